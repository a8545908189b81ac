O=gpurun_out/r2s3x
mkdir -p $O
for C in 0 73 147; do for B in 1 16; do TRACE_CTA=$C timeout 120 python scripts/umma_trace.py hyb 4 12288 4096 $B > $O/trace_hyb4_b${B}_cta$C.txt 2>&1; done; done
