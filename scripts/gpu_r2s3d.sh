O=gpurun_out/r2s3d
mkdir -p $O
timeout 300 python scripts/stage_flags.py hyb 4 1 7 > $O/flags_hyb4_b1_impl7.txt 2>&1
for B in 1 4 16; do timeout 120 python scripts/umma_trace.py hyb 4 12288 4096 $B > $O/trace_hyb4_12288_b$B.txt 2>&1; done
timeout 120 python scripts/umma_trace.py 3inst 2 12288 4096 16 > $O/trace_3inst_12288_b16.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --steps 10 > $O/hyb4_auto.json 2>&1
