O=gpurun_out/r2s3b
mkdir -p $O
for B in 1 8 16; do timeout 300 python scripts/stage_flags.py hyb 4 $B 0 > $O/flags_hyb4_b$B.txt 2>&1; done
timeout 300 python scripts/stage_flags.py hyb 4 1 6 qkv,gateup > $O/flags_hyb4_b1_impl6.txt 2>&1
timeout 300 python scripts/stage_flags.py hyb 4 16 7 > $O/flags_hyb4_b16_impl7.txt 2>&1
timeout 300 python scripts/stage_flags.py 3inst 2 16 0 > $O/flags_3inst_b16.txt 2>&1
timeout 300 python scripts/stage_flags.py 3inst 2 1 0 > $O/flags_3inst_b1.txt 2>&1
