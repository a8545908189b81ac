O=gpurun_out/r2s3w
mkdir -p $O
timeout 300 python scripts/stage_flags.py 3inst 2 1 7 > $O/flags_3inst_b1_impl7.txt 2>&1
timeout 300 python scripts/stage_flags.py hyb 4 1 7 o > $O/flags_hyb4_b1_impl7_o.txt 2>&1
timeout 300 python scripts/stage_flags.py 1mad 2 1 7 > $O/flags_1mad_b1_impl7.txt 2>&1
timeout 300 python scripts/stage_flags.py 1mad 2 1 0 > $O/flags_1mad_b1_impl0.txt 2>&1
