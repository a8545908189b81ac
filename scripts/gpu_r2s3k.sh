O=gpurun_out/r2s3k
mkdir -p $O
for B in 1 16; do for I in 0 3 7; do timeout 300 python scripts/stage_flags.py hyb 4 $B $I > $O/flags_hyb4_b${B}_impl$I.txt 2>&1; done; done
for B in 1 16; do for I in 0 7; do timeout 300 python scripts/stage_flags.py 3inst 2 $B $I > $O/flags_3inst_b${B}_impl$I.txt 2>&1; done; done
timeout 300 python scripts/stage_flags.py 3inst 2 1 6 > $O/flags_3inst_b1_impl6.txt 2>&1
timeout 300 python scripts/stage_flags.py hyb 4 4 0 > $O/flags_hyb4_b4_impl0.txt 2>&1
timeout 300 python scripts/stage_flags.py hyb 4 4 7 > $O/flags_hyb4_b4_impl7.txt 2>&1
