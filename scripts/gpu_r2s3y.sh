O=gpurun_out/r2s3y
mkdir -p $O
for B in 1 16; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"umma|rht" -c 400 --csv --log-file $O/launches_big_b$B.csv python scripts/stage_flags.py hyb 4 $B 7 big > $O/flags_big_b$B.txt 2>&1; done
