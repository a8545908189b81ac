O=gpurun_out/r2s3z
mkdir -p $O
for B in 1 16; do timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma -s 20 -c 1 -o $O/umma_big_b$B python scripts/stage_flags.py hyb 4 $B 7 big > $O/ncu_b$B.log 2>&1; done
