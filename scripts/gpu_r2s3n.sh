O=gpurun_out/r2s3n
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rht_kernel --launch-skip 3 -c 1 -o $O/rht11008_b16 python scripts/rht_bench.py 16 11008 > $O/ncu_rht.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_gemv --launch-skip 40 -c 2 -o $O/umma_hyb4 python bench.py --code hyb --k 4 --steps 1 --warmup 3 --no-cpu-baseline --no-70b > $O/ncu_umma.log 2>&1
