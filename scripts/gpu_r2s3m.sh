O=gpurun_out/r2s3m
mkdir -p $O
timeout 200 python scripts/rht_bench.py > $O/rht_bench.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --steps 10 > $O/3inst_auto.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch 16 --steps 10 > $O/c3_hyb4_b16.json 2> $O/c3_hyb4_b16.err
timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch 8 --steps 10 > $O/c3_hyb4_b8.json 2> $O/c3_hyb4_b8.err
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "rht" > $O/pytest_rht.txt 2>&1
