O=gpurun_out/r2s3t
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "rht or matvec_small" > $O/pytest_rht.txt 2>&1
timeout 200 python scripts/rht_bench.py > $O/rht_bench.txt 2>&1
timeout 300 python scripts/stage_flags.py hyb 4 16 0 > $O/flags_hyb4_b16.txt 2>&1
for B in 8 16; do timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch $B --steps 10 > $O/c3_hyb4_b$B.json 2> $O/c3_hyb4_b$B.err; done
timeout 400 python bench.py --no-cpu-baseline --no-70b --batch 16 --steps 10 > $O/c1_3inst_b16.json 2> $O/c1_3inst_b16.err
