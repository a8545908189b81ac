O=gpurun_out/r2s3l
mkdir -p $O
timeout 300 python scripts/stage_flags.py 3inst 2 1 7 > $O/flags_3inst_b1_impl7.txt 2>&1
timeout 300 python scripts/stage_flags.py 3inst 2 16 7 > $O/flags_3inst_b16_impl7.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --steps 10 > $O/3inst_auto.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --steps 10 --matvec-impl 7 > $O/3inst_impl7.json 2>&1
for B in 1 2 4 8 16; do timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch $B --steps 10 > $O/c3_hyb4_b$B.json 2> $O/c3_hyb4_b$B.err; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_path.py -q -x -m gpu > $O/pytest.txt 2>&1
