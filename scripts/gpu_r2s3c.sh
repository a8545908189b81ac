O=gpurun_out/r2s3c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_path.py -q -x -m gpu > $O/pytest.txt 2>&1
for B in 1 16; do timeout 300 python scripts/stage_flags.py hyb 4 $B 7 > $O/flags_hyb4_b${B}_impl7.txt 2>&1; done
timeout 300 python scripts/stage_flags.py hyb 4 16 0 > $O/flags_hyb4_b16.txt 2>&1
timeout 300 python scripts/stage_flags.py 3inst 2 16 7 > $O/flags_3inst_b16_impl7.txt 2>&1
timeout 300 python scripts/stage_flags.py 3inst 2 16 0 > $O/flags_3inst_b16.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --steps 10 > $O/hyb4_auto.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --steps 10 --matvec-impl 6 > $O/hyb4_impl6.json 2>&1
