O=gpurun_out/r2s3p
mkdir -p $O
timeout 120 python scripts/umma_trace.py hyb 4 12288 4096 1 > $O/trace_hyb4_b1.txt 2>&1
timeout 300 python scripts/stage_flags.py hyb 4 1 7 > $O/flags_hyb4_b1_impl7.txt 2>&1
timeout 300 python scripts/stage_flags.py 3inst 2 1 7 > $O/flags_3inst_b1_impl7.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --steps 10 > $O/hyb4_auto.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --steps 10 > $O/3inst_auto.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch 16 --steps 10 > $O/c3_hyb4_b16.json 2> $O/c3_hyb4_b16.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_path.py -q -x -m gpu -k "umma or impl7 or 7 or bench" > $O/pytest.txt 2>&1
