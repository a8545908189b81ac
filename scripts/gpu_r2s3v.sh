O=gpurun_out/r2s3v
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_path.py -q -x -m gpu -k "umma or impl7 or 7 or bench or slab" > $O/pytest.txt 2>&1
timeout 120 python scripts/umma_trace.py hyb 4 12288 4096 1 > $O/trace_hyb4_b1.txt 2>&1
timeout 300 python scripts/stage_flags.py hyb 4 1 0 > $O/flags_hyb4_b1.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --steps 10 > $O/hyb4.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --steps 10 > $O/3inst.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch 16 --steps 10 > $O/hyb4_b16.json 2>&1
