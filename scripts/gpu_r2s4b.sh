O=gpurun_out/r2s4b
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_path.py -q -x -m gpu -k "umma or impl7 or 7 or bench or slab or grouped or deterministic" > $O/pytest.txt 2>&1
for B in 1 16; do timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch $B --steps 10 > $O/c3_hyb4_b$B.json 2> $O/c3_hyb4_b$B.err; done
timeout 400 python bench.py --no-cpu-baseline --no-70b --steps 10 > $O/c1_3inst_b1.json 2> $O/c1_3inst_b1.err
timeout 120 python scripts/umma_trace.py hyb 4 12288 4096 1 > $O/trace_hyb4_b1.txt 2>&1
