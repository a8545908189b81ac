O=gpurun_out/r2s4a
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_path.py -q -x -m gpu -k "umma or impl7 or 7 or bench or slab or grouped or deterministic" > $O/pytest.txt 2>&1
timeout 300 python scripts/stage_flags.py hyb 4 16 0 > $O/flags_hyb4_b16.txt 2>&1
timeout 300 python scripts/stage_flags.py 3inst 2 16 0 > $O/flags_3inst_b16.txt 2>&1
for B in 1 4 8 16; do timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch $B --steps 10 > $O/c3_hyb4_b$B.json 2> $O/c3_hyb4_b$B.err; done
for B in 1 16; do timeout 400 python bench.py --no-cpu-baseline --no-70b --batch $B --steps 10 > $O/c1_3inst_b$B.json 2> $O/c1_3inst_b$B.err; done
