O=gpurun_out/r2s4e
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_path.py -q -x -m gpu -k "umma or impl7 or 7 or bench or slab or grouped or deterministic" > $O/pytest.txt 2>&1
for B in 1 16; do timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch $B --steps 10 > $O/c3_hyb4_b$B.json 2> $O/c3_hyb4_b$B.err; done
timeout 400 python bench.py --no-cpu-baseline --no-70b --steps 10 > $O/c1_3inst_b1.json 2> $O/c1_3inst_b1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"umma" -s 40 -c 1 -o $O/prof_umma_hyb4 python bench.py --code hyb --k 4 --steps 1 --warmup 3 --no-cpu-baseline --no-70b > $O/prof_umma.log 2>&1
