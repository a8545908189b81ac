# Round-2 baseline pass (run on the GPU box from the repo root): GPU suite, smoke, default bench,
# C3 HYB k=4 batch sweep, 1MAD, C4/C5 on one GPU, impl-7 probe.  Output in gpurun_out/<tag>/.
set -x
O=gpurun_out/${1:-r2a}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
for B in 1 2 4 8 16; do timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch $B --steps 10 > $O/c3_hyb4_b$B.json 2> $O/c3_hyb4_b$B.err; done
timeout 400 python bench.py --no-cpu-baseline --no-70b --code 1mad --k 2 --steps 10 > $O/c2_1mad.json 2> $O/c2_1mad.err
timeout 900 python bench.py --no-cpu-baseline --no-70b --workload llama2-70b --steps 3 --warmup 3 > $O/c5_70b_hyb3_1gpu.json 2> $O/c5_70b_hyb3_1gpu.err
timeout 300 python scripts/umma_probe.py time > $O/umma_probe.txt 2>&1
