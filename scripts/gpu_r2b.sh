# chain-kernel bench pass: default bench, HYB k=4 batch sweep, 1MAD, C5 70B stack, C4.
set -x
O=gpurun_out/${1:-r2b}
mkdir -p $O
timeout 300 python bench.py --no-cpu-baseline --no-70b --blocks 2 --steps 2 > gpurun_out/${1:-r2b}/quick.json 2> gpurun_out/${1:-r2b}/quick.err


timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
for B in 1 4 16; do timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch $B --steps 10 > $O/c3_hyb4_b$B.json 2> $O/c3_hyb4_b$B.err; done
timeout 900 python bench.py --no-cpu-baseline --no-70b --workload llama2-70b --steps 3 --warmup 3 > $O/c5_70b_hyb3_1gpu.json 2> $O/c5_70b_hyb3_1gpu.err
timeout 600 python bench.py --no-cpu-baseline --no-70b --workload c4-70b --steps 10 > $O/c4_70b.json 2> $O/c4_70b.err
