# Round-2 final measurement pass (session 3): GPU suite, smoke, bench lines of every config, ncu launch
# list + --set full of the step's GEMV kernels, sanitizers on the changed kernels.  Output in
# gpurun_out/<tag>/.
set -x
O=gpurun_out/${1:-r2g}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for B in 1 2 4 8 16; do timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch $B --steps 10 > $O/c3_hyb4_b$B.json 2> $O/c3_hyb4_b$B.err; done
for B in 4 16; do timeout 400 python bench.py --no-cpu-baseline --no-70b --batch $B --steps 10 > $O/c1_3inst_b$B.json 2> $O/c1_3inst_b$B.err; done
timeout 400 python bench.py --no-cpu-baseline --no-70b --code 1mad --k 2 --steps 10 > $O/c2_1mad.json 2> $O/c2_1mad.err
timeout 600 python bench.py --no-cpu-baseline --no-70b --workload c4-70b --steps 10 > $O/c4_70b_1gpu.json 2> $O/c4_70b_1gpu.err
timeout 900 python bench.py --no-cpu-baseline --no-70b --workload llama2-70b --steps 3 --warmup 3 > $O/c5_70b_hyb3_1gpu.json 2> $O/c5_70b_hyb3_1gpu.err
timeout 300 python scripts/rht_bench.py > $O/rht_bench.txt 2>&1
for B in 1 16; do timeout 300 python scripts/stage_flags.py hyb 4 $B 0 > $O/flags_hyb4_b$B.txt 2>&1; timeout 300 python scripts/stage_flags.py 3inst 2 $B 0 > $O/flags_3inst_b$B.txt 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-70b > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemv|layer_kernel|umma" -s 700 -c 4 -o $O/prof_gemv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-70b > $O/prof_gemv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"umma" -s 40 -c 2 -o $O/prof_umma_hyb4 python bench.py --code hyb --k 4 --steps 1 --warmup 3 --no-cpu-baseline --no-70b > $O/prof_umma.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv >> $O/gpu.txt 2>&1
