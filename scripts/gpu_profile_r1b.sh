# Round-1 (second session) measurement pass, run on the GPU box from the repo root: bench lines of
# the default and other configs, the ncu launch list of the bench command, ncu --set full of the
# step's GEMV launches, microbenchmarks, steady-state GEMV rates, phase traces, quantizer timing.
# Everything lands in gpurun_out/<tag>/ (bash scripts/gpu_profile_r1b.sh <tag>, default r1b);
# python scripts/summarize_r1b.py <tag> copies the summaries to profiles/<tag>_*.
set -x
O=gpurun_out/${1:-r1b}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for B in 1 2 4 8 16; do timeout 400 python bench.py --no-cpu-baseline --code hyb --k 4 --batch $B --steps 10 > $O/c3_hyb4_b$B.json 2> $O/c3_hyb4_b$B.err; done
timeout 400 python bench.py --no-cpu-baseline --code 1mad --k 2 --steps 10 > $O/c2_1mad.json 2> $O/c2_1mad.err
timeout 600 python bench.py --no-cpu-baseline --workload c4-70b --steps 10 > $O/c4_70b_1gpu.json 2> $O/c4_70b_1gpu.err
timeout 900 python bench.py --no-cpu-baseline --workload llama2-70b --steps 3 --warmup 3 > $O/c5_70b_hyb3_1gpu.json 2> $O/c5_70b_hyb3_1gpu.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemv|layer_kernel" -s 700 -c 4 -o $O/prof_gemv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/prof_gemv.log 2>&1
timeout 120 ./scripts/pipe_mix_microbench > $O/pipe_mix.txt 2>&1
timeout 120 ./scripts/decode_microbench > $O/decode_microbench.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:loop -c 1 -o $O/prof_decode_loop ./scripts/decode_microbench > $O/prof_decode_loop.log 2>&1
timeout 120 ./scripts/gridbar_microbench > $O/gridbar.txt 2>&1
for i in 3 4 6; do timeout 200 python scripts/gemv_rate.py $i 3inst 2 >> $O/gemv_rate.txt 2>&1; timeout 200 python scripts/gemv_rate.py $i hyb 4 >> $O/gemv_rate.txt 2>&1; done
timeout 300 ncu --set full --clock-control none -k regex:layer_kernel -s 3 -c 1 -o $O/prof_gemv6 python scripts/gemv_rate.py 6 3inst 2 37888 4096 1 18944 > $O/prof_gemv6.log 2>&1
for s in "4096 4096" "11008 4096" "4096 11008"; do timeout 120 python scripts/trace_fused.py $s 3inst 2 3 1 0 1 5 >> $O/trace_fused_impl5.txt 2>&1; timeout 120 python scripts/trace_fused.py $s 3inst 2 3 1 0 1 6 >> $O/trace_fused_impl6.txt 2>&1; done
OMP_NUM_THREADS=1 timeout 300 python scripts/viterbi_bench.py 3inst 2 4096 256 > $O/viterbi.txt 2>&1
OMP_NUM_THREADS=1 timeout 300 python scripts/viterbi_bench.py 3inst 3 2048 256 >> $O/viterbi.txt 2>&1
OMP_NUM_THREADS=1 timeout 300 python scripts/viterbi_bench.py 1mad 2 2048 256 >> $O/viterbi.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
