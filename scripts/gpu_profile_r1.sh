# Round-1 profiling pass (run on the GPU box from the repo root): bench line, ncu launch list of
# the same command, ncu --set full of one block's GEMV launches and of the RHT kernels, summaries.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_r1f.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_r1f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv -s 700 -c 7 -o gpurun_out/prof_gemv_r1f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_gemv_r1f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rht|reduce" -s 700 -c 8 -o gpurun_out/prof_rht_r1f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_rht_r1f.log 2>&1
python scripts/ncu_traffic.py gpurun_out/prof_gemv_r1f.ncu-rep llama2-7b/3inst/k2 gpurun_out/traffic.json > gpurun_out/traffic_gemv_r1f.txt 2>&1
python scripts/ncu_traffic.py gpurun_out/prof_rht_r1f.ncu-rep llama2-7b/3inst/k2 gpurun_out/traffic_rht.json > gpurun_out/traffic_rht_r1f.txt 2>&1
