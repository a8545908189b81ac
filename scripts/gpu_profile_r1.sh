set -x
timeout 600 python bench.py > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r1e.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_r1e.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv -s 700 -c 7 -o gpurun_out/prof_gemv_r1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_gemv_r1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rht|reduce" -s 700 -c 6 -o gpurun_out/prof_rht_r1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_rht_r1.log 2>&1
python scripts/ncu_traffic.py gpurun_out/prof_gemv_r1.ncu-rep llama2-7b/3inst/k2 gpurun_out/traffic.json > gpurun_out/traffic_gemv.txt 2>&1
python scripts/ncu_traffic.py gpurun_out/prof_rht_r1.ncu-rep llama2-7b/3inst/k2 gpurun_out/traffic_rht.json > gpurun_out/traffic_rht.txt 2>&1
