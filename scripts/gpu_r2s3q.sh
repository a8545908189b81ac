O=gpurun_out/r2s3q
mkdir -p $O
timeout 300 python scripts/stage_flags.py 3inst 2 1 0 > $O/flags_3inst_b1_impl0.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --steps 10 > $O/3inst_auto.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --steps 10 --code 1mad > $O/1mad_auto.json 2>&1
