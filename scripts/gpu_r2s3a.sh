# session-3 probe: MMA rate (A in TMEM vs smem, N), decode loops, a fresh default bench and stage breakdown
O=gpurun_out/r2s3a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 120 ./scripts/umma_rate > $O/umma_rate.txt 2>&1
timeout 120 ./scripts/decode_microbench > $O/decode_microbench.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-70b --steps 10 > $O/bench.json 2> $O/bench.err
timeout 300 python scripts/stage_breakdown.py 3inst 2 1 > $O/stage_3inst.txt 2>&1
timeout 300 python scripts/stage_breakdown.py hyb 4 1 > $O/stage_hyb4.txt 2>&1
