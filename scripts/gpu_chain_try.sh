set -x
O=gpurun_out/${1:-chain1}
mkdir -p $O
timeout 300 python scripts/xform_bench.py > $O/xform.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_chain.py -q -x > $O/t2.txt 2>&1
timeout 300 python scripts/chain_trace.py 3inst 2 4 1 > $O/trace_3inst_y1.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-70b --steps 5 > $O/bench.json 2> $O/bench.err
