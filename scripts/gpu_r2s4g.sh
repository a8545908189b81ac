O=gpurun_out/r2s4g
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_path.py tests/test_gpu_ldlq.py -q -x -m gpu > $O/pytest.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
