O=gpurun_out/r2s3s
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bench_path.py -q -x -m gpu -k "slab" > $O/pytest_slab.txt 2>&1
