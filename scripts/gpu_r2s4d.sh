O=gpurun_out/r2s4d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ldlq.py -q -m gpu > $O/pytest_ldlq.txt 2>&1
