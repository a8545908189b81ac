set -x
O=gpurun_out/${1:-chain1}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_viterbi.py -q -x > $O/viterbi.txt 2>&1
