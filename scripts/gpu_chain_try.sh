set -x
O=gpurun_out/${1:-chain1}
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chain_kernel -s 3 -c 1 -o $O/chain_prof python scripts/chain_trace.py 3inst 2 4 1 > $O/ncu.log 2>&1
