set -x
O=gpurun_out/${1:-chain1}
mkdir -p $O
for B in 16 32 64; do
  for impl in 0 7; do
    timeout 400 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --batch $B --steps 5 --matvec-impl $impl > $O/hyb4_b${B}_impl$impl.json 2> $O/hyb4_b${B}_impl$impl.err
  done
done
for B in 8 16 32; do
  for impl in 0 7; do
    timeout 400 python bench.py --no-cpu-baseline --no-70b --code 3inst --k 2 --batch $B --steps 5 --matvec-impl $impl > $O/3inst_b${B}_impl$impl.json 2> $O/3inst_b${B}_impl$impl.err
  done
done
