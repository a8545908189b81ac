O=gpurun_out/r2s3r
mkdir -p $O
for PF in 0 64; do
QTIP_L2_PREFETCH=$PF timeout 300 python scripts/stage_flags.py 3inst 2 1 0 > $O/flags_3inst_b1_pf$PF.txt 2>&1
QTIP_L2_PREFETCH=$PF timeout 300 python scripts/stage_flags.py hyb 4 1 0 > $O/flags_hyb4_b1_pf$PF.txt 2>&1
QTIP_L2_PREFETCH=$PF timeout 300 python bench.py --no-cpu-baseline --no-70b --steps 10 > $O/3inst_pf$PF.json 2>&1
QTIP_L2_PREFETCH=$PF timeout 300 python bench.py --no-cpu-baseline --no-70b --code hyb --k 4 --steps 10 > $O/hyb4_pf$PF.json 2>&1
done
QTIP_L2_PREFETCH=16 timeout 300 python bench.py --no-cpu-baseline --no-70b --steps 10 > $O/3inst_pf16.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_path.py tests/test_gpu_ldlq.py -q -x -m gpu > $O/pytest.txt 2>&1
