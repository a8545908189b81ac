O=gpurun_out/r2s3e
mkdir -p $O
timeout 200 python scripts/rht_bench.py > $O/rht_bench.txt 2>&1
for B in 1 16; do timeout 120 python scripts/umma_trace.py hyb 4 12288 4096 $B > $O/trace_new_hyb4_b$B.txt 2>&1; done
timeout 300 python scripts/stage_flags.py hyb 4 16 7 > $O/flags_new_hyb4_b16_impl7.txt 2>&1
cp paper_2406_11235_b200/libqtip.so /tmp/libqtip_new.so
cp scripts/libqtip_old.so paper_2406_11235_b200/libqtip.so
for B in 1 16; do timeout 120 python scripts/umma_trace.py hyb 4 12288 4096 $B > $O/trace_old_hyb4_b$B.txt 2>&1; done
timeout 300 python scripts/stage_flags.py hyb 4 1 7 > $O/flags_old_hyb4_b1_impl7.txt 2>&1
cp /tmp/libqtip_new.so paper_2406_11235_b200/libqtip.so
