# Build the tcgen05 GEMV (impl 2) ablation variants (k_gemv_tc.cu QTIP_TC_* switches) as separate
# libraries here, then on the GPU box run scripts/gemv_rate.py against each (QTIP_LIB=...):
#   bash scripts/tc_ablation.sh build      (CPU container)
#   bash scripts/tc_ablation.sh run        (GPU box) -> gpurun_out/tc_ablation.txt
set -e
V="base:-DQTIP_TC_PIPE=0 pipe:-DQTIP_TC_PIPE=1,-DQTIP_TC_EPI_H=1 nodec_nomma:-DQTIP_TC_PIPE=1,-DQTIP_TC_EPI_H=1,-DQTIP_TC_NODECODE=1,-DQTIP_TC_NOMMA=1 nodec_nomma_nost:-DQTIP_TC_PIPE=1,-DQTIP_TC_EPI_H=1,-DQTIP_TC_NODECODE=1,-DQTIP_TC_NOMMA=1,-DQTIP_TC_NOST=1 nodec_nomma_nosync:-DQTIP_TC_PIPE=1,-DQTIP_TC_EPI_H=1,-DQTIP_TC_NODECODE=1,-DQTIP_TC_NOMMA=1,-DQTIP_TC_NOSYNC=1 skeleton:-DQTIP_TC_PIPE=1,-DQTIP_TC_EPI_H=1,-DQTIP_TC_NODECODE=1,-DQTIP_TC_NOMMA=1,-DQTIP_TC_NOSYNC=1,-DQTIP_TC_NOST=1 decode_only:-DQTIP_TC_PIPE=1,-DQTIP_TC_EPI_H=1,-DQTIP_TC_NOMMA=1,-DQTIP_TC_NOSYNC=1,-DQTIP_TC_NOST=1"
if [ "$1" = build ]; then
  for v in $V; do n=${v%%:*}; f=${v#*:}; python - "$n" ${f//,/ } <<'PY'
import os, sys
sys.path.insert(0, '.')
from paper_2406_11235_b200 import build as b
n, fl = sys.argv[1], sys.argv[2:]
b.BUILD = '/tmp/tc_ablation/' + n
os.makedirs(b.BUILD, exist_ok=True)
b.LIB = os.path.abspath('paper_2406_11235_b200/libqtip_abl_%s.so' % n)
b.FLAGS = b.FLAGS + fl
b.build()
PY
  done
else
  mkdir -p gpurun_out
  for v in $V; do n=${v%%:*}
    QTIP_LIB=$PWD/paper_2406_11235_b200/libqtip_abl_$n.so timeout 100 python scripts/gemv_rate.py 2 3inst 2 | sed "s/^/$n: /"
  done > gpurun_out/tc_ablation.txt 2>&1
fi
