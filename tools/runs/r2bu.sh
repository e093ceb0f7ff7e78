mkdir -p gpurun_out
for cfg in "1 0" "1 1" "1 2" "1 3" "0 0"; do set -- $cfg; BMM_COLSQ_WIDE=$1 BMM_COLSQ_WIDE_CFG=$2 timeout 300 python tools/cfg4_norms_hot_probe.py 2>&1 | tail -1; done | tee gpurun_out/bu_norms_hot.txt
