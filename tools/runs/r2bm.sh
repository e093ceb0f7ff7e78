mkdir -p gpurun_out
for cfg in "4 4" "4 8" "4 4" "4 8"; do set -- $cfg; BMM_F16_GROUP_M=$1 BMM_F16_CHUNK=$2 timeout 300 python tools/cfg4_gemm_sweep.py 2>&1 | tail -1; done | tee gpurun_out/bm_gemm_sweep.txt
