mkdir -p gpurun_out
for g in 8 4 16 32 2; do BMM_F16_GROUP_M=$g timeout 300 python tools/cfg4_gemm_sweep.py 2>&1 | tail -1; done | tee gpurun_out/bi_gemm_sweep.txt
BMM_F16_CHUNK=4 timeout 300 python tools/cfg4_gemm_sweep.py 2>&1 | tail -1 | tee -a gpurun_out/bi_gemm_sweep.txt
