mkdir -p gpurun_out
BMM_COLSQ_DIRECT=2 timeout 600 python -m pytest tests/test_gpu_norms_wide.py tests/test_gpu_cfg4.py -x -q -m gpu 2>&1 | tail -2
for d in 0 1 2 3; do BMM_COLSQ_DIRECT=$d timeout 300 python tools/cfg4_norms_hot_probe.py 2>&1 | tail -1 | sed "s/^/direct=$d /"; done | tee gpurun_out/bv_colsq_direct.txt
