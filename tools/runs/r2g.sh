mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_norms_wide.py tests/test_gpu_pipeline.py -x -q > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?"
for c in 0 1 2 3; do BMM_PROBE_ONLY=colsq BMM_COLSQ_WIDE_CFG=$c timeout 300 python tools/cfg4_norms_probe.py >> gpurun_out/g_norms.txt 2>&1; done
for c in 0 1 2; do BMM_PROBE_ONLY=rowsq BMM_ROWSQ_TMA_CFG=$c timeout 300 python tools/cfg4_norms_probe.py >> gpurun_out/g_norms.txt 2>&1; done
timeout 300 python tools/cfg4_norms_probe.py >> gpurun_out/g_norms.txt 2>&1
timeout 300 python tools/norms_sweep.py > gpurun_out/g_norms_sweep.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_cfg4.py -x -q > gpurun_out/g_cfg4.log 2>&1; echo "cfg4 full rc=$?"
