mkdir -p gpurun_out
BMM_F16_COLLECTOR=1 timeout 900 python -m pytest tests/test_gpu_tf32.py -x -q -m gpu > gpurun_out/bp_pytest.log 2>&1; echo "pytest (collector) rc=$?"; tail -2 gpurun_out/bp_pytest.log
for c in 0 1 0 1; do BMM_F16_COLLECTOR=$c timeout 300 python tools/cfg4_gemm_sweep.py 2>&1 | tail -1 | sed "s/^/collector=$c /"; done | tee gpurun_out/bp_collector.txt
