mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -x -q > gpurun_out/al_test.log 2>&1; echo "test rc=$?"; tail -3 gpurun_out/al_test.log
