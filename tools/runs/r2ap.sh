mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram_blocks.py tests/test_gpu_pipeline.py -x -q > gpurun_out/ap_test.log 2>&1; echo "test rc=$?"; tail -15 gpurun_out/ap_test.log
timeout 600 python tools/timeline.py 3 cfg4 > gpurun_out/ap_tl4.txt 2>&1; tail -5 gpurun_out/ap_tl4.txt
