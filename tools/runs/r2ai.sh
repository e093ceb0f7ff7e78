mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tf32.py -x -q -k fused_gather > gpurun_out/ai_test.log 2>&1; echo "test rc=$?"
tail -15 gpurun_out/ai_test.log
timeout 600 python tools/cfg5_waves_probe.py 4096,1 > gpurun_out/ai_fused.txt 2>&1
cat gpurun_out/ai_fused.txt | tail -3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_f16split_gather -c 1 -o gpurun_out/ai_fused python tools/cfg5_waves_probe.py 4096,1 > gpurun_out/ai_ncu.log 2>&1; echo "ncu rc=$?"
