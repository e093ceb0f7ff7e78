mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tf32.py -x -q -k fused_gather > gpurun_out/ag_test.log 2>&1; echo "test rc=$?"
tail -5 gpurun_out/ag_test.log
timeout 600 python bench.py --workload cfg5 > gpurun_out/ag_cfg5.json 2> gpurun_out/ag_cfg5.err; echo "bench rc=$?"
tail -3 gpurun_out/ag_cfg5.err
BMM_F16_FUSED=0 timeout 600 python tools/cfg5_waves_probe.py 4096,1 > gpurun_out/ag_unfused.txt 2>&1
timeout 600 python tools/cfg5_waves_probe.py 4096,1 > gpurun_out/ag_fused.txt 2>&1
cat gpurun_out/ag_unfused.txt gpurun_out/ag_fused.txt
