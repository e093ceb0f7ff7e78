mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tf32.py -x -q -k fused_gather > gpurun_out/aj_test.log 2>&1; echo "test rc=$?"; tail -2 gpurun_out/aj_test.log
timeout 900 python -m pytest tests/test_gpu_cfg5.py tests/test_gpu_pipeline.py -x -q > gpurun_out/aj_test5.log 2>&1; echo "cfg5 tests rc=$?"; tail -2 gpurun_out/aj_test5.log
timeout 600 python tools/cfg5_waves_probe.py 4096,1 > gpurun_out/aj_fused.txt 2>&1; tail -1 gpurun_out/aj_fused.txt
timeout 900 python bench.py --workload cfg5 > gpurun_out/aj_cfg5.json 2> gpurun_out/aj_cfg5.err; echo "bench rc=$?"; tail -2 gpurun_out/aj_cfg5.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_f16split_gather -c 1 -o gpurun_out/aj_fused python tools/cfg5_waves_probe.py 4096,1 > gpurun_out/aj_ncu.log 2>&1; echo "ncu rc=$?"
