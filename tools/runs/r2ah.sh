mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_f16split_gather -c 1 -o gpurun_out/ah_fused python tools/cfg5_waves_probe.py 4096,1 > gpurun_out/ah_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ah_ncu.log
