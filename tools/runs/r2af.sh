mkdir -p gpurun_out
timeout 900 python tools/cfg5_waves_probe.py > gpurun_out/af_waves.txt 2>&1; echo "waves rc=$?"
