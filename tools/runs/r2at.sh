mkdir -p gpurun_out
timeout 900 python tools/cfg5_waves_probe.py 4096,1 2048,2 1024,2 1024,4 512,2 512,4 > gpurun_out/at_waves.txt 2>&1; echo "waves rc=$?"
tail -8 gpurun_out/at_waves.txt
