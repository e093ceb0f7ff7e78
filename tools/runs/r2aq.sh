mkdir -p gpurun_out
BMM_GRAM_NORMS_SIDES=3 timeout 600 python tools/gram_norms_probe.py > gpurun_out/aq_probe3.txt 2>&1
BMM_GRAM_NORMS_SIDES=1 timeout 600 python tools/gram_norms_probe.py > gpurun_out/aq_probe1.txt 2>&1
tail -3 gpurun_out/aq_probe3.txt gpurun_out/aq_probe1.txt
