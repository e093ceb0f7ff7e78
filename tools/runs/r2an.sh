mkdir -p gpurun_out
timeout 600 python tools/timeline.py 3 cfg4 > gpurun_out/an_tl4_fork.txt 2>&1
BMM_GSQ_FORK=0 timeout 600 python tools/timeline.py 3 cfg4 > gpurun_out/an_tl4_nofork.txt 2>&1
tail -5 gpurun_out/an_tl4_fork.txt; tail -5 gpurun_out/an_tl4_nofork.txt
