mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_segsq_i8.py -x -q 2>&1 | tail -3
timeout 200 python tools/segsq_i8_bench.py 2>&1 | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"oz_" -c 40 --csv python tools/segsq_i8_bench.py 2>&1 | grep -E "oz_" | awk -F'","' '{print substr($5,1,28), $NF}'
