mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_segsq_i8.py tests/test_gpu_engines.py -x -q 2>&1 | tail -2
timeout 200 python tools/segsq_i8_bench.py 2>&1 | tail -7
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"oz_" --csv python tools/segsq_i8_bench.py > /tmp/l.csv 2>&1
python tools/summarize_ncu.py launches /tmp/l.csv /tmp/ls.csv >/dev/null 2>&1; cat /tmp/ls.csv
