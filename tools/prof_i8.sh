mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'oz_|segsq' --csv --log-file gpurun_out/i8_launches.csv python tools/segsq_i8_bench.py > gpurun_out/i8_ncu1.log 2>&1; echo "launch rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'oz_' -c 5 -o gpurun_out/i8_full python tools/segsq_i8_bench.py > gpurun_out/i8_ncu2.log 2>&1; echo "full rc=$?"
