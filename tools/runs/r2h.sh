mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/h_bench_cfg4.json 2> gpurun_out/h_bench_cfg4.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/h_bench_ref.json 2> gpurun_out/h_bench_ref.err; echo "ref rc=$?"
for w in cfg2 cfg3 cfg5 cfg1; do
timeout 900 python bench.py --workload $w > gpurun_out/h_bench_$w.json 2> gpurun_out/h_bench_$w.err; echo "bench $w rc=$?"
done
timeout 300 python tools/timeline.py 5 > gpurun_out/h_timeline_cfg2.txt 2>&1; echo "timeline rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -o /tmp/h_cfg4 python tools/profile_cfg4.py > gpurun_out/h_ncu_cfg4.log 2>&1; echo "ncu rc=$?"
python tools/summarize_ncu.py full /tmp/h_cfg4.ncu-rep gpurun_out/h_ncu_cfg4_summary.csv > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/h_launches_cfg4.csv python bench.py --steps 1 --warmup 1 > gpurun_out/h_ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/summarize_ncu.py launches gpurun_out/h_launches_cfg4.csv gpurun_out/h_launches_cfg4_summary.csv > /dev/null 2>&1
