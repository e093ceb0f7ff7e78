mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/bl_smi.txt 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/bl_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/bl_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bl_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/bl_bench_cfg4.json 2> gpurun_out/bl_bench_cfg4.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bl_bench_ref.json 2> gpurun_out/bl_bench_ref.err; echo "ref rc=$?"
for w in cfg5 cfg2 cfg3 cfg1 mc; do
timeout 900 python bench.py --workload $w > gpurun_out/bl_bench_$w.json 2> gpurun_out/bl_bench_$w.err; echo "bench $w rc=$?"
done
timeout 300 python tools/timeline.py 5 > gpurun_out/bl_timeline_cfg2.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/bl_launches_cfg4.csv python bench.py --steps 1 --warmup 1 > gpurun_out/bl_ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/summarize_ncu.py launches gpurun_out/bl_launches_cfg4.csv gpurun_out/bl_launches_cfg4_summary.csv > /dev/null 2>&1
