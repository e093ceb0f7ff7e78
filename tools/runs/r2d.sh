mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/d_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/d_bench_cfg4.json 2> gpurun_out/d_bench_cfg4.err; echo "bench rc=$?"
for w in cfg2 cfg3 cfg5; do
timeout 900 python bench.py --workload $w > gpurun_out/d_bench_$w.json 2> gpurun_out/d_bench_$w.err; echo "bench $w rc=$?"
done
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -o /tmp/d_cfg4 python tools/profile_cfg4.py > gpurun_out/d_ncu_cfg4.log 2>&1; echo "ncu rc=$?"
python tools/summarize_ncu.py full /tmp/d_cfg4.ncu-rep gpurun_out/d_ncu_cfg4_summary.csv > /dev/null 2>&1
ncu -i /tmp/d_cfg4.ncu-rep --page raw --csv > gpurun_out/d_ncu_cfg4_raw.csv 2>/dev/null; echo "raw rc=$?"
ls -la /tmp/d_cfg4.ncu-rep
