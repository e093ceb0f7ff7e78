mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/i_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python tools/cfg4_norms_probe.py > gpurun_out/i_norms.txt 2>&1
timeout 300 python tools/timeline.py 5 > gpurun_out/i_timeline_cfg2.txt 2>&1; echo "timeline rc=$?"
for w in cfg2 cfg5; do
timeout 900 python bench.py --workload $w > gpurun_out/i_bench_$w.json 2> gpurun_out/i_bench_$w.err; echo "bench $w rc=$?"
done
timeout 1200 python bench.py > gpurun_out/i_bench_cfg4.json 2> gpurun_out/i_bench_cfg4.err; echo "bench rc=$?"
