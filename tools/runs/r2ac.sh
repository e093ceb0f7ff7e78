mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/ac_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ac_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/ac_bench_cfg4.json 2> gpurun_out/ac_bench_cfg4.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ac_bench_ref.json 2> gpurun_out/ac_bench_ref.err; echo "ref rc=$?"
for w in cfg2 cfg3 cfg1 cfg5 mc; do
timeout 900 python bench.py --workload $w > gpurun_out/ac_bench_$w.json 2> gpurun_out/ac_bench_$w.err; echo "bench $w rc=$?"
done
timeout 300 python tools/timeline.py 5 > gpurun_out/ac_timeline_cfg2.txt 2>&1
