mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/bc_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/bc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bc_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/bc_bench_cfg4.json 2> gpurun_out/bc_bench_cfg4.err; echo "bench rc=$?"
for w in cfg5 cfg2 cfg3 cfg1 mc; do
timeout 900 python bench.py --workload $w > gpurun_out/bc_bench_$w.json 2> gpurun_out/bc_bench_$w.err; echo "bench $w rc=$?"
done
