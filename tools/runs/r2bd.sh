mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/bd_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/bd_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bd_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/bd_smoke.log
for w in cfg2 cfg3 cfg1; do
timeout 900 python bench.py --workload $w > gpurun_out/bd_bench_$w.json 2> gpurun_out/bd_bench_$w.err; echo "bench $w rc=$?"
done
