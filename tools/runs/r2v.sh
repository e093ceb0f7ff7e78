mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/v_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?"
for w in cfg2 cfg3 cfg1 cfg5; do
timeout 900 python bench.py --workload $w > gpurun_out/v_bench_$w.json 2> gpurun_out/v_bench_$w.err; echo "bench $w rc=$?"
done
