mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --workload cfg4 > gpurun_out/a_bench_cfg4.json 2> gpurun_out/a_bench_cfg4.err; echo "bench cfg4 rc=$?"
