mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_analytics.py -x -q -m gpu > gpurun_out/bb_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/bb_pytest.log
timeout 900 python bench.py --workload mc > gpurun_out/bb_bench_mc.json 2> gpurun_out/bb_bench_mc.err; echo "bench rc=$?"
grep -o '"value": [0-9.]*, "unit": "[^"]*", "n_gpus"' gpurun_out/bb_bench_mc.json; tail -3 gpurun_out/bb_bench_mc.err
