mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -m gpu -k "waves or many_small or cfg5" > gpurun_out/au_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/au_pytest.log
timeout 900 python bench.py --workload cfg5 > gpurun_out/au_bench_cfg5.json 2> gpurun_out/au_bench_cfg5.err; echo "bench rc=$?"
BMM_CFG5_WAVES=0 timeout 900 python bench.py --workload cfg5 > gpurun_out/au_bench_cfg5_nowaves.json 2> gpurun_out/au_bench_cfg5_nowaves.err; echo "bench rc=$?"
BMM_CFG5_WAVES=512,4 timeout 900 python bench.py --workload cfg5 > gpurun_out/au_bench_cfg5_512x4.json 2> gpurun_out/au_bench_cfg5_512x4.err; echo "bench rc=$?"
BMM_CFG5_WAVES=1024,3 timeout 900 python bench.py --workload cfg5 > gpurun_out/au_bench_cfg5_1024x3.json 2> gpurun_out/au_bench_cfg5_1024x3.err; echo "bench rc=$?"
grep -o '"value": [0-9.]*' gpurun_out/au_bench_cfg5*.json
