mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_cfg5.py tests/test_gpu_parity.py tests/test_gpu_random.py -x -q > gpurun_out/o_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python tools/stage_breakdown.py cfg5 > gpurun_out/o_stages_cfg5.txt 2>&1
timeout 900 python bench.py --workload cfg5 > gpurun_out/o_bench_cfg5.json 2> gpurun_out/o_bench_cfg5.err; echo "bench rc=$?"
