mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -m gpu -k "plan_small or waves or many_small or cfg5" > gpurun_out/av_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/av_pytest.log
timeout 600 python tools/cfg5_stages.py > gpurun_out/av_cfg5_stages.txt 2>&1; cat gpurun_out/av_cfg5_stages.txt
timeout 900 python bench.py --workload cfg5 > gpurun_out/av_bench_cfg5.json 2> gpurun_out/av_bench_cfg5.err; echo "bench rc=$?"
BMM_CFG5_WAVES=0 timeout 900 python bench.py --workload cfg5 > gpurun_out/av_bench_cfg5_nowaves.json 2> gpurun_out/av_bench_cfg5_nowaves.err; echo "bench rc=$?"
BMM_CFG5_WAVES=512,4 timeout 900 python bench.py --workload cfg5 > gpurun_out/av_bench_cfg5_512x4.json 2> gpurun_out/av_bench_cfg5_512x4.err; echo "bench rc=$?"
BMM_CFG5_WAVES=2048,2 timeout 900 python bench.py --workload cfg5 > gpurun_out/av_bench_cfg5_2048x2.json 2> gpurun_out/av_bench_cfg5_2048x2.err; echo "bench rc=$?"
grep -o '"value": [0-9.]*, "unit": "ms/step", "n_gpus"' gpurun_out/av_bench_cfg5*.json
tail -3 gpurun_out/av_bench_cfg5.err
