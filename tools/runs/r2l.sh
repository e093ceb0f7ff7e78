mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_cfg5.py tests/test_gpu_pipeline.py tests/test_gpu_tf32.py -x -q > gpurun_out/l_pytest.log 2>&1; echo "pytest rc=$?"
for v in "BMM_F16=0" "BMM_F16=1"; do
env $v timeout 900 python bench.py --workload cfg5 > gpurun_out/l_bench_cfg5_$v.json 2> gpurun_out/l_bench_cfg5_$v.err; echo "bench $v rc=$?"
done
