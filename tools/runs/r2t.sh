mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q > gpurun_out/t_pytest.log 2>&1; echo "pytest rc=$?"
for v in "BMM_GROUP_SERIAL=0" "BMM_GROUP_SERIAL=1"; do
  env $v timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/t_bench_$v.json 2> gpurun_out/t_bench_$v.err; echo "bench $v rc=$?"
done
