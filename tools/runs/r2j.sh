mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tf32.py -x -q > gpurun_out/j_tf32.log 2>&1; echo "tf32 rc=$?"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/j_pytest.log 2>&1; echo "pytest rc=$?"
for v in "BMM_F16=0" "BMM_F16=1"; do
  env $v timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/j_bench_$v.json 2> gpurun_out/j_bench_$v.err; echo "bench $v rc=$?"
done
