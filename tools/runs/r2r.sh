mkdir -p gpurun_out
for v in "BMM_JOINT_BY=width" "BMM_JOINT_BY=method" "BMM_JOINT=0"; do
  env $v timeout 600 python bench.py --workload cfg2 --steps 20 --warmup 5 > gpurun_out/r_bench_cfg2_$v.json 2> gpurun_out/r_bench_cfg2_$v.err; echo "bench $v rc=$?"
  env $v timeout 300 python tools/timeline.py 5 > gpurun_out/r_timeline_$v.txt 2>&1
done
BMM_JOINT_BY=method timeout 600 python -m pytest tests/test_gpu_pipeline.py -x -q -k joint > gpurun_out/r_pytest.log 2>&1; echo "pytest rc=$?"
