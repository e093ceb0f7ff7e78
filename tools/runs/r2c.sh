mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/c_pytest.log 2>&1; echo "pytest rc=$?"
for v in "BMM_COLSQ_WIDE=0" "BMM_COLSQ_WIDE=1"; do
  env $v timeout 300 python tools/cfg4_norms_probe.py >> gpurun_out/c_norms.txt 2>&1
done
timeout 1200 python bench.py > gpurun_out/c_bench_cfg4.json 2> gpurun_out/c_bench_cfg4.err; echo "bench rc=$?"
timeout 600 python bench.py --workload cfg2 > gpurun_out/c_bench_cfg2.json 2> gpurun_out/c_bench_cfg2.err; echo "bench cfg2 rc=$?"
