mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_cfg5.py -x -q -m gpu > gpurun_out/bg_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/bg_pytest.log
timeout 300 python tools/plan_small_probe.py > gpurun_out/bg_plan_probe.txt 2>&1; cat gpurun_out/bg_plan_probe.txt
for cfg in "1024,4" "0,0"; do
  IFS=, read P S <<< "$cfg"
  W="$P,$S"; if [ "$P" = "0" ]; then W=0; fi
  BMM_CFG5_WAVES=$W timeout 900 python bench.py --workload cfg5 > gpurun_out/bg_bench_cfg5_${P}x${S}.json 2> gpurun_out/bg_bench_cfg5_${P}x${S}.err; echo "bench $cfg rc=$?"
done
grep -o '"value": [0-9.]*, "unit": "ms/step", "n_gpus"' gpurun_out/bg_bench_cfg5*.json
