mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -m gpu -k "plan_small or waves or many_small or cfg5" > gpurun_out/ay_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/ay_pytest.log
timeout 300 python tools/plan_small_probe.py > gpurun_out/ay_plan_probe.txt 2>&1; cat gpurun_out/ay_plan_probe.txt
for cfg in "1024,4,0" "0,0,0" "2048,2,0"; do
  IFS=, read P S PIPE <<< "$cfg"
  W="$P,$S"; if [ "$P" = "0" ]; then W=0; fi
  BMM_WAVE_PIPE=$PIPE BMM_CFG5_WAVES=$W timeout 900 python bench.py --workload cfg5 > gpurun_out/ay_bench_cfg5_${P}x${S}_pipe${PIPE}.json 2> gpurun_out/ay_bench_cfg5_${P}x${S}_pipe${PIPE}.err; echo "bench $cfg rc=$?"
done
grep -o '"value": [0-9.]*, "unit": "ms/step", "n_gpus"' gpurun_out/ay_bench_cfg5*.json
