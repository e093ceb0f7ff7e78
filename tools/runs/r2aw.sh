mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -m gpu -k "plan_small or waves or many_small or cfg5" > gpurun_out/aw_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/aw_pytest.log
for cfg in "1024,4,1" "1024,4,0" "512,4,1" "512,6,1" "512,8,1" "256,6,1" "2048,2,1"; do
  IFS=, read P S PR <<< "$cfg"
  BMM_WAVE_PRIO=$PR BMM_CFG5_WAVES=$P,$S timeout 900 python bench.py --workload cfg5 > gpurun_out/aw_bench_cfg5_${P}x${S}_p${PR}.json 2> gpurun_out/aw_bench_cfg5_${P}x${S}_p${PR}.err; echo "bench $cfg rc=$?"
done
grep -o '"value": [0-9.]*, "unit": "ms/step", "n_gpus"' gpurun_out/aw_bench_cfg5*.json
