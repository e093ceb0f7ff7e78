mkdir -p gpurun_out
for cfg in "342,12" "256,16" "512,8" "342,12" "256,16" "128,32"; do
  BMM_CFG5_WAVES=$cfg timeout 600 python bench.py --workload cfg5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', round(d['value'],3), d['gpu_launches'])"
done | tee gpurun_out/by_waves_plan_small.txt
