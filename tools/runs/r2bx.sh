mkdir -p gpurun_out
for cfg in "512,8" "1024,4" "512,8" "1024,4" "342,12" "512,6"; do
  BMM_CFG5_WAVES=$cfg timeout 600 python bench.py --workload cfg5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', round(d['value'],3), d['gpu_launches'])"
done | tee gpurun_out/bx_waves_plan_small.txt
