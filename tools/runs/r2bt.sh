mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_analytics.py tests/test_gpu_pipeline.py -x -q -m gpu > gpurun_out/bt_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/bt_pytest.log
for t in 1 0 1 0; do BMM_DMMA_TALL=$t timeout 600 python bench.py --workload mc > gpurun_out/bt_mc_$t.json 2> gpurun_out/bt_mc_$t.err; python - <<PY
import json
d=json.loads(open('gpurun_out/bt_mc_$t.json').read().strip().splitlines()[-1])
print('tall=$t', d['value'], d['kernel_ms'], d['e2e']['value'], d['roofline']['frac'])
PY
done
