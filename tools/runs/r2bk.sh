mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_cfg4.py tests/test_gpu_sharded.py tests/test_gpu_pipeline.py -x -q -m gpu > gpurun_out/bk_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/bk_pytest.log
timeout 1500 python bench.py > gpurun_out/bk_bench_cfg4.json 2> gpurun_out/bk_bench_cfg4.err; echo "bench rc=$?"
tail -3 gpurun_out/bk_bench_cfg4.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bk_bench_cfg4.json').read().strip().splitlines()[-1])
print(d['value'], d['kernel_ms'], d['clocks'], d['parity'].get('cd_rel_err_vs_f64_same_sketch'), d['e2e']['value'], d['roofline']['frac'])
PY
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -o /tmp/bk_cfg4 python tools/profile_cfg4.py > gpurun_out/bk_ncu_cfg4.log 2>&1; echo "ncu rc=$?"
python tools/summarize_ncu.py full /tmp/bk_cfg4.ncu-rep gpurun_out/bk_ncu_cfg4_summary.csv > /dev/null 2>&1
cat gpurun_out/bk_ncu_cfg4_summary.csv | cut -c1-200
