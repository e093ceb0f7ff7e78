mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/br_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/br_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/br_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/br_smoke.log
timeout 1500 python bench.py > gpurun_out/br_bench_cfg4.json 2> gpurun_out/br_bench_cfg4.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/br_bench_cfg4.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['parity']['ok'], d['gpu_launches'])
PY
