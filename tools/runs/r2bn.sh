mkdir -p gpurun_out
s=$(date +%s); timeout 1800 python bench.py --impl reference --gpus 1 --steps 10 --warmup 3 > gpurun_out/bn_ref.json 2> gpurun_out/bn_ref.err; echo "ref rc=$? $(( $(date +%s) - s )) s"
s=$(date +%s); timeout 1800 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/bn_cfg4.json 2> gpurun_out/bn_cfg4.err; echo "bench rc=$? $(( $(date +%s) - s )) s"
python - <<'PY'
import json
for f in ('bn_ref','bn_cfg4'):
    d=json.loads(open(f'gpurun_out/{f}.json').read().strip().splitlines()[-1])
    print(f, d['value'], d['steps'], d['warmup'], (d.get('e2e') or {}).get('value'))
PY
