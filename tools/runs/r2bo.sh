mkdir -p gpurun_out
BMM_FORCE_SHARDED=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/bo_sharded_w1.json 2> gpurun_out/bo_sharded_w1.err; echo "sharded world-1 rc=$?"
tail -2 gpurun_out/bo_sharded_w1.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bo_sharded_w1.json').read().strip().splitlines()[-1])
print(d['value'], d['n_gpus'], d['scaling'], d['config'], (d.get('e2e') or {}).get('value'), d.get('parity'))
PY
