mkdir -p gpurun_out
run() { env "$@" timeout 600 python bench.py --workload cfg2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['value'],4), round(d['e2e']['value'],3))"; }
run X=1; run X=1
run BMM_BRANCH_PRIORITY=0; run BMM_BRANCH_PRIORITY=1
run BMM_GSQ_FORK=0
run BMM_JOINT_BY=method
run BMM_JOINT=0
run BMM_OZ_CTAS=128
