mkdir -p gpurun_out
export BMM_FORCE_SHARDED=1 BMM_EXCHANGE_WORLD1=1 NCCL_DEBUG=INFO NCCL_DEBUG_FILE=/dev/stderr
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 1 > gpurun_out/s_sharded_w1.json 2> gpurun_out/s_sharded_w1.err; echo "sharded w1 rc=$?"
unset BMM_FORCE_SHARDED
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --workload cfg5 --steps 2 --warmup 1 > gpurun_out/s_cfg5_w1.json 2> gpurun_out/s_cfg5_w1.err; echo "cfg5 w1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --workload cfg2 --steps 2 --warmup 1 > gpurun_out/s_cfg2_w1.json 2> gpurun_out/s_cfg2_w1.err; echo "cfg2 w1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 1 --impl reference --steps 2 --warmup 1 > gpurun_out/s_ref_w1.json 2> gpurun_out/s_ref_w1.err; echo "ref w1 rc=$?"
