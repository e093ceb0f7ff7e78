mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g_smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "smoke rc=$?"
for w in cfg2 cfg1 cfg3 cfg5 cfg4 mc; do
  timeout 600 python bench.py --workload $w > gpurun_out/g_bench_$w.json 2> gpurun_out/g_bench_$w.err; echo "bench $w rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g_bench_ref.json 2> gpurun_out/g_bench_ref.err; echo "ref rc=$?"
