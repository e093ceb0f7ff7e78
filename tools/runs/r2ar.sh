mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ar_smi.txt 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/ar_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ar_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/ar_bench_cfg4.json 2> gpurun_out/ar_bench_cfg4.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ar_bench_ref.json 2> gpurun_out/ar_bench_ref.err; echo "ref rc=$?"
timeout 600 python tools/cfg5_stages.py > gpurun_out/ar_cfg5_stages.txt 2>&1; echo "cfg5 stages rc=$?"
