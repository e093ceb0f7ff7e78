mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/ao_bench_cfg4.json 2> gpurun_out/ao_bench_cfg4.err; echo "bench rc=$?"
tail -2 gpurun_out/ao_bench_cfg4.err
