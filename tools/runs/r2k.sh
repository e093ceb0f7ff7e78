mkdir -p gpurun_out
for w in cfg2 cfg3 cfg1 mc; do
timeout 900 python bench.py --workload $w > gpurun_out/k_bench_$w.json 2> gpurun_out/k_bench_$w.err; echo "bench $w rc=$?"
done
timeout 300 python tools/timeline.py 5 > gpurun_out/k_timeline_cfg2.txt 2>&1; echo "timeline rc=$?"
