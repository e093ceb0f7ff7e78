mkdir -p gpurun_out
for v in "BMM_F16_CHUNK=2" "BMM_F16_CHUNK=4"; do
  env $v timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/m_bench_$v.json 2> gpurun_out/m_bench_$v.err; echo "bench $v rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/m_launches_cfg5.csv python bench.py --workload cfg5 --steps 1 --warmup 1 > gpurun_out/m_ncu_cfg5.log 2>&1; echo "ncu rc=$?"
python tools/summarize_ncu.py launches gpurun_out/m_launches_cfg5.csv gpurun_out/m_launches_cfg5_summary.csv > /dev/null 2>&1
