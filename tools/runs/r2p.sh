mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/p_bench_cfg4.json 2> gpurun_out/p_bench_cfg4.err; echo "bench rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -o /tmp/p_cfg4 python tools/profile_cfg4.py > gpurun_out/p_ncu_cfg4.log 2>&1; echo "ncu rc=$?"
python tools/summarize_ncu.py full /tmp/p_cfg4.ncu-rep gpurun_out/p_ncu_cfg4_summary.csv > /dev/null 2>&1
ncu -i /tmp/p_cfg4.ncu-rep --page raw --csv > gpurun_out/p_ncu_cfg4_raw.csv 2>/dev/null
ncu -i /tmp/p_cfg4.ncu-rep --page details --csv > gpurun_out/p_ncu_cfg4_details.csv 2>/dev/null
