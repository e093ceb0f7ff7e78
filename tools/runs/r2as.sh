mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_datagen.py tests/test_abi.py -x -q -m gpu > gpurun_out/as_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -o /tmp/as_cfg4 python tools/profile_cfg4.py > gpurun_out/as_ncu_cfg4.log 2>&1; echo "ncu rc=$?"
python tools/summarize_ncu.py full /tmp/as_cfg4.ncu-rep gpurun_out/as_ncu_cfg4_summary.csv > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/as_launches_cfg4.csv python bench.py --steps 1 --warmup 1 > gpurun_out/as_ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/summarize_ncu.py launches gpurun_out/as_launches_cfg4.csv gpurun_out/as_launches_cfg4_summary.csv > /dev/null 2>&1
