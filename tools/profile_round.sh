#!/bin/bash
# One profiling pass on the GPU box (run under gpurun from the repo root):
#   1. the default bench line (plain run), then the launch list of the same command under ncu
#   2. a full ncu capture of the hot kernels at profiling sizes (tools/profile_kernels.py),
#      summarised on the box (the .ncu-rep is kept only when small enough to ship back)
# Outputs land in gpurun_out/; copy the summaries worth keeping into profiles/.
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/summarize_ncu.py launches gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_launches_summary.csv
python tools/profile_kernels.py > gpurun_out/${TAG}_pk_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on \
    -k regex:'gemm_f64_kernel|segsq_f64_kernel|oz_|colsq|rowsq|gemm_f32split|gather|compact|block_probs|budgets|sample_kernel' -c ${NCU_COUNT:-40} \
    -o /tmp/${TAG}_full python tools/profile_kernels.py > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full capture rc=$?"
python tools/summarize_ncu.py full /tmp/${TAG}_full.ncu-rep gpurun_out/${TAG}_ncu_full_summary.csv
ncu -i /tmp/${TAG}_full.ncu-rep --page details --csv > gpurun_out/${TAG}_ncu_details.csv 2>/dev/null
ncu -i /tmp/${TAG}_full.ncu-rep --page raw --csv > /tmp/${TAG}_raw.csv 2>/dev/null && gzip -c /tmp/${TAG}_raw.csv > gpurun_out/${TAG}_ncu_raw.csv.gz
echo "summaries rc=$?"
