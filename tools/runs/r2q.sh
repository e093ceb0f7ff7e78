mkdir -p gpurun_out
for g in 4 8 16 32; do
  BMM_F16_GROUP_M=$g timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_f16 --csv python tools/profile_cfg4.py > gpurun_out/q_ncu_g$g.csv 2>&1; echo "g$g rc=$?"
done
