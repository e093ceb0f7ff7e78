mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tf32.py -x -q > gpurun_out/e_tf32.log 2>&1; echo "tf32 rc=$?"
timeout 900 python -m pytest tests/test_gpu_norms_wide.py tests/test_gpu_sharded.py -x -q > gpurun_out/e_misc.log 2>&1; echo "misc rc=$?"
for v in "BMM_TF32_2SM=0" "BMM_TF32_2SM=1"; do
  env $v timeout 600 python bench.py --steps 3 --warmup 2 > gpurun_out/e_bench_$v.json 2> gpurun_out/e_bench_$v.err; echo "bench $v rc=$?"
done
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:gemm_f32split -o /tmp/e_gemm python tools/profile_cfg4.py > gpurun_out/e_ncu.log 2>&1; echo "ncu rc=$?"
python tools/summarize_ncu.py full /tmp/e_gemm.ncu-rep gpurun_out/e_ncu_gemm_summary.csv > /dev/null 2>&1
mkdir -p conformance_stage
