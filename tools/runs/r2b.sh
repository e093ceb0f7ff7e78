mkdir -p gpurun_out
free -g > gpurun_out/b_free.txt; nproc >> gpurun_out/b_free.txt; lscpu | head -20 >> gpurun_out/b_free.txt
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_gram_blocks.py -x -q > gpurun_out/b_pytest.log 2>&1; echo "pytest rc=$?"
for v in "" "BMM_COLSQ_R=16" "BMM_ROWSQ_VARIANT=1" "BMM_ROWSQ_VARIANT=1 BMM_ROWSQ_STREAM=2" "BMM_ROWSQ_VARIANT=1 BMM_ROWSQ_STREAM=3"; do
  env $v timeout 300 python tools/cfg4_norms_probe.py >> gpurun_out/b_norms.txt 2>&1
done
timeout 1200 python bench.py > gpurun_out/b_bench_cfg4.json 2> gpurun_out/b_bench_cfg4.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/b_bench_ref.json 2> gpurun_out/b_bench_ref.err; echo "ref rc=$?"
