mkdir -p gpurun_out
timeout 1200 python tools/conformance.py conformance_stage > gpurun_out/f_conformance.log 2>&1; echo "conformance rc=$?"
CS=/usr/local/cuda/bin/compute-sanitizer
for part in f32 f64; do
  timeout 900 $CS --tool memcheck --print-limit 20 python tools/sanitize_kernels.py $part > gpurun_out/f_memcheck_$part.log 2>&1; echo "memcheck $part rc=$?"
done
BMM_COLSQ_WIDE=2 timeout 600 $CS --tool memcheck --print-limit 20 python tools/sanitize_kernels.py wide > gpurun_out/f_memcheck_wide.log 2>&1; echo "memcheck wide rc=$?"
for part in f32 f64; do
  timeout 1200 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_kernels.py $part > gpurun_out/f_racecheck_$part.log 2>&1; echo "racecheck $part rc=$?"
done
BMM_COLSQ_WIDE=2 timeout 600 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_kernels.py wide > gpurun_out/f_racecheck_wide.log 2>&1; echo "racecheck wide rc=$?"
timeout 900 $CS --tool synccheck --print-limit 20 python tools/sanitize_kernels.py f32 > gpurun_out/f_synccheck_f32.log 2>&1; echo "synccheck f32 rc=$?"
for c in 0 1 2 3 4; do
  BMM_COLSQ_WIDE_CFG=$c timeout 300 python tools/cfg4_norms_probe.py >> gpurun_out/f_norms.txt 2>&1
done
timeout 2400 python -m pytest tests/test_gpu_cfg4.py tests/test_gpu_cfg5.py -x -q > gpurun_out/f_full.log 2>&1; echo "full-size rc=$?"
