python -m pytest -q -x tests/test_gpu_parity.py -k "rowsq or norms" 2>&1 | tail -3
for v in 0 1 2 3; do
  echo "stream cfg=$v"; BMM_FLUSH=wr BMM_ROWSQ_STREAM=$v timeout 300 python tools/norms_sweep.py 2>&1 | grep "rowsq cfg[23]"
done
echo "leaf"; BMM_FLUSH=wr BMM_ROWSQ_VARIANT=1 timeout 300 python tools/norms_sweep.py 2>&1 | grep "rowsq cfg[23]"
