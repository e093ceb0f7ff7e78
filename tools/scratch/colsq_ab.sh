for f in w wr; do for v in 1 3 7; do
  echo "flush=$f variant=$v"
  BMM_FLUSH=$f BMM_COLSQ_VARIANT=$v timeout 300 python tools/norms_sweep.py 2>&1
done; done
