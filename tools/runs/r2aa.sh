for v in 0 2 3 8 9; do BMM_COLSQ_VARIANT=$v timeout 300 python tools/norms_sweep.py 2>&1 | grep colsq | sed "s/^/v$v /"; done > gpurun_out/aa_variants.txt
