for v in "BMM_GSQ_FORK=1" "BMM_GSQ_FORK=0" "BMM_SHARED=0"; do
  echo "== $v"; env $v timeout 600 python tools/stress_group.py 40
done
