mkdir -p gpurun_out
for mode in "default" "BMM_GROUP_SERIAL=1" "BMM_BRANCH_PRIORITY=0" "default" "BMM_GROUP_SERIAL=1"; do
  if [ "$mode" = "default" ]; then timeout 900 python tools/timeline.py 5 cfg4 2>&1 | grep "step (stamp" | sed "s/^/$mode: /";
  else env $mode timeout 900 python tools/timeline.py 5 cfg4 2>&1 | grep "step (stamp" | sed "s/^/$mode: /"; fi
done | tee gpurun_out/bq_group_modes.txt
