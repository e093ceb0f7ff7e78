mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:plan_small -c 1 -o /tmp/bf_plan python tools/plan_small_probe.py > gpurun_out/bf_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/bf_plan.ncu-rep --page raw --csv > /tmp/bf_raw.csv 2>/dev/null
python - <<'PY'
import csv
rows=list(csv.reader(open('/tmp/bf_raw.csv')))
hdr=rows[0]; vals=rows[2] if len(rows)>2 else rows[1]
keep=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__occupancy_limit_shared_mem','launch__occupancy_limit_registers','smsp__inst_executed.sum','sm__inst_executed_pipe_fp64.sum','smsp__inst_executed_pipe_fp64.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']
out=[]
for h,v in zip(hdr,vals):
    if h in keep or 'issue_stalled' in h and 'per_issue_active' in h or 'pipe_fp64' in h:
        out.append(f"{h:90s} {v}")
open('gpurun_out/bf_plan_small_ncu.txt','w').write("\n".join(out)+"\n")
PY
ncu -i /tmp/bf_plan.ncu-rep --page source --csv > /tmp/bf_src.csv 2>/dev/null; python - <<'PY'
import csv
rows=list(csv.reader(open('/tmp/bf_src.csv')))
hdr=rows[0]
# find the sampling column
idx=[i for i,h in enumerate(hdr) if 'Sampl' in h and 'All' in h] or [i for i,h in enumerate(hdr) if 'Sampl' in h]
si=idx[0]; src=[i for i,h in enumerate(hdr) if h.strip() in ('Source','# Source')] 
tot=0; data=[]
for r in rows[1:]:
    try: c=float(r[si])
    except: continue
    tot+=c; data.append((c,r))
data.sort(key=lambda x:-x[0])
with open('gpurun_out/bf_plan_small_hot.txt','w') as f:
    f.write(f"total samples {tot}\n")
    for c,r in data[:40]:
        f.write(f"{c:8.0f} {100*c/max(tot,1):5.1f}%  {' | '.join(x for x in r[:3])}\n")
PY
head -50 gpurun_out/bf_plan_small_ncu.txt
