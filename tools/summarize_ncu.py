"""Summaries of ncu outputs for profiles/ (run here, no GPU needed).

  python tools/summarize_ncu.py launches <launches.csv> <out.csv>
      per-kernel total/avg device time and share of the profiled launches
  python tools/summarize_ncu.py full <capture.ncu-rep> <out.csv>
      one row per captured launch: duration, DRAM bytes, DRAM / tensor-pipe /
      SM throughput, occupancy, registers, grid/block
"""
import collections
import csv
import io
import subprocess
import sys

FULL = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    tot, cnt = collections.Counter(), collections.Counter()
    for r in data:
        name = r[ki].split("(")[0].strip()
        tot[name] += float(r[mi].replace(",", "")) * scale[r[ui]]
        cnt[name] += 1
    grand = sum(tot.values())
    with open(dst, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel", "launches", "total_us", "avg_us", "share_pct"])
        for name, t in tot.most_common():
            w.writerow([name, cnt[name], f"{t:.1f}", f"{t / cnt[name]:.2f}", f"{100 * t / grand:.1f}"])
    print(open(dst).read())


def full(src, dst):
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    cols = ["Kernel Name"] + FULL
    idx = [h.index(c) for c in cols]
    with open(dst, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow([c if i == 0 else f"{c} [{units[j]}]" for i, (c, j) in enumerate(zip(cols, idx))])
        for r in data:
            w.writerow([r[idx[0]].split("(")[0].strip()] + [r[j] for j in idx[1:]])
    print(open(dst).read())


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
