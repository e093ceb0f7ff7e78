"""Summarise one kernel of an ncu report: time, DRAM bytes, issue activity, the
stall reasons and the SASS lines with the most stall samples.

  python tools/ncu_summary.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def page(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    rows = page(rep, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
            "sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"{w:70s} {vals[i]} {units[i]}")
    for i, h in enumerate(hdr):
        if "stall" in h and h.endswith("per_issue_active.ratio"):
            try:
                if float(vals[i]) > 0.3:
                    print(f"  {h:68s} {vals[i]}")
            except ValueError:
                pass
    src = page(rep, "--page", "source", "--print-source", "sass")
    h2, data = src[1], src[2:]
    isrc, ist = h2.index("Source"), h2.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[ist] or 0) for r in data) or 1.0
    for k in sorted(range(len(data)), key=lambda k: -float(data[k][ist] or 0))[:top]:
        print(f"  {k:6d} {100 * float(data[k][ist]) / tot:5.1f}%  {data[k][isrc][:90]}")


if __name__ == "__main__":
    main()
