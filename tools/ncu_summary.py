"""Summarise an ncu report: per-kernel time / pipes / DRAM, and SASS stall hot spots.

usage: python tools/ncu_summary.py report.ncu-rep [kernel-substring] [--sass N]
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def ncu(*args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    sub = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else ""
    nsass = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 0
    metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
               "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
               "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
               "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
               "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
    txt = ncu(rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics))
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if sub and sub not in d["Kernel Name"]:
            continue
        name = d["Kernel Name"].split("(")[0][-40:]
        print(f"{name:40s} t={d['gpu__time_duration.sum']}{units[hdr.index('gpu__time_duration.sum')]} dram_r={d['dram__bytes_read.sum']}"
              f"{units[hdr.index('dram__bytes_read.sum')]} dram_w={d['dram__bytes_write.sum']}"
              f"{units[hdr.index('dram__bytes_write.sum')]} fp64={d[metrics[3]]}% dmma={d[metrics[4]]}% "
              f"warps={d[metrics[5]]}% issue={d[metrics[7]]}% regs={d[metrics[6]]} grid={d[metrics[8]]} "
              f"dram%={d[metrics[10]]}")
    if nsass:
        txt = ncu(rep, "--page", "source", "--csv", "--print-source", "sass")
        rows = list(csv.reader(io.StringIO(txt)))
        starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
        pick = next(k for k in range(len(starts) - 1) if sub in rows[starts[k]][1].replace("(int)", ""))
        blk = rows[starts[pick] + 1:starts[pick + 1]]
        hdr, data = blk[0], blk[1:]
        iS, iSrc, iA = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Address")
        tot = sum(float(r[iS] or 0) for r in data) or 1.0
        c = Counter()
        for r in data:
            t = r[iSrc].strip().split()
            if t:
                c[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += float(r[iS] or 0)
        print("stall samples by opcode:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in c.most_common(12)))
        for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:nsass]:
            print(f"  {r[iA][-5:]} {float(r[iS]) / tot * 100:5.2f}%  {r[iSrc][:90]}")


if __name__ == "__main__":
    main()
