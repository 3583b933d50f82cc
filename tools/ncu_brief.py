"""Brief summary of an ncu capture: time, FP64 / DMMA pipes, issue, stall reasons, and the instruction and
stall-sample split between the roles of a warp-specialised kernel (by SASS address range).
Usage: python tools/ncu_brief.py report.ncu-rep [role_split_hex ...]"""
import collections
import csv
import io
import re
import subprocess
import sys


def page(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = page(rep, "--page", "raw")
    d = dict(zip(rows[0], rows[2]))
    for k in ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed.sum.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]:
        print(f"{k:80s} {d.get(k)}")
    st = {k: float(v) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("not_issued") and v not in ("", "n/a")}
    tot = sum(st.values()) or 1
    print("stalls:", " ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v / tot * 100:.1f}%"
                              for k, v in sorted(st.items(), key=lambda x: -x[1])[:9]))
    src = page(rep, "--page", "source", "--print-source=sass")
    hdr = src[1]
    ia, isamp, isrc, iad = (hdr.index(x) for x in ("Instructions Executed", "Warp Stall Sampling (All Samples)",
                                                      "Source", "Address"))
    data = []
    for r in src[2:]:
        try:
            data.append((int(r[iad], 16), int(r[ia]), int(r[isamp]), r[isrc].strip()))
        except (ValueError, IndexError):
            pass
    base = data[0][0]
    cuts = [0] + [int(x, 16) for x in sys.argv[2:]] + [1 << 40]
    ti = sum(x[1] for x in data) or 1
    ts = sum(x[2] for x in data) or 1
    for lo, hi in zip(cuts, cuts[1:]):
        n = sum(x[1] for x in data if lo <= x[0] - base < hi)
        s = sum(x[2] for x in data if lo <= x[0] - base < hi)
        print(f"[{hex(lo)}, {hex(hi) if hi < 1 << 40 else 'end'}) inst {n / ti * 100:5.1f}%  samples {s / ts * 100:5.1f}%")
    ops = collections.Counter()
    for a, n, s, t in data:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", t)
        ops[m.group(2) if m else t] += n
    print("mix:", " ".join(f"{o}={n / ti * 100:.1f}%" for o, n in ops.most_common(16)))
    bars = [(hex(a - base), t[:40], s) for a, n, s, t in data if t.startswith("BAR") or "TRYWAIT" in t]
    print("barriers/waits (addr, insn, samples at it):", bars[:24])


if __name__ == "__main__":
    main()
