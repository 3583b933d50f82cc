"""Stall reasons of a warp-specialized kernel split by role: instructions between the
setmaxnreg.dec and setmaxnreg.inc (the eval warps) vs after the setmaxnreg.inc (MMA warps).
usage: python tools/ncu_regions.py report.ncu-rep [kernel-substring]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    rep, sub = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    pick = next(k for k in range(len(starts) - 1) if sub in rows[starts[k]][1])
    blk = rows[starts[pick] + 1:starts[pick + 1]]
    hdr, data = blk[0], blk[1:]
    iS = hdr.index("Source")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    region, acc, n_inst = "prologue", {}, Counter()
    for r in data:
        src = r[iS]
        if "SETMAXREG.DEALLOC" in src:
            region = "eval"
        elif "SETMAXREG.ALLOC" in src or "SETMAXREG.TRY_ALLOC" in src:
            region = "mma"
        c = acc.setdefault(region, Counter())
        for h in reasons:
            c[h] += float(r[hdr.index(h)] or 0)
        n_inst[region] += float(r[hdr.index("Instructions Executed")] or 0)
    tot = sum(sum(c.values()) for c in acc.values()) or 1
    for reg, c in acc.items():
        s = sum(c.values())
        top = ", ".join(f"{k[6:]}={100 * v / s:.1f}%" for k, v in c.most_common(8) if v)
        print(f"{reg:9s} {100 * s / tot:5.1f}% of samples, {n_inst[reg]:.3g} warp-instr | {top}")


if __name__ == "__main__":
    main()
