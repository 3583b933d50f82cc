"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel launch
count, total and mean duration, and each kernel's share of the fused-pass step (k_gram +
k_gram_reduce + k_gram_finish). usage: python tools/launch_share.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = re.sub(r"\(.*", "", r[4])
        name = re.sub(r"^.*::", "", name) if "kid::" in r[4] else name[-60:]
        agg[name][0] += 1
        agg[name][1] += float(r[-1])
    print(f"{'kernel':48s} {'n':>4s} {'total_us':>10s} {'mean_us':>9s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:48s} {n:4d} {t / 1e3:10.1f} {t / n / 1e3:9.2f}")
    step = {k: v[1] / v[0] for k, v in agg.items() if k.startswith(("k_gram", "k_gram_reduce", "k_gram_finish"))}
    tot = sum(step.values())
    if tot:
        print("\nfused-pass step (cold-cache, serialised launches):")
        for k, t in step.items():
            print(f"  {k:44s} {t / 1e3:8.2f} us  {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main()
