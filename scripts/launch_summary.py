"""Summarise an ncu --csv launch list (gpu__time_duration per kernel) -> per-kernel totals."""
import csv
import sys
from collections import defaultdict


def main(path, steps):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki][:100]].append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    print(f"{'total us':>10} {'n':>4} {'avg us':>9}  kernel   ({path}, {steps} measured steps incl. warmup)")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(v)/1e3:10.1f} {len(v):4d} {sum(v)/len(v)/1e3:9.1f}  {k}")
    print(f"{total/1e3:10.1f} total")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "?")
