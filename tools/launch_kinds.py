"""Per-kernel totals of the LAST step in an ncu launch list (gpu__time_duration.sum):
    python tools/launch_kinds.py gpurun_out/<tag>/launches_config1.csv [--seq]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
mi = h.index("Metric Name") if "Metric Name" in h else None
seq = [(r[ki].split("(")[0].replace("void ", ""), float(r[vi].replace(",", "")) / 1e3)
       for r in rows[hi + 1:] if len(r) > vi and "at::" not in r[ki]
       and (mi is None or r[mi] == "gpu__time_duration.sum")]
starts = [i for i, (n, _) in enumerate(seq) if n.endswith("k_gather")] or [0]
step = seq[starts[-1]:] if len(starts) > 1 else seq[len(seq) // 2:]
agg = collections.OrderedDict()
for n, t in step:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(t for _, t in step)
print(f"{len(step)} launches, {tot:.1f} us")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {n:32s} {c:4d} x {t / c:7.2f} us = {t:8.1f} us  {100 * t / tot:5.1f} %")
if "--seq" in sys.argv:
    for n, t in step:
        print(f"    {n:32s} {t:8.2f}")
