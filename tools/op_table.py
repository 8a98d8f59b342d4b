"""Per-op device times of one packed conv step (pk_cnn_prog_profile: un-graphed,
a spin ahead of every op) with each op's shape and algorithmic bytes / FLOPs:
    python tools/op_table.py config1 [reps] > table.txt
Columns: op index, kind, lane, problems, first problem's shape, us, GB/s or TF/s."""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2002_02885_b200 import _lib, cnn, data, packing  # noqa: E402
from tools import bench_cnn  # noqa: E402

wl = dict(bench_cnn.WORKLOADS[sys.argv[1]])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
c, h, w = wl["image"]
ds = data.synth_dataset(wl["n"], c * h * w, wl["classes"], seed=0, spread=1.0)
arch, hs = bench_cnn._handles(wl, packing, cnn)
packed = packing.dedup_inputs(packing.pack_models(hs))
for _ in range(3):
    packing.packed_step(packed, {"train": ds})
cp = packed._cp
prog = next(iter(cp._progs.values()))
torch.cuda.synchronize()
tot = None
for _ in range(reps):
    t = prog.profile(cp.stream.cuda_stream)
    tot = t if tot is None else [min(a, b) for a, b in zip(tot, t)]
names = {v: k for k, v in _lib.CNN.items()}


def work(kind, s):
    """(bytes, flops) of one problem."""
    k = names[kind]
    if k.startswith("CONV"):
        M = s.n * s.p * s.q
        mac = M * s.k * s.r * s.s * s.c
        if k == "CONV_FPROP":
            by = 2 * (s.n * s.h * s.w * s.c + M * s.k)
        elif k == "CONV_DGRAD":
            by = 2 * (s.n * s.h * s.w * s.c + M * s.k)
        else:
            by = 2 * (s.n * s.h * s.w * s.c + M * s.k) + 4 * s.k * s.r * s.s * s.c * max(1, s.splits)
        return by, 2 * mac, f"n{s.n} {s.h}x{s.w}x{s.c} -> {s.p}x{s.q}x{s.k} {s.r}x{s.s}/{s.stride}"
    if k.startswith("BN"):
        e = s.rows * s.c * 2
        mult = {"BN_STATS": 1, "BN_APPLY": 3 if s.res else 2, "BN_BWD_REDUCE": 3,
                "BN_BWD_APPLY": 5 if s.res else 4}[k]
        return e * mult, 0, f"rows {s.rows} c {s.c}"
    if k.startswith("DW"):
        ex = s.n * s.h * s.w * s.c * 2
        ey = s.n * s.p * s.q * s.c * 2
        return ex + ey, 0, f"n{s.n} {s.h}x{s.w}x{s.c} -> {s.p}x{s.q} /{s.stride}"
    return 0, 0, ""


ops = prog._keep
agg = collections.OrderedDict()
print(f"{'i':>4} {'kind':14} {'ln':>3} {'np':>3} {'us':>8} {'GB/s':>7} {'TF/s':>6}  shape")
for i, (kind, buf, ms) in enumerate(zip(prog.kinds, ops, tot)):
    by = fl = 0
    desc = ""
    for j, s in enumerate(buf):
        b, f, d = work(kind, s)
        by += b
        fl += f
        if j == 0:
            desc = d
    us = ms * 1e3
    gbs = by / (us * 1e-6) / 1e9 if us > 0 and by else 0
    tfs = fl / (us * 1e-6) / 1e12 if us > 0 and fl else 0
    print(f"{i:4d} {names[kind]:14} {prog.lanes[i]:3d} {len(buf):3d} {us:8.1f} {gbs:7.0f} {tfs:6.1f}  {desc}")
    a = agg.setdefault(names[kind], [0, 0.0, 0])
    a[0] += 1
    a[1] += us
    a[2] += by
print()
for k, (n, us, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:14} {n:4d} ops {us:9.1f} us  {by / max(us, 1e-9) / 1e3:7.0f} GB/s")
print(f"total {sum(tot) * 1e3:.1f} us, {len(tot)} ops")
