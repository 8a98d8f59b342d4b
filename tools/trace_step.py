"""Stage timeline of one packed step from in-kernel %globaltimer stamps.

    python tools/trace_step.py [--workload config0] [--warm]   (sets plan option trace=1)

Runs warm-up steps, flushes L2 (unless --warm), runs one traced step through
the CUDA graph and prints, per phase, when its CTAs entered, had operands,
finished the GEMM / epilogue parts and retired — relative to the first CTA
of the step.  A profiling aid, not a benchmark.
"""
import argparse
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2002_02885_b200 import _lib, data, packing, runtime  # noqa: E402

_lib.set_plan_options(trace=1)

STAGES = ("entry", "ready", "gemm", "epi1", "epi2", "done", "fin0", "fin1",
          "s8", "s9", "s10", "s11", "s12", "s13", "s14", "s15")

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config0", choices=sorted(bench.WORKLOADS) + sorted(bench.HB_SHAPES))
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"])
    ap.add_argument("--warm", action="store_true", help="no L2 flush before the traced step")
    ap.add_argument("--steps", type=int, default=3, help="traced steps (last one printed)")
    a = ap.parse_args()
    import torch
    runtime.set_precision(a.precision)
    rt = runtime.runtime()
    stream = torch.cuda.Stream()
    rt.set_stream(stream.cuda_stream)
    wl = bench.WORKLOADS.get(a.workload) or bench.HB_SHAPES[a.workload]
    datasets, hs = bench._make(wl, data, packing)
    packed = packing.dedup_inputs(packing.pack_models(hs))
    for _ in range(5):
        packing.packed_step(packed, datasets)
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    for _ in range(a.steps):
        if not a.warm:
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
        packing.packed_step(packed, datasets)
    dp = packed._dev[1]
    n = rt.lib.pk_pack_trace(dp.ptr, None, 0)
    if n < 0:
        sys.exit("tracing is off (plan option trace=1 must be set before the pack is created)")
    buf = (C.c_uint64 * n)()
    rt.lib.pk_pack_trace(dp.ptr, buf, n)
    arr = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(-1, len(STAGES))
    code, phases, _ = dp.profile()  # only for per-phase CTA counts
    t0 = arr[arr[:, 0] > 0, 0].min()
    off = 0
    plan = bench._phase_plan(wl, 8 if a.precision == "f64" else 4)
    for i, (kind, layer, ctas, _) in enumerate(phases):
        blk = arr[off:off + ctas]
        off += ctas
        label = plan[i][0] if i < len(plan) else f"phase{i}"
        print(f"phase {i} {label:16s} ctas={ctas}")
        for s, name in enumerate(STAGES):
            v = blk[:, s]
            v = v[v > 0] - t0
            if len(v):
                print(f"   {name:6s} min {v.min() / 1e3:8.2f}  med {statistics.median(v) / 1e3:8.2f}"
                      f"  max {v.max() / 1e3:8.2f} us   (n={len(v)})")
        if os.environ.get("PK_TRACE_BY_MEMBER") and i == len(phases) - 1:
            # last phase: per-member medians of ready→done (tiles are member-major)
            per = max(1, ctas // len(hs))
            t0m = blk[:, 1]
            for k, h in enumerate(hs):
                seg = blk[k * per:(k + 1) * per]
                d = (seg[:, 5] - seg[:, 1]) / 1e3
                print(f"   member {k} {h.optimizer.kind:9s} ready→done med {statistics.median(d):6.2f}"
                      f"  max {d.max():6.2f} us")
        if int(os.environ.get("PK_M1X_DEBUG", "0")) & 32:  # k_m1x: clock64 at chunks 4 / 8
            cyc = (blk[:, 7] - blk[:, 6]) / 4.0
            ns = (blk[:, 12] - blk[:, 11]) / 4.0
            print(f"   chunk 4..8: {statistics.median(cyc):.0f} cycles/iter, "
                  f"{statistics.median(ns):.0f} ns/iter → {statistics.median(cyc / ns):.3f} GHz")


if __name__ == "__main__":
    main()
