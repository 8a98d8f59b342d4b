"""Drive N packed steps of a bench workload through the public API, for
`ncu` captures (see profiles/README.md).  Not a benchmark: numbers printed
under a profiler are never bench values.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 20
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2002_02885_b200 import data, packing, runtime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config0", choices=sorted(bench.WORKLOADS) + sorted(bench.HB_SHAPES))
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"])
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    wl = bench.WORKLOADS.get(a.workload) or bench.HB_SHAPES[a.workload]
    runtime.set_precision(a.precision)
    datasets, hs = bench._make(wl, data, packing)
    packed = packing.dedup_inputs(packing.pack_models(hs))
    for _ in range(a.steps):
        losses = packing.packed_step(packed, datasets)
    print("ok", losses)


if __name__ == "__main__":
    main()
