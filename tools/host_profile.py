"""cProfile of the public packed_step loop (host overhead per step).

    python tools/host_profile.py [--mode stream|resident] [--steps 2000]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2002_02885_b200 import data, packing, runtime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="resident")
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--workload", default="config0")
    a = ap.parse_args()
    runtime.set_input_mode(a.mode)
    wl = bench.WORKLOADS[a.workload]
    datasets, hs = bench._make(wl, data, packing)
    packed = packing.dedup_inputs(packing.pack_models(hs))
    for _ in range(20):
        packing.packed_step(packed, datasets)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        packing.packed_step(packed, datasets)
    dt = time.perf_counter() - t0
    print(f"{a.mode}: {dt / a.steps * 1e6:.1f} us/step wall")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(a.steps):
        packing.packed_step(packed, datasets)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
