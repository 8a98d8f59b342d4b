"""Where the Hyperband (knn) wall time goes: cProfile of one R=81 run on the
B200 executor, plus the packed-step count.  A profiling aid, not a benchmark.

    python tools/hb_profile.py [--strategy knn] [--precision f64] [--top 30]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2002_02885_b200 import data, hyperband_pool, runtime, tuner  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--strategy", default="knn")
    ap.add_argument("--precision", default="f64", choices=["f32", "f64"])
    ap.add_argument("--R", type=int, default=81)
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    HB = bench.HB
    runtime.set_precision(a.precision)
    warm = tuner.B200Executor(data.synth_dataset(64, HB["dim"], HB["classes"], seed=1),
                              hidden=HB["hidden"], seed=HB["seed"])
    warm.evaluate([tuner.ConfigSpace().config(0), tuner.ConfigSpace().config(1)], 1)
    ds = data.synth_dataset(HB["n"], HB["dim"], HB["classes"], seed=0)
    for rep in range(2):
        ex = tuner.B200Executor(ds, hidden=HB["hidden"], seed=HB["seed"])
        prof = cProfile.Profile() if rep == 1 else None
        t0 = time.perf_counter()
        if prof:
            prof.enable()
        res, pool = hyperband_pool.sharded_hyperband(a.R, HB["eta"], ex, HB["seed"],
                                                     strategy=a.strategy)
        if prof:
            prof.disable()
        wall = time.perf_counter() - t0
        print(f"rep {rep}: wall {wall:.3f} s  packed steps {ex.steps}  "
              f"evaluations {len(res.records)}  epochs {res.total_epochs}  "
              f"{1e6 * wall / max(ex.steps, 1):.1f} us/step (wall)", flush=True)
    st = pstats.Stats(prof)
    st.sort_stats("tottime").print_stats(a.top)
    st.sort_stats("cumulative").print_stats(a.top)


if __name__ == "__main__":
    main()
