"""cProfile of a pack-aware Hyperband run on the B200 executor (host vs device split).

    python tools/hb_profile.py [--R 27] [--precision f64]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_02885_b200 import data, runtime, tuner  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--R", type=int, default=27)
    ap.add_argument("--precision", default="f64")
    a = ap.parse_args()
    runtime.set_precision(a.precision)
    ds = data.synth_dataset(2000, 784, 10, seed=0)
    ex = tuner.B200Executor(ds, hidden=(16,), seed=0)
    t0 = time.perf_counter()
    pr = cProfile.Profile()
    pr.enable()
    res = tuner.packed_hyperband(a.R, 3, ex, 0, strategy="knn")
    pr.disable()
    print(f"wall {time.perf_counter() - t0:.2f} s, packed/standalone steps {ex.steps}, "
          f"best {res.best_config.config_id}")
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(30)


if __name__ == "__main__":
    main()
