"""cProfile of one conv pack-aware Hyperband run (configs[4] shape):
    python tools/hb_prof_conv.py [R] [n] [strategy]"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2002_02885_b200 import data, tuner  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 27
n = int(sys.argv[2]) if len(sys.argv) > 2 else 600
strat = sys.argv[3] if len(sys.argv) > 3 else "knn"
ds = data.synth_dataset(n, 3 * 32 * 32, 10, seed=0, spread=1.0)
warm = tuner.B200ConvExecutor(data.synth_dataset(64, 3 * 32 * 32, 10, seed=1, spread=1.0))
warm.evaluate([tuner.ConfigSpace().config(0), tuner.ConfigSpace().config(1)], 1)
ex = tuner.B200ConvExecutor(ds)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = tuner.packed_hyperband(R, 3, ex, 0, strategy=strat)
pr.disable()
print(f"{strat}: wall {time.perf_counter() - t0:.2f} s, steps {ex.steps}, evals {len(res.records)}")
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(40)
st.sort_stats("tottime").print_stats(25)
