"""Probe: the conv Hyperband leg (bench_cnn.run_hyperband, R=27, 600 rows) with the
pool's concurrent packs per GPU set to each given value.
    python tools/hb_conc.py 1 4 8"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import bench_cnn  # noqa: E402
from paper_2002_02885_b200 import tuner  # noqa: E402

for conc in [int(a) for a in sys.argv[1:]] or [1, 4]:
    tuner.B200ConvExecutor.concurrent_groups = conc
    line = bench_cnn.run_hyperband(27, 600, 1, None)
    st = line["strategies"]
    print(f"concurrent {conc}: " + "  ".join(
        f"{k}: wall {v['wall_s']:.2f} s best {v['best_config']} loss {v['best_loss']:.6f} "
        f"evals {v['evaluations']}" for k, v in st.items()), flush=True)
