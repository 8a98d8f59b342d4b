"""Probe: the conv Hyperband leg as the bench runs it (bench_cnn.run_hyperband,
R=27, 600 rows): serial and concurrent-pack walls of both strategies.
    python tools/hb_conc.py [repeats]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import bench_cnn  # noqa: E402

for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    line = bench_cnn.run_hyperband(27, 600, 1, None)
    for mode, st in (("serial", line["strategies"]),
                     ("concurrent", line["concurrent_packs"]["strategies"])):
        print(f"{mode:10s} " + "  ".join(
            f"{k}: wall {v['wall_s']:.2f} s best {v['best_config']} loss {v['best_loss']:.6f}"
            for k, v in st.items()), flush=True)
