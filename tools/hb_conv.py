"""Probe: conv pack-aware Hyperband wall time (BASELINE configs[4] shape).
    python tools/hb_conv.py [R] [n] [family] [strategies...]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2002_02885_b200 import data, tuner  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 27
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
fam = sys.argv[3] if len(sys.argv) > 3 else "mobilenetv2"
strats = sys.argv[4:] or ["original", "knn"]
ds = data.synth_dataset(n, 3 * 32 * 32, 10, seed=0, spread=1.0)
for s in strats:
    ex = tuner.B200ConvExecutor(ds, family=fam, width=0.5 if fam == "mobilenetv2" else 1.0)
    t0 = time.perf_counter()
    res = tuner.packed_hyperband(R, 3, ex, seed=0, strategy=s)
    wall = time.perf_counter() - t0
    busy = sum(r.time_ms for r in res.records) / 1e3
    print(f"{s}: wall {wall:.2f} s  evals {len(res.records)}  epochs {res.total_epochs}  "
          f"steps {ex.steps}  best {res.best_config.config_id} {res.best_loss:.4f}", flush=True)
