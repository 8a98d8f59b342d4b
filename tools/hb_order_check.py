"""Check: the conv executor's Hyperband records do not depend on evaluation order
(serial tuner.packed_hyperband vs hyperband_pool.overlapped_hyperband, 1 rank)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2002_02885_b200 import data, hyperband_pool, tuner  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 9
fam = sys.argv[2] if len(sys.argv) > 2 else "lenet5"
ds = data.synth_dataset(300, 3 * 32 * 32, 10, seed=0, spread=1.0)
w = 0.5 if fam == "mobilenetv2" else 1.0
a = tuner.packed_hyperband(R, 3, tuner.B200ConvExecutor(ds, family=fam, width=w), 0,
                           strategy="knn")
b, _ = hyperband_pool.overlapped_hyperband(R, 3, tuner.B200ConvExecutor(ds, family=fam, width=w),
                                           0, strategy="knn")
ka = [(r.bracket, r.rung, r.group, r.config_id, r.epochs, r.loss) for r in a.records]
kb = [(r.bracket, r.rung, r.group, r.config_id, r.epochs, r.loss) for r in b.records]
print("identical:", ka == kb, "best", a.best_config.config_id, b.best_config.config_id)
for x, y in zip(ka, kb):
    if x != y:
        print("  first diff", x, y)
        break
