"""Debug: wide16 shape one step vs the f64 oracle, per member/tensor error stats."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from _helpers import oracle_dataset, oracle_from_handle  # noqa: E402
from oracle import mlp64 as O  # noqa: E402
from paper_2002_02885_b200 import _lib, data, packing  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
K = int(sys.argv[3]) if len(sys.argv) > 3 else 16
fwd = sys.argv[4] if len(sys.argv) > 4 else "auto"
_lib.set_plan_options(fwd=fwd)
ds = {"t": data.synth_dataset(1000, 784, 10, seed=43, spread=0.5)}
arch = packing.MLPArch(784, (H,), 10, "relu")
opts = ("sgd", "adam", "momentum", "adagrad")
hs = [packing.make_handle(f"w{i}", arch, opts[i % 4], 10.0 ** -(1 + i % 4), B, 20, "t", i)
      for i in range(K)]
packed = packing.dedup_inputs(packing.pack_models(hs))
odata = {k: oracle_dataset(v) for k, v in ds.items()}
oms = [oracle_from_handle(h) for h in packed.members]
gout = {}
want, _ = O.oracle_packed_step(oms, odata, grads_out=gout)
got = packing.packed_step(packed, ds)
print("H", H, "B", B, "K", K, "fwd", fwd)
for h, m in zip(hs, oms):
    line = [f"{h.model_id} {h.optimizer.kind:8s} loss {got[h.model_id]:.6f}/{want[h.model_id]:.6f}"]
    for i, (w, b) in enumerate(m.layers):
        for j, (nm, ref) in enumerate(((f"L{i}/W", w), (f"L{i}/b", b))):
            g = h.params[f"{h.model_id}/{nm}"]
            err = np.abs(g - ref) - (1e-4 * np.abs(ref) + 1e-6)
            nbad = int((err > 0).sum())
            if nbad:
                idx = np.unravel_index(np.argmax(err), err.shape)
                gr = gout[h.model_id][0][i][j][idx]
                sc = gout[h.model_id][1][i][j][idx]
                line.append(f"{nm}: {nbad} bad, worst {np.abs(g - ref).max():.2e} at {idx} "
                            f"g {gr:.2e} scale {sc:.2e}")
    print("  ".join(line), flush=True)
for h, m in zip(hs, oms):
    for i, (w, b) in enumerate(m.layers):
        for j, (nm, ref) in enumerate(((f"L{i}/W", w), (f"L{i}/b", b))):
            g = h.params[f"{h.model_id}/{nm}"]
            err = np.abs(g - ref) - (1e-4 * np.abs(ref) + 1e-6)
            bad = err > 0
            if bad.any():
                r = np.abs(gout[h.model_id][0][i][j])[bad] / gout[h.model_id][1][i][j][bad]
                print(h.model_id, nm, "max |g|/scale of off elements", float(r.max()))
