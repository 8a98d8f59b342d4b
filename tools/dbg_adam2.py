"""Debug: wide16 shape, step 2 (after one profiled step) vs the oracle: the off
elements of an Adam member with their g, m, v on both sides."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from _helpers import oracle_dataset, oracle_from_handle  # noqa: E402
from oracle import mlp64 as O  # noqa: E402
from paper_2002_02885_b200 import data, packing  # noqa: E402

ds = {"t": data.synth_dataset(1000, 784, 10, seed=43, spread=0.5)}
arch = packing.MLPArch(784, (1024,), 10, "relu")
opts = ("sgd", "adam", "momentum", "adagrad")
hs = [packing.make_handle(f"w{i}", arch, opts[i % 4], 10.0 ** -(1 + i % 4), 128, 20, "t", i)
      for i in range(16)]
packed = packing.dedup_inputs(packing.pack_models(hs))
odata = {k: oracle_dataset(v) for k, v in ds.items()}
mode = sys.argv[1] if len(sys.argv) > 1 else "profile"
if mode == "profile":
    active = packing._active_members(packed, ds, False)
    plan_ = packing._plan_step(packed, active, ds, None, None)
    code, phases, losses = plan_.dpack.profile()
    packing._apply_result(packed, active, plan_, code, -1, -1, losses)
else:
    packing.packed_step(packed, ds)
for step in range(2):
    oms = [oracle_from_handle(h) for h in packed.members]
    before = {h.model_id: {k: v.copy() for k, v in h.params.items()} for h in hs}
    gout = {}
    want, _ = O.oracle_packed_step(oms, odata, grads_out=gout)
    got = packing.packed_step(packed, ds)
    for h, m in zip(hs, oms):
        if h.optimizer.kind != "adam":
            continue
        for i, (w, b) in enumerate(m.layers):
            for j, (nm, ref) in enumerate(((f"L{i}/W", w), (f"L{i}/b", b))):
                full = f"{h.model_id}/{nm}"
                g = h.params[full]
                err = np.abs(g - ref) - (1e-4 * np.abs(ref) + 1e-6)
                bad = np.argwhere(err > 0)
                if len(bad) == 0:
                    continue
                print(f"step {step} {full}: {len(bad)} off", flush=True)
                gr, sc = gout[h.model_id][0][i][j], gout[h.model_id][1][i][j]
                mo = m.slots[(i, "W" if j == 0 else "b")]
                md = h.optimizer.slots[f"{h.model_id}/L{i}/{'W' if j == 0 else 'b'}"]
                for idx in bad[:6]:
                    idx = tuple(idx)
                    print(f"   {idx} w0 {before[h.model_id][full][idx]:+.6e} dev {g[idx]:+.6e} "
                          f"ref {ref[idx]:+.6e} g {gr[idx]:+.3e} scale {sc[idx]:.3e} "
                          f"m dev {md['m'][idx]:+.3e} ref {mo['m'][idx]:+.3e} "
                          f"v dev {md['v'][idx]:.3e} ref {mo['v'][idx]:.3e}", flush=True)
