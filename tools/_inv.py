import numpy as np, sys
sys.path.insert(0, ".")
from paper_2002_02885_b200 import data, packing
ds = {"t": data.synth_dataset(3000, 784, 10, seed=31, spread=0.5)}
arch = packing.MLPArch(784, (256,), 10, "relu")
opts = ("sgd", "adam", "momentum", "adagrad")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
hs = [packing.make_handle(f"x{i}", arch, opts[i % 4], 0.01 / (1 + i), 32, 50, "t", i) for i in range(K)]
packed = packing.dedup_inputs(packing.pack_models(hs))
packing.packed_step(packed, ds)
for i in range(K):
    solo = packing.make_handle(f"x{i}", arch, opts[i % 4], 0.01 / (1 + i), 32, 50, "t", i)
    packing.standalone_step(solo, ds)
    d = {k: float(np.max(np.abs(hs[i].params[k] - solo.params[k]))) for k in solo.params}
    n = {k: int(np.sum(hs[i].params[k] != solo.params[k])) for k in solo.params}
    print(i, opts[i % 4], d, n)
