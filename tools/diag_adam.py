import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import numpy as np
from paper_2002_02885_b200 import data, packing
from oracle import mlp64 as O
from _helpers import oracle_from_handle, oracle_dataset
ds = {"t": data.synth_dataset(3000, 784, 10, seed=7, spread=0.5)}
arch = packing.MLPArch(784, (256,), 10, "tanh")
for opt in ("sgd", "adam"):
    h = packing.make_handle("g1", arch, opt, 0.005, 32, 50, "t", 1)
    m = oracle_from_handle(h)
    od = {"t": oracle_dataset(ds["t"])}
    # oracle gradient of step 1
    x, y, idx, take = O._next_batch(m, od["t"]) if False else (None, None, None, None)
    want, _ = O.oracle_packed_step([m], od)
    packing.packed_step(packing.pack_models([h]), ds)
    W = h.params["g1/L0/W"]; Wr = m.layers[0][0]
    d = np.abs(W - Wr); i = np.unravel_index(np.argmax(d), d.shape)
    print(opt, "max |dW|", d.max(), "at", i, "rel-excess count", int(((d - (1e-4*np.abs(Wr)+1e-6)) > 0).sum()), "of", d.size)
