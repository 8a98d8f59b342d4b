"""One un-graphed conv pack step of a bench workload (for ncu):
    ncu ... python tools/cnn_profile_step.py config1 [K]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2002_02885_b200 import cnn, data, packing  # noqa: E402
from tools import bench_cnn  # noqa: E402

wl = dict(bench_cnn.WORKLOADS[sys.argv[1]])
K = int(sys.argv[2]) if len(sys.argv) > 2 else wl["K"]
c, h, w = wl["image"]
ds = data.synth_dataset(wl["n"], c * h * w, wl["classes"], seed=0, spread=1.0)
arch, hs = bench_cnn._handles(wl, packing, cnn, K=K)
packed = packing.dedup_inputs(packing.pack_models(hs))
packing.packed_step(packed, {"train": ds})   # builds + runs the program once (graph)
cp = packed._cp
prog = next(iter(cp._progs.values()))
torch.cuda.synchronize()
prog.run(cp.stream.cuda_stream, graph=False)  # the profiled step: one launch per op
torch.cuda.synchronize()
print("ok", prog.launches)
