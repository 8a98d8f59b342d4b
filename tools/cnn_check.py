"""Diagnostic: one conv packed step on the GPU vs the fp64 oracle (per-tensor errors).

    python tools/cnn_check.py [family] [K] [batch] [image]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import cnn64 as O  # noqa: E402
from paper_2002_02885_b200 import cnn, data, packing  # noqa: E402


def main():
    fam = sys.argv[1] if len(sys.argv) > 1 else "lenet5"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    b = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    img = int(sys.argv[4]) if len(sys.argv) > 4 else 32
    width = 0.5 if fam == "mobilenetv2" else 1.0
    arch = cnn.ConvArch(fam, 10, (3, img, img), width)
    ds = data.synth_dataset(512, 3 * img * img, 10, seed=1, spread=0.5)
    opts = ["sgd", "momentum", "adam", "adagrad"]
    hs = [packing.make_handle(f"m{i}", arch, opts[i % 4], 0.05 / (i + 1), b, 10, "train", 0)
          for i in range(K)]
    init = [{k: v.copy() for k, v in h.params.items()} for h in hs]
    packed = packing.dedup_inputs(packing.pack_models(hs))
    t0 = time.time()
    losses = packing.packed_step(packed, {"train": ds})
    torch.cuda.synchronize()
    print("first step wall", time.time() - t0, "losses", losses, packed.last_step_stats)
    cp = packed._cp
    spec = O.Spec(fam, 10, (3, img, img), width)
    perm = packing.epoch_permutation(ds.dataset_id, ds.n, 0)
    rows = perm[:b]
    x = O.batch_images(ds.features, (3, img, img), rows)
    y = torch.from_numpy(ds.labels[rows].astype(np.int64))
    worst = 0.0
    for k, h in enumerate(hs):
        p0 = {n.split("/", 1)[1]: v for n, v in init[k].items()}
        tr = {}
        loss, grads, _ = O.forward_backward(spec, p0, x, y, mirror=True, trace=tr)
        A = cp.acts[k]
        for name, t in h.net.tensors.items():
            if name == "input" or name not in tr:
                continue
            dv = A["val"][name].float().cpu().numpy().reshape(b, t.h, t.w, t.c)[..., :t.creal]
            ov = tr[name].permute(0, 2, 3, 1).numpy()
            e = np.linalg.norm(dv - ov) / max(np.linalg.norm(ov), 1e-30)
            if e > 1e-2 or k == 0 and name == h.net.logits:
                print(f"   fwd {name:10s} rel {e:.2e}")
        loss64, grads64, _ = O.forward_backward(spec, p0, x, y, mirror=False)
        print(f"member {k}: loss dev {losses[h.model_id]:.6f} oracle(mirror) {loss:.6f} "
              f"oracle(fp64) {loss64:.6f}")
        for p in h.net.params:
            g = cp.grad_of(k, p.name)
            ref = grads[p.name]
            ref64 = grads64[p.name]
            e = np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30)
            e64 = np.linalg.norm(g - ref64) / max(np.linalg.norm(ref64), 1e-30)
            worst = max(worst, e)
            if e > 1e-3 or p.name in ("L0/W",) or p is h.net.params[-1]:
                print(f"   {p.name:12s} {str(p.shape):22s} rel(mirror) {e:.2e} rel(fp64) {e64:.2e}"
                      f"  |g| {np.linalg.norm(ref):.3e}")
    print("worst normwise grad error vs mirrored oracle:", worst)
    # timing
    st = cp.stream.cuda_stream
    prog = next(iter(cp._progs.values()))
    for _ in range(3):
        prog.run(st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record(cp.stream)
    for _ in range(n):
        prog.run(st)
    e1.record(cp.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"step {ms:.3f} ms  launches {prog.launches}  samples/s x K {K * b / ms * 1e3:.0f}")
    prof = prog.profile(st)
    names = _KN = {v: k for k, v in cnn.CNN.items()}
    agg = {}
    for kind, t in zip(prog.kinds, prof):
        agg[names[kind]] = agg.get(names[kind], 0.0) + t
    for kname, t in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"   {kname:14s} {t:8.3f} ms")


if __name__ == "__main__":
    main()
