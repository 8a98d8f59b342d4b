"""Probe: device time of one packed conv step (bench_cnn's timing loop, L2
flushed before every step) for a workload, optionally with a planner knob
overridden.   python tools/exp_step.py config1 [steps] [knob=value ...]
knobs: rpt=<rows per thread of the column reductions (cnn.rows_per_block)>,
       nt=wide (256-wide N tiles for N >= 256), wgnt=<WGRAD N tile for co > 64>"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import bench_cnn  # noqa: E402
from paper_2002_02885_b200 import cnn, data, packing  # noqa: E402

wl_name = sys.argv[1] if len(sys.argv) > 1 else "config1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
knobs = dict(a.split("=") for a in sys.argv[3:])
if "rpt" in knobs:
    rpt = int(knobs["rpt"])
    orig = cnn.rows_per_block
    cnn.rows_per_block = lambda rows, c=8, per_thread=4: orig(rows, c, rpt)

if "async" in knobs:  # conv WGRAD on an async lane (1) or in the chain (0)
    cnn.ASYNC_WGRAD = bool(int(knobs["async"]))
if "dwcp" in knobs:  # depthwise WGRAD channel-pixels per block
    cnn.DW_CHANNEL_PIXELS_PER_BLOCK = int(knobs["dwcp"])
if "nt" in knobs:  # N tile rule: "wide" prefers 256-wide tiles for N >= 256
    if knobs["nt"] == "wide":
        cnn._pick_ntile = lambda n, cap=256: cnn.rup(n, 16) if n <= cap else 256
if "wgnt" in knobs:  # WGRAD N tile for co > 64 (rsc > 64): 128 (default) or 256
    wg = int(knobs["wgnt"])
    orig_wg = cnn._wgrad_cfg

    def _wgcfg(k, rsc, pix, _o=orig_wg, _w=wg):
        nt, sp = _o(k, rsc, pix)
        if k > 64 and rsc > 64:
            base = cnn.cdiv(k, 128) * cnn.cdiv(rsc, _w)
            want = max(1, min(pix // 1024, cnn.cdiv(2 * 148, base)))
            kper = cnn.rup(cnn.cdiv(pix, want), 64)
            return _w, cnn.cdiv(pix, kper)
        return nt, sp
    cnn._wgrad_cfg = _wgcfg
wl = bench_cnn.WORKLOADS[wl_name]
K, b = wl["K"], wl["batch"]
c, h, w = wl["image"]
ds = data.synth_dataset(wl["n"], c * h * w, wl["classes"], seed=0, spread=1.0)
datasets = {"train": ds}
_, hs = bench_cnn._handles(wl, packing, cnn)
packed = packing.dedup_inputs(packing.pack_models(hs))
for _ in range(3):
    packing.packed_step(packed, datasets)
cp = packed._cp
prog = [p for key, p in cp._progs.items() if key[0] == tuple([b] * K)][0]
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
st = cp.stream
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
      for _ in range(steps)]
for i in range(steps):
    with torch.cuda.stream(st):
        flush.fill_(1.0)
        torch.cuda._sleep(100_000)
    ev[i][0].record(st)
    prog.run(st.cuda_stream)
    ev[i][1].record(st)
torch.cuda.synchronize()
ms = [a.elapsed_time(z) for a, z in ev]
print(f"{wl_name} {knobs} launches {prog.launches}: median {statistics.median(ms):.3f} ms  "
      f"min {min(ms):.3f}  mean {statistics.mean(ms):.3f}", flush=True)
