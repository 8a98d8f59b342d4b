"""Pipelined packed_run time per step (native driver), streamed and resident inputs:
    python tools/pipeline_bench.py [config0|k16|wide16]
(_lib.set_plan_options(run_batch=n) sets the steps per graph launch)."""
import sys, time
sys.path.insert(0, ".")
import bench
from paper_2002_02885_b200 import data, packing, runtime
wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "config0"]
datasets, hs = bench._make(wl, data, packing, seed=0)
for h in hs:
    h.target_steps = 10 ** 9
packed = packing.dedup_inputs(packing.pack_models(hs))
for mode in ("stream", "resident"):
    runtime.set_input_mode(mode)
    packing.packed_run(packed, datasets, 64)
    t0 = time.perf_counter(); n = len(packing.packed_run(packed, datasets, 3000)); dt = time.perf_counter() - t0
    print(f"{sys.argv[1:]} {mode}: packed_run {dt / n * 1e6:.1f} us/step")
