"""Host-side cost of one pipelined step, piece by piece (no profiler)."""
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
    t0 = time.perf_counter(); n = len(packing.packed_run(packed, datasets, 2000)); dt = time.perf_counter() - t0
    print(f"{mode}: packed_run {dt / n * 1e6:.1f} us/step")
    # host pieces of one step, device drained (synchronous)
    acc = dict(active=0, plan=0, launch=0, wait=0, apply=0)
    N = 500
    for _ in range(N):
        t = time.perf_counter_ns(); act = packing._active_members(packed, datasets, False)
        t1 = time.perf_counter_ns(); plan = packing._plan_step(packed, act, datasets, None, None)
        t2 = time.perf_counter_ns(); tk = plan.dpack.step_async()
        t3 = time.perf_counter_ns(); r = plan.dpack.wait(tk)
        t4 = time.perf_counter_ns(); packing._apply_result(packed, act, plan, *r[:3], r[4])
        t5 = time.perf_counter_ns()
        for k, v in zip(acc, (t1 - t, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
            acc[k] += v
    print("  sync step pieces (us):", {k: round(v / N / 1e3, 1) for k, v in acc.items()})
