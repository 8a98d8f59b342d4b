"""Conv-pack workloads of bench.py (BASELINE configs 1-3).

A step = one packed train step of all K conv members over one batch each
(forward, backward, every member's optimizer update): ONE pk_cnn_prog replay.
  value  = K·b / device time of the step (CUDA events on the pack's stream,
           inputs resident in HBM, L2 flushed before every timed step — the
           step's activations are also far larger than L2); max over ranks.
  e2e    = the same metric through the drop-in API, packing.packed_step, with
           the dataset in page-locked HOST memory: every step the GPU gathers
           the batch rows over PCIe (h2d bytes = the batch) and the host reads
           losses + commit verdicts back (d2h), one synchronous step at a time.
  speedup_vs_unpacked = the same members trained one after another as
           one-member packs (the reference's standalone_step) on the same GPU.
"""
from __future__ import annotations

import json
import os
import statistics
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPTS = ("sgd", "momentum", "adam", "adagrad")

WORKLOADS = {
    # configs[1]: K small CNNs on CIFAR-shape 32x32 (the headline: K = 16, b = 128)
    "config1": dict(family="mobilenetv2", width=0.5, image=(3, 32, 32), classes=10, n=4096,
                    batch=128, K=16, sweep=(2, 4, 8, 16),
                    members=[(OPTS[i % 4], 10.0 ** -(1 + i % 4), 0.0) for i in range(16)]),
    "config1_lenet": dict(family="lenet5", width=1.0, image=(3, 32, 32), classes=10, n=4096,
                          batch=128, K=16, sweep=(2, 4, 8, 16),
                          members=[(OPTS[i % 4], 10.0 ** -(1 + i % 4), 0.0)
                                   for i in range(16)]),
    # configs[3]: heterogeneous MobileNetV2 + ResNet-18 + DenseNet-121 on one input stream
    "config3": dict(family="hetero", width=1.0, image=(3, 224, 224), classes=1000, n=256,
                    batch=32, K=3, sweep=(3,),
                    archs=[("mobilenetv2", 1.0), ("resnet18", 1.0), ("densenet121", 1.0)],
                    members=[("momentum", 0.05, 1e-4), ("momentum", 0.1, 1e-4),
                             ("momentum", 0.1, 1e-4)]),
    # configs[2]: K = 4 ResNet-18 variants differing in lr / weight decay, 224², b = 32
    "config2": dict(family="resnet18", width=1.0, image=(3, 224, 224), classes=1000, n=512,
                    batch=32, K=4, sweep=(2, 4),
                    members=[("momentum", lr, wd) for lr, wd in
                             ((0.1, 1e-4), (0.05, 5e-4), (0.02, 1e-3), (0.01, 5e-3))]),
}


def _traffic(workload, kind):
    """measured DRAM bytes per step of a kernel kind (ncu, profiles/ncu_traffic.json,
    tools/traffic_summary.py) or None"""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[workload][kind]
    except Exception:
        return None


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def _arch(wl, cnn, i):
    fam, width = wl["archs"][i] if "archs" in wl else (wl["family"], wl["width"])
    return cnn.ConvArch(fam, wl["classes"], tuple(wl["image"]), width)


def _handles(wl, packing, cnn, K=None, prefix="m"):
    ms = wl["members"][:K or wl["K"]]
    return _arch(wl, cnn, 0), [
        packing.make_handle(f"{prefix}{i}", _arch(wl, cnn, i), o, lr, wl["batch"], 10 ** 9,
                            "train", i, weight_decay=wd) for i, (o, lr, wd) in enumerate(ms)]


# ---------------------------------------------------------------- work model --
def layer_work(net, b):
    """Algorithmic FLOPs (real channel counts) and bytes per kernel kind for ONE
    member-step of batch b: GEMM kinds count 2·M·N·K; the
    HBM-bound kinds count every tensor they must touch once (bf16 activations,
    fp32 params / slots / grads)."""
    fl, by = {}, {}

    def add(d, k, v):
        d[k] = d.get(k, 0) + v

    T = net.tensors
    for op in net.ops:
        if op.kind == "conv":
            tx, ty = T[op.x], T[op.y]
            macs = b * ty.h * ty.w * ty.creal * op.a["r"] * op.a["s"] * tx.creal
            add(fl, "CONV_FPROP", 2 * macs)
            add(fl, "CONV_WGRAD", 2 * macs)
            if op.x != "input":
                add(fl, "CONV_DGRAD", 2 * macs)
        elif op.kind == "bn":
            e = b * T[op.x].h * T[op.x].w * T[op.x].c * 2
            add(by, "BN_STATS", e)
            add(by, "BN_APPLY", e * (3 if op.res else 2))
            add(by, "BN_BWD_REDUCE", 3 * e)
            add(by, "BN_BWD_APPLY", e * (5 if op.res else 4))
        elif op.kind == "dw":
            ex = b * T[op.x].h * T[op.x].w * T[op.x].c * 2
            ey = b * T[op.y].h * T[op.y].w * T[op.y].c * 2
            add(by, "DW_FPROP", ex + ey)
            add(by, "DW_DGRAD", ex + ey)
            add(by, "DW_WGRAD", ex + ey)
            macs = b * T[op.y].h * T[op.y].w * T[op.y].c * op.a["r"] * op.a["s"]
            add(fl, "DW", 6 * macs)
        elif op.kind in ("maxpool", "avgpool"):
            ex = b * T[op.x].h * T[op.x].w * T[op.x].c * 2
            ey = b * T[op.y].h * T[op.y].w * T[op.y].c * 2
            kind = "MAXPOOL" if op.kind == "maxpool" else "AVGPOOL"
            add(by, kind + "_FWD", ex + ey * (1.5 if kind == "MAXPOOL" else 1))
            add(by, kind + "_BWD", ex + ey * (1.5 if kind == "MAXPOOL" else 1))
    return fl, by


def opt_bytes(net, opt):
    P = sum(p.numel for p in net.params)
    slots = {"sgd": 0, "momentum": 1, "adagrad": 1, "adam": 2}[opt]
    w16 = sum(p.numel for p in net.params if p.w16)
    return 4 * P * (3 + 2 * slots) + 2 * w16


# ------------------------------------------------------------------- GPU arm --
def run_b200(args, world, rank, local, Clocks, flush_bytes):
    import torch
    import torch.distributed as dist

    from paper_2002_02885_b200 import cnn, data, packing, runtime

    wl = WORKLOADS[args.workload]
    K, b = wl["K"], wl["batch"]
    c, h, w = wl["image"]
    ds = data.synth_dataset(wl["n"], c * h * w, wl["classes"], seed=rank, spread=1.0)
    datasets = {"train": ds}
    arch, hs = _handles(wl, packing, cnn)
    packed = packing.dedup_inputs(packing.pack_models(hs))
    flush = torch.empty(flush_bytes // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        packing.packed_step(packed, datasets)
    cp = packed._cp
    full = [b] * K
    leads = [0] * K
    dd = next(iter(cp._progs))[2]
    prog = [p for key, p in cp._progs.items() if key[0] == tuple(full)][0]

    def device_ms(cpk, pr, steps):
        """Σ per-step device time of program `pr` on pack `cpk`'s stream, L2 cold."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        st = cpk.stream
        for i in range(steps):
            with torch.cuda.stream(st):
                flush.fill_(1.0)
                torch.cuda._sleep(100_000)
            ev[i][0].record(st)
            pr.run(st.cuda_stream)
            ev[i][1].record(st)
        torch.cuda.synchronize()
        return [a.elapsed_time(z) for a, z in ev]

    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    per = device_ms(cp, prog, args.steps)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    dev_ms = sum(per)

    # per-kind profile: events around every op, un-graphed, a device spin ahead of
    # each op so host enqueue latency is not counted (pk_cnn_prog_profile)
    kinds = {v: k for k, v in cnn.CNN.items()}
    prof = []
    for _ in range(5):
        with torch.cuda.stream(cp.stream):
            flush.fill_(1.0)
        prof.append(prog.profile(cp.stream.cuda_stream))
    op_ms = [statistics.median(p[i] for p in prof) for i in range(len(prog.kinds))]
    by_kind = {}
    for kd, t in zip(prog.kinds, op_ms):
        by_kind[kinds[kd]] = by_kind.get(kinds[kd], 0.0) + t
    top_ops = []
    for i in sorted(range(len(op_ms)), key=lambda i: -op_ms[i])[:12]:
        st = prog._keep[i][0]
        desc = {f: getattr(st, f) for f in ("n", "h", "w", "c", "k", "r", "s", "stride", "rows",
                                             "p", "q") if hasattr(st, f)}
        top_ops.append({"op": i, "kernel": kinds[prog.kinds[i]], "ms": op_ms[i],
                        "problems": prog.sizes[i], "shape": desc})

    # algorithmic work per step, all members
    flops, nbytes = {}, {}
    for hnd in hs:
        f, bb = layer_work(hnd.net, b)
        for k2, v in f.items():
            flops[k2] = flops.get(k2, 0) + v
        for k2, v in bb.items():
            nbytes[k2] = nbytes.get(k2, 0) + v
        nbytes["OPT"] = nbytes.get("OPT", 0) + opt_bytes(hnd.net, hnd.optimizer.kind)
    peaks, peak_kind = _peaks()
    table = []
    for kname, t in sorted(by_kind.items(), key=lambda kv: -kv[1]):
        if kname in flops:
            ach = flops[kname] / (t / 1e3) / 1e12
            table.append({"kernel": kname, "ms": t, "bound": "tensor", "achieved": ach,
                          "unit": "TFLOP/s", "frac": ach / peaks["bf16_tflops"],
                          "flops": flops[kname]})
        elif kname in nbytes:
            ach = nbytes[kname] / (t / 1e3) / 1e9
            table.append({"kernel": kname, "ms": t, "bound": "hbm", "achieved": ach,
                          "unit": "GB/s", "frac": ach / peaks["hbm_gbs"], "bytes": nbytes[kname]})
        else:
            table.append({"kernel": kname, "ms": t})
    top = next(r for r in table if "frac" in r)
    gemm_ms = sum(r["ms"] for r in table if r.get("bound") == "tensor")
    gemm_fl = sum(r["flops"] for r in table if r.get("bound") == "tensor")

    # unpacked: each member alone (one-member pack), same kernels, one after another
    _, solo = _handles(wl, packing, cnn, prefix="m")
    solo_ms = []
    for hnd in solo:
        sp = packing.pack_models([hnd])
        for _ in range(3):
            packing.packed_step(sp, datasets)
        spr = [p for key, p in sp._cp._progs.items() if key[0] == (b,)][0]
        solo_ms.append(statistics.median(device_ms(sp._cp, spr, max(5, args.steps // 4))))
        del sp
    un_ms_step = sum(solo_ms)
    sweep = {}
    for k2 in wl["sweep"]:
        if k2 == K:
            pk_ms = dev_ms / args.steps
        else:
            _, hk = _handles(wl, packing, cnn, K=k2, prefix="s")
            pk = packing.dedup_inputs(packing.pack_models(hk))
            for _ in range(3):
                packing.packed_step(pk, datasets)
            pr = [p for key, p in pk._cp._progs.items() if key[0] == tuple([b] * k2)][0]
            pk_ms = statistics.median(device_ms(pk._cp, pr, max(5, args.steps // 4)))
            del pk
        sweep[str(k2)] = {"packed_ms": pk_ms, "unpacked_ms": sum(solo_ms[:k2]),
                          "speedup": sum(solo_ms[:k2]) / pk_ms}

    # e2e through the public API with host-resident (pinned) inputs
    runtime.set_input_mode("stream")
    for _ in range(3):
        packing.packed_step(packed, datasets)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        packing.packed_step(packed, datasets)
    e2e_s = time.perf_counter() - t0
    runtime.set_input_mode("resident")
    row_bytes = h * w * cnn.rup(c, 8) * 2

    t = torch.tensor([dev_ms, e2e_s * 1e3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, e2e_ms = t.tolist()
    if rank != 0:
        return None
    ms_step = dev_ms / args.steps
    line = {
        "value": world * K * b * args.steps / (dev_ms / 1e3), "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (reference synth_dataset, seeded, spread 1.0; rows read as NCHW "
                "images), random-init weights (the reference's Xavier draw per member)",
        "config": {"workload": args.workload, "family": wl["family"], "width": wl["width"],
                   "archs": wl.get("archs"),
                   "image": list(wl["image"]), "classes": wl["classes"], "members": K,
                   "batch": b, "optimizers": [o for o, _, _ in wl["members"][:K]],
                   "lr": [lr for _, lr, _ in wl["members"][:K]],
                   "weight_decay": [wd for _, _, wd in wl["members"][:K]],
                   "parallelism": f"independent pack per GPU x{world}",
                   "precision": "bf16 activations / GEMM operands, fp32 accumulate, fp32 "
                                "master weights, slots, BN statistics",
                   "l2": "flushed (256 MiB write) before every timed step; per-step "
                         "activations exceed the 126 MB L2"},
        "speedup_vs_unpacked": un_ms_step / ms_step,
        "unpacked_ms_per_step": un_ms_step,
        "speedup_by_K": sweep,
        "e2e": {"value": world * K * b * args.steps / (e2e_ms / 1e3),
                "h2d_bytes_per_step": b * (row_bytes + 8),
                "d2h_bytes_per_step": 16 * K,
                "api": "packing.packed_step one synchronous step at a time, input_mode=stream: "
                       "the dataset lives in page-locked host memory and each step's GATHER "
                       "op pulls its batch rows over PCIe; losses + commit verdicts D2H"},
        "roofline": {"bound": top["bound"], "kernel": top["kernel"], "achieved": top["achieved"],
                     "peak": peaks["bf16_tflops"] if top["bound"] == "tensor" else peaks["hbm_gbs"],
                     "unit": top["unit"], "frac": top["frac"], "traffic": _traffic(args.workload, top["kernel"]),
                     "launch_ms": top["ms"], "peak_source": peak_kind,
                     "gemm_all": {"ms": gemm_ms, "tflops": gemm_fl / (gemm_ms / 1e3) / 1e12,
                                  "frac": gemm_fl / (gemm_ms / 1e3) / 1e12 / peaks["bf16_tflops"]}},
        "kernels": table,
        "top_ops": top_ops,
        "step_flops": sum(flops.values()),
        "gpu_launches": prog.launches * args.steps,
        "clocks": clk,
    }
    return line


# ------------------------------------------------------------- CPU baseline --
def cpu_baseline(workload, seconds=10.0, steps=None):
    """The oracle port (oracle/cnn64.py, torch CPU float64 — the reference has no
    conv path) on this host's cores: one member's train step on a
    batch at a time, bounded to ~`seconds` (or `steps`); value scaled to the
    metric (samples/s x members processed)."""
    import torch

    from oracle import cnn64 as O
    from paper_2002_02885_b200 import data

    wl = WORKLOADS[workload]
    cores = len(os.sched_getaffinity(0))
    torch.set_num_threads(cores)
    c, h, w = wl["image"]
    b = wl["batch"]
    ds = data.synth_dataset(max(b, 64), c * h * w, wl["classes"], seed=0, spread=1.0)
    specs = [O.Spec(*(wl["archs"][i] if "archs" in wl else (wl["family"], wl["width"]))[:1],
                    wl["classes"], tuple(wl["image"]),
                    (wl["archs"][i] if "archs" in wl else (wl["family"], wl["width"]))[1])
             for i in range(wl["K"])]
    rows = np.arange(b) % ds.n
    x = O.batch_images(ds.features, wl["image"], rows)
    y = torch.from_numpy(ds.labels[rows].astype(np.int64))
    done, t0 = 0, time.perf_counter()
    ts = []
    while True:
        i = done % wl["K"]
        o, lr, wd = wl["members"][i]
        spec = specs[i]
        p = spec.init(f"m{i}", i)
        t1 = time.perf_counter()
        _, g, _ = O.forward_backward(spec, p, x, y, mirror=False)
        O.apply_update(o, lr, wd, 0, p, g, {}, mirror=False)
        ts.append(time.perf_counter() - t1)
        done += 1
        if (steps is not None and done >= steps) or (steps is None and
                                                      time.perf_counter() - t0 >= seconds):
            break
    per = statistics.median(ts)
    return {"value": b / per, "unit": "samples/s (x K members)", "cores": cores, "kind": "port",
            "ms_per_member_step": per * 1e3,
            "sample": f"{done} member-steps of {wl['family']} at batch {b} (members cycled), "
                      f"oracle/cnn64.py float64 on torch CPU, {cores} threads; a K-member step "
                      f"costs K member-steps on the CPU"}


# ------------------------------------------------- configs[4]: conv Hyperband --
def run_hyperband(R, n, world, group, cpu_ms_per_sample=None, family="mobilenetv2",
                  width=0.5, seed=0):
    """BASELINE configs[4]: pack-aware Hyperband (tuner.packed_hyperband,
    reference tuner.py:285-337) over the Table-4 space with conv members
    (B200ConvExecutor: MobileNetV2-w0.5 on synthetic CIFAR-shape data, 10 %
    validation split), rung groups sharded over the job's GPUs by
    hyperband_pool (LPT, gloo control plane, no NCCL).  `original` trains every
    config alone (the unpacked Hyperband), `knn` packs similar configs.  Wall
    time is the max over ranks.  The reference has no conv engine, so the CPU
    figure is an estimate: the oracle's measured float64 time per sample times
    the samples the schedule trains."""
    import torch
    import torch.distributed as dist

    from paper_2002_02885_b200 import data, hyperband_pool, tuner

    ds = data.synth_dataset(n, 3 * 32 * 32, 10, seed=seed, spread=1.0)
    # context, programs' code and the kernels' first launches outside the timing
    warm = tuner.B200ConvExecutor(data.synth_dataset(64, 3 * 32 * 32, 10, seed=1, spread=1.0),
                                  family=family, width=width, seed=seed)
    warm.evaluate([tuner.ConfigSpace().config(0), tuner.ConfigSpace().config(1)], 1)
    out, conc = {}, {}
    for mode, strategy in (("serial", "original"), ("serial", "knn"),
                           ("concurrent", "original"), ("concurrent", "knn")):
        ex = tuner.B200ConvExecutor(ds, family=family, width=width, seed=seed)
        # serial: a rank's groups one after another, as the reference evaluates them;
        # concurrent: up to 4 packs at once per GPU (hyperband_pool._run_local)
        ex.concurrent_groups = 1 if mode == "serial" else tuner.B200ConvExecutor.concurrent_groups
        if world > 1:
            dist.barrier(group=group)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res, pool = hyperband_pool.overlapped_hyperband(R, 3, ex, seed, strategy=strategy,
                                                     group=group)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        t = torch.tensor([wall], dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        samples = res.total_epochs * ex.train.n
        (out if mode == "serial" else conc)[strategy] = {
                         "wall_s": float(t.item()), "best_config": res.best_config.config_id,
                         "best_loss": res.best_loss, "epochs": res.total_epochs,
                         "evaluations": len(res.records), "packed_steps": ex.steps,
                         "migrations": pool.migrations, "rounds": pool.rungs,
                         "samples_trained": samples}
    line = {"R": R, "eta": 3, "n": n, "n_train": out["knn"]["samples_trained"]
            // max(1, out["knn"]["epochs"]), "family": family, "width": width,
            "image": [3, 32, 32], "dtype": "bf16", "n_gpus": world,
            "sharding": "independent brackets overlapped; each round's groups LPT over GPUs; member state moves point to point (gloo control plane, no NCCL)",
            "strategies": out,
            "speedup_knn_vs_original": out["original"]["wall_s"] / out["knn"]["wall_s"],
            "concurrent_packs": {
                "packs_per_gpu": tuner.B200ConvExecutor.concurrent_groups,
                "note": "a round's groups as concurrent packs (one host thread + CUDA stream "
                        "each); records and selection identical to the serial run",
                "strategies": conc,
                "speedup_vs_serial_original": out["original"]["wall_s"] / min(
                    v["wall_s"] for v in conc.values())}}
    if cpu_ms_per_sample:
        line["cpu_estimate"] = {
            "original_s": out["original"]["samples_trained"] * cpu_ms_per_sample / 1e3,
            "method": "oracle/cnn64.py float64 torch-CPU time per sample (bench cpu_baseline, "
                      "batch 128) x samples the schedule trains; the reference has no conv "
                      "engine (SPEC.md:15)"}
    return line
