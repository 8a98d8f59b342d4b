"""B200-calibrated step-time model and the training-time distance.

The reference groups configs with a *calibrated simulator* of a 16 GB
P5000-era GPU (device_sim.py:33-138, Eqs. 1-3 of the paper):

    single  = t_fix + b·(t_tx + t_pre) + b·c                         (Eq. 1)
    packed  = t_fix + Σ_groups driver·(t_tx + t_pre) + κ·Σ_k b_k·c    (Eq. 2)
    IMPV    = (seq − packed) / seq                                   (Eq. 3)

and its "traintime" kNN distance is |T(pack{a,b}) − (T(a)+T(b))| / (T(a)+T(b))
(tuner.py:118-127).  Here the same model is *fitted to packed steps measured
on the B200* through the real kernels: `calibrate()` times one-member packs
over batch sizes and K-member packs over K, and least-squares fits t_fix,
the per-sample input cost, a per-optimizer per-sample compute cost and the
packing contention κ.  `make_traintime_metric()` then gives the reference's
distance with B200 numbers, usable as `packed_hyperband(..., metric=...)`.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

OPT_KINDS = ("sgd", "momentum", "adagrad", "adam")


@dataclass(frozen=True)
class DeviceProfile:
    """device_sim.py:33-45 (t_tx and t_pre are folded into one input cost)."""
    memory_capacity: int
    fixed_step_overhead_ms: float
    transfer_ms_per_sample: float
    preprocess_ms_per_sample: float = 0.0
    contention_factor: float = 1.0
    switch_overhead_ms: float = 0.0


@dataclass(frozen=True)
class ModelProfile:
    """device_sim.py:48-54, with the compute cost per optimizer kind (the
    update's HBM passes differ: SGD 1, momentum/adagrad 2, Adam 3)."""
    name: str
    parameter_bytes: int
    activation_bytes_per_sample: int
    compute_ms_per_sample: dict = field(default_factory=dict)  # kind -> ms


@dataclass(frozen=True)
class StepTimeReport:
    t_s_seq_ms: float
    t_s_pack_ms: float

    @property
    def impv(self) -> float:
        return (self.t_s_seq_ms - self.t_s_pack_ms) / self.t_s_seq_ms


def _io(d: DeviceProfile) -> float:
    return d.transfer_ms_per_sample + d.preprocess_ms_per_sample


def single_step_ms(model: ModelProfile, kind: str, batch: int, d: DeviceProfile) -> float:
    """Eq. 1 (device_sim.py:102-106)."""
    return d.fixed_step_overhead_ms + batch * _io(d) + batch * model.compute_ms_per_sample[kind]


def estimate_step_time(members, d: DeviceProfile, input_groups=None) -> StepTimeReport:
    """Eq. 2 (device_sim.py:109-131).  members: (ModelProfile, kind, batch)."""
    if not members:
        raise ValueError("estimate_step_time needs at least one member")
    if input_groups is None:
        input_groups = [[i] for i in range(len(members))]
    t_seq = sum(single_step_ms(m, k, b, d) for m, k, b in members)
    driver = max(b for _, _, b in members)
    io = sum(driver * _io(d) for _ in input_groups)
    compute = sum(b * m.compute_ms_per_sample[k] for m, k, b in members)
    kappa = d.contention_factor if len(members) > 1 else 1.0
    return StepTimeReport(t_seq, d.fixed_step_overhead_ms + io + kappa * compute)


def fit(samples, memory_capacity: int, name="mlp", parameter_bytes=0, act_bytes=0):
    """Fit Eqs. 1-2 to measured steps (closed form on the calibration design).

    samples: [(ms, [(kind, batch), ...], n_groups)] — one packed step each:
    one-member steps over batch sizes (per kind: t = t_fix + b·(io + c_k))
    and n-member same-kind same-batch packs sharing one input group
    (t = t_fix + b·io + κ·n·b·c_k).  Singles give t_fix and io + c_k; the
    packs' intercept separates io, their slope over n gives κ."""
    singles, packs = {}, {}
    for t, ms, ng in samples:
        k0 = ms[0][0]
        if len(ms) == 1:
            singles.setdefault(k0, []).append((ms[0][1], t))
        else:
            packs.setdefault(k0, []).append((len(ms), ms[0][1], t))
    kinds = sorted(singles)
    t_fixes, slopes = [], {}
    for k in kinds:
        b, t = np.array(singles[k], dtype=float).T
        m, c0 = np.polyfit(b, t, 1) if len(b) > 1 else (t[0] / b[0], 0.0)
        slopes[k] = float(m)
        t_fixes.append(float(c0))
    t_fix = max(float(np.mean(t_fixes)), 0.0)
    ios, kappas = [], []
    for k, rows in packs.items():
        n, b, t = np.array(rows, dtype=float).T
        if len(n) > 1:
            s, a0 = np.polyfit(n, t, 1)
            ios.append((a0 - t_fix) / b[0])
            kappas.append((k, s / b[0]))
    io = max(float(np.mean(ios)), 0.0) if ios else 0.0
    c = {k: max(slopes[k] - io, 1e-9) for k in kinds}
    kap = [s / c[k] for k, s in kappas if k in c]
    kappa = max(float(np.mean(kap)), 0.0) if kap else 1.0
    for k in OPT_KINDS:  # kinds never measured borrow a measured cost
        c.setdefault(k, c.get("adam" if k in ("momentum", "adagrad") and "adam" in c
                              else kinds[0]))
    dev = DeviceProfile(memory_capacity, t_fix, io, 0.0, kappa)
    model = ModelProfile(name, parameter_bytes, act_bytes, c)
    return dev, model


def _measure(handles, datasets, steps, packing):
    packed = packing.dedup_inputs(packing.pack_models(handles))
    for _ in range(3):
        packing.packed_step(packed, datasets)
    t0 = time.perf_counter()
    for _ in range(steps):
        packing.packed_step(packed, datasets)
    return (time.perf_counter() - t0) * 1e3 / steps


def calibrate(input_dim=784, hidden=(16,), classes=10, batches=(20, 45, 70),
              kinds=("sgd", "adam"), pack_sizes=(2, 4, 8), steps=50, seed=0, measure=None):
    """Measure packed steps on the current GPU and fit the model.

    `measure(handles, datasets, steps) -> ms per step` defaults to timing
    `packing.packed_step` (host + device, the quantity Hyperband waits on)."""
    from . import data, packing, runtime
    from .device import B200Device, member_device_bytes
    ds = data.synth_dataset(2000, input_dim, classes, seed=seed)
    datasets = {"cal": ds}
    arch = packing.MLPArch(input_dim, tuple(hidden), classes, "relu")
    meas = measure or (lambda hs, dsets, n: _measure(hs, dsets, n, packing))
    samples = []

    def hs(specs):
        return [packing.make_handle(f"cal{i}", arch, k, 1e-3, b, 10 ** 9, "cal", seed)
                for i, (k, b) in enumerate(specs)]

    for k in kinds:
        for b in batches:
            samples.append((meas(hs([(k, b)]), datasets, steps), [(k, b)], 1))
        for n in pack_sizes:
            specs = [(k, batches[len(batches) // 2])] * n
            samples.append((meas(hs(specs), datasets, steps), specs, 1))
    cap = B200Device.detect().memory_capacity
    pbytes = member_device_bytes(arch, "sgd", 1, runtime.default_precision())
    return fit(samples, cap, name=f"mlp{input_dim}-{'-'.join(map(str, hidden))}-{classes}",
               parameter_bytes=pbytes, act_bytes=4 * (sum(hidden) + classes))


def make_traintime_metric(model: ModelProfile, device: DeviceProfile):
    """tuner.py:118-127 with the B200-calibrated model: normalized
    |T(pack{a,b}) − (T(a)+T(b))|; same-batch pairs share one input group."""
    def metric(a, b):
        members = [(model, a.optimizer, a.batch_size), (model, b.optimizer, b.batch_size)]
        groups = [[0, 1]] if a.batch_size == b.batch_size else [[0], [1]]
        r = estimate_step_time(members, device, groups)
        return abs(r.t_s_seq_ms - r.t_s_pack_ms) / r.t_s_seq_ms
    return metric


def epoch_time_ms(model: ModelProfile, kind: str, batch: int, d: DeviceProfile, n: int) -> float:
    """device_sim.py:134-137."""
    return math.ceil(n / batch) * single_step_ms(model, kind, batch, d)
