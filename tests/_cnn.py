"""Helpers for the conv pack parity tests: read device tensors back and check
every kernel against oracle/cnn64.py "teacher-forced" — each layer's oracle
output is computed from the DEVICE's own inputs to that layer, so a kernel is
judged on its own arithmetic, not on the chaotic propagation of bf16 rounding
through an untrained deep net (an fp64 gradient of these nets moves by 15-60 %
under a 1e-3 input perturbation).

Stated bf16 tolerances (elementwise, `ref` = oracle of the same inputs):
  * bf16 activations:            |Δ| <= 2^-7 |ref| + 2e-3 max|ref|   (1-ulp flips)
  * bf16 activation gradients:   |Δ| <= 2^-7 (1 + √n) |ref| + 4e-3 max|ref|, n = the
                                 contributions accumulated in bf16 into that tensor
                                 (n = 1 → 2^-6; DenseNet block buffers take up to 17)
  * fp32 parameter gradients:    |Δ| <= 1e-3 |ref| + 1e-4 max|ref|,  normwise <= 1e-3
                                 (BN dgamma sums g·xhat with heavy cancellation)
  * fp32 logits / loss:          rel 1e-5
  * optimizer update (fp32):     |Δ| <= 2e-6 |w| + 1e-7 + 1e-4 |Δw_ref|
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import cnn64 as O


def dev_tensor(cp, k, name, which, take):
    """member k's tensor `name` (a view reads its slice of the base buffer) as
    NCHW float64"""
    t = cp.members[k].net.tensors[name]
    rows = take * t.h * t.w
    v = cp.tensor(k, name, which, rows).float().cpu().numpy().astype(np.float64)
    v = v.reshape(take, t.h, t.w, t.c)[..., :t.creal]
    return torch.from_numpy(np.ascontiguousarray(v.transpose(0, 3, 1, 2)))


def _check(got, ref, rtol, ftol, what, report):
    got = got.double()
    err = (got - ref).abs()
    scale = ref.abs().max().item()
    bound = rtol * ref.abs() + ftol * scale + 1e-30
    bad = (err > bound)
    frac = bad.double().mean().item()
    report.append((what, float(err.max()), scale, frac))
    assert not bool(bad.any()), (what, float(err.max()), scale, frac)


def spec_of(arch):
    return O.Spec(arch.family, arch.classes, tuple(arch.image), arch.width)


def teacher_forced(cp, k, params_before, x, labels, take, loss_dev, report=None):
    """Per-layer parity of member k's last step.  params_before: member-
    relative {name: array} the step started from; x: the batch [b, C, H, W]."""
    report = [] if report is None else report
    m = cp.members[k]
    spec = spec_of(m.net.arch)
    T = O.params_tensors(params_before)
    vals = {"input": O._rnd(x, True)}
    for name in m.net.tensors:
        if name != "input":
            vals[name] = dev_tensor(cp, k, name, "val", take)
    caches = {}
    for L in spec.layers:
        ref, caches[L["name"]] = O.fwd_op(L, vals, T)
        got = vals[L["y"]]
        if L["kind"] == "conv" and L["out_f32"]:
            _check(got, ref, 1e-5, 1e-6, "fwd " + L["y"], report)
        else:
            _check(got, ref, 2.0 ** -7, 2e-3, "fwd " + L["y"], report)
    logits = vals[spec.logits].reshape(take, -1)
    loss, d, dbias = O.xent(logits, labels, spec.classes)
    assert abs(loss_dev - loss) <= 1e-5 * abs(loss) + 1e-6, (loss_dev, loss)
    gdev = {n: dev_tensor(cp, k, n, "grad", take) for n in m.net.tensors if n != "input"}
    _check(gdev[spec.logits].reshape(take, -1)[:, :spec.classes], d, 2.0 ** -7, 1e-3,
           "dlogits", report)
    pgrads = {spec.layers[-1]["name"] + "/b": dbias}
    contrib = {}   # base tensor -> summed input-gradient contributions (channel space)
    ncontrib = {}

    def add(n, t):
        base, ch0 = n, 0
        if n in spec.views:
            base, ch0, _ = spec.views[n]
        if base not in contrib:
            C, H, W = spec.shapes[base]
            contrib[base] = torch.zeros(take, C, H, W, dtype=torch.float64)
        contrib[base][:, ch0:ch0 + t.shape[1]] += t
        ncontrib[base] = ncontrib.get(base, 0) + 1

    for L in reversed(spec.layers):
        g, c, _ = O.bwd_op(L, gdev[L["y"]], vals, T, caches[L["name"]])
        pgrads.update(g)
        for n, t in c.items():
            add(n, t)
    producer = {L["y"]: L for L in spec.layers}
    for n, ref in contrib.items():
        L = producer.get(n)
        if L is not None and L["kind"] == "conv" and L["bias"] and not L["out_f32"]:
            ref = ref * O._dact(vals[n], L["act"])  # the device folds act' in place (BIAS_ACT_BWD)
        got = gdev[n] if n in gdev else dev_tensor(cp, k, n, "grad", take)
        _check(got, ref, 2.0 ** -7 * (1 + ncontrib[n] ** 0.5), 4e-3, "grad " + n, report)
    for p in m.net.params:
        got = torch.from_numpy(cp.grad_of(k, p.name))
        ref = pgrads[p.name]
        nrm = float((got - ref).norm() / max(float(ref.norm()), 1e-30))
        assert nrm <= 1e-3 or float(ref.abs().max()) < 1e-9, (p.name, nrm)
        _check(got, ref, 1e-3, 1e-4, "dparam " + p.name, report)
    return report


def check_update(cp, k, kind, lr, wd, step, before, slots_before):
    """The device's new masters / slots == the fp32 optimizer applied to the
    device's own gradients (engine.py:295-326)."""
    m = cp.members[k]
    grads = {p.name: cp.grad_of(k, p.name) for p in m.net.params}
    P, S = O.apply_update(kind, lr, wd, step, before, grads, slots_before, mirror=True)
    params, slots, st, _ = cp.get_member_state(k)
    assert st == step + 1
    for p in m.net.params:
        full = f"{m.model_id}/{p.name}"
        got = params[full]
        ref = P[p.name]
        dw = np.abs(ref - np.asarray(before[p.name], np.float32).astype(np.float64))
        bound = 2e-6 * np.abs(ref) + 1e-7 + 1e-4 * dw
        assert np.all(np.abs(got - ref) <= bound), (p.name, float(np.abs(got - ref).max()))
