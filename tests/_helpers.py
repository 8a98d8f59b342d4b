"""Shared test helpers: lockstep device-vs-oracle comparison."""
from __future__ import annotations

import numpy as np

from oracle import mlp64 as O

# fp32 device vs float64 oracle, one step from identical state
# (BASELINE north_star: "rel 1e-4 per step"; SURVEY §8c absolute floor 1e-6)
RTOL, ATOL = 1e-4, 1e-6


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def oracle_dataset(ds, round32=True):
    x = f32(ds.features) if round32 else ds.features
    return O.OracleDataset(ds.dataset_id, x, ds.labels)


def oracle_from_handle(h):
    """An OracleMember holding exactly the handle's current device state."""
    params = h.params
    n = len(h.arch.hidden) + 1
    layers = [[params[f"{h.model_id}/L{i}/W"].copy(), params[f"{h.model_id}/L{i}/b"].copy()]
              for i in range(n)]
    slots = {}
    for pname, d in h.optimizer.slots.items():
        i = int(pname.split("/L")[1].split("/")[0])
        which = pname.rsplit("/", 1)[1]
        slots[(i, which)] = {k: v.copy() for k, v in d.items()}
    c = h.cursor
    m = O.OracleMember(h.model_id, h.arch.dims, h.arch.activation, h.optimizer.kind,
                       h.optimizer.learning_rate, h.batch_size, h.target_steps,
                       h.dataset_binding, layers, slots, h.optimizer.step_counter,
                       c.steps_done, c.epoch_index, c.pos,
                       None if c.samples_used is None else c.samples_used.copy(),
                       weight_decay=h.weight_decay)
    return m


# Normalizing optimizers (Adam, Adagrad) step by ~lr·sign(·) of a quantity
# that can sit near zero: Adagrad's g, Adam's first moment m_t = 0.9 m_{t-1} +
# 0.1 g.  When that quantity is a near-cancellation of its terms, rounding
# upstream (a ReLU' flip on a near-zero pre-activation, softmax's absolute
# error) moves the update by a few percent in ANY fp32 engine (the FFMA kernels
# flip 3 of 200,704 W0 elements on the same case the tcgen05 path flips 7).
# Stated tolerance: an element may exceed rel 1e-4 + abs 1e-6 only if
#   (a) its update's sign source cancels at least 10:1 against its terms:
#       |g| <= FLIP_EPS · (|x|ᵀ|d|)  (Adagrad), or
#       |m_t| <= FLIP_EPS · (0.9 |m_{t-1}| + 0.1 (|x|ᵀ|d|))  (Adam), FLIP_EPS = 0.1
#       (measured on the wide16 shape: <= 0.087; a wrong product, a misplaced
#       tile or a wrong bias correction is O(1)),
#   (b) it is off by no more than one maximal Adam step (7·lr), and
#   (c) at most 1e-4 of the tensor's elements (min 2) are off.
# Without the oracle's gradient (grad=None) (b) and (c) apply.
SIGN_FLIP_FRACTION = 1e-4
FLIP_EPS = 0.1


def _assert_param_close(got, ref, rtol, atol, what, kind, lr, grad=None):
    err = np.abs(got - ref) - (rtol * np.abs(ref) + atol)
    if err.max() <= 0:
        return
    if kind in ("adam", "adagrad"):
        bad = err > 0
        allowed = max(2, int(SIGN_FLIP_FRACTION * got.size))
        assert bad.sum() <= allowed, f"{what}: {bad.sum()} elements off (> {allowed})"
        worst = np.abs(got - ref)[bad].max()
        assert worst <= 7 * lr + atol, f"{what}: flip larger than an Adam step ({worst:.3e})"
        if grad is not None:
            src, terms = grad  # the update's sign source and the magnitude of its terms
            ratio = np.abs(src)[bad] / np.maximum(terms[bad], 1e-300)
            assert ratio.max() <= FLIP_EPS, \
                f"{what}: off element whose update source is not a near-cancellation " \
                f"({ratio.max():.3e} > {FLIP_EPS})"
        return
    raise AssertionError(f"{what}: worst excess {err.max():.3e}")


def assert_close_member(h, m, rtol=RTOL, atol=ATOL, what="", grads=None):
    """grads: the oracle step's (grads, scales) of this member (oracle
    oracle_packed_step(grads_out=...)), narrowing the Adam/Adagrad allowance"""
    p = h.params
    kind, lr = h.optimizer.kind, h.optimizer.learning_rate
    for i, (w, b) in enumerate(m.layers):
        for j, (name, ref) in enumerate(((f"{h.model_id}/L{i}/W", w),
                                         (f"{h.model_id}/L{i}/b", b))):
            g = None
            if grads is not None:
                g = (grads[0][i][j], grads[1][i][j])   # (g, |x|ᵀ|d|)
                if kind == "adam":  # sign source: the first moment after the step
                    mt = m.slots[(i, "W" if j == 0 else "b")]["m"]
                    g = (mt, np.abs(mt - 0.1 * g[0]) + 0.1 * g[1])
            _assert_param_close(p[name], ref, rtol, atol, f"{what} {name}", kind, lr, g)
    for (i, which), d in m.slots.items():
        for sname, ref in d.items():
            got = h.optimizer.slots[f"{h.model_id}/L{i}/{which}"][sname]
            err = np.abs(got - ref) - (rtol * np.abs(ref) + atol)
            assert err.max() <= 0, f"{what} slot {i}{which}/{sname}: excess {err.max():.3e}"
    assert h.optimizer.step_counter == m.t
    assert h.cursor.steps_done == m.steps_done
    assert h.cursor.pos == m.pos and h.cursor.epoch_index == m.epoch


def lockstep(packed, datasets, steps, share_inputs=True, packing=None):
    """Run `steps` packed steps; before each, load the oracle with the
    device's exact state and compare one step (losses, params, slots,
    cursors, stats)."""
    odata = {k: oracle_dataset(v) for k, v in datasets.items()}
    for s in range(steps):
        oms = [oracle_from_handle(h) for h in packed.members]
        gout = {}
        try:
            want, wstats = O.oracle_packed_step(oms, odata, share_inputs=share_inputs,
                                                grads_out=gout)
        except StopIteration:
            return
        got = packing.packed_step(packed, datasets)
        assert set(got) == set(want)
        for k in want:
            assert abs(got[k] - want[k]) <= RTOL * abs(want[k]) + ATOL, (s, k, got[k], want[k])
        assert packed.last_step_stats == wstats
        for h, m in zip(packed.members, oms):
            assert_close_member(h, m, what=f"step {s}", grads=gout.get(h.model_id))
