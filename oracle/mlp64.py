"""ORACLE (test infrastructure only): float64 CPU restatement of the pack path.

Each function names the reference lines it restates; paths are relative to
`/root/reference/pkg/src/packtrain/`.  Layers are held as plain lists of
(W, b) numpy pairs instead of the reference's node graph, but the arithmetic,
the seeding and the cursor/grouping rules are the reference's.

This module is the checker for the CUDA path and the timed CPU baseline
(`bench.py --impl reference`, `cpu_baseline` key).  The product package
never imports it.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

# engine.py:14-22
LEAKY = 0.01
MOM = 0.9
B1, B2, ADAM_EPS = 0.9, 0.999, 1e-8
ADAGRAD_EPS = 1e-10
ACTIVATIONS = ("sigmoid", "leaky_relu", "tanh", "relu")
OPTIMIZERS = ("sgd", "momentum", "adam", "adagrad")


class OracleValueError(Exception):
    """Non-finite forward value (engine.py:233-235)."""


class OracleGradError(Exception):
    """Non-finite gradient (engine.py:297-299)."""

    def __init__(self, param):
        self.param = param
        super().__init__(param)


# ----------------------------------------------------------------- seeding --

def seeded_rng(text: str) -> np.random.Generator:
    """sha256(text)[:8] little-endian → PCG64 (engine.py:157-159, data.py:124-128)."""
    seed = int.from_bytes(hashlib.sha256(text.encode()).digest()[:8], "little")
    return np.random.default_rng(seed)


def synth_blobs(n, d, classes, seed, spread=4.0):
    """Gaussian blobs; returns (dataset_id, features f64 [n,d], labels i64 [n]).

    Same generator call order as data.py:46-49; id format data.py:51."""
    g = np.random.default_rng(seed)
    centers = g.normal(scale=spread, size=(classes, d))
    labels = g.integers(0, classes, size=n)
    feats = centers[labels] + g.normal(size=(n, d))
    return f"synth-{n}x{d}c{classes}s{seed}", feats, labels.astype(np.int64)


def epoch_order(dataset_id: str, n: int, epoch: int) -> np.ndarray:
    """Per-epoch permutation (data.py:124-128)."""
    return seeded_rng(f"{dataset_id}|epoch{epoch}").permutation(n)


def xavier_layers(member_id: str, dims, seed: int):
    """Xavier-uniform W, zero b per affine layer (engine.py:162-177)."""
    out = []
    for i in range(len(dims) - 1):
        fi, fo = int(dims[i]), int(dims[i + 1])
        lim = np.sqrt(6.0 / (fi + fo))
        w = seeded_rng(f"{member_id}|{i}|{seed}").uniform(-lim, lim, size=(fi, fo))
        out.append([w, np.zeros(fo)])
    return out


# ------------------------------------------------------------- arithmetic --

def _act(kind, z):
    """engine.py:202-210."""
    if kind == "sigmoid":
        return 1.0 / (1.0 + np.exp(-z))
    if kind == "tanh":
        return np.tanh(z)
    if kind == "relu":
        return np.maximum(z, 0.0)
    if kind == "leaky_relu":
        return np.where(z >= 0, z, LEAKY * z)
    raise ValueError(kind)


def _act_grad(kind, z, a, d):
    """engine.py:274-290 (relu keys on pre-activation > 0, leaky on >= 0)."""
    if kind == "sigmoid":
        return d * a * (1.0 - a)
    if kind == "tanh":
        return d * (1.0 - a * a)
    if kind == "relu":
        return d * (z > 0)
    if kind == "leaky_relu":
        return d * np.where(z >= 0, 1.0, LEAKY)
    raise ValueError(kind)


def member_forward_loss(layers, act, x, y, n_valid=None, check=True):
    """Forward of one member's MLP + softmax-xent head (engine.py:180-238).

    Returns (loss, cache) where cache holds the per-layer inputs, pre- and
    post-activations and the softmax probabilities for the backward pass.
    `n_valid` masks trailing pad rows (engine.py:217, :224-225)."""
    x = np.asarray(x, dtype=np.float64)
    rows = x.shape[0]
    nv = rows if n_valid is None else int(n_valid)
    names = []

    def _chk(v, name):
        if check and not np.all(np.isfinite(v)):
            raise OracleValueError(name)

    _chk(x, "in")
    ins, pre, post = [], [], []
    h = x
    last = len(layers) - 1
    for i, (w, b) in enumerate(layers):
        ins.append(h)
        z = h @ w + b
        _chk(z, f"aff{i}")
        pre.append(z)
        if i < last:
            h = _act(act, z)
            _chk(h, f"act{i}")
        else:
            h = z
        post.append(h)
    logits = h
    zz = logits - logits.max(axis=1, keepdims=True)
    ez = np.exp(zz)
    s = ez.sum(axis=1, keepdims=True)
    p = ez / s
    logp = zz - np.log(s)
    y = np.asarray(y).astype(np.int64)
    loss = -logp[np.arange(nv), y[:nv]].mean() if nv else 0.0
    _chk(loss, "loss")
    del names
    return float(loss), {"ins": ins, "pre": pre, "post": post, "p": p,
                         "y": y, "nv": nv}


def member_backward(layers, act, cache, scales=None):
    """Backward of the summed head (engine.py:241-292); returns [(dW, db)].
    scales (test tolerance support): receives [(|x|ᵀ|d|, Σ|d|)] per layer, the
    magnitude an fp32 GEMM's rounding error of each gradient element scales with."""
    p, y, nv = cache["p"], cache["y"], cache["nv"]
    d = np.zeros_like(p)
    if nv:
        d[:nv] = p[:nv]
        d[np.arange(nv), y[:nv]] -= 1.0
        d[:nv] /= nv
    grads = [None] * len(layers)
    for i in range(len(layers) - 1, -1, -1):
        w, _ = layers[i]
        x_in = cache["ins"][i]
        grads[i] = (x_in.T @ d, d.sum(axis=0))
        if scales is not None:
            scales.insert(0, (np.abs(x_in).T @ np.abs(d), np.abs(d).sum(axis=0)))
        if i == 0:
            break
        da = d @ w.T
        d = _act_grad(act, cache["pre"][i - 1], cache["post"][i - 1], da)
    return grads


def forward_backward(layers, act, x, y, n_valid=None):
    loss, cache = member_forward_loss(layers, act, x, y, n_valid)
    return loss, member_backward(layers, act, cache), cache


def grad_order(n_layers):
    """Parameter names in the reference's grads-dict order: the backward walk
    visits the last affine first (engine.py:251, :270-271)."""
    out = []
    for i in range(n_layers - 1, -1, -1):
        out += [(i, "W"), (i, "b")]
    return out


def optimizer_step(kind, lr, t_prev, layers, slots, grads, weight_decay=0.0):
    """In-place update of one member (engine.py:295-326).

    `slots` maps (layer, 'W'|'b') -> {slot_name: array}; created lazily as
    zeros (engine.py:92-96).  Raises OracleGradError before mutating anything
    if a gradient is non-finite (engine.py:297-299).  Returns t_prev + 1.
    `weight_decay` is the coupled-L2 extension (0 = reference semantics)."""
    order = grad_order(len(layers))
    for li, which in order:
        g = grads[li][0 if which == "W" else 1]
        if not np.all(np.isfinite(g)):
            raise OracleGradError((li, which))
    t = t_prev + 1
    for li, which in order:
        k = 0 if which == "W" else 1
        w = layers[li][k]
        g = grads[li][k]
        if weight_decay:
            g = g + weight_decay * w
        st = slots.setdefault((li, which), {})
        if kind == "sgd":
            w -= lr * g
        elif kind == "momentum":
            v = st.setdefault("velocity", np.zeros_like(w))
            v *= MOM
            v += g
            w -= lr * v
        elif kind == "adagrad":
            a = st.setdefault("accum", np.zeros_like(w))
            a += g * g
            w -= lr * g / (np.sqrt(a) + ADAGRAD_EPS)
        elif kind == "adam":
            m = st.setdefault("m", np.zeros_like(w))
            v = st.setdefault("v", np.zeros_like(w))
            m *= B1
            m += (1.0 - B1) * g
            v *= B2
            v += (1.0 - B2) * g * g
            mh = m / (1.0 - B1 ** t)
            vh = v / (1.0 - B2 ** t)
            w -= lr * mh / (np.sqrt(vh) + ADAM_EPS)
        else:
            raise ValueError(kind)
    return t


# ------------------------------------------------------------ pack layer --

@dataclass
class OracleDataset:
    dataset_id: str
    features: np.ndarray
    labels: np.ndarray

    @property
    def n(self):
        return len(self.features)


@dataclass
class OracleMember:
    """One packed member: params, optimizer state and data cursor
    (packing.py:40-66)."""
    model_id: str
    dims: tuple
    act: str
    opt: str
    lr: float
    batch: int
    target_steps: int
    binding: str
    layers: list
    slots: dict = field(default_factory=dict)
    t: int = 0
    steps_done: int = 0
    epoch: int = 0
    pos: int = 0
    samples_used: np.ndarray | None = None
    weight_decay: float = 0.0

    @classmethod
    def make(cls, model_id, dims, act, opt, lr, batch, target_steps, binding,
             seed, weight_decay=0.0):
        return cls(model_id, tuple(int(d) for d in dims), act, opt, float(lr),
                   int(batch), int(target_steps), binding,
                   xavier_layers(model_id, dims, seed),
                   weight_decay=weight_decay)

    @property
    def finished(self):
        return self.steps_done >= self.target_steps

    def _ensure_epoch(self, n):
        if self.samples_used is None:
            self.pos = 0
            self.samples_used = np.zeros(n, dtype=np.int64)

    def roll(self, n):
        """packing.py:175-182."""
        self._ensure_epoch(n)
        if self.pos >= n:
            self.epoch += 1
            self.pos = 0
            self.samples_used = np.zeros(n, dtype=np.int64)

    def flat_params(self):
        return np.concatenate([np.concatenate([w.ravel(), b.ravel()])
                               for w, b in self.layers])


def _next_batch(m: OracleMember, ds: OracleDataset):
    """packing.py:161-172 → data.py:131-136 (permutation recomputed per call,
    as the reference does)."""
    m._ensure_epoch(ds.n)
    take = min(m.batch, ds.n - m.pos)
    perm = epoch_order(ds.dataset_id, ds.n, m.epoch)
    idx = perm[m.pos:m.pos + take]
    return ds.features[idx], ds.labels[idx], idx, take


def oracle_packed_step(members, datasets, share_inputs=True,
                       stop_at_epoch_end=False, grads_out=None):
    """One synchronized packed step (packing.py:185-264).

    Pads each input group to the driver batch and masks the pad rows exactly
    as the reference does; returns ({model_id: loss}, stats)."""
    active = [m for m in members if not m.finished]
    if not stop_at_epoch_end:
        for m in active:
            m.roll(datasets[m.binding].n)
    else:
        for m in active:
            m._ensure_epoch(datasets[m.binding].n)
        active = [m for m in active if m.pos < datasets[m.binding].n]
    if not active:
        raise StopIteration("replan")
    driver = max(m.batch for m in active)
    groups = {}
    for m in active:
        groups.setdefault((m.binding, m.epoch, m.pos, m.batch), []).append(m)
    feeds, takes, physical = {}, {}, 0
    for key in sorted(groups):
        grp = groups[key]
        x, y, idx, take = _next_batch(grp[0], datasets[grp[0].binding])
        xp = np.zeros((driver, x.shape[1]))
        xp[:take] = x
        yp = np.zeros(driver, dtype=np.int64)
        yp[:take] = y
        physical += 1 if share_inputs else len(grp)
        for m in grp:
            feeds[m.model_id] = (xp, yp, take)
            takes[m.model_id] = (idx, take)
    # forward of every member first (the fused graph checks node by node in
    # member order, engine.py:189-235), then backward, then the update loop
    caches = {}
    losses = {}
    for m in active:
        xp, yp, take = feeds[m.model_id]
        loss, cache = member_forward_loss(m.layers, m.act, xp, yp, take)
        caches[m.model_id] = cache
        losses[m.model_id] = loss
    grads = {}
    for m in active:
        sc = [] if grads_out is not None else None
        grads[m.model_id] = member_backward(m.layers, m.act, caches[m.model_id], sc)
        if grads_out is not None:
            grads_out[m.model_id] = (grads[m.model_id], sc)
    for m in active:
        m.t = optimizer_step(m.opt, m.lr, m.t, m.layers, m.slots,
                             grads[m.model_id], m.weight_decay)
        idx, take = takes[m.model_id]
        m.steps_done += 1
        m.pos += take
        m.samples_used[idx] += 1
    stats = {"physical_inputs": physical, "groups": len(groups),
             "driver_batch": driver}
    return losses, stats


def oracle_standalone_step(m: OracleMember, datasets):
    """packing.py:267-282."""
    ds = datasets[m.binding]
    m.roll(ds.n)
    x, y, idx, take = _next_batch(m, ds)
    loss, grads, _ = forward_backward(m.layers, m.act, x, y)
    m.t = optimizer_step(m.opt, m.lr, m.t, m.layers, m.slots, grads,
                         m.weight_decay)
    m.steps_done += 1
    m.pos += take
    m.samples_used[idx] += 1
    return loss
