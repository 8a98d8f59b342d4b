"""float64 CPU restatement of the conv pack step — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module; the product package never does.

Parity status: UNPINNED BY THE REFERENCE for the conv layers themselves.  The
reference engine has no conv, batch norm, pooling, ReLU6 or weight decay
(/root/reference/SPEC.md:15, :90, :100); its CNNs exist only as simulator
profiles.  What the reference does define is restated from it:
  * Xavier-uniform init, draw per (member, layer, seed) from
    sha256("{member}|{layer}|{seed}")[:8] LE → PCG64   (pt/engine.py:157-177)
  * softmax cross-entropy, mean over the member's valid rows (pt/engine.py:211-230),
    dlogits = (p - onehot) / n_valid (pt/engine.py:252-264)
  * SGD / Momentum(0.9) / Adagrad(1e-10) / Adam(0.9, 0.999, 1e-8, bias-corrected)
    (pt/engine.py:295-326), coupled weight decay g += wd·w as the extension
  * batch rows = perm[pos:pos+take] of the epoch permutation (pt/data.py:124-136,
    pt/packing.py:161-172).
The conv-layer semantics (torch conventions: NCHW math, BN with batch
statistics and biased variance for normalisation, unbiased for the running
update, momentum 0.1, eps 1e-5; max pool keeping the FIRST maximal tap) are
stated here and in DESIGN.md; parity for them is self-consistency (packed ==
standalone on the device) plus this restatement.

`mirror=True` rounds to bfloat16 exactly where the device stores bf16 (inputs,
GEMM weights, every activation and activation gradient; logits, BN statistics,
weight gradients and masters stay fp32-class), so device-vs-oracle differences
are only fp32-vs-fp64 accumulation order and the occasional 1-ulp bf16 flip it
causes; `mirror=False` is the plain fp64 reference of the same network.
"""
from __future__ import annotations

import hashlib
import math

import numpy as np
import torch
import torch.nn.functional as F

BN_EPS = 1e-5
BN_MOMENTUM = 0.1


def _rnd(t, on):
    return t.float().bfloat16().double() if on else t


def _rng(member, layer, seed):
    h = hashlib.sha256(f"{member}|{layer}|{seed}".encode()).digest()
    return np.random.default_rng(int.from_bytes(h[:8], "little"))


def _div8(v, divisor=8):
    nv = max(divisor, int(v + divisor / 2) // divisor * divisor)
    return nv + divisor if nv < 0.9 * v else nv


class Spec:
    """Layer list of one conv member, in the device's layer numbering."""

    def __init__(self, family, classes=10, image=(3, 32, 32), width=1.0):
        self.family, self.classes, self.image, self.width = family, classes, image, width
        self.layers = []   # dicts
        self.shapes = {"input": (image[0], image[1], image[2])}   # name -> (C, H, W)
        self.views = {}    # name -> (base, ch0, c): a channel slice of a concat buffer
        self.n = 0
        getattr(self, "_" + family)()

    def buffer(self, c, h, w):
        name = f"B{sum(1 for n in self.shapes if n.startswith('B'))}"
        self.shapes[name] = (c, h, w)
        return name

    def view(self, base, ch0, c):
        bc, h, w = self.shapes[base]
        if ch0 == 0 and c == bc:
            return base
        name = f"{base}[{ch0}:{ch0 + c}]"
        self.shapes[name] = (c, h, w)
        self.views[name] = (base, ch0, c)
        return name

    # builders (same order / numbering as the device planner) -----------------
    def _new(self):
        name = f"L{self.n}"
        self.n += 1
        return name

    def conv(self, x, k, r, stride=1, pad=0, bias=False, act="none", out_f32=False, s=None,
             out=None):
        s = r if s is None else s
        c, h, w = self.shapes[x]
        name = self._new()
        y = out if out is not None else name + ".y"
        self.shapes[y] = (k, (h + 2 * pad - r) // stride + 1, (w + 2 * pad - s) // stride + 1)
        self.layers.append(dict(kind="conv", name=name, x=x, y=y, k=k, c=c, r=r, s=s,
                                stride=stride, pad=pad, bias=bias, act=act, out_f32=out_f32))
        return y

    def bn(self, x, act="none", res=None):
        name = self._new()
        y = name + ".out"
        self.shapes[y] = self.shapes[x]
        self.layers.append(dict(kind="bn", name=name, x=x, y=y, act=act, res=res,
                                c=self.shapes[x][0]))
        return y

    def dw(self, x, r=3, stride=1, pad=1):
        c, h, w = self.shapes[x]
        name = self._new()
        y = name + ".y"
        self.shapes[y] = (c, (h + 2 * pad - r) // stride + 1, (w + 2 * pad - r) // stride + 1)
        self.layers.append(dict(kind="dw", name=name, x=x, y=y, c=c, r=r, stride=stride, pad=pad))
        return y

    def pool(self, kind, x, r, stride, pad=0, out=None):
        c, h, w = self.shapes[x]
        name = self._new()
        y = out if out is not None else name + ".y"
        self.shapes[y] = (c, (h + 2 * pad - r) // stride + 1, (w + 2 * pad - r) // stride + 1)
        self.layers.append(dict(kind=kind, name=name, x=x, y=y, r=r, stride=stride, pad=pad))
        return y

    # families -----------------------------------------------------------------
    def _lenet5(self):
        x = self.conv("input", 6, 5, bias=True, act="relu")
        x = self.pool("maxpool", x, 2, 2)
        x = self.conv(x, 16, 5, bias=True, act="relu")
        x = self.pool("maxpool", x, 2, 2)
        _, h, w = self.shapes[x]
        x = self.conv(x, 120, h, s=w, bias=True, act="relu")
        x = self.conv(x, 84, 1, bias=True, act="relu")
        self.logits = self.conv(x, self.classes, 1, bias=True, out_f32=True)

    def _mobilenetv2(self):
        cfg = ((1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1),
               (6, 160, 3, 2), (6, 320, 1, 1))
        wm = self.width
        cin = _div8(32 * wm)
        last = _div8(1280 * max(1.0, wm))
        x = self.bn(self.conv("input", cin, 3, stride=2, pad=1), "relu6")
        for t, c, n, s in cfg:
            cout = _div8(c * wm)
            for i in range(n):
                st = s if i == 0 else 1
                hdim = int(round(cin * t))
                h = x
                if t != 1:
                    h = self.bn(self.conv(h, hdim, 1), "relu6")
                h = self.bn(self.dw(h, 3, st, 1), "relu6")
                res = x if (st == 1 and cin == cout) else None
                x = self.bn(self.conv(h, cout, 1), "none", res=res)
                cin = cout
        x = self.bn(self.conv(x, last, 1), "relu6")
        x = self.pool("avgpool", x, self.shapes[x][1], 1)
        self.logits = self.conv(x, self.classes, 1, bias=True, out_f32=True)

    def _resnet18(self):
        x = self.bn(self.conv("input", 64, 7, stride=2, pad=3), "relu")
        x = self.pool("maxpool", x, 3, 2, 1)
        cin = 64
        for cout, stride in ((64, 1), (128, 2), (256, 2), (512, 2)):
            for i in range(2):
                st = stride if i == 0 else 1
                h = self.bn(self.conv(x, cout, 3, stride=st, pad=1), "relu")
                y2 = self.conv(h, cout, 3, stride=1, pad=1)
                sc = self.bn(self.conv(x, cout, 1, stride=st), "none") \
                    if (st != 1 or cin != cout) else x
                x = self.bn(y2, "relu", res=sc)
                cin = cout
        x = self.pool("avgpool", x, self.shapes[x][1], 1)
        self.logits = self.conv(x, self.classes, 1, bias=True, out_f32=True)

    def _densenet121(self, blocks=(6, 12, 24, 16), growth=32, bn_size=4, c0=64):
        """torchvision DenseNet-121; torch.cat of the dense layers restated as
        writes into channel slices of one buffer per block."""
        x = self.bn(self.conv("input", c0, 7, stride=2, pad=3), "relu")
        _, h, w = self.shapes[x]
        h, w = (h + 2 - 3) // 2 + 1, (w + 2 - 3) // 2 + 1
        c = c0
        buf = self.buffer(c + blocks[0] * growth, h, w)
        self.pool("maxpool", x, 3, 2, 1, out=self.view(buf, 0, c))
        for bi, nl in enumerate(blocks):
            for _ in range(nl):
                y = self.bn(self.view(buf, 0, c), "relu")
                y = self.conv(y, bn_size * growth, 1)
                y = self.bn(y, "relu")
                self.conv(y, growth, 3, pad=1, out=self.view(buf, c, growth))
                c += growth
            if bi + 1 < len(blocks):
                y = self.conv(self.bn(buf, "relu"), c // 2, 1)
                c //= 2
                h, w = h // 2, w // 2
                nbuf = self.buffer(c + blocks[bi + 1] * growth, h, w)
                self.pool("avgpool", y, 2, 2, out=self.view(nbuf, 0, c))
                buf = nbuf
        x = self.bn(buf, "relu")
        x = self.pool("avgpool", x, self.shapes[x][1], 1)
        self.logits = self.conv(x, self.classes, 1, bias=True, out_f32=True)

    # parameters -----------------------------------------------------------------
    def param_names(self):
        out = []
        for L in self.layers:
            if L["kind"] == "conv":
                out.append(L["name"] + "/W")
                if L["bias"]:
                    out.append(L["name"] + "/b")
            elif L["kind"] == "bn":
                out += [L["name"] + "/gamma", L["name"] + "/beta"]
            elif L["kind"] == "dw":
                out.append(L["name"] + "/W")
        return out

    def init(self, member, seed):
        """engine.py:162-177 extended: Xavier-uniform on (fan_in, fan_out) =
        (C·R·S, K·R·S), zero bias / beta, unit gamma.  Shapes: conv W (K,R,S,C),
        depthwise W (R,S,C)."""
        p = {}
        for li, L in enumerate(self.layers):
            n = L["name"]
            li = int(n[1:])
            if L["kind"] == "conv":
                k, c, r, s = L["k"], L["c"], L["r"], L["s"]
                lim = math.sqrt(6.0 / (c * r * s + k * r * s))
                p[n + "/W"] = _rng(member, li, seed).uniform(-lim, lim, size=(k, r, s, c))
                if L["bias"]:
                    p[n + "/b"] = np.zeros(k)
            elif L["kind"] == "bn":
                p[n + "/gamma"] = np.ones(L["c"])
                p[n + "/beta"] = np.zeros(L["c"])
            elif L["kind"] == "dw":
                r = L["r"]
                lim = math.sqrt(6.0 / (2 * r * r))
                p[n + "/W"] = _rng(member, li, seed).uniform(-lim, lim, size=(r, r, L["c"]))
        return p


def _act(y, act):
    if act == "relu":
        return y.clamp_min(0)
    if act == "relu6":
        return y.clamp(0, 6)
    return y


def _dact(out, act):
    if act == "relu":
        return (out > 0).double()
    if act == "relu6":
        return ((out > 0) & (out < 6)).double()
    return torch.ones_like(out)


def _maxpool_arg(x, r, stride, pad):
    """argmax tap (first maximal, scan order r-major) and values of every window."""
    n, c, h, w = x.shape
    xp = F.pad(x, (pad, pad, pad, pad), value=-math.inf)
    u = F.unfold(xp, r, stride=stride)           # [n, c*r*r, L]
    u = u.view(n, c, r * r, -1)
    val, arg = u.max(dim=2)                      # first maximal index
    p = (h + 2 * pad - r) // stride + 1
    q = (w + 2 * pad - r) // stride + 1
    return val.view(n, c, p, q), arg.view(n, c, p, q)


class Store(dict):
    """name -> NCHW tensor, with channel views of concat buffers resolved to
    slices of their base (writes go into the base)."""

    def __init__(self, spec, batch):
        super().__init__()
        self.spec, self.batch = spec, batch

    def _base(self, name):
        base, ch0, c = self.spec.views[name]
        if not dict.__contains__(self, base):
            C, H, W = self.spec.shapes[base]
            dict.__setitem__(self, base, torch.zeros(self.batch, C, H, W, dtype=torch.float64))
        return dict.__getitem__(self, base), ch0, c

    def __getitem__(self, name):
        if name in self.spec.views:
            b, ch0, c = self._base(name)
            return b[:, ch0:ch0 + c]
        return dict.__getitem__(self, name)

    def __setitem__(self, name, value):
        if name in self.spec.views:
            b, ch0, c = self._base(name)
            b[:, ch0:ch0 + c] = value
        else:
            dict.__setitem__(self, name, value)

    def __contains__(self, name):
        if name in self.spec.views:
            return dict.__contains__(self, self.spec.views[name][0])
        return dict.__contains__(self, name)


def fwd_op(L, vals, T, mirror=True, train=True, run_stats=None):
    """Forward of one layer L given input tensors `vals` (NCHW float64) and
    params T (member-relative names → float64 tensors, fp32-valued when
    mirror).  Returns (output, cache)."""
    R = lambda t: _rnd(t, mirror)  # noqa: E731
    kind, n = L["kind"], L["name"]
    xin = vals[L["x"]]
    if kind == "conv":
        W = R(T[n + "/W"]).permute(0, 3, 1, 2)          # (K, C, R, S)
        y = F.conv2d(xin, W, stride=L["stride"], padding=L["pad"])
        if L["bias"]:
            y = y + T[n + "/b"].view(1, -1, 1, 1)
        y = _act(y, L["act"])
        if L["out_f32"]:
            return (y.float().double() if mirror else y), None
        return R(y), None
    if kind == "bn":
        if train:
            mean = xin.mean(dim=(0, 2, 3))
            var = ((xin * xin).mean(dim=(0, 2, 3)) - mean * mean).clamp_min(0)
            m = xin.shape[0] * xin.shape[2] * xin.shape[3]
        else:
            a, bb = run_stats[n]
            mean, var, m = torch.from_numpy(a), torch.from_numpy(bb), None
        rstd = 1.0 / torch.sqrt(var + BN_EPS)
        if mirror:
            mean, rstd = mean.float().double(), rstd.float().double()
        xh = (xin - mean.view(1, -1, 1, 1)) * rstd.view(1, -1, 1, 1)
        y = xh * T[n + "/gamma"].view(1, -1, 1, 1) + T[n + "/beta"].view(1, -1, 1, 1)
        if L["res"]:
            y = y + vals[L["res"]]
        return R(_act(y, L["act"])), (mean, rstd, m, var)
    if kind == "dw":
        W = R(T[n + "/W"]).permute(2, 0, 1).unsqueeze(1)   # (C, 1, R, R)
        return R(F.conv2d(xin, W, stride=L["stride"], padding=L["pad"], groups=L["c"])), None
    if kind == "maxpool":
        v, arg = _maxpool_arg(xin, L["r"], L["stride"], L["pad"])
        return v, arg
    if kind == "avgpool":
        return R(F.avg_pool2d(xin, L["r"], stride=L["stride"], padding=L["pad"])), None
    raise ValueError(kind)


def bwd_op(L, dy, vals, T, cache, mirror=True):
    """Backward of layer L given the gradient `dy` of its output, its forward
    input/output tensors in `vals` and its forward cache.  Returns
    (param grads {name: tensor}, input-gradient contributions {tensor: grad},
    dy after the fused activation backward for bias layers)."""
    R = lambda t: _rnd(t, mirror)  # noqa: E731
    kind, n = L["kind"], L["name"]
    xin = vals[L["x"]]
    grads, contrib = {}, {}
    if kind == "conv":
        if L["bias"] and not L["out_f32"]:
            dy = dy * _dact(vals[L["y"]], L["act"])
            grads[n + "/b"] = dy.sum(dim=(0, 2, 3))
            dy = R(dy)
        W = R(T[n + "/W"]).permute(0, 3, 1, 2)
        gw = torch.nn.grad.conv2d_weight(xin, W.shape, dy, stride=L["stride"], padding=L["pad"])
        grads[n + "/W"] = gw.permute(0, 2, 3, 1)
        if L["x"] != "input":
            contrib[L["x"]] = torch.nn.grad.conv2d_input(xin.shape, W, dy, stride=L["stride"],
                                                         padding=L["pad"])
    elif kind == "bn":
        mean, rstd, m, _ = cache
        g = dy * _dact(vals[L["y"]], L["act"])
        xh = (xin - mean.view(1, -1, 1, 1)) * rstd.view(1, -1, 1, 1)
        sg = g.sum(dim=(0, 2, 3))
        sgx = (g * xh).sum(dim=(0, 2, 3))
        grads[n + "/gamma"] = sgx
        grads[n + "/beta"] = sg
        mg, mgx = sg / m, sgx / m
        if mirror:
            mg, mgx = mg.float().double(), mgx.float().double()
        contrib[L["x"]] = T[n + "/gamma"].view(1, -1, 1, 1) * rstd.view(1, -1, 1, 1) * (
            g - mg.view(1, -1, 1, 1) - xh * mgx.view(1, -1, 1, 1))
        if L["res"]:
            contrib[L["res"]] = g
    elif kind == "dw":
        c = L["c"]
        W = R(T[n + "/W"]).permute(2, 0, 1).unsqueeze(1)
        gw = torch.nn.grad.conv2d_weight(xin, W.shape, dy, stride=L["stride"], padding=L["pad"],
                                         groups=c)
        grads[n + "/W"] = gw.squeeze(1).permute(1, 2, 0)
        contrib[L["x"]] = torch.nn.grad.conv2d_input(xin.shape, W, dy, stride=L["stride"],
                                                     padding=L["pad"], groups=c)
    elif kind in ("maxpool", "avgpool"):
        r, pad = L["r"], L["pad"]
        nb, c, p, q = dy.shape
        h, w = xin.shape[2], xin.shape[3]
        if kind == "maxpool":
            cols = torch.zeros(nb, c, r * r, p * q, dtype=torch.float64)
            cols.scatter_(2, cache.view(nb, c, 1, p * q), dy.reshape(nb, c, 1, p * q))
        else:
            cols = (dy / (r * r)).reshape(nb, c, 1, p * q).expand(nb, c, r * r, p * q)
        dx = F.fold(cols.reshape(nb, c * r * r, p * q), (h + 2 * pad, w + 2 * pad), r,
                    stride=L["stride"])
        contrib[L["x"]] = dx[:, :, pad:pad + h, pad:pad + w]
    return grads, contrib, dy


def xent(z, labels, classes, mirror=True):
    """softmax cross-entropy over fp32 logits z [b, >=classes] (engine.py:211-230)
    and its gradient (engine.py:252-264): (loss, dlogits (bf16-rounded when
    mirror), dbias)."""
    b = z.shape[0]
    z = z[:, :classes]
    zmax = z.max(dim=1, keepdim=True).values
    logp = z - (torch.log(torch.exp(z - zmax).sum(dim=1, keepdim=True)) + zmax)
    loss = float(-logp[torch.arange(b), labels].mean())
    d = torch.exp(logp)
    d[torch.arange(b), labels] -= 1.0
    d = d / b
    return loss, _rnd(d, mirror), d.sum(dim=0)


def params_tensors(params, mirror=True):
    T = {k: torch.from_numpy(np.asarray(v, dtype=np.float64)) for k, v in params.items()}
    return {k: v.float().double() for k, v in T.items()} if mirror else T


def forward_backward(spec: Spec, params: dict, x, labels, mirror=True, run_stats=None,
                     train=True, trace=None):
    """One training forward + backward of one member on batch x [b, C, H, W]
    (float64 torch), labels [b] int64.  params: {layer param name: np array}
    (member-relative names).  Returns (loss, grads {name: np}, new run_stats)."""
    R = lambda t: _rnd(t, mirror)  # noqa: E731
    T = params_tensors(params, mirror)
    vals = Store(spec, x.shape[0])
    vals["input"] = R(x)
    cache = {}
    rs_new = {} if run_stats is None else {k: (a.copy(), b.copy()) for k, (a, b) in
                                           run_stats.items()}
    b = x.shape[0]
    for L in spec.layers:
        y, c = fwd_op(L, vals, T, mirror, train, run_stats)
        vals[L["y"]] = y
        cache[L["name"]] = c
        if L["kind"] == "bn" and train and run_stats is not None:
            mean, _, m, var = c
            a, bb = rs_new.get(L["name"], (np.zeros(L["c"]), np.ones(L["c"])))
            unb = var.numpy() * m / max(m - 1, 1)
            rs_new[L["name"]] = ((1 - BN_MOMENTUM) * a + BN_MOMENTUM * mean.numpy(),
                                 (1 - BN_MOMENTUM) * bb + BN_MOMENTUM * unb)
    if trace is not None:
        trace.update(vals)
    loss, d, dbias = xent(vals[spec.logits].reshape(b, -1), labels, spec.classes, mirror)
    if not train:
        return loss, None, rs_new
    grads = {spec.layers[-1]["name"] + "/b": dbias}
    gv = Store(spec, b)
    gv[spec.logits] = d.view(b, -1, 1, 1)
    for L in reversed(spec.layers):
        if L["y"] not in gv:
            continue
        g, contrib, _ = bwd_op(L, gv[L["y"]], vals, T, cache[L["name"]], mirror)
        grads.update(g)
        for name, t in contrib.items():
            gv[name] = R(t if name not in gv else gv[name] + t)
    if trace is not None:
        trace.update({"grad:" + k: v for k, v in gv.items()})
    return loss, {k: v.numpy().astype(np.float64) for k, v in grads.items()}, rs_new


SLOTS = {"sgd": (), "momentum": ("velocity",), "adagrad": ("accum",), "adam": ("m", "v")}


def apply_update(kind, lr, wd, step, params, grads, slots, mirror=True):
    """engine.py:295-326 (+ coupled weight decay), in fp32 when mirror (the
    device keeps fp32 masters), else fp64.  Returns (params, slots)."""
    dt = np.float32 if mirror else np.float64
    t = step + 1
    P, S = {}, {}
    for name, w0 in params.items():
        w = np.asarray(w0, dtype=dt).copy()
        g = np.asarray(grads[name], dtype=dt)
        if wd:
            g = g + dt(wd) * w
        sl = {k: np.asarray(v, dtype=dt).copy() for k, v in (slots.get(name) or {}).items()}
        lr_ = dt(lr)
        if kind == "sgd":
            w = w - lr_ * g
        elif kind == "momentum":
            v = dt(0.9) * sl.get("velocity", np.zeros_like(w)) + g
            sl["velocity"] = v
            w = w - lr_ * v
        elif kind == "adagrad":
            a = sl.get("accum", np.zeros_like(w)) + g * g
            sl["accum"] = a
            w = w - lr_ * g / (np.sqrt(a) + dt(1e-10))
        else:
            m = dt(0.9) * sl.get("m", np.zeros_like(w)) + dt(0.1) * g
            v = dt(0.999) * sl.get("v", np.zeros_like(w)) + dt(0.001) * (g * g)
            sl["m"], sl["v"] = m, v
            c1, c2 = dt(1.0 - 0.9 ** t), dt(1.0 - 0.999 ** t)
            w = w - lr_ * (m / c1) / (np.sqrt(v / c2) + dt(1e-8))
        P[name] = w.astype(np.float64)
        S[name] = {k: v.astype(np.float64) for k, v in sl.items()}
    return P, S


def batch_images(features, image, rows):
    """dataset rows (NCHW-flattened) → [b, C, H, W] float64 tensor."""
    c, h, w = image
    return torch.from_numpy(np.asarray(features[rows], dtype=np.float64).reshape(-1, c, h, w))
