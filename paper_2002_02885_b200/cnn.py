"""Conv pack path: member nets, their HBM layout, and the packed step program.

The reference engine has affine layers only (SPEC.md:15, :90 — MobileNet /
ResNet / DenseNet exist there only as simulator profiles, e.g.
pkg/src/packtrain/profiles/mobilenet.profile).  BASELINE configs 1-4 pack
conv nets, so this module extends the reference's pack primitive
(packing.py:185-264: shared input groups, per-member valid rows, one
optimizer step per member per packed step) to conv members.  Everything the
reference does define is kept: the Xavier-uniform init drawn from
sha256("{member}|{layer}|{seed}") (engine.py:157-177), the four optimizers and
their constants (engine.py:295-326), softmax cross-entropy with a mean over
the member's valid rows (engine.py:211-230), and the rule that a member with a
non-finite gradient is not updated (engine.py:297-299).  Extensions the
reference has no semantics for are defined here and restated by the oracle
(oracle/cnn64.py): batch norm (batch statistics over the member's own rows,
torch's running-statistics rule), ReLU6, pooling, depthwise conv, residual
adds, and coupled weight decay (g += wd·w, the torch.optim rule).

Device layout: activations NHWC bf16, one [rows][C] matrix per
tensor per member (rows = b·H·W, C padded to a multiple of 8); conv weights
fp32 masters [K][kpad] (k = (r, s, c) with c fastest, kpad = roundup(R·S·C, 64))
plus a bf16 mirror the GEMM reads by TMA and, for layers with a data
gradient, a transposed bf16 copy [C][roundup(R·S·K, 64)]; BN statistics,
optimizer slots and gradients fp32.  A packed step is one program of grouped
launches (pk_cnn_prog, include/packtrain_b200.h): each launch covers one layer
of every member, so K identical nets cost the launches of one.  The first
conv of members that share an input group runs as ONE concatenated-N GEMM
(their bf16 weights are laid out contiguously): each im2col tile of the
shared input is staged once and multiplied by all members' filters.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import CNN, CNN_ACT, OPT_CODES

_BN_EPS = 1e-5
_BN_MOMENTUM = 0.1


def rup(a, b):
    return (a + b - 1) // b * b


def cdiv(a, b):
    return (a + b - 1) // b


def input_channels(c):
    """Padded channel count of a network input: 16 for narrow images (the first
    conv then reads 16-channel im2col boxes by TMA, csrc/pk_convgemm.cuh
    a_mode 3), else a multiple of 8."""
    return 16 if c < 16 else rup(c, 8)


# =============================================================================
# Member architectures
# =============================================================================
@dataclass(frozen=True)
class ConvArch:
    """A conv member's architecture (the conv counterpart of MLPArch,
    packing.py:32-38).  `image` is the (C, H, W) shape a dataset row holds in
    NCHW order; `width` is MobileNetV2's width multiplier."""
    family: str                 # lenet5 | mobilenetv2 | resnet18 | densenet121
    classes: int = 10
    image: tuple = (3, 32, 32)
    width: float = 1.0

    @property
    def input_dim(self):
        c, h, w = self.image
        return c * h * w

    @property
    def dims(self):  # for code that reports an arch's shape
        return (self.input_dim, self.family, self.classes)


@dataclass
class TSpec:
    h: int
    w: int
    c: int          # padded channels (multiple of 8)
    creal: int
    base: str | None = None   # a view: channels [ch0, ch0 + c) of tensor `base`
    ch0: int = 0


@dataclass
class PSpec:
    name: str       # member-relative, e.g. "L3/W"
    kind: str       # convw | dww | bias | gamma | beta
    shape: tuple    # logical (host) shape
    dev_shape: tuple
    layer: int
    fan: tuple = ()
    w16: bool = False
    dgrad: bool = False   # conv weight whose layer needs a data gradient (Wt16 copy)
    cin_p: int = 0        # conv weight: padded input channels of the device layout
    im2col: int = 0       # first conv on a narrow input: dense (tap, channel) columns

    @property
    def numel(self):
        return int(np.prod(self.dev_shape))


@dataclass
class Op:
    kind: str       # conv | bn | dw | maxpool | avgpool | head
    name: str
    x: str
    y: str
    a: dict
    params: list = field(default_factory=list)
    res: str | None = None


class Net:
    def __init__(self, arch: ConvArch):
        self.arch = arch
        c, h, w = arch.image
        self.tensors = {"input": TSpec(h, w, input_channels(c), c)}
        self.ops: list[Op] = []
        self.params: list[PSpec] = []
        self.n = 0
        self.logits = None

    @property
    def op_index(self):
        """op name -> position in ops (ops are dataclasses: list.index compares
        every field)"""
        d = self.__dict__.get("_op_index")
        if d is None or len(d) != len(self.ops):
            d = {op.name: i for i, op in enumerate(self.ops)}
            self.__dict__["_op_index"] = d
        return d

    @property
    def signature(self):
        """identical nets (same architecture) share launches in a pack"""
        return (self.arch.family, self.arch.classes, tuple(self.arch.image), self.arch.width)

    # -- builders -------------------------------------------------------------
    def _layer(self):
        name = f"L{self.n}"
        self.n += 1
        return name

    def buffer(self, h, w, c):
        """A tensor no op produces whole: a concat buffer written through views."""
        name = f"B{sum(1 for n in self.tensors if n.startswith('B'))}"
        self.tensors[name] = TSpec(h, w, c, c)
        return name

    def view(self, base, ch0, c):
        """Channels [ch0, ch0 + c) of `base` (row stride = base's channels)."""
        b = self.tensors[base]
        if ch0 == 0 and c == b.c:
            return base
        name = f"{base}[{ch0}:{ch0 + c}]"
        self.tensors[name] = TSpec(b.h, b.w, c, c, base=base, ch0=ch0)
        return name

    def conv(self, x, k, r, s=None, stride=1, pad=0, bias=False, act="none", out_f32=False,
             out=None):
        s = r if s is None else s
        tx = self.tensors[x]
        kp = rup(k, 8)
        p = (tx.h + 2 * pad - r) // stride + 1
        q = (tx.w + 2 * pad - s) // stride + 1
        name = self._layer()
        li = self.n - 1
        kpad = rup(r * s * tx.c, 64)
        cols = 0
        if x == "input" and DENSE_FIRST and tx.creal < tx.c and tx.creal <= 8 \
                and rup(r * s * tx.creal, 8) <= 256 and r * (63 * stride + s) <= 1024:
            # a narrow input's first conv runs as a 1x1 GEMM over dense im2col rows
            # (IM2COL op): K = r·s·creal (rounded to 8) instead of r·s·cp
            cols = rup(r * s * tx.creal, 8)
            kpad = rup(cols, 64)
        W = PSpec(f"{name}/W", "convw", (k, r, s, tx.creal), (kp, kpad), li,
                  fan=(tx.creal * r * s, k * r * s), w16=True, dgrad=(x != "input"),
                  cin_p=tx.c, im2col=cols)
        ps = [W]
        if bias:
            ps.append(PSpec(f"{name}/b", "bias", (k,), (kp,), li))
        self.params += ps
        if out is not None:
            t = self.tensors[out]
            assert (t.h, t.w, t.c) == (p, q, kp), (out, t, p, q, kp)
            y = out
        else:
            y = f"{name}.y"
            self.tensors[y] = TSpec(p, q, kp, k)
        self.ops.append(Op("conv", name, x, y,
                           dict(k=kp, r=r, s=s, stride=stride, pad=pad, act=act,
                                out_f32=out_f32, bias=bias),
                           [pp.name for pp in ps]))
        return y

    def bn(self, x, act="none", res=None):
        tx = self.tensors[x]
        name = self._layer()
        li = self.n - 1
        ps = [PSpec(f"{name}/gamma", "gamma", (tx.creal,), (tx.c,), li),
              PSpec(f"{name}/beta", "beta", (tx.creal,), (tx.c,), li)]
        self.params += ps
        y = f"{name}.out"
        self.tensors[y] = TSpec(tx.h, tx.w, tx.c, tx.creal)
        self.ops.append(Op("bn", name, x, y, dict(act=act), [pp.name for pp in ps], res=res))
        return y

    def dw(self, x, r=3, stride=1, pad=1):
        tx = self.tensors[x]
        name = self._layer()
        li = self.n - 1
        p = (tx.h + 2 * pad - r) // stride + 1
        q = (tx.w + 2 * pad - r) // stride + 1
        W = PSpec(f"{name}/W", "dww", (r, r, tx.creal), (r * r, tx.c), li, fan=(r * r, r * r),
                  w16=True)
        self.params.append(W)
        y = f"{name}.y"
        self.tensors[y] = TSpec(p, q, tx.c, tx.creal)
        self.ops.append(Op("dw", name, x, y, dict(r=r, s=r, stride=stride, pad=pad), [W.name]))
        return y

    def pool(self, kind, x, r, stride, pad=0, out=None):
        tx = self.tensors[x]
        name = self._layer()
        p = (tx.h + 2 * pad - r) // stride + 1
        q = (tx.w + 2 * pad - r) // stride + 1
        if out is not None:
            t = self.tensors[out]
            assert (t.h, t.w, t.c) == (p, q, tx.c), (out, t, p, q)
            y = out
        else:
            y = f"{name}.y"
            self.tensors[y] = TSpec(p, q, tx.c, tx.creal)
        self.ops.append(Op(kind, name, x, y, dict(r=r, s=r, stride=stride, pad=pad)))
        return y

    def head(self, logits):
        self.logits = logits
        self.ops.append(Op("head", "head", logits, "", dict(classes=self.arch.classes)))

    # -- queries ----------------------------------------------------------------
    def param(self, name) -> PSpec:
        for p in self.params:
            if p.name == name:
                return p
        raise KeyError(name)

    @property
    def param_count(self):
        return int(sum(np.prod(p.shape) for p in self.params))


def _make_div(v, divisor=8):
    """torchvision's _make_divisible (MobileNetV2 channel rounding)."""
    new_v = max(divisor, int(v + divisor / 2) // divisor * divisor)
    if new_v < 0.9 * v:
        new_v += divisor
    return new_v


def _lenet5(net: Net):
    x = net.conv("input", 6, 5, bias=True, act="relu")
    x = net.pool("maxpool", x, 2, 2)
    x = net.conv(x, 16, 5, bias=True, act="relu")
    x = net.pool("maxpool", x, 2, 2)
    t = net.tensors[x]
    x = net.conv(x, 120, t.h, t.w, bias=True, act="relu")     # fc1 = conv over the 5x5 map
    x = net.conv(x, 84, 1, bias=True, act="relu")
    x = net.conv(x, net.arch.classes, 1, bias=True, out_f32=True)
    net.head(x)


_MBV2_CFG = ((1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1),
             (6, 160, 3, 2), (6, 320, 1, 1))


def _mobilenetv2(net: Net):
    """torchvision MobileNetV2 topology (ImageNet strides) without dropout."""
    wm = net.arch.width
    cin = _make_div(32 * wm)
    last = _make_div(1280 * max(1.0, wm))
    x = net.bn(net.conv("input", cin, 3, stride=2, pad=1), "relu6")
    for t, c, n, s in _MBV2_CFG:
        cout = _make_div(c * wm)
        for i in range(n):
            stride = s if i == 0 else 1
            hidden = int(round(cin * t))
            h = x
            if t != 1:
                h = net.bn(net.conv(h, hidden, 1), "relu6")
            h = net.bn(net.dw(h, 3, stride, 1), "relu6")
            res = x if (stride == 1 and cin == cout) else None
            x = net.bn(net.conv(h, cout, 1), "none", res=res)
            cin = cout
    x = net.bn(net.conv(x, last, 1), "relu6")
    t = net.tensors[x]
    x = net.pool("avgpool", x, t.h, 1)
    x = net.conv(x, net.arch.classes, 1, bias=True, out_f32=True)
    net.head(x)


def _resnet18(net: Net):
    """torchvision ResNet-18 topology (7x7/2 stem + 3x3/2 max pool, BasicBlocks)."""
    x = net.bn(net.conv("input", 64, 7, stride=2, pad=3), "relu")
    x = net.pool("maxpool", x, 3, 2, 1)
    cin = 64
    for cout, stride in ((64, 1), (128, 2), (256, 2), (512, 2)):
        for i in range(2):
            st = stride if i == 0 else 1
            h = net.bn(net.conv(x, cout, 3, stride=st, pad=1), "relu")
            y2 = net.conv(h, cout, 3, stride=1, pad=1)
            if st != 1 or cin != cout:
                sc = net.bn(net.conv(x, cout, 1, stride=st), "none")
            else:
                sc = x
            x = net.bn(y2, "relu", res=sc)
            cin = cout
    t = net.tensors[x]
    x = net.pool("avgpool", x, t.h, 1)
    x = net.conv(x, net.arch.classes, 1, bias=True, out_f32=True)
    net.head(x)


def _densenet121(net: Net, blocks=(6, 12, 24, 16), growth=32, bn_size=4, c0=64):
    """torchvision DenseNet-121 topology (pre-activation dense layers, 2x2
    average-pool transitions, norm5 + ReLU before the classifier).  The
    concatenations are block buffers: every layer's 3x3 conv writes its
    `growth` channels straight into its slice, and every BN reads a channel
    prefix of the buffer (no copies)."""
    x = net.bn(net.conv("input", c0, 7, stride=2, pad=3), "relu")
    t = net.tensors[x]
    h, w = (t.h + 2 - 3) // 2 + 1, (t.w + 2 - 3) // 2 + 1
    c = c0
    buf = net.buffer(h, w, c + blocks[0] * growth)
    net.pool("maxpool", x, 3, 2, 1, out=net.view(buf, 0, c))
    for bi, nl in enumerate(blocks):
        for _ in range(nl):
            y = net.bn(net.view(buf, 0, c), "relu")
            y = net.conv(y, bn_size * growth, 1)
            y = net.bn(y, "relu")
            net.conv(y, growth, 3, pad=1, out=net.view(buf, c, growth))
            c += growth
        if bi + 1 < len(blocks):
            y = net.bn(buf, "relu")
            y = net.conv(y, c // 2, 1)
            c //= 2
            h, w = h // 2, w // 2
            nbuf = net.buffer(h, w, c + blocks[bi + 1] * growth)
            net.pool("avgpool", y, 2, 2, out=net.view(nbuf, 0, c))
            buf = nbuf
    x = net.bn(buf, "relu")
    x = net.pool("avgpool", x, net.tensors[x].h, 1)
    x = net.conv(x, net.arch.classes, 1, bias=True, out_f32=True)
    net.head(x)


FAMILIES = {"lenet5": _lenet5, "mobilenetv2": _mobilenetv2, "resnet18": _resnet18,
            "densenet121": _densenet121}
_NET_CACHE: dict = {}


def build_net(arch: ConvArch) -> Net:
    if arch not in _NET_CACHE:
        if arch.family not in FAMILIES:
            raise ValueError(f"unknown conv family {arch.family!r}; known: {sorted(FAMILIES)}")
        net = Net(arch)
        FAMILIES[arch.family](net)
        _NET_CACHE[arch] = net
    return _NET_CACHE[arch]


# =============================================================================
# Host state <-> device layout
# =============================================================================
def _param_rng(member: str, layer_index: int, seed: int) -> np.random.Generator:
    """The reference's per-(member, layer, seed) stream (engine.py:157-159)."""
    h = hashlib.sha256(f"{member}|{layer_index}|{seed}".encode()).digest()
    return np.random.default_rng(int.from_bytes(h[:8], "little"))


def init_parameters(net: Net, model_id: str, seed: int) -> dict:
    """Xavier-uniform weights (fan_in = C·R·S, fan_out = K·R·S, the torch conv
    convention), zero bias / beta, unit gamma; the draw for layer i is the
    reference's _param_rng(member, i, seed) (engine.py:162-177)."""
    out = {}
    for p in net.params:
        full = f"{model_id}/{p.name}"
        if p.kind in ("convw", "dww"):
            lim = math.sqrt(6.0 / (p.fan[0] + p.fan[1]))
            out[full] = _param_rng(model_id, p.layer, seed).uniform(-lim, lim, size=p.shape)
        elif p.kind == "gamma":
            out[full] = np.ones(p.shape)
        else:
            out[full] = np.zeros(p.shape)
    return out


def to_dev_layout(p: PSpec, a: np.ndarray) -> np.ndarray:
    """Logical (host) array → padded device layout, float32."""
    out = np.zeros(p.dev_shape, dtype=np.float32)
    a = np.asarray(a, dtype=np.float64)
    if p.kind == "convw" and p.im2col:  # dense (tap, channel) columns
        k, r, s, c = p.shape
        out[:k, :r * s * c] = a.reshape(k, r * s * c)
    elif p.kind == "convw":
        k, r, s, c = p.shape
        kp, kpad = p.dev_shape
        cp = p.cin_p
        v = np.zeros((kp, r, s, cp), dtype=np.float32)
        v[:k, :, :, :c] = a
        out[:, :r * s * cp] = v.reshape(kp, r * s * cp)
    elif p.kind == "dww":
        r, s, c = p.shape
        out[:, :c] = a.reshape(r * s, c)
    else:
        out[:p.shape[0]] = a
    return out


def from_dev_layout(p: PSpec, d: np.ndarray) -> np.ndarray:
    d = np.asarray(d, dtype=np.float32).reshape(p.dev_shape)
    if p.kind == "convw" and p.im2col:
        k, r, s, c = p.shape
        return d[:k, :r * s * c].reshape(k, r, s, c).astype(np.float64)
    if p.kind == "convw":
        k, r, s, c = p.shape
        kp, kpad = p.dev_shape
        cp = p.cin_p
        return d[:, :r * s * cp].reshape(kp, r, s, cp)[:k, :, :, :c].astype(np.float64)
    if p.kind == "dww":
        r, s, c = p.shape
        return d[:, :c].reshape(r, s, c).astype(np.float64)
    return d[:p.shape[0]].astype(np.float64)


def bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 → bfloat16 bit patterns, round to nearest even (= __float2bfloat16_rn)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + 0x7FFF
    out = ((u + r) >> 16).astype(np.uint16)
    nan = np.isnan(np.asarray(a, dtype=np.float32))
    out[nan] = 0x7FC0
    return out


def bf16_round(a: np.ndarray) -> np.ndarray:
    """float → nearest bfloat16 value (as float64)."""
    b = bf16_bits(np.asarray(a, dtype=np.float32)).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


SLOTS = {"sgd": (), "momentum": ("velocity",), "adagrad": ("accum",), "adam": ("m", "v")}


def member_device_bytes(net: Net, optimizer: str, batch: int) -> int:
    """HBM a conv member occupies in a pack (ConvPack allocations): fp32
    masters, gradients and slots, bf16 GEMM mirrors, bf16 activations and
    their gradients for `batch` rows, BN statistics / workspaces (~5 %)."""
    P = sum(p.numel for p in net.params)
    mirrors = sum(2 * p.numel for p in net.params if p.w16) * 2
    act = 0
    for name, t in net.tensors.items():
        if name == "input" or t.base is not None:
            continue
        act += batch * t.h * t.w * t.c * 2 * 2
    op0 = net.ops[0]
    if op0.kind == "conv" and net.param(op0.params[0]).im2col:  # IM2COL rows
        t = net.tensors[op0.y]
        act += batch * t.h * t.w * net.param(op0.params[0]).im2col * 2
    return int((4 * P * (2 + len(SLOTS[optimizer])) + mirrors + act) * 1.05)


# =============================================================================
# Device pack: buffers + programs
# =============================================================================
def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the conv pack path needs a CUDA device (there is no CPU fallback)")
    return torch


def _ptr(t):
    return 0 if t is None else t.data_ptr()


class DeviceConvDataset:
    """A dataset as NHWC bf16 [n][H][W][Cp] (rows are the reference's NCHW
    feature rows, data.py:18-39) plus int64 labels: resident in HBM, or
    (host=True, the streamed e2e mode) in page-locked host memory that the
    step's GATHER op reads over PCIe."""

    def __init__(self, ds, image, device, host=False):
        torch = _torch()
        c, h, w = image
        n = ds.features.shape[0]
        if ds.features.shape[1] != c * h * w:
            raise ValueError(f"dataset rows hold {ds.features.shape[1]} features, "
                             f"the conv members expect {c}x{h}x{w}")
        cp = input_channels(c)
        self.n, self.image, self.cp = n, image, cp
        x = np.zeros((n, h, w, cp), dtype=np.float32)
        x[..., :c] = np.asarray(ds.features, dtype=np.float32).reshape(n, c, h, w).transpose(
            0, 2, 3, 1)
        bits = torch.from_numpy(bf16_bits(x).view(np.int16))
        labels = torch.from_numpy(np.asarray(ds.labels, dtype=np.int64))
        self.host = bool(host)
        if self.host:
            self.x = bits.pin_memory().view(torch.bfloat16)
            self.y = labels.pin_memory()
        else:
            self.x = bits.to(device).view(torch.bfloat16)
            self.y = labels.to(device)
        self.row_bytes = h * w * cp * 2
        self.max_label = int(np.max(ds.labels)) if n else -1


# conv / depthwise WGRAD and split sums on an async lane of the step program
# (single-architecture packs): they overlap the data-gradient chain and join before
# the commit
ASYNC_WGRAD = True

# a narrow input's first conv: dense im2col rows + a 1x1 GEMM (Net.conv, IM2COL op)
DENSE_FIRST = True

# depthwise WGRAD fast path: channel-pixels per partial block (the planner's
# trade-off between per-thread serial latency and partial-record traffic)
DW_CHANNEL_PIXELS_PER_BLOCK = 8192


def _cgp(c):
    """channel groups (of 8) rounded up to a power of two (csrc lanes_of)"""
    g = 1
    while g < max(1, c // 8):
        g *= 2
    return g


def rows_per_block(rows, c=8, per_thread=8):
    """Rows per partial block of a column reduction over `c` channels: a
    function of the member's own shape only (K-invariant).  Each of a block's
    256/pow2(c/8) row lanes sums ~`per_thread` rows; at most 256 blocks (the
    kernels' two-level ticket tree); a multiple of 32."""
    cgp = 1
    while cgp < max(1, c // 8):
        cgp *= 2
    lanes = max(1, 256 // cgp)
    return rup(max(32, lanes * per_thread, cdiv(rows, 256)), 32)


def red_blocks_max(rows, nout):
    """upper bound of cdiv(r, rows_per_block(r)) over r <= rows (ws sizing)"""
    return min(256, cdiv(rows, 32))


def _red_ws(nout_per_blk, nblk, nout):
    """floats for nblk partial records + fp64 group records and totals
    (tree_reduce in csrc/pk_cnn_ops.cuh)."""
    return rup(nout_per_blk * nblk, 2) + 2 * nout * (cdiv(nblk, 16) + 1) + 2


def _pick_ntile(n, cap=256):
    if n <= cap:
        return rup(n, 16)
    return 128 if rup(n, 128) - n <= rup(n, 256) - n else 256


def _stages(ntile, budget=110 * 1024):
    """Pipeline depth for an N tile: the deepest ring within ~110 KB of shared
    memory, so two CTAs share an SM (one's epilogue overlaps the other's
    mainloop)."""
    return max(2, min(6, budget // (16384 + ntile * 128)))


def _wgrad_cfg(k, rsc, pix):
    """(N tile, pixel splits) of a WGRAD problem from the member's own shape.
    co <= 64: the swapped orientation (GEMM M = r·s·c, N = co, N tile 64);
    else M = co, N = r·s·c with 128-wide tiles (two persistent CTAs per SM)."""
    if k <= 64:
        ntile = 64
        base = cdiv(rsc, 128)
    else:
        ntile = 64 if rsc <= 64 else 128
        base = cdiv(k, 128) * cdiv(rsc, ntile)
    want = max(1, min(pix // 1024, cdiv(2 * 148, base)))
    kper = rup(cdiv(pix, want), 64)
    splits = cdiv(pix, kper)
    return ntile, splits


class MemberSpec:
    def __init__(self, model_id, net: Net, batch, optimizer, lr, wd=0.0):
        if optimizer not in OPT_CODES:
            raise ValueError(f"unknown optimizer {optimizer!r}")
        self.model_id, self.net, self.batch = model_id, net, int(batch)
        self.optimizer, self.lr, self.wd = optimizer, float(lr), float(wd)


class _Arena:
    """Bump allocator for a ConvPack's buffers: zeros(*shape, dt=) returns a view
    of a large uint8 chunk (256-byte aligned); finish() zeroes every chunk's
    used bytes with one memset each.  The views are only read after finish()."""

    CHUNK = 64 << 20

    def __init__(self, torch, dev):
        self.torch, self.dev = torch, dev
        self.chunks = []  # [buffer, used bytes]
        self._es = {}

    def zeros(self, *shape, dt=None):
        torch = self.torch
        dt = torch.float32 if dt is None else dt
        n = 1
        for d in shape:
            n *= int(d)
        es = self._es.get(dt)
        if es is None:
            es = self._es[dt] = torch.empty((), dtype=dt).element_size()
        nbytes = n * es
        if not self.chunks or self.chunks[-1][1] + nbytes > self.chunks[-1][0].numel():
            self.chunks.append([torch.empty(max(self.CHUNK, rup(nbytes, 256)),
                                            dtype=torch.uint8, device=self.dev), 0])
        buf, off = self.chunks[-1]
        self.chunks[-1][1] = rup(off + nbytes, 256)
        return buf[off:off + nbytes].view(dt).view(*shape)

    def finish(self):
        for buf, used in self.chunks:
            if used:
                buf[:used].zero_()


class ConvPack:
    """HBM state and step programs of one conv pack.

    members: MemberSpec list; groups: list of member-index lists that share an
    input stream (the reference's input_groups, packing.py:121-128).  Buffers
    are sized for each member's batch_size; programs are built per distinct
    tuple of per-member valid rows ("takes") and cached."""

    def __init__(self, members, groups, device=0):
        torch = _torch()
        self.torch = torch
        self.dev = torch.device("cuda", device)
        self.device = device
        self.members = members
        self.groups = [list(g) for g in groups]
        self.group_of = {}
        for gi, g in enumerate(self.groups):
            for k in g:
                self.group_of[k] = gi
        K = len(members)
        # the pack's buffers come from a few large zeroed chunks (one allocation and
        # one memset per 64 MiB instead of one fill kernel per tensor)
        arena = _Arena(torch, self.dev)
        z = arena.zeros
        self._z = z
        self.state = z(K, 4, dt=torch.int32)        # step, flag, verdict, loss bits
        self.eval_loss = z(K)                        # eval-program loss per member
        # batch image indices, one buffer per member; a step's program reads the
        # buffer of each input group's leader (the first member of the group)
        self.idx = [z(m.batch, dt=torch.int64) for m in members]
        self.params, self.grads, self.slots, self.w16, self.wt16 = [], [], [], [], []
        self.run_stats = []
        self._alloc_params()
        self.acts = []
        for m in members:
            self.acts.append(self._alloc_acts(m))
        arena.finish()
        self._z = lambda *s, dt=torch.float32: torch.zeros(*s, dtype=dt, device=self.dev)  # noqa: E731
        self._arena = arena
        self._progs = {}
        self.staging = {}   # leader -> device batch buffer (streamed inputs)
        # programs are captured / replayed on this stream (graph capture cannot use the
        # legacy default stream); it is ordered after the caller's stream on entry
        self.stream = torch.cuda.Stream(device=self.dev)
        self.lib = _lib.lib()
        self.dataset = None

    # -- allocation ---------------------------------------------------------------
    def _shared_first(self):
        """Per group: the member indices whose first op is a conv on the input
        with one geometry (the concatenated-N first layer)."""
        out = {}
        for gi, g in enumerate(self.groups):
            sig = {}
            for k in g:
                op = self.members[k].net.ops[0]
                if op.kind != "conv" or op.x != "input":
                    continue
                key = (tuple(sorted((kk, v) for kk, v in op.a.items())),
                       self.members[k].batch)
                sig.setdefault(key, []).append(k)
            out[gi] = [ks for ks in sig.values() if len(ks) > 1]
        return out

    def _alloc_params(self):
        torch, z = self.torch, self._z
        K = len(self.members)
        self.first_shared = {}    # member -> (gi, slot index j, member list)
        self.shared_w16, self.shared_bias = {}, {}
        for gi, lists in self._shared_first().items():
            for li, ks in enumerate(lists):
                net = self.members[ks[0]].net
                op = net.ops[0]
                W = net.param(op.params[0])
                kp, kpad = W.dev_shape
                self.shared_w16[(gi, li)] = z(len(ks) * kp, kpad, dt=torch.bfloat16)
                if op.a["bias"]:
                    self.shared_bias[(gi, li)] = z(len(ks) * kp)
                for j, k in enumerate(ks):
                    self.first_shared[k] = (gi, li, j, ks)
        for k, m in enumerate(self.members):
            P, G, S, W16, WT = {}, {}, {}, {}, {}
            slots = SLOTS[m.optimizer]
            first = m.net.ops[0]
            for p in m.net.params:
                shared = k in self.first_shared and p.name in first.params
                gi, li, j, ks = self.first_shared.get(k, (None,) * 4)
                if shared and p.kind == "bias":
                    kp = p.dev_shape[0]
                    P[p.name] = self.shared_bias[(gi, li)][j * kp:(j + 1) * kp]
                else:
                    P[p.name] = z(*p.dev_shape)
                G[p.name] = z(*p.dev_shape)
                S[p.name] = [z(*p.dev_shape) for _ in slots]
                if p.w16:
                    if shared:
                        kp = p.dev_shape[0]
                        W16[p.name] = self.shared_w16[(gi, li)][j * kp:(j + 1) * kp]
                    else:
                        W16[p.name] = z(*p.dev_shape, dt=torch.bfloat16)
                if p.dgrad:
                    kp, kpad = p.dev_shape
                    _, r, s, _c = p.shape
                    cp = p.cin_p
                    WT[p.name] = z(cp, rup(r * s * kp, 64), dt=torch.bfloat16)
            self.params.append(P)
            self.grads.append(G)
            self.slots.append(S)
            self.w16.append(W16)
            self.wt16.append(WT)
            rs = {}
            for op in m.net.ops:
                if op.kind == "bn":
                    c = m.net.tensors[op.x].c
                    rs[op.name] = (z(c), torch.ones(c, dtype=torch.float32, device=self.dev))
            self.run_stats.append(rs)

    def _alloc_acts(self, m: MemberSpec):
        torch, z = self.torch, self._z
        b = m.batch
        net = m.net
        A = {"val": {}, "grad": {}, "ws": {}, "stats": {}, "arg": {}, "split": {}, "dwcnt": {}}
        k = self.members.index(m)
        shared = self.first_shared.get(k)
        for name, t in net.tensors.items():
            if name == "input" or t.base is not None:
                continue  # the network input lives in the group batch buffer; views alias
            rows = b * t.h * t.w
            if name == net.logits:
                A["val"][name] = z(rows, t.c)
                A["grad"][name] = z(rows, t.c, dt=torch.bfloat16)
                continue
            if shared is not None and name == net.ops[0].y:
                continue  # lives in the group's concatenated buffer (below)
            A["val"][name] = z(rows, t.c, dt=torch.bfloat16)
            A["grad"][name] = z(rows, t.c, dt=torch.bfloat16)
        if shared is not None:
            gi, li, j, ks = shared
            key = ("first", gi, li)
            if not hasattr(self, "_first_out"):
                self._first_out, self._first_grad, self._first_split = {}, {}, {}
            t = net.tensors[net.ops[0].y]
            rows = b * t.h * t.w
            if key not in self._first_out:
                self._first_out[key] = z(len(ks), rows, t.c, dt=torch.bfloat16)
                # gradients of the first output and the WGRAD split partials also
                # back to back per member: one concatenated-N WGRAD reads them all
                self._first_grad[key] = z(len(ks), rows, t.c, dt=torch.bfloat16)
                op0 = net.ops[0]
                W0 = net.param(op0.params[0])
                _, sp0 = _wgrad_cfg(t.c, W0.im2col or op0.a["r"] * op0.a["s"] *
                                    net.tensors[op0.x].c, rows)
                if sp0 > 1:
                    self._first_split[key] = z(len(ks), sp0 * W0.numel)
            A["val"][net.ops[0].y] = self._first_out[key][j]
            A["grad"][net.ops[0].y] = self._first_grad[key][j]
        for op in net.ops:
            tx = net.tensors[op.x]
            if op.kind in ("bn",):
                rows = b * tx.h * tx.w
                nb = red_blocks_max(rows, 2 * tx.c)
                A["ws"][op.name] = z(_red_ws(2 * tx.c, nb, 2 * tx.c))
                A["stats"][op.name] = z(4 * tx.c)
            elif op.kind == "conv" and op.a["bias"] and not op.a["out_f32"]:
                ty = net.tensors[op.y]
                rows = b * ty.h * ty.w
                nb = red_blocks_max(rows, ty.c)
                A["ws"][op.name] = z(_red_ws(2 * ty.c, nb, 2 * ty.c))
            elif op.kind == "dw":
                ty = net.tensors[op.y]
                pix = b * ty.h * ty.w
                nout = op.a["r"] * op.a["s"] * tx.c
                # generic path: <= 256 blocks of [r·s·c] records; 3x3 path: per chunk of
                # <= 64 channels, <= 256 / chunks splits of [9][64] records + tree_reduce
                cgb = min(_cgp(tx.c), 8)
                nch = cdiv(tx.c // 8, cgb)
                n9 = 9 * 8 * cgb
                A["ws"][op.name] = z(max(_red_ws(nout, 256, nout),
                                         nch * _red_ws(n9, 256 // nch, n9)))
                A["dwcnt"][op.name] = z(17 * nch, dt=torch.int32)
            elif op.kind == "maxpool":
                ty = net.tensors[op.y]
                A["arg"][op.name] = z(b * ty.h * ty.w * ty.c, dt=torch.uint8)
            if op.kind == "conv":
                ty = net.tensors[op.y]
                W = net.param(op.params[0])
                _, splits = _wgrad_cfg(ty.c, W.im2col or op.a["r"] * op.a["s"] * tx.c,
                                       b * ty.h * ty.w)
                if splits > 1:
                    fkey = ("first",) + shared[:2] if shared is not None and op is net.ops[0] \
                        else None
                    if fkey is not None and fkey in self._first_split:
                        A["split"][op.name] = self._first_split[fkey][shared[2]]
                    else:
                        A["split"][op.name] = z(splits * W.numel)
        A["counters"] = z(17 * (4 * len(net.ops) + 4), dt=torch.int32)
        return A

    # -- state transfer ------------------------------------------------------------
    def set_member_state(self, k, params: dict, slots: dict, step: int, run_stats=None):
        """Upload a member's float64 host state (rounded to float32, the bf16
        mirrors rounded from those) — params {full name: array}, slots
        {full name: {slot: array}}."""
        torch = self.torch
        m = self.members[k]
        for p in m.net.params:
            full = f"{m.model_id}/{p.name}"
            d = to_dev_layout(p, params[full])
            self.params[k][p.name].copy_(torch.from_numpy(d))
            for si, sname in enumerate(SLOTS[m.optimizer]):
                sv = (slots or {}).get(full, {}).get(sname)
                src = to_dev_layout(p, sv) if sv is not None else np.zeros(p.dev_shape, np.float32)
                self.slots[k][p.name][si].copy_(torch.from_numpy(src))
            if p.w16:
                bits = bf16_bits(d)
                self.w16[k][p.name].copy_(torch.from_numpy(bits.view(np.int16)).view(
                    torch.bfloat16))
            if p.dgrad:
                kp, kpad = p.dev_shape
                _, r, s, c = p.shape
                cp = p.cin_p
                wt = np.zeros(tuple(self.wt16[k][p.name].shape), dtype=np.float32)
                v = d[:, :r * s * cp].reshape(kp, r * s, cp).transpose(2, 1, 0)  # [cp][rs][kp]
                wt[:, :r * s * kp] = v.reshape(cp, r * s * kp)
                self.wt16[k][p.name].copy_(torch.from_numpy(bf16_bits(wt).view(np.int16)).view(
                    torch.bfloat16))
        for name, (rm, rv) in self.run_stats[k].items():
            if run_stats and name in run_stats:
                c = rm.shape[0]
                a, b = run_stats[name]
                ra = np.zeros(c, np.float32)
                rb = np.ones(c, np.float32)
                ra[:len(a)] = a
                rb[:len(b)] = b
                rm.copy_(torch.from_numpy(ra))
                rv.copy_(torch.from_numpy(rb))
            else:
                rm.zero_()
                rv.fill_(1.0)
        st = torch.tensor([step, 0, 0, 0], dtype=torch.int32)
        self.state[k].copy_(st)

    def get_member_state(self, k, want_slots=True):
        m = self.members[k]
        # the pack's steps and the caller's uploads — not a device-wide sync, which
        # would stall (and, mid-capture, break) other threads' concurrent packs
        self.stream.synchronize()
        self.torch.cuda.current_stream(self.dev).synchronize()
        params, slots = {}, {}
        for p in m.net.params:
            full = f"{m.model_id}/{p.name}"
            params[full] = from_dev_layout(p, self.params[k][p.name].cpu().numpy())
            if want_slots and SLOTS[m.optimizer]:
                slots[full] = {s: from_dev_layout(p, self.slots[k][p.name][i].cpu().numpy())
                               for i, s in enumerate(SLOTS[m.optimizer])}
        rs = {n: (a.cpu().numpy()[:m.net.tensors[self._bn_x(m, n)].creal].astype(np.float64),
                  b.cpu().numpy()[:m.net.tensors[self._bn_x(m, n)].creal].astype(np.float64))
              for n, (a, b) in self.run_stats[k].items()}
        step = int(self.state[k, 0].item())
        return params, slots, step, rs

    @staticmethod
    def _bn_x(m, name):
        for op in m.net.ops:
            if op.name == name:
                return op.x
        raise KeyError(name)

    def set_lr(self, k, lr):
        self.members[k].lr = float(lr)
        self._progs.clear()

    def grad_of(self, k, pname):
        p = self.members[k].net.param(pname)
        return from_dev_layout(p, self.grads[k][pname].cpu().numpy())

    # -- program construction -------------------------------------------------------
    def _ptr(self, k, name, which):
        """device address of tensor `name` ("val" or "grad") of member k; a
        view points into its base buffer"""
        t = self.members[k].net.tensors[name]
        A = self.acts[k]
        if t.base is not None:
            return A[which][t.base].data_ptr() + 2 * t.ch0
        return A[which][name].data_ptr()

    def _ld(self, k, name):
        """row (pixel) stride in elements of tensor `name` of member k"""
        net = self.members[k].net
        t = net.tensors[name]
        return net.tensors[t.base].c if t.base is not None else t.c

    def tensor(self, k, name, which, rows):
        """[rows][c] torch view of a member tensor (tests / diagnostics)"""
        net = self.members[k].net
        t = net.tensors[name]
        A = self.acts[k]
        if t.base is not None:
            return A[which][t.base][:rows, t.ch0:t.ch0 + t.c]
        return A[which][name][:rows]

    def _counter(self, k, slot):
        """int32[17] ticket counters of (op, slot) of member k (tree_reduce)"""
        c = self.acts[k]["counters"]
        return c.data_ptr() + 4 * 17 * slot

    def _flag(self, k):
        return self.state.data_ptr() + 16 * k + 4

    def _fwd_steps(self, k, take, lead, data, train=True):
        """Per-member forward kernel steps: list of (kind, cfg, struct, tag).
        train=False: the eval forward (BN normalises with the running
        statistics and leaves them untouched; the head only sums the loss)."""
        m = self.members[k]
        net, A = m.net, self.acts[k]
        steps = []
        idx = self.idx[lead].data_ptr()
        for oi, op in enumerate(net.ops):
            tx = net.tensors[op.x] if op.x else None
            if op.kind == "conv":
                ty = net.tensors[op.y]
                first = op.x == "input"
                src, fidx = self._input(lead, data) if first else (self._ptr(k, op.x, "val"), 0)
                cs = _lib.CnnConv()
                cs.src = src
                cs.idx = fidx
                cs.wt = self.w16[k][op.params[0]].data_ptr()
                cs.dst = self._ptr(k, op.y, "val")
                cs.bias = self.params[k][op.params[1]].data_ptr() if op.a["bias"] else 0
                cs.n, cs.h, cs.w, cs.c = take, tx.h, tx.w, tx.c
                cs.k, cs.r, cs.s = ty.c, op.a["r"], op.a["s"]
                cs.stride, cs.pad, cs.p, cs.q = op.a["stride"], op.a["pad"], ty.h, ty.w
                cs.ldx = tx.c if first else self._ld(k, op.x)
                if first:
                    self._dense_geometry(cs, k, op, lead, take)
                cs.ldo = self._ld(k, op.y)
                cs.act = CNN_ACT[op.a["act"]]
                cs.out_f32 = int(op.a["out_f32"])
                nt = _pick_ntile(ty.c)
                tag = None
                if train and first and k in self.first_shared:
                    gi2, li, j, ks = self.first_shared[k]
                    tag = ("first", gi2, li, j, lead)
                steps.append((CNN["CONV_FPROP"], (nt, _stages(nt)), cs, tag))
            elif op.kind == "bn":
                rows = take * tx.h * tx.w
                for kind in ("BN_STATS", "BN_APPLY") if train else ("BN_APPLY",):
                    b = self._bn_struct(k, op, rows)
                    b.use_running = 0 if train else 1
                    steps.append((CNN[kind], None, b, None))
            elif op.kind == "dw":
                ty = net.tensors[op.y]
                d = self._dw_struct(k, op, take)
                steps.append((CNN["DW_FPROP"], None, d, None))
            elif op.kind in ("maxpool", "avgpool"):
                pl = self._pool_struct(k, op, take)
                steps.append((CNN["MAXPOOL_FWD" if op.kind == "maxpool" else "AVGPOOL_FWD"],
                              None, pl, None))
            elif op.kind == "head":
                t = net.tensors[op.x]
                h = _lib.CnnHead()
                h.logits = self._ptr(k, op.x, "val")
                h.labels = data.y.data_ptr()
                h.idx = idx
                last = net.ops[oi - 1]
                if train:
                    h.dlogits = self._ptr(k, op.x, "grad")
                    h.dbias = self.grads[k][last.params[1]].data_ptr()
                    h.loss = self.state.data_ptr() + 16 * k + 12
                    h.flag = self._flag(k)
                else:
                    h.loss = self.eval_loss.data_ptr() + 4 * k
                h.rows, h.classes, h.ldl = take, op.a["classes"], t.c
                steps.append((CNN["XENT"], None, h, None))
        return steps

    def _input(self, lead, data):
        """(source, index list) the first conv of a member led by `lead` reads:
        the leader's batch buffer, which the step's first op (GATHER) fills
        from the dataset rows idx[...] — in HBM, or over PCIe from page-locked
        host memory (streamed inputs).  One contiguous batch per input group
        keeps the index indirection out of the GEMMs' operand loads."""
        st = self.staging.get(lead)
        if st is None:
            _, h, w = self.members[lead].net.arch.image
            st = self._z(self.members[lead].batch, h, w, data.cp, dt=self.torch.bfloat16)
            self.staging[lead] = st
        return st.data_ptr(), 0

    def _cols_key(self, k, lead):
        """(lead, r, s, stride, pad, columns) of member k's dense first conv, or None"""
        op = self.members[k].net.ops[0]
        if op.kind != "conv" or op.x != "input":
            return None
        W = self.members[k].net.param(op.params[0])
        if not W.im2col:
            return None
        return (lead, op.a["r"], op.a["s"], op.a["stride"], op.a["pad"], W.im2col)

    def _cols(self, key):
        """the IM2COL rows buffer [batch·p·q][columns] of an input group's leader
        and first-conv geometry"""
        buf = self._cols_bufs.get(key) if hasattr(self, "_cols_bufs") else None
        if buf is None:
            if not hasattr(self, "_cols_bufs"):
                self._cols_bufs = {}
            lead, r, s, stv, pad, cols = key
            net = self.members[lead].net
            ty = net.tensors[net.ops[0].y]
            buf = self._z(self.members[lead].batch * ty.h * ty.w, cols, dt=self.torch.bfloat16)
            self._cols_bufs[key] = buf
        return buf

    def _dense_geometry(self, cs, k, op, lead, take):
        """a dense first conv as a 1x1 GEMM over its IM2COL rows"""
        key = self._cols_key(k, lead)
        if key is None:
            return
        ty = self.members[k].net.tensors[op.y]
        cs.src, cs.idx = self._cols(key).data_ptr(), 0
        cs.n, cs.h, cs.w, cs.c = take, ty.h, ty.w, key[5]
        cs.r = cs.s = cs.stride = 1
        cs.pad = 0
        cs.ldx = key[5]

    def _im2col_op(self, pairs, data):
        """one IM2COL launch filling the dense first-conv rows of every
        (member, lead) pair's input group (after GATHER), or None"""
        seen, ims = set(), []
        for k, lead, take in pairs:
            key = self._cols_key(k, lead)
            if key is None or key in seen:
                continue
            seen.add(key)
            _, r, s, stv, pad, cols = key
            net = self.members[lead].net
            tx, ty = net.tensors["input"], net.tensors[net.ops[0].y]
            im = _lib.CnnIm2col()
            im.src = self._input(lead, data)[0]
            im.dst = self._cols(key).data_ptr()
            im.n, im.h, im.w, im.cp, im.c = take, tx.h, tx.w, data.cp, tx.creal
            im.r, im.s, im.stride, im.pad, im.p, im.q, im.ldo = r, s, stv, pad, ty.h, ty.w, cols
            ims.append(im)
        return (CNN["IM2COL"], None, ims) if ims else None

    def _bn_struct(self, k, op, rows):
        """member k's BN problem over `rows` rows: a copy of the (k, op) template
        (every pointer / stride field is fixed for the pack's life) with the row
        count and partition filled in — program builds are host work per new
        takes tuple, so the Hyperband legs make hundreds of them"""
        tpl = self._bn_tpl.get((k, op.name)) if hasattr(self, "_bn_tpl") else None
        if tpl is None:
            if not hasattr(self, "_bn_tpl"):
                self._bn_tpl = {}
            tpl = self._bn_tpl[(k, op.name)] = self._bn_template(k, op)
        b = _lib.CnnBn.from_buffer_copy(tpl)
        b.rows = rows
        b.rpb = rows_per_block(rows, b.c)
        return b

    def _bn_template(self, k, op):
        m = self.members[k]
        net, A = m.net, self.acts[k]
        tx = net.tensors[op.x]
        b = _lib.CnnBn()
        b.x = self._ptr(k, op.x, "val")
        b.res = self._ptr(k, op.res, "val") if op.res else 0
        b.out = self._ptr(k, op.y, "val")
        b.dout = self._ptr(k, op.y, "grad")
        b.fout = self._ptr(k, op.y, "val")
        b.dx = self._ptr(k, op.x, "grad")
        b.gamma = self.params[k][op.params[0]].data_ptr()
        b.beta = self.params[k][op.params[1]].data_ptr()
        b.dgamma = self.grads[k][op.params[0]].data_ptr()
        b.dbeta = self.grads[k][op.params[1]].data_ptr()
        b.stats = A["stats"][op.name].data_ptr()
        rm, rv = self.run_stats[k][op.name]
        b.run_mean, b.run_var = rm.data_ptr(), rv.data_ptr()
        b.ws = A["ws"][op.name].data_ptr()
        b.counter = self._counter(k, 4 * net.op_index[op.name])
        b.flag = self._flag(k)
        b.c = tx.c
        b.ldx = b.ldx2 = self._ld(k, op.x)
        b.ldo = b.ldd = self._ld(k, op.y)
        b.ldr = self._ld(k, op.res) if op.res else 0
        b.act = CNN_ACT[op.a["act"]]
        b.eps, b.momentum = _BN_EPS, _BN_MOMENTUM
        return b

    def _dw_struct(self, k, op, take):
        m = self.members[k]
        net, A = m.net, self.acts[k]
        tx, ty = net.tensors[op.x], net.tensors[op.y]
        d = _lib.CnnDw()
        d.x = self._ptr(k, op.x, "val")
        d.wt = self.w16[k][op.params[0]].data_ptr()
        d.dy = self._ptr(k, op.y, "grad")
        d.y = self._ptr(k, op.y, "val")
        d.dw = self.grads[k][op.params[0]].data_ptr()
        d.ws = A["ws"][op.name].data_ptr()
        d.counter = self._counter(k, 4 * net.op_index[op.name])
        d.flag = self._flag(k)
        d.n, d.h, d.w, d.c = take, tx.h, tx.w, tx.c
        d.r, d.s, d.stride, d.pad, d.p, d.q = (op.a["r"], op.a["s"], op.a["stride"], op.a["pad"],
                                               ty.h, ty.w)
        d.ldx, d.ldy = self._ld(k, op.x), self._ld(k, op.y)
        if d.r == 3 and d.s == 3 and d.stride in (1, 2):
            # 3x3 fast path (csrc/pk_cnn_ops.cuh dw_fast_wgrad): blocks own a chunk of
            # <= 64 channels x one of <= 16 pixel splits (~DW_CHANNEL_PIXELS_PER_BLOCK
            # channel-pixels each), a multiple of the block's pixel lanes
            cgb = min(_cgp(tx.c), 8)
            lanes = (256 // cgb) // 3
            pix = take * ty.h * ty.w
            nchunk = cdiv(tx.c // 8, cgb)
            nsplit = min(256 // nchunk, max(1, cdiv(pix * 8 * cgb, DW_CHANNEL_PIXELS_PER_BLOCK)))
            d.ppb = rup(cdiv(pix, nsplit), lanes)
        else:
            d.ppb = rows_per_block(take * ty.h * ty.w, tx.c, per_thread=4)
        return d

    def _pool_struct(self, k, op, take):
        m = self.members[k]
        net, A = m.net, self.acts[k]
        tx, ty = net.tensors[op.x], net.tensors[op.y]
        p = _lib.CnnPool()
        p.x = self._ptr(k, op.x, "val")
        p.y = self._ptr(k, op.y, "val")
        p.dy = self._ptr(k, op.y, "grad")
        p.dx = self._ptr(k, op.x, "grad")
        p.arg = A["arg"][op.name].data_ptr() if op.kind == "maxpool" else 0
        p.n, p.h, p.w, p.c = take, tx.h, tx.w, tx.c
        p.r, p.s, p.stride, p.pad, p.p, p.q = (op.a["r"], op.a["s"], op.a["stride"], op.a["pad"],
                                               ty.h, ty.w)
        p.ldx, p.ldy = self._ld(k, op.x), self._ld(k, op.y)
        return p

    def _bwd_steps(self, k, take, lead, data):
        m = self.members[k]
        net, A = m.net, self.acts[k]
        idx = self.idx[lead].data_ptr()
        steps = []
        written = {}   # base tensor -> channel intervals whose gradient holds a contribution

        def acc(name):
            """1 if the gradient of `name` (a tensor or a channel view) already
            holds a contribution — the next writer accumulates — else 0"""
            t = net.tensors[name]
            base = t.base or name
            lo, hi = t.ch0, t.ch0 + t.c
            iv = written.setdefault(base, [])
            cov = sum(max(0, min(hi, b) - max(lo, a)) for a, b in iv)
            if cov == hi - lo:
                return 1
            if cov == 0:
                iv.append((lo, hi))
                return 0
            raise NotImplementedError(f"gradient of {name} is partially accumulated")

        for op in reversed(net.ops):
            tx = net.tensors[op.x] if op.x else None
            if op.kind == "head":
                continue  # the XENT step (forward list) already wrote dlogits + dbias
            if op.kind == "conv":
                ty = net.tensors[op.y]
                first = op.x == "input"
                if op.a["bias"] and not op.a["out_f32"]:
                    rows = take * ty.h * ty.w
                    bs = _lib.CnnBias()
                    bs.dy = bs.g = self._ptr(k, op.y, "grad")
                    bs.fout = self._ptr(k, op.y, "val")
                    bs.dbias = self.grads[k][op.params[1]].data_ptr()
                    bs.ws = A["ws"][op.name].data_ptr()
                    bs.counter = self._counter(k, 4 * net.op_index[op.name] + 1)
                    bs.flag = self._flag(k)
                    bs.rows, bs.c, bs.ld = rows, ty.c, self._ld(k, op.y)
                    bs.rpb = rows_per_block(rows, ty.c)
                    bs.act = CNN_ACT[op.a["act"]]
                    steps.append((CNN["BIAS_ACT_BWD"], None, bs, None))
                W = net.param(op.params[0])
                pix = take * ty.h * ty.w
                rsc = W.im2col or op.a["r"] * op.a["s"] * tx.c
                nt, splits = _wgrad_cfg(ty.c, rsc, pix)
                bsplits = _wgrad_cfg(ty.c, rsc, m.batch * ty.h * ty.w)[1]
                splits = min(splits, bsplits) if op.name in A["split"] else 1
                cs = _lib.CnnConv()
                cs.src, cs.idx = self._input(lead, data) if first else (
                    self._ptr(k, op.x, "val"), 0)
                cs.dy = self._ptr(k, op.y, "grad")
                cs.n, cs.h, cs.w, cs.c = take, tx.h, tx.w, tx.c
                cs.k, cs.r, cs.s = ty.c, op.a["r"], op.a["s"]
                cs.stride, cs.pad, cs.p, cs.q = op.a["stride"], op.a["pad"], ty.h, ty.w
                cs.ldx = tx.c if first else self._ld(k, op.x)
                if first:
                    self._dense_geometry(cs, k, op, lead, take)
                cs.ldy = self._ld(k, op.y)
                cs.flag = self._flag(k)
                # fix the split count so the pixel partition is valid for this take
                while splits > 1 and cdiv(pix, rup(cdiv(pix, splits), 64)) != splits:
                    splits -= 1
                cs.splits = splits
                if splits > 1:
                    cs.dst = A["split"][op.name].data_ptr()
                else:
                    cs.dst = self.grads[k][op.params[0]].data_ptr()
                wtag = None
                if first and k in self.first_shared and splits > 1 and ty.c == 64 \
                        and nt == 64:
                    gi2, li, j, ks = self.first_shared[k]
                    wtag = ("firstw", gi2, li, j, lead)
                steps.append((CNN["CONV_WGRAD"], (nt, _stages(nt)), cs, wtag))
                if splits > 1:
                    rd = _lib.CnnReduce()
                    rd.src = A["split"][op.name].data_ptr()
                    rd.dst = self.grads[k][op.params[0]].data_ptr()
                    rd.flag = self._flag(k)
                    rd.len, rd.splits = W.numel, splits
                    steps.append((CNN["SPLIT_REDUCE"], None, rd, None))
                if not first:
                    ds = _lib.CnnConv()
                    ds.src = self._ptr(k, op.y, "grad")
                    ds.wt = self.wt16[k][op.params[0]].data_ptr()
                    ds.dst = self._ptr(k, op.x, "grad")
                    ds.n, ds.h, ds.w, ds.c = take, tx.h, tx.w, tx.c
                    ds.k, ds.r, ds.s = ty.c, op.a["r"], op.a["s"]
                    ds.stride, ds.pad, ds.p, ds.q = op.a["stride"], op.a["pad"], ty.h, ty.w
                    ds.ldy, ds.ldo = self._ld(k, op.y), self._ld(k, op.x)
                    ds.accumulate = acc(op.x)
                    ntd = _pick_ntile(tx.c)
                    steps.append((CNN["CONV_DGRAD"], (ntd, _stages(ntd)), ds, None))
            elif op.kind == "bn":
                rows = take * tx.h * tx.w
                b = self._bn_struct(k, op, rows)
                b.counter = self._counter(k, 4 * net.op_index[op.name] + 1)
                steps.append((CNN["BN_BWD_REDUCE"], None, b, None))
                b2 = self._bn_struct(k, op, rows)
                b2.counter = self._counter(k, 4 * net.op_index[op.name] + 1)
                b2.accumulate = acc(op.x)
                if op.res:
                    b2.dres = self._ptr(k, op.res, "grad")
                    b2.res_accumulate = acc(op.res)
                steps.append((CNN["BN_BWD_APPLY"], None, b2, None))
            elif op.kind == "dw":
                d = self._dw_struct(k, op, take)
                d.counter = A["dwcnt"][op.name].data_ptr()  # 17 ints per channel chunk
                steps.append((CNN["DW_WGRAD"], None, d, None))
                d2 = self._dw_struct(k, op, take)
                d2.y = self._ptr(k, op.x, "grad")
                if acc(op.x):
                    raise NotImplementedError("depthwise input with two consumers")
                steps.append((CNN["DW_DGRAD"], None, d2, None))
            elif op.kind in ("maxpool", "avgpool"):
                pl = self._pool_struct(k, op, take)
                pl.accumulate = acc(op.x)
                steps.append((CNN["MAXPOOL_BWD" if op.kind == "maxpool" else "AVGPOOL_BWD"],
                              None, pl, None))
        return steps

    def _opt_steps(self, k):
        m = self.members[k]
        steps = []
        for p in m.net.params:
            s = _lib.CnnOptSeg()
            s.w = self.params[k][p.name].data_ptr()
            s.g = self.grads[k][p.name].data_ptr()
            sl = self.slots[k][p.name]
            s.s1 = sl[0].data_ptr() if len(sl) > 0 else 0
            s.s2 = sl[1].data_ptr() if len(sl) > 1 else 0
            s.w16 = self.w16[k][p.name].data_ptr() if p.w16 else 0
            s.step = self.state.data_ptr() + 16 * k
            s.flag = self.state.data_ptr() + 16 * k + 8   # commit verdict (COMMIT mode 0)
            s.len = p.numel
            s.kind = OPT_CODES[m.optimizer]
            s.lr, s.wd = m.lr, m.wd
            steps.append((CNN["OPT"], None, s, None))
        return steps

    def _publish_steps(self, k):
        m = self.members[k]
        steps = []
        for p in m.net.params:
            if not p.dgrad:
                continue
            kp, kpad = p.dev_shape
            _, r, s, c = p.shape
            t = _lib.CnnTpose()
            t.src = self.w16[k][p.name].data_ptr()
            t.dst = self.wt16[k][p.name].data_ptr()
            t.k, t.c, t.taps = kp, p.cin_p, r * s
            t.kpad, t.kpadt = kpad, self.wt16[k][p.name].shape[1]
            steps.append((CNN["PUBLISH_T"], None, t, None))
        return steps

    def _group(self, per_member):
        """Zip per-member step lists by position; one launch per (position,
        kind, cfg).  Concatenated-N first-layer problems are merged."""
        ops = []
        L = max((len(s) for s in per_member), default=0)
        for i in range(L):
            buckets = {}
            order = []
            for steps in per_member:
                if i >= len(steps):
                    continue
                kind, cfg, st, tag = steps[i]
                key = (kind, cfg)
                if key not in buckets:
                    buckets[key] = []
                    order.append(key)
                buckets[key].append((st, tag))
            for key in order:
                kind, cfg = key
                items = buckets[key]
                if kind == CNN["CONV_FPROP"]:
                    n0 = len(items)
                    items = self._merge_first(items)
                    if len(items) != n0:  # a concatenated-N problem: tile over its full N
                        nt = max(_pick_ntile(st.k) for st, _ in items)
                        cfg = (nt, _stages(nt))
                elif kind == CNN["CONV_WGRAD"] and any(t is not None for _, t in items):
                    merged = self._merge_first_wgrad(items)
                    plain = [(st, None) for st, t in items if t is None]
                    if plain:
                        ops.append((kind, cfg, [st for st, _ in plain]))
                    for st in merged:  # one launch per concatenated problem, N tile <= 256
                        nt = min(256, st.k)
                        ops.append((kind, (nt, _stages(nt)), [st]))
                    continue
                ops.append((kind, cfg, [st for st, _ in items]))
        return ops

    def _merge_first_wgrad(self, items):
        """The first-layer WGRAD problems of a shared input group (tag
        ("firstw", gi, li, j, lead)) as one concatenated-N problem: GEMM
        M = r·s·c over the shared input, N = members x 64 (csrc pk_cnn.cu
        conv_to_launches, cg::Problem::wseg); each member keeps its own pixel
        splits, so its partials are bit-identical to its standalone WGRAD."""
        merged, order = {}, []
        for st, tag in items:
            if tag is None:
                continue
            _, gi, li, j, lead = tag
            if (gi, li, lead) not in merged:
                merged[(gi, li, lead)] = []
                order.append((gi, li, lead))
            merged[(gi, li, lead)].append((j, st))
        res = []
        for key in order:
            parts = sorted(merged[key], key=lambda t: t[0])
            js = [j for j, _ in parts]
            base = parts[0][1]
            fkey = ("first",) + key[:2]
            if len(parts) == 1 or js != list(range(js[0], js[0] + len(js))):
                res += [p for _, p in parts]  # (kept as separate launches below)
                continue
            m = _lib.CnnConv()
            C.pointer(m)[0] = base
            g = self._first_grad[fkey]
            m.k = 64 * len(parts)
            m.nseg = 64
            m.dy = g[js[0]].data_ptr()
            m.dseg = g.shape[1] * g.shape[2]
            m.dst = self._first_split[fkey][js[0]].data_ptr()
            res.append(m)
        return res

    def _merge_first(self, items):
        out, merged = [], {}
        for st, tag in items:
            if tag is None:
                out.append((st, None))
                continue
            _, gi, li, j, lead = tag
            if (gi, li, lead) not in merged:
                merged[(gi, li, lead)] = []
                out.append(((gi, li, lead), "M"))
            merged[(gi, li, lead)].append((j, st))
        res = []
        for st, tag in out:
            if tag != "M":
                res.append((st, None))
                continue
            parts = sorted(merged[st], key=lambda t: t[0])
            js = [j for j, _ in parts]
            if len(parts) == 1 or js != list(range(js[0], js[0] + len(js))):
                res += [(p, None) for _, p in parts]
                continue
            st = st[:2]
            base = parts[0][1]
            m = _lib.CnnConv()
            C.pointer(m)[0] = base
            kseg = base.k
            m.wt = self.shared_w16[st].data_ptr()
            if base.bias:
                m.bias = self.shared_bias[st].data_ptr()
            m.k = kseg * len(parts)
            m.nseg = kseg
            rows = base.n * base.p * base.q
            full_rows = self._first_out[("first",) + st].shape[1]
            m.dseg = full_rows * kseg
            m.dst = self._first_out[("first",) + st][js[0]].data_ptr()
            m.wt = self.shared_w16[st][js[0] * kseg:].data_ptr()
            if base.bias:
                m.bias = self.shared_bias[st][js[0] * kseg:].data_ptr()
            assert rows <= full_rows
            res.append((m, None))
        return res

    def _lanes(self, act):
        """Active members split by architecture (identical nets are grouped into
        shared launches; different nets go to separate lanes, at most 8)."""
        by = {}
        for k in act:
            by.setdefault(self.members[k].net.signature, []).append(k)
        lanes = list(by.values())
        while len(lanes) > 8:  # fold the smallest lanes together
            lanes.sort(key=len)
            lanes = [lanes[0] + lanes[1]] + lanes[2:]
        return lanes

    def _build_ops(self, takes, leads, data, with_update=True):
        K = len(self.members)
        act = [k for k in range(K) if takes[k] > 0]
        ops = []
        # each input group's batch rows, gathered once (over PCIe when data.host)
        gs = []
        for lead in sorted({leads[k] for k in act}):
            g = _lib.CnnGather()
            g.src = data.x.data_ptr()
            g.dst = self._input(lead, data)[0]
            g.idx = self.idx[lead].data_ptr()
            g.row_bytes, g.rows = data.row_bytes, takes[lead]
            gs.append(g)
        ops.append((CNN["GATHER"], None, gs))
        im = self._im2col_op([(k, leads[k], takes[leads[k]]) for k in act], data)
        if im is not None:
            ops.append(im)
        fwd = {k: self._fwd_steps(k, takes[k], leads[k], data) for k in act}
        bwd = {k: self._bwd_steps(k, takes[k], leads[k], data) for k in act}
        lanes = self._lanes(act)
        if len(lanes) == 1:
            ops += self._group([fwd[k] for k in act])
            # weight gradients (and their split sums) only feed the optimizer: an async
            # lane (pk_cnn_op.lane 16 + 1) runs them beside the data-gradient chain
            for op in self._group([bwd[k] for k in act]):
                async_ok = op[0] in (CNN["CONV_WGRAD"], CNN["SPLIT_REDUCE"],
                                     CNN["DW_WGRAD"]) and ASYNC_WGRAD
                ops.append(op + (17,) if async_ok else op)
        else:
            # heterogeneous pack: one lane (stream) per architecture, so the
            # different nets' launches overlap; the shared-input first layer's
            # concatenated FPROP runs before the fork, its WGRAD after the join
            pre, post = [], []
            for k in act:
                if fwd[k] and fwd[k][0][3] is not None:
                    pre.append([fwd[k].pop(0)])
                cut = next((i for i, st in enumerate(bwd[k])
                            if st[3] is not None and st[3][0] == "firstw"), None)
                if cut is not None:
                    post.append(bwd[k][cut:])
                    bwd[k] = bwd[k][:cut]
            ops += self._group(pre)
            for li, lane in enumerate(lanes, 1):
                for op in self._group([fwd[k] for k in lane]):
                    ops.append(op + (li,))
                for op in self._group([bwd[k] for k in lane]):
                    async_ok = op[0] in (CNN["CONV_WGRAD"], CNN["SPLIT_REDUCE"],
                                         CNN["DW_WGRAD"]) and ASYNC_WGRAD
                    ops.append(op + ((16 + li) if async_ok else li,))
            ops += self._group(post)
        if with_update:
            cm = []
            for k in act:
                c = _lib.CnnCommit()
                c.step = self.state.data_ptr() + 16 * k
                c.flag = self._flag(k)
                c.verdict = self.state.data_ptr() + 16 * k + 8
                cm.append(c)
            ops.append((CNN["COMMIT"], (0, 0), cm))
            opt = [s for k in act for s in self._opt_steps(k)]
            ops.append((CNN["OPT"], None, [st for _, _, st, _ in opt]))
            pub = [s for k in act for s in self._publish_steps(k)]
            if pub:
                ops.append((CNN["PUBLISH_T"], None, [st for _, _, st, _ in pub]))
            ops.append((CNN["COMMIT"], (1, 0), cm))
        return ops

    def eval_program(self, k, take, data):
        """forward-only program of member k on `take` rows (its own batch buffer
        as the input group): the validation loss of tuner.py:460-464"""
        key = ("eval", k, take, id(data))
        pr = self._progs.get(key)
        if pr is None:
            g = _lib.CnnGather()
            g.src = data.x.data_ptr()
            g.dst = self._input(k, data)[0]
            g.idx = self.idx[k].data_ptr()
            g.row_bytes, g.rows = data.row_bytes, take
            ops = [(CNN["GATHER"], None, [g])]
            im = self._im2col_op([(k, k, take)], data)
            if im is not None:
                ops.append(im)
            ops += self._group([self._fwd_steps(k, take, k, data, train=False)])
            pr = CnnProgram(ops, self.device)
            self._progs[key] = pr
        return pr

    def val_loss(self, k, data, rows_dev, n):
        """mean softmax cross-entropy of member k over dataset rows rows_dev[:n]
        (device int64), in chunks of its batch size; BN in eval mode."""
        torch = self.torch
        b = self.members[k].batch
        tot = 0.0
        with torch.cuda.stream(self.stream):
            for i0 in range(0, n, b):
                take = min(b, n - i0)
                self.idx[k][:take].copy_(rows_dev[i0:i0 + take], non_blocking=True)
                self.eval_program(k, take, data).run(self.stream.cuda_stream)
                tot += float(self.eval_loss[k].item()) * take
        return tot / n

    def program(self, takes, leads, data):
        """The step program for per-member valid rows `takes` (0 = inactive)
        and input-group leaders `leads` (members with one leader read the same
        batch rows from that leader's index buffer)."""
        key = (tuple(takes), tuple(leads), id(data))
        pr = self._progs.get(key)
        if pr is None:
            pr = CnnProgram(self._build_ops(takes, leads, data), self.device)
            self._progs[key] = pr
        return pr


class CnnProgram:
    """A pk_cnn_prog built from (kind, cfg, [structs]) launch groups."""

    def __init__(self, ops, device):
        self.lib = _lib.lib()
        self.kinds = [op[0] for op in ops]
        self.sizes = [len(op[2]) for op in ops]
        self.lanes = [op[3] if len(op) > 3 else 0 for op in ops]
        self._keep = []
        arr = (_lib.CnnOp * len(ops))()
        for i, op in enumerate(ops):
            kind, cfg, structs = op[:3]
            arr[i].lane = op[3] if len(op) > 3 else 0
            T = _lib.CNN_STRUCT[kind]
            buf = (T * len(structs))(*structs)
            self._keep.append(buf)
            arr[i].kind = kind
            arr[i].nprob = len(structs)
            arr[i].cfg0, arr[i].cfg1 = cfg if cfg else (0, 0)
            arr[i].probs = C.cast(buf, C.c_void_p)
        self.handle = C.c_void_p()
        rc = self.lib.pk_cnn_prog_create(arr, len(ops), device, C.byref(self.handle))
        if rc != 0:
            raise _lib.PKError(rc, self.lib.pk_cnn_last_error().decode())
        self.launches = self.lib.pk_cnn_prog_launches(self.handle)

    def run(self, stream, graph=True):
        rc = self.lib.pk_cnn_prog_run(self.handle, C.c_void_p(stream), int(graph))
        if rc != 0:
            raise _lib.PKError(rc, self.lib.pk_cnn_last_error().decode())

    def profile(self, stream):
        out = (C.c_float * len(self.kinds))()
        rc = self.lib.pk_cnn_prog_profile(self.handle, C.c_void_p(stream), out)
        if rc != 0:
            raise _lib.PKError(rc, self.lib.pk_cnn_last_error().decode())
        return list(out)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.pk_cnn_prog_destroy(h)
            self.handle = None
