"""B200 memory model for pack grouping.

The reference sizes packs with a calibrated 16 GB simulator
(device_sim.py:72-85, :222-244).  Here a member's footprint is the exact
size of its device slab (csrc/pk_runtime.cu pk_member_create): ping-pong
parameters, ping-pong optimizer slots, per-layer Z/A/dZ workspace for
`batch_size` rows and the control block, each 256-byte aligned; capacity is
the GPU's real HBM.  `OOMError` / `DeviceAccountant` keep the reference's
interface so `pack_opt_*` and `load_model(device=...)` work unchanged.
"""
from __future__ import annotations

from dataclasses import dataclass

_CTL_BYTES = 80          # sizeof(pk::MemberCtl)
_ALIGN = 256
_SLOTS = {"sgd": 0, "momentum": 1, "adagrad": 1, "adam": 2}


class OOMError(Exception):
    def __init__(self, demand, capacity, what="pack"):
        self.demand = int(demand)
        self.capacity = int(capacity)
        self.deficit = int(demand - capacity)
        self.what = what
        super().__init__(f"{what}: demand {self.demand} B exceeds capacity "
                         f"{self.capacity} B by {self.deficit} B")

    def __reduce__(self):  # pickles across the Hyperband pool's gather
        return (type(self), (self.demand, self.capacity, self.what))


def _al(v):
    return (v + _ALIGN - 1) // _ALIGN * _ALIGN


_SMEM_OPTIN = 232448     # B200 opt-in shared memory per block (227 KB)
_STATIC_MARGIN = 16384   # kStaticSmemMargin (csrc/pk_pack.cuh)
_M1_BC, _M1_KC, _M1_STAGES, _M1_MAXR, _M1_MAXC = 8, 32, 4, 128, 32


def _m1_rows_pad(r):
    return 32 if r <= 32 else (64 if r <= 64 else 128)


_T_KS, _T_UM, _T_BK, _T_BU, _T_XLD, _T_BXLD, _T_LB, _T_MAXC, _T_MAXR = (
    64, 128, 128, 32, 68, 132, 32, 32, 128)


def _cdiv(a, b):
    return -(-a // b)


_X_KC, _X_LD, _X_UB, _X_FS, _X_RED, _X_MAXC, _X_MAXR, _X_MAXCS = 64, 68, 16, 4, 4096, 32, 64, 16


def _r4(n):
    return (n + 3) & ~3


def _m1x_smem(RP, U, C, ns, Sb):
    """M1X::smem (csrc/pk_m1x.cuh)."""
    wld = U + 4
    ring = max(_X_FS * (RP * _X_LD + _X_KC * wld), Sb * (RP * _X_LD + (1 + ns) * _X_KC * wld))
    return 4 * (ring + _X_RED + 3 * RP * U + _r4(U * C) + _r4((U // _X_UB) * RP * C)
                + _r4(RP * (C + 1)) + _r4(U) + 32) + 8 * RP


def _plan():
    """the library's current kernel plan (csrc eligibility reads the same)"""
    from . import _lib
    return _lib.plan_options()


def uses_m1x(arch, optimizer: str, batch_size: int, precision="f32") -> bool:
    """Mirror of csrc m1x_eligible(): the one-launch cluster step (fp32, one
    hidden layer, <= 32 classes, <= 64 rows, H and D multiples of 4, one
    cluster of <= 16 CTAs covers the hidden layer within the smem budget)."""
    if precision != "f32" or len(arch.hidden) != 1 or not _plan()["m1x"]:
        return False
    D, H, C = arch.input_dim, arch.hidden[0], arch.classes
    if C > _X_MAXC or batch_size > _X_MAXR or H % 4 or D % 4:
        return False
    RP, ns = _m1_rows_pad(batch_size), _SLOTS[optimizer.lower()]
    budget = _SMEM_OPTIN - _STATIC_MARGIN
    b = 4 if RP <= 32 else 2
    while b >= 1 and _m1x_smem(RP, _X_UB * b, C, ns, 2) > budget:
        b //= 2
    return b >= 1 and _cdiv(_cdiv(H, _X_UB), b) <= _X_MAXCS


def uses_m1t(arch, optimizer: str, batch_size: int, precision="f32") -> bool:
    """Mirror of csrc m1t_eligible(): the tcgen05 3xTF32 one-hidden-layer
    step (fp32, <= 32 classes, <= 128 rows, H and D multiples of 4, smem fits),
    for members the one-launch cluster step does not take."""
    if precision != "f32" or len(arch.hidden) != 1 or not _plan()["tcgen05"]:
        return False
    if uses_m1x(arch, optimizer, batch_size, precision):
        return False
    D, H, C = arch.input_dim, arch.hidden[0], arch.classes
    if C > _T_MAXC or batch_size > _T_MAXR or H % 4 or D % 4 or _cdiv(D, _T_KS) > 16:
        return False
    RP = _m1_rows_pad(batch_size)
    ns = _SLOTS[optimizer.lower()]
    fwd = _T_KS * _T_UM * 4 + RP * _T_XLD * 4 + 2 * _T_UM * _T_KS * 4 + 2 * RP * _T_KS * 4 \
        + _T_UM * C * 4 + _T_UM * 4 + RP * 4 + 64
    bwd = (_T_BK * (_T_BU + 4) * 4 + RP * _T_BXLD * 4 + 2 * _T_BK * 32 * 4
           + 2 * _T_BU * 32 * 4 + RP * (C + 1) * 4 + 2 * RP * _T_BU * 4
           + (1 + ns) * _T_BU * C * 4 + _T_MAXC * 4 + 2 * RP * 4 + 128)
    budget = _SMEM_OPTIN - _STATIC_MARGIN
    return fwd <= budget and bwd <= budget


def uses_fused_mlp1(arch, optimizer: str, batch_size: int, precision="f32") -> bool:
    """Mirror of csrc mlp1_eligible() (the FFMA fused path, taken when the
    tensor path is not): one hidden layer, <= 32 classes, batch <= 128 and
    the fused kernels' shared memory fits."""
    if uses_m1t(arch, optimizer, batch_size, precision) or \
            uses_m1x(arch, optimizer, batch_size, precision):
        return False
    if len(arch.hidden) != 1 or arch.classes > _M1_MAXC or batch_size > _M1_MAXR:
        return False
    if precision == "f64" or not _plan()["mlp1"]:  # phase kernels win in f64
        return False
    es = 8 if precision == "f64" else 4
    vec = 16 // es
    D, C, RP = arch.input_dim, arch.classes, _m1_rows_pad(batch_size)
    ns = _SLOTS[optimizer.lower()]
    xld = _M1_KC + vec
    fwd = (_M1_STAGES * (RP * xld + _M1_KC * _M1_BC) * es + (128 // RP) * RP * _M1_BC * es
           + RP * _M1_BC * es + _M1_BC * C * es + RP * 4)
    bwd = (D * _M1_BC * (1 + ns) * es + _M1_STAGES * RP * xld * es + RP * (_M1_MAXC + 1) * es
           + 2 * RP * _M1_BC * es + _M1_BC * C * (1 + ns) * es + 2 * RP * 4)
    budget = _SMEM_OPTIN - _STATIC_MARGIN
    return fwd <= budget and bwd <= budget


def member_device_bytes(arch, optimizer: str, batch_size: int, precision="f32") -> int:
    """Bytes pk_member_create allocates for this member (exact)."""
    es = 8 if precision == "f64" else 4
    dims = (arch.input_dim, *arch.hidden, arch.classes)
    P = sum(dims[i] * dims[i + 1] + dims[i + 1] for i in range(len(dims) - 1))
    ss = _cdiv(P * es, 32) * 32 // es  # slot blocks are 32-byte strided
    ns = _SLOTS[optimizer.lower()]
    total = 2 * _al(P * es) + 2 * _al(ns * ss * es)
    n = len(dims) - 1
    tensor = uses_m1t(arch, optimizer, batch_size, precision)
    fused = uses_fused_mlp1(arch, optimizer, batch_size, precision)
    for layer in range(n):
        act = batch_size * dims[layer + 1] * es
        z = act
        if fused and layer == 1:  # Z_1 doubles as the partial-logit exchange
            z = max(act, -(-dims[1] // _M1_BC) * act)
        if tensor and layer == 1:
            z = max(act, _cdiv(dims[1], _T_LB) * act)
        total += _al(z) + _al(act if layer + 1 < n else 0) + _al(act)
    total += _al(batch_size * 8)  # per-row loss terms (float64)
    return total + _al(_CTL_BYTES)


@dataclass(frozen=True)
class B200Device:
    """Device profile consumed by the tuner's grouping (`memory_capacity`)."""
    memory_capacity: int
    name: str = "NVIDIA B200"

    @classmethod
    def detect(cls, reserve_fraction=0.05):
        from .runtime import runtime
        free, total, _ = runtime().mem_info()
        return cls(memory_capacity=int(total * (1.0 - reserve_fraction)))


class DeviceAccountant:
    """Which members occupy a device and how many bytes (device_sim.py:222-244)."""

    def __init__(self, device):
        self.device = device
        self.resident: dict = {}

    @property
    def used(self) -> int:
        return sum(self.resident.values())

    def register(self, model_id: str, nbytes: int):
        if model_id in self.resident:
            raise ValueError(f"{model_id!r} is already resident")
        if self.used + nbytes > self.device.memory_capacity:
            raise OOMError(self.used + nbytes, self.device.memory_capacity,
                           what=f"load {model_id!r}")
        self.resident[model_id] = int(nbytes)

    def release(self, model_id: str) -> int:
        if model_id not in self.resident:
            raise ValueError(f"{model_id!r} is not resident")
        return self.resident.pop(model_id)
