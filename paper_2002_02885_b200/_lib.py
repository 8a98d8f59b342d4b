"""ctypes binding of the C-ABI in include/packtrain_b200.h.

The library is built in-tree (`libpk_b200.so`, see csrc/Makefile).  There is
no fallback: if the library or a CUDA device is missing, `lib()` raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpk_b200.so")

PK_MAX_LAYERS = 8
PK_OK, PK_ERR_ARG, PK_ERR_NONFINITE_VALUE, PK_ERR_NONFINITE_GRAD = 0, 1, 2, 3
PK_ERR_OOM, PK_ERR_CUDA, PK_ERR_STATE, PK_SKIPPED = 4, 5, 6, 7
PK_F32, PK_F64 = 0, 1
# enum order = the reference tuples (engine.py:21-22)
ACT_CODES = {"sigmoid": 0, "leaky_relu": 1, "tanh": 2, "relu": 3}
OPT_CODES = {"sgd": 0, "momentum": 1, "adam": 2, "adagrad": 3}

# every symbol the header declares (checked by tests/test_abi.py)
EXPORTS = (
    "pk_abi_version", "pk_plan_options_get", "pk_plan_options_set", "pk_ctx_create", "pk_ctx_destroy", "pk_ctx_last_error",
    "pk_ctx_set_stream", "pk_ctx_synchronize", "pk_ctx_mem_info",
    "pk_dataset_create", "pk_dataset_write", "pk_dataset_write_rows", "pk_dataset_gather_rows",
    "pk_pack_run", "pk_host_map", "pk_host_unmap",
    "pk_dataset_destroy",
    "pk_order_create", "pk_order_destroy",
    "pk_member_create", "pk_member_destroy", "pk_member_param_count",
    "pk_member_slot_count", "pk_member_device_bytes", "pk_member_set_lr",
    "pk_member_set_state", "pk_member_get_state", "pk_member_inject_fault",
    "pk_pack_create", "pk_pack_destroy", "pk_pack_step", "pk_pack_step_async",
    "pk_pack_step_wait", "pk_pack_eval", "pk_pack_profile_step", "pk_pack_trace",
    "pk_pack_launches_per_step",
    "pk_conv_gemm_test",
    "pk_cnn_prog_create", "pk_cnn_prog_destroy", "pk_cnn_prog_run", "pk_cnn_prog_profile",
    "pk_cnn_prog_launches", "pk_cnn_last_error",
)


class PlanOptions(C.Structure):
    """packtrain_b200.h pk_plan_options: the MLP path's kernel plan."""
    _fields_ = [(n, C.c_int32) for n in ("fwd", "fwd_cluster", "tcgen05", "mlp1", "m1x",
                                         "fwd_split", "wgrad_narrow", "inline_desc",
                                         "run_batch", "trace", "conv_cluster", "conv_halo")] \
        + [("reserved", C.c_int32 * 4)]


PLAN_FIELDS = ("fwd", "fwd_cluster", "tcgen05", "mlp1", "m1x", "fwd_split", "wgrad_narrow",
               "inline_desc", "run_batch", "trace", "conv_cluster", "conv_halo")
FWD_PLANS = {"auto": 0, "split": 1, "stream": 2}


def plan_options() -> dict:
    """The current kernel plan (pk_plan_options_get) as a dict."""
    o = PlanOptions()
    if lib().pk_plan_options_get(C.byref(o)) != PK_OK:
        raise PKError(PK_ERR_ARG, "pk_plan_options_get failed")
    return {f: int(getattr(o, f)) for f in PLAN_FIELDS}


def set_plan_options(**kw) -> dict:
    """Update fields of the kernel plan (read when a pack is created); returns
    the previous plan.  set_plan_options() with no fields restores the defaults."""
    prev = plan_options()
    if not kw:
        lib().pk_plan_options_set(None)
        return prev
    o = PlanOptions()
    cur = dict(prev)
    for k, v in kw.items():
        if k not in cur:
            raise KeyError(f"unknown plan option {k!r}")
        cur[k] = FWD_PLANS[v] if k == "fwd" and isinstance(v, str) else int(v)
    for f in PLAN_FIELDS:
        setattr(o, f, cur[f])
    if lib().pk_plan_options_set(C.byref(o)) != PK_OK:
        raise PKError(PK_ERR_ARG, f"invalid kernel plan {kw}")
    return prev


class kernel_plan:
    """with kernel_plan(fwd="stream"): ... — a scoped kernel plan."""

    def __init__(self, **kw):
        self.kw = kw

    def __enter__(self):
        self.prev = set_plan_options(**self.kw)
        return self

    def __exit__(self, *exc):
        set_plan_options(**self.prev)


class MemberDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32),
                ("dims", C.c_int32 * (PK_MAX_LAYERS + 1)),
                ("activation", C.c_int32),
                ("optimizer", C.c_int32),
                ("learning_rate", C.c_double),
                ("weight_decay", C.c_double),
                ("max_rows", C.c_int32),
                ("reserved", C.c_int32)]


class Feed(C.Structure):
    _fields_ = [("data", C.c_void_p),
                ("order", C.c_void_p),
                ("pos", C.c_int64),
                ("take", C.c_int32),
                ("group", C.c_int32)]


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("member", C.c_int32),
                ("index", C.c_int32), ("committed", C.c_int32)]


class RunMember(C.Structure):
    _fields_ = [("dataset", C.c_int32), ("batch", C.c_int32),
                ("epoch", C.c_int64), ("pos", C.c_int64), ("steps_done", C.c_int64),
                ("target_steps", C.c_int64), ("samples_used", C.c_void_p)]


class RunDataset(C.Structure):
    _fields_ = [("n", C.c_int64), ("dim", C.c_int32), ("max_label", C.c_int32),
                ("host_x", C.c_void_p), ("host_ld", C.c_int64), ("host_y", C.c_void_p),
                ("device", C.c_void_p), ("epoch0", C.c_int64), ("n_epochs", C.c_int32),
                ("perm", C.c_void_p), ("order", C.c_void_p),
                ("mapped_x", C.c_void_p), ("mapped_y", C.c_void_p)]


PK_RUN_MAX_STEPS, PK_RUN_NO_MEMBER, PK_RUN_NEED_PERM, PK_RUN_LABEL_BOUNDS, PK_RUN_FAILED = range(5)


class ConvGeom(C.Structure):
    _fields_ = [(f, C.c_int32) for f in ("n", "h", "w", "c", "k", "r", "s", "stride", "pad",
                                         "p", "q")]


# ---- conv pack program (packtrain_b200.h pk_cnn_*) ----------------------------------
CNN_KINDS = ("CONV_FPROP", "CONV_DGRAD", "CONV_WGRAD", "BN_STATS", "BN_APPLY", "BN_BWD_REDUCE",
             "BN_BWD_APPLY", "DW_FPROP", "DW_DGRAD", "DW_WGRAD", "MAXPOOL_FWD", "MAXPOOL_BWD",
             "AVGPOOL_FWD", "AVGPOOL_BWD", "XENT", "BIAS_ACT_BWD", "SPLIT_REDUCE", "OPT",
             "PUBLISH_T", "COMMIT", "GATHER", "IM2COL")
CNN = {k: i for i, k in enumerate(CNN_KINDS)}
CNN_ACT = {"none": 0, "relu": 1, "relu6": 2}
_vp, _i32, _i64, _f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float


def _ints(*names):
    return [(n, _i32) for n in names]


class CnnConv(C.Structure):
    _fields_ = ([("src", _vp), ("dy", _vp), ("wt", _vp), ("dst", _vp), ("idx", _vp),
                 ("bias", _vp), ("flag", _vp), ("dseg", _i64)]
                + _ints("n", "h", "w", "c", "k", "r", "s", "stride", "pad", "p", "q",
                        "ldx", "ldy", "ldo", "act", "out_f32", "accumulate", "splits", "nseg"))


class CnnBn(C.Structure):
    _fields_ = ([(n, _vp) for n in ("x", "res", "out", "dout", "fout", "dx", "dres", "gamma",
                                    "beta", "dgamma", "dbeta", "stats", "run_mean", "run_var",
                                    "ws", "counter", "flag")]
                + _ints("rows", "c", "ldx", "ldo", "ldr", "ldd", "ldx2", "act", "accumulate",
                        "res_accumulate", "use_running")
                + [("eps", _f32), ("momentum", _f32), ("rpb", _i32), ("pad0", _i32)])


class CnnDw(C.Structure):
    _fields_ = ([(n, _vp) for n in ("x", "wt", "dy", "y", "dw", "ws", "counter", "flag")]
                + _ints("n", "h", "w", "c", "r", "s", "stride", "pad", "p", "q", "ldx", "ldy",
                        "ppb", "pad0"))


class CnnPool(C.Structure):
    _fields_ = ([(n, _vp) for n in ("x", "y", "dy", "dx", "arg")]
                + _ints("n", "h", "w", "c", "r", "s", "stride", "pad", "p", "q", "ldx", "ldy",
                        "accumulate"))


class CnnHead(C.Structure):
    _fields_ = ([(n, _vp) for n in ("logits", "labels", "idx", "dlogits", "dbias", "loss",
                                    "flag")]
                + _ints("rows", "classes", "ldl"))


class CnnBias(C.Structure):
    _fields_ = ([(n, _vp) for n in ("dy", "fout", "g", "dbias", "ws", "counter", "flag")]
                + _ints("rows", "c", "ld", "act", "rpb", "pad0"))


class CnnReduce(C.Structure):
    _fields_ = [("src", _vp), ("dst", _vp), ("flag", _vp), ("len", _i64), ("splits", _i32),
                ("pad0", _i32)]


class CnnOptSeg(C.Structure):
    _fields_ = ([(n, _vp) for n in ("w", "g", "s1", "s2", "w16", "step", "flag")]
                + [("len", _i64), ("kind", _i32), ("lr", _f32), ("wd", _f32)])


class CnnTpose(C.Structure):
    _fields_ = [("src", _vp), ("dst", _vp)] + _ints("k", "c", "taps", "kpad", "kpadt", "pad0")


class CnnCommit(C.Structure):
    _fields_ = [("step", _vp), ("flag", _vp), ("verdict", _vp)]


class CnnGather(C.Structure):
    _fields_ = [("src", _vp), ("dst", _vp), ("idx", _vp), ("row_bytes", _i64), ("rows", _i32),
                ("pad0", _i32)]


class CnnIm2col(C.Structure):
    _fields_ = [("src", _vp), ("dst", _vp)] + _ints("n", "h", "w", "cp", "c", "r", "s", "stride",
                                                    "pad", "p", "q", "ldo")


class CnnOp(C.Structure):
    _fields_ = [("kind", _i32), ("nprob", _i32), ("cfg0", _i32), ("cfg1", _i32),
                ("lane", _i32), ("pad0", _i32), ("probs", _vp)]


CNN_STRUCT = {}
for _k in ("CONV_FPROP", "CONV_DGRAD", "CONV_WGRAD"):
    CNN_STRUCT[CNN[_k]] = CnnConv
for _k in ("BN_STATS", "BN_APPLY", "BN_BWD_REDUCE", "BN_BWD_APPLY"):
    CNN_STRUCT[CNN[_k]] = CnnBn
for _k in ("DW_FPROP", "DW_DGRAD", "DW_WGRAD"):
    CNN_STRUCT[CNN[_k]] = CnnDw
for _k in ("MAXPOOL_FWD", "MAXPOOL_BWD", "AVGPOOL_FWD", "AVGPOOL_BWD"):
    CNN_STRUCT[CNN[_k]] = CnnPool
CNN_STRUCT[CNN["XENT"]] = CnnHead
CNN_STRUCT[CNN["BIAS_ACT_BWD"]] = CnnBias
CNN_STRUCT[CNN["SPLIT_REDUCE"]] = CnnReduce
CNN_STRUCT[CNN["OPT"]] = CnnOptSeg
CNN_STRUCT[CNN["PUBLISH_T"]] = CnnTpose
CNN_STRUCT[CNN["COMMIT"]] = CnnCommit
CNN_STRUCT[CNN["GATHER"]] = CnnGather
CNN_STRUCT[CNN["IM2COL"]] = CnnIm2col


class PKError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        super().__init__(f"pk error {code}: {msg}")


_LIB = None
_LOCK = threading.Lock()


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load the shared library and declare signatures (no device needed)."""
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    L = C.CDLL(path)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    sig = {
        "pk_abi_version": (C.c_int, []),
        "pk_ctx_create": (C.c_int, [i32, i32, P(vp)]),
        "pk_ctx_destroy": (C.c_int, [vp]),
        "pk_ctx_last_error": (C.c_char_p, [vp]),
        "pk_ctx_set_stream": (C.c_int, [vp, vp]),
        "pk_ctx_synchronize": (C.c_int, [vp]),
        "pk_ctx_mem_info": (C.c_int, [vp, P(C.c_uint64), P(C.c_uint64), P(C.c_uint64)]),
        "pk_dataset_create": (C.c_int, [vp, i64, i32, P(vp)]),
        "pk_dataset_write": (C.c_int, [vp, i64, i64, vp, vp]),
        "pk_dataset_write_rows": (C.c_int, [vp, i64, i64, vp, vp]),
        "pk_dataset_gather_rows": (C.c_int, [vp, i64, vp, i64, vp, vp, vp, vp]),
        "pk_host_map": (C.c_int, [vp, vp, i64, vp]),
        "pk_host_unmap": (C.c_int, [vp, vp]),
        "pk_pack_run": (C.c_int, [vp, vp, vp, C.c_int32, C.c_int32, i64, C.c_int32, vp, vp, vp,
                                  vp, vp, vp]),
        "pk_dataset_destroy": (C.c_int, [vp]),
        "pk_order_create": (C.c_int, [vp, vp, i64, P(vp)]),
        "pk_order_destroy": (C.c_int, [vp]),
        "pk_member_create": (C.c_int, [vp, P(MemberDesc), P(vp)]),
        "pk_member_destroy": (C.c_int, [vp]),
        "pk_member_param_count": (i64, [vp]),
        "pk_member_slot_count": (i32, [vp]),
        "pk_member_device_bytes": (i64, [vp]),
        "pk_member_set_lr": (C.c_int, [vp, dbl]),
        "pk_member_set_state": (C.c_int, [vp, vp, vp, i64]),
        "pk_member_get_state": (C.c_int, [vp, vp, vp, P(i64)]),
        "pk_member_inject_fault": (C.c_int, [vp, i32]),
        "pk_pack_create": (C.c_int, [vp, P(vp), i32, P(vp)]),
        "pk_pack_destroy": (C.c_int, [vp]),
        "pk_pack_step": (C.c_int, [vp, P(Feed), P(dbl), P(Status)]),
        "pk_pack_step_async": (C.c_int, [vp, P(Feed), P(i64)]),
        "pk_pack_step_wait": (C.c_int, [vp, i64, P(dbl), P(Status)]),
        "pk_pack_eval": (C.c_int, [vp, vp, vp, i64, i64, P(dbl), P(Status)]),
        "pk_pack_profile_step": (C.c_int, [vp, P(Feed), P(C.c_float), P(i32), P(i32),
                                           P(i32), P(dbl), P(Status)]),
        "pk_pack_trace": (i64, [vp, vp, i64]),
        "pk_pack_launches_per_step": (i32, [vp]),
        "pk_plan_options_get": (C.c_int, [P(PlanOptions)]),
        "pk_plan_options_set": (C.c_int, [P(PlanOptions)]),
        "pk_conv_gemm_test": (C.c_int, [i32, P(ConvGeom), vp, vp, vp, vp, i32, i32, i32, vp]),
        "pk_cnn_prog_create": (C.c_int, [P(CnnOp), i32, i32, P(vp)]),
        "pk_cnn_prog_destroy": (None, [vp]),
        "pk_cnn_prog_run": (C.c_int, [vp, vp, i32]),
        "pk_cnn_prog_profile": (C.c_int, [vp, vp, P(C.c_float)]),
        "pk_cnn_prog_launches": (i32, [vp]),
        "pk_cnn_last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def lib() -> C.CDLL:
    global _LIB
    with _LOCK:
        if _LIB is None:
            _LIB = load_library()
    return _LIB


def check(ctx_ptr, rc):
    """Raise PKError for non-OK codes that are not step outcomes."""
    if rc in (PK_OK,):
        return rc
    msg = lib().pk_ctx_last_error(ctx_ptr) if ctx_ptr else b""
    raise PKError(rc, (msg or b"").decode(errors="replace"))
