"""Device objects over the C-ABI: runtime (one per process/GPU), resident
datasets and epoch orders, member slabs and packs.

This is plumbing for `packing.py`; it keeps no numerics of its own.  Every
call goes to `libpk_b200.so` — if the library or the GPU is missing the
first use raises (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from collections import OrderedDict

import numpy as np

from . import _lib as L

_RUNTIMES: dict = {}
_DEFAULT = {"device": None, "dtype": None, "inputs": None}
# environment defaults, read once (the step path asks for them every call)
_ENV = {"inputs": os.environ.get("PACKTRAIN_INPUTS", "resident"),
        "device": int(os.environ.get("PACKTRAIN_DEVICE", "0")),
        "dtype": os.environ.get("PACKTRAIN_PRECISION", "f32")}


def set_input_mode(mode: str):
    """'resident' (default): datasets are uploaded once and steps gather
    their rows on the device.  'stream': every step gathers its batch rows on
    the host into pinned memory and copies them H2D (the reference's
    per-step `_next_batch`, packing.py:161-172, as a real host→device feed)."""
    if mode not in ("resident", "stream"):
        raise ValueError("input mode must be 'resident' or 'stream'")
    _DEFAULT["inputs"] = mode


# host-side transport / driver options (the device kernel plan is
# _lib.set_plan_options): host_gather = streamed inputs gathered by the host into
# pinned memory + H2D copy instead of the device pulling rows over PCIe;
# py_run = packed_run stepped from Python instead of the native pk_pack_run
_OPTIONS = {"host_gather": False, "py_run": False}


def set_options(**kw) -> dict:
    """Set host-side runtime options; returns the previous values."""
    prev = dict(_OPTIONS)
    for k, v in kw.items():
        if k not in _OPTIONS:
            raise KeyError(f"unknown runtime option {k!r}")
        _OPTIONS[k] = bool(v)
    return prev


def option(name: str) -> bool:
    return _OPTIONS[name]


def input_mode() -> str:
    return _DEFAULT["inputs"] or _ENV["inputs"]


def set_device(device: int):
    """Select the GPU used by subsequently created handles/packs."""
    _DEFAULT["device"] = int(device)


def set_precision(dtype: str):
    """'f32' (default) or 'f64' device arithmetic for new runtimes."""
    if dtype not in ("f32", "f64"):
        raise ValueError("precision must be 'f32' or 'f64'")
    _DEFAULT["dtype"] = dtype


def default_device() -> int:
    if _DEFAULT["device"] is not None:
        return _DEFAULT["device"]
    return _ENV["device"]


def default_precision() -> str:
    return _DEFAULT["dtype"] or _ENV["dtype"]


def runtime(device: int | None = None, dtype: str | None = None) -> "Runtime":
    dev = default_device() if device is None else int(device)
    dt = dtype or default_precision()
    key = (dev, dt)
    rt = _RUNTIMES.get(key)
    if rt is None:
        rt = Runtime(dev, dt)
        _RUNTIMES[key] = rt
    return rt


class Runtime:
    """One pk_ctx: a device, a precision, a stream and the resident data."""

    ORDER_CACHE = 16

    def __init__(self, device: int, dtype: str):
        self.lib = L.lib()
        self.device = device
        self.dtype = dtype
        ptr = C.c_void_p()
        rc = self.lib.pk_ctx_create(device, L.PK_F64 if dtype == "f64" else L.PK_F32,
                                    C.byref(ptr))
        if rc != L.PK_OK:
            raise L.PKError(rc, f"cannot create context on cuda:{device} "
                                "(is a GPU visible and libpk_b200.so built for sm_100a?)")
        self.ptr = ptr
        self._datasets: dict = {}
        self._orders: OrderedDict = OrderedDict()
        self._host_orders: OrderedDict = OrderedDict()
        self._mapped: list = []

    def check(self, rc):
        return L.check(self.ptr, rc)

    def set_stream(self, stream_handle: int | None):
        self.check(self.lib.pk_ctx_set_stream(self.ptr, C.c_void_p(stream_handle or 0)))

    def synchronize(self):
        self.check(self.lib.pk_ctx_synchronize(self.ptr))

    def mem_info(self):
        f, t, m = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.check(self.lib.pk_ctx_mem_info(self.ptr, C.byref(f), C.byref(t), C.byref(m)))
        return f.value, t.value, m.value

    # ---- data -------------------------------------------------------------
    def dataset(self, ds) -> "DeviceDataset":
        """Device-resident copy of a reference-style Dataset (uploaded once)."""
        key = (ds.dataset_id, id(ds.features), ds.features.shape)
        d = self._datasets.get(key)
        if d is None:
            d = DeviceDataset(self, ds.n, ds.dim)
            d.write(0, ds.features, ds.labels)
            d._src = weakref.ref(ds.features) if _weakrefable(ds.features) else None
            self._datasets[key] = d
        return d

    def preprocessed(self, ds, spec):
        """Device-resident copy of `ds` with every sample through `spec`
        (SURVEY §8f-2): materialized once per (dataset, spec digest) on the
        host with the reference's per-index formulas, uploaded once; steps then
        gather rows on the device like any dataset.  Returns (device dataset,
        host f64 table)."""
        from .data import preprocess_all
        key = ("pre", ds.dataset_id, spec.digest(), id(ds.features), ds.features.shape)
        got = self._datasets.get(key)
        if got is None:
            table = preprocess_all(spec, ds.features)
            d = DeviceDataset(self, ds.n, ds.dim)
            d.write(0, table, ds.labels)
            got = (d, table)
            self._datasets[key] = got
        return got

    def host_rows_source(self, ds):
        """(features in device precision, int32 labels) host copies of `ds` for
        streamed gathers, made once per dataset."""
        key = ("rows", ds.dataset_id, id(ds.features), ds.features.shape)
        got = self._datasets.get(key)
        if got is None:
            got = (np.ascontiguousarray(ds.features,
                                        dtype=np.float64 if self.dtype == "f64" else np.float32),
                   np.ascontiguousarray(ds.labels, dtype=np.int32))
            self._datasets[key] = got
        return got

    def host_rows_mapped(self, ds):
        """Device views (x, y) of host_rows_source(ds), page-locked and mapped
        once per dataset: pk_pack_run's streamed steps let the GPU pull the
        batch rows over PCIe itself (no host memcpy per step)."""
        key = ("mapped", ds.dataset_id, id(ds.features), ds.features.shape)
        got = self._datasets.get(key)
        if got is None:
            x, y = self.host_rows_source(ds)
            dx, dy = C.c_void_p(), C.c_void_p()
            self.check(self.lib.pk_host_map(self.ptr, x.ctypes.data, x.nbytes, C.byref(dx)))
            self.check(self.lib.pk_host_map(self.ptr, y.ctypes.data, y.nbytes, C.byref(dy)))
            got = (dx.value, dy.value)
            self._datasets[key] = got
            self._mapped.append((x, y))  # page-locked for the runtime's lifetime
        return got

    def host_order(self, dataset_id: str, n: int, epoch: int, make) -> np.ndarray:
        key = (dataset_id, n, epoch)
        o = self._host_orders.get(key)
        if o is None:
            o = make()
            self._host_orders[key] = o
            while len(self._host_orders) > self.ORDER_CACHE:
                self._host_orders.popitem(last=False)
        else:
            self._host_orders.move_to_end(key)
        return o

    def order(self, dataset_id: str, n: int, epoch: int, make) -> "DeviceOrder":
        key = (dataset_id, n, epoch)
        o = self._orders.get(key)
        if o is None:
            o = DeviceOrder(self, self.host_order(dataset_id, n, epoch, make))
            self._orders[key] = o
            while len(self._orders) > self.ORDER_CACHE:
                self._orders.popitem(last=False)
        else:
            self._orders.move_to_end(key)
        return o


def _weakrefable(a):
    try:
        weakref.ref(a)
        return True
    except TypeError:
        return False


class DeviceDataset:
    def __init__(self, rt: Runtime, n: int, dim: int):
        self.rt, self.n, self.dim = rt, int(n), int(dim)
        ptr = C.c_void_p()
        rt.check(rt.lib.pk_dataset_create(rt.ptr, self.n, self.dim, C.byref(ptr)))
        self.ptr = ptr

    def write_rows_ptr(self, rows: int, x, y):
        """write_rows(0, x[:rows], y[:rows]) for contiguous pinned buffers,
        with their ctypes pointers cached."""
        key = (x.ctypes.data, y.ctypes.data)
        ptrs = getattr(self, "_wr_ptrs", None)
        if ptrs is None or ptrs[0] != key:
            ptrs = (key, C.c_void_p(key[0]), C.c_void_p(key[1]))
            self._wr_ptrs = ptrs
        self.rt.check(self.rt.lib.pk_dataset_write_rows(self.ptr, 0, int(rows), ptrs[1], ptrs[2]))

    def gather_rows(self, rows: int, x, y, idx, hx, hy):
        """Rows idx of the host source (x, y) → pinned staging (hx, hy) → H2D
        into rows [0, rows), in one library call (pointers of the long-lived
        buffers cached)."""
        key = (x.ctypes.data, y.ctypes.data, hx.ctypes.data, hy.ctypes.data)
        ptrs = getattr(self, "_gr_ptrs", None)
        if ptrs is None or ptrs[0] != key:
            ptrs = (key, *(C.c_void_p(v) for v in key), x.strides[0] // x.itemsize)
            self._gr_ptrs = ptrs
        if idx.dtype != np.int64 or not idx.flags.c_contiguous:
            idx = np.ascontiguousarray(idx, dtype=np.int64)
        self.rt.check(self.rt.lib.pk_dataset_gather_rows(
            self.ptr, int(rows), ptrs[1], ptrs[5], ptrs[2], idx.ctypes.data, ptrs[3], ptrs[4]))

    def write_rows(self, row0: int, x, y):
        """Async H2D of rows already in device precision (x) / int32 (y);
        x and y must stay alive until the stream syncs (pinned: true DMA)."""
        self.rt.check(self.rt.lib.pk_dataset_write_rows(
            self.ptr, int(row0), int(x.shape[0]), x.ctypes.data_as(C.c_void_p),
            y.ctypes.data_as(C.c_void_p)))

    def write(self, row0: int, features, labels):
        x = np.ascontiguousarray(features, dtype=np.float64)
        y = np.ascontiguousarray(labels, dtype=np.int64)
        rows = x.shape[0]
        self.rt.check(self.rt.lib.pk_dataset_write(
            self.ptr, int(row0), rows, x.ctypes.data_as(C.c_void_p),
            y.ctypes.data_as(C.c_void_p)))

    def __del__(self):
        try:
            if self.ptr:
                self.rt.lib.pk_dataset_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


class DeviceOrder:
    def __init__(self, rt: Runtime, perm: np.ndarray):
        self.rt = rt
        p = np.ascontiguousarray(perm, dtype=np.int64)
        self.n = len(p)
        ptr = C.c_void_p()
        rt.check(rt.lib.pk_order_create(rt.ptr, p.ctypes.data_as(C.c_void_p), self.n,
                                        C.byref(ptr)))
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr:
                self.rt.lib.pk_order_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


class DeviceMember:
    """A member's device slab: ping-pong params/slots, workspace, control."""

    def __init__(self, rt: Runtime, dims, activation: str, optimizer: str, lr: float,
                 max_rows: int, weight_decay: float = 0.0):
        if len(dims) - 1 > L.PK_MAX_LAYERS:
            raise ValueError(f"at most {L.PK_MAX_LAYERS} affine layers per member")
        self.rt = rt
        d = L.MemberDesc()
        d.n_layers = len(dims) - 1
        for i, v in enumerate(dims):
            d.dims[i] = int(v)
        d.activation = L.ACT_CODES[activation]
        d.optimizer = L.OPT_CODES[optimizer]
        d.learning_rate = float(lr)
        d.weight_decay = float(weight_decay)
        d.max_rows = int(max_rows)
        ptr = C.c_void_p()
        rt.check(rt.lib.pk_member_create(rt.ptr, C.byref(d), C.byref(ptr)))
        self.ptr = ptr
        self.desc = d
        self.n_params = rt.lib.pk_member_param_count(ptr)
        self.n_slots = rt.lib.pk_member_slot_count(ptr)
        self.device_bytes = rt.lib.pk_member_device_bytes(ptr)

    def inject_fault(self, grad_position: int):
        """Testing hook: NaN in gradient tensor `grad_position` next step."""
        self.rt.check(self.rt.lib.pk_member_inject_fault(self.ptr, int(grad_position)))

    def set_lr(self, lr: float):
        self.rt.check(self.rt.lib.pk_member_set_lr(self.ptr, float(lr)))

    def upload(self, flat_params: np.ndarray, flat_slots, step_counter: int):
        p = np.ascontiguousarray(flat_params, dtype=np.float64)
        assert p.size == self.n_params
        sp = None
        if flat_slots is not None and self.n_slots:
            s = np.ascontiguousarray(flat_slots, dtype=np.float64)
            assert s.size == self.n_slots * self.n_params
            sp = s.ctypes.data_as(C.c_void_p)
        self.rt.check(self.rt.lib.pk_member_set_state(
            self.ptr, p.ctypes.data_as(C.c_void_p), sp, int(step_counter)))

    def download(self, want_slots=True):
        p = np.empty(self.n_params, dtype=np.float64)
        s = np.empty(self.n_slots * self.n_params, dtype=np.float64) if (
            want_slots and self.n_slots) else None
        t = C.c_int64()
        self.rt.check(self.rt.lib.pk_member_get_state(
            self.ptr, p.ctypes.data_as(C.c_void_p),
            s.ctypes.data_as(C.c_void_p) if s is not None else None, C.byref(t)))
        return p, s, t.value

    def __del__(self):
        try:
            if self.ptr:
                self.rt.lib.pk_member_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


class DevicePack:
    """pk_pack over an ordered list of DeviceMembers (kept alive here)."""

    def __init__(self, rt: Runtime, members):
        self.rt = rt
        self.members = list(members)  # keep member slabs alive
        self.K = len(self.members)
        arr = (C.c_void_p * self.K)(*[m.ptr.value for m in self.members])
        ptr = C.c_void_p()
        rt.check(rt.lib.pk_pack_create(rt.ptr, arr, self.K, C.byref(ptr)))
        self.ptr = ptr
        self._feeds = (L.Feed * self.K)()
        self._losses = (C.c_double * self.K)()
        self._status = L.Status()
        self.launches = rt.lib.pk_pack_launches_per_step(ptr)

    def set_feed(self, k, ddata, dorder, pos, take, group=0):
        f = self._feeds[k]
        f.data = ddata.ptr.value if ddata is not None else None
        f.order = dorder.ptr.value if dorder is not None else None
        f.pos = int(pos)
        f.take = int(take)
        f.group = int(group)

    def clear_feeds(self):
        for k in range(self.K):
            self._feeds[k].take = 0
            self._feeds[k].data = None
            self._feeds[k].order = None

    def step(self):
        """Synchronous step: returns (status code, member, index, committed, losses)."""
        rc = self.rt.lib.pk_pack_step(self.ptr, self._feeds, self._losses,
                                      C.byref(self._status))
        if rc not in (L.PK_OK, L.PK_ERR_NONFINITE_VALUE, L.PK_ERR_NONFINITE_GRAD):
            self.rt.check(rc)
        st = self._status
        return st.code, st.member, st.index, st.committed, list(self._losses)

    def step_async(self) -> int:
        t = C.c_int64()
        self.rt.check(self.rt.lib.pk_pack_step_async(self.ptr, self._feeds, C.byref(t)))
        return t.value

    def wait(self, ticket: int):
        rc = self.rt.lib.pk_pack_step_wait(self.ptr, int(ticket), self._losses,
                                           C.byref(self._status))
        if rc not in (L.PK_OK, L.PK_ERR_NONFINITE_VALUE, L.PK_ERR_NONFINITE_GRAD):
            self.rt.check(rc)
        st = self._status
        return st.code, st.member, st.index, st.committed, list(self._losses)

    def profile(self):
        """One real step, un-graphed, timed per phase with CUDA events.
        Returns (status code, [(kind, layer, ctas, ms)], losses)."""
        n = self.launches
        ms = (C.c_float * n)()
        kind, layer, ctas = (C.c_int32 * n)(), (C.c_int32 * n)(), (C.c_int32 * n)()
        rc = self.rt.lib.pk_pack_profile_step(self.ptr, self._feeds, ms, kind, layer, ctas,
                                              self._losses, C.byref(self._status))
        if rc not in (L.PK_OK, L.PK_ERR_NONFINITE_VALUE, L.PK_ERR_NONFINITE_GRAD):
            self.rt.check(rc)
        phases = [(kind[i], layer[i], ctas[i], ms[i]) for i in range(n)]
        return self._status.code, phases, list(self._losses)

    def eval(self, ddata, dorder, pos, rows):
        rc = self.rt.lib.pk_pack_eval(self.ptr, ddata.ptr,
                                      dorder.ptr if dorder is not None else None,
                                      int(pos), int(rows), self._losses,
                                      C.byref(self._status))
        if rc not in (L.PK_OK, L.PK_ERR_NONFINITE_VALUE):
            self.rt.check(rc)
        st = self._status
        return st.code, st.member, st.index, list(self._losses)

    def __del__(self):
        try:
            if self.ptr:
                self.rt.lib.pk_pack_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass
