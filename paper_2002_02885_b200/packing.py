"""The pack / load / free primitives — drop-in for the reference's
`packtrain.packing` (packing.py:1-489) with the step executed on a B200.

Host side (this file): member handles, cursors, input grouping, epoch plans,
checkpoints — the same observable semantics as the reference.  Device side
(`pk_pack_step`): the whole packed train step — batch gather through the
epoch order, forward, softmax-xent, backward and every member's optimizer
update — as one CUDA-graph launch over all K members, with losses and a
commit status returned through a host-mapped ring.

State ownership: a handle's parameters and optimizer slots live on the GPU
once it has stepped.  `handle.params` / `handle.optimizer.slots` download on
read (float32 → float64 exactly) and mark the host copy authoritative, so an
in-place edit made by the caller is uploaded before the next step.
"""
from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass, field, replace

import numpy as np

from . import engine
from . import runtime as _rt
from .data import Dataset, account_cache, epoch_permutation, preprocess
from .engine import ComputationGraph
import ctypes as C

from . import _lib
from ._lib import PK_ERR_NONFINITE_GRAD, PK_ERR_NONFINITE_VALUE, PK_SKIPPED

CHECKPOINT_MAGIC = b"PKCK"
CHECKPOINT_VERSION = 1


class PackError(Exception):
    pass


class ReplanNeeded(PackError):
    """No member can take a step under the current epoch plan."""


@dataclass(frozen=True)
class MLPArch:
    input_dim: int
    hidden: tuple
    classes: int
    activation: str = "relu"

    @property
    def dims(self):
        return (self.input_dim, *self.hidden, self.classes)


@dataclass
class ProgressCursor:
    steps_done: int = 0
    epoch_index: int = 0
    pos: int = 0
    samples_used: np.ndarray | None = None

    def start_epoch(self, n: int):
        self.pos = 0
        self.samples_used = np.zeros(n, dtype=np.int64)


def _param_names(model_id, n_layers):
    out = []
    for i in range(n_layers):
        out += [f"{model_id}/L{i}/W", f"{model_id}/L{i}/b"]
    return out


class ModelHandle:
    """One member: arch, params, optimizer, batch size, target, cursor
    (packing.py:52-66), with its state mirrored in a device slab."""

    def __init__(self, model_id, arch: MLPArch, graph: ComputationGraph, params: dict,
                 optimizer: engine.OptimizerState, batch_size: int, target_steps: int,
                 dataset_binding: str, cursor: ProgressCursor | None = None,
                 weight_decay: float = 0.0):
        self.model_id = model_id
        self.arch = arch
        self.graph = graph
        self._params = params
        self.optimizer = optimizer
        optimizer._owner = self
        self.batch_size = batch_size
        self.target_steps = target_steps
        self.dataset_binding = dataset_binding
        self.cursor = cursor if cursor is not None else ProgressCursor()
        self.weight_decay = float(weight_decay)
        self._dev = None          # runtime.DeviceMember
        self._where = "host"      # host | device | synced
        self._solo = None         # cached singleton pack for standalone_step

    # -- observable state ---------------------------------------------------
    @property
    def params(self) -> dict:
        self._pull()
        self._host_authoritative()
        return self._params

    @params.setter
    def params(self, value):
        self._pull()
        self._params = value
        self._where = "host"

    @property
    def finished(self) -> bool:
        return self.cursor.steps_done >= self.target_steps

    @property
    def n_layers(self):
        return len(self.arch.hidden) + 1

    def __repr__(self):
        return (f"ModelHandle(model_id={self.model_id!r}, arch={self.arch!r}, "
                f"batch_size={self.batch_size}, target_steps={self.target_steps}, "
                f"steps_done={self.cursor.steps_done})")

    # -- device sync ----------------------------------------------------------
    def _flat_params(self, params):
        return np.concatenate([np.asarray(params[n], dtype=np.float64).ravel()
                               for n in _param_names(self.model_id, self.n_layers)])

    def _flat_slots(self):
        names = engine.SLOT_NAMES[self.optimizer.kind]
        slots = self.optimizer._slots
        if not names or not slots:
            return None
        parts = []
        for s in names:
            for n in _param_names(self.model_id, self.n_layers):
                arr = slots.get(n, {}).get(s)
                parts.append(np.zeros(int(np.prod(self._params[n].shape)))
                             if arr is None else np.asarray(arr, dtype=np.float64).ravel())
        return np.concatenate(parts)

    def _device(self, rt) -> "_rt.DeviceMember":
        """The member's device slab on runtime `rt`, uploaded if stale."""
        if self._dev is None or self._dev.rt is not rt:
            if self._dev is not None:
                self._pull()
            self._dev = _rt.DeviceMember(rt, self.arch.dims, self.arch.activation,
                                         self.optimizer.kind, self.optimizer.learning_rate,
                                         self.batch_size, self.weight_decay)
            self._where = "host"
            self._solo = None
        if self._where == "host":
            self._dev.upload(self._flat_params(self._params), self._flat_slots(),
                             self.optimizer._step)
            self._where = "synced"
        return self._dev

    def _pull(self):
        if self._where != "device":
            return
        flat, sflat, step = self._dev.download()
        off = 0
        for n in _param_names(self.model_id, self.n_layers):
            a = self._params[n]
            cnt = a.size
            np.copyto(a, flat[off:off + cnt].reshape(a.shape))
            off += cnt
        self.optimizer._step = int(step)
        names = engine.SLOT_NAMES[self.optimizer.kind]
        if names and (step > 0 or self.optimizer._slots):
            slots = self.optimizer._slots
            off = 0
            for s in names:
                for n in _param_names(self.model_id, self.n_layers):
                    shape = self._params[n].shape
                    cnt = int(np.prod(shape))
                    per = slots.setdefault(n, {})
                    v = sflat[off:off + cnt].reshape(shape)
                    if s in per and per[s].shape == shape:
                        np.copyto(per[s], v)
                    else:
                        per[s] = v.copy()
                    off += cnt
        self._where = "synced"

    def _host_authoritative(self):
        if self._where == "synced":
            self._where = "host"

    def _lr_changed(self):
        if self._dev is not None:
            self._dev.set_lr(self.optimizer.learning_rate)

    def _committed(self):
        self.optimizer._step += 1
        self._where = "device"


def make_handle(model_id, arch: MLPArch, optimizer, learning_rate, batch_size,
                target_steps, dataset_binding, seed, weight_decay=0.0) -> ModelHandle:
    """packing.py:69-81; `weight_decay` is the coupled-L2 extension.  A
    ConvArch member (BASELINE configs 1-4) gets a convpack.ConvModelHandle."""
    from .cnn import ConvArch
    if isinstance(arch, ConvArch):
        from .convpack import make_conv_handle
        return make_conv_handle(model_id, arch, optimizer, learning_rate, batch_size,
                                target_steps, dataset_binding, seed, weight_decay)
    if batch_size < 1 or target_steps < 1:
        raise PackError("batch_size and target_steps must be >= 1")
    graph = engine.build_mlp(model_id, arch.input_dim, arch.hidden, arch.classes,
                             arch.activation, dataset_binding)
    if len(arch.hidden) + 1 > 8:
        raise PackError("at most 7 hidden layers per member on the device path")
    return ModelHandle(model_id, arch, graph, engine.init_parameters(graph, seed),
                       engine.make_optimizer(optimizer, learning_rate), batch_size,
                       target_steps, dataset_binding, weight_decay=weight_decay)


def _fuse(members) -> ComputationGraph:
    """Merged graph description (packing.py:84-100)."""
    nodes, ins, labels, outs, heads, shapes = [], {}, {}, {}, {}, {}
    for h in members:
        g = h.graph
        nodes += g.nodes
        ins.update(g.input_ports)
        labels.update(g.label_ports)
        outs.update(g.output_ports)
        heads.update(g.loss_heads)
        shapes.update(g.param_shapes)
    return ComputationGraph("pack(" + ",".join(h.model_id for h in members) + ")",
                            nodes, ins, labels, outs, heads, shapes)


@dataclass
class PackedModel:
    members: list
    fused_graph: ComputationGraph
    share_inputs: bool = False
    last_step_stats: dict = field(default_factory=dict)
    _dev: object = field(default=None, repr=False, compare=False)
    _spec: object = field(default=None, repr=False, compare=False)  # speculated next plan
    _buf: int = field(default=0, repr=False, compare=False)         # stream staging parity

    @property
    def driver_batch(self) -> int:
        b = [m.batch_size for m in self.members if not m.finished]
        return max(b) if b else 0

    def member(self, model_id) -> ModelHandle:
        for h in self.members:
            if h.model_id == model_id:
                return h
        raise PackError(f"unknown model_id {model_id!r}")

    def _stream(self, rt, gi, x, y, buf=0):
        dev, hx, hy = _stream_staging(self, rt, (gi, buf), x.shape[0], x.shape[1])
        n = x.shape[0]
        hx[:n] = x  # f64 → device precision, round-to-nearest (as pk_dataset_write)
        hy[:n] = y
        dev.write_rows(0, hx[:n], hy[:n])
        return dev

    def _stream_rows(self, rt, gi, ds, idx, buf=0):
        """Streamed batch rows `idx` of `ds`: one np.take from the host copy in
        device precision (made once per dataset; float32(x) is what the H2D
        copy would carry anyway) into the pinned staging buffer, then H2D."""
        x, y = rt.host_rows_source(ds)
        n = len(idx)
        dev, hx, hy = _stream_staging(self, rt, (gi, buf), n, ds.dim)
        dev.gather_rows(n, x, y, idx, hx, hy)
        return dev

    def input_groups(self):
        """Members partitioned by (dataset, epoch, cursor, batch) (packing.py:121-128)."""
        g: dict = {}
        for h in self.members:
            g.setdefault((h.dataset_binding, h.cursor.epoch_index, h.cursor.pos,
                          h.batch_size), []).append(h)
        return [g[k] for k in sorted(g)]

    def pad_slice_plan(self):
        return {h.model_id: (0, h.batch_size) for h in self.members if not h.finished}

    def _device_pack(self, rt):
        """The pk_pack over all members (finished ones simply get take=0)."""
        key = (rt, tuple(id(h) for h in self.members))
        cached = self._dev
        devs = [h._device(rt) for h in self.members]
        if cached is None or cached[0] != key or any(
                a is not b for a, b in zip(cached[1].members, devs)):
            self._dev = (key, _rt.DevicePack(rt, devs), {})
        return self._dev[1]


def _pinned(shape, dtype):
    import torch
    t = torch.empty(shape, dtype={np.float32: torch.float32, np.float64: torch.float64,
                                  np.int32: torch.int32}[dtype], pin_memory=True)
    return t.numpy()


def _stream_staging(packed, rt, gi, rows, dim):
    """Per (pack, input group): a device staging dataset and pinned host
    buffers for streamed inputs (input_mode 'stream')."""
    stg = packed._dev[2]
    d = stg.get(gi)
    if d is None or d[0].n < rows or d[0].dim != dim:
        n = max(rows, packed.driver_batch)
        d = (_rt.DeviceDataset(rt, n, dim),
             _pinned((n, dim), np.float64 if rt.dtype == "f64" else np.float32),
             _pinned((n,), np.int32))
        stg[gi] = d
    return d


def pack_models(handles) -> PackedModel:
    """packing.py:136-142."""
    if not handles:
        raise PackError("pack needs at least one model")
    ids = [h.model_id for h in handles]
    if len(set(ids)) != len(ids):
        raise PackError(f"duplicate model_id in pack: {sorted(ids)}")
    from .convpack import ConvModelHandle, conv_pack_models
    conv = [isinstance(h, ConvModelHandle) for h in handles]
    if any(conv):
        if not all(conv):
            raise PackError("a pack holds either MLP or conv members, not both")
        return conv_pack_models(handles)
    return PackedModel(members=list(handles), fused_graph=_fuse(handles))


def dedup_inputs(packed: PackedModel) -> PackedModel:
    """Members of one input group share one physical input (packing.py:145-151).
    On the device every group is always read once; this flag only changes the
    reported `physical_inputs`, exactly as in the reference."""
    return replace(packed, share_inputs=True)


def _dataset_max_label(rt, ds):
    key = ("maxlabel", ds.dataset_id, id(ds.labels))
    v = rt._datasets.get(key)
    if v is None:
        v = int(np.max(ds.labels))
        rt._datasets[key] = v
    return v


def _order_fn(ds, epoch):
    return lambda: epoch_permutation(ds.dataset_id, ds.n, epoch)


def _roll_if_needed(handle: ModelHandle, datasets):
    """packing.py:175-182."""
    n = datasets[handle.dataset_binding].n
    cur = handle.cursor
    if cur.samples_used is None:
        cur.start_epoch(n)
    if cur.pos >= n:
        cur.epoch_index += 1
        cur.start_epoch(n)


def _node_name(h: ModelHandle, idx: int) -> str:
    n = h.n_layers
    if idx == 0:
        return f"{h.model_id}/in"
    if idx == 2 * n:
        return f"{h.model_id}/loss"
    return f"{h.model_id}/aff{(idx - 1) // 2}" if idx % 2 == 1 else f"{h.model_id}/act{(idx - 2) // 2}"


def _grad_name(h: ModelHandle, pos: int) -> str:
    layer = h.n_layers - 1 - pos // 2
    return f"{h.model_id}/L{layer}/{'W' if pos % 2 == 0 else 'b'}"


class _StepPlan:
    __slots__ = ("dpack", "index", "takes", "n_groups", "physical", "driver")


def _plan_step(packed: PackedModel, active, datasets, preprocess_spec, cache, curs=None,
               buf=0, dpack=None):
    """Host half of a packed step: input groups, batch rows and the per-member
    device feeds (packing.py:206-239).  Reads cursors (or the (epoch, pos)
    overrides in `curs`, for speculation), changes no member state."""
    rt = _rt.runtime()
    plan = _StepPlan()
    plan.driver = max(h.batch_size for h in active)
    groups: dict = {}
    for h in active:
        ep, ps = curs[id(h)] if curs is not None else (h.cursor.epoch_index, h.cursor.pos)
        groups.setdefault((h.dataset_binding, ep, ps, h.batch_size), []).append(h)
    if dpack is None:
        dpack = packed._device_pack(rt)
    plan.dpack = dpack
    plan.index = index = {id(h): k for k, h in enumerate(packed.members)}
    dpack.clear_feeds()
    plan.takes = takes = {}
    physical = 0
    for gi, key in enumerate(sorted(groups)):
        grp = groups[key]
        lead = grp[0]
        ds: Dataset = datasets[lead.dataset_binding]
        for h in grp:
            if ds.dim != h.arch.input_dim:
                raise engine.ShapeMismatch(f"{h.model_id}/x", ("batch", h.arch.input_dim),
                                           (plan.driver, ds.dim))
        _, c_epoch, c_pos, _ = key
        take = min(lead.batch_size, ds.n - c_pos)
        perm = rt.host_order(ds.dataset_id, ds.n, c_epoch, _order_fn(ds, c_epoch))
        idx = perm[c_pos:c_pos + take]
        if _dataset_max_label(rt, ds) >= min(h.arch.classes for h in grp):
            bad = [h for h in grp if int(ds.labels[idx].max()) >= h.arch.classes]
            if bad:
                raise IndexError(f"label out of bounds for member {bad[0].model_id!r} "
                                 f"with {bad[0].arch.classes} classes")
        if _rt.input_mode() == "stream":
            # host gather (+ per-sample preprocess) into pinned staging, H2D
            if preprocess_spec is not None and preprocess_spec.stages:
                x = preprocess(preprocess_spec, ds.features[idx], idx, ds.dataset_id, cache)
                src = packed._stream(rt, gi, x, ds.labels[idx], buf)
            else:  # gather straight from a device-precision host copy into pinned memory
                src = packed._stream_rows(rt, gi, ds, idx, buf)
            order, pos = None, 0
        else:
            if preprocess_spec is not None and preprocess_spec.stages:
                # device-resident preprocessed copy (memo over the whole
                # dataset); the PreprocessCache sees the reference's per-sample
                # bookkeeping
                src, table = rt.preprocessed(ds, preprocess_spec)
                if cache is not None:
                    account_cache(preprocess_spec, table, idx, ds.dataset_id, cache)
            else:
                src = rt.dataset(ds)
            order = rt.order(ds.dataset_id, ds.n, c_epoch, _order_fn(ds, c_epoch))
            pos = c_pos
        physical += 1 if packed.share_inputs else len(grp)
        for h in grp:
            dpack.set_feed(index[id(h)], src, order, pos, take, gi)
            takes[id(h)] = (idx, take)
    plan.n_groups = len(groups)
    plan.physical = physical
    return plan


def _apply_result(packed: PackedModel, active, plan: _StepPlan, code, who, where, losses):
    """Device status → the reference's exceptions and cursor updates
    (packing.py:246-257): a forward error commits nothing; a gradient error
    at member k leaves members before k committed."""
    if code == PK_SKIPPED:
        raise PackError("step skipped: an earlier in-flight step failed")
    if code == PK_ERR_NONFINITE_VALUE:
        raise engine.EngineError(
            f"non-finite value at node {_node_name(packed.members[who], where)!r}")
    out = {}
    for h in active:
        k = plan.index[id(h)]
        if code == PK_ERR_NONFINITE_GRAD and k == who:
            raise engine.NonFiniteGradient(_grad_name(h, where))
        h._committed()
        idx, take = plan.takes[id(h)]
        h.cursor.steps_done += 1
        h.cursor.pos += take
        h.cursor.samples_used[idx] += 1
        out[h.model_id] = losses[k]
    return out


def _state_key(packed, active, curs, datasets, stop_at_epoch_end, dpack):
    """Everything a step plan depends on besides member parameters."""
    return (dpack, stop_at_epoch_end, _rt.input_mode(), packed.share_inputs,
            tuple((id(h), curs[id(h)] if curs is not None else
                   (h.cursor.epoch_index, h.cursor.pos), h.batch_size, h.dataset_binding,
                   id(datasets[h.dataset_binding])) for h in active))


def _speculate(packed, active, plan, datasets, stop_at_epoch_end, buf):
    """While step n runs on the device, plan step n+1 assuming step n
    commits: shadow cursors advance by their take and roll epochs exactly as
    _active_members would (packing.py:175-204).  The plan is used only if the
    real state at the next call matches its key."""
    try:
        shadow, nxt = {}, []
        for h in packed.members:
            c = h.cursor
            ep, pos, steps = c.epoch_index, c.pos, c.steps_done
            if id(h) in plan.takes:
                steps += 1
                pos += plan.takes[id(h)][1]
            if steps >= h.target_steps:
                continue
            n = datasets[h.dataset_binding].n
            if c.samples_used is None:
                pos = 0
            if pos >= n:
                if stop_at_epoch_end:
                    continue
                ep, pos = ep + 1, 0
            shadow[id(h)] = (ep, pos)
            nxt.append(h)
        if not nxt:
            return None
        nplan = _plan_step(packed, nxt, datasets, None, None, curs=shadow, buf=buf)
        return _state_key(packed, nxt, shadow, datasets, stop_at_epoch_end, nplan.dpack), nplan
    except Exception:  # the real call recomputes (and raises) if needed
        return None


def _native_run(packed: PackedModel, datasets, max_steps: int, depth: int):
    """packed_run through the library's native driver (pk_pack_run): the same
    plan / apply semantics as the Python loop below, host cost per step a few
    microseconds.  Returns (loss dicts, finished) — finished False means the
    remaining steps need the Python loop (a label out of bounds)."""
    rt = _rt.runtime()
    out = []
    K = len(packed.members)
    stream = _rt.input_mode() == "stream"
    bindings = sorted({h.dataset_binding for h in packed.members})
    for h in packed.members:
        if datasets[h.dataset_binding].dim != h.arch.input_dim:
            return out, False  # the Python planner raises ShapeMismatch
    while len(out) < max_steps:
        try:
            active = _active_members(packed, datasets, False)
        except ReplanNeeded:
            return out, True
        dpack = packed._device_pack(rt)
        mem = (_lib.RunMember * K)()
        keep = []
        for k, h in enumerate(packed.members):
            c = h.cursor
            m = mem[k]
            m.dataset = bindings.index(h.dataset_binding)
            m.batch = h.batch_size
            m.epoch, m.pos, m.steps_done = c.epoch_index, c.pos, c.steps_done
            m.target_steps = h.target_steps
            su = c.samples_used
            if su is not None:
                if su.dtype != np.int64 or not su.flags.c_contiguous:
                    c.samples_used = su = np.ascontiguousarray(su, dtype=np.int64)
                m.samples_used = su.ctypes.data
        dsa = (_lib.RunDataset * len(bindings))()
        for i, b in enumerate(bindings):
            ds = datasets[b]
            # every epoch the remaining steps can reach (each re-entry drains the
            # in-flight window, so give the driver the whole horizon at once)
            mine = [h for h in packed.members if h.dataset_binding == b]
            e0 = min(h.cursor.epoch_index for h in mine)
            e1 = e0
            for h in mine:
                left = min(h.target_steps - h.cursor.steps_done, max_steps - len(out))
                if left > 0:
                    reach = h.cursor.pos + left * h.batch_size
                    e1 = max(e1, h.cursor.epoch_index + -(-reach // ds.n))
            e1 = min(e1, e0 + 64)
            perms = [np.ascontiguousarray(rt.host_order(ds.dataset_id, ds.n, e, _order_fn(ds, e)),
                                          dtype=np.int64) for e in range(e0, e1 + 1)]
            pa = (C.c_void_p * len(perms))(*[q.ctypes.data for q in perms])
            x, y = rt.host_rows_source(ds)
            d = dsa[i]
            d.n, d.dim, d.max_label = ds.n, ds.dim, _dataset_max_label(rt, ds)
            d.host_y = y.ctypes.data
            d.epoch0, d.n_epochs, d.perm = e0, len(perms), C.cast(pa, C.c_void_p)
            keep += [perms, pa, x, y]
            # device orders: the resident gather, and the GPU's own gather of
            # streamed rows from page-locked host memory
            orders = [rt.order(ds.dataset_id, ds.n, e, _order_fn(ds, e)) for e in range(e0, e1 + 1)]
            oa = (C.c_void_p * len(orders))(*[o.ptr.value for o in orders])
            d.order = C.cast(oa, C.c_void_p)
            keep += [orders, oa]
            if stream:
                d.host_x, d.host_ld = x.ctypes.data, x.strides[0] // x.itemsize
                if not _rt.option("host_gather"):
                    d.mapped_x, d.mapped_y = rt.host_rows_mapped(ds)
            else:
                dev = rt.dataset(ds)
                d.device = dev.ptr.value
                keep.append(dev)
        n = max_steps - len(out)
        losses = np.empty((n, K), dtype=np.float64)
        act = np.empty((n, K), dtype=np.uint8)
        stats = np.empty((n, 3), dtype=np.int32)
        done, stop, st = C.c_int64(), C.c_int32(), _lib.Status()
        rt.check(rt.lib.pk_pack_run(dpack.ptr, mem, dsa, len(bindings), int(packed.share_inputs),
                                    n, int(depth), losses.ctypes.data, act.ctypes.data,
                                    stats.ctypes.data, C.byref(done), C.byref(st), C.byref(stop)))
        nd = done.value
        code = stop.value
        rows = nd + (1 if code == _lib.PK_RUN_FAILED and nd < n else 0)  # + a partial commit
        for k, h in enumerate(packed.members):  # cursors → handles
            c = h.cursor
            c.epoch_index, c.pos = int(mem[k].epoch), int(mem[k].pos)
            stepped = int(act[:rows, k].sum())
            c.steps_done = int(mem[k].steps_done)
            for _ in range(stepped):
                h._committed()
        mids = [h.model_id for h in packed.members]
        for i in range(nd):
            out.append({mids[k]: float(losses[i, k]) for k in range(K) if act[i, k]})
        if nd:
            g, ph, dr = (int(v) for v in stats[nd - 1])
            packed.last_step_stats = {"physical_inputs": ph, "groups": g, "driver_batch": dr}
        if code == _lib.PK_RUN_FAILED:
            who = packed.members[st.member]
            # on a gradient error the members before `who` committed inside the
            # library; the failed step's losses are not returned (as in Python)
            if st.code == PK_ERR_NONFINITE_VALUE:
                raise engine.EngineError(f"non-finite value at node {_node_name(who, st.index)!r}")
            raise engine.NonFiniteGradient(_grad_name(who, st.index))
        if code == _lib.PK_RUN_LABEL_BOUNDS:
            return out, False
        if code == _lib.PK_RUN_NO_MEMBER and len(out) < max_steps:
            return out, True
        # PK_RUN_NEED_PERM: loop with the next epochs' permutations
    return out, True


def packed_run(packed: PackedModel, datasets, max_steps: int, depth: int = 16,
               native: bool = True) -> list:
    """Up to `max_steps` packed_step calls with up to `depth` in flight.  The
    native driver (pk_pack_run) plans and applies the steps in the library;
    the Python sliding window below is the same loop (and the fallback for
    anything the native loop hands back).  Both produce the reference
    packed_step loop's state bit for bit."""
    out = []
    if native and max_steps > 0 and not _rt.option("py_run"):
        out, finished = _native_run(packed, datasets, max_steps, depth)
        packed._spec = None
        if finished or len(out) >= max_steps:
            return out
    return out + _py_run(packed, datasets, max_steps - len(out), depth)


def _py_run(packed: PackedModel, datasets, max_steps: int, depth: int = 16) -> list:
    """Up to `max_steps` packed_step calls (reference semantics, packing.py:185-264)
    with up to `depth` steps in flight on the device: a sliding window — the
    host plans step n+depth from shadow cursors (epoch rolls and finished
    members exactly as _active_members) and enqueues it as soon as step n's
    result has been applied, so the device never drains between steps.  If a
    step raises (non-finite value / gradient), the device has skipped every
    later step (halt flag), so the state is exactly the reference's at that
    exception.  Stops early when no member is left; returns the per-step loss
    dicts."""
    from collections import deque
    out = []
    if max_steps <= 0:
        return out
    try:
        act = _active_members(packed, datasets, False)
    except ReplanNeeded:
        return out
    shadow = {id(h): (h.cursor.epoch_index, h.cursor.pos, h.cursor.steps_done)
              for h in packed.members}
    dpack = packed._device_pack(_rt.runtime())  # host-side edits synced once
    inflight = deque()
    curs, planned, more = None, 0, True
    try:
        while len(out) < max_steps:
            while more and len(inflight) < depth and planned < max_steps:
                # stream mode: every in-flight step owns a pinned + device
                # staging slot; a slot is reused only after its step was waited
                plan = _plan_step(packed, act, datasets, None, None, curs=curs, dpack=dpack,
                                  buf=2 + planned % depth)
                inflight.append((act, plan, plan.dpack.step_async()))
                planned += 1
                nact, ncurs = [], {}
                for h in packed.members:  # shadow state after this step commits
                    ep, pos, steps = shadow[id(h)]
                    if id(h) in plan.takes:
                        steps += 1
                        pos += plan.takes[id(h)][1]
                    shadow[id(h)] = (ep, pos, steps)
                    if steps >= h.target_steps:
                        continue
                    n = datasets[h.dataset_binding].n
                    if pos >= n:
                        ep, pos = ep + 1, 0
                        shadow[id(h)] = (ep, pos, steps)
                    ncurs[id(h)] = (ep, pos)
                    nact.append(h)
                more = bool(nact)
                act, curs = nact, ncurs
            if not inflight:
                break
            a, plan, ticket = inflight.popleft()
            code, who, where, _, losses = plan.dpack.wait(ticket)
            if out:  # the reference rolls epochs at the top of each packed_step
                for h in a:
                    _roll_if_needed(h, datasets)
            out.append(_apply_result(packed, a, plan, code, who, where, losses))
            packed.last_step_stats = {"physical_inputs": plan.physical,
                                      "groups": plan.n_groups, "driver_batch": plan.driver}
    finally:
        # a raised step: the later in-flight steps were skipped on the device;
        # drain their tickets so no staging slot or ring entry is left busy
        for _, plan, ticket in inflight:
            try:
                plan.dpack.wait(ticket)
            except _lib.PKError:  # PK_SKIPPED: nothing was committed
                pass
        packed._spec = None
    return out


def _device_step(packed: PackedModel, active, datasets, preprocess_spec, cache,
                 stop_at_epoch_end=False):
    spec = packed._spec
    packed._spec = None
    plan = None
    plain = preprocess_spec is None or not preprocess_spec.stages
    if spec is not None and plain:
        dpack = packed._device_pack(_rt.runtime())  # syncs host-side parameter edits
        if spec[0] == _state_key(packed, active, None, datasets, stop_at_epoch_end, dpack):
            plan = spec[1]
    if plan is None:
        packed._buf ^= 1
        plan = _plan_step(packed, active, datasets, preprocess_spec, cache, buf=packed._buf)
    ticket = plan.dpack.step_async()
    if plain:  # host planning of the next step overlaps this one on the device
        packed._buf ^= 1
        packed._spec = _speculate(packed, active, plan, datasets, stop_at_epoch_end, packed._buf)
    code, who, where, _, losses = plan.dpack.wait(ticket)
    out = _apply_result(packed, active, plan, code, who, where, losses)
    return out, plan.n_groups, plan.physical, plan.driver


def _active_members(packed, datasets, stop_at_epoch_end):
    active = [h for h in packed.members if not h.finished]
    if not stop_at_epoch_end:
        for h in active:
            _roll_if_needed(h, datasets)
    else:
        for h in active:
            if h.cursor.samples_used is None:
                h.cursor.start_epoch(datasets[h.dataset_binding].n)
        active = [h for h in active if h.cursor.pos < datasets[h.dataset_binding].n]
    if not active:
        raise ReplanNeeded("no member has both remaining steps and epoch data")
    return active


def packed_step(packed: PackedModel, datasets, preprocess_spec=None, cache=None,
                stop_at_epoch_end=False):
    """Train every active member for exactly one synchronized step
    (packing.py:185-264).  Returns {model_id: loss}."""
    from .convpack import ConvPackedModel, conv_packed_step
    if isinstance(packed, ConvPackedModel):
        return conv_packed_step(packed, datasets, preprocess_spec, cache, stop_at_epoch_end)
    active = _active_members(packed, datasets, stop_at_epoch_end)
    losses, n_groups, physical, driver = _device_step(packed, active, datasets,
                                                      preprocess_spec, cache,
                                                      stop_at_epoch_end)
    packed.last_step_stats = {"physical_inputs": physical, "groups": n_groups,
                              "driver_batch": driver}
    return losses


def standalone_step(handle: ModelHandle, datasets, preprocess_spec=None, cache=None):
    """One unpacked step (packing.py:267-282): the same device kernels on a
    one-member pack, so a packed member's trajectory equals its standalone
    one bit for bit."""
    from .convpack import ConvModelHandle, conv_standalone_step
    if isinstance(handle, ConvModelHandle):
        return conv_standalone_step(handle, datasets, preprocess_spec, cache)
    if handle.finished:
        raise PackError(f"{handle.model_id}: no remaining steps")
    _roll_if_needed(handle, datasets)
    if handle._solo is None or handle._solo.members[0] is not handle:
        handle._solo = pack_models([handle])
    losses, _, _, _ = _device_step(handle._solo, [handle], datasets, preprocess_spec, cache)
    return losses[handle.model_id]


def make_epoch_plan(members, datasets):
    """Phases (driver model_id, steps) covering one epoch (packing.py:285-319)."""
    if not members:
        raise PackError("epoch plan needs at least one member")
    state = {}
    for h in members:
        n = datasets[h.dataset_binding].n
        state[h.model_id] = [h.cursor.pos if h.cursor.samples_used is not None else 0, n]
    batch = {h.model_id: h.batch_size for h in members}
    plan = []
    while any(p < n for p, n in state.values()):
        live = [mid for mid, (p, n) in state.items() if p < n]
        driver = min(live, key=lambda mid: (-batch[mid], mid))
        steps = 0
        done = False
        while not done:
            for mid in live:
                p, n = state[mid]
                if p >= n:
                    continue
                p += min(batch[mid], n - p)
                state[mid][0] = p
                done = done or p >= n
            steps += 1
        plan.append((driver, steps))
    return plan


def run_epoch(packed: PackedModel, datasets, preprocess_spec=None, cache=None):
    """Packed steps until every member's epoch is exhausted (packing.py:322-330)."""
    out = []
    while True:
        try:
            out.append(packed_step(packed, datasets, preprocess_spec, cache,
                                   stop_at_epoch_end=True))
        except ReplanNeeded:
            return out


# ------------------------------------------------------------ checkpoints --
# PKCK v1, byte-compatible with packing.py:333-417: magic, u32 version,
# payload, sha256(payload).

@dataclass(frozen=True)
class Checkpoint:
    model_id: str
    payload: bytes
    digest: bytes

    def to_bytes(self) -> bytes:
        return CHECKPOINT_MAGIC + struct.pack("<I", CHECKPOINT_VERSION) + self.payload + self.digest

    @classmethod
    def from_bytes(cls, raw: bytes) -> "Checkpoint":
        if raw[:4] != CHECKPOINT_MAGIC:
            raise PackError("bad checkpoint magic")
        (ver,) = struct.unpack_from("<I", raw, 4)
        if ver != CHECKPOINT_VERSION:
            raise PackError(f"unsupported checkpoint version {ver}")
        payload, digest = raw[8:-32], raw[-32:]
        if hashlib.sha256(payload).digest() != digest:
            raise PackError("checkpoint digest mismatch")
        mid, _ = _Reader(payload).str_()
        return cls(model_id=mid, payload=payload, digest=digest)


class _Writer:
    def __init__(self):
        self.parts = []

    def raw(self, fmt, *v):
        self.parts.append(struct.pack(fmt, *v))

    def str_(self, s: str):
        b = s.encode()
        self.raw("<H", len(b))
        self.parts.append(b)

    def tensor(self, a):
        a = np.asarray(a, dtype=np.float64)
        self.raw("<B", a.ndim)
        if a.ndim:
            self.raw(f"<{a.ndim}Q", *a.shape)
        self.parts.append(a.astype("<f8").tobytes())

    def bytes(self):
        return b"".join(self.parts)


class _Reader:
    def __init__(self, buf):
        self.buf, self.off = buf, 0

    def raw(self, fmt):
        v = struct.unpack_from(fmt, self.buf, self.off)
        self.off += struct.calcsize(fmt)
        return v

    def str_(self):
        (n,) = self.raw("<H")
        s = self.buf[self.off:self.off + n].decode()
        self.off += n
        return s, self.off

    def tensor(self):
        (nd,) = self.raw("<B")
        shape = self.raw(f"<{nd}Q") if nd else ()
        cnt = int(np.prod(shape)) if shape else 1
        a = np.frombuffer(self.buf, dtype="<f8", count=cnt, offset=self.off)
        self.off += 8 * cnt
        return a.reshape(shape).copy()


def checkpoint_model(handle: ModelHandle) -> Checkpoint:
    """Device → host download into the PKCK payload (packing.py:387-417)."""
    params = handle.params
    opt = handle.optimizer
    w = _Writer()
    w.str_(handle.model_id)
    a = handle.arch
    w.raw("<IIB", a.input_dim, a.classes, len(a.hidden))
    if a.hidden:
        w.raw(f"<{len(a.hidden)}I", *a.hidden)
    w.str_(a.activation)
    w.str_(handle.dataset_binding)
    w.raw("<IQ", handle.batch_size, handle.target_steps)
    w.str_(opt.kind)
    w.raw("<dQ", opt.learning_rate, opt.step_counter)
    names = sorted(params)
    w.raw("<I", len(names))
    for n in names:
        w.str_(n)
        w.tensor(params[n])
    slots = opt.slots
    items = [(p, s, slots[p][s]) for p in sorted(slots) for s in sorted(slots[p])]
    w.raw("<I", len(items))
    for p, s, arr in items:
        w.str_(p)
        w.str_(s)
        w.tensor(arr)
    c = handle.cursor
    w.raw("<QQQ", c.steps_done, c.epoch_index, c.pos)
    payload = w.bytes()
    return Checkpoint(handle.model_id, payload, hashlib.sha256(payload).digest())


def restore_handle(ckpt: Checkpoint, datasets=None) -> ModelHandle:
    """packing.py:420-465."""
    r = _Reader(ckpt.payload)
    mid, _ = r.str_()
    input_dim, classes, nh = r.raw("<IIB")
    hidden = r.raw(f"<{nh}I") if nh else ()
    act, _ = r.str_()
    binding, _ = r.str_()
    batch, target = r.raw("<IQ")
    kind, _ = r.str_()
    lr, step = r.raw("<dQ")
    (np_,) = r.raw("<I")
    params = {}
    for _ in range(np_):
        n, _ = r.str_()
        params[n] = r.tensor()
    (ns,) = r.raw("<I")
    opt = engine.make_optimizer(kind, lr)
    opt._step = step
    for _ in range(ns):
        p, _ = r.str_()
        s, _ = r.str_()
        opt._slots.setdefault(p, {})[s] = r.tensor()
    steps_done, epoch, pos = r.raw("<QQQ")
    arch = MLPArch(input_dim, tuple(hidden), classes, act)
    graph = engine.build_mlp(mid, input_dim, tuple(hidden), classes, act, binding)
    cur = ProgressCursor(steps_done=steps_done, epoch_index=epoch, pos=pos)
    if datasets is not None and binding in datasets:
        ds = datasets[binding]
        cur.samples_used = np.zeros(ds.n, dtype=np.int64)
        cur.samples_used[epoch_permutation(ds.dataset_id, ds.n, epoch)[:pos]] = 1
    return ModelHandle(mid, arch, graph, params, opt, batch, target, binding, cur)


def free_model(packed: PackedModel, model_id):
    """Checkpoint one member and drop it from the pack (packing.py:468-478)."""
    h = packed.member(model_id)
    rest = [m for m in packed.members if m.model_id != model_id]
    ckpt = checkpoint_model(h)
    h._dev = None  # release the member's device slab
    h._where = "host"
    h._solo = None
    return ckpt, PackedModel(members=rest, fused_graph=_fuse(rest),
                             share_inputs=packed.share_inputs)


def load_model(obj, device=None, datasets=None) -> ModelHandle:
    """Restore a checkpoint (or take a handle) and register its device bytes
    with an accountant (packing.py:481-489).  `device` is any object with a
    `register(model_id, nbytes)` method, e.g. device.DeviceAccountant."""
    h = restore_handle(obj, datasets) if isinstance(obj, Checkpoint) else obj
    if device is not None:
        from .device import member_device_bytes
        device.register(h.model_id, member_device_bytes(h.arch, h.optimizer.kind,
                                                        h.batch_size, _rt.default_precision()))
    return h
