"""Conv members behind the reference's pack API (make_handle / pack_models /
dedup_inputs / packed_step / standalone_step, packing.py:69-282).

`packing.make_handle(..., arch=ConvArch(...), ...)` returns a ConvModelHandle;
`packing.pack_models` of conv handles returns a ConvPackedModel, and
`packing.packed_step` / `standalone_step` dispatch here.  The host semantics
are the reference's: active members and epoch rolls (packing.py:193-204), the
driver batch (:206), input groups keyed (binding, epoch, pos, batch) (:207-211),
take = min(b, n - pos) per group (:167), cursor advance and samples_used
(:255-257), last_step_stats (:259-263), and a non-finite gradient stopping the
per-member update loop at that member (:250-253, engine.py:297-299).  The step
itself is one pk_cnn_prog launch sequence (cnn.py) on the current torch
stream; losses and commit verdicts come back in one 16·K-byte read.
"""
from __future__ import annotations

import threading
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import cnn, engine
from . import runtime as _rt
from .cnn import ConvArch
from .data import epoch_permutation


class ConvModelHandle:
    """One conv member (the ModelHandle of packing.py:52-66 for a ConvArch).
    Parameters / optimizer slots live on the device once the member has
    stepped; `params`, `optimizer.slots` and `run_stats` download on read."""

    def __init__(self, model_id, arch: ConvArch, params: dict,
                 optimizer: engine.OptimizerState, batch_size: int, target_steps: int,
                 dataset_binding: str, cursor=None, weight_decay: float = 0.0):
        from .packing import ProgressCursor
        self.model_id = model_id
        self.arch = arch
        self.net = cnn.build_net(arch)
        self._params = params
        self.optimizer = optimizer
        optimizer._owner = self
        self.batch_size = int(batch_size)
        self.target_steps = int(target_steps)
        self.dataset_binding = dataset_binding
        self.cursor = cursor if cursor is not None else ProgressCursor()
        self.weight_decay = float(weight_decay)
        self._run_stats = {}
        self._home = None       # (ConvPack, member index) holding the device state
        self._where = "host"    # host | synced | device
        self._solo = None

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
    def run_stats(self) -> dict:
        """BN running (mean, var) per BN layer name (eval-mode statistics)."""
        self._pull()
        return self._run_stats

    @property
    def finished(self) -> bool:
        return self.cursor.steps_done >= self.target_steps

    def __repr__(self):
        return (f"ConvModelHandle(model_id={self.model_id!r}, arch={self.arch!r}, "
                f"batch_size={self.batch_size}, target_steps={self.target_steps}, "
                f"steps_done={self.cursor.steps_done})")

    # -- device sync -------------------------------------------------------------
    def _pull(self):
        if self._where != "device":
            return
        cp, k = self._home
        params, slots, step, rs = cp.get_member_state(k)
        for n, a in params.items():
            self._params[n] = a
        self.optimizer._slots = slots if slots else self.optimizer._slots
        self.optimizer._step = step
        self._run_stats = rs
        self._where = "synced"

    def _host_authoritative(self):
        if self._where == "synced":
            self._where = "host"

    def _lr_changed(self):
        if self._home is not None:
            cp, k = self._home
            cp.set_lr(k, self.optimizer.learning_rate)

    def _bind(self, cp, k):
        """Make (cp, k) hold this member's current state."""
        if self._home is None or self._home[0] is not cp or self._home[1] != k:
            self._pull()
            self._home = (cp, k)
            self._where = "host"
        if self._where == "host":
            cp.members[k].lr = self.optimizer.learning_rate
            cp.set_member_state(k, self._params, self.optimizer._slots, self.optimizer._step,
                                self._run_stats)
            self._where = "synced"

    def _committed(self):
        self.optimizer._step += 1
        self._where = "device"


def make_conv_handle(model_id, arch: ConvArch, optimizer, learning_rate, batch_size,
                     target_steps, dataset_binding, seed, weight_decay=0.0):
    from .packing import PackError
    if batch_size < 1 or target_steps < 1:
        raise PackError("batch_size and target_steps must be >= 1")
    net = cnn.build_net(arch)
    return ConvModelHandle(model_id, arch, cnn.init_parameters(net, model_id, seed),
                           engine.make_optimizer(optimizer, learning_rate), batch_size,
                           target_steps, dataset_binding, weight_decay=weight_decay)


@dataclass
class ConvPackedModel:
    members: list
    share_inputs: bool = False
    last_step_stats: dict = field(default_factory=dict)
    _cp: object = field(default=None, repr=False, compare=False)

    @property
    def driver_batch(self) -> int:
        b = [m.batch_size for m in self.members if not m.finished]
        return max(b) if b else 0

    def member(self, model_id):
        from .packing import PackError
        for h in self.members:
            if h.model_id == model_id:
                return h
        raise PackError(f"unknown model_id {model_id!r}")

    def input_groups(self):
        g: dict = {}
        for h in self.members:
            g.setdefault((h.dataset_binding, h.cursor.epoch_index, h.cursor.pos,
                          h.batch_size), []).append(h)
        return [g[k] for k in sorted(g)]

    def pad_slice_plan(self):
        return {h.model_id: (0, h.batch_size) for h in self.members if not h.finished}

    def device_pack(self, device=None):
        """The ConvPack over all members (finished members get take = 0)."""
        if self._cp is None:
            import torch
            dev = torch.cuda.current_device() if device is None else device
            specs = [cnn.MemberSpec(h.model_id, h.net, h.batch_size, h.optimizer.kind,
                                    h.optimizer.learning_rate, h.weight_decay)
                     for h in self.members]
            groups: dict = {}
            for k, h in enumerate(self.members):
                groups.setdefault((h.dataset_binding, h.batch_size), []).append(k)
            self._cp = cnn.ConvPack(specs, [groups[g] for g in sorted(groups)], dev)
        for k, h in enumerate(self.members):
            h._bind(self._cp, k)
        return self._cp


def conv_pack_models(handles) -> ConvPackedModel:
    return ConvPackedModel(members=list(handles))


# ---- device datasets and epoch orders ---------------------------------------------
_DATA: dict = {}   # id(dataset) -> {(image, device): DeviceConvDataset}
_LOCK = threading.RLock()  # the caches below are shared by concurrent packs' threads


def device_dataset(ds, image, device, host=False):
    """The NHWC bf16 copy of `ds` the step reads (made once per dataset object,
    device and placement): HBM-resident, or page-locked host memory for the
    streamed input mode (runtime.set_input_mode("stream"))."""
    with _LOCK:
        per = _DATA.get(id(ds))
        if per is None:
            per = {}
            _DATA[id(ds)] = per
            weakref.finalize(ds, _DATA.pop, id(ds), None)
        key = (tuple(image), device, host)
        d = per.get(key)
        if d is None:
            import torch
            d = cnn.DeviceConvDataset(ds, image, device, host)
            torch.cuda.current_stream(device).synchronize()  # read on other packs' streams
            per[key] = d
        return d


class _Orders:
    """Host + device epoch permutations, one per (dataset, epoch), LRU of 64.
    A new order is uploaded from page-locked memory on a side stream and
    published with an event: the step that needs it waits on the GPU
    (`cudaStreamWaitEvent`), so an epoch boundary does not drain the
    pipelined step loop, and concurrent packs on other streams see the copy."""

    def __init__(self):
        self.cache = {}
        self.side = {}

    def get(self, ds, epoch, device):
        """(host order, device order, ready event)"""
        import torch
        key = (ds.dataset_id, ds.n, epoch, device)
        with _LOCK:
            v = self.cache.pop(key, None)
            if v is None:
                perm = epoch_permutation(ds.dataset_id, ds.n, epoch)
                st = self.side.get(device)
                if st is None:
                    st = self.side[device] = torch.cuda.Stream(device=device)
                host = torch.from_numpy(perm.astype(np.int64)).pin_memory()
                with torch.cuda.stream(st):
                    dev = host.to(torch.device("cuda", device), non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(st)
                v = (perm, dev, ev, host)  # host: the pinned source lives as long as the copy
            self.cache[key] = v
            while len(self.cache) > 64:  # members of a pack sit at different epochs
                old = self.cache.pop(next(iter(self.cache)))
                old[2].synchronize()      # (long done) before its pinned source goes
            return v[:3]


_ORDERS = _Orders()


class ConvStep:
    """The host half of one conv packed step: groups, takes, leaders."""
    __slots__ = ("takes", "leads", "rows", "n_groups", "driver", "data")


def _plan(packed: ConvPackedModel, active, datasets, cp):
    from .packing import PackError
    import torch
    plan = ConvStep()
    K = len(packed.members)
    plan.takes = [0] * K
    plan.leads = list(range(K))
    plan.rows = {}
    plan.driver = max(h.batch_size for h in active)
    index = {id(h): k for k, h in enumerate(packed.members)}
    groups: dict = {}
    for h in active:
        groups.setdefault((h.dataset_binding, h.cursor.epoch_index, h.cursor.pos,
                           h.batch_size), []).append(h)
    plan.n_groups = len(groups)
    data = None
    for key in sorted(groups):
        grp = groups[key]
        binding, epoch, pos, b = key
        ds = datasets[binding]
        image = grp[0].arch.image
        for h in grp:
            if h.arch.image != image or ds.dim != h.arch.input_dim:
                raise engine.ShapeMismatch(f"{h.model_id}/x", ("batch", h.arch.input_dim),
                                           (b, ds.dim))
        d = device_dataset(ds, image, cp.device, host=_rt.input_mode() == "stream")
        if data is None:
            data = d
        elif d is not data:
            raise PackError("conv packs read one dataset per step (all groups bound to "
                            f"{packed.members[0].dataset_binding!r})")
        for h in grp:
            if d.max_label >= h.arch.classes:
                raise IndexError(f"label out of bounds for member {h.model_id!r} "
                                 f"with {h.arch.classes} classes")
        take = min(b, ds.n - pos)
        perm, dperm, ready = _ORDERS.get(ds, epoch, cp.device)
        lead = index[id(grp[0])]
        torch.cuda.current_stream(cp.device).wait_event(ready)
        cp.idx[lead][:take].copy_(dperm[pos:pos + take], non_blocking=True)
        rows = perm[pos:pos + take]
        for h in grp:
            k = index[id(h)]
            plan.takes[k] = take
            plan.leads[k] = lead
            plan.rows[k] = rows
    plan.data = data
    return plan


def _apply(packed, active, plan, state):
    """Cursor / optimizer bookkeeping after the device step (packing.py:250-257)."""
    from .engine import NonFiniteGradient
    index = {id(h): k for k, h in enumerate(packed.members)}
    losses = {}
    bad = None
    for h in active:
        k = index[id(h)]
        verdict = int(state[k, 2])
        if verdict & 1:
            if verdict & 2 and bad is None:
                bad = h
            continue
        h._committed()
        c = h.cursor
        c.steps_done += 1
        c.pos += plan.takes[k]
        np.add.at(c.samples_used, plan.rows[k], 1)
        losses[h.model_id] = float(np.array([state[k, 3]], dtype=np.int32).view(np.float32)[0])
    if bad is not None:
        cp, k = bad._home
        for p in bad.net.params:
            g = cp.grads[k][p.name]
            import torch
            if not bool(torch.isfinite(g).all()):
                raise NonFiniteGradient(f"{bad.model_id}/{p.name}")
        raise NonFiniteGradient(f"{bad.model_id}/loss")
    return losses


def conv_packed_step(packed: ConvPackedModel, datasets, preprocess_spec=None, cache=None,
                     stop_at_epoch_end=False):
    """packing.py:185-264 for conv members."""
    from .packing import _active_members
    import torch
    if preprocess_spec is not None and getattr(preprocess_spec, "stages", None):
        raise NotImplementedError("preprocess stages are not supported for conv members")
    active = _active_members(packed, datasets, stop_at_epoch_end)
    cp = packed.device_pack()
    caller = torch.cuda.current_stream(cp.dev)
    cp.stream.wait_stream(caller)          # host→device state uploads happen on the caller
    with torch.cuda.stream(cp.stream):
        plan = _plan(packed, active, datasets, cp)
        prog = cp.program(plan.takes, plan.leads, plan.data)
        prog.run(cp.stream.cuda_stream)
        state = cp.state.cpu().numpy()     # the step's one sync: losses + verdicts
    caller.wait_stream(cp.stream)
    losses = _apply(packed, active, plan, state)
    packed.last_step_stats = {
        "physical_inputs": plan.n_groups if packed.share_inputs else len(active),
        "groups": plan.n_groups, "driver_batch": plan.driver}
    return losses


def conv_packed_run(packed: ConvPackedModel, datasets, max_steps, depth=3):
    """Up to `max_steps` packed steps (fewer when no member is active any more),
    pipelined: the host plans and launches step i+1 while the device runs step i;
    every step's losses and commit verdicts come back through a pinned ring (one
    async D2H copy per step) instead of a synchronous read.  Cursors advance as
    packed_step advances them, assuming each step commits; a step that did not
    (non-finite value or gradient, engine.py:297-299) is found when its verdicts
    arrive — at most `depth` steps later — and NonFiniteGradient is raised then
    (the reference raises at that step; steps already in flight are not rolled
    back, so the pack's state is unspecified after the exception).  Returns the
    per-step {model_id: loss} dicts.  Used by B200ConvExecutor.evaluate."""
    import collections
    import torch
    from .engine import NonFiniteGradient
    from .packing import ReplanNeeded, _active_members
    cp = packed.device_pack()
    K = len(packed.members)
    depth = max(1, int(depth))
    ring = torch.empty((depth, K, 4), dtype=torch.int32, pin_memory=True)
    evs = [torch.cuda.Event() for _ in range(depth)]
    index = {id(h): k for k, h in enumerate(packed.members)}
    fly = collections.deque()
    out = []

    def drain():
        slot, active, plan = fly.popleft()
        evs[slot].synchronize()
        st = ring[slot].numpy()
        losses = {}
        for h in active:
            k = index[id(h)]
            if int(st[k, 2]) & 1:
                raise NonFiniteGradient(f"{h.model_id}/step {h.cursor.steps_done}")
            losses[h.model_id] = float(np.array([st[k, 3]], dtype=np.int32)
                                       .view(np.float32)[0])
        out.append(losses)

    caller = torch.cuda.current_stream(cp.dev)
    cp.stream.wait_stream(caller)
    with torch.cuda.stream(cp.stream):
        for i in range(int(max_steps)):
            try:
                active = _active_members(packed, datasets, False)
            except ReplanNeeded:
                break
            plan = _plan(packed, active, datasets, cp)
            cp.program(plan.takes, plan.leads, plan.data).run(cp.stream.cuda_stream)
            if len(fly) == depth:
                drain()
            slot = i % depth
            ring[slot].copy_(cp.state, non_blocking=True)
            evs[slot].record(cp.stream)
            for h in active:  # the bookkeeping of a committed step (packing.py:255-257)
                k = index[id(h)]
                h._committed()
                c = h.cursor
                c.steps_done += 1
                c.pos += plan.takes[k]
                np.add.at(c.samples_used, plan.rows[k], 1)
            fly.append((slot, active, plan))
            packed.last_step_stats = {
                "physical_inputs": plan.n_groups if packed.share_inputs else len(active),
                "groups": plan.n_groups, "driver_batch": plan.driver}
        while fly:
            drain()
    caller.wait_stream(cp.stream)
    return out


def conv_standalone_step(handle: ConvModelHandle, datasets, preprocess_spec=None, cache=None):
    """packing.py:267-282: the same kernels on a one-member pack."""
    from .packing import PackError, _roll_if_needed
    if handle.finished:
        raise PackError(f"{handle.model_id}: no remaining steps")
    _roll_if_needed(handle, datasets)
    if handle._solo is None or handle._solo.members[0] is not handle:
        handle._solo = conv_pack_models([handle])
    losses = conv_packed_step(handle._solo, datasets, preprocess_spec, cache)
    return losses[handle.model_id]
