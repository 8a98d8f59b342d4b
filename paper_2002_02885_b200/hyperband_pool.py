"""Pack-aware Hyperband sharded over the GPUs of one box.

Packs are independent, so the only parallelism is *which GPU trains which
pack*.  The driver loop stays the reference's (`tuner.packed_hyperband`,
tuner.py:285-337, unchanged grouping and selection); this module supplies
its `rung_runner`:

* SPMD: one process per GPU (torchrun / `spawn`), every rank runs the same
  `packed_hyperband` call.  Grouping is deterministic (seeded by
  `("group", seed, s, i)`), so every rank computes the same groups and the
  same assignment without talking.
* Assignment: longest-processing-time first over the rung's groups, cost =
  Σ members' samples this rung (epochs · ceil(n_train/b) · b, the unit the
  packed kernels scale with); ties go to the rank already holding most of
  the group's member state, then to the lowest rank.
* Member state (params + optimizer slots + cursor) persists per config_id
  across rungs and brackets exactly as in EngineExecutor (tuner.py:446-458).
  It lives on the rank that last trained it; when a later rung places the
  member elsewhere its state moves as a PKCK checkpoint (packing.py:335-417,
  bit-exact f64 carrier of the device's values) before the rung runs.
* The rung barrier is the gather of per-group (losses, ms): a host
  collective on the control-plane process group (gloo), never NCCL — no
  tensor of the training path crosses GPUs.  Results merge in group order,
  so records, selection and best config are identical to a 1-GPU run.
* Failures: OOM degrades a group to singletons on the rank that owns it
  (tuner.py:309-314).  Any other exception a group raises on its rank
  (ExecutorError, EngineError / NonFiniteGradient from a diverging config,
  an OOMError from the singleton fallback, ...) is caught, shipped through
  the rung's gather as (type, message, pickled exception) and re-raised on
  EVERY rank after the merge, first failing group in group order — so all
  ranks fail together exactly as the 1-GPU run does (ExecutorError aborts
  the bracket, tuner.py:332-334; anything else propagates) instead of the
  healthy ranks blocking in the gather.

Executors used with the pool expose, besides the reference protocol
(`device`, `memory_bytes(cfg)`, `evaluate(cfgs, epochs)`):
`export_state(config_id) -> bytes | None`, `import_state(config_id, bytes)`
and `drop_state(config_id)`; optional `group_cost(cfgs, epochs)`.
"""
from __future__ import annotations

import math
import pickle
import time

from . import tuner
from .device import OOMError


def _dist():
    import torch.distributed as dist
    return dist


class PackPool:
    """`rung_runner` for `tuner.packed_hyperband` over a process group.

    `group` is a torch.distributed process group whose backend can move
    Python objects (gloo); None = the default group.  With world size 1 it
    degenerates to the serial reference order."""

    def __init__(self, group=None):
        dist = _dist()
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.owner: dict = {}          # config_id -> rank holding its state
        self.migrations = 0            # member states moved between ranks
        self.migrated_bytes = 0
        self.busy_ms = 0.0             # this rank's evaluate time
        self.rungs = 0

    # ---- collectives (host objects only) ------------------------------------
    def _all_gather(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        _dist().all_gather_object(out, obj, group=self.group)
        return out

    # ---- placement ------------------------------------------------------------
    @staticmethod
    def group_cost(executor, members, epochs) -> float:
        fn = getattr(executor, "group_cost", None)
        if fn is not None:
            return float(fn(members, epochs))
        return float(epochs * len(members))

    def assign(self, executor, groups, epochs) -> list:
        """Deterministic LPT: returns the rank of every group."""
        costs = [self.group_cost(executor, g.members, epochs) for g in groups]
        order = sorted(range(len(groups)), key=lambda i: (-costs[i], i))
        load = [0.0] * self.world
        where = [0] * len(groups)
        for i in order:
            held = [0] * self.world
            for c in groups[i].members:
                r = self.owner.get(c.config_id)
                if r is not None:
                    held[r] += 1
            best = min(range(self.world), key=lambda r: (load[r], -held[r], r))
            where[i] = best
            load[best] += costs[i]
        return where

    # ---- state movement --------------------------------------------------------
    def _migrate(self, executor, groups, where):
        moves = {}  # config_id -> (src, dst)
        for g, dst in zip(groups, where):
            for c in g.members:
                src = self.owner.get(c.config_id)
                if src is not None and src != dst:
                    moves[c.config_id] = (src, dst)
        if not moves:
            return
        mine = {}
        for cid, (src, _dst) in sorted(moves.items()):
            if src == self.rank:
                raw = executor.export_state(cid)
                if raw is not None:
                    mine[cid] = raw
                executor.drop_state(cid)
        for payload in self._all_gather(mine):
            for cid, raw in payload.items():
                if moves[cid][1] == self.rank:
                    executor.import_state(cid, raw)
                self.migrated_bytes += len(raw)
        self.migrations += len(moves)

    # ---- the rung -------------------------------------------------------------
    def __call__(self, executor, groups, r_i):
        where = self.assign(executor, groups, r_i)
        self._migrate(executor, groups, where)
        mine = {}
        t0 = time.perf_counter()
        for gi, (g, r) in enumerate(zip(groups, where)):
            if r != self.rank:
                continue
            try:
                got, t_ms = tuner.run_rung_groups(executor, [g], r_i)[0]
                mine[gi] = ("ok", got, t_ms)
            except Exception as exc:  # noqa: BLE001 - re-raised on every rank below
                mine[gi] = ("error", _pack_exc(exc), 0.0)
        self.busy_ms += (time.perf_counter() - t0) * 1000.0
        merged = {}
        for part in self._all_gather(mine):
            merged.update(part)
        for gi, g in enumerate(groups):
            for c in g.members:
                self.owner[c.config_id] = where[gi]
        self.rungs += 1
        for gi in range(len(groups)):
            kind, a, _ = merged[gi]
            if kind == "error":
                raise _unpack_exc(a)
        return [(merged[gi][1], merged[gi][2]) for gi in range(len(groups))]


def _pack_exc(exc):
    try:
        blob = pickle.dumps(exc)
        pickle.loads(blob)
    except Exception:  # noqa: BLE001 - unpicklable: keep type name + message
        blob = None
    return (type(exc).__name__, str(exc), blob)


def _unpack_exc(packed):
    name, msg, blob = packed
    if blob is not None:
        return pickle.loads(blob)
    if name == "ExecutorError":
        return tuner.ExecutorError(msg)
    return RuntimeError(f"{name}: {msg}")


def sharded_hyperband(R, eta, executor, seed, strategy="knn", group=None, **kw):
    """`tuner.packed_hyperband` with its rungs sharded over the process
    group's ranks (one GPU each).  Every rank must call it with the same
    arguments; every rank returns the same TuneResult (its wall time is this
    rank's; take the max over ranks for the job's)."""
    pool = PackPool(group)
    res = tuner.packed_hyperband(R, eta, executor, seed, strategy=strategy,
                                 rung_runner=pool, **kw)
    return res, pool


def predicted_samples(n_train, members, epochs) -> int:
    """Σ_k epochs · ceil(n_train / b_k) · b_k: the rows the group's members
    consume in one rung (the LPT cost of B200Executor.group_cost)."""
    return sum(epochs * math.ceil(n_train / c.batch_size) * c.batch_size for c in members)
