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
  bit-exact f64 carrier of the device's values) before the rung runs —
  point to point from the owning rank to the new one on the control group.
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

* Concurrent packs on one GPU: a rank's groups of one round are independent
  packs, each a chain of small latency-bound launches that fills a fraction of
  the B200.  Executors that declare `concurrent_groups = n > 1` (the conv
  executor) run up to n of them at once, one host thread and CUDA stream per
  pack; results are keyed by group, so records are the serial run's.

Executors used with the pool expose, besides the reference protocol
(`device`, `memory_bytes(cfg)`, `evaluate(cfgs, epochs)`):
`export_state(config_id) -> bytes | None`, `import_state(config_id, bytes)`
and `drop_state(config_id)`; optional `group_cost(cfgs, epochs)` and
`concurrent_groups`.
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


def _evaluate_group(executor, g, r_i, own_stream):
    """One group's rung: ("ok", losses, ms) or ("error", packed exception, 0).
    own_stream: run on a private CUDA stream (concurrent packs must not meet on
    the legacy default stream, which serialises against every other stream)."""
    try:
        import torch
        if own_stream and torch.cuda.is_available():
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                got, t_ms = tuner.run_rung_groups(executor, [g], r_i)[0]
            st.synchronize()
        else:
            got, t_ms = tuner.run_rung_groups(executor, [g], r_i)[0]
        return ("ok", got, t_ms)
    except Exception as exc:  # noqa: BLE001 - re-raised after the merge
        return ("error", _pack_exc(exc), 0.0)


def _run_local(executor, items):
    """items = [(key, group, r_i)] this rank trains: sequentially, or up to
    executor.concurrent_groups packs at once (largest first)."""
    n = int(getattr(executor, "concurrent_groups", 1) or 1)
    if n <= 1 or len(items) <= 1:
        return {key: _evaluate_group(executor, g, r_i, False) for key, g, r_i in items}
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(n, len(items))) as tp:
        futs = {key: tp.submit(_evaluate_group, executor, g, r_i, True)
                for key, g, r_i in items}
        return {key: f.result() for key, f in futs.items()}


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
        if self.world == 1:
            self.migrations += len(moves)
            return
        # point to point: each moved state travels once, src → dst (a length
        # header, then the bytes), posted asynchronously in config_id order
        import torch
        dist = _dist()
        reqs, inbox = [], []
        for cid, (src, dst) in sorted(moves.items()):
            if src == self.rank:
                raw = executor.export_state(cid)
                executor.drop_state(cid)
                raw = raw or b""
                hdr = torch.tensor([len(raw)], dtype=torch.int64)
                reqs.append(dist.isend(hdr, dst, group=self.group))
                if raw:
                    buf = torch.frombuffer(bytearray(raw), dtype=torch.uint8)
                    reqs.append(dist.isend(buf, dst, group=self.group))
                    inbox.append((None, buf))  # keep the buffer alive until sent
                self.migrated_bytes += len(raw)
            elif dst == self.rank:
                hdr = torch.zeros(1, dtype=torch.int64)
                dist.recv(hdr, src, group=self.group)
                n = int(hdr.item())
                if n:
                    buf = torch.empty(n, dtype=torch.uint8)
                    dist.recv(buf, src, group=self.group)
                    executor.import_state(cid, bytes(buf.numpy()))
                self.migrated_bytes += n
        for r in reqs:
            r.wait()
        self.migrations += len(moves)

    # ---- the rung -------------------------------------------------------------
    def __call__(self, executor, groups, r_i):
        where = self.assign(executor, groups, r_i)
        self._migrate(executor, groups, where)
        t0 = time.perf_counter()
        mine = _run_local(executor, [(gi, g, r_i) for gi, (g, r) in enumerate(zip(groups, where))
                                     if r == self.rank])
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


    def run_many(self, executor, tasks):
        """One round over several rungs (overlapped brackets): tasks =
        [(groups, r_i)]; all their groups are placed together (LPT), run, and
        gathered in one collective.  Returns per task either ("ok", [(losses,
        t_ms)] in group order) or ("error", exception) — the first failing group
        of the task in group order, as the task's own rung would have raised."""
        flat = [(ti, gi, g, r_i) for ti, (groups, r_i) in enumerate(tasks)
                for gi, g in enumerate(groups)]
        costs = [self.group_cost(executor, g.members, r_i) for _, _, g, r_i in flat]
        order = sorted(range(len(flat)), key=lambda i: (-costs[i], i))
        load = [0.0] * self.world
        where = [0] * len(flat)
        for i in order:
            held = [0] * self.world
            for c in flat[i][2].members:
                r = self.owner.get(c.config_id)
                if r is not None:
                    held[r] += 1
            best = min(range(self.world), key=lambda r: (load[r], -held[r], r))
            where[i] = best
            load[best] += costs[i]
        self._migrate(executor, [g for _, _, g, _ in flat], where)
        t0 = time.perf_counter()
        local = sorted((i for i in range(len(flat)) if where[i] == self.rank),
                       key=lambda i: (-costs[i], i))  # largest packs start first
        mine = _run_local(executor, [(i, flat[i][2], flat[i][3]) for i in local])
        self.busy_ms += (time.perf_counter() - t0) * 1000.0
        merged = {}
        for part in self._all_gather(mine):
            merged.update(part)
        for i, (_, _, g, _) in enumerate(flat):
            for c in g.members:
                self.owner[c.config_id] = where[i]
        self.rungs += 1
        out = [None] * len(tasks)
        for i, (ti, gi, g, r_i) in enumerate(flat):
            kind, a, t_ms = merged[i]
            if out[ti] is not None and out[ti][0] == "error":
                continue
            if kind == "error":
                out[ti] = ("error", _unpack_exc(a))
            else:
                out[ti] = out[ti] or ("ok", [])
                out[ti][1].append((a, t_ms))
        return out


def overlapped_hyperband(R, eta, executor, seed, strategy="knn", group=None, space=None,
                         threshold=6.0, m=27, metric="indexsum"):
    """`tuner.packed_hyperband` (reference tuner.py:285-337) with independent
    brackets overlapped: each round runs the next rung of every bracket whose
    predecessors are done, all their groups placed over the ranks together.
    Brackets are independent except through member state, which is kept per
    config_id across brackets (tuner.py:446-458): a bracket sharing a config_id
    with an earlier bracket waits for it, so every member sees the serial
    order of its training.  Sampling and grouping are seeded per (bracket,
    rung), so records, survivors, failures and the best config equal the
    serial run's (records are reported in the serial order).  A non-executor
    exception is raised as the serial run would raise it: that of the earliest
    failing bracket, after every earlier bracket has finished."""
    import math as _m
    space = space or tuner.ConfigSpace()
    pool = PackPool(group)
    t0 = time.perf_counter()
    br = []
    for bi, (s, n, r) in enumerate(tuner.bracket_schedule(R, eta)):
        cfgs = tuner.sample_configs(space, n, (seed, s))
        ids = {c.config_id for c in cfgs}
        br.append({"s": s, "r": r, "configs": cfgs, "ids": ids, "i": 0, "done": False,
                   "deps": [bj for bj in range(bi) if ids & br[bj]["ids"]], "records": [],
                   "bests": [], "ms": 0.0, "epochs": 0, "failure": None, "raised": None})
    while True:
        raised = [bi for bi, b in enumerate(br) if b["raised"] is not None]
        stop_at = raised[0] if raised else len(br)
        live = [bi for bi in range(stop_at) if not br[bi]["done"]]
        if not live:
            break
        runnable = [bi for bi in live if all(br[d]["done"] for d in br[bi]["deps"])]
        tasks = []
        for bi in runnable:
            b = br[bi]
            r_i = max(1, int(round(b["r"] * eta ** b["i"])))
            groups = tuner.make_groups(strategy, b["configs"], executor,
                                       tuner._rng("group", seed, b["s"], b["i"]), threshold, m,
                                       metric)
            tasks.append((bi, groups, r_i))
        results = pool.run_many(executor, [(g, r_i) for _, g, r_i in tasks])
        for (bi, groups, r_i), res in zip(tasks, results):
            b = br[bi]
            if res[0] == "error":
                exc = res[1]
                b["done"] = True
                if isinstance(exc, tuner.ExecutorError):
                    b["failure"] = (b["s"], str(exc))
                else:
                    b["raised"] = exc
                continue
            losses = {}
            for gi, (g, (got, t_ms)) in enumerate(zip(groups, res[1])):
                b["ms"] += t_ms
                losses.update(got)
                for cfg in sorted(g.members, key=lambda c: c.config_id):
                    b["records"].append(tuner.AuditRecord(b["s"], b["i"], gi, cfg.config_id, r_i,
                                                          got[cfg.config_id], t_ms))
                b["epochs"] += r_i * len(g.members)
            ranked = sorted(b["configs"], key=lambda c: (losses[c.config_id], c.config_id))
            b["bests"].append((losses[ranked[0].config_id], ranked[0]))
            b["configs"] = ranked[:len(b["configs"]) // eta]
            b["i"] += 1
            if not b["configs"] or b["i"] > b["s"]:
                b["done"] = True
    raised = [b["raised"] for b in br if b["raised"] is not None]
    if raised:
        raise raised[0]
    records, failures, total_ms, total_epochs = [], [], 0.0, 0
    best_loss, best = _m.inf, None
    for b in br:
        records += b["records"]
        total_ms += b["ms"]
        total_epochs += b["epochs"]
        for loss, cfg in b["bests"]:
            if loss < best_loss:
                best_loss, best = loss, cfg
        if b["failure"] is not None:
            failures.append(b["failure"])
    res = tuner.TuneResult(best, best_loss, records, total_ms, total_epochs, failures,
                           wall_time_ms=(time.perf_counter() - t0) * 1000.0)
    return res, pool


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
