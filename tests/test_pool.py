"""Multi-GPU Hyperband sharding (hyperband_pool) on CPU: world
size 2 over gloo, with a stateful stub executor whose losses depend on each
config's accumulated training — so a lost or duplicated state migration
changes the selection.  The sharded run must reproduce the serial run's
records, survivors and best config exactly (results merge in group order)."""
import math
import os
import pickle
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2002_02885_b200 import engine, hyperband_pool, tuner


class StatefulStub:
    """Loss = f(config, cumulative epochs trained), state kept per config_id
    like EngineExecutor (tuner.py:446-458); state moves as bytes."""

    device = None

    def __init__(self, fail_on=None, diverge_on=None):
        self.state = {}
        self.fail_on = fail_on
        self.diverge_on = diverge_on

    def memory_bytes(self, cfg):
        return 0

    def group_cost(self, cfgs, epochs):
        return hyperband_pool.predicted_samples(1000, cfgs, epochs)

    def evaluate(self, cfgs, epochs):
        out = {}
        for c in cfgs:
            if self.fail_on is not None and c.config_id == self.fail_on:
                raise tuner.ExecutorError(f"injected failure at {c.config_id}")
            if self.diverge_on is not None and c.config_id == self.diverge_on:
                raise engine.NonFiniteGradient(f"cfg{c.config_id:04d}/L0/W")
            e = self.state.get(c.config_id, 0) + epochs
            self.state[c.config_id] = e
            out[c.config_id] = ((c.config_id * 7919) % 101) / (1.0 + math.log1p(e)) \
                + 0.01 * c.indices[2]
        return out, 1.0

    def export_state(self, cid):
        return pickle.dumps(self.state[cid]) if cid in self.state else None

    def import_state(self, cid, raw):
        self.state[cid] = pickle.loads(raw)

    def drop_state(self, cid):
        self.state.pop(cid, None)


def _summary(res):
    return ([(r.bracket, r.rung, r.group, r.config_id, r.epochs, r.loss)
             for r in res.records],
            res.best_config.config_id, res.best_loss, res.total_epochs, res.failures)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, strategy, fail_on, q, diverge_on=None, overlap=False, R=27):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        run = hyperband_pool.overlapped_hyperband if overlap else hyperband_pool.sharded_hyperband
        res, pool = run(R, 3, StatefulStub(fail_on, diverge_on), seed=3, strategy=strategy)
        q.put((rank, _summary(res), pool.migrations, pool.rungs))
    except Exception as exc:  # noqa: BLE001 - reported to the test
        q.put((rank, ("raised", type(exc).__name__, str(exc)), -1, -1))
    finally:
        dist.destroy_process_group()


def _run_world(world, strategy, fail_on=None, diverge_on=None, overlap=False, R=27):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, strategy, fail_on, q, diverge_on,
                                            overlap, R))
          for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    return sorted(out)


@pytest.mark.parametrize("strategy", ["knn", "original", "random"])
def test_sharded_hyperband_matches_serial(strategy):
    serial = tuner.packed_hyperband(27, 3, StatefulStub(), seed=3, strategy=strategy)
    out = _run_world(2, strategy)
    for rank, summ, migrations, rungs in out:
        assert summ == _summary(serial), f"rank {rank} diverged from the serial run"
    assert out[0][3] > 0
    # both ranks saw the same migrations (replicated ownership map), and
    # knn/original regroupings do move member state between ranks
    assert out[0][2] == out[1][2]
    if strategy != "random":
        assert out[0][2] > 0


def test_sharded_executor_error_aborts_bracket_on_all_ranks():
    serial = tuner.packed_hyperband(27, 3, StatefulStub(fail_on=None), seed=3, strategy="knn")
    victim = serial.records[5].config_id
    ref = tuner.packed_hyperband(27, 3, StatefulStub(fail_on=victim), seed=3, strategy="knn")
    assert ref.failures
    out = _run_world(2, "knn", fail_on=victim)
    for _, summ, _, _ in out:
        assert summ == _summary(ref)


def test_lpt_assignment_balances_and_prefers_owner():
    pool = hyperband_pool.PackPool.__new__(hyperband_pool.PackPool)
    pool.world, pool.rank, pool.owner = 3, 0, {}
    space = tuner.ConfigSpace()
    cfgs = [space.config(i) for i in range(0, 60, 4)]
    groups = [tuner.PackGroup(cfgs[i:i + 3], 0, cfgs[i].config_id) for i in range(0, 15, 3)]
    ex = StatefulStub()
    where = pool.assign(ex, groups, 3)
    costs = [pool.group_cost(ex, g.members, 3) for g in groups]
    load = [sum(c for c, w in zip(costs, where) if w == r) for r in range(3)]
    assert max(load) - min(load) <= max(costs)
    # equal-cost tie: the group goes to the rank already holding its members
    pool.owner = {c.config_id: 2 for c in groups[0].members}
    same = [tuner.PackGroup(groups[0].members, 0, 0)]
    assert pool.assign(ex, same, 3) == [2]


def test_sharded_engine_error_raises_on_every_rank():
    """A diverging config (NonFiniteGradient, not an ExecutorError) propagates
    out of the serial run; sharded, every rank raises it together instead of
    the healthy rank blocking in the rung gather."""
    serial = tuner.packed_hyperband(27, 3, StatefulStub(), seed=3, strategy="knn")
    victim = serial.records[7].config_id
    with pytest.raises(engine.NonFiniteGradient) as ref:
        tuner.packed_hyperband(27, 3, StatefulStub(diverge_on=victim), seed=3, strategy="knn")
    out = _run_world(2, "knn", diverge_on=victim)
    for _, summ, _, _ in out:
        assert summ == ("raised", "NonFiniteGradient", str(ref.value))


@pytest.mark.parametrize("strategy", ["knn", "original"])
def test_overlapped_brackets_match_serial_world4(strategy):
    """Brackets that share no config_id overlap (one round runs the next rung of
    every ready bracket, all their groups LPT-placed over 4 ranks): records,
    survivors, best config and failures equal the serial run's, in fewer
    synchronised rounds than serial rungs."""
    serial = tuner.packed_hyperband(81, 3, StatefulStub(), seed=3, strategy=strategy)
    out = _run_world(4, strategy, overlap=True, R=81)
    rungs_serial = len({(r.bracket, r.rung) for r in serial.records})
    for rank, summ, migrations, rounds in out:
        assert summ == _summary(serial), f"rank {rank} diverged from the serial run"
        assert 0 < rounds < rungs_serial
    assert len({o[2] for o in out}) == 1  # replicated ownership: same migrations everywhere


def test_overlapped_failures_match_serial():
    """An ExecutorError aborts only its bracket; a diverging config raises on every
    rank the exception the serial run raises (earliest failing bracket first)."""
    serial = tuner.packed_hyperband(27, 3, StatefulStub(), seed=3, strategy="knn")
    victim = serial.records[5].config_id
    ref = tuner.packed_hyperband(27, 3, StatefulStub(fail_on=victim), seed=3, strategy="knn")
    got, _ = hyperband_pool.overlapped_hyperband(27, 3, StatefulStub(fail_on=victim), seed=3,
                                                 strategy="knn")
    assert _summary(got) == _summary(ref)
    victim = serial.records[7].config_id
    with pytest.raises(engine.NonFiniteGradient) as a:
        tuner.packed_hyperband(27, 3, StatefulStub(diverge_on=victim), seed=3, strategy="knn")
    out = _run_world(2, "knn", diverge_on=victim, overlap=True)
    for _, summ, _, _ in out:
        assert summ == ("raised", "NonFiniteGradient", str(a.value))


class ConcurrentStub(StatefulStub):
    """The stub with the pool's concurrent packs switched on (a round's groups
    evaluated by a thread pool, as the conv executor's packs are)."""
    concurrent_groups = 4


@pytest.mark.parametrize("strategy", ["original", "knn"])
def test_concurrent_groups_match_serial(strategy):
    """Groups of a round evaluated concurrently (hyperband_pool._run_local):
    records, selection and failures equal the serial run's, including an
    ExecutorError aborting its bracket and a diverging config raising the serial
    run's exception."""
    serial = tuner.packed_hyperband(81, 3, StatefulStub(), seed=3, strategy=strategy)
    got, _ = hyperband_pool.overlapped_hyperband(81, 3, ConcurrentStub(), seed=3,
                                                 strategy=strategy)
    assert _summary(got) == _summary(serial)
    serial = tuner.packed_hyperband(27, 3, StatefulStub(), seed=3, strategy=strategy)
    victim = serial.records[5].config_id
    ref = tuner.packed_hyperband(27, 3, StatefulStub(fail_on=victim), seed=3, strategy=strategy)
    got, _ = hyperband_pool.overlapped_hyperband(27, 3, ConcurrentStub(fail_on=victim), seed=3,
                                                 strategy=strategy)
    assert _summary(got) == _summary(ref)
    victim = serial.records[7].config_id
    with pytest.raises(engine.NonFiniteGradient) as a:
        tuner.packed_hyperband(27, 3, StatefulStub(diverge_on=victim), seed=3, strategy=strategy)
    with pytest.raises(engine.NonFiniteGradient) as b:
        hyperband_pool.overlapped_hyperband(27, 3, ConcurrentStub(diverge_on=victim), seed=3,
                                            strategy=strategy)
    assert str(a.value) == str(b.value)
