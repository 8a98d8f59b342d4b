"""Host-side logic of the drop-in (CPU only): seeding, epoch plans, the
Hyperband driver and grouping strategies, the PKCK checkpoint format and
the device memory model — checked against the reference's own outputs."""
import json
import math
import os

import numpy as np
import pytest

from paper_2002_02885_b200 import data, device, engine, packing, tuner

G = os.path.join(os.path.dirname(__file__), "golden")
ARCH = packing.MLPArch(input_dim=6, hidden=(8,), classes=3)


def _h(mid, batch=10, steps=20, opt="sgd", lr=0.05, seed=0, arch=ARCH):
    return packing.make_handle(mid, arch, opt, lr, batch, steps, "d", seed)


def test_synth_and_permutation_match_reference():
    z = np.load(os.path.join(G, "config0.npz"))
    ds = data.synth_dataset(10000, 784, 10, seed=0)
    assert ds.dataset_id == str(z["dataset_id"])
    np.testing.assert_array_equal(data.epoch_permutation(ds.dataset_id, 10000, 0)[:64],
                                  z["perm_head"])


def test_init_matches_reference_bitwise():
    z = np.load(os.path.join(G, "config0.npz"))
    h = packing.make_handle("m0", packing.MLPArch(784, (256,), 10), "sgd", 0.1, 32, 1, "t", 0)
    flat = h._flat_params(h.params)
    np.testing.assert_array_equal(flat[:4096], z["init_m0_head"])
    np.testing.assert_array_equal([flat.sum(), (flat ** 2).sum()], z["init_m0_sum"])


def test_init_respects_xavier_bound_and_is_member_scoped():
    """tests/test_engine.py:182-203."""
    g1 = engine.build_mlp("a", 4, (5,), 3)
    g3 = engine.build_mlp("b", 4, (5,), 3)
    p1, p3 = engine.init_parameters(g1, 11), engine.init_parameters(g3, 11)
    assert not np.array_equal(p1["a/L0/W"], p3["b/L0/W"])
    g = engine.build_mlp("m", 10, (20,), 5)
    ps = engine.init_parameters(g, 0)
    for i, (fi, fo) in enumerate([(10, 20), (20, 5)]):
        bound = np.sqrt(6.0 / (fi + fo))
        assert np.all(np.abs(ps[f"m/L{i}/W"]) <= bound)
        np.testing.assert_array_equal(ps[f"m/L{i}/b"], 0.0)


def test_graph_node_names_match_reference_convention():
    g = engine.build_mlp("m", 3, (4, 5), 2, "tanh")
    assert [n.name for n in g.nodes] == ["m/in", "m/aff0", "m/act0", "m/aff1", "m/act1",
                                        "m/aff2", "m/loss"]
    assert g.param_shapes["m/L1/W"] == (4, 5)


def test_error_node_and_grad_naming():
    h = packing.make_handle("m", packing.MLPArch(3, (4, 5), 2), "sgd", 0.1, 4, 1, "d", 0)
    assert [packing._node_name(h, i) for i in range(7)] == [
        "m/in", "m/aff0", "m/act0", "m/aff1", "m/act1", "m/aff2", "m/loss"]
    assert [packing._grad_name(h, p) for p in range(6)] == [
        "m/L2/W", "m/L2/b", "m/L1/W", "m/L1/b", "m/L0/W", "m/L0/b"]


def test_epoch_plan_phases():
    """tests/test_pack.py:153-172."""
    datasets = {"d": data.synth_dataset(100, 6, 3, seed=0)}
    members = [_h("a", batch=50, steps=100), _h("b", batch=20, steps=100)]
    assert packing.make_epoch_plan(members, datasets) == [("a", 2), ("b", 3)]
    members = [_h("z", batch=25, steps=10), _h("a", batch=25, steps=10)]
    assert packing.make_epoch_plan(members, datasets) == [("a", 4)]


def test_pack_rejects_duplicates_and_empty():
    with pytest.raises(packing.PackError):
        packing.pack_models([_h("m"), _h("m")])
    with pytest.raises(packing.PackError):
        packing.pack_models([])


def test_driver_batch_and_groups_before_stepping():
    h1, h2, h3 = _h("a", batch=10), _h("b", batch=10), _h("c", batch=20)
    p = packing.pack_models([h1, h2, h3])
    assert p.driver_batch == 20
    assert sorted(len(g) for g in p.input_groups()) == [1, 2]
    assert packing.dedup_inputs(p).share_inputs


def test_optimizer_construction_errors():
    with pytest.raises(engine.EngineError):
        engine.make_optimizer("newton", 0.1)
    with pytest.raises(engine.EngineError):
        engine.make_optimizer("sgd", 0.0)
    with pytest.raises(engine.EngineError):
        engine.build_mlp("m", 3, (4,), 2, activation="swish")


# ---------------------------------------------------------------- PKCK --

def test_checkpoint_bytes_identical_to_reference_for_fresh_handle():
    raw = open(os.path.join(G, "ckpt_fresh.pkck"), "rb").read()
    h = packing.make_handle("m", ARCH, "adam", 0.001, 10, 30, "d", 0)
    assert packing.checkpoint_model(h).to_bytes() == raw


def test_reference_checkpoint_round_trips_byte_exact():
    raw = open(os.path.join(G, "ckpt_adam7.pkck"), "rb").read()
    ck = packing.Checkpoint.from_bytes(raw)
    ds = data.synth_dataset(120, 6, 3, seed=0)
    back = packing.restore_handle(ck, {"d": ds})
    assert back.optimizer.kind == "adam" and back.optimizer.step_counter == 7
    assert back.cursor.steps_done == 7 and back.cursor.pos == 70
    assert int(back.cursor.samples_used.sum()) == 70
    assert packing.checkpoint_model(back).to_bytes() == raw


def test_checkpoint_detects_corruption():
    raw = bytearray(packing.checkpoint_model(_h("m")).to_bytes())
    raw[20] ^= 0xFF
    with pytest.raises(packing.PackError):
        packing.Checkpoint.from_bytes(bytes(raw))
    with pytest.raises(packing.PackError):
        packing.Checkpoint.from_bytes(b"XXXX" + bytes(raw[4:]))


# -------------------------------------------------------------- tuner --

def _tuning():
    return json.load(open(os.path.join(G, "tuning.json")))


def test_bracket_schedule():
    assert tuner.bracket_schedule(81, 3) == [(4, 81, 1), (3, 34, 3), (2, 15, 9), (1, 8, 27),
                                             (0, 5, 81)]


def test_stub_hyperband_chain_matches_reference():
    res = tuner.hyperband(81, 3, tuner.StubExecutor(lambda c, e: c.config_id), seed=1)
    got = [[r.bracket, r.rung, r.group, r.config_id, r.epochs] for r in res.records]
    assert got == _tuning()["stub_chain"]
    assert res.total_epochs == sum(r[4] for r in got)


@pytest.mark.parametrize("strategy", ["original", "batchsize", "random", "knn"])
def test_grouping_and_selection_match_reference(strategy):
    ref = _tuning()["stub_winners"]
    for seed in range(5):
        ex = tuner.StubExecutor(lambda c, e, s=seed: float(
            tuner._rng("accept7", s, c.config_id).uniform()))
        r = tuner.packed_hyperband(81, 3, ex, seed=seed, strategy=strategy)
        best, epochs, recs = ref[f"{seed}_{strategy}"]
        assert r.best_config.config_id == best
        assert r.total_epochs == epochs
        assert [[x.bracket, x.rung, x.group, x.config_id] for x in r.records] == recs


def test_distance_worked_example_and_axioms():
    space = tuner.ConfigSpace()
    by = {(c.batch_size, c.optimizer, c.learning_rate, c.activation): c
          for c in (space.config(i) for i in range(space.size))}
    assert tuner.config_distance(by[(20, "sgd", 1e-2, "relu")],
                                 by[(40, "adagrad", 1e-2, "relu")]) == 5.0
    rng = np.random.default_rng(6)
    for _ in range(500):
        i, j, k = (space.config(int(x)) for x in rng.integers(space.size, size=3))
        d = tuner.config_distance(i, j)
        assert d == tuner.config_distance(j, i) and d >= 0
        assert d <= tuner.config_distance(i, k) + tuner.config_distance(k, j)


def test_oom_degrades_to_singletons():
    class Ex(tuner.StubExecutor):
        def evaluate(self, configs, epochs):
            if len(configs) > 1:
                raise device.OOMError(2, 1)
            return super().evaluate(configs, epochs)
    r = tuner.packed_hyperband(9, 3, Ex(lambda c, e: c.config_id), seed=0, strategy="knn")
    assert r.best_config is not None and not r.failures


def test_executor_failure_is_recorded_per_bracket():
    class Flaky(tuner.StubExecutor):
        calls = 0

        def evaluate(self, configs, epochs):
            Flaky.calls += 1
            if Flaky.calls == 2:
                raise tuner.ExecutorError("boom")
            return super().evaluate(configs, epochs)
    r = tuner.packed_hyperband(9, 3, Flaky(lambda c, e: c.config_id), seed=0,
                               strategy="original")
    assert len(r.failures) == 1 and r.failures[0][1] == "boom"


# ------------------------------------------------------- memory model --

def test_member_device_bytes_formula():
    arch = packing.MLPArch(784, (256,), 10)
    b = device.member_device_bytes(arch, "adam", 32)
    P = 784 * 256 + 256 + 256 * 10 + 10
    assert b >= 6 * P * 4  # ping-pong params + two ping-pong slots
    assert device.member_device_bytes(arch, "sgd", 32) < b
    assert device.member_device_bytes(arch, "sgd", 32, "f64") > device.member_device_bytes(
        arch, "sgd", 32)


def test_accountant_registers_and_overflows():
    acct = device.DeviceAccountant(device.B200Device(memory_capacity=10_000_000))
    nb = device.member_device_bytes(ARCH, "adam", 10)
    h = packing.load_model(_h("m"), device=acct)
    assert acct.used == device.member_device_bytes(ARCH, "sgd", 10) and h.model_id == "m"
    big = packing.make_handle("big", packing.MLPArch(784, (2048,), 10), "adam", 0.1, 512, 1,
                              "d", 0)
    with pytest.raises(device.OOMError):
        packing.load_model(big, device=acct)
    assert "big" not in acct.resident and nb > 0


def test_preprocess_memo_matches_per_sample_path():
    """§8f-2: the whole-dataset preprocessed table equals the per-sample
    `preprocess` output row for row, and account_cache reproduces its
    hit/miss/entry bookkeeping (reference data.py:176-194)."""
    ds = data.synth_dataset(50, 6, 3, seed=4)
    spec = data.PreprocessSpec(stages=(("normalize", 0.5, 2.0), ("jitter", 7)))
    table = data.preprocess_all(spec, ds.features)
    idx = np.array([3, 17, 3, 42, 0])
    want = data.preprocess(spec, ds.features[idx], idx, ds.dataset_id)
    np.testing.assert_array_equal(table[idx], want)
    c1, c2 = data.PreprocessCache(), data.PreprocessCache()
    for batch in (idx, idx[::-1], np.array([1, 2])):
        data.preprocess(spec, ds.features[batch], batch, ds.dataset_id, c1)
        data.account_cache(spec, table, batch, ds.dataset_id, c2)
    assert (c1.hits, c1.misses) == (c2.hits, c2.misses)
    assert c1.entries.keys() == c2.entries.keys()
    for k in c1.entries:
        np.testing.assert_array_equal(c1.entries[k], c2.entries[k])


def test_costmodel_fit_recovers_known_coefficients_and_metric():
    """§8f-4: the Eq. 1-2 fit recovers t_fix / io / c_kind / κ from exact
    synthetic measurements, and the traintime metric follows tuner.py:118-127."""
    from paper_2002_02885_b200 import costmodel as cm
    true_dev = cm.DeviceProfile(1 << 30, 0.02, 1e-4, 0.0, 0.6)
    true_model = cm.ModelProfile("m", 0, 0, {"sgd": 2e-4, "adam": 5e-4, "momentum": 3e-4,
                                             "adagrad": 3e-4})

    def fake(hs, dsets, n):
        specs = [(h.optimizer.kind, h.batch_size) for h in hs]
        r = cm.estimate_step_time([(true_model, k, b) for k, b in specs], true_dev,
                                  [list(range(len(specs)))])
        return r.t_s_pack_ms if len(specs) > 1 else r.t_s_seq_ms

    samples = []
    for k in ("sgd", "adam"):
        for b in (20, 45, 70):
            samples.append((fake([_h("x", batch=b, opt=k)], None, 0), [(k, b)], 1))
        for n in (2, 4, 8):
            specs = [(k, 45)] * n
            hs = [_h(f"x{i}", batch=45, opt=k) for i in range(n)]
            samples.append((fake(hs, None, 0), specs, 1))
    dev, model = cm.fit(samples, 1 << 30)
    assert abs(dev.fixed_step_overhead_ms - 0.02) < 1e-6
    assert abs(dev.contention_factor - 0.6) < 1e-3
    for k in ("sgd", "adam"):
        assert abs(model.compute_ms_per_sample[k] - true_model.compute_ms_per_sample[k]) < 1e-6
    metric = cm.make_traintime_metric(model, dev)
    space = tuner.ConfigSpace()
    a, b = space.config(0), space.config(4)
    assert metric(a, b) == metric(b, a) and metric(a, b) > 0
    # usable as the kNN distance of the reference driver
    r = tuner.packed_hyperband(9, 3, tuner.StubExecutor(lambda c, e: c.config_id), seed=0,
                               strategy="knn", metric=metric, threshold=0.5)
    assert r.total_epochs > 0
