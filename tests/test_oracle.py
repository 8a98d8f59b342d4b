"""Pin the float64 oracle against the reference's golden vectors (CPU only).

The fixtures were produced by running the reference itself
(`tests/golden/make_golden.py`); the known answers are the reference's own
hand-evaluated tests (`pkg/tests/test_engine.py:56-179`).
"""
import json
import os

import numpy as np
import pytest

from oracle import mlp64 as O

G = os.path.join(os.path.dirname(__file__), "golden")


def _npz(name):
    return np.load(os.path.join(G, name))


def test_known_answers_match_reference_hand_evaluations():
    ka = json.load(open(os.path.join(G, "known_answers.json")))
    layers = [[np.array([[1.0, -1.0], [0.5, 0.5]]), np.array([0.0, 1.0])]]
    loss, _ = O.member_forward_loss(layers, "relu", [[1.0, 2.0]], [0])
    assert loss == ka["linear_softmax_loss"]
    assert loss == pytest.approx(-np.log(np.exp(2) / (np.exp(2) + np.exp(1))),
                                 abs=1e-12)
    # optimizers: run through optimizer_step on a 1-layer "net" whose W is the
    # vector under test (bias grads zero)
    for kind, lr, gs, w0 in [("sgd", 0.1, [[0.5, -1.0]], [1.0, 2.0]),
                             ("momentum", 0.1, [[1.0], [1.0]], [0.0]),
                             ("adagrad", 0.5, [[2.0]], [1.0]),
                             ("adam", 0.01, [[1.0], [2.0]], [0.0])]:
        layers = [[np.array(w0, dtype=float), np.zeros(1)]]
        slots, t = {}, 0
        for g in gs:
            t = O.optimizer_step(kind, lr, t, layers, slots,
                                 [(np.array(g, dtype=float), np.zeros(1))])
        np.testing.assert_allclose(layers[0][0], ka["optimizer_seq"][kind],
                                   rtol=0, atol=1e-15)
    np.testing.assert_allclose(ka["optimizer_seq"]["sgd"], [0.95, 2.1], atol=1e-15)
    np.testing.assert_allclose(ka["optimizer_seq"]["momentum"], [-0.29], atol=1e-15)


def test_zero_weights_give_log_classes():
    """tests/test_engine.py:46-53."""
    for c in (2, 3, 7):
        layers = [[np.zeros((4, 5)), np.zeros(5)], [np.zeros((5, c)), np.zeros(c)]]
        x = np.random.default_rng(0).normal(size=(6, 4))
        loss, _ = O.member_forward_loss(layers, "relu", x, np.zeros(6, int))
        assert loss == pytest.approx(np.log(c), abs=1e-12)


@pytest.mark.parametrize("act", O.ACTIVATIONS)
def test_oracle_gradients_match_finite_differences(act):
    """tests/test_engine.py:69-80 restated on the oracle."""
    rng = np.random.default_rng(5)
    layers = O.xavier_layers("m", (3, 4, 2), 1)
    x = rng.normal(size=(5, 3))
    y = rng.integers(0, 2, size=5)
    _, grads, _ = O.forward_backward(layers, act, x, y)
    h = 1e-6
    for li in range(2):
        for k in range(2):
            arr = layers[li][k]
            flat = arr.reshape(-1)
            gnum = np.zeros_like(flat)
            for i in range(flat.size):
                o = flat[i]
                flat[i] = o + h
                lp, _ = O.member_forward_loss(layers, act, x, y)
                flat[i] = o - h
                lm, _ = O.member_forward_loss(layers, act, x, y)
                flat[i] = o
                gnum[i] = (lp - lm) / (2 * h)
            ga = grads[li][k].reshape(-1)
            rel = np.abs(ga - gnum) / np.maximum(np.abs(ga) + np.abs(gnum), 1.0)
            assert rel.max() <= 1e-4


def test_padding_rows_are_inert_bit_exact():
    """tests/test_engine.py:113-129."""
    layers = O.xavier_layers("m", (3, 4, 2), 9)
    rng = np.random.default_rng(9)
    x = rng.normal(size=(3, 3))
    y = rng.integers(0, 2, size=3)
    xp = np.zeros((7, 3))
    xp[:3] = x
    yp = np.zeros(7, dtype=np.int64)
    yp[:3] = y
    l0, g0, _ = O.forward_backward(layers, "relu", x, y)
    l1, g1, _ = O.forward_backward(layers, "relu", xp, yp, n_valid=3)
    assert l0 == l1
    for a, b in zip(g0, g1):
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])


def test_config0_golden_trajectory():
    """BASELINE configs[0] run by the reference: dataset, permutation, init,
    step-1 params and three steps of losses (SURVEY §8c values)."""
    z = _npz("config0.npz")
    did, feats, labels = O.synth_blobs(10000, 784, 10, 0)
    assert did == str(z["dataset_id"])
    np.testing.assert_array_equal(
        [feats.std(), np.abs(feats).max(), feats[0, :8].sum()], z["feat_stats"])
    np.testing.assert_array_equal(O.epoch_order(did, 10000, 0)[:64], z["perm_head"])
    datasets = {"train": O.OracleDataset(did, feats, labels)}
    ms = [O.OracleMember.make(f"m{i}", (784, 256, 10), "relu", "sgd", lr, 32,
                              100, "train", 0) for i, lr in ((0, 0.1), (1, 0.01))]
    init = ms[0].flat_params()
    np.testing.assert_array_equal(init[:4096], z["init_m0_head"])
    losses = []
    for s in range(3):
        out, stats = O.oracle_packed_step(ms, datasets)
        losses.append([out["m0"], out["m1"]])
        if s == 0:
            p0, p1 = ms[0].flat_params(), ms[1].flat_params()
            np.testing.assert_allclose(p0[:4096], z["step1_m0_head"], rtol=1e-12, atol=1e-15)
            np.testing.assert_allclose(p1[784 * 256:784 * 256 + 256], z["step1_m1_b0"],
                                       rtol=1e-12, atol=1e-15)
            np.testing.assert_allclose([p0.sum(), (p0 ** 2).sum()], z["step1_m0_sum"], rtol=1e-12)
    np.testing.assert_allclose(losses, z["losses"], rtol=1e-9)
    assert list(stats.values()) == list(z["stats"])
    # SURVEY §8c quoted values
    assert losses[0][0] == pytest.approx(6.486935308541392, rel=1e-12)
    assert losses[0][1] == pytest.approx(6.3139062633732586, rel=1e-12)


@pytest.mark.parametrize("opt", O.OPTIMIZERS)
def test_small_pairs_golden(opt):
    z = _npz("small_pairs.npz")
    did, feats, labels = O.synth_blobs(120, 6, 3, 0)
    datasets = {"d": O.OracleDataset(did, feats, labels)}
    for act in O.ACTIVATIONS:
        a = O.OracleMember.make("a", (6, 8, 3), act, opt, 0.05, 10, 20, "d", 1)
        b = O.OracleMember.make("b", (6, 8, 3), act, opt, 0.01, 10, 20, "d", 2)
        ls = []
        for s in range(5):
            out, _ = O.oracle_packed_step([a, b], datasets)
            ls.append([out["a"], out["b"]])
            if s == 0:
                np.testing.assert_allclose(a.flat_params(), z[f"{opt}_{act}_a_p1"],
                                           rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(ls, z[f"{opt}_{act}_losses"], rtol=1e-10)
        np.testing.assert_allclose(b.flat_params(), z[f"{opt}_{act}_b_p5"],
                                   rtol=1e-10, atol=1e-13)


def test_deep_and_misaligned_golden():
    z = _npz("deep_misaligned.npz")
    did, feats, labels = O.synth_blobs(400, 5, 3, 8)
    datasets = {"d": O.OracleDataset(did, feats, labels)}
    for opt in O.OPTIMIZERS:
        ms = [O.OracleMember.make(f"m{i}", (5, 8, 8, 3), "relu", opt, 0.01, 16,
                                  50, "d", i) for i in (1, 2)]
        for _ in range(50):
            O.oracle_packed_step(ms, datasets)
        np.testing.assert_allclose(ms[0].flat_params(), z[f"c2_{opt}_m1"],
                                   rtol=1e-9, atol=1e-12)
    did, feats, labels = O.synth_blobs(1000, 6, 3, 4)
    datasets = {"d": O.OracleDataset(did, feats, labels)}
    specs = [("m20", 20, 50), ("m50", 50, 20), ("m100", 100, 10)]
    ms = [O.OracleMember.make(mid, (6, 8, 3), "relu", "sgd", 0.05, b, s, "d", i)
          for i, (mid, b, s) in enumerate(specs)]
    stats = []
    while any(not m.finished for m in ms):
        _, st = O.oracle_packed_step(ms, datasets, share_inputs=False)
        stats.append(list(st.values()))
    np.testing.assert_array_equal(stats, z["mis_stats"])
    for m in ms:
        np.testing.assert_allclose(m.flat_params(), z[f"mis_{m.model_id}"],
                                   rtol=1e-9, atol=1e-12)
        np.testing.assert_array_equal(m.samples_used, 1)
