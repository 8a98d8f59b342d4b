"""GPU parity of the packed train step (runs on a B200).

Two kinds of checks, mirroring the reference's test strategy:
  * lockstep parity: before every step the float64 oracle is loaded with the
    device's exact state and both take one step; losses, params, optimizer
    slots, cursors and stats must agree to rel 1e-4 + abs 1e-6 (fp32 device
    vs f64 oracle, BASELINE north_star).  Integer/indexing state is exact.
  * self-consistency, exact: packed == standalone, gradient isolation and
    dedup are bit-identical on the device (tests/test_pack.py:31-82).
"""
import json
import math
import os

import numpy as np
import pytest

from _helpers import (ATOL, RTOL, _assert_param_close, assert_close_member, has_gpu, lockstep,
                      oracle_dataset, oracle_from_handle)
from oracle import mlp64 as O

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

from paper_2002_02885_b200 import data, engine, packing, runtime, tuner  # noqa: E402

ARCH = packing.MLPArch(input_dim=6, hidden=(8,), classes=3)
G = os.path.join(os.path.dirname(__file__), "golden")


def _ds(n=120, seed=0, d=6, c=3):
    return {"d": data.synth_dataset(n, d, c, seed=seed)}


def _h(mid, batch=10, steps=20, opt="sgd", lr=0.05, seed=0, arch=ARCH, binding="d"):
    return packing.make_handle(mid, arch, opt, lr, batch, steps, binding, seed)


def _maxdiff(a, b):
    return max(float(np.max(np.abs(a.params[k] - b.params[k]))) for k in a.params)


# ------------------------------------------------------- oracle parity --

def test_config0_lockstep_three_steps():
    """BASELINE configs[0]: K=2 784-256-10, SGD 0.1 / 0.01, b=32."""
    ds = data.synth_dataset(10000, 784, 10, seed=0)
    arch = packing.MLPArch(784, (256,), 10, "relu")
    hs = [packing.make_handle(f"m{i}", arch, "sgd", lr, 32, 100, "train", 0)
          for i, lr in ((0, 0.1), (1, 0.01))]
    packed = packing.dedup_inputs(packing.pack_models(hs))
    lockstep(packed, {"train": ds}, 3, packing=packing)
    z = np.load(os.path.join(G, "config0.npz"))
    assert packed.last_step_stats == {"physical_inputs": 1, "groups": 1, "driver_batch": 32}
    # the first-step losses agree with the reference's own numbers
    hs2 = [packing.make_handle(f"m{i}", arch, "sgd", lr, 32, 100, "train", 0)
           for i, lr in ((0, 0.1), (1, 0.01))]
    out = packing.packed_step(packing.dedup_inputs(packing.pack_models(hs2)), {"train": ds})
    np.testing.assert_allclose([out["m0"], out["m1"]], z["losses"][0], rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("opt", engine.OPTIMIZERS)
@pytest.mark.parametrize("act", engine.ACTIVATIONS)
def test_small_pair_lockstep(opt, act):
    arch = packing.MLPArch(6, (8,), 3, act)
    hs = [_h("a", opt=opt, seed=1, arch=arch), _h("b", opt=opt, lr=0.01, seed=2, arch=arch)]
    lockstep(packing.dedup_inputs(packing.pack_models(hs)), _ds(), 6, packing=packing)


@pytest.mark.parametrize("opt", engine.OPTIMIZERS)
def test_deep_ragged_pack_lockstep(opt):
    """Members of different depth/width/activation/optimizer in one pack."""
    datasets = _ds(n=300, d=5, seed=8)
    hs = [packing.make_handle("deep", packing.MLPArch(5, (8, 8, 7), 3, "tanh"), opt, 0.01,
                              16, 50, "d", 1),
          packing.make_handle("wide", packing.MLPArch(5, (40,), 3, "sigmoid"), "adam", 0.003,
                              16, 50, "d", 2),
          packing.make_handle("lin", packing.MLPArch(5, (), 3, "relu"), "momentum", 0.02, 9,
                              50, "d", 3)]
    lockstep(packing.dedup_inputs(packing.pack_models(hs)), datasets, 8, packing=packing)


def test_wide_layers_cross_tile_boundaries():
    """Dims not multiples of the tile sizes, batch > one row tile."""
    datasets = _ds(n=500, d=77, c=13, seed=3)
    hs = [packing.make_handle("x", packing.MLPArch(77, (45, 33), 13, "leaky_relu"), "adam",
                              0.002, 70, 20, "d", 1),
          packing.make_handle("y", packing.MLPArch(77, (130,), 13, "relu"), "adagrad", 0.05,
                              37, 20, "d", 2)]
    lockstep(packing.pack_models(hs), datasets, 5, share_inputs=False, packing=packing)


def test_misaligned_batches_coverage_and_parity():
    """tests/test_pack.py:113-138 + per-step oracle parity."""
    n = 1000
    datasets = {"d": data.synth_dataset(n, 6, 3, seed=4)}
    specs = [("m20", 20, 50), ("m50", 50, 20), ("m100", 100, 10)]
    members = [_h(mid, batch=b, steps=s, seed=i) for i, (mid, b, s) in enumerate(specs)]
    packed = packing.pack_models(members)
    lockstep(packed, datasets, 10, share_inputs=False, packing=packing)
    assert members[2].finished
    assert members[1].cursor.pos == n // 2
    while any(not h.finished for h in members):
        packing.packed_step(packed, datasets)
    for h, (mid, b, s) in zip(members, specs):
        assert h.cursor.steps_done == s
        np.testing.assert_array_equal(h.cursor.samples_used, 1)
    z = np.load(os.path.join(G, "deep_misaligned.npz"))
    for h in members:  # whole trajectory vs the reference (fp32 drift bound)
        flat = h._flat_params(h.params)
        np.testing.assert_allclose(flat, z[f"mis_{h.model_id}"], rtol=1e-3, atol=1e-4)


def test_golden_trajectories_f32():
    """5 packed steps from the reference's init vs its golden params."""
    z = np.load(os.path.join(G, "small_pairs.npz"))
    for opt in engine.OPTIMIZERS:
        arch = packing.MLPArch(6, (8,), 3, "tanh")
        a = _h("a", opt=opt, seed=1, arch=arch)
        b = _h("b", opt=opt, lr=0.01, seed=2, arch=arch)
        packed = packing.dedup_inputs(packing.pack_models([a, b]))
        ls = [list(packing.packed_step(packed, _ds()).values()) for _ in range(5)]
        np.testing.assert_allclose(ls, z[f"{opt}_tanh_losses"], rtol=1e-3, atol=1e-5)
        np.testing.assert_allclose(b._flat_params(b.params), z[f"{opt}_tanh_b_p5"],
                                   rtol=1e-3, atol=1e-5)


# ------------------------------------------------ exact self-consistency --

def test_singleton_pack_matches_standalone_exactly():
    datasets = _ds()
    ph, solo = _h("m", seed=3), _h("m", seed=3)
    packed = packing.pack_models([ph])
    for _ in range(20):
        packing.packed_step(packed, datasets)
        packing.standalone_step(solo, datasets)
    assert _maxdiff(ph, solo) == 0.0


@pytest.mark.parametrize("opt", engine.OPTIMIZERS)
def test_packed_pair_reproduces_standalone_bitwise(opt):
    datasets = _ds()
    pa, pb = _h("a", opt=opt, seed=1), _h("b", opt=opt, seed=2)
    sa, sb = _h("a", opt=opt, seed=1), _h("b", opt=opt, seed=2)
    packed = packing.pack_models([pa, pb])
    for _ in range(20):
        packing.packed_step(packed, datasets)
    for _ in range(20):
        packing.standalone_step(sa, datasets)
        packing.standalone_step(sb, datasets)
    assert _maxdiff(pa, sa) == 0.0 and _maxdiff(pb, sb) == 0.0


def test_gradient_isolation_members_do_not_interact():
    datasets = _ds()
    alone, with_b = _h("a", seed=1), _h("a", seed=1)
    packed = packing.pack_models([with_b, _h("b", batch=7, seed=9, opt="adam", lr=0.001)])
    packing.standalone_step(alone, datasets)
    packing.packed_step(packed, datasets)
    assert _maxdiff(alone, with_b) == 0.0


def test_k_invariance_large_pack():
    """A member's trajectory is bit-identical inside a 16-member pack."""
    datasets = {"t": data.synth_dataset(2000, 64, 10, seed=5)}
    arch = packing.MLPArch(64, (96,), 10, "relu")
    hs = [packing.make_handle(f"k{i}", arch, ("sgd", "adam", "momentum", "adagrad")[i % 4],
                              0.01 * (1 + i % 3), 32 + 4 * (i % 3), 30, "t", i)
          for i in range(16)]
    solo = packing.make_handle("k5", arch, "adam", 0.01 * (1 + 5 % 3), 32 + 4 * (5 % 3), 30,
                               "t", 5)
    packed = packing.dedup_inputs(packing.pack_models(hs))
    for _ in range(12):
        packing.packed_step(packed, datasets)
        packing.standalone_step(solo, datasets)
    assert _maxdiff(hs[5], solo) == 0.0


def test_dedup_inputs_is_value_preserving_and_collapses_transfers():
    datasets = _ds()
    plain = [_h("a", seed=1), _h("b", seed=2)]
    deduped = [_h("a", seed=1), _h("b", seed=2)]
    p1, p2 = packing.pack_models(plain), packing.dedup_inputs(packing.pack_models(deduped))
    for _ in range(10):
        packing.packed_step(p1, datasets)
        packing.packed_step(p2, datasets)
    assert p1.last_step_stats["physical_inputs"] == 2
    assert p2.last_step_stats["physical_inputs"] == 1
    for a, b in zip(plain, deduped):
        assert _maxdiff(a, b) == 0.0


# --------------------------------------------------------- pack semantics --

def test_driver_batch_tracks_largest_active_member():
    datasets = _ds(n=100)
    big, small = _h("big", batch=50, steps=2), _h("small", batch=10, steps=10)
    packed = packing.pack_models([big, small])
    packing.packed_step(packed, datasets)
    assert packed.last_step_stats["driver_batch"] == 50
    packing.packed_step(packed, datasets)
    assert big.finished
    packing.packed_step(packed, datasets)
    assert packed.driver_batch == 10 and packed.last_step_stats["driver_batch"] == 10


def test_partial_final_batch_never_spans_epochs():
    datasets = _ds(n=25)
    h = _h("m", batch=10, steps=6)
    packed = packing.pack_models([h])
    for _ in range(3):
        packing.packed_step(packed, datasets)
    assert h.cursor.pos == 25 and h.cursor.epoch_index == 0
    packing.packed_step(packed, datasets)
    assert h.cursor.epoch_index == 1 and h.cursor.pos == 10


def test_run_epoch_and_replan():
    datasets = _ds(n=100)
    members = [_h("a", batch=50, steps=100), _h("b", batch=20, steps=100)]
    plan = packing.make_epoch_plan(members, datasets)
    losses = packing.run_epoch(packing.pack_models(members), datasets)
    assert len(losses) == sum(s for _, s in plan)
    for h in members:
        np.testing.assert_array_equal(h.cursor.samples_used, 1)


def test_finished_members_are_left_alone():
    datasets = _ds()
    done, working = _h("done", steps=1), _h("working", steps=3)
    packed = packing.pack_models([done, working])
    packing.packed_step(packed, datasets)
    frozen = {k: v.copy() for k, v in done.params.items()}
    packing.packed_step(packed, datasets)
    for k in frozen:
        np.testing.assert_array_equal(done.params[k], frozen[k])
    working.cursor.steps_done = working.target_steps
    with pytest.raises(packing.ReplanNeeded):
        packing.packed_step(packed, datasets)


def test_host_edit_of_params_is_uploaded():
    datasets = _ds()
    a, b = _h("a", seed=1), _h("a", seed=1)
    pa = packing.pack_models([a])
    packing.packed_step(pa, datasets)
    packing.standalone_step(b, datasets)
    a.params["a/L0/W"][0, 0] += 0.5  # in-place edit, as reference users do
    b.params["a/L0/W"][0, 0] += 0.5
    packing.packed_step(pa, datasets)
    packing.standalone_step(b, datasets)
    assert _maxdiff(a, b) == 0.0


# ------------------------------------------------------------ failures --

def test_nonfinite_input_raises_engine_error_and_commits_nothing():
    ds = data.synth_dataset(120, 6, 3, seed=0)
    x = ds.features.copy()
    perm = data.epoch_permutation(ds.dataset_id + "-nan", ds.n, 0)
    x[perm[3], 2] = np.nan
    bad = data.Dataset(ds.dataset_id + "-nan", x, ds.labels, 3)
    a, b = _h("a", seed=1), _h("b", seed=2)
    packed = packing.pack_models([a, b])
    before = {k: v.copy() for k, v in a.params.items()}
    with pytest.raises(engine.EngineError, match="non-finite value at node 'a/in'"):
        packing.packed_step(packed, {"d": bad})
    assert a.cursor.steps_done == 0 and a.optimizer.step_counter == 0
    for k in before:
        np.testing.assert_array_equal(a.params[k], before[k])


def test_nonfinite_param_names_the_affine_node():
    a = _h("a", seed=1)
    a.params["a/L1/W"][0, 0] = np.inf
    with pytest.raises(engine.EngineError, match="a/aff1"):
        packing.packed_step(packing.pack_models([a]), _ds())


def test_nonfinite_gradient_commit_rules():
    """engine.py:297-299 + packing.py:250-253: members before the bad one
    commit, the bad one and later ones do not; counters stay put."""
    datasets = _ds()
    a, b, c = _h("a", seed=1), _h("b", seed=2), _h("c", seed=3)
    sa = _h("a", seed=1)
    packed = packing.pack_models([a, b, c])
    rt = runtime.runtime()
    packed._device_pack(rt)
    pb = {k: v.copy() for k, v in b.params.items()}
    pc = {k: v.copy() for k, v in c.params.items()}
    b._dev.inject_fault(2)  # grads order: L1/W, L1/b, L0/W, L0/b → "b/L0/W"
    with pytest.raises(engine.NonFiniteGradient) as err:
        packing.packed_step(packed, datasets)
    assert err.value.param == "b/L0/W"
    packing.standalone_step(sa, datasets)
    assert _maxdiff(a, sa) == 0.0 and a.optimizer.step_counter == 1
    assert a.cursor.steps_done == 1
    assert b.optimizer.step_counter == 0 and b.cursor.steps_done == 0
    assert c.optimizer.step_counter == 0 and c.cursor.steps_done == 0
    for k in pb:
        np.testing.assert_array_equal(b.params[k], pb[k])
    for k in pc:
        np.testing.assert_array_equal(c.params[k], pc[k])
    # the fault is one-shot: the next step succeeds for b and c
    out = packing.packed_step(packed, datasets)
    assert set(out) == {"a", "b", "c"}


def test_shape_mismatch_names_the_port():
    h = packing.make_handle("m", packing.MLPArch(5, (4,), 3), "sgd", 0.1, 4, 2, "d", 0)
    with pytest.raises(engine.ShapeMismatch) as err:
        packing.packed_step(packing.pack_models([h]), _ds())
    assert err.value.port == "m/x"


# ---------------------------------------------------------- checkpoints --

def test_checkpoint_round_trip_is_exact():
    datasets = _ds()
    h = _h("m", opt="adam", lr=0.001, steps=30)
    for _ in range(7):
        packing.standalone_step(h, datasets)
    raw = packing.checkpoint_model(h).to_bytes()
    back = packing.restore_handle(packing.Checkpoint.from_bytes(raw), datasets)
    assert back.optimizer.step_counter == 7 and back.cursor.pos == h.cursor.pos
    for k in h.params:
        np.testing.assert_array_equal(back.params[k], h.params[k])
    for p in h.optimizer.slots:
        for s in h.optimizer.slots[p]:
            np.testing.assert_array_equal(back.optimizer.slots[p][s], h.optimizer.slots[p][s])


def test_free_load_resume_equals_uninterrupted():
    datasets = _ds()
    interrupted = _h("m", opt="momentum", steps=40, seed=5)
    straight = _h("m", opt="momentum", steps=40, seed=5)
    packed = packing.pack_models([interrupted])
    for _ in range(15):
        packing.packed_step(packed, datasets)
    ckpt, packed = packing.free_model(packed, "m")
    assert packed.members == []
    resumed = packing.load_model(packing.Checkpoint.from_bytes(ckpt.to_bytes()),
                                 datasets=datasets)
    packed = packing.pack_models([resumed])
    while not resumed.finished:
        packing.packed_step(packed, datasets)
    while not straight.finished:
        packing.standalone_step(straight, datasets)
    assert _maxdiff(resumed, straight) == 0.0


def test_mid_pack_replacement_scenario():
    datasets = _ds(n=200)
    short = _h("short", batch=20, steps=10, seed=1)
    long_p, long_s = _h("long", batch=10, steps=40, seed=2), _h("long", batch=10, steps=40, seed=2)
    packed = packing.pack_models([short, long_p])
    for _ in range(10):
        packing.packed_step(packed, datasets)
    assert short.finished and not long_p.finished
    ckpt, packed = packing.free_model(packed, "short")
    newcomer = _h("late", batch=30, steps=15, seed=3)
    packed = packing.pack_models(packed.members + [newcomer])
    while any(not h.finished for h in packed.members):
        packing.packed_step(packed, datasets)
    assert long_p.cursor.steps_done == 40 and newcomer.cursor.steps_done == 15
    while not long_s.finished:
        packing.standalone_step(long_s, datasets)
    assert _maxdiff(long_p, long_s) == 0.0


def test_preprocessing_inside_pack_matches_standalone():
    datasets = _ds()
    spec = data.PreprocessSpec(stages=(("normalize", 0.5, 2.0), ("jitter", 7)))
    cache = data.PreprocessCache()
    pa, sa = _h("a", seed=1), _h("a", seed=1)
    packed = packing.dedup_inputs(packing.pack_models([pa, _h("b", seed=2)]))
    for _ in range(5):
        packing.packed_step(packed, datasets, preprocess_spec=spec, cache=cache)
        packing.standalone_step(sa, datasets, preprocess_spec=spec, cache=cache)
    assert _maxdiff(pa, sa) == 0.0
    assert cache.hits > 0


# ------------------------------------------------------------ f64 mode --

def test_f64_context_reproduces_reference_golden_to_1e10():
    """With a float64 device context the B200 path reproduces the reference's
    own trajectories (tests/golden/small_pairs.npz) to ~1e-12."""
    z = np.load(os.path.join(G, "small_pairs.npz"))
    runtime.set_precision("f64")
    try:
        for opt in engine.OPTIMIZERS:
            for act in engine.ACTIVATIONS:
                arch = packing.MLPArch(6, (8,), 3, act)
                a = _h("a", opt=opt, seed=1, arch=arch)
                b = _h("b", opt=opt, lr=0.01, seed=2, arch=arch)
                packed = packing.dedup_inputs(packing.pack_models([a, b]))
                ls = [list(packing.packed_step(packed, _ds()).values()) for _ in range(5)]
                np.testing.assert_allclose(ls, z[f"{opt}_{act}_losses"], rtol=1e-10, atol=1e-13)
                np.testing.assert_allclose(b._flat_params(b.params), z[f"{opt}_{act}_b_p5"],
                                           rtol=1e-10, atol=1e-13)
    finally:
        runtime.set_precision("f32")


def test_f64_packed_run_reproduces_reference_golden():
    """The native multi-step driver in the float64 context (the Hyperband
    executor's mode): the reference's own 5-step trajectories, streamed and
    resident inputs."""
    z = np.load(os.path.join(G, "small_pairs.npz"))
    runtime.set_precision("f64")
    try:
        for mode in ("resident", "stream"):
            runtime.set_input_mode(mode)
            for opt in engine.OPTIMIZERS:
                arch = packing.MLPArch(6, (8,), 3, "tanh")
                a = _h("a", opt=opt, seed=1, arch=arch)
                b = _h("b", opt=opt, lr=0.01, seed=2, arch=arch)
                packed = packing.dedup_inputs(packing.pack_models([a, b]))
                ls = [list(d.values()) for d in packing.packed_run(packed, _ds(), 5)]
                np.testing.assert_allclose(ls, z[f"{opt}_tanh_losses"], rtol=1e-10, atol=1e-13)
                np.testing.assert_allclose(b._flat_params(b.params), z[f"{opt}_tanh_b_p5"],
                                           rtol=1e-10, atol=1e-13)
    finally:
        runtime.set_input_mode("resident")
        runtime.set_precision("f32")


def test_fwd_input_ranges_lockstep_parity():
    """Generic forward with input ranges (in=300: 3 ranges of 2 chunks) and
    tiles shared by several CTAs: per-step parity with the f64 oracle."""
    datasets = _ds(n=400, d=300, c=10, seed=11)
    hs = [packing.make_handle(f"r{i}", packing.MLPArch(300, (40, 24), 10, "relu"), opt, lr,
                              b, 20, "d", i)
          for i, (opt, lr, b) in enumerate((("sgd", 0.05, 40), ("adam", 0.002, 33),
                                            ("momentum", 0.02, 64)))]
    lockstep(packing.dedup_inputs(packing.pack_models(hs)), datasets, 5, packing=packing)


def test_narrow_wgrad_tiles_match_square_tiles_bitwise(plan):
    """Weight-gradient tiles of narrow layers (out <= 16) are 64x16 instead of
    32x32: the per-element sums keep their order, so the trajectories are
    bit-identical to the 32x32 tiles (plan option wgrad_narrow=0)."""
    datasets = _ds(n=300, d=100, c=10, seed=4)
    arch = packing.MLPArch(100, (16, 12), 10, "tanh")
    runs = []
    for narrow in (True, False):
        plan(wgrad_narrow=int(narrow))
        hs = [packing.make_handle(f"w{i}", arch, opt, 0.01, 24, 20, "d", i)
              for i, opt in enumerate(("adam", "momentum"))]
        packed = packing.pack_models(hs)
        for _ in range(5):
            packing.packed_step(packed, datasets)
        runs.append(hs)
    for a, b in zip(*runs):
        assert _maxdiff(a, b) == 0.0


def test_f64_fwd_input_ranges_k_invariant():
    """Hyperband shape (784-16-10, float64): a member alone shares each forward
    tile among 7 CTAs, inside an 8-member pack among 4; the input-range sums
    are the same, so the trajectories are bit-identical."""
    runtime.set_precision("f64")
    try:
        ds = {"t": data.synth_dataset(600, 784, 10, seed=7)}
        arch = packing.MLPArch(784, (16,), 10, "relu")

        def mk(i):
            return packing.make_handle(f"h{i}", arch, ("sgd", "adam", "momentum", "adagrad")[i % 4],
                                       0.01 * (1 + i % 3), 40, 30, "t", i)
        hs, solo = [mk(i) for i in range(8)], [mk(i) for i in range(8)]
        packed = packing.dedup_inputs(packing.pack_models(hs))
        for _ in range(6):
            packing.packed_step(packed, ds)
        for h in solo:
            for _ in range(6):
                packing.standalone_step(h, ds)
        for a, b in zip(hs, solo):
            assert _maxdiff(a, b) == 0.0
    finally:
        runtime.set_precision("f32")


# ------------------------------------------------------ device memory --

def test_member_device_bytes_matches_allocation():
    from paper_2002_02885_b200 import device
    rt = runtime.runtime()
    for arch, opt, b in [(ARCH, "sgd", 10), (packing.MLPArch(784, (256,), 10), "adam", 32),
                         (packing.MLPArch(5, (8, 8, 7), 3), "momentum", 17)]:
        m = runtime.DeviceMember(rt, arch.dims, arch.activation, opt, 0.1, b)
        assert m.device_bytes == device.member_device_bytes(arch, opt, b)


# ------------------------------------------------------------- tuning --

def test_val_loss_matches_oracle():
    ds = data.synth_dataset(300, 5, 3, seed=30)
    ex = tuner.B200Executor(ds, hidden=(6,), seed=0)
    space = tuner.ConfigSpace()
    cfgs = [space.config(i) for i in (3, 100, 555)]
    hs = [ex._handle(c) for c in cfgs]
    got = ex.val_losses(hs)
    vx = oracle_dataset(ex.val).features
    for h, g in zip(hs, got):
        m = oracle_from_handle(h)
        want, _ = O.member_forward_loss(m.layers, m.act, vx, ex.val.labels)
        assert abs(g - want) <= RTOL * abs(want) + ATOL


def test_engine_micro_tuning_matches_reference_records():
    """Acceptance C10 on the device: original and knn agree per config
    (<= 1e-6), and both agree with the reference's own records."""
    ref = json.load(open(os.path.join(G, "tuning.json")))
    dataset = data.synth_dataset(120, 5, 3, seed=30)
    space = tuner.ConfigSpace(batch_sizes=(10, 20, 30), optimizers=("sgd", "adam"),
                              learning_rates=(1e-3, 1e-2), activations=("relu", "tanh"))
    res = {}
    for strategy in ("original", "knn"):
        ex = tuner.B200Executor(dataset, hidden=(6,), seed=0)
        res[strategy] = tuner.packed_hyperband(4, 2, ex, seed=0, strategy=strategy, space=space)
    by = {(r.bracket, r.rung, r.config_id): r.loss for r in res["original"].records}
    for r in res["knn"].records:
        assert abs(r.loss - by[(r.bracket, r.rung, r.config_id)]) <= 1e-6
    assert res["knn"].best_config.config_id == res["original"].best_config.config_id
    for strategy in ("original", "knn"):
        want = {(b, ru, c): loss for b, ru, g, c, e, loss in ref[strategy]["records"]}
        for r in res[strategy].records:
            w = want[(r.bracket, r.rung, r.config_id)]
            assert abs(r.loss - w) <= 1e-3 * abs(w) + 1e-4
        assert res[strategy].best_config.config_id == ref[strategy]["best"]


def test_pool_world1_matches_serial_and_migrates_state_bitwise():
    """hyperband_pool on one GPU reproduces the serial packed_hyperband records
    exactly, and a member's state survives the pool's PKCK migration hooks
    (export → drop → import) bit for bit."""
    from paper_2002_02885_b200 import hyperband_pool
    dataset = data.synth_dataset(120, 8, 3, seed=31)
    space = tuner.ConfigSpace(batch_sizes=(10, 20), optimizers=("sgd", "adam"),
                              learning_rates=(1e-3, 1e-2), activations=("relu", "tanh"))
    serial = tuner.packed_hyperband(4, 2, tuner.B200Executor(dataset, hidden=(8,), seed=0),
                                    seed=0, strategy="knn", space=space)
    res, pool = hyperband_pool.sharded_hyperband(
        4, 2, tuner.B200Executor(dataset, hidden=(8,), seed=0), seed=0, strategy="knn",
        space=space)
    assert [(r.bracket, r.rung, r.group, r.config_id, r.loss) for r in res.records] == \
        [(r.bracket, r.rung, r.group, r.config_id, r.loss) for r in serial.records]
    assert res.best_config.config_id == serial.best_config.config_id
    # migration round trip on a trained member (adam: params + both slots)
    ex = tuner.B200Executor(dataset, hidden=(8,), seed=0)
    cfg = space.config(5)
    ex.evaluate([cfg], 2)
    h = ex.handles[cfg.config_id]
    before = (h._flat_params(h.params), h._flat_slots(), h.optimizer.step_counter,
              h.cursor.steps_done, h.cursor.pos)
    raw = ex.export_state(cfg.config_id)
    ex.drop_state(cfg.config_id)
    ex.import_state(cfg.config_id, raw)
    g = ex.handles[cfg.config_id]
    after = (g._flat_params(g.params), g._flat_slots(), g.optimizer.step_counter,
             g.cursor.steps_done, g.cursor.pos)
    np.testing.assert_array_equal(before[0], after[0])
    if before[1] is not None:
        np.testing.assert_array_equal(before[1], after[1])
    assert before[2:] == after[2:]
    # and the migrated member keeps training identically to an unmigrated twin
    twin = tuner.B200Executor(dataset, hidden=(8,), seed=0)
    twin.evaluate([cfg], 2)
    l1, _ = ex.evaluate([cfg], 1)
    l2, _ = twin.evaluate([cfg], 1)
    assert l1 == l2


def test_streamed_inputs_match_resident_bitwise():
    """input_mode 'stream' (host gather → pinned → H2D per step) trains the
    same bits as the device-resident gather, with and without preprocessing."""
    spec = data.PreprocessSpec(stages=(("normalize", 0.5, 2.0), ("jitter", 7)))
    out = {}
    for mode in ("resident", "stream"):
        runtime.set_input_mode(mode)
        try:
            datasets = _ds()
            hs = [_h("a", seed=1), _h("b", seed=2, opt="adam")]
            packed = packing.dedup_inputs(packing.pack_models(hs))
            cache = data.PreprocessCache()
            losses = [packing.packed_step(packed, datasets, preprocess_spec=spec if i % 2 else None,
                                          cache=cache) for i in range(6)]
            out[mode] = (losses, [h._flat_params(h.params) for h in hs], cache.hits, cache.misses)
        finally:
            runtime.set_input_mode("resident")
    assert out["resident"][0] == out["stream"][0]
    for a, b in zip(out["resident"][1], out["stream"][1]):
        np.testing.assert_array_equal(a, b)
    assert out["resident"][2:] == out["stream"][2:]


def test_packed_run_streamed_inputs_match_resident_bitwise():
    """packed_run with 16 steps in flight in input_mode 'stream': every
    in-flight step owns its pinned + device staging slot, so the trajectory
    equals the resident packed_step loop bit for bit (epoch rolls included)."""
    out = {}
    for mode in ("resident", "stream"):
        runtime.set_input_mode(mode)
        try:
            datasets = _ds(n=50)
            hs = [_h("a", seed=1, steps=40), _h("b", seed=2, opt="adam", batch=7, steps=40)]
            packed = packing.dedup_inputs(packing.pack_models(hs))
            if mode == "stream":
                losses = packing.packed_run(packed, datasets, 30, depth=16)
            else:
                losses = [packing.packed_step(packed, datasets) for _ in range(30)]
            out[mode] = (losses, [h._flat_params(h.params) for h in hs])
        finally:
            runtime.set_input_mode("resident")
    assert out["resident"][0] == out["stream"][0]
    for a, b in zip(out["resident"][1], out["stream"][1]):
        np.testing.assert_array_equal(a, b)


def test_costmodel_calibrates_on_device():
    """§8f-4: Eqs. 1-2 fitted to packed steps timed on this GPU; packing K
    same-batch members must be predicted (and measured) cheaper than K
    sequential steps."""
    from paper_2002_02885_b200 import costmodel as cm
    dev, model = cm.calibrate(input_dim=64, hidden=(16,), classes=4, batches=(20, 40),
                              kinds=("sgd",), pack_sizes=(2, 4), steps=10)
    assert dev.fixed_step_overhead_ms > 0
    assert all(v > 0 for v in model.compute_ms_per_sample.values())
    r = cm.estimate_step_time([(model, "sgd", 40)] * 4, dev, [[0, 1, 2, 3]])
    assert r.impv > 0
    metric = cm.make_traintime_metric(model, dev)
    space = tuner.ConfigSpace()
    assert metric(space.config(0), space.config(1)) >= 0


def test_hyperband_with_calibrated_traintime_metric():
    """§8f-4 in use: a pack-aware Hyperband run grouping by the training-time
    distance with the B200-calibrated cost model (tuner.py:118-127 with measured
    coefficients) instead of the index-sum distance.  Grouping changes which
    configs share packs, never a config's trajectory: every (config, rung) loss
    and the selected config equal the unpacked run's."""
    from paper_2002_02885_b200 import costmodel as cm
    dev, model = cm.calibrate(input_dim=784, hidden=(16,), classes=10, batches=(20, 45, 70),
                              kinds=("sgd", "adam", "momentum", "adagrad"), pack_sizes=(2, 4),
                              steps=10)
    metric = cm.make_traintime_metric(model, dev)
    ds = data.synth_dataset(600, 784, 10, seed=11, spread=0.1)
    res = {}
    for strat, kw in (("original", {}), ("knn", {"metric": metric, "threshold": 0.5})):
        ex = tuner.B200Executor(ds, hidden=(16,), seed=0)
        res[strat] = tuner.packed_hyperband(9, 3, ex, seed=4, strategy=strat, **kw)
    key = lambda r: sorted((x.config_id, x.epochs, x.loss) for x in r.records)  # noqa: E731
    assert key(res["original"]) == key(res["knn"])
    assert res["original"].best_config.config_id == res["knn"].best_config.config_id
    sizes = {}
    for x in res["knn"].records:
        sizes[(x.bracket, x.rung, x.group)] = sizes.get((x.bracket, x.rung, x.group), 0) + 1
    assert max(sizes.values()) >= 2  # the traintime distance really packed configs


# ------------------------------------------- tcgen05 path: schedule shapes --

def test_tensor_path_grouped_input_tiles_lockstep(plan):
    """8 wide members (mixed optimizers) on the tcgen05 path: the backward
    groups several 128-input tiles per CTA (G > 1) with two cp.async stages;
    one-step parity with the f64 oracle and packed == standalone bitwise."""
    plan(m1x=0)  # exercise the tcgen05 path
    from paper_2002_02885_b200 import device
    ds = {"t": data.synth_dataset(3000, 784, 10, seed=7, spread=0.5)}
    arch = packing.MLPArch(784, (256,), 10, "tanh")
    opts = ("sgd", "adam", "momentum", "adagrad")
    hs = [packing.make_handle(f"g{i}", arch, opts[i % 4], 0.01 / (1 + i), 32, 50, "t", i)
          for i in range(8)]
    assert all(device.uses_m1t(arch, h.optimizer.kind, 32) for h in hs)
    packed = packing.dedup_inputs(packing.pack_models(hs))
    lockstep(packed, ds, 2, packing=packing)
    solo = packing.make_handle("g5", arch, opts[5 % 4], 0.01 / 6, 32, 50, "t", 5)
    for _ in range(2):
        packing.standalone_step(solo, ds)
    assert _maxdiff(hs[5], solo) == 0.0


def test_tensor_path_batch_128_rows_lockstep(plan):
    """RP = 128 rows (batch 100): four 32-row K chunks per backward tile and
    one input-tile stage; parity with the oracle."""
    plan(m1x=0)  # exercise the tcgen05 path
    from paper_2002_02885_b200 import device
    ds = {"t": data.synth_dataset(1000, 200, 7, seed=8, spread=0.5)}
    arch = packing.MLPArch(200, (36,), 7, "sigmoid")
    hs = [packing.make_handle("r0", arch, "adagrad", 0.01, 100, 20, "t", 1),
          packing.make_handle("r1", arch, "momentum", 0.05, 100, 20, "t", 2)]
    assert all(device.uses_m1t(arch, h.optimizer.kind, 100) for h in hs)
    lockstep(packing.dedup_inputs(packing.pack_models(hs)), ds, 3, packing=packing)


def test_pack_beyond_inline_descriptors():
    """K = 40 > 32: step descriptors go through the H2D copy and finalize
    takes its general path; still parity and K-invariance."""
    ds = {"t": data.synth_dataset(400, 12, 4, seed=9)}
    arch = packing.MLPArch(12, (8,), 4, "relu")
    hs = [packing.make_handle(f"w{i}", arch, ("sgd", "adam")[i % 2], 0.02, 16, 10, "t", i)
          for i in range(40)]
    packed = packing.dedup_inputs(packing.pack_models(hs))
    lockstep(packed, ds, 2, packing=packing)
    solo = packing.make_handle("w7", arch, "adam", 0.02, 16, 10, "t", 7)
    for _ in range(2):
        packing.standalone_step(solo, ds)
    assert _maxdiff(hs[7], solo) == 0.0


def test_streaming_forward_large_pack_lockstep(plan):
    """12 x 784-256-10 members under the default plan: the forward is the
    cluster-resident k_m1c_fwd here (its clusters fit one wave; the streaming
    k_m1s_fwd is pinned by test_forced_streaming_forward_lockstep_and_kernel and
    reached by default at the wide16 shape); parity with the oracle, packed ==
    standalone (split-K cluster forward) bitwise."""
    plan(m1x=0)  # exercise the tcgen05 path
    ds = {"t": data.synth_dataset(3000, 784, 10, seed=11, spread=0.5)}
    arch = packing.MLPArch(784, (256,), 10, "leaky_relu")
    opts = ("sgd", "momentum", "adagrad", "adam")
    hs = [packing.make_handle(f"s{i}", arch, opts[i % 4], 0.02 / (1 + i), 32, 50, "t", i)
          for i in range(12)]
    packed = packing.dedup_inputs(packing.pack_models(hs))
    lockstep(packed, ds, 2, packing=packing)
    # the one-member pack takes the split-K cluster forward; the streaming
    # forward reproduces its arithmetic exactly → bit-identical trajectories
    solo = packing.make_handle("s4", arch, "sgd", 0.02 / 5, 32, 50, "t", 4)
    for _ in range(2):
        packing.standalone_step(solo, ds)
    assert _maxdiff(hs[4], solo) == 0.0


def test_tensor_path_ragged_heterogeneous_pack(plan):
    """Config-3-style heterogeneous pack on the tensor path: members with
    different hidden widths, class counts, batch sizes and input datasets
    (dimensions) share one pack — dummy cluster splits for the shallower
    inputs, ragged unit tiles; oracle parity and K-invariance."""
    plan(m1x=0)  # exercise the tcgen05 path
    from paper_2002_02885_b200 import device
    ds = {"a": data.synth_dataset(800, 784, 10, seed=12, spread=0.5),
          "b": data.synth_dataset(600, 256, 32, seed=13, spread=0.5)}
    specs = [("h0", packing.MLPArch(784, (16,), 10, "relu"), "adam", 0.01, 20, "a"),
             ("h1", packing.MLPArch(784, (100,), 10, "tanh"), "sgd", 0.05, 45, "a"),
             ("h2", packing.MLPArch(256, (256,), 32, "sigmoid"), "momentum", 0.02, 64, "b"),
             ("h3", packing.MLPArch(256, (36,), 32, "leaky_relu"), "adagrad", 0.02, 64, "b")]
    hs = [packing.make_handle(m, a, o, lr, b, 30, d, i) for i, (m, a, o, lr, b, d) in enumerate(specs)]
    assert all(device.uses_m1t(h.arch, h.optimizer.kind, h.batch_size) for h in hs)
    packed = packing.dedup_inputs(packing.pack_models(hs))
    lockstep(packed, ds, 3, packing=packing)
    solo = packing.make_handle("h2", specs[2][1], "momentum", 0.02, 64, 30, "b", 2)
    for _ in range(3):
        packing.standalone_step(solo, ds)
    assert _maxdiff(hs[2], solo) == 0.0


# ------------------------------------- one-launch cluster step (k_m1x) --

def test_m1x_mixed_optimizers_lockstep_and_cluster_size_invariance(plan):
    """8 x 784-256-10 members (all four optimizers) on the one-launch cluster
    step: parity with the f64 oracle per step, and the packed member equals
    its standalone run bit for bit although the pack runs 8-CTA clusters
    (2 unit blocks per CTA) and the singleton 16-CTA clusters (1 block)."""
    plan(m1x=1)
    from paper_2002_02885_b200 import device
    ds = {"t": data.synth_dataset(3000, 784, 10, seed=31, spread=0.5)}
    arch = packing.MLPArch(784, (256,), 10, "relu")
    opts = ("sgd", "adam", "momentum", "adagrad")
    hs = [packing.make_handle(f"x{i}", arch, opts[i % 4], 0.01 / (1 + i), 32, 50, "t", i)
          for i in range(8)]
    assert all(device.uses_m1x(arch, h.optimizer.kind, 32) for h in hs)
    packed = packing.dedup_inputs(packing.pack_models(hs))
    lockstep(packed, ds, 3, packing=packing)
    for i in (1, 6):
        solo = packing.make_handle(f"x{i}", arch, opts[i % 4], 0.01 / (1 + i), 32, 50, "t", i)
        for _ in range(3):
            packing.standalone_step(solo, ds)
        assert _maxdiff(hs[i], solo) == 0.0


def test_m1x_ragged_units_rows_and_classes_lockstep(plan):
    """Members whose hidden width is not a multiple of the 16-unit block
    (partial last block, idle cluster ranks), 64-row padding (batch 50),
    odd class counts and every activation, in one heterogeneous pack with two
    input datasets; oracle parity and packed == standalone."""
    plan(m1x=1)
    from paper_2002_02885_b200 import device
    ds = {"a": data.synth_dataset(700, 64, 7, seed=32, spread=0.5),
          "b": data.synth_dataset(500, 100, 3, seed=33, spread=0.5)}
    specs = [("r0", packing.MLPArch(64, (100,), 7, "sigmoid"), "adam", 0.01, 50, "a"),
             ("r1", packing.MLPArch(64, (40,), 7, "tanh"), "momentum", 0.05, 32, "a"),
             ("r2", packing.MLPArch(100, (212,), 3, "leaky_relu"), "adagrad", 0.02, 20, "b"),
             ("r3", packing.MLPArch(100, (4,), 3, "relu"), "sgd", 0.1, 64, "b")]
    hs = [packing.make_handle(m, a, o, lr, b, 30, d, i)
          for i, (m, a, o, lr, b, d) in enumerate(specs)]
    assert all(device.uses_m1x(h.arch, h.optimizer.kind, h.batch_size) for h in hs)
    packed = packing.dedup_inputs(packing.pack_models(hs))
    lockstep(packed, ds, 3, packing=packing)
    solo = packing.make_handle("r2", specs[2][1], "adagrad", 0.02, 20, 30, "b", 2)
    for _ in range(3):
        packing.standalone_step(solo, ds)
    assert _maxdiff(hs[2], solo) == 0.0


def test_m1x_and_tensor_path_agree(plan):
    """The same member trained by the one-launch FFMA step and by the tcgen05
    3xTF32 path: both within the stated fp32 tolerance of each other."""
    ds = {"t": data.synth_dataset(2000, 784, 10, seed=34, spread=0.5)}
    arch = packing.MLPArch(784, (128,), 10, "tanh")
    out = {}
    for path in ("m1x", "m1t"):
        plan(m1x=int(path == "m1x"))
        h = packing.make_handle("a", arch, "momentum", 0.02, 32, 50, "t", 3)
        for _ in range(4):
            loss = packing.standalone_step(h, ds)
        out[path] = (h, loss)
    (a, la), (b, lb) = out["m1x"], out["m1t"]
    for k in a.params:
        _assert_param_close(a.params[k], b.params[k], RTOL, ATOL, k, "momentum", 0.02)
    assert la == pytest.approx(lb, rel=1e-5)


# ------------------------------------------------- pipelined packed_run --

def _run_pair(ds, steps, depth):
    arch = packing.MLPArch(40, (24,), 5, "tanh")
    hs = [packing.make_handle("p0", arch, "adam", 0.01, 16, 23, "t", 1),
          packing.make_handle("p1", arch, "sgd", 0.05, 16, 40, "t", 2),
          packing.make_handle("p2", arch, "momentum", 0.02, 12, 31, "t", 3)]
    return hs, packing.dedup_inputs(packing.pack_models(hs))


def test_packed_run_equals_packed_step_loop():
    """packed_run (16 steps in flight, shadow cursors) reproduces the
    packed_step loop bit for bit across epoch rolls, ragged batches and members
    finishing at different steps."""
    ds = {"t": data.synth_dataset(100, 40, 5, seed=21)}
    ha, pa = _run_pair(ds, 0, 0)
    la = []
    while any(not h.finished for h in ha):
        la.append(packing.packed_step(pa, ds))
    hb, pb = _run_pair(ds, 0, 0)
    lb = packing.packed_run(pb, ds, 1 << 30, depth=16)
    assert la == lb
    for a, b in zip(ha, hb):
        assert _maxdiff(a, b) == 0.0
        assert (a.cursor.steps_done, a.cursor.epoch_index, a.cursor.pos) == \
            (b.cursor.steps_done, b.cursor.epoch_index, b.cursor.pos)
        np.testing.assert_array_equal(a.cursor.samples_used, b.cursor.samples_used)
        assert a.optimizer.step_counter == b.optimizer.step_counter
    assert pa.last_step_stats == pb.last_step_stats


@pytest.mark.parametrize("mode", ["resident", "stream"])
def test_native_run_matches_python_loop_two_datasets(mode):
    """pk_pack_run (the library's multi-step driver) against the Python
    sliding window and the packed_step loop: two datasets, four batch sizes
    (several input groups), many epoch rolls (the driver returns for the next
    epochs' permutations), members finishing at different steps; losses,
    params, cursors, samples_used and last_step_stats bit-identical."""
    ds = {"a": data.synth_dataset(70, 12, 4, seed=41), "b": data.synth_dataset(45, 8, 3, seed=42)}

    def make():
        spec = [("n0", 12, 4, "a", "adam", 16, 60), ("n1", 12, 4, "a", "sgd", 16, 45),
                ("n2", 12, 4, "a", "momentum", 9, 80), ("n3", 8, 3, "b", "adagrad", 7, 70),
                ("n4", 8, 3, "b", "sgd", 20, 33)]
        hs = [packing.make_handle(m, packing.MLPArch(d, (8,), c, "tanh"), o, 0.03, b, t, bind, i)
              for i, (m, d, c, bind, o, b, t) in enumerate(spec)]
        return hs, packing.dedup_inputs(packing.pack_models(hs))

    runtime.set_input_mode(mode)
    try:
        hl, pl = make()
        ll = []
        while any(not h.finished for h in hl):
            ll.append(packing.packed_step(pl, ds))
        hn, pn = make()
        ln = packing.packed_run(pn, ds, 1 << 30, depth=8)
        runtime.set_options(py_run=True)
        hp, pp = make()
        lp = packing.packed_run(pp, ds, 1 << 30, depth=8)
    finally:
        runtime.set_options(py_run=False)
        runtime.set_input_mode("resident")
    assert ll == ln == lp
    for a, b, c in zip(hl, hn, hp):
        assert _maxdiff(a, b) == 0.0 and _maxdiff(a, c) == 0.0
        for x in (b, c):
            assert (a.cursor.steps_done, a.cursor.epoch_index, a.cursor.pos) == \
                (x.cursor.steps_done, x.cursor.epoch_index, x.cursor.pos)
            np.testing.assert_array_equal(a.cursor.samples_used, x.cursor.samples_used)
            assert a.optimizer.step_counter == x.optimizer.step_counter
    assert pl.last_step_stats == pn.last_step_stats == pp.last_step_stats


def test_native_run_hands_label_errors_back():
    """A batch whose labels exceed a member's classes: the native driver stops
    before that step and the Python planner raises the reference's IndexError
    at exactly the same step."""
    d = data.synth_dataset(60, 6, 5, seed=43)
    ds = {"d": d}
    hs = [packing.make_handle("z0", packing.MLPArch(6, (4,), 3, "relu"), "sgd", 0.05, 10, 100, "d", 0)]
    packed = packing.pack_models(hs)
    with pytest.raises(IndexError):
        packing.packed_run(packed, ds, 100)
    ref = packing.make_handle("z0", packing.MLPArch(6, (4,), 3, "relu"), "sgd", 0.05, 10, 100, "d", 0)
    pr = packing.pack_models([ref])
    with pytest.raises(IndexError):
        for _ in range(100):
            packing.packed_step(pr, ds)
    assert hs[0].cursor.steps_done == ref.cursor.steps_done
    assert _maxdiff(hs[0], ref) == 0.0


def test_native_run_failure_inside_a_multi_step_graph():
    """A non-finite input row reached at the 4th step of a run: the native
    driver launches 8 steps per graph, the failing step's finalize sets the
    halt flag and steps 5..8 of the same graph skip; the exception, the step
    it happens at and every member's state equal the packed_step loop's."""
    from paper_2002_02885_b200.data import epoch_permutation

    def make():
        d = data.synth_dataset(200, 12, 4, seed=44)
        perm = epoch_permutation(d.dataset_id, d.n, 0)
        d.features[perm[3 * 10 + 2]] = np.inf  # a row of step 3's batch (b = 10)
        hs = [packing.make_handle(f"q{i}", packing.MLPArch(12, (8,), 4, "tanh"), o, 0.05, 10,
                                  100, "d", i) for i, o in enumerate(("sgd", "adam", "momentum"))]
        return {"d": d}, hs, packing.dedup_inputs(packing.pack_models(hs))

    out = []
    for mode in ("loop", "run"):
        ds, hs, pk = make()
        done = []
        with pytest.raises(engine.EngineError):
            if mode == "loop":
                for _ in range(20):
                    done.append(packing.packed_step(pk, ds))
            else:
                done = packing.packed_run(pk, ds, 20, depth=16)
        steps = [h.cursor.steps_done for h in hs]
        out.append((steps, [h._flat_params(h.params) for h in hs]))
    assert out[0][0] == out[1][0] == [3, 3, 3]
    for a, b in zip(out[0][1], out[1][1]):
        np.testing.assert_array_equal(a, b)


def test_native_run_without_inline_descriptors():
    """K = 36 > 32 members: step descriptors travel by H2D copy and the driver
    launches one step per graph; packed_run still equals the packed_step loop."""
    ds = {"t": data.synth_dataset(300, 12, 4, seed=45)}

    def make():
        hs = [packing.make_handle(f"w{i}", packing.MLPArch(12, (8,), 4, "relu"),
                                  ("sgd", "adam")[i % 2], 0.02, 16, 12, "t", i) for i in range(36)]
        return hs, packing.dedup_inputs(packing.pack_models(hs))

    ha, pa = make()
    la = [packing.packed_step(pa, ds) for _ in range(12)]
    hb, pb = make()
    lb = packing.packed_run(pb, ds, 12)
    assert la == lb
    for a, b in zip(ha, hb):
        assert _maxdiff(a, b) == 0.0
        assert a.cursor.pos == b.cursor.pos and a.cursor.steps_done == b.cursor.steps_done


def test_packed_run_stops_exactly_at_a_failing_step():
    """A non-finite gradient inside a pipelined run raises at that step; the
    device skipped every step enqueued behind it, so the state equals the
    packed_step loop's at the same exception (commit rules packing.py:246-253)."""
    ds = {"t": data.synth_dataset(100, 40, 5, seed=22)}
    results = []
    for mode in ("loop", "run"):
        hs, pk = _run_pair(ds, 0, 0)
        for _ in range(3):
            packing.packed_step(pk, ds)
        rt = runtime.runtime()
        hs[1]._device(rt).inject_fault(2)  # member p1's next step: NaN in dW0
        with pytest.raises(engine.NonFiniteGradient):
            if mode == "loop":
                for _ in range(10):
                    packing.packed_step(pk, ds)
            else:
                packing.packed_run(pk, ds, 10, depth=8)
        # the pack keeps training normally afterwards
        after = packing.packed_step(pk, ds)
        results.append((hs, after))
    (ha, la), (hb, lb) = results
    assert la == lb
    for a, b in zip(ha, hb):
        assert _maxdiff(a, b) == 0.0
        assert a.cursor.steps_done == b.cursor.steps_done
        assert a.optimizer.step_counter == b.optimizer.step_counter


# ------------------------------- which kernel a step launched (kind codes) --
# pk_pack_profile_step kind codes (packtrain_b200.h): 17 k_mlp1_fwd, 18 k_mlp1_bwd,
# 19 k_m1t_fwd, 20 k_m1t_bwd, 21 k_m1s_fwd, 22 k_m1c_fwd, 23 k_m1x_step
K_M1T_FWD, K_M1T_BWD, K_M1S_FWD, K_M1C_FWD = 19, 20, 21, 22


def _profiled_step(packed, datasets):
    """one real packed step run un-graphed through pk_pack_profile_step; returns
    the launched kernels' kind codes (the step commits like packed_step)"""
    active = packing._active_members(packed, datasets, False)
    plan_ = packing._plan_step(packed, active, datasets, None, None)
    code, phases, losses = plan_.dpack.profile()
    packing._apply_result(packed, active, plan_, code, -1, -1, losses)
    return [kind for kind, _, _, _ in phases]


def test_forced_streaming_forward_lockstep_and_kernel(plan):
    """plan fwd='stream': the tensor-path forward is k_m1s_fwd even for a small
    pack; it is checked launched, one-step parity with the f64 oracle for all
    four optimizers, and its trajectory equals the default plan's (k_m1c_fwd /
    split-K) bit for bit — the streaming forward reproduces the split order."""
    ds = {"t": data.synth_dataset(2000, 784, 10, seed=41, spread=0.5)}
    arch = packing.MLPArch(784, (256,), 10, "relu")
    opts = ("sgd", "adam", "momentum", "adagrad")

    def mk(prefix):
        return [packing.make_handle(f"{prefix}{i}", arch, opts[i], 0.01 / (1 + i), 32, 50, "t", i)
                for i in range(4)]
    plan(fwd="stream")
    hs = mk("s")
    packed = packing.dedup_inputs(packing.pack_models(hs))
    kinds = _profiled_step(packed, ds)
    assert K_M1S_FWD in kinds and K_M1T_BWD in kinds, kinds
    lockstep(packed, ds, 2, packing=packing)
    plan(fwd="auto")
    ref = mk("s")
    pr = packing.dedup_inputs(packing.pack_models(ref))
    kinds = _profiled_step(pr, ds)
    assert K_M1S_FWD not in kinds and (K_M1C_FWD in kinds or K_M1T_FWD in kinds), kinds
    for _ in range(2):
        packing.packed_step(pr, ds)
    for a, b in zip(hs, ref):
        assert _maxdiff(a, b) == 0.0


def test_k16_shape_default_plan_uses_cluster_forward():
    """BASELINE k16 mix (16 x 784-256-10, b = 32, four optimizers): the default
    plan's forward is the cluster-resident k_m1c_fwd (one wave); parity per step
    with the oracle."""
    ds = {"t": data.synth_dataset(2000, 784, 10, seed=42, spread=0.5)}
    arch = packing.MLPArch(784, (256,), 10, "relu")
    opts = ("sgd", "adam", "momentum", "adagrad")
    hs = [packing.make_handle(f"k{i}", arch, opts[i % 4], 10.0 ** -(1 + i % 4), 32, 50, "t", i)
          for i in range(16)]
    packed = packing.dedup_inputs(packing.pack_models(hs))
    kinds = _profiled_step(packed, ds)
    assert K_M1C_FWD in kinds and K_M1T_BWD in kinds, kinds
    lockstep(packed, ds, 1, packing=packing)


def test_wide16_shape_streaming_forward_lockstep():
    """The wide16 bench shape (16 x 784-1024-10, b = 128, four optimizers): no
    cluster size fits one wave, so the default plan streams (k_m1s_fwd); four
    32-row chunks per backward tile, H = 1024; one-step parity per member."""
    ds = {"t": data.synth_dataset(1000, 784, 10, seed=43, spread=0.5)}
    arch = packing.MLPArch(784, (1024,), 10, "relu")
    opts = ("sgd", "adam", "momentum", "adagrad")
    hs = [packing.make_handle(f"w{i}", arch, opts[i % 4], 10.0 ** -(1 + i % 4), 128, 20, "t", i)
          for i in range(16)]
    packed = packing.dedup_inputs(packing.pack_models(hs))
    kinds = _profiled_step(packed, ds)
    assert K_M1S_FWD in kinds and K_M1T_BWD in kinds, kinds
    lockstep(packed, ds, 1, packing=packing)


def test_f64_hyperband_shape_lockstep():
    """The f64 Hyperband member shape (784-16-10 on k_phase<double> with forward
    input ranges), 8 members with every optimizer: lockstep against the oracle
    at the f64 tolerance (rel 1e-10)."""
    runtime.set_precision("f64")
    try:
        ds = {"t": data.synth_dataset(600, 784, 10, seed=44)}
        arch = packing.MLPArch(784, (16,), 10, "relu")
        opts = ("sgd", "adam", "momentum", "adagrad")
        hs = [packing.make_handle(f"f{i}", arch, opts[i % 4], 0.01 * (1 + i % 3), 40, 30, "t", i)
              for i in range(8)]
        packed = packing.dedup_inputs(packing.pack_models(hs))
        odata = {k: oracle_dataset(v, round32=False) for k, v in ds.items()}
        for s in range(3):
            oms = [oracle_from_handle(h) for h in packed.members]
            want, _ = O.oracle_packed_step(oms, odata)
            got = packing.packed_step(packed, ds)
            for k in want:
                assert abs(got[k] - want[k]) <= 1e-10 * abs(want[k]) + 1e-12, (s, k)
            for h, m in zip(packed.members, oms):
                assert_close_member(h, m, rtol=1e-10, atol=1e-12, what=f"f64 step {s}")
    finally:
        runtime.set_precision("f32")
