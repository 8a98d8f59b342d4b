"""GPU parity of the conv pack path (BASELINE configs 1-3) through the
reference's pack API (packing.make_handle / pack_models / dedup_inputs /
packed_step / standalone_step) and the pk_cnn_* C-ABI behind it.

* every kernel teacher-forced against oracle/cnn64.py (tests/_cnn.py states the
  bf16 tolerances), for LeNet-5, MobileNetV2-w0.5 and ResNet-18 members with
  mixed optimizers, shared-input (concatenated-N) first layer included;
* the fused optimizer against engine.py:295-326 in fp32 on the device's grads;
* packed == standalone bit for bit (K-invariant kernels);
* the reference's step semantics: non-finite gradient stops the update loop at
  that member, misaligned batches form separate input groups, the last batch
  of an epoch is short, cursors and samples_used advance exactly.
"""
import numpy as np
import pytest

from _helpers import has_gpu

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

import torch  # noqa: E402

from oracle import cnn64 as O  # noqa: E402
from paper_2002_02885_b200 import cnn, data, engine, packing  # noqa: E402
import _cnn  # noqa: E402

OPTS = ("sgd", "momentum", "adam", "adagrad")


def _arch(fam, img=32):
    return cnn.ConvArch(fam, 10, (3, img, img), 0.5 if fam == "mobilenetv2" else 1.0)


def _ds(n=256, img=32, seed=1):
    return data.synth_dataset(n, 3 * img * img, 10, seed=seed, spread=0.5)


def _handles(arch, K, b, opts=OPTS, lr0=0.05, target=50, wd=0.0, prefix="m"):
    return [packing.make_handle(f"{prefix}{i}", arch, opts[i % len(opts)], lr0 / (i + 1), b,
                                target, "train", 0, weight_decay=wd) for i in range(K)]


def _batch(ds, arch, epoch, pos, take):
    perm = data.epoch_permutation(ds.dataset_id, ds.n, epoch)
    rows = perm[pos:pos + take]
    return O.batch_images(ds.features, arch.image, rows), torch.from_numpy(
        ds.labels[rows].astype(np.int64))


@pytest.mark.parametrize("fam,K,b", [("lenet5", 2, 32), ("mobilenetv2", 2, 32),
                                     ("resnet18", 2, 16), ("lenet5", 5, 20),
                                     ("densenet121", 2, 8)])
def test_teacher_forced_step(fam, K, b):
    arch = _arch(fam)
    ds = _ds()
    hs = _handles(arch, K, b, wd=1e-3)
    before = [{n.split("/", 1)[1]: v.copy() for n, v in h.params.items()} for h in hs]
    packed = packing.dedup_inputs(packing.pack_models(hs))
    losses = packing.packed_step(packed, {"train": ds})
    assert packed.last_step_stats == {"physical_inputs": 1, "groups": 1, "driver_batch": b}
    cp = packed._cp
    x, y = _batch(ds, arch, 0, 0, b)
    for k, h in enumerate(hs):
        _cnn.teacher_forced(cp, k, before[k], x, y, b, losses[h.model_id])
        _cnn.check_update(cp, k, h.optimizer.kind, h.optimizer.learning_rate, 1e-3, 0,
                          before[k], {})
        assert h.optimizer.step_counter == 1 and h.cursor.steps_done == 1 and h.cursor.pos == b


@pytest.mark.parametrize("fam,K,b,img", [("mobilenetv2", 2, 4, 56), ("resnet18", 2, 2, 40),
                                         ("lenet5", 2, 8, 28)])
def test_teacher_forced_odd_planes(fam, K, b, img):
    """Planes whose widths are odd or not a multiple of the depthwise strip (56²:
    28, 14, 7, 4, 2; 40²: 20, 10, 5, 3, 2), stride-2 layers on odd planes, and the
    dense first conv (IM2COL) off the 32² / 224² shapes: every kernel of one packed
    step teacher-forced against the oracle, packed == standalone bit for bit."""
    arch = _arch(fam, img)
    ds = _ds(n=64, img=img)
    hs = _handles(arch, K, b, wd=1e-3)
    before = [{n.split("/", 1)[1]: v.copy() for n, v in h.params.items()} for h in hs]
    packed = packing.dedup_inputs(packing.pack_models(hs))
    losses = packing.packed_step(packed, {"train": ds})
    x, y = _batch(ds, arch, 0, 0, b)
    for k, h in enumerate(hs):
        _cnn.teacher_forced(packed._cp, k, before[k], x, y, b, losses[h.model_id])
    solo = _handles(arch, K, b, wd=1e-3)
    for h in solo:
        assert packing.standalone_step(h, {"train": ds}) == losses[h.model_id]
    for a, s_ in zip(hs, solo):
        for n in a.params:
            assert np.array_equal(a.params[n], s_.params[n]), n


def test_end_to_end_loss_vs_oracle():
    """Whole-net forward from identical state: LeNet (no BN) matches the
    mirrored oracle to fp32 precision; BN nets within 1 % (bf16 chaos)."""
    ds = _ds()
    for fam, b, tol in (("lenet5", 32, 1e-4), ("resnet18", 16, 1e-2)):
        arch = _arch(fam)
        hs = _handles(arch, 2, b)
        init = [{n.split("/", 1)[1]: v.copy() for n, v in h.params.items()} for h in hs]
        losses = packing.packed_step(packing.dedup_inputs(packing.pack_models(hs)),
                                     {"train": ds})
        x, y = _batch(ds, arch, 0, 0, b)
        spec = _cnn.spec_of(arch)
        for k, h in enumerate(hs):
            ref, _, _ = O.forward_backward(spec, init[k], x, y)
            assert abs(losses[h.model_id] - ref) <= tol * ref, (fam, losses, ref)


@pytest.mark.parametrize("fam,b", [("lenet5", 32), ("mobilenetv2", 16), ("resnet18", 8)])
def test_packed_equals_standalone_bitwise(fam, b):
    arch = _arch(fam)
    ds = _ds()
    K = 3
    hs = _handles(arch, K, b)
    solo = _handles(arch, K, b)
    packed = packing.dedup_inputs(packing.pack_models(hs))
    for _ in range(3):
        lp = packing.packed_step(packed, {"train": ds})
        for h in solo:
            ls = packing.standalone_step(h, {"train": ds})
            assert ls == lp[h.model_id]
    for a, s in zip(hs, solo):
        pa, ps = a.params, s.params
        for n in pa:
            assert np.array_equal(pa[n], ps[n]), n
        assert a.optimizer.step_counter == s.optimizer.step_counter == 3


def test_nonfinite_stops_update_loop_at_member():
    """engine.py:297-299 + packing.py:250-253: members before the bad one are
    updated, the bad one and every later member are not; NonFiniteGradient."""
    arch = _arch("lenet5")
    ds = _ds()
    hs = _handles(arch, 3, 16, opts=("sgd",))
    packed = packing.pack_models(hs)
    packing.packed_step(packed, {"train": ds})
    before = [{n: v.copy() for n, v in h.params.items()} for h in hs]
    p = hs[1].params
    p["m1/L2/W"][0, 0, 0, 0] = np.nan
    before[1]["m1/L2/W"][0, 0, 0, 0] = np.nan
    with pytest.raises(engine.NonFiniteGradient):
        packing.packed_step(packed, {"train": ds})
    assert [h.optimizer.step_counter for h in hs] == [2, 1, 1]
    assert [h.cursor.steps_done for h in hs] == [2, 1, 1]
    for k in (1, 2):
        after = hs[k].params
        for n in after:
            np.testing.assert_array_equal(after[n], np.asarray(before[k][n], np.float32))
    assert not np.array_equal(hs[0].params["m0/L0/W"], before[0]["m0/L0/W"])


def test_misaligned_and_partial_batches_match_standalone():
    """Batches 20 / 32 on n = 84: separate input groups, short last batches
    (packing.py:167), each member's trajectory == its standalone one."""
    arch = _arch("lenet5")
    ds = _ds(n=84)
    hs = [packing.make_handle(f"m{i}", arch, o, 0.05, b, 30, "train", 0)
          for i, (o, b) in enumerate((("sgd", 20), ("adam", 32), ("momentum", 20)))]
    solo = [packing.make_handle(f"m{i}", arch, o, 0.05, b, 30, "train", 0)
            for i, (o, b) in enumerate((("sgd", 20), ("adam", 32), ("momentum", 20)))]
    packed = packing.dedup_inputs(packing.pack_models(hs))
    for step in range(7):
        lp = packing.packed_step(packed, {"train": ds})
        assert packed.last_step_stats["groups"] == 2
        assert packed.last_step_stats["physical_inputs"] == 2
        for h in solo:
            assert packing.standalone_step(h, {"train": ds}) == lp[h.model_id]
    for a, s in zip(hs, solo):
        assert (a.cursor.epoch_index, a.cursor.pos) == (s.cursor.epoch_index, s.cursor.pos)
        np.testing.assert_array_equal(a.cursor.samples_used, s.cursor.samples_used)
        for n in a.params:
            assert np.array_equal(a.params[n], s.params[n]), n
    # b=32 over n=84: 32, 32, 20 | 32, 32, 20 | 32 → epoch 2, pos 32
    assert (hs[1].cursor.epoch_index, hs[1].cursor.pos) == (2, 32)


def test_training_reduces_loss():
    arch = _arch("lenet5")
    ds = data.synth_dataset(512, 3 * 32 * 32, 10, seed=3, spread=1.0)
    hs = _handles(arch, 4, 32, opts=("sgd", "momentum", "adam", "adagrad"), lr0=0.02)
    packed = packing.dedup_inputs(packing.pack_models(hs))
    first = packing.packed_step(packed, {"train": ds})
    for _ in range(40):
        last = packing.packed_step(packed, {"train": ds})
    for h in hs:
        assert last[h.model_id] < first[h.model_id], (first, last)


def _hetero(prefix="h", b=8):
    """BASELINE configs[3] shape at 32x32: MobileNetV2 + ResNet-18 + DenseNet-121
    on one input stream (ragged grouped launches; ResNet and DenseNet share the
    concatenated-N 7x7 stem)."""
    out = []
    for i, (fam, w, opt) in enumerate((("mobilenetv2", 1.0, "sgd"), ("resnet18", 1.0, "adam"),
                                       ("densenet121", 1.0, "momentum"))):
        arch = cnn.ConvArch(fam, 10, (3, 32, 32), w)
        out.append(packing.make_handle(f"{prefix}{i}", arch, opt, 0.01, b, 20, "train", 0,
                                       weight_decay=1e-4))
    return out


def test_heterogeneous_pack_teacher_forced_and_standalone():
    ds = _ds()
    hs = _hetero()
    before = [{n.split("/", 1)[1]: v.copy() for n, v in h.params.items()} for h in hs]
    packed = packing.dedup_inputs(packing.pack_models(hs))
    losses = packing.packed_step(packed, {"train": ds})
    assert packed.last_step_stats == {"physical_inputs": 1, "groups": 1, "driver_batch": 8}
    x, y = _batch(ds, hs[0].arch, 0, 0, 8)
    for k, h in enumerate(hs):
        _cnn.teacher_forced(packed._cp, k, before[k], x, y, 8, losses[h.model_id])
    solo = _hetero()
    for h in solo:
        assert packing.standalone_step(h, {"train": ds}) == losses[h.model_id]
    for _ in range(2):
        lp = packing.packed_step(packed, {"train": ds})
        for h in solo:
            assert packing.standalone_step(h, {"train": ds}) == lp[h.model_id]
    for a, s_ in zip(hs, solo):
        pa, ps = a.params, s_.params
        for n in pa:
            assert np.array_equal(pa[n], ps[n]), n


def test_conv_hyperband_packed_matches_unpacked():
    """BASELINE configs[4] at toy scale: pack-aware Hyperband (tuner.py:285-337)
    over LeNet-5 members with the conv executor.  Every config trains the same
    trajectory packed (knn groups) or alone (original) — the kernels are
    K-invariant — so records (config, rung epochs, loss) and the selected
    config are identical across strategies."""
    from paper_2002_02885_b200 import tuner
    ds = data.synth_dataset(400, 3 * 32 * 32, 10, seed=5, spread=1.0)
    res = {}
    for strat in ("original", "knn"):
        ex = tuner.B200ConvExecutor(ds, family="lenet5", width=1.0, seed=0)
        res[strat] = tuner.packed_hyperband(9, 3, ex, seed=1, strategy=strat)
    key = lambda r: sorted((x.config_id, x.epochs, x.loss) for x in r.records)  # noqa: E731
    assert key(res["original"]) == key(res["knn"])
    assert res["original"].best_config.config_id == res["knn"].best_config.config_id
    assert all(np.isfinite(x.loss) for x in res["knn"].records)
    sizes = {}
    for x in res["knn"].records:
        sizes[(x.bracket, x.rung, x.group)] = sizes.get((x.bracket, x.rung, x.group), 0) + 1
    assert max(sizes.values()) >= 2  # knn really packed members


def test_conv_hyperband_concurrent_packs_match_serial():
    """The pool's concurrent packs (executor.concurrent_groups > 1: a round's
    groups train at once, one host thread and CUDA stream per pack) give the
    serial run's records, selection and member trajectories."""
    from paper_2002_02885_b200 import hyperband_pool, tuner
    ds = data.synth_dataset(300, 3 * 32 * 32, 10, seed=7, spread=1.0)
    res = {}
    for conc in (1, 4):
        ex = tuner.B200ConvExecutor(ds, family="lenet5", width=1.0, seed=0)
        ex.concurrent_groups = conc
        res[conc] = hyperband_pool.overlapped_hyperband(9, 3, ex, seed=2, strategy="knn")[0]
    key = lambda r: [(x.bracket, x.rung, x.group, x.config_id, x.epochs, x.loss)  # noqa: E731
                     for x in r.records]
    assert key(res[1]) == key(res[4])
    assert res[1].best_config.config_id == res[4].best_config.config_id
    assert len(res[4].records) > 8


def test_pipelined_run_matches_step_loop():
    """convpack.conv_packed_run (host planning overlapped with the device, verdicts
    through a pinned ring) == the same number of packed_step calls, bit for bit:
    losses per step, parameters, cursors and samples_used."""
    from paper_2002_02885_b200 import convpack
    arch = _arch("lenet5")
    ds = _ds(n=200)
    a = _handles(arch, 3, 32, target=9)
    b = _handles(arch, 3, 32, target=9)
    pa = packing.dedup_inputs(packing.pack_models(a))
    la = [packing.packed_step(pa, {"train": ds}) for _ in range(9)]
    pb = packing.dedup_inputs(packing.pack_models(b))
    lb = convpack.conv_packed_run(pb, {"train": ds}, 50, depth=3)
    assert lb == la and all(h.finished for h in b)
    for x, y in zip(a, b):
        for n in x.params:
            assert np.array_equal(x.params[n], y.params[n]), n
        assert x.cursor.steps_done == y.cursor.steps_done and x.cursor.pos == y.cursor.pos
        assert np.array_equal(x.cursor.samples_used, y.cursor.samples_used)
        assert x.optimizer.step_counter == y.optimizer.step_counter
