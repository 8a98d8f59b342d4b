"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_golden.py

It imports `packtrain` from /root/reference/pkg/src, drives its public
pack API (make_handle / pack_models / dedup_inputs / packed_step /
standalone_step, engine.forward/backward/apply_update, EngineExecutor +
packed_hyperband) on seeded synthetic data and writes small .npz fixtures
next to this script.  The fixtures pin `oracle/` (tests/test_oracle.py)
and, through the oracle, the CUDA path.  Nothing at test or bench time
reads /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    from packtrain import data, engine, packing, tuner  # noqa: F401
    return data, engine, packing, tuner


def _flat(h):
    """Flatten params in layer order W0,b0,W1,b1,... (the C-ABI order)."""
    n = len(h.arch.hidden) + 1
    return np.concatenate([np.concatenate(
        [h.params[f"{h.model_id}/L{i}/W"].ravel(),
         h.params[f"{h.model_id}/L{i}/b"].ravel()]) for i in range(n)])


def _flat_slots(h):
    n = len(h.arch.hidden) + 1
    names = {"sgd": [], "momentum": ["velocity"], "adagrad": ["accum"],
             "adam": ["m", "v"]}[h.optimizer.kind]
    out = []
    for s in names:
        for i in range(n):
            for p in ("W", "b"):
                out.append(h.optimizer.slots[f"{h.model_id}/L{i}/{p}"][s].ravel())
    return np.concatenate(out) if out else np.zeros(0)


def config0(data, packing):
    """BASELINE configs[0]: K=2 MLP 784-256-10, SGD lr 0.1 / 0.01, b=32."""
    ds = data.synth_dataset(10000, 784, 10, seed=0)
    datasets = {"train": ds}
    arch = packing.MLPArch(784, (256,), 10, "relu")
    m0 = packing.make_handle("m0", arch, "sgd", 0.1, 32, 100, "train", 0)
    m1 = packing.make_handle("m1", arch, "sgd", 0.01, 32, 100, "train", 0)
    init0 = _flat(m0).copy()
    packed = packing.dedup_inputs(packing.pack_models([m0, m1]))
    losses = []
    p1 = None
    for step in range(3):
        out = packed_step_losses(packing, packed, datasets)
        losses.append([out["m0"], out["m1"]])
        if step == 0:
            p1 = (_flat(m0).copy(), _flat(m1).copy())
    perm = data.epoch_permutation(ds.dataset_id, ds.n, 0)
    np.savez_compressed(
        os.path.join(HERE, "config0.npz"),
        losses=np.array(losses),
        perm_head=perm[:64],
        init_m0_head=init0[:4096],
        init_m0_sum=np.array([init0.sum(), (init0 ** 2).sum()]),
        step1_m0_sum=np.array([p1[0].sum(), (p1[0] ** 2).sum()]),
        step1_m1_sum=np.array([p1[1].sum(), (p1[1] ** 2).sum()]),
        step1_m0_head=p1[0][:4096],
        step1_m1_b0=p1[1][784 * 256:784 * 256 + 256],
        feat_stats=np.array([ds.features.std(), np.abs(ds.features).max(),
                             ds.features[0, :8].sum()]),
        stats=np.array([packed.last_step_stats[k] for k in
                        ("physical_inputs", "groups", "driver_batch")]),
        dataset_id=np.array(ds.dataset_id),
    )


def packed_step_losses(packing, packed, datasets, **kw):
    return packing.packed_step(packed, datasets, **kw)


def small_pairs(data, packing, engine):
    """Pairs of 6-8-3 MLPs for every optimizer x activation: per-step losses
    and full flat params/slots after steps 1 and 5 (packed, dedup)."""
    ds = data.synth_dataset(120, 6, 3, seed=0)
    datasets = {"d": ds}
    out = {}
    for opt in engine.OPTIMIZERS:
        for act in engine.ACTIVATIONS:
            arch = packing.MLPArch(6, (8,), 3, act)
            a = packing.make_handle("a", arch, opt, 0.05, 10, 20, "d", 1)
            b = packing.make_handle("b", arch, opt, 0.01, 10, 20, "d", 2)
            packed = packing.dedup_inputs(packing.pack_models([a, b]))
            ls = []
            for s in range(5):
                r = packing.packed_step(packed, datasets)
                ls.append([r["a"], r["b"]])
                if s == 0:
                    out[f"{opt}_{act}_a_p1"] = _flat(a).copy()
                    out[f"{opt}_{act}_b_p1"] = _flat(b).copy()
            out[f"{opt}_{act}_losses"] = np.array(ls)
            out[f"{opt}_{act}_a_p5"] = _flat(a).copy()
            out[f"{opt}_{act}_b_p5"] = _flat(b).copy()
            out[f"{opt}_{act}_a_s5"] = _flat_slots(a).copy()
            out[f"{opt}_{act}_b_s5"] = _flat_slots(b).copy()
    np.savez_compressed(os.path.join(HERE, "small_pairs.npz"), **out)


def deep_and_misaligned(data, packing, engine):
    """Acceptance C2 shape (5-(8,8)-3, 50 packed steps, all optimizers) and
    the misaligned 20/50/100 scenario (tests/test_pack.py:113-138)."""
    out = {}
    ds = data.synth_dataset(400, 5, 3, seed=8)
    arch = packing.MLPArch(5, (8, 8), 3)
    for opt in engine.OPTIMIZERS:
        hs = [packing.make_handle(f"m{i}", arch, opt, 0.01, 16, 50, "d", i)
              for i in (1, 2)]
        packed = packing.dedup_inputs(packing.pack_models(hs))
        ls = []
        for _ in range(50):
            r = packing.packed_step(packed, {"d": ds})
            ls.append([r["m1"], r["m2"]])
        out[f"c2_{opt}_losses"] = np.array(ls)
        out[f"c2_{opt}_m1"] = _flat(hs[0])
        out[f"c2_{opt}_m2"] = _flat(hs[1])
    n = 1000
    ds = data.synth_dataset(n, 6, 3, seed=4)
    arch = packing.MLPArch(6, (8,), 3)
    specs = [("m20", 20, 50), ("m50", 50, 20), ("m100", 100, 10)]
    hs = [packing.make_handle(mid, arch, "sgd", 0.05, b, s, "d", i)
          for i, (mid, b, s) in enumerate(specs)]
    packed = packing.pack_models(hs)
    trace = []
    stats = []
    while any(not h.finished for h in hs):
        r = packing.packed_step(packed, {"d": ds})
        trace.append([r.get(mid, np.nan) for mid, _, _ in specs])
        stats.append([packed.last_step_stats[k] for k in
                      ("physical_inputs", "groups", "driver_batch")])
    out["mis_losses"] = np.array(trace)
    out["mis_stats"] = np.array(stats)
    for h in hs:
        out[f"mis_{h.model_id}"] = _flat(h)
    np.savez_compressed(os.path.join(HERE, "deep_misaligned.npz"), **out)


def known_answers(engine):
    """The engine known-answer tests (tests/test_engine.py:56-179) evaluated
    by the reference itself."""
    out = {}
    g = engine.build_mlp("m", 2, (), 2)
    params = {"m/L0/W": np.array([[1.0, -1.0], [0.5, 0.5]]),
              "m/L0/b": np.array([0.0, 1.0])}
    st = engine.forward(g, params, {"m/x": np.array([[1.0, 2.0]]),
                                    "m/y": np.array([0])})
    out["linear_softmax_loss"] = st.losses["m"]
    seq = {}
    for kind, lr, gs, w0 in [("sgd", 0.1, [[0.5, -1.0]], [1.0, 2.0]),
                             ("momentum", 0.1, [[1.0], [1.0]], [0.0]),
                             ("adagrad", 0.5, [[2.0]], [1.0]),
                             ("adam", 0.01, [[1.0], [2.0]], [0.0])]:
        p = {"w": np.array(w0, dtype=float)}
        opt = engine.make_optimizer(kind, lr)
        for gv in gs:
            engine.apply_update(opt, p, {"w": np.array(gv, dtype=float)})
        seq[kind] = p["w"].tolist()
    out["optimizer_seq"] = seq
    with open(os.path.join(HERE, "known_answers.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def micro_tuning(data, tuner):
    """Acceptance C10 (tests/test_acceptance.py:330-356): engine-backed
    Hyperband R=4 eta=2 under original and knn; the audit records."""
    dataset = data.synth_dataset(120, 5, 3, seed=30)
    space = tuner.ConfigSpace(batch_sizes=(10, 20, 30),
                              optimizers=("sgd", "adam"),
                              learning_rates=(1e-3, 1e-2),
                              activations=("relu", "tanh"))
    out = {}
    for strategy in ("original", "knn"):
        ex = tuner.EngineExecutor(dataset, hidden=(6,), seed=0)
        res = tuner.packed_hyperband(4, 2, ex, seed=0, strategy=strategy,
                                     space=space)
        out[strategy] = {
            "records": [[r.bracket, r.rung, r.group, r.config_id, r.epochs,
                         r.loss] for r in res.records],
            "best": res.best_config.config_id,
            "best_loss": res.best_loss,
            "total_epochs": res.total_epochs,
        }
    # schedule + stub-executor selection (tests/test_acceptance.py:247-265)
    res = tuner.hyperband(81, 3, tuner.StubExecutor(lambda c, e: c.config_id),
                          seed=1)
    out["stub_chain"] = [[r.bracket, r.rung, r.group, r.config_id, r.epochs]
                         for r in res.records]
    winners = {}
    for seed in range(5):
        for strategy in ("original", "batchsize", "random", "knn"):
            ex = tuner.StubExecutor(lambda c, e, s=seed: float(
                tuner._rng("accept7", s, c.config_id).uniform()))
            r = tuner.packed_hyperband(81, 3, ex, seed=seed, strategy=strategy)
            winners[f"{seed}_{strategy}"] = [
                r.best_config.config_id, r.total_epochs,
                [[x.bracket, x.rung, x.group, x.config_id] for x in r.records]]
    out["stub_winners"] = winners
    with open(os.path.join(HERE, "tuning.json"), "w") as fh:
        json.dump(out, fh, sort_keys=True)


def checkpoints(data, packing):
    """PKCK bytes of a fresh handle and of one after 7 Adam steps
    (tests/test_pack.py:197-215 scenario)."""
    ds = data.synth_dataset(120, 6, 3, seed=0)
    arch = packing.MLPArch(6, (8,), 3)
    fresh = packing.make_handle("m", arch, "adam", 0.001, 10, 30, "d", 0)
    h = packing.make_handle("m", arch, "adam", 0.001, 10, 30, "d", 0)
    for _ in range(7):
        packing.standalone_step(h, {"d": ds})
    with open(os.path.join(HERE, "ckpt_fresh.pkck"), "wb") as fh:
        fh.write(packing.checkpoint_model(fresh).to_bytes())
    with open(os.path.join(HERE, "ckpt_adam7.pkck"), "wb") as fh:
        fh.write(packing.checkpoint_model(h).to_bytes())


def main():
    data, engine, packing, tuner = _ref()
    checkpoints(data, packing)
    known_answers(engine)
    config0(data, packing)
    small_pairs(data, packing, engine)
    deep_and_misaligned(data, packing, engine)
    micro_tuning(data, tuner)
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
