"""Datasets, epoch orders and the preprocessing stage — host side.

Mirrors the reference's `packtrain.data` interface (data.py:14-194) for the
pieces the pack path consumes.  Seeding is bit-compatible with the
reference (sha256-derived PCG64 streams), so epoch orders, synthetic data and
jitter noise are identical numbers; the device keeps resident copies of the
features and of each epoch order (runtime.Runtime.dataset / .order) and
gathers batch rows itself.  The PTDS/CSV file formats are out of scope
(SURVEY §2.1).
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np


class DataError(Exception):
    pass


def _hashed_generator(text: str) -> np.random.Generator:
    # first 8 digest bytes, little endian (data.py:126-127, :158-159)
    return np.random.default_rng(
        int.from_bytes(hashlib.sha256(text.encode()).digest()[:8], "little"))


@dataclass(frozen=True)
class Dataset:
    """N x D float64 features with int64 labels (data.py:18-39)."""
    dataset_id: str
    features: np.ndarray
    labels: np.ndarray
    class_count: int

    def __post_init__(self):
        f = self.features
        if f.ndim != 2 or f.shape[0] < 1:
            raise DataError("features must be a non-empty N x D matrix")
        if len(self.labels) != f.shape[0]:
            raise DataError("label count does not match feature rows")
        lo, hi = int(np.min(self.labels)), int(np.max(self.labels))
        if lo < 0 or hi >= self.class_count:
            raise DataError("label out of range for class_count")

    @property
    def n(self) -> int:
        return self.features.shape[0]

    @property
    def dim(self) -> int:
        return self.features.shape[1]


def synth_dataset(n, d, classes, seed, spread=4.0) -> Dataset:
    """Gaussian class blobs (data.py:42-54); same draws in the same order."""
    if min(n, d, classes) < 1:
        raise DataError("n, d and classes must all be >= 1")
    g = np.random.default_rng(seed)
    centers = g.normal(scale=spread, size=(classes, d))
    y = g.integers(0, classes, size=n)
    x = centers[y] + g.normal(size=(n, d))
    return Dataset(f"synth-{n}x{d}c{classes}s{seed}", x, y.astype(np.int64), classes)


def epoch_permutation(dataset_id: str, n: int, epoch: int) -> np.ndarray:
    """Sample order of one epoch (data.py:124-128)."""
    return _hashed_generator(f"{dataset_id}|epoch{epoch}").permutation(n)


def batch_at(ds: Dataset, perm: np.ndarray, cursor: int, b: int):
    """Rows perm[cursor:cursor+b] (data.py:131-136)."""
    if cursor + b > ds.n:
        raise DataError(f"batch [{cursor}, {cursor + b}) exceeds dataset size {ds.n}")
    idx = perm[cursor:cursor + b]
    return ds.features[idx], ds.labels[idx], idx


@dataclass(frozen=True)
class PreprocessSpec:
    """Ordered pure stages ("normalize", mean, std) / ("jitter", seed)
    (data.py:139-147)."""
    stages: tuple = ()

    def digest(self) -> str:
        text = ";".join(",".join(str(p) for p in st) for st in self.stages)
        return hashlib.sha256(text.encode()).hexdigest()[:16]


@dataclass
class PreprocessCache:
    entries: dict = field(default_factory=dict)
    hits: int = 0
    misses: int = 0


def _stage_row(spec: PreprocessSpec, row: np.ndarray, index: int) -> np.ndarray:
    out = row
    for st in spec.stages:
        kind = st[0]
        if kind == "normalize":
            out = (out - st[1]) / st[2]
        elif kind == "jitter":
            noise = _hashed_generator(f"jitter|{st[1]}|{index}").normal(
                scale=0.01, size=out.shape)
            out = out + noise
        else:
            raise DataError(f"unknown preprocess stage {kind!r}")
    return out


def preprocess_all(spec: PreprocessSpec, features: np.ndarray) -> np.ndarray:
    """Every sample through the stage list (row i keyed by dataset index i) —
    the whole-dataset form of the per-sample memo, values identical to
    `preprocess` row by row (pure per-index stages, data.py:156-173)."""
    x = np.asarray(features, dtype=np.float64)
    return np.stack([_stage_row(spec, x[i], i) for i in range(x.shape[0])]) if len(x) else x


def account_cache(spec: PreprocessSpec, table: np.ndarray, indices, dataset_id: str,
                  cache: PreprocessCache):
    """The cache bookkeeping `preprocess` does for a batch (hits, misses,
    entries keyed (dataset, spec digest, index)), with values taken from an
    already materialized `table` (data.py:183-193)."""
    dig = spec.digest()
    for i in np.asarray(indices):
        key = (dataset_id, dig, int(i))
        if key in cache.entries:
            cache.hits += 1
        else:
            cache.misses += 1
            cache.entries[key] = table[int(i)].copy()


def preprocess(spec: PreprocessSpec, batch: np.ndarray, indices, dataset_id: str,
               cache: PreprocessCache | None = None) -> np.ndarray:
    """Per-sample stages memoized on (dataset, spec digest, index)
    (data.py:176-194)."""
    if not spec.stages:
        return batch
    dig = spec.digest()
    out = np.empty_like(batch)
    for r, i in enumerate(np.asarray(indices)):
        key = (dataset_id, dig, int(i))
        if cache is not None and key in cache.entries:
            cache.hits += 1
            out[r] = cache.entries[key]
            continue
        v = _stage_row(spec, batch[r], int(i))
        if cache is not None:
            cache.misses += 1
            cache.entries[key] = v
        out[r] = v
    return out
