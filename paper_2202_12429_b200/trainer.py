"""Stub trainer math on the GPU (reference trainer.py:1-179).

The reference's "dense model" is a deterministic gradient stub
g = c_value*v + c_label*(label - 0.5), accumulated per key in occurrence
order (np.add.at), combined across trainers in ascending rank order and
applied by single-precision SGD.  All three cores run in
``csrc/trainer.cu``; the engine uses the fused ``bp_stub_step`` (one kernel
for gradient + combine + SGD + dirty marking), the functions below expose
the same cores with the reference's numpy signatures.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .device import DevicePrep
from .errors import CacheMissError, ConfigurationError

BP_STUB_SGD = 0
BP_STUB_GRAD = 1


@dataclass(frozen=True)
class StubModelConfig:
    """g = c_value*v + c_label*(label - 0.5), per embedding component."""

    lr: float = 0.01
    c_value: float = 0.01
    c_label: float = 0.001

    def __post_init__(self):
        if not self.lr > 0:
            raise ConfigurationError("lr must be > 0")


def f32(x: float) -> float:
    """The float32 rounding numpy applies to np.float32(x)."""
    return float(np.float32(x))


def _index_prep(idx: np.ndarray, labels: np.ndarray) -> DevicePrep:
    """Registry-mode prep whose keys are the indices (table 0): the CSR of
    occurrences per index in input order."""
    keys = np.ascontiguousarray(idx, dtype=np.int64).astype(np.uint64)
    n = len(keys)
    return DevicePrep(keys, labels, np.asarray([0, n], dtype=np.int64), 0, schema=None)


def gradient_core(occ_unique_idx, occ_labels, unique_values, cfg: StubModelConfig) -> np.ndarray:
    """Per-unique-key gradients; per-key sums in occurrence order, float32."""
    values = np.ascontiguousarray(unique_values, dtype=np.float32)
    u, dim = values.shape
    out = np.zeros_like(values)
    idx = np.asarray(occ_unique_idx, dtype=np.int64)
    if len(idx) == 0 or u == 0:
        return out
    labels = np.asarray(occ_labels, dtype=np.float32)
    if not np.array_equal(labels, np.round(labels)) or labels.min() < 0 or labels.max() > 255:
        raise ConfigurationError("labels must be small non-negative integers")
    prep = _index_prep(idx, labels.astype(np.uint8))
    nu = prep.num_unique
    d_rows = L.to_device(values)
    row_index = torch.empty(nu, dtype=torch.int32, device="cuda")
    L.check(L.lib().bp_prep_key_rows(prep.handle, L.ptr(row_index), L.stream_ptr()), "bp_prep_key_rows")
    grad = torch.empty((nu, dim), dtype=torch.float32, device="cuda")
    L.check(L.lib().bp_stub_step(L.Context.get().handle, prep.handle, L.ptr(d_rows), L.ptr(row_index), None, dim,
                                 f32(cfg.c_value), f32(cfg.c_label), f32(cfg.lr), BP_STUB_GRAD, L.ptr(grad),
                                 None, 0, None, L.stream_ptr()), "bp_stub_step")
    rows = row_index.cpu().numpy()
    out[rows] = grad.cpu().numpy()
    return out


def combine_core(rank_batch_idx, rank_grads, num_unique: int, emb_dim: int) -> np.ndarray:
    """Sum per-rank gradient blocks into batch-unique rows in ascending rank order."""
    out = np.zeros((num_unique, emb_dim), dtype=np.float32)
    nonempty = [i for i in range(len(rank_grads)) if len(rank_grads[i])]
    if not nonempty:
        return out
    idx = np.concatenate([np.asarray(rank_batch_idx[i], dtype=np.int64) for i in nonempty])
    grads = np.ascontiguousarray(np.concatenate([rank_grads[i] for i in nonempty]), dtype=np.float32)
    prep = _index_prep(idx, np.zeros(len(idx), dtype=np.uint8))
    d_out = L.to_device(out)
    d_grads = L.to_device(grads)  # keep alive until the kernel is enqueued after every upload
    L.check(L.lib().bp_add_at_rows(prep.handle, L.ptr(d_grads), emb_dim, L.ptr(d_out), L.stream_ptr()),
            "bp_add_at_rows")
    return d_out.cpu().numpy()


def sgd_step(values, grads, lr: float) -> np.ndarray:
    """v - lr*g in single precision (two roundings, no FMA)."""
    v = np.ascontiguousarray(values, dtype=np.float32)
    g = np.ascontiguousarray(grads, dtype=np.float32)
    if v.size == 0:
        return v.copy()
    d_out = torch.empty(v.shape, dtype=torch.float32, device="cuda")
    d_v, d_g = L.to_device(v), L.to_device(g)
    L.check(L.lib().bp_sgd(L.ptr(d_v), L.ptr(d_g), f32(lr), v.size, L.ptr(d_out), L.stream_ptr()), "bp_sgd")
    return d_out.cpu().numpy()


def local_gradients(sub_batch, values, cfg: StubModelConfig) -> dict:
    """Gradients of one trainer's sub-batch keyed by its unique keys (first-occurrence order)."""
    unique: dict = {}
    occ_idx: list = []
    occ_labels: list = []
    for ex in sub_batch:
        for key in ex.sparse:
            pos = unique.setdefault(key, len(unique))
            occ_idx.append(pos)
            occ_labels.append(ex.label)
    if not unique:
        return {}
    try:
        mat = np.stack([np.asarray(values[k], dtype=np.float32) for k in unique])
    except KeyError as exc:
        raise CacheMissError(exc.args[0]) from None
    grads = gradient_core(np.asarray(occ_idx), np.asarray(occ_labels, dtype=np.float32), mat, cfg)
    return {key: grads[i] for key, i in unique.items()}


def combine_gradients(per_trainer) -> dict:
    """Sum gradient maps across trainers in ascending rank order (union of keys)."""
    union: dict = {}
    for g in per_trainer:
        for key in g:
            union.setdefault(key, len(union))
    if not union:
        return {}
    dim = None
    rank_idx, rank_mats = [], []
    for g in per_trainer:
        keys = list(g)
        if keys:
            dim = len(next(iter(g.values())))
        rank_idx.append(np.asarray([union[k] for k in keys], dtype=np.int64))
        rank_mats.append(np.stack([np.asarray(g[k], dtype=np.float32) for k in keys]) if keys
                         else np.zeros((0, 0), dtype=np.float32))
    out = combine_core(rank_idx, rank_mats, len(union), dim)
    return {key: out[i] for key, i in union.items()}


def apply_updates(cache, combined, cfg: StubModelConfig) -> set:
    """Apply combined gradients to a cache; zero-gradient rows stay clean."""
    keys = list(combined)
    if not keys:
        return set()
    slots = cache.resolve_slots(keys)
    grads = np.stack([np.asarray(combined[k], dtype=np.float32) for k in keys])
    new_values = sgd_step(cache.values_at(slots), grads, cfg.lr)
    cache.update_rows(slots, new_values, np.any(grads != 0, axis=1))
    return set(keys)


def split_sync_sets(updated: set, next_batch_keys: set) -> tuple:
    """(critical, background): updated keys needed / not needed by the next batch, each sorted."""
    return sorted(updated & next_batch_keys), sorted(updated - next_batch_keys)
