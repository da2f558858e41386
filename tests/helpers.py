"""Shared builders for the lookup-path tests (small synthetic tasks)."""
from __future__ import annotations

import numpy as np

from paper_2210_02023_b200.api import PlacementTask, TableDesc, table_memory_gb


def make_tables(dims, rows, pfs, hot=None):
    tables = []
    for i, (d, r, pf) in enumerate(zip(dims, rows, pfs)):
        dist = [0.0] * 17
        h = 0.0 if hot is None else hot[i]
        dist[12] = h
        dist[0] = 0.5 * (1 - h)
        dist[1] = 0.3 * (1 - h)
        dist[2] = 0.2 * (1 - h)
        tables.append(TableDesc(i, int(d), int(r), float(pf), table_memory_gb(r, d, 4), dist))
    return tables


def as_dicts(tables):
    return [t.to_dict() for t in tables]


def random_task(seed, dims, D, B, rows_range=(1, 3000), pf_range=(0.0, 12.0), hot_p=0.5):
    rng = np.random.default_rng(seed)
    T = len(dims)
    rows = rng.integers(rows_range[0], rows_range[1], size=T)
    pfs = rng.uniform(pf_range[0], pf_range[1], size=T)
    hot = rng.uniform(0, 1, size=T) * (rng.uniform(0, 1, size=T) < hot_p)
    tables = make_tables(dims, rows, pfs, hot)
    placement = rng.integers(0, D, size=T).astype(np.int32)
    return PlacementTask(tables, D, 0.0, B), placement


def random_weights(seed, tables):
    rng = np.random.default_rng(seed)
    return [rng.uniform(0.5, 1.0, size=(t.hash_size, t.dim)).astype(np.float32)
            for t in tables]


def grad_cols(seed, B, cols):
    """The SURVEY 8d gradient generator (synth.cuh grad_value), vectorised:
    columns `cols` (global pooled columns) of dL/dpooled for every bag."""
    def mix64(x):
        x = x + np.uint64(0x9e3779b97f4a7c15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
        return x ^ (x >> np.uint64(31))
    tag = np.uint64(0x6772616469656e74)
    with np.errstate(over="ignore"):
        s = mix64(np.array([np.uint64(seed) ^ tag], dtype=np.uint64))
        hb = mix64(s ^ np.arange(B, dtype=np.uint64))[:, None]
        h = mix64(hb ^ np.asarray(cols, dtype=np.uint64)[None, :])
    return (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)


def table_cols(dims, t):
    """Global pooled columns of table t."""
    g = int(sum(dims[:t]))
    return np.arange(g, g + dims[t])


def sub_batch(off, idx, B, picks):
    """The CSR of tables `picks` alone (segments rebased), for the oracle."""
    sub_off = [np.zeros(1, dtype=np.int64)]
    sub_idx = []
    base = 0
    for t in picks:
        seg = off[t * B:(t + 1) * B + 1]
        sub_off.append(seg[1:] - seg[0] + base)
        sub_idx.append(idx[seg[0]:seg[-1]])
        base += int(seg[-1] - seg[0])
    return np.concatenate(sub_off), np.concatenate(sub_idx)


def sgd_rows_expected(off, idx, B, t, rows_sel, before_rows, grad_t, lr):
    """Row-wise SGD of a few rows of table t, restated in numpy: every
    occurrence of the row adds dL/dpooled of its bag (fp64), then
    W[row] -= lr * sum. grad_t = [B, dim_t] gradient columns of table t."""
    seg = off[t * B:(t + 1) * B + 1]
    ids = idx[seg[0]:seg[-1]]
    bag = np.repeat(np.arange(B), np.diff(seg))
    out = []
    for r, w in zip(rows_sel, before_rows):
        s = grad_t[bag[ids == r]].astype(np.float64).sum(axis=0)
        out.append((w.astype(np.float64) - lr * s).astype(np.float32))
    return np.stack(out) if out else np.zeros((0, grad_t.shape[1]), dtype=np.float32)
