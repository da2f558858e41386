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
