"""Parity at BASELINE.json's full cfg3 size (100 tables, B = 65536, 44 M
lookups, 9.2 GB of fp32 tables, one device): the same synthetic batch and
weights on the GPU and in the CPU oracle (generator-defined weights, so the
oracle never materialises the tables).
  - the backward's sorted (key, bag) pairs and run heads == std::stable_sort
    over the whole batch, bit for bit;
  - all pooled rows (every bag of every table) == the oracle's
    fp64-accumulated forward (rtol 1e-5);
  - ten whole tables (the heaviest, a dim-16, a dim-128 one and every 14th) after one
    SGD step == the oracle's row-wise SGD over all of their lookups (rtol 1e-5).
"""
import json
import os

import numpy as np
import pytest

from oracle import lookup as orc
from paper_2210_02023_b200.api import EmbeddingShard, PlacementTask, TableDesc
from tests.helpers import grad_cols

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 2210
LR = 0.01


@pytest.fixture(scope="module")
def cfg3():
    with open(os.path.join(ROOT, "paper_2210_02023_b200", "data", "pools.json")) as f:
        pool = json.load(f)["cfg3"]
    tables = [TableDesc.from_dict(t) for t in pool["tables"]]
    B = int(pool["batch_size"])
    task = PlacementTask(tables, 1, 0.0, B)
    sh = EmbeddingShard(task, np.zeros(len(tables), dtype=np.int32), lr=LR)
    sh.init_tables(SEED)
    sh.synth_batch(SEED)
    off, idx = orc.synth_batch([t.to_dict() for t in tables], B, SEED)
    assert sh.nnz == len(idx)
    yield task, sh, off, idx
    sh.close()


def test_fullsize_sort_bit_exact(cfg3):
    task, sh, off, idx = cfg3
    keys, bags, heads = sh.sorted(0)
    rows = [t.hash_size for t in task.tables]
    wk, wb, wh = orc.sorted_keys(rows, off, idx, task.batch_size, list(range(len(rows))))
    np.testing.assert_array_equal(keys, wk)
    np.testing.assert_array_equal(bags, wb)
    np.testing.assert_array_equal(heads, wh)


def test_fullsize_forward_all_bags(cfg3):
    """Every pooled row of the 65536 x 6224 output (1.6 GB), in bag chunks."""
    task, sh, off, idx = cfg3
    B = task.batch_size
    dims = [t.dim for t in task.tables]
    rows = [t.hash_size for t in task.tables]
    sh.forward()
    sh.a2a_forward()
    pooled = sh.pooled()
    for lo in range(0, B, 8192):
        hi = lo + 8192
        want = orc.tbe_forward(dims, rows, None, off, idx, B, wseed=SEED, bag_lo=lo, bag_hi=hi)
        np.testing.assert_allclose(pooled[lo:hi], want, rtol=1e-5, atol=1e-5)


def test_fullsize_sgd_whole_tables(cfg3):
    task, sh, off, idx = cfg3
    B = task.batch_size
    T = len(task.tables)
    dims = [t.dim for t in task.tables]
    nnz = np.diff(off[::B])
    heavy = int(np.argmax(nnz * np.array(dims)))
    d16 = next(i for i in range(T) if dims[i] == 16 and i != heavy)
    d128 = next(i for i in range(T) if dims[i] == 128 and i != heavy)
    picks = sorted({heavy, d16, d128} | set(range(0, T, 14)))
    before = {t: sh.get_table(t) for t in picks}
    gcol = np.concatenate([[0], np.cumsum(dims)[:-1]])
    sh.synth_grad(SEED)
    sh.backward_sgd()
    # the oracle on a task of just the picked tables (their CSR segments rebased)
    sub_off = [np.zeros(1, dtype=np.int64)]
    sub_idx = []
    base = 0
    for t in picks:
        seg = off[t * B:(t + 1) * B + 1]
        sub_off.append(seg[1:] - seg[0] + base)
        sub_idx.append(idx[seg[0]:seg[-1]])
        base += seg[-1] - seg[0]
    sub_off = np.concatenate(sub_off)
    sub_idx = np.concatenate(sub_idx)
    cols = np.concatenate([np.arange(gcol[t], gcol[t] + dims[t]) for t in picks])
    grad = grad_cols(SEED, B, cols)
    sub_dims = [dims[t] for t in picks]
    sub_rows = [task.tables[t].hash_size for t in picks]
    want = orc.tbe_backward_sgd(sub_dims, sub_rows, [before[t] for t in picks], sub_off,
                                sub_idx, B, grad, LR, list(range(len(picks))))
    for k, t in enumerate(picks):
        np.testing.assert_allclose(sh.get_table(t), want[k], rtol=1e-5, atol=1e-6)
