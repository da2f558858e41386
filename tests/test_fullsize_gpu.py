"""Parity at BASELINE.json's full cfg3 size (100 tables, B = 65536, 44 M
lookups, 9.2 GB of fp32 tables, one device): the same synthetic batch and
weights on the GPU and in the CPU oracle (generator-defined weights, so the
oracle never materialises the tables).
  - the backward's sorted (key, bag) pairs and run heads == std::stable_sort
    over the whole batch, bit for bit;
  - pooled rows of the first and last 512 bags of every table == the oracle's
    fp64-accumulated forward (rtol 1e-5);
  - three whole tables (the heaviest, a dim-16 and a dim-128 one) after one
    SGD step == the oracle's row-wise SGD over all of their lookups (rtol 1e-5).
"""
import json
import os

import numpy as np
import pytest

from oracle import lookup as orc
from paper_2210_02023_b200.api import EmbeddingShard, PlacementTask, TableDesc

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


def test_fullsize_forward_sampled_bags(cfg3):
    task, sh, off, idx = cfg3
    B = task.batch_size
    dims = [t.dim for t in task.tables]
    rows = [t.hash_size for t in task.tables]
    sh.forward()
    sh.a2a_forward()
    pooled = sh.pooled()
    for lo, hi in ((0, 512), (B - 512, B)):
        want = orc.tbe_forward(dims, rows, None, off, idx, B, wseed=SEED, bag_lo=lo, bag_hi=hi)
        np.testing.assert_allclose(pooled[lo:hi], want, rtol=1e-5, atol=1e-5)


def _grad_cols(seed, B, cols):
    """The SURVEY 8d gradient generator (synth.cuh grad_value), vectorised:
    columns `cols` of dL/dpooled for every bag."""
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


def test_fullsize_sgd_whole_tables(cfg3):
    task, sh, off, idx = cfg3
    B = task.batch_size
    T = len(task.tables)
    dims = [t.dim for t in task.tables]
    nnz = np.diff(off[::B])
    heavy = int(np.argmax(nnz * np.array(dims)))
    d16 = next(i for i in range(T) if dims[i] == 16 and i != heavy)
    d128 = next(i for i in range(T) if dims[i] == 128 and i != heavy)
    picks = [heavy, d16, d128]
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
    grad = _grad_cols(SEED, B, cols)
    sub_dims = [dims[t] for t in picks]
    sub_rows = [task.tables[t].hash_size for t in picks]
    want = orc.tbe_backward_sgd(sub_dims, sub_rows, [before[t] for t in picks], sub_off,
                                sub_idx, B, grad, LR, [0, 1, 2])
    for k, t in enumerate(picks):
        np.testing.assert_allclose(sh.get_table(t), want[k], rtol=1e-5, atol=1e-6)
