"""Lookup-path parity at BASELINE.json's configurations, every
one through the C-ABI against the CPU oracle on the same generator-defined
tables, batch and gradient:

  cfg1  10 x dim 16, 1e5 rows, pf 8, D = 2, B = 512 — emulated on one GPU
        (every device's K1 / sort / SGD, the exchange as the device-local
        re-layout): all pooled rows, sorted keys, every table after SGD.
  cfg2  50 x dim 16, D = 4, B = 65536, the DreamShard placement (m50_d4
        checkpoint, greedy rollout on the GPU evaluator) — emulated: all
        65536 x 800 pooled rows, every device's sorted keys, all 50 tables.
  cfg3  D = 8, each of the 8 DreamShard ranks as its own one-rank context
        (world 8, no peers: what one process per GPU runs, sp_run_local):
        the rank's pre-exchange pooled rows for all bags, its sorted keys,
        and its heaviest and lightest tables after SGD.
  cfg4  the fewest- and the most-lookup rank's shard of 200 tables of 1e7
        rows (~62 GB on the device, one 28-bit key space): sorted keys of the
        whole shard, all pooled rows, one whole dim-16 table after SGD and
        sampled rows (hot and cold) of the shard's heaviest table.
  cfg3  with bf16 tables (D = 1): the sorted keys, pooled rows of every bag
        for 12 tables, and 3 whole tables after SGD within the double-rounding
        bound.

Tolerances: bit-exact sort; rtol 1e-5 pooled and tables (north star)."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import lookup as orc
from paper_2210_02023_b200 import api
from paper_2210_02023_b200.api import EmbeddingShard, PlacementTask, TableDesc
from tests.helpers import grad_cols, sgd_rows_expected, sub_batch, table_cols

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DATA = os.path.join(ROOT, "paper_2210_02023_b200", "data")
SEED = 2210
LR = 0.01
RTOL = 1e-5


def _pool(cfg):
    with open(os.path.join(DATA, "pools.json")) as f:
        p = json.load(f)[cfg]
    return ([TableDesc.from_dict(t) for t in p["tables"]], int(p["batch_size"]),
            float(p["mem_cap_gb"]))


def _dreamshard(task, ckpt):
    placement, _ = api.infer(api.load_checkpoint(os.path.join(DATA, ckpt)), task)
    return np.asarray(placement, dtype=np.int32)


def _check_pooled(got, task, off, idx, tables_list, chunk=8192):
    """got = [B, sum dims of tables_list] (tables in id order) == the
    oracle's fp64-accumulated forward over the generator's weights, in bag
    chunks (bounded host memory)."""
    dims = [t.dim for t in task.tables]
    rows = [t.hash_size for t in task.tables]
    B = task.batch_size
    cols = np.concatenate([table_cols(dims, t) for t in sorted(tables_list)])
    for lo in range(0, B, chunk):
        hi = min(B, lo + chunk)
        want = orc.tbe_forward(dims, rows, None, off, idx, B, tables_list=tables_list,
                               wseed=SEED, bag_lo=lo, bag_hi=hi)
        np.testing.assert_allclose(got[lo:hi], want[:, cols], rtol=RTOL, atol=1e-5)


def _check_sorted(sh, dev, task, off, idx, tables_list):
    rows = [t.hash_size for t in task.tables]
    k, b, h = sh.sorted(dev)
    wk, wb, wh = orc.sorted_keys(rows, off, idx, task.batch_size, sorted(tables_list))
    np.testing.assert_array_equal(k, wk)
    np.testing.assert_array_equal(b, wb)
    np.testing.assert_array_equal(h, wh)


def _check_sgd_tables(sh, task, off, idx, picks, before):
    """Whole tables `picks` after one SGD step == the oracle's row-wise SGD
    over all of their lookups, with the generator's gradient."""
    B = task.batch_size
    dims = [t.dim for t in task.tables]
    sub_off, sub_idx = sub_batch(off, idx, B, picks)
    cols = np.concatenate([table_cols(dims, t) for t in picks])
    grad = grad_cols(SEED, B, cols)
    want = orc.tbe_backward_sgd([dims[t] for t in picks],
                                [task.tables[t].hash_size for t in picks],
                                [before[t] for t in picks], sub_off, sub_idx, B, grad, LR,
                                list(range(len(picks))))
    for k, t in enumerate(picks):
        np.testing.assert_allclose(sh.get_table(t), want[k], rtol=RTOL, atol=1e-6)


def _emulated(cfg, D, placement_fn):
    tables, B, cap = _pool(cfg)
    task = PlacementTask(tables, D, cap, B)
    placement = placement_fn(task)
    off, idx = orc.synth_batch([t.to_dict() for t in tables], B, SEED)
    sh = EmbeddingShard(task, placement, lr=LR)
    sh.init_tables(SEED)
    sh.synth_batch(SEED)
    sh.synth_grad(SEED)
    assert sh.nnz == len(idx)
    before = {t: sh.get_table(t) for t in range(len(tables))}
    # the generator's weights, spot-checked against the oracle's
    for t in (0, len(tables) - 1):
        for r in (0, tables[t].hash_size - 1):
            assert before[t][r, 3] == orc.lib().or_weight(SEED, t, r, 3)
    bd = sh.run_iteration()
    assert abs(bd.overall_ms - (max(bd.fwd_ms) + bd.fwd_comm_stage_ms + bd.bwd_comm_stage_ms +
                                max(bd.bwd_ms))) < 1e-9
    for d in range(D):
        _check_sorted(sh, d, task, off, idx, [t for t in range(len(tables)) if placement[t] == d])
    _check_pooled(sh.pooled(), task, off, idx, list(range(len(tables))))
    _check_sgd_tables(sh, task, off, idx, list(range(len(tables))), before)
    sh.close()


def test_cfg1_emulated_d2():
    _emulated("cfg1", 2, lambda task: _dreamshard(task, "dreamshard_m50_d4.dshd"))


def test_cfg2_emulated_d4_dreamshard():
    _emulated("cfg2", 4, lambda task: _dreamshard(task, "dreamshard_m50_d4.dshd"))


@pytest.fixture(scope="module")
def cfg3_d8():
    tables, B, cap = _pool("cfg3")
    task = PlacementTask(tables, 8, cap, B)
    placement = _dreamshard(task, "dreamshard_m100_d8.dshd")
    off, idx = orc.synth_batch([t.to_dict() for t in tables], B, SEED)
    return task, placement, off, idx


@pytest.mark.parametrize("rank", range(8))
def test_cfg3_d8_rank_context(cfg3_d8, rank):
    task, placement, off, idx = cfg3_d8
    B = task.batch_size
    sh = EmbeddingShard(task, placement, lr=LR, rank=rank, world_size=8, nccl_id=None)
    local = sh.local_tables()
    assert local == [t for t in range(len(task.tables)) if placement[t] == rank]
    sh.init_tables(SEED)
    sh.synth_batch(SEED)
    sh.synth_grad(SEED)
    nnz = np.diff(off[::B])
    dims = np.array([t.dim for t in task.tables])
    heavy = max(local, key=lambda t: nnz[t] * dims[t])
    light = min(local, key=lambda t: (dims[t], nnz[t]))
    picks = sorted({heavy, light})
    before = {t: sh.get_table(t) for t in picks}
    sh.run_local()  # K1, the sort, then the SGD on the delivered gradient
    _check_sorted(sh, rank, task, off, idx, local)
    _check_pooled(sh.local_pooled(rank), task, off, idx, local)
    _check_sgd_tables(sh, task, off, idx, picks, before)
    sh.close()


@pytest.mark.parametrize("which", ["fewest", "most"])
def test_cfg4_rank_shard(which):
    """One of 8 DreamShard ranks of cfg4 (200 tables x 1e7 rows, 64 GB cap):
    the fewest- and the most-lookup rank (~30 M lookups in one 28-bit key
    space: the largest sort of any config), ~62 GB of fp32 tables each."""
    tables, B, cap = _pool("cfg4")
    task = PlacementTask(tables, 8, cap, B)
    placement = _dreamshard(task, "dreamshard_m100_d8.dshd")
    off, idx = orc.synth_batch([t.to_dict() for t in tables], B, SEED)
    nnz = np.diff(off[::B])
    dims = np.array([t.dim for t in tables])
    per_rank = [int(nnz[placement == r].sum()) for r in range(8)]
    rank = int(np.argmin(per_rank) if which == "fewest" else np.argmax(per_rank))
    local = [t for t in range(len(tables)) if placement[t] == rank]
    torch.cuda.empty_cache()
    sh = EmbeddingShard(task, placement, lr=LR, rank=rank, world_size=8, nccl_id=None)
    assert sh.device_bytes > 40e9
    sh.init_tables(SEED)
    sh.synth_batch(SEED)
    sh.synth_grad(SEED)
    assert sh.nnz == per_rank[rank]
    heavy = max(local, key=lambda t: nnz[t] * dims[t])
    small = min((t for t in local if t != heavy), key=lambda t: (dims[t], nnz[t]))
    before_small = sh.get_table(small)
    before_heavy = sh.get_table(heavy)
    sh.run_local()
    _check_sorted(sh, rank, task, off, idx, local)
    _check_pooled(sh.local_pooled(rank), task, off, idx, local)
    _check_sgd_tables(sh, task, off, idx, [small], {small: before_small})
    # heaviest table: hot rows (the generator's k * rows/1024), cold touched
    # rows and an untouched row
    R = tables[heavy].hash_size
    seg = off[heavy * B:(heavy + 1) * B + 1]
    ids = idx[seg[0]:seg[-1]]
    rng = np.random.default_rng(0)
    hot = [k * (R // 1024) for k in (0, 1, 511, 1023)]
    cold = rng.choice(ids, size=12, replace=False).tolist()
    untouched = next(r for r in range(1, R) if r % (R // 1024) and not np.any(ids == r))
    rows_sel = sorted(set(hot + cold + [untouched]))
    after = sh.get_table(heavy)[rows_sel]
    want = sgd_rows_expected(off, idx, B, heavy, rows_sel, before_heavy[rows_sel],
                             grad_cols(SEED, B, table_cols(list(dims), heavy)), LR)
    np.testing.assert_allclose(after, want, rtol=RTOL, atol=1e-6)
    np.testing.assert_array_equal(after[rows_sel.index(untouched)], before_heavy[untouched])
    sh.close()


def _to_bf16(x):
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def test_cfg3_bf16_tables():
    """cfg3 at full size with bf16 storage (the 2-byte paths: raw 16-byte
    slices in K1, 32-byte gradient loads in the SGD, REDG.ADD.BF16x8)."""
    from paper_2210_02023_b200.api import table_memory_gb
    tables, B, cap = _pool("cfg3")
    tables = [TableDesc(t.id, t.dim, t.hash_size, t.pooling_factor,
                        table_memory_gb(t.hash_size, t.dim, 2), t.dist) for t in tables]
    task = PlacementTask(tables, 1, 0.0, B)
    off, idx = orc.synth_batch([t.to_dict() for t in tables], B, SEED)
    sh = EmbeddingShard(task, np.zeros(len(tables), dtype=np.int32), lr=LR, storage="bf16")
    sh.init_tables(SEED)
    sh.synth_batch(SEED)
    _check_sorted(sh, 0, task, off, idx, list(range(len(tables))))
    nnz = np.diff(off[::B])
    dims = [t.dim for t in tables]
    rows = [t.hash_size for t in tables]
    heavy = int(np.argmax(nnz * np.array(dims)))
    picks = sorted({heavy} | set(range(3, len(tables), 9)))
    w = {t: sh.get_table(t) for t in picks}
    for t in picks[:3]:  # the generator's weights, rounded to bf16
        np.testing.assert_array_equal(w[t][:64, :4], _to_bf16(
            np.array([[orc.lib().or_weight(SEED, t, r, c) for c in range(4)] for r in range(64)],
                     dtype=np.float32)))
    sh.forward()
    sh.a2a_forward()
    pooled = sh.pooled()
    cols = np.concatenate([table_cols(dims, t) for t in picks])
    wl = [w.get(t) for t in range(len(tables))]
    for lo in range(0, B, 16384):
        want = orc.tbe_forward(dims, rows, wl, off, idx, B, tables_list=picks,
                               bag_lo=lo, bag_hi=lo + 16384)
        np.testing.assert_allclose(pooled[lo:lo + 16384][:, cols], want[:, cols], rtol=1e-5,
                                   atol=1e-5)
    sh.synth_grad(SEED)
    sh.backward_sgd()
    three = [heavy] + [t for t in picks if t != heavy][:2]
    sub_off, sub_idx = sub_batch(off, idx, B, three)
    g = grad_cols(SEED, B, np.concatenate([table_cols(dims, t) for t in three]))
    ref = orc.tbe_backward_sgd([dims[t] for t in three], [rows[t] for t in three],
                               [w[t] for t in three], sub_off, sub_idx, B, g, LR, [0, 1, 2])

    def ulp(x):
        x = np.abs(x.astype(np.float32))
        return 2.0 ** (np.floor(np.log2(np.maximum(x, 2.0 ** -126))) - 7)
    for k, t in enumerate(three):
        got = sh.get_table(t)
        bound = 0.5 * ulp(ref[k]) + 0.5 * ulp(ref[k] - w[t]) + 1e-7
        assert np.all(np.abs(got - ref[k]) <= bound), t
    sh.close()


@pytest.mark.parametrize("cfg,D", [("cfg1", 2), ("cfg2", 4)])
def test_against_torch_embedding_bag(cfg, D):
    """The GPU iteration against a third-party implementation of the same
    operator: PyTorch's embedding_bag(mode="sum") per table and the SGD
    step from its autograd (CPU), on the generator's tables, batch and
    gradient; every pooled value and every table after the step. Both sides
    accumulate in fp32 in their own order (hot rows sum thousands of
    gradient rows), so the tables get atol 5e-6 beside rtol 1e-5."""
    tables, B, cap = _pool(cfg)
    task = PlacementTask(tables, D, cap, B)
    placement = _dreamshard(task, "dreamshard_m50_d4.dshd")
    off, idx = orc.synth_batch([t.to_dict() for t in tables], B, SEED)
    sh = EmbeddingShard(task, placement, lr=LR)
    sh.init_tables(SEED)
    sh.synth_batch(SEED)
    sh.synth_grad(SEED)
    weights = [sh.get_table(t) for t in range(len(tables))]
    sh.run_iteration()
    dims = [t.dim for t in tables]
    grad = grad_cols(SEED, B, np.arange(sum(dims)))
    pooled = sh.pooled()
    col = 0
    for t, tab in enumerate(tables):
        seg = off[t * B:(t + 1) * B + 1]
        ids = torch.from_numpy(idx[seg[0]:seg[-1]].astype(np.int64))
        offs = torch.from_numpy((seg[:-1] - seg[0]).astype(np.int64))
        w = torch.tensor(weights[t], requires_grad=True)
        p = torch.nn.functional.embedding_bag(ids, w, offs, mode="sum")
        (p * torch.from_numpy(np.ascontiguousarray(grad[:, col:col + tab.dim]))).sum().backward()
        np.testing.assert_allclose(pooled[:, col:col + tab.dim], p.detach().numpy(),
                                   rtol=RTOL, atol=1e-5)
        np.testing.assert_allclose(sh.get_table(t), (w - LR * w.grad).detach().numpy(),
                                   rtol=RTOL, atol=5e-6)
        col += tab.dim
    sh.close()
