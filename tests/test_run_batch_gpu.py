"""sp_run_batch — the pipelined upload + iteration with host buffers (the e2e
path of bench.py) — against the CPU oracle and against the unpipelined
upload_batch + run_iteration, including many upload chunks, each sorted on its own
(sp_ctx_set_upload_chunk) with many small sort buckets (sp_ctx_set_sort_target), and its deferred validation: a bad
batch raises like upload_batch and leaves every table untouched."""
import os

import numpy as np
import pytest

from oracle import lookup as orc
from paper_2210_02023_b200.api import EmbeddingShard, LookupBatch, ShardplanError
from tests.helpers import as_dicts, random_task, random_weights

pytestmark = pytest.mark.gpu

RTOL = 1e-5


@pytest.fixture(params=["default", "chunked"])
def chunking(request):
    return request.param


def _shard(task, placement, weights, lr, chunking="default", overlap=True):
    sh = EmbeddingShard(task, placement, lr=lr)
    if chunking == "chunked":
        sh.set_upload_chunk(700)
        sh.set_sort_target(9)
    sh.set_overlap(overlap)
    for i, w in enumerate(weights):
        sh.set_table(i, w)
    return sh


@pytest.mark.parametrize("D", [1, 3])
@pytest.mark.parametrize("overlap", [True, False])
def test_run_batch_matches_oracle(D, overlap, chunking):
    B = 96
    dims = [16, 32, 64, 128, 16, 64, 12, 4]
    task, placement = random_task(31 + D, dims, D, B)
    weights = random_weights(13, task.tables)
    off, idx = orc.synth_batch(as_dicts(task.tables), B, seed=9)
    W = sum(dims)
    grad = np.random.default_rng(4).uniform(-1, 1, size=(B, W)).astype(np.float32)
    lr = 0.02
    sh = _shard(task, placement, weights, lr, chunking, overlap)
    sh.set_grad(grad)
    bd = sh.run_batch(LookupBatch(idx, off, len(dims), B))
    assert bd.overall_ms > 0 and len(bd.fwd_ms) == D
    rows = [t.hash_size for t in task.tables]
    np.testing.assert_allclose(sh.pooled(), orc.tbe_forward(dims, rows, weights, off, idx, B),
                               rtol=RTOL, atol=1e-5)
    want = orc.tbe_backward_sgd(dims, rows, weights, off, idx, B, grad, lr,
                                list(range(len(dims))))
    got = [sh.get_table(i) for i in range(len(dims))]
    for i in range(len(dims)):
        np.testing.assert_allclose(got[i], want[i], rtol=RTOL, atol=1e-5)
    # identical to the unpipelined path on a fresh shard (same kernels, same order)
    ref = _shard(task, placement, weights, lr)
    ref.set_grad(grad)
    ref.upload_batch(LookupBatch(idx, off, len(dims), B))
    ref.run_iteration()
    for i in range(len(dims)):
        np.testing.assert_array_equal(got[i], ref.get_table(i))
    # the batch stays current: a plain iteration on it works
    sh.run_iteration()
    sh.close()
    ref.close()


def test_run_batch_rejects_bad_batch_without_update(chunking):
    B = 64
    dims = [16, 64, 32]
    task, placement = random_task(5, dims, 1, B)
    weights = random_weights(3, task.tables)
    off, idx = orc.synth_batch(as_dicts(task.tables), B, seed=2)
    sh = _shard(task, placement, weights, 0.1, chunking)
    sh.set_grad(np.ones((B, sum(dims)), dtype=np.float32))
    bad = idx.copy()
    bad[len(bad) // 2] = task.tables[1].hash_size + 5  # out of range in table 1
    with pytest.raises(ShardplanError) as e:
        sh.run_batch(LookupBatch(bad, off, 3, B))
    assert e.value.kind == "bad_input"
    for i in range(3):
        np.testing.assert_array_equal(sh.get_table(i), weights[i])
    with pytest.raises(ShardplanError):  # no batch is current after the failure
        sh.run_iteration()
    bad_off = off.copy()
    bad_off[5] = bad_off[7] + 1  # decreases inside table 0
    with pytest.raises(ShardplanError) as e:
        sh.run_batch(LookupBatch(idx, bad_off, 3, B))
    assert e.value.kind == "malformed_batch"
    for i in range(3):
        np.testing.assert_array_equal(sh.get_table(i), weights[i])
    # a good batch afterwards works
    sh.run_batch(LookupBatch(idx, off, 3, B))
    sh.close()


def test_run_batches_equals_sequential_steps(chunking):
    """sp_run_batches (step s's H2D under step s-1's compute) == the same
    steps one sp_run_batch at a time, bit for bit; a bad step in the middle
    updates nothing and is reported by index."""
    B = 96
    dims = [16, 64, 32, 128, 8]
    task, placement = random_task(77, dims, 1, B)
    weights = random_weights(21, task.tables)
    batches = []
    for seed in (3, 4, 5):
        off, idx = orc.synth_batch(as_dicts(task.tables), B, seed=seed)
        batches.append(LookupBatch(idx, off, len(dims), B))
    grad = np.random.default_rng(8).uniform(-1, 1, size=(B, sum(dims))).astype(np.float32)
    a = _shard(task, placement, weights, 0.02, chunking)
    a.set_grad(grad)
    ms = a.run_batches(batches)
    assert len(ms) == 3 and all(m > 0 for m in ms)
    b = _shard(task, placement, weights, 0.02, chunking)
    b.set_grad(grad)
    for bt in batches:
        b.run_batch(bt)
    for i in range(len(dims)):
        np.testing.assert_array_equal(a.get_table(i), b.get_table(i))
    # bad middle step
    bad_idx = batches[1].indices.copy()
    bad_idx[0] = -1
    bad = LookupBatch(bad_idx, batches[1].offsets, len(dims), B)
    c = _shard(task, placement, weights, 0.02, chunking)
    c.set_grad(grad)
    with pytest.raises(ShardplanError) as e:
        c.run_batches([batches[0], bad, batches[2]])
    assert e.value.kind == "bad_input" and "step 1" in str(e.value)
    d = _shard(task, placement, weights, 0.02, chunking)
    d.set_grad(grad)
    d.run_batch(batches[0])
    d.run_batch(batches[2])
    for i in range(len(dims)):
        np.testing.assert_array_equal(c.get_table(i), d.get_table(i))
    for sh in (a, b, c, d):
        sh.close()
