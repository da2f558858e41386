"""fp16 table storage (2 B/param: the paper's fp16 tables, and
the reference's default sizing, table_memory_gb in table.hpp:55-63). The
storage type follows each table's table_size_gb; pooled outputs, gradients
and sums stay fp32. Forward: exact fp16 inputs summed in fp32 -> rtol 1e-5 vs
the fp64 oracle. Backward: W <- fp16(W + fp16(-lr * sum)) by an L2 fp16x8
reduction -> within half an fp16 ulp of the result plus half an fp16 ulp of
the update of the fp64 oracle."""
import numpy as np
import pytest

from oracle import lookup as orc
from paper_2210_02023_b200.api import (EmbeddingShard, LookupBatch, PlacementTask,
                                       ShardplanError, TableDesc, table_memory_gb)
from tests.helpers import as_dicts

pytestmark = pytest.mark.gpu


def _tables(dims, rows, pfs, hot, bpp=2):
    out = []
    for i, (d, r, pf, h) in enumerate(zip(dims, rows, pfs, hot)):
        dist = [0.0] * 17
        dist[12] = h
        dist[0], dist[1], dist[2] = 0.5 * (1 - h), 0.3 * (1 - h), 0.2 * (1 - h)
        out.append(TableDesc(i, d, r, pf, table_memory_gb(r, d, bpp), dist))
    return out


def _half_weights(seed, tables):
    rng = np.random.default_rng(seed)
    return [rng.uniform(0.5, 1.0, size=(t.hash_size, t.dim)).astype(np.float16).astype(np.float32)
            for t in tables]


def _ulp16(x):
    x = np.abs(x.astype(np.float32))
    e = np.floor(np.log2(np.maximum(x, 2.0 ** -14)))
    return 2.0 ** (e - 10)


@pytest.mark.parametrize("D", [1, 2])
def test_fp16_forward_backward_matches_oracle(D):
    B = 128
    dims = [8, 16, 32, 64, 128, 256, 12, 16]
    rows = [700, 3000, 50, 900, 400, 300, 200, 20]
    pfs = [3.0, 8.0, 2.0, 5.0, 12.0, 4.0, 3.0, 30.0]
    hot = [0.0, 0.5, 0.0, 0.9, 0.3, 0.0, 0.2, 1.0]
    tables = _tables(dims, rows, pfs, hot)
    task = PlacementTask(tables, D, 0.0, B)
    placement = [i % D for i in range(len(dims))]
    weights = _half_weights(3, tables)
    off, idx = orc.synth_batch(as_dicts(tables), B, seed=12)
    W = sum(dims)
    grad = np.random.default_rng(5).uniform(-1, 1, size=(B, W)).astype(np.float32)
    lr = 0.05
    sh = EmbeddingShard(task, placement, lr=lr)
    for i, w in enumerate(weights):
        sh.set_table(i, w)
        np.testing.assert_array_equal(sh.get_table(i), w)  # exact round trip
    sh.upload_batch(LookupBatch(idx, off, len(dims), B))
    sh.forward()
    sh.a2a_forward()
    want = orc.tbe_forward(dims, rows, weights, off, idx, B)
    np.testing.assert_allclose(sh.pooled(), want, rtol=1e-5, atol=1e-5)
    sh.set_grad(grad)
    sh.a2a_backward()
    sh.backward_sgd()
    ref = orc.tbe_backward_sgd(dims, rows, weights, off, idx, B, grad, lr, list(range(len(dims))))
    for i in range(len(dims)):
        got = sh.get_table(i)
        # two roundings: the delta to fp16, then the sum at L2
        bound = 0.5 * _ulp16(ref[i]) + 0.5 * _ulp16(ref[i] - weights[i]) + 1e-7
        err = np.abs(got - ref[i])
        assert np.all(err <= bound), (i, float((err - bound).max()))
    sh.close()


def test_fp16_pipelined_batch_and_synth():
    B = 256
    dims = [16, 64, 128]
    tables = _tables(dims, [5000, 800, 300], [6.0, 3.0, 9.0], [0.3, 0.0, 0.6])
    task = PlacementTask(tables, 1, 0.0, B)
    sh = EmbeddingShard(task, [0, 0, 0], lr=0.01)
    sh.init_tables(7)
    w0 = [sh.get_table(i) for i in range(3)]
    assert all(np.all((w >= 0.5) & (w <= 1.0)) for w in w0)
    sh.synth_grad(7)
    off, idx = orc.synth_batch(as_dicts(tables), B, seed=4)
    bd = sh.run_batch(LookupBatch(idx, off, 3, B))
    assert bd.overall_ms > 0
    rows = [t.hash_size for t in tables]
    np.testing.assert_allclose(sh.pooled(), orc.tbe_forward(dims, rows, w0, off, idx, B),
                               rtol=1e-5, atol=1e-5)
    sh.synth_batch(9)
    sh.run_iteration()
    sh.close()


def test_mixed_bytes_per_param_rejected():
    t = _tables([16, 16], [100, 100], [1.0, 1.0], [0.0, 0.0])
    t[1] = TableDesc(1, 16, 100, 1.0, table_memory_gb(100, 16, 4), t[1].dist)
    with pytest.raises(ShardplanError) as e:
        EmbeddingShard(PlacementTask(t, 1, 0.0, 4), [0, 0])
    assert e.value.kind == "bad_input"
