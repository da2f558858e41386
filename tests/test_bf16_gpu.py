"""bf16 table storage (2 B/param like the paper's fp16 tables, PAPER.md:709,
and the reference's default sizing, table.hpp:30 / table_memory_gb; fp32's
exponent range), selected with sp_ctx_create_ex(SP_STORAGE_BF16). Pooled
outputs, gradients and sums stay fp32. Forward: exact bf16 inputs summed in
fp32 -> rtol 1e-5 vs the fp64 oracle. Backward: W <- bf16(W + bf16(-lr *
sum)) by an L2 bf16x8 reduction (REDG.ADD.BF16x8) -> within half a bf16 ulp
of the result plus half a bf16 ulp of the update of the fp64 oracle."""
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


def _to_bf16(x):
    """Round-to-nearest-even fp32 -> bf16 -> fp32."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def _ulp_bf16(x):
    x = np.abs(x.astype(np.float32))
    e = np.floor(np.log2(np.maximum(x, 2.0 ** -126)))
    return 2.0 ** (e - 7)


@pytest.mark.parametrize("D", [1, 2])
def test_bf16_forward_backward_matches_oracle(D):
    B = 128
    dims = [8, 16, 32, 64, 128, 256, 12, 16]
    rows = [700, 3000, 50, 900, 400, 300, 200, 20]
    pfs = [3.0, 8.0, 2.0, 5.0, 12.0, 4.0, 3.0, 30.0]
    hot = [0.0, 0.5, 0.0, 0.9, 0.3, 0.0, 0.2, 1.0]
    tables = _tables(dims, rows, pfs, hot)
    task = PlacementTask(tables, D, 0.0, B)
    placement = [i % D for i in range(len(dims))]
    rng = np.random.default_rng(3)
    weights = [_to_bf16(rng.uniform(0.5, 1.0, size=(t.hash_size, t.dim))) for t in tables]
    off, idx = orc.synth_batch(as_dicts(tables), B, seed=12)
    W = sum(dims)
    grad = np.random.default_rng(5).uniform(-1, 1, size=(B, W)).astype(np.float32)
    lr = 0.05
    sh = EmbeddingShard(task, placement, lr=lr, storage="bf16")
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
    changed = 0
    for i in range(len(dims)):
        got = sh.get_table(i)
        # two roundings: the delta to bf16, then the sum at L2
        bound = 0.5 * _ulp_bf16(ref[i]) + 0.5 * _ulp_bf16(ref[i] - weights[i]) + 1e-7
        err = np.abs(got - ref[i])
        assert np.all(err <= bound), (i, float((err - bound).max()))
        changed += int(np.sum(got != weights[i]))
    assert changed > 0
    sh.close()


def test_bf16_synth_and_pipelined_batch():
    B = 256
    dims = [16, 64, 128]
    tables = _tables(dims, [5000, 800, 300], [6.0, 3.0, 9.0], [0.3, 0.0, 0.6])
    task = PlacementTask(tables, 1, 0.0, B)
    sh = EmbeddingShard(task, [0, 0, 0], lr=0.01, storage="bf16")
    sh.init_tables(7)
    w0 = [sh.get_table(i) for i in range(3)]
    # the generator's fp32 weights, rounded to bf16
    for i in range(3):
        for r in (0, 17):
            want = np.array([orc.lib().or_weight(7, i, r, c) for c in range(dims[i])],
                            dtype=np.float32)
            np.testing.assert_array_equal(w0[i][r], _to_bf16(want))
    sh.synth_grad(7)
    off, idx = orc.synth_batch(as_dicts(tables), B, seed=4)
    bd = sh.run_batch(LookupBatch(idx, off, 3, B))
    assert bd.overall_ms > 0
    rows = [t.hash_size for t in tables]
    np.testing.assert_allclose(sh.pooled(), orc.tbe_forward(dims, rows, w0, off, idx, B),
                               rtol=1e-5, atol=1e-5)
    sh.close()


def test_storage_must_match_sizing():
    t4 = _tables([16, 16], [100, 100], [1.0, 1.0], [0.0, 0.0], bpp=4)
    with pytest.raises(ShardplanError) as e:
        EmbeddingShard(PlacementTask(t4, 1, 0.0, 4), [0, 0], storage="bf16")
    assert e.value.kind == "bad_input"
    t2 = _tables([16, 16], [100, 100], [1.0, 1.0], [0.0, 0.0], bpp=2)
    with pytest.raises(ShardplanError):
        EmbeddingShard(PlacementTask(t2, 1, 0.0, 4), [0, 0], storage="fp32")
    with pytest.raises(ShardplanError):
        EmbeddingShard(PlacementTask(t2, 1, 0.0, 4), [0, 0], storage="int8")
