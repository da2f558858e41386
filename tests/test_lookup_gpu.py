"""GPU parity of the embedding hot path (K1 forward, exchange layout, K4
backward) against the CPU oracle (oracle/lookup_oracle.cpp), through the
C-ABI. Tolerances follow BASELINE.json's north star: rtol 1e-5 for fp32
pooled outputs and updated tables; bit-exact for sorted keys, bag payloads
and segment boundaries."""
import numpy as np
import pytest

from oracle import lookup as orc
from paper_2210_02023_b200.api import (EmbeddingShard, LookupBatch, PlacementTask,
                                       ShardplanError)
from tests.helpers import as_dicts, make_tables, random_task, random_weights

pytestmark = pytest.mark.gpu

RTOL = 1e-5
ATOL = 1e-5

DIM_SETS = {
    "pow2": [16, 32, 64, 128, 16, 64],
    "small": [4, 8, 4, 8],
    "generic": [12, 3, 256, 20, 1, 136],
}


def _shard(task, placement, weights, lr=0.01):
    sh = EmbeddingShard(task, placement, lr=lr)
    for i, w in enumerate(weights):
        sh.set_table(i, w)
    return sh


def _oracle_pooled(task, weights, off, idx):
    dims = [t.dim for t in task.tables]
    rows = [t.hash_size for t in task.tables]
    return orc.tbe_forward(dims, rows, weights, off, idx, task.batch_size)


@pytest.mark.parametrize("dims", list(DIM_SETS))
@pytest.mark.parametrize("D", [1, 3])
def test_forward_matches_oracle(dims, D):
    B = 96
    task, placement = random_task(7 + D, DIM_SETS[dims], D, B)
    weights = random_weights(11, task.tables)
    off, idx = orc.synth_batch(as_dicts(task.tables), B, seed=5)
    sh = _shard(task, placement, weights)
    sh.upload_batch(LookupBatch(idx, off, len(task.tables), B))
    sh.forward()
    sh.a2a_forward()
    got = sh.pooled()
    want = _oracle_pooled(task, weights, off, idx)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)
    # each (virtual) device's pre-exchange output, its tables in id order
    for d in range(D):
        cols = np.concatenate([np.arange(sum(t.dim for t in task.tables[:i]),
                                         sum(t.dim for t in task.tables[:i + 1]))
                               for i in range(len(task.tables)) if placement[i] == d] or
                              [np.zeros(0, dtype=int)])
        np.testing.assert_allclose(sh.local_pooled(d), want[:, cols], rtol=RTOL, atol=ATOL)


def test_forward_hand_case():
    """Hand-computed: 2 tables (dim 4, dim 8), B = 3, empty bag included."""
    tables = make_tables([4, 8], [3, 2], [1.0, 1.0])
    task = PlacementTask(tables, 1, 0.0, 3)
    w0 = np.arange(12, dtype=np.float32).reshape(3, 4)
    w1 = np.arange(16, dtype=np.float32).reshape(2, 8) * 10
    # table 0: bags {0,2}, {}, {1,1,1}; table 1: bags {1}, {0,1}, {}
    off = np.array([0, 2, 2, 5, 6, 8, 8])
    idx = np.array([0, 2, 1, 1, 1, 1, 0, 1])
    sh = _shard(task, [0, 0], [w0, w1])
    sh.upload_batch(LookupBatch(idx, off, 2, 3))
    sh.forward()
    got = sh.pooled()
    want = np.zeros((3, 12), dtype=np.float32)
    want[0, :4] = w0[0] + w0[2]
    want[2, :4] = 3 * w0[1]
    want[0, 4:] = w1[1]
    want[1, 4:] = w1[0] + w1[1]
    np.testing.assert_array_equal(got, want)


@pytest.fixture(params=[0, 7])
def sort_target(request):
    """The default K4a sort plan, and one forced to buckets / warp-tiles of ~7
    lookups (many buckets and tiles per table even at B = 64)."""
    return request.param


@pytest.mark.parametrize("dims", list(DIM_SETS))
@pytest.mark.parametrize("D", [1, 2])
def test_backward_matches_oracle(dims, D, sort_target):
    B = 64
    task, placement = random_task(19 + D, DIM_SETS[dims], D, B, rows_range=(1, 200))
    weights = random_weights(3, task.tables)
    off, idx = orc.synth_batch(as_dicts(task.tables), B, seed=9)
    W = sum(t.dim for t in task.tables)
    grad = np.random.default_rng(4).uniform(-1, 1, size=(B, W)).astype(np.float32)
    lr = 0.05
    sh = _shard(task, placement, weights, lr=lr)
    sh.set_sort_target(sort_target)
    sh.upload_batch(LookupBatch(idx, off, len(task.tables), B))
    sh.set_grad(grad)
    sh.a2a_backward()
    # sorted keys / bags / segment heads: bit-exact vs std::stable_sort
    rows = [t.hash_size for t in task.tables]
    for d in range(D):
        lst = [i for i in range(len(task.tables)) if placement[i] == d]
        k, b, h = sh.sorted(d)
        ok, ob, oh = orc.sorted_keys(rows, off, idx, B, lst)
        np.testing.assert_array_equal(k, ok)
        np.testing.assert_array_equal(b, ob)
        np.testing.assert_array_equal(h, oh)
    sh.backward_sgd()
    dims_l = [t.dim for t in task.tables]
    want = orc.tbe_backward_sgd(dims_l, rows, weights, off, idx, B, grad, lr,
                                list(range(len(task.tables))))
    for i in range(len(task.tables)):
        np.testing.assert_allclose(sh.get_table(i), want[i], rtol=RTOL, atol=ATOL)


def test_device_generator_matches_oracle(sort_target):
    """sp_synth_batch / sp_init_tables / sp_synth_grad are bit-identical to the
    oracle generator: same sorted keys, same pooled sums, same update."""
    B = 128
    task, placement = random_task(23, [16, 32, 64, 128, 8], 2, B, rows_range=(500, 5000))
    seed = 2210
    sh = EmbeddingShard(task, placement, lr=0.01)
    sh.set_sort_target(sort_target)
    sh.init_tables(seed)
    sh.synth_batch(seed)
    off, idx = orc.synth_batch(as_dicts(task.tables), B, seed)
    assert sh.nnz == len(idx)
    rows = [t.hash_size for t in task.tables]
    for d in range(2):
        lst = [i for i in range(len(task.tables)) if placement[i] == d]
        k, b, h = sh.sorted(d)
        ok, ob, oh = orc.sorted_keys(rows, off, idx, B, lst)
        np.testing.assert_array_equal(k, ok)
        np.testing.assert_array_equal(b, ob)
    for i, t in enumerate(task.tables):
        np.testing.assert_array_equal(sh.get_table(i), orc.weights(seed, i, t.hash_size, t.dim))
    sh.forward()
    sh.a2a_forward()
    want = orc.tbe_forward([t.dim for t in task.tables], rows, None, off, idx, B, wseed=seed)
    np.testing.assert_allclose(sh.pooled(), want, rtol=RTOL, atol=ATOL)


def test_run_iteration_composition():
    B = 256
    task, placement = random_task(31, [16, 32, 64, 128] * 3, 4, B, rows_range=(100, 20000))
    sh = EmbeddingShard(task, placement)
    sh.init_tables(1)
    sh.synth_batch(1)
    sh.synth_grad(1)
    bd = sh.run_iteration()
    assert len(bd.fwd_ms) == 4
    want = max(bd.fwd_ms) + bd.fwd_comm_stage_ms + bd.bwd_comm_stage_ms + max(bd.bwd_ms)
    assert abs(bd.overall_ms - want) < 1e-9
    assert all(x >= 0 for x in bd.fwd_ms + bd.bwd_ms + bd.comm_ms)
    ev = bd.events
    assert len(ev) == 16


def test_graph_replay_matches_eager():
    B = 128
    task, placement = random_task(41, [16, 64, 128, 32], 2, B, rows_range=(50, 400))
    outs = []
    for mode in ("eager", "graph"):
        sh = EmbeddingShard(task, placement, lr=0.02)
        sh.init_tables(3)
        sh.synth_batch(3)
        sh.synth_grad(3)
        if mode == "eager":
            for _ in range(3):
                sh.enqueue_iteration()
        else:
            k = sh.graph_replay(3)
            assert k >= 5
        outs.append([sh.get_table(i) for i in range(len(task.tables))])
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


def test_malformed_batches_rejected():
    tables = make_tables([16], [10], [1.0])
    task = PlacementTask(tables, 1, 0.0, 2)
    sh = EmbeddingShard(task, [0])
    with pytest.raises(ShardplanError) as e:
        sh.upload_batch(LookupBatch(np.array([1, 2]), np.array([0, 2, 1]), 1, 2))
    assert e.value.kind == "malformed_batch"
    with pytest.raises(ShardplanError) as e:
        sh.upload_batch(LookupBatch(np.array([1, 99]), np.array([0, 1, 2]), 1, 2))
    assert e.value.kind == "bad_input"
    with pytest.raises(ShardplanError) as e:
        sh.upload_batch(LookupBatch(np.array([1]), np.array([0, 1]), 1, 2))
    assert e.value.kind == "malformed_batch"


def test_memory_cap_enforced():
    tables = make_tables([16, 16], [1000, 1000], [1.0, 1.0])
    cap = tables[0].table_size_gb * 1.5
    task = PlacementTask(tables, 2, cap, 4)
    EmbeddingShard(task, [0, 1]).close()
    with pytest.raises(ShardplanError) as e:
        EmbeddingShard(task, [0, 0])
    assert e.value.kind == "memory_violation" and e.value.exit_code == 2


def test_hot_rows_and_empty_tables(sort_target):
    """All-hot table (long duplicate runs), a never-accessed table (pf 0)."""
    B = 512
    tables = make_tables([32, 16, 128], [5000, 300, 70], [20.0, 0.0, 3.0], hot=[1.0, 0.0, 0.9])
    task = PlacementTask(tables, 2, 0.0, B)
    placement = [0, 1, 0]
    weights = random_weights(8, tables)
    off, idx = orc.synth_batch(as_dicts(tables), B, seed=77)
    W = sum(t.dim for t in tables)
    grad = np.random.default_rng(2).uniform(-1, 1, size=(B, W)).astype(np.float32)
    sh = _shard(task, placement, weights, lr=0.001)
    sh.set_sort_target(sort_target)
    sh.upload_batch(LookupBatch(idx, off, 3, B))
    sh.forward()
    sh.a2a_forward()
    np.testing.assert_allclose(sh.pooled(), _oracle_pooled(task, weights, off, idx),
                               rtol=RTOL, atol=ATOL)
    sh.set_grad(grad)
    sh.a2a_backward()
    sh.backward_sgd()
    want = orc.tbe_backward_sgd([t.dim for t in tables], [t.hash_size for t in tables], weights,
                                off, idx, B, grad, 0.001, [0, 1, 2])
    for i in range(3):
        np.testing.assert_allclose(sh.get_table(i), want[i], rtol=RTOL, atol=1e-4)


def test_runs_spanning_many_sgd_tiles(sort_target):
    """Tables of 1-3 rows at B = 4096: every row's run covers thousands of
    sorted positions, i.e. dozens of segmented-SGD tiles (1024 positions),
    so the per-chunk partials and the cross-tile carries are all exercised;
    plus a 4-row fp32 table of dim 8 and a generic dim (12)."""
    B = 4096
    dims = [16, 64, 128, 8, 12]
    tables = make_tables(dims, [1, 2, 3, 4, 3], [8.0, 6.0, 5.0, 4.0, 3.0])
    task = PlacementTask(tables, 1, 0.0, B)
    weights = random_weights(9, tables)
    off, idx = orc.synth_batch(as_dicts(tables), B, seed=31)
    grad = np.random.default_rng(5).uniform(-1, 1, size=(B, sum(dims))).astype(np.float32)
    sh = _shard(task, [0] * len(dims), weights, lr=0.001)
    sh.set_sort_target(sort_target)
    sh.upload_batch(LookupBatch(idx, off, len(dims), B))
    sh.set_grad(grad)
    sh.run_iteration()
    want = orc.tbe_backward_sgd(dims, [t.hash_size for t in tables], weights, off, idx, B, grad,
                                0.001, list(range(len(dims))))
    for i in range(len(dims)):
        np.testing.assert_allclose(sh.get_table(i), want[i], rtol=RTOL, atol=1e-5)
    sh.close()


def _golden_cases():
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lookup_cases.json")
    with open(p) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda c: c["name"])
def test_golden_cases_bit_exact(case, sort_target):
    """K1, the K4a sort and the SGD against the hand-worked golden cases
    (tests/golden/gen_lookup_cases.py; integer data: exact)."""
    dims, rows, B = case["dims"], case["rows"], case["B"]
    placement = case["placement"]
    D = max(placement) + 1
    tables = make_tables(dims, rows, [1.0] * len(dims))
    task = PlacementTask(tables, D, 0.0, B)
    w = [np.array(x, dtype=np.float32).reshape(r, d) for x, r, d in
         zip(case["weights"], rows, dims)]
    sh = _shard(task, placement, w, lr=case["lr"])
    sh.set_sort_target(sort_target)
    off = np.array(case["offsets"], dtype=np.int64)
    idx = np.array(case["indices"], dtype=np.int64)
    sh.upload_batch(LookupBatch(idx, off, len(dims), B))
    sh.forward()
    sh.a2a_forward()
    np.testing.assert_array_equal(sh.pooled(), np.array(case["pooled"], dtype=np.float32))
    for d, want in enumerate(case["sorted"]):
        k, b, h = sh.sorted(d)
        assert k.tolist() == want["keys"] and b.tolist() == want["bags"]
        assert h.tolist() == want["heads"]
    sh.set_grad(np.array(case["grad"], dtype=np.float32))
    sh.a2a_backward()
    sh.backward_sgd()
    for t, (x, r, d) in enumerate(zip(case["updated"], rows, dims)):
        np.testing.assert_array_equal(sh.get_table(t),
                                      np.array(x, dtype=np.float32).reshape(r, d))
    sh.close()
