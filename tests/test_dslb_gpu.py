"""The DSLB loader straight to device (SURVEY §8f row 2, table.hpp:283-305):
sp_upload_batch_file and sp_ingest_batch_file against the reference's own
file and answers (tests/golden/ref_batch.dslb + ref_dslb.json, written by
the reference's save_lookup_batch / ingest_lookup_batch), and against the
host-buffer paths on the same batch: identical device CSR (sorted pairs,
pooled rows, updated tables), for emulated multi-device placements, a rank
context that reads only its own tables, bad data, and cfg3 at full size."""
import json
import os
import time

import numpy as np
import pytest

from oracle import lookup as orc
from paper_2210_02023_b200.api import (EmbeddingShard, LookupBatch, PlacementTask,
                                       ShardplanError, TableDesc, ingest_batch_file,
                                       ingest_lookup_batch, load_lookup_batch,
                                       save_lookup_batch, synth_lookup_batch)
from tests.helpers import as_dicts, random_task, random_weights

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ingest_file_matches_reference_golden():
    with open(os.path.join(GOLD, "ref_dslb.json")) as f:
        g = json.load(f)
    path = os.path.join(GOLD, "ref_batch.dslb")
    tables, mean, std, B = ingest_batch_file(path, g["dims"], g["hash_sizes"],
                                             g["bytes_per_param"])
    assert B == g["batch_size"] and len(tables) == g["num_tables"]
    for t, want in zip(tables, g["ingest"]):
        assert t.pooling_factor == want["pooling_factor"]      # bit-exact
        assert t.table_size_gb == want["table_size_gb"]
        assert list(t.dist) == want["dist"]
    assert list(mean) == g["feature_mean"] and list(std) == g["feature_std"]
    # and the same as the host-buffer ingest of the host-loaded batch
    t2, _, _ = ingest_lookup_batch(load_lookup_batch(path), g["dims"], g["hash_sizes"],
                                   g["bytes_per_param"])
    assert [list(t.dist) for t in t2] == [list(t.dist) for t in tables]


def _shard(task, placement, weights, lr):
    sh = EmbeddingShard(task, placement, lr=lr)
    for i, w in enumerate(weights):
        sh.set_table(i, w)
    return sh


@pytest.mark.parametrize("D", [1, 3])
def test_upload_file_equals_upload_batch(tmp_path, D):
    B = 96
    dims = [16, 32, 64, 128, 16, 64, 12, 4]
    task, placement = random_task(50 + D, dims, D, B)
    weights = random_weights(8, task.tables)
    off, idx = orc.synth_batch(as_dicts(task.tables), B, seed=11)
    path = str(tmp_path / "b.dslb")
    save_lookup_batch(LookupBatch(idx, off, len(dims), B), path)
    grad = np.random.default_rng(2).uniform(-1, 1, size=(B, sum(dims))).astype(np.float32)
    a = _shard(task, placement, weights, 0.03)
    b = _shard(task, placement, weights, 0.03)
    a.set_upload_chunk(500)  # many chunks / ring refills
    a.upload_batch_file(path)
    b.upload_batch(LookupBatch(idx, off, len(dims), B))
    assert a.nnz == b.nnz == len(idx)
    for sh in (a, b):
        sh.forward()
        sh.a2a_forward()
    np.testing.assert_array_equal(a.pooled(), b.pooled())
    for dev in range(D):
        for x, y in zip(a.sorted(dev), b.sorted(dev)):
            np.testing.assert_array_equal(x, y)
    for sh in (a, b):
        sh.set_grad(grad)
        sh.a2a_backward()
        sh.backward_sgd()
    for i in range(len(dims)):
        np.testing.assert_array_equal(a.get_table(i), b.get_table(i))
    # a second file on the same context (ring and offset buffers reused)
    off2, idx2 = orc.synth_batch(as_dicts(task.tables), B, seed=12)
    save_lookup_batch(LookupBatch(idx2, off2, len(dims), B), path)
    a.upload_batch_file(path)
    assert a.nnz == len(idx2)
    a.close()
    b.close()


def test_rank_context_reads_its_own_tables(tmp_path):
    B = 64
    dims = [16, 32, 64, 128, 16, 8]
    task, placement = random_task(9, dims, 2, B)
    placement = np.array([0, 1, 1, 0, 1, 0], dtype=np.int32)
    off, idx = orc.synth_batch(as_dicts(task.tables), B, seed=5)
    path = str(tmp_path / "b.dslb")
    save_lookup_batch(LookupBatch(idx, off, len(dims), B), path)
    for rank in (0, 1):
        a = EmbeddingShard(task, placement, lr=0.01, rank=rank, world_size=2, nccl_id=None)
        b = EmbeddingShard(task, placement, lr=0.01, rank=rank, world_size=2, nccl_id=None)
        a.init_tables(3)
        b.init_tables(3)
        a.upload_batch_file(path)
        b.upload_batch(LookupBatch(idx, off, len(dims), B))
        local = [t for t in range(len(dims)) if placement[t] == rank]
        assert a.local_tables() == local
        assert a.nnz == b.nnz == sum(int(off[(t + 1) * B] - off[t * B]) for t in local)
        for x, y in zip(a.sorted(rank), b.sorted(rank)):
            np.testing.assert_array_equal(x, y)
        a.close()
        b.close()


def test_bad_file_data_raises_like_upload_batch(tmp_path):
    B = 64
    dims = [16, 64, 32]
    task, placement = random_task(5, dims, 1, B)
    weights = random_weights(3, task.tables)
    off, idx = orc.synth_batch(as_dicts(task.tables), B, seed=2)
    sh = _shard(task, placement, weights, 0.1)
    bad = idx.copy()
    bad[len(bad) // 2] = task.tables[1].hash_size + 5
    path = str(tmp_path / "bad.dslb")
    save_lookup_batch(LookupBatch(bad, off, 3, B), path)
    with pytest.raises(ShardplanError) as e:
        sh.upload_batch_file(path)
    assert e.value.kind == "bad_input"
    with pytest.raises(ShardplanError):  # no batch is current after the failure
        sh.run_iteration()
    # shape from another task
    other = str(tmp_path / "other.dslb")
    save_lookup_batch(LookupBatch(idx, off, 3, B), other)
    with open(other, "r+b") as f:  # rewrite batch_size: 64 -> 32 (offsets length now wrong)
        f.seek(12)
        f.write(np.array([32], "<u4").tobytes())
    with pytest.raises(ShardplanError) as e:
        sh.upload_batch_file(other)
    assert e.value.kind == "malformed_batch"
    small = str(tmp_path / "small.dslb")
    off_s, idx_s = orc.synth_batch(as_dicts(task.tables), 32, seed=2)
    save_lookup_batch(LookupBatch(idx_s, off_s, 3, 32), small)
    with pytest.raises(ShardplanError) as e:
        sh.upload_batch_file(small)
    assert e.value.kind == "shape_mismatch"
    with pytest.raises(ShardplanError) as e:
        sh.upload_batch_file(str(tmp_path / "missing.dslb"))
    assert e.value.kind == "bad_input"
    # a good file afterwards works and nothing was updated before
    save_lookup_batch(LookupBatch(idx, off, 3, B), path)
    sh.upload_batch_file(path)
    for i in range(3):
        np.testing.assert_array_equal(sh.get_table(i), weights[i])
    sh.close()


def test_fullsize_cfg3_file(tmp_path):
    """cfg3 (100 tables, B = 65536, 45 M lookups, a 400 MB file): the batch
    loaded from its DSLB file gives the same device sort as the device
    generator's batch, bit for bit; prints the file -> device rate."""
    with open(os.path.join(ROOT, "paper_2210_02023_b200", "data", "pools.json")) as f:
        pool = json.load(f)["cfg3"]
    tables = [TableDesc.from_dict(t) for t in pool["tables"]]
    B = int(pool["batch_size"])
    task = PlacementTask(tables, 1, 0.0, B)
    b, _ = synth_lookup_batch(tables, B, 2210)
    path = str(tmp_path / "cfg3.dslb")
    save_lookup_batch(b, path)
    size = os.path.getsize(path)
    del b
    a = EmbeddingShard(task, np.zeros(len(tables), dtype=np.int32), lr=0.01)
    ref = EmbeddingShard(task, np.zeros(len(tables), dtype=np.int32), lr=0.01)
    a.upload_batch_file(path)  # warm (ring allocation, page cache)
    t0 = time.perf_counter()
    a.upload_batch_file(path)
    dt = time.perf_counter() - t0
    print(f"\ncfg3 DSLB file {size / 1e6:.0f} MB -> device in {dt * 1e3:.1f} ms "
          f"({size / dt / 1e9:.1f} GB/s)")
    ref.synth_batch(2210)
    assert a.nnz == ref.nnz
    for x, y in zip(a.sorted(0), ref.sorted(0)):
        np.testing.assert_array_equal(x, y)
    a.close()
    ref.close()
