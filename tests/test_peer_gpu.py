"""Peer-memory exchange (sp_ipc_export / sp_ipc_import): K1 stores every batch
slice's pooled rows straight into the receiving rank's buffer and the
backward pulls this rank's gradient slices from the peers. Two processes
share cuda:0 (CUDA IPC works between processes on one device), exchange
their IPC handles over gloo, and drive the stages from the host with rank
barriers in between (a peer-only context: no NCCL id). Checked against the
CPU oracle: each rank's received pooled slice and its updated tables."""
import os
import socket
import traceback

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WORLD = 2
B = 64
LR = 0.03


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(name="random"):
    from tests.helpers import random_task, random_weights
    if name == "cfg1":
        # BASELINE.json cfg1: 10 x dim 16, 1e5 rows, pf 8, D = 2, B = 512
        import json
        from paper_2210_02023_b200.api import PlacementTask, TableDesc
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        with open(os.path.join(root, "paper_2210_02023_b200", "data", "pools.json")) as f:
            pool = json.load(f)["cfg1"]
        tables = [TableDesc.from_dict(t) for t in pool["tables"]]
        task = PlacementTask(tables, WORLD, 0.0, int(pool["batch_size"]))
        placement = (np.arange(len(tables)) % WORLD).astype(np.int32)
        return task, placement, random_weights(17, task.tables)
    dims = [16, 64, 32, 128, 12, 16, 64]
    task, placement = random_task(101, dims, WORLD, B)
    placement[0], placement[1] = 0, 1  # both ranks own tables
    weights = random_weights(17, task.tables)
    return task, placement, weights


def _worker(rank, port, q, name="random"):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        from oracle import lookup as orc
        from paper_2210_02023_b200.api import EmbeddingShard, LookupBatch
        from tests.helpers import as_dicts
        task, placement, weights = _case(name)
        B = task.batch_size
        dims = [t.dim for t in task.tables]
        rows = [t.hash_size for t in task.tables]
        off, idx = orc.synth_batch(as_dicts(task.tables), B, seed=23)
        W = sum(dims)
        grad = np.random.default_rng(6).uniform(-1, 1, size=(B, W)).astype(np.float32)
        R = B // WORLD
        sh = EmbeddingShard(task, placement, lr=LR, rank=rank, world_size=WORLD,
                            nccl_id=None, device=0)
        local = sh.local_tables()
        for t in local:
            sh.set_table(t, weights[t])
        handles = [None] * WORLD
        dist.all_gather_object(handles, sh.ipc_export())
        sh.ipc_import(handles)
        sh.upload_batch(LookupBatch(idx, off, len(dims), B))
        dist.barrier()
        sh.forward()  # K1 stores the pooled rows at their receivers
        sh.synchronize()
        dist.barrier()
        sh.a2a_forward()  # no-op with peer memory
        want = orc.tbe_forward(dims, rows, weights, off, idx, B)
        np.testing.assert_allclose(sh.pooled(), want[rank * R:(rank + 1) * R], rtol=1e-5,
                                   atol=1e-5)
        sh.set_grad(grad[rank * R:(rank + 1) * R])
        sh.synchronize()
        dist.barrier()
        sh.a2a_backward()  # pull this rank's gradient slices from the peers
        sh.synchronize()
        dist.barrier()
        sh.backward_sgd()
        sh.synchronize()
        want_w = orc.tbe_backward_sgd(dims, rows, weights, off, idx, B, grad, LR,
                                      list(range(len(dims))))
        for t in local:
            np.testing.assert_allclose(sh.get_table(t), want_w[t], rtol=1e-5, atol=1e-5)
        # a whole on-device iteration needs device-side barriers (NCCL)
        try:
            sh.run_iteration()
            raise AssertionError("peer-only run_iteration should be rejected")
        except Exception as e:  # noqa: BLE001
            assert "peer-only" in str(e), e
        dist.barrier()
        sh.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException:  # noqa: BLE001
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("name", ["random", "cfg1"])
def test_peer_exchange_two_processes_one_gpu(name):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, name)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(WORLD):
            r, msg = q.get(timeout=240)
            results[r] = msg
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(WORLD):
        assert results.get(r) == "ok", results.get(r)
