"""The multi-GPU exchange with one process per GPU: NCCL grouped
send/recv all-to-all (ctx.cu a2a_fwd_rank / a2a_bwd_rank), its device-side
barriers, the breakdown AllGather, and the NCCL + peer-memory mode (K1
stores pooled rows straight into the receivers' buffers over NVLink, the
backward pulls gradient slices from the peers, NCCL barriers order them).
A whole on-device iteration (sp_run_iteration) per rank, checked against
the CPU oracle: each rank's received pooled slice, its updated tables, and
the breakdown's composition (oracle.hpp:222-227).

Needs >= 2 GPUs (NCCL refuses two ranks on one device); skipped otherwise —
the peer path alone is covered on one GPU by tests/test_peer_gpu.py and the
exchange plan by tests/test_dist_cpu.py."""
import os
import socket
import traceback

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2,
                                 reason="NCCL exchange needs >= 2 GPUs")]

LR = 0.03


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(name, world):
    from tests.helpers import random_task, random_weights
    if name == "random":
        B = 128 * world
        dims = [16, 64, 32, 128, 12, 16, 64, 8, 128, 32]
        task, placement = random_task(202 + world, dims, world, B)
        placement[:world] = np.arange(world)  # every rank owns a table
    else:  # cfg1 of BASELINE.json: 10 x dim 16, 1e5 rows, pf 8, B = 512
        import json
        from paper_2210_02023_b200.api import PlacementTask, TableDesc
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        with open(os.path.join(root, "paper_2210_02023_b200", "data", "pools.json")) as f:
            pool = json.load(f)["cfg1"]
        tables = [TableDesc.from_dict(t) for t in pool["tables"]]
        task = PlacementTask(tables, world, 0.0, int(pool["batch_size"]))
        placement = (np.arange(len(tables)) % world).astype(np.int32)
    weights = random_weights(29, task.tables)
    return task, placement, weights


def _worker(rank, world, port, name, peer, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import lookup as orc
        from paper_2210_02023_b200 import api
        from paper_2210_02023_b200.api import EmbeddingShard, LookupBatch
        from tests.helpers import as_dicts
        task, placement, weights = _case(name, world)
        B = task.batch_size
        dims = [t.dim for t in task.tables]
        rows = [t.hash_size for t in task.tables]
        off, idx = orc.synth_batch(as_dicts(task.tables), B, seed=37)
        W = sum(dims)
        grad = np.random.default_rng(8).uniform(-1, 1, size=(B, W)).astype(np.float32)
        R = B // world
        obj = [api.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        sh = EmbeddingShard(task, placement, lr=LR, rank=rank, world_size=world,
                            nccl_id=obj[0], device=rank)
        for t in sh.local_tables():
            sh.set_table(t, weights[t])
        if peer:
            handles = [None] * world
            dist.all_gather_object(handles, sh.ipc_export())
            sh.ipc_import(handles)
        sh.upload_batch(LookupBatch(idx, off, len(dims), B))
        sh.set_grad(grad[rank * R:(rank + 1) * R])
        bd = sh.run_iteration()
        assert len(bd.fwd_ms) == world and len(bd.bwd_ms) == world
        want_total = (max(bd.fwd_ms) + bd.fwd_comm_stage_ms + bd.bwd_comm_stage_ms +
                      max(bd.bwd_ms))
        assert abs(bd.overall_ms - want_total) < 1e-9
        want = orc.tbe_forward(dims, rows, weights, off, idx, B)
        np.testing.assert_allclose(sh.pooled(), want[rank * R:(rank + 1) * R], rtol=1e-5,
                                   atol=1e-5)
        want_w = orc.tbe_backward_sgd(dims, rows, weights, off, idx, B, grad, LR,
                                      list(range(len(dims))))
        for t in sh.local_tables():
            np.testing.assert_allclose(sh.get_table(t), want_w[t], rtol=1e-5, atol=1e-5)
        # every rank sees the same breakdown (the AllGather)
        got = [None] * world
        dist.all_gather_object(got, (bd.fwd_ms, bd.bwd_ms, bd.overall_ms))
        assert all(g == got[0] for g in got)
        dist.barrier()
        sh.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException:  # noqa: BLE001
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("peer", [False, True], ids=["nccl", "nccl+peer"])
@pytest.mark.parametrize("name", ["random", "cfg1"])
def test_nccl_exchange_iteration(name, peer):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, peer, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(world):
            r, msg = q.get(timeout=300)
            results[r] = msg
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert results.get(r) == "ok", results.get(r)
