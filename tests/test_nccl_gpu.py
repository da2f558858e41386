"""The multi-GPU exchange with one process per GPU: NCCL grouped
send/recv all-to-all (ctx.cu a2a_fwd_rank / a2a_bwd_rank), its device-side
barriers, the breakdown AllGather, and the NCCL + peer-memory mode (K1
stores pooled rows straight into the receivers' buffers over NVLink, the
backward pulls gradient slices from the peers, NCCL barriers order them).
A whole on-device iteration (sp_run_iteration) per rank, checked against
the CPU oracle: each rank's received pooled slice, its updated tables, and
the breakdown's composition (oracle.hpp:222-227).

The iterations need >= 2 GPUs (NCCL refuses two ranks on one device) and
skip otherwise — the peer path alone is covered on one GPU by
tests/test_peer_gpu.py and the exchange plan by tests/test_dist_cpu.py. On
one GPU, test_nccl_binding_reaches_comm_init still drives the NCCL binding
up to ncclCommInitRank and checks its refusal comes back as an error."""
import os
import socket
import traceback

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
needs_two = pytest.mark.skipif(torch.cuda.device_count() < 2,
                               reason="NCCL exchange needs >= 2 GPUs")

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


@needs_two
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


def _dup_worker(rank, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=2)
        from paper_2210_02023_b200 import api
        from paper_2210_02023_b200.api import EmbeddingShard, ShardplanError
        task, placement, _ = _case("random", 2)
        obj = [api.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        try:
            EmbeddingShard(task, placement, rank=rank, world_size=2, nccl_id=obj[0], device=0)
            q.put((rank, "created"))
        except ShardplanError as e:
            q.put((rank, f"{e.kind}: {e}"))
        dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        q.put((rank, traceback.format_exc()))


def test_nccl_binding_reaches_comm_init():
    """On any box: the run-time NCCL binding (csrc/nccl_loader.h, bound to the
    NCCL already in the process) creates a unique id and reaches
    ncclCommInitRank; two ranks on one device are refused by NCCL
    ("Duplicate GPU"), and the refusal comes back as a ShardplanError of
    kind nccl, not a crash."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dup_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(2):
            r, msg = q.get(timeout=300)
            results[r] = msg
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(2):
        assert "invalid usage" in results.get(r, ""), results.get(r)
        assert results[r].startswith("nccl"), results[r]
