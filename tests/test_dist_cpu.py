"""The N > 1 path's host logic on CPU: two gloo ranks execute the exact
exchange plan the NCCL path uses (sp_exchange_plan) on oracle-computed
pooled outputs / gradients, and the results must equal the single-process
oracle: pooled rows land on the right rank in global column order, and the
owner-side SGD with the returned gradients equals the global SGD."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lookup as orc
from paper_2210_02023_b200.api import exchange_plan
from tests.helpers import as_dicts, random_task, random_weights

WORLD = 2
B = 48


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange(sends, recv_sizes, rank, world):
    """Point-to-point all-to-all over gloo (isend/irecv pairs)."""
    recvs = [torch.empty(int(n), dtype=torch.float32) for n in recv_sizes]
    reqs = []
    for j in range(world):
        if j == rank:
            recvs[j].copy_(sends[j])
            continue
        reqs.append(dist.isend(sends[j], j))
        reqs.append(dist.irecv(recvs[j], j))
    for r in reqs:
        r.wait()
    return recvs


def _worker(rank, port, dims, seed, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        task, placement = random_task(seed, dims, WORLD, B, rows_range=(5, 300))
        placement[0], placement[1] = 0, 1  # both ranks own tables
        weights = random_weights(seed + 1, task.tables)
        tables = as_dicts(task.tables)
        off, idx = orc.synth_batch(tables, B, seed=seed + 2)
        tdims = [t.dim for t in task.tables]
        rows = [t.hash_size for t in task.tables]
        gcol = np.concatenate([[0], np.cumsum(tdims)])
        full = orc.tbe_forward(tdims, rows, weights, off, idx, B)  # [B, W_total]
        R = B // WORLD
        plan = exchange_plan(task, placement, rank)
        mine = [t for t in range(len(tables)) if placement[t] == rank]
        local_cols = np.concatenate([np.arange(gcol[t], gcol[t + 1]) for t in mine])
        pooled_local = np.ascontiguousarray(full[:, local_cols]).reshape(-1)

        # forward exchange
        sends = [torch.from_numpy(pooled_local[plan["send_off"][j]:plan["send_off"][j] +
                                               plan["send_count"][j]].copy())
                 for j in range(WORLD)]
        recvs = _exchange(sends, plan["recv_count"], rank, WORLD)
        grouped = torch.cat(recvs).numpy()
        assert len(grouped) == R * full.shape[1]
        got = np.zeros((R, full.shape[1]), dtype=np.float32)
        base = 0
        cm = plan["colmap"]
        c0 = 0
        for i in range(WORLD):
            Wi = int(plan["recv_count"][i] // R)
            blk = grouped[base:base + R * Wi].reshape(R, Wi)
            got[:, cm[c0:c0 + Wi]] = blk
            base += R * Wi
            c0 += Wi
        np.testing.assert_array_equal(got, full[rank * R:(rank + 1) * R])

        # backward exchange (mirror): every rank's gradient slice is drawn
        # from one global matrix so the oracle can apply the global SGD
        gfull = np.random.default_rng(seed + 3).uniform(-1, 1, size=full.shape).astype(np.float32)
        gslice = gfull[rank * R:(rank + 1) * R]
        gsend = []
        c0 = 0
        for j in range(WORLD):
            Wj = int(plan["recv_count"][j] // R)
            gsend.append(torch.from_numpy(np.ascontiguousarray(gslice[:, cm[c0:c0 + Wj]]).reshape(-1)))
            c0 += Wj
        grecv = _exchange(gsend, plan["send_count"], rank, WORLD)
        glocal = np.zeros(B * len(local_cols), dtype=np.float32)
        for j in range(WORLD):
            glocal[plan["send_off"][j]:plan["send_off"][j] + plan["send_count"][j]] = grecv[j].numpy()
        glocal = glocal.reshape(B, len(local_cols))
        np.testing.assert_array_equal(glocal, gfull[:, local_cols])

        # owner-side SGD with the returned gradient == global SGD
        lr = 0.03
        want = orc.tbe_backward_sgd(tdims, rows, weights, off, idx, B, gfull, lr, mine)
        # the same update from the rank-local view: local tables, local grad
        g_only = np.zeros_like(gfull)
        g_only[:, local_cols] = glocal
        got_w = orc.tbe_backward_sgd(tdims, rows, weights, off, idx, B, g_only, lr, mine)
        for t in mine:
            np.testing.assert_array_equal(got_w[t], want[t])
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced in the parent
        import traceback
        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")


@pytest.mark.parametrize("dims", [[16, 32, 64, 128, 16, 8], [4, 12, 256]])
def test_two_rank_exchange_plan(dims):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, dims, 17, errq)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    errors = []
    while not errq.empty():
        errors.append(errq.get())
    assert not errors, "\n".join(errors)
    assert all(p.exitcode == 0 for p in procs)


def test_plan_shapes():
    task, placement = random_task(3, [16, 32, 64], 4, 64)
    for r in range(4):
        p = exchange_plan(task, placement, r)
        W = sum(t.dim for t in task.tables)
        assert sorted(p["colmap"].tolist()) == list(range(W))
        assert p["recv_count"].sum() == (64 // 4) * W
        Wr = sum(t.dim for t, d in zip(task.tables, placement) if d == r)
        assert (p["send_count"] == (64 // 4) * Wr).all()
