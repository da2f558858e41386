"""bench.py's host-side contract (CPU): both arms describe the same config
for every N, `python bench.py --gpus N` self-launches N ranks, and the CPU
iteration the reference arm times is the oracle's arithmetic with the
exchange as a pure re-layout."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


@pytest.mark.parametrize("gpus", [1, 2, 4, 8])
def test_arms_share_config(gpus):
    """run_ours sizes the task by the world (= --gpus, enforced by
    dist_setup); run_reference by --gpus: the config objects are equal."""
    args = bench.parse_args(["--gpus", str(gpus)])
    ours = bench.config_dict(args, bench.load_task(args.config, gpus))
    ref_args = bench.parse_args(["--gpus", str(gpus), "--impl", "reference"])
    ref = bench.config_dict(ref_args, bench.load_task(ref_args.config, ref_args.gpus))
    assert ours == ref
    assert ours["devices"] == gpus


def test_world_must_match_gpus(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit):
        bench.dist_setup(bench.parse_args(["--gpus", "4"]))


def test_self_launch_reaches_world_2():
    """`python bench.py --gpus 2` with no WORLD_SIZE re-runs itself under
    torch.distributed.run; --dry-dist stops each rank after the rendezvous."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-dist"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert sorted(x["rank"] for x in lines) == [0, 1]
    assert all(x["world"] == 2 for x in lines)


def test_cpu_iteration_exchange_is_a_relayout():
    """The D > 1 CPU step: the backward all-to-all hands every owner exactly
    the gradient columns of its tables (the mirror of the forward re-layout),
    so the SGD result equals the D = 1 step's."""
    from paper_2210_02023_b200.api import PlacementTask, TableDesc
    dims = [8, 16, 4, 8]
    tabs = [TableDesc(i, d, 50 + 10 * i, 3.0, 0.0, [0.5] + [0.0] * 11 + [0.5] + [0.0] * 4)
            for i, d in enumerate(dims)]
    res = []
    for D, pl in ((1, [0, 0, 0, 0]), (2, [1, 0, 1, 0])):
        it = bench.CpuIteration(PlacementTask(tabs, D, 0.0, 64), pl)
        it.step(1)
        res.append([w.copy() for w in it.weights])
    for a, b in zip(*res):
        np.testing.assert_array_equal(a, b)


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref",
                                                    "libshardplan_ref.so")),
                    reason="the reference build (oracle/_ref) places the reference arm's tables")
def test_reference_arm_two_ranks_prints_one_line():
    """`bench.py --impl reference --gpus 2` (self-launched as two ranks, as the
    driver's torchrun would): rank 0 alone times the full-batch CPU iteration
    at D = 2 and prints one JSON line; the other rank exits 0 without work."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--config", "cfg1", "--steps", "2", "--warmup", "3",
                          "--no-cpu-single"], capture_output=True, text=True, timeout=600,
                         env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["devices"] == 2 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0


def _mode_worker(rank, world, port, fail_rank, q):
    """One rank of make_rank_shard with a stand-in shard (no GPU): rank
    `fail_rank` cannot map its peers."""
    import traceback
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2210_02023_b200 import api
        built = []

        class FakeShard:
            def __init__(self, task, placement, **kw):
                self.kw, self.closed, self.peer = kw, False, False
                built.append(self)

            def ipc_export(self):
                return bytes([self.kw["rank"]]) * 4

            def ipc_import(self, handles):
                assert [h[0] for h in handles] == list(range(world))
                if self.kw["rank"] == fail_rank:
                    raise api.ShardplanError(4, "no peer access")
                self.peer = True

            def close(self):
                self.closed = True

        api.EmbeddingShard = FakeShard
        api.nccl_unique_id = lambda: b"id"
        args = bench.parse_args(["--gpus", str(world)])
        shard, mode = bench.make_rank_shard(args, None, None, world, rank, rank)
        q.put((rank, mode, len(built), built[0].closed, shard.peer))
        dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        q.put((rank, traceback.format_exc(), 0, False, False))


@pytest.mark.parametrize("fail_rank", [-1, 1])
def test_exchange_mode_agreed_over_ranks(fail_rank):
    """--exchange peer (the N > 1 default): every rank maps the others'
    buffers; if any rank cannot, all ranks rebuild NCCL-only (mixed modes
    would deadlock the barriers)."""
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_mode_worker, args=(r, 2, port, fail_rank, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for rank, mode, n_built, first_closed, peer in out:
        if fail_rank < 0:
            assert (mode, n_built, first_closed, peer) == ("nccl+peer", 1, False, True), out
        else:
            assert mode.startswith("nccl (peer mapping failed)"), out
            assert (n_built, first_closed, peer) == (2, True, False), out
