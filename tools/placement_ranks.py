"""Placement study with every rank measured alone (sp_run_local): cfg3 on 8
GPUs, each rank's shard on this B200 in turn — its K1, the sort forked
after it, its SGD — for DreamShard (the reference's oracle-trained
m100_d8 checkpoint and the B200-measured one), random, and the greedy
size / lookup experts. Prints one JSON object: per placement the max-over-
rank forward, backward and their sum (the compute part of the metric).

    python tools/placement_ranks.py [--config cfg3] [--devices 8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2210_02023_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--devices", type=int, default=8)
    args = ap.parse_args()
    task = bench.load_task(args.config, args.devices)
    data = os.path.join(ROOT, "paper_2210_02023_b200", "data")
    placements = {}
    for name, ck in (("dreamshard_oracle", f"dreamshard_m100_d{args.devices}.dshd"),
                     ("dreamshard_measured", f"dreamshard_measured_m100_d{args.devices}.dshd")):
        path = os.path.join(data, ck)
        if os.path.exists(path):
            placements[name] = api.infer(api.load_checkpoint(path), task)[0]
    placements["random"] = api.random_placement(task, bench.SEED)
    for how in ("size", "lookup"):
        placements[how] = api.expert_placement(task, how)
    out = {}
    for name, p in placements.items():
        r = bench.bench_ranks(args.config, args.devices, 0, placement=p)
        out[name] = {"max_fwd_ms": r["max_fwd_ms"], "max_bwd_ms": r["max_bwd_ms"],
                     "compute_ms": round(r["max_fwd_ms"] + r["max_bwd_ms"], 4),
                     "overall_estimate_ms": r["overall_estimate"]["ms"],
                     "peer_fused_estimate_ms": r["overall_estimate"]["peer_fused_ms"],
                     "rank_compute_ms": [x["compute_ms"] for x in r["ranks"]]}
        print(name, out[name], flush=True)
    print(json.dumps({"config": args.config, "devices": args.devices, "placements": out}))


if __name__ == "__main__":
    main()
