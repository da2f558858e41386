"""DreamShard on B200-measured costs, end to end (first row).

1. trains the reference's DreamShard (tools/_bin/train_measured: the
   reference's training loop with every collect-phase cost measured on the
   GPU by MeasuredCostProvider) on the synthetic training pool;
2. places the evaluation tasks with it, with the checkpoint the reference's
   own train() produced on its synthetic oracle, and with the baselines;
3. measures every placement on the GPU (all devices emulated on one B200:
   max-over-device fwd + bwd compute, median of 5).

    python tools/measured_dreamshard.py [--iterations N] [--out DIR]
Prints one JSON object (also written to DIR/measured_dreamshard.json).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2210_02023_b200 import api  # noqa: E402

DATA = os.path.join(ROOT, "paper_2210_02023_b200", "data")
TOOL = os.path.join(ROOT, "tools", "_bin", "train_measured")


def load(config, D):
    with open(os.path.join(DATA, "pools.json")) as f:
        pool = json.load(f)[config]
    tables = [api.TableDesc.from_dict(t) for t in pool["tables"]]
    return api.PlacementTask(tables, D, float(pool["mem_cap_gb"]), int(pool["batch_size"])), pool


def measure(task, placement, device=0):
    """(max-over-device fwd + bwd compute, the metric with the exchange
    stages from the NVLink 5 model): median of 5 after one warm-up."""
    sh = api.EmbeddingShard(task, placement, lr=0.01, device=device)
    sh.set_comm_model(True)
    sh.init_tables(2210)
    sh.synth_batch(2210)
    sh.synth_grad(2210)
    runs = sorted((sh.run_iteration() for _ in range(6)), key=lambda b: b.overall_ms)[1:]
    bd = runs[2]
    sh.close()
    return {"compute_ms": round(max(bd.fwd_ms) + max(bd.bwd_ms), 4),
            "overall_ms": round(bd.overall_ms, 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iterations", type=int, default=10)
    ap.add_argument("--tables", type=int, default=50)
    ap.add_argument("--devices", type=int, default=4)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out"))
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    _, train_pool = load("train", 1)
    specs = api._specs([api.TableDesc.from_dict(t) for t in train_pool["tables"]])
    pool_bin = os.path.join(args.out, "pool_train.bin")
    with open(pool_bin, "wb") as f:
        f.write(bytes(specs))
    ckpt = os.path.join(args.out, f"dreamshard_measured_m{args.tables}_d{args.devices}.dshd")
    t0 = time.time()
    r = subprocess.run([TOOL, pool_bin, str(train_pool["batch_size"]), str(args.tables),
                        str(args.devices), str(train_pool["mem_cap_gb"]), str(args.iterations),
                        ckpt], capture_output=True, text=True)
    train_s = time.time() - t0
    if r.returncode != 0:
        raise SystemExit(f"train_measured failed: {r.stderr[-2000:]}")
    metrics = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    oracle_ckpt = os.path.join(DATA, f"dreamshard_m{args.tables}_d{args.devices}.dshd")
    if not os.path.exists(oracle_ckpt):
        oracle_ckpt = os.path.join(DATA, "dreamshard_m50_d4.dshd")
    models = {"dreamshard_oracle": api.load_checkpoint(oracle_ckpt),
              "dreamshard_measured": api.load_checkpoint(ckpt)}
    results = {}
    for cfg, D in (("cfg2", 4), ("cfg3", 4), ("cfg3", 8)):
        task, _ = load(cfg, D)
        row = {}
        for name, ck in models.items():
            p, _ = api.infer(ck, task)
            row[name] = measure(task, p)
        row["random"] = measure(task, api.random_placement(task, 2210))
        for how in ("size", "lookup"):
            row[how] = measure(task, api.expert_placement(task, how))
        results[f"{cfg}_d{D}"] = row
    out = {"train_seconds": round(train_s, 1), "iterations": args.iterations,
           "train_tables": args.tables, "train_devices": args.devices,
           "oracle_checkpoint": os.path.basename(oracle_ckpt),
           "train_metrics": metrics, "placements": results,
           "note": "placements measured on one B200 with every device emulated: compute_ms = "
                   "max over devices of the measured fwd + bwd compute; overall_ms = that plus "
                   "the two all-to-all stages from the NVLink 5 model (sp_comm_model: 770 GB/s "
                   "per direction + 10 us; a model, not a measurement), median of 5. The "
                   "measured checkpoint is trained with the same comm term "
                   "(MeasuredCostProvider comm_model)"}
    name = f"measured_dreamshard_m{args.tables}_d{args.devices}.json"
    with open(os.path.join(args.out, name), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
