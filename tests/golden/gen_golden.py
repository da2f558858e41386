"""Generates the committed fixtures from the REFERENCE ITSELF (oracle/_ref).

Run here (where /root/reference exists), never on the GPU box:

    make -C oracle all ref
    python tests/golden/gen_golden.py pools        # workload pools (JSON)
    python tests/golden/gen_golden.py checkpoints  # DreamShard checkpoints (minutes)
    python tests/golden/gen_golden.py golden       # reference outputs for tests

Outputs
  paper_2210_02023_b200/data/pools.json   table descriptors of cfg1-cfg4 and
      the training pool, from synth_pool (synth.hpp:72-119, bytes_per_param 4,
      SURVEY §8d); cfg1 overrides pooling_factor to 8 as BASELINE.json says.
  paper_2210_02023_b200/data/*.dshd       checkpoints from train() (harness.hpp:220,
      RunConfig defaults config.hpp:19-39) saved with save_checkpoint
      (checkpoint.hpp:114).
  tests/golden/ref_*.npz / *.json         reference answers used by the tests.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

DATA = os.path.join(ROOT, "paper_2210_02023_b200", "data")
GOLD = os.path.join(ROOT, "tests", "golden")

MIXED_DIMS = [(16, 1.0), (32, 1.0), (64, 1.0), (128, 1.0)]

# name -> (num_tables, dim_choices, hash_log10, D, B, mem_cap_gb, seed, pf override)
POOLS = {
    "cfg1": (10, [(16, 1.0)], (5.0, 5.0), 2, 512, 64.0, 2210, 8.0),
    "cfg2": (50, [(16, 1.0)], (5.0, 6.0), 4, 65536, 64.0, 2210, None),
    "cfg3": (100, MIXED_DIMS, (5.0, 6.0), 8, 65536, 64.0, 2210, None),
    "cfg4": (200, MIXED_DIMS, (7.0, 7.0), 8, 65536, 64.0, 2210, None),
    "train": (856, MIXED_DIMS, (5.0, 6.0), 4, 65536, 64.0, 1, None),
}

CHECKPOINTS = {
    # file: (num_tables per task, num_devices, seed)
    "dreamshard_m50_d4.dshd": (50, 4, 1),
    "dreamshard_m100_d8.dshd": (100, 8, 1),
}


def make_pools():
    os.makedirs(DATA, exist_ok=True)
    out = {}
    for name, (n, dims, hr, D, B, cap, seed, pf) in POOLS.items():
        tables, mean, std = ref.synth_pool(n, dims, hash_log10=hr, batch=B,
                                           bytes_per_param=4, seed=seed)
        if pf is not None:
            for t in tables:
                t["pooling_factor"] = pf
        out[name] = {"num_devices": D, "batch_size": B, "mem_cap_gb": cap,
                     "bytes_per_param": 4, "seed": seed, "tables": tables,
                     "feature_mean": mean.tolist(), "feature_std": std.tolist()}
    with open(os.path.join(DATA, "pools.json"), "w") as f:
        json.dump(out, f)
    print("pools ->", os.path.join(DATA, "pools.json"))


def load_pools():
    with open(os.path.join(DATA, "pools.json")) as f:
        return json.load(f)


def make_checkpoints(which=None):
    pools = load_pools()
    train_pool = pools["train"]
    for fname, (m, d, seed) in CHECKPOINTS.items():
        if which and fname != which:
            continue
        path = os.path.join(DATA, fname)
        t0 = time.time()
        ref.train(train_pool["tables"], train_pool["batch_size"], m, d, 64.0, path, seed=seed)
        print(f"{fname}: trained in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    stage = sys.argv[1] if len(sys.argv) > 1 else "all"
    if stage in ("pools", "all"):
        make_pools()
    if stage in ("checkpoints", "all"):
        make_checkpoints(sys.argv[2] if len(sys.argv) > 2 else None)
    if stage in ("golden", "all"):
        from gen_golden_outputs import make_golden  # noqa: E402
        make_golden(load_pools())
