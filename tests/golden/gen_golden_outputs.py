"""Reference answers for the evaluator / ingest / placement tests, produced by
the UNMODIFIED reference (oracle/_ref/libshardplan_ref.so). Called from
gen_golden.py (`python tests/golden/gen_golden.py golden`)."""
from __future__ import annotations

import json
import os

import numpy as np

from oracle import ref

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DATA = os.path.join(ROOT, "paper_2210_02023_b200", "data")

# (name, pool, checkpoint, table subset (None = all), D, cap, n_random, n_sampled)
EVAL_CASES = [
    ("cfg1", "cfg1", "dreamshard_m50_d4.dshd", None, 2, 64.0, 64, 16),
    ("cfg2", "cfg2", "dreamshard_m50_d4.dshd", None, 4, 64.0, 64, 16),
    ("cfg3", "cfg3", "dreamshard_m100_d8.dshd", None, 8, 64.0, 64, 8),
    ("cfg3_d4", "cfg3", "dreamshard_m50_d4.dshd", None, 4, 64.0, 32, 8),
    # capacity-bound: caps at 1.3x the balanced share force legality masks
    ("cfg3_cap", "cfg3", "dreamshard_m100_d8.dshd", None, 8, "tight", 32, 8),
    ("sweep_m20_d1", "train", "dreamshard_m50_d4.dshd", 20, 1, 64.0, 16, 4),
    ("sweep_m20_d2", "train", "dreamshard_m50_d4.dshd", 20, 2, 64.0, 16, 4),
    ("sweep_m60_d8", "train", "dreamshard_m50_d4.dshd", 60, 8, 64.0, 16, 4),
    ("sweep_m200_d8", "train", "dreamshard_m100_d8.dshd", 200, 8, 64.0, 16, 4),
]


def _tables(pools, pool, subset, seed=7):
    tables = pools[pool]["tables"]
    if subset is not None:
        rng = np.random.default_rng(seed + subset)
        ids = np.sort(rng.choice(len(tables), size=subset, replace=False))
        tables = [dict(tables[i], id=k) for k, i in enumerate(ids)]
    return tables


def make_eval_golden(pools):
    out = {}
    for name, pool, ck, subset, D, cap, n_rand, n_samp in EVAL_CASES:
        tables = _tables(pools, pool, subset)
        M = len(tables)
        if cap == "tight":
            cap = 1.3 * sum(t["table_size_gb"] for t in tables) / D
        ckpt = os.path.join(DATA, ck)
        B = pools[pool]["batch_size"]
        placement, pred, order = ref.infer(ckpt, tables, D, cap, B)
        rng = np.random.default_rng(1234)
        rand = np.stack([ref.random_placement(tables, D, cap, B, int(rng.integers(1 << 62)))
                         for _ in range(n_rand)])
        overall, q = ref.costnet_overall(ckpt, tables, D, rand)
        seed = 99
        sp, so = ref.sampled_rollouts(ckpt, tables, D, cap, B, seed, n_samp)
        uniforms = ref.rng_u01(seed, n_samp * M).reshape(n_samp, M)
        rows, single = ref.task_features(ckpt, tables)
        out[name] = {
            "pool": pool, "checkpoint": ck, "subset": subset, "D": D, "cap": cap, "B": B,
            "tables": tables, "infer_placement": placement.tolist(), "infer_predicted": pred,
            "order": order.tolist(), "random_placements": rand.tolist(),
            "random_overall": overall.tolist(), "random_q": q.tolist(),
            "sampled_placements": sp.tolist(), "sampled_overall": so.tolist(),
            "uniforms": uniforms.tolist(), "feature_rows": rows.tolist(),
            "single_cost": single.tolist(),
        }
    with open(os.path.join(HERE, "ref_evaluator.json"), "w") as f:
        json.dump(out, f)
    print("golden evaluator cases:", list(out))


def make_ingest_golden():
    cases = {}
    # SPEC.md:51-53 worked examples
    cases["spec_one_hot"] = {"offsets": [0, 1, 2, 3, 4], "indices": [7, 7, 7, 7], "T": 1, "B": 4,
                             "dims": [16], "hash": [10]}
    cases["spec_empty"] = {"offsets": [0, 0, 0, 0, 0], "indices": [], "T": 1, "B": 4,
                           "dims": [16], "hash": [10]}
    cases["spec_two_tables"] = {"offsets": [0, 2, 4, 5, 6], "indices": [1, 2, 3, 4, 9, 9],
                                "T": 2, "B": 2, "dims": [16, 32], "hash": [10, 10]}
    # a random multi-table batch with hot rows (counts spanning many bins)
    rng = np.random.default_rng(5)
    T, B = 6, 500
    lens = rng.integers(0, 40, size=T * B)
    offsets = np.concatenate([[0], np.cumsum(lens)])
    hs = [50, 1000, 100000, 7, 3000, 1 << 20]
    idx = []
    for t in range(T):
        n = int(lens[t * B:(t + 1) * B].sum())
        hot = rng.integers(0, min(hs[t], 8), size=n)
        cold = rng.integers(0, hs[t], size=n)
        idx.append(np.where(rng.random(n) < 0.6, hot, cold))
    cases["random_hot"] = {"offsets": offsets.tolist(), "indices": np.concatenate(idx).tolist(),
                           "T": T, "B": B, "dims": [4, 8, 16, 32, 64, 128], "hash": hs}
    for name, c in cases.items():
        tables, mean, std = ref.ingest(c["offsets"], c["indices"], c["T"], c["B"], c["dims"],
                                       c["hash"], bytes_per_param=2)
        c["expected_tables"] = tables
        c["expected_mean"] = mean.tolist()
        c["expected_std"] = std.tolist()
    with open(os.path.join(HERE, "ref_ingest.json"), "w") as f:
        json.dump(cases, f)
    print("golden ingest cases:", list(cases))


def make_oracle_golden(pools):
    """Known answers of the reference's cost model and placements."""
    out = {"device_comm": [[256, 4, 65536, ref.lib().ref_device_comm(256, 4, 65536)],
                           [832, 4, 65536, ref.lib().ref_device_comm(832, 4, 65536)]],
           "fusion_speedup": [[k, ref.lib().ref_fusion_speedup(k)] for k in (1, 2, 10, 200)]}
    expert = {}
    for cfg in ("cfg2", "cfg3", "cfg4"):
        p = pools[cfg]
        for s in ref.EXPERT:
            expert[f"{cfg}/{s}"] = ref.expert_placement(p["tables"], p["num_devices"],
                                                        p["mem_cap_gb"], p["batch_size"],
                                                        s).tolist()
    out["expert"] = expert
    ev = {}
    for cfg in ("cfg2", "cfg3"):
        p = pools[cfg]
        pl = np.array(expert[f"{cfg}/lookup"])
        ev[cfg] = ref.evaluate_placement(p["tables"], p["num_devices"], p["mem_cap_gb"],
                                         p["batch_size"], pl)
        ev[cfg] = {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in ev[cfg].items()}
    out["evaluate_lookup"] = ev
    with open(os.path.join(HERE, "ref_oracle.json"), "w") as f:
        json.dump(out, f)
    print("golden oracle answers written")


def make_golden(pools):
    make_oracle_golden(pools)
    make_ingest_golden()
    make_eval_golden(pools)
