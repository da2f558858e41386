"""Writes a DSLB lookup-batch fixture WITH THE REFERENCE ITSELF and records
the reference's ingest of it (run here, where oracle/_ref is built):

    make -C oracle all ref && python tests/golden/gen_golden_dslb.py

Outputs
  tests/golden/ref_batch.dslb   save_lookup_batch (table.hpp:268-281) of a
      6-table, B = 64 batch from the SURVEY §8d generator (seed 7).
  tests/golden/ref_dslb.json    the batch's shape, a checksum of its arrays,
      and ingest_lookup_batch(load_lookup_batch(file)) (table.hpp:188-305)
      by the reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import lookup as orc  # noqa: E402
from oracle import ref  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
DIMS = [16, 32, 64, 128, 16, 8]
ROWS = [300, 1000, 200, 500, 50, 64]
PFS = [4.0, 2.5, 6.0, 3.0, 10.0, 1.0]
B = 64
SEED = 7


def tables():
    out = []
    for i, (d, r, pf) in enumerate(zip(DIMS, ROWS, PFS)):
        dist = [0.0] * 17
        dist[0], dist[1], dist[2], dist[12] = 0.35, 0.21, 0.14, 0.3
        out.append({"id": i, "dim": d, "hash_size": r, "pooling_factor": pf,
                    "table_size_gb": r * d * 4 / 2 ** 30, "dist": dist})
    return out


def main():
    off, idx = orc.synth_batch(tables(), B, SEED)
    path = os.path.join(GOLD, "ref_batch.dslb")
    ref.save_lookup_batch(path, off, idx, len(DIMS), B)
    l_off, l_idx, T, Bl = ref.load_lookup_batch(path)
    assert T == len(DIMS) and Bl == B
    assert np.array_equal(l_off, off) and np.array_equal(l_idx, idx)
    specs, mean, std = ref.ingest(l_off, l_idx, T, Bl, DIMS, ROWS, 2)
    rec = {"num_tables": T, "batch_size": Bl, "offsets_len": int(len(l_off)),
           "indices_len": int(len(l_idx)), "offsets_sum": int(l_off.sum()),
           "indices_sum": int(l_idx.sum()), "dims": DIMS, "hash_sizes": ROWS,
           "bytes_per_param": 2,
           "ingest": [{"pooling_factor": s["pooling_factor"], "table_size_gb": s["table_size_gb"],
                       "dist": list(s["dist"])} for s in specs],
           "feature_mean": list(mean), "feature_std": list(std)}
    with open(os.path.join(GOLD, "ref_dslb.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
