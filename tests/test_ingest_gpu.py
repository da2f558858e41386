"""K5: ingest_lookup_batch on the GPU, bit-exact against the reference's own
answers (tests/golden/ref_ingest.json) including SPEC.md:51-53's examples,
and against the oracle restatement at cfg3 scale."""
import json
import os

import numpy as np
import pytest

from oracle import lookup as orc
from paper_2210_02023_b200.api import LookupBatch, ShardplanError, ingest_lookup_batch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "ref_ingest.json")) as f:
    GOLD = json.load(f)


@pytest.mark.parametrize("name", sorted(GOLD))
def test_ingest_bit_exact(name):
    c = GOLD[name]
    b = LookupBatch(np.array(c["indices"], dtype=np.int64), np.array(c["offsets"]), c["T"], c["B"])
    tables, mean, std = ingest_lookup_batch(b, c["dims"], c["hash"], bytes_per_param=2)
    for got, want in zip(tables, c["expected_tables"]):
        assert got.pooling_factor == want["pooling_factor"]
        assert got.table_size_gb == want["table_size_gb"]
        assert list(got.dist) == want["dist"]
    np.testing.assert_allclose(mean, c["expected_mean"], rtol=1e-12)
    np.testing.assert_allclose(std, c["expected_std"], rtol=1e-9, atol=1e-12)


def test_ingest_cfg3_scale_matches_oracle(pools):
    tables = pools["cfg3"]["tables"][:20]
    B = 65536
    off, idx = orc.synth_batch(tables, B, seed=2210)
    b = LookupBatch(idx, off, len(tables), B)
    got, _, _ = ingest_lookup_batch(b, [t["dim"] for t in tables], [t["hash_size"] for t in tables],
                                    bytes_per_param=4)
    rc, pf, dist = orc.ingest(off, idx, len(tables), B)
    assert rc == 0
    for i, t in enumerate(got):
        assert t.pooling_factor == pf[i]
        assert list(t.dist) == dist[i].tolist()


def test_ingest_rejects_malformed():
    with pytest.raises(ShardplanError) as e:
        ingest_lookup_batch(LookupBatch(np.array([1, 2]), np.array([0, 2, 1]), 1, 2), [4], [10])
    assert e.value.kind == "malformed_batch"
    with pytest.raises(ShardplanError) as e:
        ingest_lookup_batch(LookupBatch(np.array([1]), np.array([0, 1, 1]), 1, 2), [0], [10])
    assert e.value.kind == "bad_input"
