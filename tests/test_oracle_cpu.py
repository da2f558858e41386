"""CPU-only checks of the oracle (oracle/) against the reference's golden
vectors and SPEC.md's worked examples, plus the host mirror's pure-host
logic (expert placements, feature stats, checkpoint reader). No GPU."""
import json
import math
import os

import numpy as np
import pytest

from oracle import lookup as orc
from oracle import nets as onets
from oracle import ref
from paper_2210_02023_b200.api import (EXPERT_STRATEGIES, LookupBatch, PlacementTask,
                                       ShardplanError, TableDesc, compute_feature_stats,
                                       expert_placement, load_checkpoint, table_memory_gb,
                                       validate_batch)

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
DATA = os.path.join(os.path.dirname(HERE), "paper_2210_02023_b200", "data")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---- cost-model known answers ---------------------------

def test_reference_known_answers():
    g = _load("ref_oracle.json")
    comm = {tuple(x[:3]): x[3] for x in g["device_comm"]}
    assert abs(comm[(256, 4, 65536)] - 11.24) <= 0.02
    assert abs(comm[(832, 4, 65536)] - 17.65) <= 0.02
    fs = dict((k, v) for k, v in g["fusion_speedup"])
    assert fs[1] == 1.0 and abs(fs[10] - 2.35) < 0.01 and fs[200] <= 3.0


# ---- table.hpp -------------------------------------------------------------

def test_table_memory_gb_spec():
    assert table_memory_gb(1 << 20, 16, 2) == 0.03125
    assert table_memory_gb(1 << 30, 1, 2) == 2.0
    assert abs(table_memory_gb(10**6, 16, 2) - 0.0298) < 1e-4


@pytest.mark.parametrize("count,want", [(0, 0), (1, 0), (2, 1), (3, 2), (4, 2), (5, 3),
                                        (8, 3), (9, 4), (32768, 15), (32769, 16),
                                        (10**9, 16)])
def test_access_count_bin(count, want):
    assert orc.lib().or_access_count_bin(count) == want


@pytest.mark.parametrize("name", ["spec_one_hot", "spec_empty", "spec_two_tables", "random_hot"])
def test_oracle_ingest_matches_reference(name):
    c = _load("ref_ingest.json")[name]
    rc, pf, dist = orc.ingest(c["offsets"], c["indices"], c["T"], c["B"])
    assert rc == 0
    for i, t in enumerate(c["expected_tables"]):
        assert pf[i] == t["pooling_factor"]
        assert dist[i].tolist() == t["dist"]


def test_ingest_spec_examples():
    # index 7 accessed 4 times -> all mass in bin (2,4]
    rc, pf, dist = orc.ingest([0, 1, 2, 3, 4], [7, 7, 7, 7], 1, 4)
    assert pf[0] == 1.0 and dist[0][2] == 1.0 and dist[0].sum() == 1.0
    # two tables, batch 2 -> pf 2 and 1
    rc, pf, dist = orc.ingest([0, 2, 4, 5, 6], [1, 2, 3, 4, 9, 9], 2, 2)
    assert pf.tolist() == [2.0, 1.0]
    # malformed (validate_batch, table.hpp:167-184)
    assert orc.ingest([0, 2, 1], [1, 2], 1, 2)[0] == 3
    assert orc.ingest([1, 2, 2], [1, 2], 1, 2)[0] == 3


def test_feature_stats_match_reference():
    c = _load("ref_ingest.json")["random_hot"]
    tables = [TableDesc.from_dict(t) for t in c["expected_tables"]]
    mean, std = compute_feature_stats(tables)
    np.testing.assert_allclose(mean, c["expected_mean"], rtol=1e-12)
    np.testing.assert_allclose(std, c["expected_std"], rtol=1e-9, atol=1e-12)


def test_validate_batch_errors():
    with pytest.raises(ShardplanError) as e:
        validate_batch(LookupBatch(np.array([1]), np.array([0, 1]), 1, 2))
    assert e.value.kind == "malformed_batch" and e.value.exit_code == 3
    validate_batch(LookupBatch(np.array([1, 1]), np.array([0, 1, 2]), 1, 2))


# ---- generator --------------------------------------------------

def test_generator_properties(pools):
    tables = pools["cfg3"]["tables"][:12]
    B = 4096
    off, idx = orc.synth_batch(tables, B, seed=2210)
    off2, idx2 = orc.synth_batch(tables, B, seed=2210)
    assert (off == off2).all() and (idx == idx2).all()          # deterministic
    lens = np.diff(off).reshape(len(tables), B)
    for t, row in zip(tables, lens):
        assert row.min() >= 0 and row.max() <= math.floor(2 * t["pooling_factor"])
        assert abs(row.mean() - math.floor(2 * t["pooling_factor"]) / 2) < 0.1 * t["pooling_factor"] + 0.2
    for i, t in enumerate(tables):
        seg = idx[off[i * B]:off[(i + 1) * B]]
        assert seg.min() >= 0 and seg.max() < t["hash_size"]
    # round trip: ingest recovers the pooling factors (statistically)
    rc, pf, dist = orc.ingest(off, idx, len(tables), B)
    for t, p in zip(tables, pf):
        assert abs(p - math.floor(2 * t["pooling_factor"]) / 2) < 0.1 * t["pooling_factor"] + 0.2


def test_weights_and_grads_exact_fp32():
    for t, r, c in [(0, 0, 0), (3, 12345, 17), (99, 999999, 127)]:
        w = orc.lib().or_weight(7, t, r, c)
        assert 0.5 <= w < 1.0 and np.float32(w) == w
    g = orc.lib().or_grad(7, 100, 5000)
    assert -1.0 <= g < 1.0


# ---- lookup oracle vs hand-computed and independent numpy ----------------

def test_forward_hand_case():
    w0 = np.arange(12, dtype=np.float32).reshape(3, 4)
    w1 = np.arange(16, dtype=np.float32).reshape(2, 8) * 10
    off = np.array([0, 2, 2, 5, 6, 8, 8])
    idx = np.array([0, 2, 1, 1, 1, 1, 0, 1])
    got = orc.tbe_forward([4, 8], [3, 2], [w0, w1], off, idx, 3)
    want = np.zeros((3, 12), dtype=np.float32)
    want[0, :4] = w0[0] + w0[2]
    want[2, :4] = 3 * w0[1]
    want[0, 4:] = w1[1]
    want[1, 4:] = w1[0] + w1[1]
    np.testing.assert_array_equal(got, want)


def test_backward_hand_case():
    # one table dim 4, B = 3; row 1 used by bags 0 and 2, row 0 by bag 1
    w = np.ones((2, 4), dtype=np.float32)
    off = np.array([0, 1, 2, 3])
    idx = np.array([1, 0, 1])
    grad = np.array([[1, 2, 3, 4], [10, 10, 10, 10], [0.5, 0.5, 0.5, 0.5]], dtype=np.float32)
    k, b, h = orc.sorted_keys([2], off, idx, 3, [0])
    assert k.tolist() == [0, 1, 1] and b.tolist() == [1, 0, 2] and h.tolist() == [0, 1]
    out = orc.tbe_backward_sgd([4], [2], [w], off, idx, 3, grad, 0.1, [0])[0]
    lr = float(np.float32(0.1))  # the SGD step is an fp32 parameter
    np.testing.assert_array_equal(out[0], np.float32(1 - lr * 10.0))
    np.testing.assert_array_equal(out[1], (1 - lr * (grad[0].astype(np.float64) +
                                                     grad[2])).astype(np.float32))


def test_sorted_keys_match_numpy_stable_sort():
    rng = np.random.default_rng(1)
    B, dims, rows = 50, [4, 8, 16], [7, 30, 1000]
    lens = rng.integers(0, 6, size=3 * B)
    off = np.concatenate([[0], np.cumsum(lens)])
    idx = np.concatenate([rng.integers(0, rows[t], size=int(lens[t * B:(t + 1) * B].sum()))
                          for t in range(3)])
    lst = [0, 2]
    k, b, h = orc.sorted_keys(rows, off, idx, B, lst)
    base, keys, bags = 0, [], []
    for t in lst:
        for bb in range(B):
            for p in range(off[t * B + bb], off[t * B + bb + 1]):
                keys.append(base + idx[p])
                bags.append(bb)
        base += rows[t]
    keys, bags = np.array(keys), np.array(bags)
    o = np.argsort(keys, kind="stable")
    assert (k == keys[o]).all() and (b == bags[o]).all()
    assert (h == np.flatnonzero(np.r_[True, np.diff(keys[o]) != 0])).all()


# ---- expert placements / checkpoint ------------------------------------------

@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg4"])
def test_expert_placements_match_reference(pools, cfg):
    g = _load("ref_oracle.json")["expert"]
    p = pools[cfg]
    task = PlacementTask([TableDesc.from_dict(t) for t in p["tables"]], p["num_devices"],
                         p["mem_cap_gb"], p["batch_size"])
    for s in EXPERT_STRATEGIES:
        assert expert_placement(task, s).tolist() == g[f"{cfg}/{s}"]


def test_checkpoint_reader():
    for f in ("dreamshard_m50_d4.dshd", "dreamshard_m100_d8.dshd"):
        ck = load_checkpoint(os.path.join(DATA, f))
        assert ck.reductions == (0, 2)
        assert len(ck.sections["cost.table_mlp"]) == 6944
    with pytest.raises(ShardplanError):
        load_checkpoint(os.path.join(DATA, "pools.json"))


# ---- nets oracle pinned to the reference -----------------------------------

@pytest.mark.parametrize("name", ["sweep_m20_d1", "sweep_m20_d2", "cfg1"])
def test_nets_oracle_matches_reference(name):
    g = _load("ref_evaluator.json")[name]
    ck = load_checkpoint(os.path.join(DATA, g["checkpoint"]))
    nets = onets.Nets(ck.sections)
    rows = onets.feature_rows(g["tables"], ck.feature_mean, ck.feature_std, ck.feature_mask)
    np.testing.assert_allclose(rows, g["feature_rows"], rtol=0, atol=0)
    assert onets.predicted_order(nets, rows) == g["order"]
    pl, overall = onets.rollout(nets, g["tables"], rows, g["D"], g["cap"])
    assert pl == g["infer_placement"]
    assert abs(max(0.0, overall) - g["infer_predicted"]) <= 1e-9 * max(1.0, abs(overall))
    est = onets.Estimated(nets, rows)
    for p, want in zip(g["random_placements"][:8], g["random_overall"][:8]):
        assert abs(est.overall(p, g["D"]) - want) <= 1e-9 * max(1.0, abs(want))
    u = g["uniforms"][0]
    pl, overall = onets.rollout(nets, g["tables"], rows, g["D"], g["cap"], uniforms=u)
    assert pl == g["sampled_placements"][0]


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (needs /root/reference)")
def test_live_reference_agrees_with_oracle_ingest():
    rng = np.random.default_rng(3)
    T, B = 3, 64
    lens = rng.integers(0, 9, size=T * B)
    off = np.concatenate([[0], np.cumsum(lens)])
    idx = rng.integers(0, 40, size=int(off[-1]))
    tables, _, _ = ref.ingest(off, idx, T, B, [4, 8, 16], [40, 40, 40])
    rc, pf, dist = orc.ingest(off, idx, T, B)
    for i, t in enumerate(tables):
        assert t["pooling_factor"] == pf[i] and t["dist"] == dist[i].tolist()


# ---- lookup path: hand-worked golden cases (tests/golden/gen_lookup_cases.py)

@pytest.mark.parametrize("case", _load("lookup_cases.json"), ids=lambda c: c["name"])
def test_oracle_lookup_golden_cases(case):
    """The oracle's forward, stable sort and row-wise SGD against outputs
    worked out from the definitions (integer data, lr 0.5: exact)."""
    dims, rows, B = case["dims"], case["rows"], case["B"]
    w = [np.array(x, dtype=np.float32).reshape(r, d) for x, r, d in
         zip(case["weights"], rows, dims)]
    off = np.array(case["offsets"], dtype=np.int64)
    idx = np.array(case["indices"], dtype=np.int64)
    np.testing.assert_array_equal(orc.tbe_forward(dims, rows, w, off, idx, B),
                                  np.array(case["pooled"], dtype=np.float32))
    for d, want in enumerate(case["sorted"]):
        lst = [t for t in range(len(dims)) if case["placement"][t] == d]
        k, b, h = orc.sorted_keys(rows, off, idx, B, lst)
        assert k.tolist() == want["keys"] and b.tolist() == want["bags"]
        assert h.tolist() == want["heads"]
    grad = np.array(case["grad"], dtype=np.float32)
    got = orc.tbe_backward_sgd(dims, rows, w, off, idx, B, grad, case["lr"],
                               list(range(len(dims))))
    for g, x, r, d in zip(got, case["updated"], rows, dims):
        np.testing.assert_array_equal(g, np.array(x, dtype=np.float32).reshape(r, d))
