"""K6/K7 batched cost/policy evaluator vs the reference's own answers
(tests/golden/ref_evaluator.json, produced by oracle/_ref from the
unmodified reference): visit order and placements bit-exact; cost and
policy outputs rtol 1e-4 (BASELINE.json north star)."""
import json
import os

import numpy as np
import pytest

from paper_2210_02023_b200.api import (Evaluator, PlacementTask, ShardplanError, TableDesc,
                                       infer, load_checkpoint)

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "ref_evaluator.json")) as f:
    GOLD = json.load(f)
DATA = os.path.join(os.path.dirname(HERE), "paper_2210_02023_b200", "data")
CASES = sorted(GOLD)


def _setup(name):
    g = GOLD[name]
    ckpt = load_checkpoint(os.path.join(DATA, g["checkpoint"]))
    tables = [TableDesc.from_dict(t) for t in g["tables"]]
    task = PlacementTask(tables, g["D"], g["cap"], g["B"])
    return g, ckpt, task


def _close(got, want, rtol=1e-4):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    tol = rtol * np.maximum(np.abs(want), 1.0)
    assert np.all(np.abs(got - want) <= tol), np.max(np.abs(got - want) / np.maximum(np.abs(want), 1))


@pytest.mark.parametrize("name", CASES)
def test_predicted_order_bit_exact(name):
    g, ckpt, task = _setup(name)
    ev = Evaluator(ckpt, task)
    assert ev.order().tolist() == g["order"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("precision", ["guarded", "fp64"])
def test_greedy_rollout_matches_reference_infer(name, precision):
    g, ckpt, task = _setup(name)
    ev = Evaluator(ckpt, task)
    pl, pred, st, nref = ev.rollout(4, "greedy", precision=precision)
    assert (st == 0).all()
    for i in range(4):
        assert pl[i].tolist() == g["infer_placement"]
    want = g["infer_predicted"]
    _close(max(0.0, pred[0]), want, rtol=1e-4 if precision == "guarded" else 1e-12)


@pytest.mark.parametrize("name", CASES)
def test_infer_api(name):
    g, ckpt, task = _setup(name)
    placement, predicted = infer(ckpt, task)
    assert placement.tolist() == g["infer_placement"]
    _close(predicted, g["infer_predicted"])


@pytest.mark.parametrize("name", CASES)
def test_eval_batch_matches_estimated_provider(name):
    g, ckpt, task = _setup(name)
    ev = Evaluator(ckpt, task)
    rand = np.array(g["random_placements"], dtype=np.int32)
    overall, q = ev.eval_batch(rand)
    _close(overall, g["random_overall"])
    _close(q, g["random_q"])


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("precision", ["guarded", "fp64"])
def test_sampled_rollouts_match_reference(name, precision):
    g, ckpt, task = _setup(name)
    ev = Evaluator(ckpt, task)
    u = np.array(g["uniforms"])
    n = u.shape[0]
    pl, pred, st, _ = ev.rollout(n, "sample", uniforms=u, precision=precision)
    assert (st == 0).all()
    assert pl.tolist() == g["sampled_placements"]
    _close(pred, g["sampled_overall"], rtol=1e-4 if precision == "guarded" else 1e-12)


def test_infeasible_task_is_an_error():
    g, ckpt, task = _setup("cfg2")
    tight = PlacementTask(task.tables, task.num_devices,
                          0.5 * max(t.table_size_gb for t in task.tables), task.batch_size)
    ev = Evaluator(ckpt, tight)
    _, _, st, _ = ev.rollout(2, "greedy")
    assert (st == 1).all()  # SP_ERR_INFEASIBLE
    with pytest.raises(ShardplanError) as e:
        infer(ckpt, tight)
    assert e.value.kind == "infeasible" and e.value.exit_code == 2


def test_many_candidates_consistent():
    """4096 greedy candidates of one task are all the same placement; fp32
    throughput path with the fp64 guard."""
    g, ckpt, task = _setup("cfg3")
    ev = Evaluator(ckpt, task)
    pl, pred, st, nref = ev.rollout(4096, "greedy")
    assert (pl == np.array(g["infer_placement"])[None, :]).all()
    assert np.ptp(pred) == 0.0 or nref > 0
