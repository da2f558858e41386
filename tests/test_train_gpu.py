"""GPU training of the cost network (csrc/train.cu) against the
reference's own fp64 code (oracle/_ref: costnet_loss_and_grad,
costnet_train_steps): the loss to 1e-12 and the gradient to 1e-9 relative
(only the association of the minibatch sum differs), then 30 Adam steps with
the reference's Rng minibatches to 1e-8 relative, for the default and the
other reductions / output ReLU."""
import numpy as np
import pytest

from oracle import ref
from paper_2210_02023_b200.api import CostNetTrainer, costnet_subbatch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]

N_PARAMS = 15652


def _setup(seed, n=40, rows=60):
    rng = np.random.default_rng(seed)
    feats = rng.normal(size=(rows, 21))
    params = rng.normal(scale=0.15, size=N_PARAMS)
    dev_off, tab_off, tab_row, tq, tov = [0], [0], [], [], []
    for s in range(n):
        D = int(rng.integers(1, 9))
        for d in range(D):
            k = int(rng.integers(0, 7))
            tab_row.extend(rng.choice(rows, size=k, replace=False).tolist())
            tab_off.append(len(tab_row))
            tq.append(rng.uniform(0.0, 3.0, size=3))
        dev_off.append(len(tab_off) - 1)
        tov.append(rng.uniform(1.0, 9.0) if s % 2 == 0 else np.nan)
    batch = {"n": n, "dev_off": np.array(dev_off, dtype=np.int32),
             "tab_off": np.array(tab_off, dtype=np.int32),
             "tab_row": np.array(tab_row, dtype=np.int32), "target_q": np.array(tq),
             "target_overall": np.array(tov)}
    mask = np.ones(21)
    mask[[3, 7]] = 0.0
    return params, feats, batch, mask


CONFIGS = [(0, 2, 0), (1, 1, 0), (2, 0, 1)]  # (tables, devices, table output relu)


@pytest.mark.parametrize("red", CONFIGS)
def test_loss_and_grad_match_reference(red):
    params, feats, batch, mask = _setup(1)
    rt, rd, relu = red
    want_loss, want_grad = ref.costnet_loss_grad(params, batch, feats, mask, rt, rd, relu)
    tr = CostNetTrainer(params, feats, mask, rt, rd, bool(relu))
    loss, grad = tr.loss_grad(batch)
    tr.close()
    assert abs(loss - want_loss) <= 1e-12 * abs(want_loss)
    scale = np.abs(want_grad).max()
    np.testing.assert_allclose(grad, want_grad, rtol=1e-9, atol=1e-12 * scale)


@pytest.mark.parametrize("red", CONFIGS[:2])
def test_train_steps_match_reference(red):
    params, feats, batch, mask = _setup(2)
    rt, rd, relu = red
    steps, nb, lr, seed = 30, 8, 5e-3, 99
    want, want_mean = ref.costnet_train_steps(params, batch, feats, steps, nb, lr, steps, seed,
                                              mask, rt, rd, relu)
    picks = ref.rng_index(seed, steps * nb, batch["n"]).reshape(steps, nb)
    tr = CostNetTrainer(params, feats, mask, rt, rd, bool(relu), lr=lr, total_steps=steps)
    losses = [tr.step(costnet_subbatch(batch, p)) for p in picks]
    got, _, _, nstep = tr.state()
    tr.close()
    assert nstep == steps
    assert abs(np.mean(losses) - want_mean) <= 1e-9 * abs(want_mean)
    np.testing.assert_allclose(got, want, rtol=1e-8, atol=1e-12)
    assert not np.allclose(got, params)  # it trained


def _episodes(seed, n=6, rows=80):
    """Random same-shape episodes of several tasks: each step assigns the
    next table of a random order to a legal device; q and legality random."""
    from paper_2210_02023_b200.api import PolicyTrainer  # noqa: F401 (import check)
    rng = np.random.default_rng(seed)
    feats = rng.normal(size=(rows, 21))
    eps = {k: [] for k in ("row0", "ntab", "reward", "action", "tab_id", "legal", "q")}
    step_off, dev_off, tab_off = [0], [0], [0]
    for e in range(n):
        M = int(rng.integers(5, 25))
        D = int(rng.integers(2, 9))
        row0 = int(rng.integers(0, rows - M))
        eps["row0"].append(row0)
        eps["ntab"].append(M)
        eps["reward"].append(-rng.uniform(5, 20))
        sets = [[] for _ in range(D)]
        for t in rng.permutation(M):
            legal = rng.uniform(size=D) < 0.8
            if not legal.any():
                legal[int(rng.integers(D))] = True
            a = int(rng.choice(np.flatnonzero(legal)))
            for d in range(D):
                eps["tab_id"].extend(sets[d])
                tab_off.append(len(eps["tab_id"]))
                eps["legal"].append(int(legal[d]))
                eps["q"].append(rng.uniform(0.0, 2.0, size=3) if sets[d] else np.zeros(3))
            dev_off.append(len(tab_off) - 1)
            eps["action"].append(a)
            sets[a].append(int(t))
        step_off.append(len(dev_off) - 1)
    eps.update({"n": n, "step_off": step_off, "dev_off": dev_off, "tab_off": tab_off,
                "q": np.array(eps["q"]).reshape(-1, 3)})
    params = rng.normal(scale=0.2, size=9345)
    return params, feats, eps


def test_reinforce_grad_and_updates_match_reference():
    from paper_2210_02023_b200.api import PolicyTrainer
    params, feats, eps = _episodes(5)
    mask = np.ones(21)
    mask[[0, 9]] = 0.0
    w = 0.001
    want_obj, want_grad = ref.reinforce_loss_grad(params, eps, feats, w, mask)
    tr = PolicyTrainer(params, feats, mask, lr=1e-3, total_steps=10)
    obj, grad = tr.loss_grad(eps, w)
    assert abs(obj - want_obj) <= 1e-12 * max(1.0, abs(want_obj))
    scale = np.abs(want_grad).max()
    np.testing.assert_allclose(grad, want_grad, rtol=1e-9, atol=1e-12 * scale)
    # ten reinforce_update steps on the same episodes
    want_p, want_objs = ref.reinforce_updates(params, eps, feats, w, 10, 1e-3, 10, mask)
    objs = [tr.step(eps, w) for _ in range(10)]
    got, _, _, nstep = tr.state()
    tr.close()
    assert nstep == 10
    np.testing.assert_allclose(objs, want_objs, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(got, want_p, rtol=1e-8, atol=1e-12)
    assert not np.allclose(got, params)
