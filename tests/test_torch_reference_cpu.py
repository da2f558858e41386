"""The lookup path's semantics pinned to a third-party implementation: the
reference's lookups ran in FBGEMM's table-batched embedding (PAPER.md:485,
709; not vendored, not pinned), whose sum-pooled forward and row-wise SGD
are PyTorch's `embedding_bag(mode="sum")` and its gradient. On CPU, for
tasks with empty bags, repeated rows inside a bag, hot rows and several
tables: the oracle's forward == torch's embedding_bag per table, and the
oracle's SGD == W - lr * dL/dW from torch autograd (loss = sum(pooled *
grad)). fp32 torch against the fp64-accumulating oracle: rtol 1e-5."""
import numpy as np
import pytest
import torch

from oracle import lookup as orc
from tests.helpers import as_dicts, random_task, random_weights

RTOL, ATOL = 1e-5, 1e-5


def _torch_step(task, weights, off, idx, grad, lr):
    """Per table: embedding_bag(sum) forward, autograd of sum(pooled * g)."""
    B = task.batch_size
    pooled, updated = [], []
    col = 0
    for t, tab in enumerate(task.tables):
        seg = off[t * B:(t + 1) * B + 1]
        ids = torch.from_numpy(idx[seg[0]:seg[-1]].astype(np.int64))
        offs = torch.from_numpy((seg[:-1] - seg[0]).astype(np.int64))
        w = torch.tensor(weights[t], dtype=torch.float32, requires_grad=True)
        p = torch.nn.functional.embedding_bag(ids, w, offs, mode="sum")
        g = torch.from_numpy(grad[:, col:col + tab.dim])
        (p * g).sum().backward()
        pooled.append(p.detach().numpy())
        updated.append((w - lr * w.grad).detach().numpy())
        col += tab.dim
    return np.concatenate(pooled, axis=1), updated


@pytest.mark.parametrize("seed", [3, 17, 29])
def test_oracle_matches_torch_embedding_bag(seed):
    B = 96
    dims = [16, 4, 32, 12, 8, 64]
    task, _ = random_task(seed, dims, 1, B, rows_range=(1, 300), pf_range=(0.0, 9.0))
    weights = random_weights(seed + 1, task.tables)
    off, idx = orc.synth_batch(as_dicts(task.tables), B, seed=seed + 2)
    W = sum(dims)
    grad = np.random.default_rng(seed + 3).uniform(-1, 1, size=(B, W)).astype(np.float32)
    lr = 0.05
    want_p, want_w = _torch_step(task, weights, off, idx, grad, lr)
    rows = [t.hash_size for t in task.tables]
    np.testing.assert_allclose(orc.tbe_forward(dims, rows, weights, off, idx, B), want_p,
                               rtol=RTOL, atol=ATOL)
    got_w = orc.tbe_backward_sgd(dims, rows, weights, off, idx, B, grad, lr,
                                 list(range(len(dims))))
    for g, w in zip(got_w, want_w):
        np.testing.assert_allclose(g, w, rtol=RTOL, atol=ATOL)
