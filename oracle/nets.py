"""CPU ORACLE (test infrastructure only): fp64 numpy restatement of
DreamShard's cost network, policy network and Alg. 2 inference, following
the reference line by line. Pinned against the reference's own outputs in
tests/golden/ref_evaluator.json (tests/test_oracle_cpu.py).

  feature_vector ............ table.hpp:89-104
  mlp_forward ............... nn.hpp:82-111 (sequential dot products)
  costnet reductions ........ costnet.hpp:129-158
  EstimatedCostProvider ..... costnet.hpp:454-515
  policy_scores ............. policy.hpp:87-119
  softmax_masked ............ nn.hpp:207-229
  greedy/sample_action ...... policy.hpp:156-184
  PlacementEnv .............. mdp.hpp:95-159
  predicted_order / infer ... harness.hpp:112-137, 332-356
"""
from __future__ import annotations

import math

import numpy as np

SIZES = {
    "cost.table_mlp": [21, 128, 32], "cost.head_fwd": [32, 64, 1], "cost.head_bwd": [32, 64, 1],
    "cost.head_comm": [32, 64, 1], "cost.head_overall": [32, 64, 1],
    "policy.table_mlp": [21, 128, 32], "policy.cost_mlp": [3, 64, 32], "policy.head": [64, 1],
}


def mlp_forward(params, sizes, x):
    cur = [float(v) for v in x]
    off = 0
    L = len(sizes) - 1
    for l in range(L):
        i_n, o_n = sizes[l], sizes[l + 1]
        W = params[off:off + i_n * o_n]
        b = params[off + i_n * o_n: off + i_n * o_n + o_n]
        off += i_n * o_n + o_n
        nxt = []
        for o in range(o_n):
            acc = float(b[o])
            row = W[o * i_n:(o + 1) * i_n]
            for i in range(i_n):
                acc += float(row[i]) * cur[i]
            nxt.append(acc)
        if l + 1 < L:
            nxt = [v if v > 0.0 else 0.0 for v in nxt]
        cur = nxt
    return cur


def feature_rows(tables, mean, std, mask):
    rows = []
    for t in tables:
        v = [float(t["dim"]), float(t["hash_size"]), t["pooling_factor"], t["table_size_gb"]] + \
            [float(x) for x in t["dist"]]
        for f in range(4):
            sd = std[f] if std[f] > 1e-12 else 1.0
            v[f] = (math.log1p(v[f]) - mean[f]) / sd
        rows.append([v[f] if mask[f] != 0.0 else 0.0 for f in range(21)])
    return rows


def _reduce(kind, items, dim=32):
    out = [0.0] * dim
    if not items:
        return out
    if kind == 2:
        return [max(it[k] for it in items) for k in range(dim)]
    for it in items:
        for k in range(dim):
            out[k] += it[k]
    if kind == 1:
        out = [v / len(items) for v in out]
    return out


class Nets:
    def __init__(self, sections):
        self.s = {k: np.asarray(v, dtype=np.float64) for k, v in sections.items()}
        self.red_tables = int(self.s["reductions"][0])
        self.red_devices = int(self.s["reductions"][1])

    def f(self, name, x):
        return mlp_forward(self.s[name], SIZES[name], x)


class Estimated:
    """EstimatedCostProvider (costnet.hpp:454-515)."""

    def __init__(self, nets: Nets, rows):
        self.n = nets
        self.reprs = [nets.f("cost.table_mlp", r) for r in rows]

    def device_repr(self, ids):
        return _reduce(self.n.red_tables, [self.reprs[i] for i in sorted(ids)])

    def cost_features(self, sets):
        q = []
        for ids in sets:
            h = self.device_repr(ids)
            q.append([max(0.0, self.n.f(f"cost.head_{k}", h)[0]) for k in ("fwd", "bwd", "comm")])
        return q

    def overall(self, placement, D):
        sets = [[] for _ in range(D)]
        for i, d in enumerate(placement):
            sets[d].append(i)
        dev = [self.device_repr(s) for s in sets]
        return self.n.f("cost.head_overall", _reduce(self.n.red_devices, dev))[0]


def softmax_masked(logits, mask):
    zmax = -1e300
    for z, m in zip(logits, mask):
        if m:
            zmax = max(zmax, z)
    p = [math.exp(z - zmax) if m else 0.0 for z, m in zip(logits, mask)]
    s = 0.0
    for v, m in zip(p, mask):
        if m:
            s += v
    return [v / s for v in p]


def predicted_order(nets: Nets, rows):
    est = Estimated(nets, rows)
    cost = []
    for i in range(len(rows)):
        q = est.cost_features([[i]])[0]
        cost.append(q[0] + q[1] + q[2])
    return sorted(range(len(rows)), key=lambda i: (-cost[i], i))


def rollout(nets: Nets, tables, rows, D, cap, uniforms=None):
    """One episode (greedy when uniforms is None) -> (placement, raw overall)."""
    est = Estimated(nets, rows)
    preprs = [nets.f("policy.table_mlp", r) for r in rows]
    order = predicted_order(nets, rows)
    sets = [[] for _ in range(D)]
    q = [[0.0, 0.0, 0.0] for _ in range(D)]
    mem = [0.0] * D
    placement = [-1] * len(tables)
    for step, tid in enumerate(order):
        need = tables[tid]["table_size_gb"]
        legal = [mem[d] + need <= cap for d in range(D)]
        if not any(legal):
            raise RuntimeError("infeasible")
        scores = []
        for d in range(D):
            concat = [0.0] * 32
            for i in sorted(sets[d]):
                for k in range(32):
                    concat[k] += preprs[i][k]
            concat += nets.f("policy.cost_mlp", q[d])
            scores.append(nets.f("policy.head", concat)[0])
        p = softmax_masked(scores, legal)
        if uniforms is None:
            best, bp = -1, -1.0
            for d in range(D):
                if p[d] > bp:
                    bp, best = p[d], d
            a = best
        else:
            u = uniforms[step]
            acc, last, a = 0.0, -1, -1
            for d in range(D):
                if p[d] <= 0.0:
                    continue
                acc += p[d]
                last = d
                if u < acc:
                    a = d
                    break
            if a < 0:
                a = last
        sets[a].append(tid)
        mem[a] += need
        placement[tid] = a
        q = est.cost_features(sets)
    return placement, est.overall(placement, D)
