"""Writes tests/golden/lookup_cases.json: hand-specified cases for the lookup
path, with the expected outputs worked out by the definitions alone (plain
Python loops, no oracle code):

  forward   pooled[b, col(t) + c] = sum over k in [offsets[t B + b],
            offsets[t B + b + 1]) of W_t[indices[k], c]; empty bag -> 0
            (table.hpp:158-165 CSR layout, "summed")
  sort      per device: key = rowbase(t) + row (rowbase = prefix sum of the
            device's table rows in id order), payload = bag, stable in CSR
            position order; heads = first position of every run
  SGD       W_t[row] -= lr * sum over the row's occurrences of
            dL/dpooled[bag, col(t) + c]

Weights and gradients are small integers and lr = 0.5, so every expected
value is exact in fp32: the oracle and the GPU must match bit for bit.

    python tests/golden/gen_lookup_cases.py
"""
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))


def forward(dims, weights, offsets, indices, B):
    W = sum(dims)
    out = [[0.0] * W for _ in range(B)]
    col = 0
    for t, d in enumerate(dims):
        for b in range(B):
            for k in range(offsets[t * B + b], offsets[t * B + b + 1]):
                for c in range(d):
                    out[b][col + c] += weights[t][indices[k]][c]
        col += d
    return out


def sort_device(rows, offsets, indices, B, tables):
    items = []
    base = 0
    for t in tables:
        for b in range(B):
            for k in range(offsets[t * B + b], offsets[t * B + b + 1]):
                items.append((base + indices[k], b))
        base += rows[t]
    items = sorted(items, key=lambda kb: kb[0])  # Python's sort is stable
    keys = [k for k, _ in items]
    bags = [b for _, b in items]
    heads = [p for p in range(len(keys)) if p == 0 or keys[p] != keys[p - 1]]
    return keys, bags, heads


def sgd(dims, weights, offsets, indices, B, grad, lr):
    out = [[list(r) for r in w] for w in weights]
    col = 0
    for t, d in enumerate(dims):
        sums = {}
        for b in range(B):
            for k in range(offsets[t * B + b], offsets[t * B + b + 1]):
                s = sums.setdefault(indices[k], [0.0] * d)
                for c in range(d):
                    s[c] += grad[b][col + c]
        for r, s in sums.items():
            for c in range(d):
                out[t][r][c] -= lr * s[c]
        col += d
    return out


def case(name, dims, rows, offsets, indices, B, placement, lr=0.5, wseed=1, gseed=2):
    weights = [[[((wseed * 7 + t * 5 + r * 3 + c) % 9) - 4 for c in range(d)]
                for r in range(rows[t])] for t, d in enumerate(dims)]
    W = sum(dims)
    grad = [[((gseed * 11 + b * 5 + c * 3) % 7) - 3 for c in range(W)] for b in range(B)]
    D = max(placement) + 1
    return {
        "name": name, "dims": dims, "rows": rows, "B": B, "placement": placement,
        "offsets": offsets, "indices": indices, "lr": lr,
        "weights": weights, "grad": grad,
        "pooled": forward(dims, weights, offsets, indices, B),
        "sorted": [dict(zip(("keys", "bags", "heads"),
                            sort_device(rows, offsets, indices, B,
                                        [t for t in range(len(dims)) if placement[t] == d])))
                   for d in range(D)],
        "updated": sgd(dims, weights, offsets, indices, B, grad, lr),
    }


def main():
    cases = [
        # 2 tables (dim 4, dim 8), B = 3: table 0 bags {0,2}, {}, {1,1,1};
        # table 1 bags {1}, {0,1}, {} — empty bags, a row repeated in a bag
        case("two_tables_empty_bags", [4, 8], [3, 2], [0, 2, 2, 5, 6, 8, 8],
             [0, 2, 1, 1, 1, 1, 0, 1], 3, [0, 0]),
        # a table nobody reads (all bags empty), a generic dim (12), a dim-1
        # table, rows shared across bags and devices, D = 2
        case("idle_table_generic_dims", [16, 12, 1, 8], [5, 4, 3, 6],
             [0, 3, 3, 4,   6, 6, 6, 6,   6, 7, 9, 9,   12, 14, 15, 15,   19],
             [4, 4, 0, 2, 2, 2,   1, 0, 0, 2, 2, 2,   5, 5, 0, 3, 3, 3, 3], 4,
             [0, 1, 1, 0]),
        # one hot row: every lookup of table 0 hits row 1 (one long run)
        case("single_hot_row", [32, 4], [2, 7],
             [0, 4, 9, 9,   12, 13, 13, 15,   17],
             [1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1,   6, 0, 6, 3, 6], 4, [0, 0]),
    ]
    with open(os.path.join(HERE, "lookup_cases.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))


if __name__ == "__main__":
    main()
