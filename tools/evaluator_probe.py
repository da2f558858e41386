"""Times the GPU evaluator (K6/K7) at cfg3 tables: 4096 sampled rollouts,
4096 greedy rollouts and 4096 cost-net scorings, D in {4, 8}, median of 5
host-wall calls after one warm-up; SP_LIBRARY selects an A/B build.
    python tools/evaluator_probe.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CKPT, load_task  # noqa: E402
from paper_2210_02023_b200 import api  # noqa: E402

ckpt = api.load_checkpoint(CKPT)
out = {"lib": os.path.basename(os.environ.get("SP_LIBRARY", "_shardplan_b200.so"))}
for D in (4, 8):
    task = load_task("cfg3", D)
    ev = api.Evaluator(ckpt, task)
    rng = np.random.default_rng(D)
    n, M = 4096, len(task.tables)
    u = rng.random((n, M))
    pl = rng.integers(0, D, size=(n, M)).astype(np.int32)
    for name, fn in (("sampled", lambda: ev.rollout(n, "sample", uniforms=u)),
                     ("greedy", lambda: ev.rollout(n, "greedy")),
                     ("eval", lambda: ev.eval_batch(pl))):
        fn()
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        out[f"D{D}_{name}_ms"] = round(sorted(ts)[2], 3)
    ev.close()
print(json.dumps(out))
