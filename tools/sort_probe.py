"""Runs the K4a sort of the cfg3 batch (D = 1) a few times: a target for
ncu (`-k regex:sort_`) and a quick CUDA-event timing of the sort alone
(kernels serialised: K1, then the sort, then the SGD), after two warm-up
iterations. SP_LIBRARY selects an A/B build of the library.
    python tools/sort_probe.py [config] [reps] [fp32|fp16|bf16]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import SEED, load_task  # noqa: E402
from paper_2210_02023_b200 import api  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
storage = sys.argv[3] if len(sys.argv) > 3 else "fp32"
task = load_task(cfg, 1)
if storage != "fp32":  # 2 B/param sizing (table_memory_gb), same tables
    task = api.PlacementTask([api.TableDesc(t.id, t.dim, t.hash_size, t.pooling_factor,
                                            api.table_memory_gb(t.hash_size, t.dim, 2), t.dist)
                              for t in task.tables], 1, task.mem_cap_gb, task.batch_size)
sh = api.EmbeddingShard(task, [0] * len(task.tables), lr=0.01, storage=storage)
sh.init_tables(SEED)
sh.synth_batch(SEED)
sh.synth_grad(SEED)
sh.set_overlap(False)
sh.set_profiling(True)
for _ in range(2):
    sh.enqueue_iteration()
sh.kernel_ms()
for _ in range(reps):
    sh.enqueue_iteration()
k = sh.kernel_ms()
out = {n: round(v[0] / max(1, v[1]), 4) for n, v in k.items()}
out["lib"] = os.path.basename(os.environ.get("SP_LIBRARY", "_shardplan_b200.so"))
out["storage"] = storage
print(json.dumps(out))
sh.close()
