"""The modelled NVLink exchange of one GPU emulating D devices
(sp_ctx_set_comm_model, sp_comm_model) and MeasuredCostProvider's comm
term (the B200 counterpart of device_comm, oracle.hpp:178-185,244-269):
the breakdown's comm terms are the model, compute terms stay measured,
the composition is oracle.hpp:222-227's, and a table brings the same
synthetic batch to every partial assignment (generators keyed by id)."""
import numpy as np
import pytest

from paper_2210_02023_b200 import api
from paper_2210_02023_b200.api import EmbeddingShard, MeasuredCostProvider, ShardplanError
from tests.helpers import random_task

pytestmark = pytest.mark.gpu


def test_breakdown_with_modelled_exchange():
    B, D = 512, 4
    task, placement = random_task(61, [16, 32, 64, 128] * 3, D, B, rows_range=(100, 5000))
    sh = EmbeddingShard(task, placement)
    sh.init_tables(1)
    sh.synth_batch(1)
    sh.synth_grad(1)
    sh.set_comm_model(True)
    bd = sh.run_iteration()
    W = [int(sum(t.dim for t, p in zip(task.tables, placement) if p == d)) for d in range(D)]
    Wt = sum(W)
    want = [api.comm_model_ms(B, w, Wt, D) for w in W]
    np.testing.assert_allclose(bd.comm_ms, want, rtol=1e-12)
    assert bd.fwd_comm_stage_ms == max(want) and bd.bwd_comm_stage_ms == max(want)
    assert abs(bd.overall_ms - (max(bd.fwd_ms) + 2 * max(want) + max(bd.bwd_ms))) < 1e-9
    sh.set_comm_model(False)
    bd2 = sh.run_iteration()
    assert bd2.comm_ms != want  # the device-local copy's measured time
    sh.close()


def test_comm_model_rejected_for_rank_contexts():
    task, placement = random_task(62, [16, 32], 2, 64)
    sh = EmbeddingShard(task, placement, rank=0, world_size=2, nccl_id=None)
    with pytest.raises(ShardplanError):
        sh.set_comm_model(True)
    sh.close()


def test_measured_provider_comm_term_and_id_keyed_data():
    B, D = 1024, 2
    task, _ = random_task(63, [16, 64, 32, 128, 8], D, B, rows_range=(1000, 20000))
    prov = MeasuredCostProvider(task, iters=3, warmup=1)
    q = prov.cost_features([[0, 2], [3]])
    assert q[0][2] == api.comm_model_ms(B, 16 + 32, -1, D)
    assert q[1][2] == api.comm_model_ms(B, 128, -1, D)
    assert all(x > 0 for x in q[0][:2]) and all(x > 0 for x in q[1][:2])
    # table 3's synthetic lookups are the same whatever else is assigned
    a = EmbeddingShard(api.PlacementTask([task.tables[3]], 1, 0.0, B), [0])
    b = EmbeddingShard(api.PlacementTask([task.tables[1], task.tables[3]], 1, 0.0, B), [0, 0])
    for s in (a, b):
        s.synth_batch(5)
    ka, _, _ = a.sorted(0)
    kb, _, _ = b.sorted(0)
    rows1 = task.tables[1].hash_size
    np.testing.assert_array_equal(ka, kb[kb >= rows1] - rows1)
    a.close()
    b.close()
    assert prov.overall([0, 1, 0, 1, 1]) > 0
