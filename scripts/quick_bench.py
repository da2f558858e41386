import json, time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2210_02023_b200.api import *
pools = json.load(open('paper_2210_02023_b200/data/pools.json'))
for name in sys.argv[1:]:
    p = pools[name]
    tables = [TableDesc.from_dict(t) for t in p['tables']]
    D = 1
    task = PlacementTask(tables, D, 0.0, p['batch_size'])
    sh = EmbeddingShard(task, [0]*len(tables))
    t0=time.time(); sh.init_tables(1); sh.synth_batch(1); sh.synth_grad(1); print('setup', time.time()-t0, 'nnz', sh.nnz, flush=True)
    for i in range(5):
        bd = sh.run_iteration()
        print(name, 'fwd %.3f bwd %.3f overall %.3f' % (bd.fwd_ms[0], bd.bwd_ms[0], bd.overall_ms), flush=True)
    ab = sh.algorithmic_bytes()
    print('alg bytes', ab, 'fwd GB/s', ab['fwd']/bd.fwd_ms[0]/1e6, 'bwd GB/s', ab['bwd']/bd.bwd_ms[0]/1e6)
    k = sh.graph_replay(0); print('graph kernels', k)
    import ctypes
    from paper_2210_02023_b200._lib import lib
    # time 10 graph replays using torch events on the ctx stream
    import torch
    s = torch.cuda.ExternalStream(sh.stream)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    sh.graph_replay(3); torch.cuda.synchronize()
    e0.record(s); sh.graph_replay(10); e1.record(s); torch.cuda.synchronize()
    print('graph ms/iter', e0.elapsed_time(e1)/10)
    sh.close()
