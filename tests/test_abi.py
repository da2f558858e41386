"""The C-ABI library loads on a CPU-only host, exports every function
include/shardplan_b200.h declares, its struct layouts match the ctypes
mirror, and argument errors map to ErrorKind+1 before any GPU work."""
import ctypes
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2210_02023_b200 import _lib
from paper_2210_02023_b200.api import (EmbeddingShard, LookupBatch, PlacementTask,
                                       ShardplanError, TableDesc, ingest_lookup_batch,
                                       table_memory_gb)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "shardplan_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    names = header_functions()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)


def test_abi_version_and_errors():
    L = _lib.lib()
    assert L.sp_abi_version() == 2
    assert isinstance(L.sp_last_error(), bytes)


def test_struct_layout_matches_header():
    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "shardplan_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\n", sizeof(sp_table_spec), offsetof(sp_table_spec, hash_size),
         offsetof(sp_table_spec, dist), sizeof(sp_breakdown), sizeof(sp_nets));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "l")
        cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
        subprocess.run([cc, "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        got = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(_lib.SpTableSpec), _lib.SpTableSpec.hash_size.offset,
                   _lib.SpTableSpec.dist.offset, ctypes.sizeof(_lib.SpBreakdown),
                   ctypes.sizeof(_lib.SpNets)]


def _tables(n=3):
    return [TableDesc(i, 16, 100, 2.0, table_memory_gb(100, 16, 4), [1.0] + [0.0] * 16)
            for i in range(n)]


def test_ctx_argument_errors_before_gpu():
    tables = _tables()
    with pytest.raises(ShardplanError) as e:
        EmbeddingShard(PlacementTask(tables, 2, 0.0, 64), [0, 1, 2])
    assert e.value.kind == "bad_input"           # device id out of range
    with pytest.raises(ShardplanError) as e:
        EmbeddingShard(PlacementTask(tables, 3, 0.0, 64), [0, 1, 2])
    assert e.value.kind == "shape_mismatch"      # B not divisible by D
    cap = tables[0].table_size_gb * 1.5
    with pytest.raises(ShardplanError) as e:
        EmbeddingShard(PlacementTask(tables, 2, cap, 64), [0, 0, 1])
    assert e.value.kind == "memory_violation" and e.value.exit_code == 2
    with pytest.raises(ShardplanError) as e:
        EmbeddingShard(PlacementTask(tables, 2, 0.0, 64), [0, 1, 1], rank=1, world_size=3)
    assert e.value.kind == "bad_input"           # world_size is 1 (emulation) or D
    with pytest.raises(ShardplanError) as e:
        EmbeddingShard(PlacementTask(tables, 2, 0.0, 64), [0, 1, 1], rank=2, world_size=2)
    assert e.value.kind == "bad_input"           # rank out of range


def test_ingest_argument_errors_before_gpu():
    with pytest.raises(ShardplanError) as e:
        ingest_lookup_batch(LookupBatch(np.array([1, 2]), np.array([0, 2]), 1, 2), [4], [10])
    assert e.value.kind == "malformed_batch"
    with pytest.raises(ShardplanError) as e:
        ingest_lookup_batch(LookupBatch(np.array([1, 2]), np.array([1, 2, 2]), 1, 2), [4], [10])
    assert e.value.kind == "malformed_batch"


def test_comm_model_is_host_only_and_matches_formula():
    """sp_comm_model (the NVLink 5 all-to-all model used when one GPU
    emulates D devices) needs no GPU; send side vs receive side."""
    from paper_2210_02023_b200 import api
    B, D = 65536, 8
    lat, bw = api.A2A_LATENCY_MS, api.NVLINK_PEER_GBS
    sent = 4.0 * B * 800 * (D - 1) / D
    assert abs(api.comm_model_ms(B, 800, -1, D) - (lat + sent / (bw * 1e6))) < 1e-12
    recv = 4.0 * (B // D) * (6224 - 800)
    assert abs(api.comm_model_ms(B, 800, 6224, D) - (lat + max(sent, recv) / (bw * 1e6))) < 1e-12
    assert api.comm_model_ms(B, 800, 6224, 1) == 0.0
    assert api.comm_model_ms(B, 0, 6224, 8) == 0.0
