"""Host-side mirror of the reference's interface for the embedding hot path.

The reference (`shardplan`, C++ headers under proj/include/shardplan) fakes
GPU execution with CostOracle. This module keeps its names, argument meaning
and error behaviour, and routes every computation through the CUDA library
(`_shardplan_b200.so`, C-ABI in include/shardplan_b200.h):

  TableDesc, table_memory_gb ............ table.hpp:45-63
  LookupBatch, validate_batch ........... table.hpp:158-184
  ingest_lookup_batch ................... table.hpp:188-232   (GPU, K5)
  PlacementTask, Placement, CostBreakdown oracle.hpp:68-116
  EmbeddingShard.run_iteration .......... oracle.hpp:187-240  (GPU K1-K4)
  CostProvider / MeasuredCostProvider ... mdp.hpp:28-54
  Checkpoint / load_checkpoint .......... checkpoint.hpp:26-217
  Evaluator, infer ...................... costnet.hpp:454-515, policy.hpp:87-184,
                                          harness.hpp:112-137, 332-356 (GPU K6/K7)

There is no CPU fallback: a missing library raises ImportError.
"""
from __future__ import annotations

import ctypes
import math
import os
import struct
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._lib import (SpBreakdown, SpCostnetBatch, SpNets, SpReinforceBatch, SpTableSpec,
                   ShardplanError, check, lib)

NUM_BINS = 17
NUM_FEATURES = 21
DEFAULT_BATCH_SIZE = 65536
DEFAULT_BYTES_PER_PARAM = 2

__all__ = [
    "TableDesc", "table_memory_gb", "LookupBatch", "validate_batch", "PlacementTask",
    "CostBreakdown", "TraceEvent", "EmbeddingShard", "CostProvider",
    "MeasuredCostProvider", "ingest_lookup_batch", "compute_feature_stats", "Checkpoint",
    "load_checkpoint", "Evaluator", "infer", "ShardplanError", "nccl_unique_id",
    "hot_mass", "HostBuffer", "EXPERT_STRATEGIES", "expert_cost", "greedy_placement",
    "expert_placement", "exchange_plan", "synth_lookup_batch",
]


# ---------------------------------------------------------------------------
# table.hpp

@dataclass
class TableDesc:
    """shardplan::TableDesc (table.hpp:45-52)."""

    id: int = 0
    dim: int = 1
    hash_size: int = 1
    pooling_factor: float = 0.0
    table_size_gb: float = 0.0
    dist: List[float] = field(default_factory=lambda: [0.0] * NUM_BINS)

    @classmethod
    def from_dict(cls, d: dict) -> "TableDesc":
        return cls(int(d["id"]), int(d["dim"]), int(d["hash_size"]),
                   float(d["pooling_factor"]), float(d["table_size_gb"]),
                   [float(x) for x in d["dist"]])

    def to_dict(self) -> dict:
        return {"id": self.id, "dim": self.dim, "hash_size": self.hash_size,
                "pooling_factor": self.pooling_factor, "table_size_gb": self.table_size_gb,
                "dist": list(self.dist)}


def table_memory_gb(hash_size: int, dim: int, bytes_per_param: int = DEFAULT_BYTES_PER_PARAM):
    """table.hpp:55-63: rows * columns * bytes per parameter / 2^30."""
    return float(hash_size) * dim * bytes_per_param / (1024.0 * 1024.0 * 1024.0)


def hot_mass(t: TableDesc) -> float:
    """oracle.hpp:119-123: access mass in bins whose lower edge is >= 8."""
    h = 0.0
    for b in range(4, NUM_BINS):
        h += t.dist[b]
    return h


def _specs(tables: Sequence[TableDesc]):
    arr = (SpTableSpec * max(len(tables), 1))()
    for i, t in enumerate(tables):
        arr[i].id = t.id
        arr[i].dim = t.dim
        arr[i].hash_size = t.hash_size
        arr[i].pooling_factor = t.pooling_factor
        arr[i].table_size_gb = t.table_size_gb
        for b in range(NUM_BINS):
            arr[i].dist[b] = t.dist[b]
    return arr


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


@dataclass
class LookupBatch:
    """shardplan::LookupBatch (table.hpp:158-165): CSR ordered by
    (table_id, batch_offset); lookup k of table t reads
    indices[offsets[t*B + k] : offsets[t*B + k + 1]]."""

    indices: np.ndarray
    offsets: np.ndarray
    num_tables: int
    batch_size: int

    def __post_init__(self):
        self.indices = np.ascontiguousarray(self.indices, dtype=np.int64)
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.int64)


def validate_batch(b: LookupBatch) -> None:
    """table.hpp:167-184; raises ShardplanError(malformed_batch)."""
    if b.num_tables < 0 or b.batch_size <= 0:
        raise ShardplanError(3, "non-positive table or batch count")
    want = b.num_tables * b.batch_size + 1
    if len(b.offsets) != want:
        raise ShardplanError(3, f"offsets length {len(b.offsets)}, expected {want}")
    if b.offsets[0] != 0:
        raise ShardplanError(3, "offsets must start at 0")
    d = np.diff(b.offsets)
    if len(d) and d.min() < 0:
        raise ShardplanError(3, f"offsets decrease at position {int(np.argmax(d < 0)) + 1}")
    if int(b.offsets[-1]) != len(b.indices):
        raise ShardplanError(3, "last offset != indices length")


# Binary lookup-batch file (table.hpp:235-305): "DSLB", u32 version,
# u32 num_tables, u32 batch_size, u64 offsets_len, i64 offsets[],
# u64 indices_len, i64 indices[], little-endian.
BATCH_FILE_VERSION = 1  # kBatchVersion, table.hpp:240
_DSLB_HEADER = np.dtype([("magic", "S4"), ("version", "<u4"), ("num_tables", "<u4"),
                         ("batch_size", "<u4"), ("offsets_len", "<u8")])


def save_lookup_batch(b: LookupBatch, path: str) -> None:
    """save_lookup_batch (table.hpp:268-281): validates, then writes the
    DSLB file byte for byte like the reference."""
    validate_batch(b)
    hdr = np.zeros(1, dtype=_DSLB_HEADER)
    hdr["magic"], hdr["version"] = b"DSLB", BATCH_FILE_VERSION
    hdr["num_tables"], hdr["batch_size"], hdr["offsets_len"] = (b.num_tables, b.batch_size,
                                                                len(b.offsets))
    try:
        with open(path, "wb") as f:
            f.write(hdr.tobytes())
            f.write(b.offsets.astype("<i8", copy=False).tobytes())
            f.write(np.array([len(b.indices)], dtype="<u8").tobytes())
            f.write(b.indices.astype("<i8", copy=False).tobytes())
    except OSError as e:
        raise ShardplanError(10, f"cannot open {path} for writing") from e


def load_lookup_batch(path: str) -> LookupBatch:
    """load_lookup_batch (table.hpp:283-305) into host memory (the device
    path is EmbeddingShard.upload_batch_file / ingest_batch_file, which
    never hold the indices on the host)."""
    try:
        raw = np.fromfile(path, dtype=np.uint8)
    except OSError as e:
        raise ShardplanError(10, f"cannot open {path}") from e
    if len(raw) < 4 or raw[:4].tobytes() != b"DSLB":
        raise ShardplanError(10, f"{path}: not a lookup batch file")

    def u(pos, dt, n=1):
        size = np.dtype(dt).itemsize * n
        if pos + size > len(raw):
            raise ShardplanError(10, "unexpected end of file")
        return raw[pos:pos + size].view(dt)

    version = int(u(4, "<u4")[0])
    if version != BATCH_FILE_VERSION:
        raise ShardplanError(10, f"unsupported batch version {version}")
    T, B, n_off = int(u(8, "<u4")[0]), int(u(12, "<u4")[0]), int(u(16, "<u8")[0])
    if n_off > (len(raw) - 24) // 8:
        raise ShardplanError(10, "unexpected end of file")
    offsets = u(24, "<i8", n_off).astype(np.int64)
    pos = 24 + 8 * n_off
    n_idx = int(u(pos, "<u8")[0])
    if n_idx > (len(raw) - pos - 8) // 8:
        raise ShardplanError(10, "unexpected end of file")
    indices = u(pos + 8, "<i8", n_idx).astype(np.int64)
    # the reference's int fields
    T = T - (1 << 32) if T >= 1 << 31 else T
    B = B - (1 << 32) if B >= 1 << 31 else B
    b = LookupBatch(indices, offsets, T, B)
    validate_batch(b)
    return b


def compute_feature_stats(tables: Sequence[TableDesc]):
    """table.hpp:108-131: per-feature (mean, std) of ln(1+x)."""
    if not tables:
        return np.zeros(NUM_FEATURES), np.ones(NUM_FEATURES)
    raw = np.array([[t.dim, t.hash_size, t.pooling_factor, t.table_size_gb] + list(t.dist)
                    for t in tables], dtype=np.float64)
    y = np.log1p(raw)
    n = float(len(tables))
    s = np.zeros(NUM_FEATURES)
    s2 = np.zeros(NUM_FEATURES)
    for row in y:  # same accumulation order as the reference
        s += row
        s2 += row * row
    mean = s / n
    var = np.maximum(0.0, s2 / n - mean * mean)
    return mean, np.sqrt(var)


def ingest_lookup_batch(b: LookupBatch, dims: Sequence[int], hash_sizes: Sequence[int],
                        bytes_per_param: int = DEFAULT_BYTES_PER_PARAM, device: int = 0):
    """ingest_lookup_batch (table.hpp:188-232) on the GPU (K5).

    Returns (tables, feature_mean, feature_std) — the TablePool content."""
    dims_a = np.ascontiguousarray(dims, dtype=np.int32)
    hs_a = np.ascontiguousarray(hash_sizes, dtype=np.int64)
    out = (SpTableSpec * max(b.num_tables, 1))()
    check(lib().sp_ingest_lookup_batch(_ptr(b.offsets), len(b.offsets), _ptr(b.indices),
                                       len(b.indices), b.num_tables, b.batch_size,
                                       _ptr(dims_a), _ptr(hs_a), bytes_per_param, device, out))
    tables = [TableDesc(s.id, s.dim, s.hash_size, s.pooling_factor, s.table_size_gb,
                        list(s.dist)) for s in out][:b.num_tables]
    mean, std = compute_feature_stats(tables)
    return tables, mean, std


def ingest_batch_file(path: str, dims: Sequence[int], hash_sizes: Sequence[int],
                      bytes_per_param: int = DEFAULT_BYTES_PER_PARAM, device: int = 0):
    """ingest_lookup_batch(load_lookup_batch(path), ...) (table.hpp:188-232,
    283-305) with the file's indices streamed straight to the GPU.

    Returns (tables, feature_mean, feature_std, batch_size)."""
    dims_a = np.ascontiguousarray(dims, dtype=np.int32)
    hs_a = np.ascontiguousarray(hash_sizes, dtype=np.int64)
    if len(dims_a) != len(hs_a):
        raise ShardplanError(10, "dims/hash_sizes length != num_tables")
    out = (SpTableSpec * max(len(dims_a), 1))()
    nt, bs = ctypes.c_int32(), ctypes.c_int32()
    check(lib().sp_ingest_batch_file(os.fsencode(path), _ptr(dims_a), _ptr(hs_a), len(dims_a),
                                     bytes_per_param, device, out, ctypes.byref(nt),
                                     ctypes.byref(bs)))
    tables = [TableDesc(s.id, s.dim, s.hash_size, s.pooling_factor, s.table_size_gb,
                        list(s.dist)) for s in out][:nt.value]
    mean, std = compute_feature_stats(tables)
    return tables, mean, std, bs.value


# ---------------------------------------------------------------------------
# oracle.hpp types

@dataclass
class PlacementTask:
    """shardplan::PlacementTask (oracle.hpp:68-73)."""

    tables: List[TableDesc]
    num_devices: int = 1
    mem_cap_gb: float = 0.0
    batch_size: int = DEFAULT_BATCH_SIZE


@dataclass
class TraceEvent:
    device: int
    phase: str
    start_ms: float
    dur_ms: float


@dataclass
class CostBreakdown:
    """shardplan::CostBreakdown (oracle.hpp:105-116), measured on B200."""

    fwd_ms: List[float]
    bwd_ms: List[float]
    comm_ms: List[float]
    fwd_comm_stage_ms: float
    bwd_comm_stage_ms: float
    overall_ms: float

    @property
    def events(self) -> List[TraceEvent]:
        """Synchronised stage bars, laid out as oracle.hpp:229-238."""
        t1 = max(self.fwd_ms)
        t2 = t1 + self.fwd_comm_stage_ms
        t3 = t2 + self.bwd_comm_stage_ms
        ev = []
        for d in range(len(self.fwd_ms)):
            ev.append(TraceEvent(d, "fwd_comp", 0.0, self.fwd_ms[d]))
            ev.append(TraceEvent(d, "fwd_comm", t1, self.comm_ms[d]))
            ev.append(TraceEvent(d, "bwd_comm", t2, self.comm_ms[d]))
            ev.append(TraceEvent(d, "bwd_comp", t3, self.bwd_ms[d]))
        return ev

    def to_json(self) -> dict:
        return {"devices": len(self.fwd_ms), "overall_ms": self.overall_ms,
                "fwd_ms": list(self.fwd_ms), "bwd_ms": list(self.bwd_ms),
                "comm_ms": list(self.comm_ms), "fwd_comm_stage_ms": self.fwd_comm_stage_ms,
                "bwd_comm_stage_ms": self.bwd_comm_stage_ms,
                "events": [e.__dict__ for e in self.events]}


NVLINK_PEER_GBS = 770.0   # SP_NVLINK_PEER_GBS
A2A_LATENCY_MS = 0.010    # SP_A2A_LATENCY_MS


def comm_model_ms(batch: int, width_dev: int, width_total: int, D: int) -> float:
    """Modelled ms of one all-to-all direction on NVLink 5 for a device with
    width_dev pooled columns (sp_comm_model; width_total < 0: send side only)."""
    ms = ctypes.c_double()
    check(lib().sp_comm_model(int(batch), int(width_dev), int(width_total), int(D),
                              ctypes.byref(ms)))
    return ms.value


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    check(lib().sp_nccl_unique_id(buf))
    return bytes(buf)


def exchange_plan(task: PlacementTask, placement: Sequence[int], rank: int) -> dict:
    """The forward all-to-all plan the NCCL path executes for `rank`
    (sp_exchange_plan; host only). Offsets/counts are fp32 elements."""
    D = task.num_devices
    p = np.ascontiguousarray(placement, dtype=np.int32)
    W = int(sum(t.dim for t in task.tables))
    so, sc, ro, rc = (np.zeros(D, dtype=np.int64) for _ in range(4))
    colmap = np.zeros(max(W, 1), dtype=np.int32)
    check(lib().sp_exchange_plan(_specs(task.tables), len(task.tables), D, _ptr(p),
                                 task.batch_size, rank, _ptr(so), _ptr(sc), _ptr(ro), _ptr(rc),
                                 _ptr(colmap)))
    return {"send_off": so, "send_count": sc, "recv_off": ro, "recv_count": rc,
            "colmap": colmap[:W]}


class HostBuffer:
    """Page-locked host array (sp_host_alloc) for the e2e upload path."""

    def __init__(self, n: int, dtype=np.int64):
        self._p = ctypes.c_void_p()
        self.dtype = np.dtype(dtype)
        check(lib().sp_host_alloc(max(n, 1) * self.dtype.itemsize, ctypes.byref(self._p)))
        buf = (ctypes.c_char * (max(n, 1) * self.dtype.itemsize)).from_address(self._p.value)
        self.array = np.frombuffer(buf, dtype=self.dtype)[:n]

    def __del__(self):
        try:
            if getattr(self, "_p", None) and self._p.value:
                lib().sp_host_free(self._p)
                self._p = ctypes.c_void_p()
        except Exception:  # interpreter shutdown: the library binding is gone
            pass


# ---------------------------------------------------------------------------
# The measured execution of a placement (replaces CostOracle).

class EmbeddingShard:
    """One rank's shard of a placement on one B200 (sp_ctx).

    world_size == num_devices: one process per GPU, exchanges over NCCL.
    world_size == 1 < num_devices: emulation, all virtual devices on this GPU
    (compute measured per device; exchange is a device-local copy).
    storage: "auto" (2 B/param tables -> fp16, else fp32), "fp32", "fp16",
    "bf16" (sp_ctx_create_ex)."""

    STORAGE = {"auto": 0, "fp32": 1, "fp16": 2, "bf16": 3}  # SP_STORAGE_*

    def __init__(self, task: PlacementTask, placement: Sequence[int], lr: float = 0.01,
                 rank: int = 0, world_size: int = 1, nccl_id: Optional[bytes] = None,
                 device: int = 0, storage: str = "auto"):
        self.task = task
        self.placement = np.ascontiguousarray(placement, dtype=np.int32)
        if len(self.placement) != len(task.tables):
            raise ShardplanError(10, "placement length != table count")
        self.D = task.num_devices
        self.B = task.batch_size
        self.rank = rank
        self.world = world_size
        self.dims = np.array([t.dim for t in task.tables], dtype=np.int64)
        self.W_total = int(self.dims.sum())
        self._specs = _specs(task.tables)
        h = ctypes.c_void_p()
        idb = None
        if nccl_id is not None:
            idb = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        if storage not in self.STORAGE:
            raise ShardplanError(10, f"storage must be one of {sorted(self.STORAGE)}")
        check(lib().sp_ctx_create_ex(self._specs, len(task.tables), self.D,
                                     _ptr(self.placement), self.B, float(task.mem_cap_gb),
                                     float(lr), rank, world_size, idb, device,
                                     self.STORAGE[storage], ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().sp_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the library binding is gone
            pass

    # -- properties
    @property
    def stream(self) -> int:
        s = ctypes.c_void_p()
        check(lib().sp_ctx_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    @property
    def device_bytes(self) -> int:
        b = ctypes.c_uint64()
        check(lib().sp_ctx_device_bytes(self._h, ctypes.byref(b)))
        return b.value

    def local_tables(self) -> List[int]:
        n = ctypes.c_int32()
        check(lib().sp_ctx_local_tables(self._h, None, ctypes.byref(n)))
        ids = np.zeros(n.value, dtype=np.int32)
        check(lib().sp_ctx_local_tables(self._h, _ptr(ids), ctypes.byref(n)))
        return ids.tolist()

    def rows_per_rank(self) -> int:
        return self.B if self.world == 1 else self.B // self.D

    # -- tables
    def init_tables(self, seed: int):
        check(lib().sp_init_tables(self._h, seed))

    def set_table(self, table_id: int, rows: np.ndarray):
        t = self.task.tables[table_id]
        rows = np.ascontiguousarray(rows, dtype=np.float32).reshape(t.hash_size, t.dim)
        check(lib().sp_set_table(self._h, table_id, _ptr(rows)))

    def get_table(self, table_id: int) -> np.ndarray:
        t = self.task.tables[table_id]
        out = np.empty((t.hash_size, t.dim), dtype=np.float32)
        check(lib().sp_get_table(self._h, table_id, _ptr(out)))
        return out

    # -- batch
    def upload_batch(self, b: LookupBatch):
        if b.num_tables != len(self.task.tables) or b.batch_size != self.B:
            raise ShardplanError(8, "batch shape does not match the task")
        check(lib().sp_upload_batch(self._h, _ptr(b.offsets), len(b.offsets), _ptr(b.indices),
                                    len(b.indices)))

    def upload_batch_file(self, path: str):
        """load_lookup_batch(path) (table.hpp:283-305) + upload_batch, the
        indices streamed from the file straight to the device (only this
        shard's tables are read)."""
        check(lib().sp_upload_batch_file(self._h, os.fsencode(path)))

    def upload_batch_ptr(self, offsets_ptr: int, offsets_len: int, indices_ptr: int,
                         indices_len: int):
        check(lib().sp_upload_batch(self._h, ctypes.c_void_p(offsets_ptr), offsets_len,
                                    ctypes.c_void_p(indices_ptr), indices_len))

    def synth_batch(self, seed: int):
        check(lib().sp_synth_batch(self._h, seed))

    @property
    def nnz(self) -> int:
        n = ctypes.c_int64()
        check(lib().sp_batch_nnz(self._h, ctypes.byref(n)))
        return n.value

    # -- stages
    def forward(self):
        check(lib().sp_forward(self._h))

    def a2a_forward(self):
        check(lib().sp_a2a_forward(self._h))

    def a2a_backward(self):
        check(lib().sp_a2a_backward(self._h))

    def backward_sgd(self):
        check(lib().sp_backward_sgd(self._h))

    def set_grad(self, grad: np.ndarray):
        g = np.ascontiguousarray(grad, dtype=np.float32).reshape(self.rows_per_rank(),
                                                                  self.W_total)
        check(lib().sp_set_grad(self._h, _ptr(g)))

    def synth_grad(self, seed: int):
        check(lib().sp_synth_grad(self._h, seed))

    def pooled(self) -> np.ndarray:
        out = np.empty((self.rows_per_rank(), self.W_total), dtype=np.float32)
        check(lib().sp_get_pooled(self._h, _ptr(out)))
        return out

    def local_pooled(self, dev: int) -> np.ndarray:
        w = int(self.dims[self.placement == dev].sum())
        out = np.empty((self.B, w), dtype=np.float32)
        check(lib().sp_get_local_pooled(self._h, dev, _ptr(out)))
        return out

    def sorted(self, dev: int):
        """(keys, bags, run heads) of device dev's backward sort."""
        n = ctypes.c_int64()
        nu = ctypes.c_int64()
        check(lib().sp_get_sorted(self._h, dev, None, None, ctypes.byref(n), None,
                                  ctypes.byref(nu)))
        keys = np.empty(n.value, dtype=np.uint32)
        bags = np.empty(n.value, dtype=np.uint32)
        heads = np.empty(max(n.value, 1), dtype=np.uint32)
        check(lib().sp_get_sorted(self._h, dev, _ptr(keys), _ptr(bags), ctypes.byref(n),
                                  _ptr(heads), ctypes.byref(nu)))
        return keys, bags, heads[:nu.value]

    def run_iteration(self) -> CostBreakdown:
        D = self.D
        f = (ctypes.c_double * D)()
        b = (ctypes.c_double * D)()
        c = (ctypes.c_double * D)()
        bd = SpBreakdown(f, b, c, 0.0, 0.0, 0.0)
        check(lib().sp_run_iteration(self._h, ctypes.byref(bd)))
        return CostBreakdown(list(f), list(b), list(c), bd.fwd_comm_stage_ms,
                             bd.bwd_comm_stage_ms, bd.overall_ms)

    def run_local(self, with_sort: bool = False):
        """This shard's compute of one iteration, exchanges left out:
        (forward-stage ms, backward-stage ms[, sort ms]) (sp_run_local). The
        backward stage waits for the sort, which in a multi-GPU iteration
        runs under the exchanges."""
        ms = np.zeros(3)
        check(lib().sp_run_local(self._h, _ptr(ms)))
        if with_sort:
            return float(ms[0]), float(ms[1]), float(ms[2])
        return float(ms[0]), float(ms[1])

    def run_batch(self, b: LookupBatch) -> CostBreakdown:
        """upload_batch + run_iteration in one pipelined call (sp_run_batch):
        the H2D of the host LookupBatch overlaps the forward of the tables
        already uploaded; validation errors are raised like upload_batch and
        leave the tables untouched."""
        if b.num_tables != len(self.task.tables) or b.batch_size != self.B:
            raise ShardplanError(8, "batch shape does not match the task")
        D = self.D
        f = (ctypes.c_double * D)()
        bw = (ctypes.c_double * D)()
        c = (ctypes.c_double * D)()
        bd = SpBreakdown(f, bw, c, 0.0, 0.0, 0.0)
        check(lib().sp_run_batch(self._h, _ptr(b.offsets), len(b.offsets), _ptr(b.indices),
                                 len(b.indices), ctypes.byref(bd)))
        return CostBreakdown(list(f), list(bw), list(c), bd.fwd_comm_stage_ms,
                             bd.bwd_comm_stage_ms, bd.overall_ms)

    def run_batches(self, batches: list) -> list:
        """n consecutive host-buffer steps (sp_run_batches): step s's H2D
        overlaps step s-1's compute. Returns per-step device ms."""
        n = len(batches)
        for b in batches:
            if b.num_tables != len(self.task.tables) or b.batch_size != self.B:
                raise ShardplanError(8, "batch shape does not match the task")
        offs = (ctypes.c_void_p * n)(*[b.offsets.ctypes.data for b in batches])
        idxs = (ctypes.c_void_p * n)(*[b.indices.ctypes.data for b in batches])
        olen = (ctypes.c_int64 * n)(*[len(b.offsets) for b in batches])
        ilen = (ctypes.c_int64 * n)(*[len(b.indices) for b in batches])
        ms = (ctypes.c_double * n)()
        check(lib().sp_run_batches(self._h, n, offs, olen, idxs, ilen, ms))
        return list(ms)

    def enqueue_iteration(self):
        check(lib().sp_enqueue_iteration(self._h))

    def graph_replay(self, iters: int) -> int:
        k = ctypes.c_int32()
        check(lib().sp_graph_replay(self._h, iters, ctypes.byref(k)))
        return k.value

    IPC_BYTES = 128

    def ipc_export(self) -> bytes:
        """CUDA IPC handles of this rank's receive and gradient buffers
        (sp_ipc_export), to be all-gathered by the host in rank order."""
        buf = (ctypes.c_uint8 * self.IPC_BYTES)()
        check(lib().sp_ipc_export(self._h, buf))
        return bytes(buf)

    def ipc_import(self, handles: list):
        """Map every rank's buffers (sp_ipc_import): K1 then stores pooled
        rows at their receivers and the backward pulls gradients from peers."""
        if len(handles) != self.world:
            raise ShardplanError(8, "one handle blob per rank expected")
        blob = b"".join(handles)
        buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        check(lib().sp_ipc_import(self._h, buf))

    def synchronize(self):
        check(lib().sp_ctx_synchronize(self._h))

    def set_comm_model(self, on: bool):
        """One GPU emulating D devices: report the exchange terms of the
        breakdown as the modelled NVLink 5 all-to-all (sp_ctx_set_comm_model)
        instead of the device-local copy's time."""
        check(lib().sp_ctx_set_comm_model(self._h, 1 if on else 0))

    def set_overlap(self, on: bool):
        """Backward sort on the side stream, forked after K1 and concurrent
        with the exchanges (default), or on the main stream behind K1
        (sp_ctx_set_overlap)."""
        check(lib().sp_ctx_set_overlap(self._h, 1 if on else 0))

    def set_sort_target(self, lookups: int):
        """K4a sort plan override (sp_ctx_set_sort_target): buckets and
        warp-tiles of about `lookups` lookups, 0 = default. Results are
        independent of it."""
        check(lib().sp_ctx_set_sort_target(self._h, int(lookups)))

    def set_upload_chunk(self, indices: int):
        """Indices per H2D chunk of the pipelined host-buffer upload
        (sp_ctx_set_upload_chunk). Results are independent of it."""
        check(lib().sp_ctx_set_upload_chunk(self._h, int(indices)))

    def set_profiling(self, on: bool):
        check(lib().sp_ctx_set_profiling(self._h, 1 if on else 0))

    KERNELS = ("fwd", "unused", "sort", "sgd", "exchange")

    def kernel_ms(self) -> dict:
        """Summed CUDA-event ms and launch counts per hot kernel since the
        last call (profiling must be on)."""
        ms = (ctypes.c_double * 5)()
        n = (ctypes.c_int64 * 5)()
        check(lib().sp_ctx_kernel_ms(self._h, ms, n))
        return {k: (ms[i], n[i]) for i, k in enumerate(self.KERNELS)}

    def algorithmic_bytes(self) -> dict:
        out = (ctypes.c_double * 5)()
        check(lib().sp_ctx_algorithmic_bytes(self._h, out))
        return {"fwd": out[0], "a2a": out[1], "bwd": out[2], "sort": out[3],
                "fwd_unique": out[4]}


# ---------------------------------------------------------------------------
# mdp.hpp plugin boundary

class CostProvider:
    """shardplan::CostProvider (mdp.hpp:28-34)."""

    def cost_features(self, assignment: Sequence[Sequence[int]]):  # pragma: no cover
        raise NotImplementedError

    def overall(self, placement: Sequence[int]) -> float:  # pragma: no cover
        raise NotImplementedError


class MeasuredCostProvider(CostProvider):
    """CostProvider whose numbers are measured on this B200 instead of the
    synthetic oracle (the drop-in for OracleCostProvider, mdp.hpp:37-54).

    Every query builds an emulated shard of the (partial) assignment on this
    GPU — all D virtual devices, real K1/K4 kernels on the synthetic batch of
    the task — and returns median stage times over `iters` iterations after
    `warmup`. cost_features returns per device (fwd_ms, bwd_ms, comm_ms);
    a device with no tables reports (0, 0, 0) like oracle.hpp:242-269.

    One GPU cannot time NVLink, so with comm_model (default) the comm terms
    are the modelled NVLink 5 all-to-all (sp_comm_model: the B200
    counterpart of device_comm, oracle.hpp:178-185) instead of the
    emulation's device-local copy: comm_ms of a device = its send side
    (its own tables only, like device_comm); overall = max fwd + the two
    modelled stages + max bwd. Synthetic data is keyed by table id, so a
    table brings the same batch to every partial assignment."""

    def __init__(self, task: PlacementTask, seed: int = 2210, iters: int = 5, warmup: int = 2,
                 device: int = 0, comm_model: bool = True):
        self.task = task
        self.seed = seed
        self.iters = iters
        self.warmup = warmup
        self.device = device
        self.comm_model = comm_model
        self.calls = 0

    def _measure(self, placement: np.ndarray, subset: np.ndarray) -> CostBreakdown:
        tables = [self.task.tables[i] for i in subset]
        sub_task = PlacementTask(tables, self.task.num_devices, self.task.mem_cap_gb,
                                 self.task.batch_size)
        shard = EmbeddingShard(sub_task, placement[subset], device=self.device)
        try:
            shard.set_comm_model(self.comm_model)
            shard.init_tables(self.seed)
            shard.synth_batch(self.seed)
            shard.synth_grad(self.seed)
            runs = []
            for i in range(self.warmup + self.iters):
                bd = shard.run_iteration()
                if i >= self.warmup:
                    runs.append(bd)
        finally:
            shard.close()
        k = int(np.argsort([r.overall_ms for r in runs])[len(runs) // 2])
        return runs[k]

    def cost_features(self, assignment):
        self.calls += 1
        D = self.task.num_devices
        if len(assignment) != D:
            raise ShardplanError(10, "assignment has wrong device count")
        placement = np.full(len(self.task.tables), -1, dtype=np.int32)
        for d, ids in enumerate(assignment):
            for i in ids:
                if i < 0 or i >= len(self.task.tables):
                    raise ShardplanError(5, f"table id {i}")
                placement[i] = d
        subset = np.nonzero(placement >= 0)[0]
        if len(subset) == 0:
            return [(0.0, 0.0, 0.0)] * D
        bd = self._measure(placement, subset)
        out = []
        for d in range(D):
            if not len(assignment[d]):
                out.append((0.0, 0.0, 0.0))
                continue
            comm = bd.comm_ms[d]
            if self.comm_model:
                w = sum(self.task.tables[i].dim for i in assignment[d])
                comm = comm_model_ms(self.task.batch_size, w, -1, D)
            out.append((bd.fwd_ms[d], bd.bwd_ms[d], comm))
        return out

    def overall(self, placement):
        self.calls += 1
        p = np.ascontiguousarray(placement, dtype=np.int32)
        return self._measure(p, np.arange(len(p))).overall_ms


# ---------------------------------------------------------------------------
# checkpoint.hpp (DSHD) and the GPU evaluator

REDUCTIONS = {"sum": 0, "mean": 1, "max": 2}


class CostNetTrainer:
    """GPU training of the cost network (sp_costnet_trainer): the parameters
    stay on the device; each step is costnet_loss_and_grad + Adam with linear
    decay (costnet.hpp:349-446, nn.hpp:163-200) in fp64.

    A batch is a dict: n, dev_off[n+1], tab_off[devices+1], tab_row (feature
    row of each table), target_q[devices][3], target_overall[n] (NaN = none).
    """

    N_PARAMS = 15652

    def __init__(self, params, features, mask=None, red_tables: int = 0,
                 red_devices: int = 2, table_output_relu: bool = False, lr: float = 5e-4,
                 total_steps: int = 0, device: int = 0):
        p = np.ascontiguousarray(params, dtype=np.float64)
        f = np.ascontiguousarray(features, dtype=np.float64)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.float64)
        h = ctypes.c_void_p()
        check(lib().sp_costnet_trainer_create(_ptr(p), p.size, _ptr(f), f.shape[0],
                                              _ptr(m) if m is not None else None, red_tables,
                                              red_devices, int(table_output_relu), lr,
                                              total_steps, device, ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().sp_costnet_trainer_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass

    @staticmethod
    def _batch(b):
        arrs = {k: np.ascontiguousarray(b[k], dtype=np.int32) for k in ("dev_off", "tab_off",
                                                                         "tab_row")}
        arrs["target_q"] = np.ascontiguousarray(b["target_q"], dtype=np.float64)
        arrs["target_overall"] = np.ascontiguousarray(b["target_overall"], dtype=np.float64)
        sb = SpCostnetBatch(int(b["n"]), arrs["dev_off"].ctypes.data,
                                 arrs["tab_off"].ctypes.data, arrs["tab_row"].ctypes.data,
                                 arrs["target_q"].ctypes.data,
                                 arrs["target_overall"].ctypes.data)
        return sb, arrs

    def loss_grad(self, batch):
        sb, keep = self._batch(batch)
        loss = ctypes.c_double()
        grad = np.zeros(self.N_PARAMS)
        check(lib().sp_costnet_loss_grad(self._h, ctypes.byref(sb), ctypes.byref(loss),
                                         _ptr(grad)))
        return loss.value, grad

    def step(self, batch) -> float:
        sb, keep = self._batch(batch)
        loss = ctypes.c_double()
        check(lib().sp_costnet_train_step(self._h, ctypes.byref(sb), ctypes.byref(loss)))
        return loss.value

    def state(self):
        p = np.zeros(self.N_PARAMS)
        m = np.zeros(self.N_PARAMS)
        v = np.zeros(self.N_PARAMS)
        st = ctypes.c_int64()
        check(lib().sp_costnet_trainer_get(self._h, _ptr(p), _ptr(m), _ptr(v), ctypes.byref(st)))
        return p, m, v, st.value


class PolicyTrainer:
    """GPU REINFORCE on the policy network (sp_policy_trainer):
    reinforce_loss_and_grad + Adam (policy.hpp:203-296) in fp64, parameters
    resident on the device. Episodes dict: n, row0[n], ntab[n], step_off[n+1],
    reward[n], dev_off[steps+1], action[steps], tab_off[devices+1], tab_id,
    legal[devices], q[devices][3]."""

    N_PARAMS = 9345
    _INT = ("row0", "ntab", "step_off", "dev_off", "action", "tab_off", "tab_id", "legal")

    def __init__(self, params, features, mask=None, lr: float = 5e-4, total_steps: int = 0,
                 device: int = 0):
        p = np.ascontiguousarray(params, dtype=np.float64)
        f = np.ascontiguousarray(features, dtype=np.float64)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.float64)
        h = ctypes.c_void_p()
        check(lib().sp_policy_trainer_create(_ptr(p), p.size, _ptr(f), f.shape[0],
                                             _ptr(m) if m is not None else None, lr,
                                             total_steps, device, ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().sp_policy_trainer_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass

    def _batch(self, eps):
        arrs = {k: np.ascontiguousarray(eps[k], dtype=np.int32) for k in self._INT}
        arrs["reward"] = np.ascontiguousarray(eps["reward"], dtype=np.float64)
        arrs["q"] = np.ascontiguousarray(eps["q"], dtype=np.float64)
        sb = SpReinforceBatch(int(eps["n"]), *[arrs[k].ctypes.data for k in (
            "row0", "ntab", "step_off", "reward", "dev_off", "action", "tab_off", "tab_id",
            "legal", "q")])
        return sb, arrs

    def loss_grad(self, eps, w_entropy: float):
        sb, keep = self._batch(eps)
        obj = ctypes.c_double()
        grad = np.zeros(self.N_PARAMS)
        check(lib().sp_reinforce_loss_grad(self._h, ctypes.byref(sb), w_entropy,
                                           ctypes.byref(obj), _ptr(grad)))
        return obj.value, grad

    def step(self, eps, w_entropy: float) -> float:
        sb, keep = self._batch(eps)
        obj = ctypes.c_double()
        check(lib().sp_reinforce_step(self._h, ctypes.byref(sb), w_entropy, ctypes.byref(obj)))
        return obj.value

    def state(self):
        p, m, v = (np.zeros(self.N_PARAMS) for _ in range(3))
        st = ctypes.c_int64()
        check(lib().sp_policy_trainer_get(self._h, _ptr(p), _ptr(m), _ptr(v), ctypes.byref(st)))
        return p, m, v, st.value


def costnet_subbatch(batch, picks):
    """The minibatch of samples `picks` of a batch dict (replay-buffer draws)."""
    dev_off, tab_off = batch["dev_off"], batch["tab_off"]
    do, to, rows, tq, tov = [0], [0], [], [], []
    for s in picks:
        for d in range(dev_off[s], dev_off[s + 1]):
            rows.extend(batch["tab_row"][tab_off[d]:tab_off[d + 1]])
            to.append(len(rows))
            tq.append(batch["target_q"][d])
        do.append(len(to) - 1)
        tov.append(batch["target_overall"][s])
    return {"n": len(picks), "dev_off": np.array(do), "tab_off": np.array(to),
            "tab_row": np.array(rows, dtype=np.int32), "target_q": np.array(tq).reshape(-1, 3),
            "target_overall": np.array(tov)}


@dataclass
class Checkpoint:
    """shardplan::Checkpoint (checkpoint.hpp:28-33), parameters in the flat
    Mlp layout (nn.hpp:21-53)."""

    sections: dict

    @property
    def feature_mean(self):
        return self.sections["feature_mean"]

    @property
    def feature_std(self):
        return self.sections["feature_std"]

    @property
    def feature_mask(self):
        return self.sections["feature_mask"]

    @property
    def reductions(self):
        r = self.sections["reductions"]
        return int(r[0]), int(r[1])


_SECTION_SIZES = {
    "cost.table_mlp": 6944, "cost.head_fwd": 2177, "cost.head_bwd": 2177,
    "cost.head_comm": 2177, "cost.head_overall": 2177, "policy.table_mlp": 6944,
    "policy.cost_mlp": 2336, "policy.head": 65, "feature_mean": 21, "feature_std": 21,
    "feature_mask": 21, "reductions": 2, "config": 24,
}


def load_checkpoint(path: str) -> Checkpoint:
    """DSHD reader (checkpoint.hpp:149-217): magic, u32 version, u32 count,
    then (u32 name_len, name, u64 n, f64[n]) sections, little-endian."""
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != b"DSHD":
        raise ShardplanError(10, f"{path}: not a checkpoint file")
    version, count = struct.unpack_from("<II", data, 4)
    if version != 1:
        raise ShardplanError(10, f"unsupported checkpoint version {version}")
    off = 12
    sections = {}
    for _ in range(count):
        (nl,) = struct.unpack_from("<I", data, off)
        off += 4
        name = data[off:off + nl].decode()
        off += nl
        (n,) = struct.unpack_from("<Q", data, off)
        off += 8
        if off + 8 * n > len(data):
            raise ShardplanError(10, "truncated checkpoint")
        sections[name] = np.frombuffer(data, dtype="<f8", count=n, offset=off).copy()
        off += 8 * n
    for name, size in _SECTION_SIZES.items():
        if name not in sections:
            raise ShardplanError(10, f"checkpoint missing section {name}")
        if len(sections[name]) != size:
            raise ShardplanError(10, f"section {name} has wrong length")
    return Checkpoint(sections)


class Evaluator:
    """Cost network + policy network of a checkpoint bound to one placement
    task on one GPU (sp_evaluator)."""

    def __init__(self, ckpt: Checkpoint, task: PlacementTask, device: int = 0):
        s = ckpt.sections
        self._keep = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in s.items()}
        k = self._keep
        dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
        rt, rd = ckpt.reductions
        self._nets = SpNets(dp(k["cost.table_mlp"]), dp(k["cost.head_fwd"]),
                            dp(k["cost.head_bwd"]), dp(k["cost.head_comm"]),
                            dp(k["cost.head_overall"]), dp(k["policy.table_mlp"]),
                            dp(k["policy.cost_mlp"]), dp(k["policy.head"]),
                            dp(k["feature_mean"]), dp(k["feature_std"]), dp(k["feature_mask"]),
                            rt, rd)
        self.task = task
        self.M = len(task.tables)
        self.D = task.num_devices
        self._specs = _specs(task.tables)
        h = ctypes.c_void_p()
        check(lib().sp_evaluator_create(ctypes.byref(self._nets), self._specs, self.M, self.D,
                                        float(task.mem_cap_gb), device, ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().sp_evaluator_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the library binding is gone
            pass

    def order(self) -> np.ndarray:
        """predicted_order (harness.hpp:131-137)."""
        o = np.zeros(self.M, dtype=np.int32)
        check(lib().sp_evaluator_order(self._h, _ptr(o)))
        return o

    def eval_batch(self, placements: np.ndarray):
        """EstimatedCostProvider::overall for each row (raw) + clamped q."""
        p = np.ascontiguousarray(placements, dtype=np.int32).reshape(-1, self.M)
        n = p.shape[0]
        overall = np.zeros(n, dtype=np.float32)
        q = np.zeros((n, self.D, 3), dtype=np.float32)
        check(lib().sp_eval_batch(self._h, _ptr(p), n, _ptr(overall), _ptr(q)))
        return overall, q

    def rollout(self, n: int, mode: str = "greedy", uniforms: Optional[np.ndarray] = None,
                precision: str = "guarded"):
        """n estimated-MDP rollouts (greedy = Alg. 2 infer; sample = policy
        sampling with one uniform per step). Returns (placements [n, M],
        predicted overall [n], status [n], n_refined)."""
        m = {"greedy": 0, "sample": 1}[mode]
        prec = {"guarded": 0, "fp64": 1, "fp32": 2}[precision]
        if m == 1:
            if uniforms is None:
                raise ShardplanError(10, "sampled rollouts need uniforms [n, M]")
            u = np.ascontiguousarray(uniforms, dtype=np.float64).reshape(n, self.M)
            up = _ptr(u)
        else:
            u = None
            up = None
        pl = np.zeros((n, self.M), dtype=np.int32)
        pred = np.zeros(n, dtype=np.float64)
        st = np.zeros(n, dtype=np.int32)
        nref = ctypes.c_int32()
        check(lib().sp_rollout_batch(self._h, m, up, n, prec, _ptr(pl), _ptr(pred), _ptr(st),
                                     ctypes.byref(nref)))
        return pl, pred, st, nref.value


def infer(ckpt: Checkpoint, task: PlacementTask, device: int = 0):
    """harness.hpp:332-356 infer() on the GPU: (placement, predicted_ms).

    Infeasibility is a hard error, as in the reference."""
    ev = Evaluator(ckpt, task, device)
    try:
        pl, pred, st, _ = ev.rollout(1, "greedy")
    finally:
        ev.close()
    if st[0] != 0:
        raise ShardplanError(int(st[0]), "no device can hold the next table")
    return pl[0], max(0.0, float(pred[0]))


# ---------------------------------------------------------------------------
# baselines.hpp: greedy expert placements (host, microseconds)

EXPERT_STRATEGIES = ("size", "dim", "lookup", "size-lookup")


def expert_cost(strategy: str, t: TableDesc) -> float:
    """baselines.hpp:81-110."""
    if strategy == "size":
        return t.table_size_gb
    if strategy == "dim":
        return float(t.dim)
    if strategy == "lookup":
        return t.dim * t.pooling_factor
    if strategy == "size-lookup":
        return t.dim * t.pooling_factor * t.table_size_gb
    raise ShardplanError(10, f"unknown expert strategy: {strategy}")


def greedy_placement(task: PlacementTask, cost_fn) -> np.ndarray:
    """baselines.hpp:47-79: LPT greedy; sort ties to the lower id, device
    ties to the lower index; infeasible when a table fits nowhere."""
    D = task.num_devices
    cost = [cost_fn(t) for t in task.tables]
    order = sorted(range(len(cost)), key=lambda i: (-cost[i], i))
    load = [0.0] * D
    mem = [0.0] * D
    p = np.zeros(len(cost), dtype=np.int32)
    for i in order:
        need = task.tables[i].table_size_gb
        best = -1
        for d in range(D):
            if mem[d] + need > task.mem_cap_gb:
                continue
            if best < 0 or load[d] < load[best]:
                best = d
        if best < 0:
            raise ShardplanError(1, f"table {i} does not fit on any device")
        p[i] = best
        load[best] += cost[i]
        mem[best] += need
    return p


def random_placement(task: PlacementTask, seed: int = 0) -> np.ndarray:
    """baselines.hpp:23-41: table by table in id order, uniform over the
    devices that still have room (numpy's PCG64 stream here, not the
    reference's mt19937_64: a baseline, not a parity target)."""
    rng = np.random.default_rng(seed)
    mem = [0.0] * task.num_devices
    p = np.zeros(len(task.tables), dtype=np.int32)
    for i, t in enumerate(task.tables):
        legal = [d for d in range(task.num_devices)
                 if task.mem_cap_gb <= 0 or mem[d] + t.table_size_gb <= task.mem_cap_gb]
        if not legal:
            raise ShardplanError(1, f"table {i} does not fit on any device")
        d = legal[int(rng.integers(len(legal)))]
        p[i] = d
        mem[d] += t.table_size_gb
    return p


def expert_placement(task: PlacementTask, strategy: str) -> np.ndarray:
    return greedy_placement(task, lambda t: expert_cost(strategy, t))


def synth_lookup_batch(tables: Sequence[TableDesc], batch_size: int, seed: int,
                       device: int = 0, pinned: bool = False):
    """Host LookupBatch from the SURVEY §8d generator (run on the GPU).

    With pinned=True the arrays live in page-locked HostBuffers (returned
    as the third element to keep them alive)."""
    specs = _specs(tables)
    T = len(tables)
    nnz = ctypes.c_int64()
    if pinned:
        ob = HostBuffer(T * batch_size + 1, np.int64)
        off = ob.array
    else:
        ob = None
        off = np.zeros(T * batch_size + 1, dtype=np.int64)
    check(lib().sp_synth_lookup_batch(specs, T, batch_size, seed, device, _ptr(off), None,
                                      ctypes.byref(nnz)))
    if pinned:
        ib = HostBuffer(nnz.value, np.int64)
        idx = ib.array
    else:
        ib = None
        idx = np.zeros(nnz.value, dtype=np.int64)
    check(lib().sp_synth_lookup_batch(specs, T, batch_size, seed, device, _ptr(off), _ptr(idx),
                                      ctypes.byref(nnz)))
    return LookupBatch(idx, off, T, batch_size), (ob, ib)
