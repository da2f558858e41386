"""ctypes face of oracle/_build/liblookup_oracle.so — the CPU restatement of
the lookup path (see oracle/lookup_oracle.h for what it restates and the
import rule: tests/, smoke() and bench.py's CPU legs only)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liblookup_oracle.so")

_lib = None
c_vp = ctypes.c_void_p


def build():
    env = dict(os.environ)
    env.pop("CXX", None)
    subprocess.run(["make", "-C", HERE, "all"], check=True, capture_output=True, env=env)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.or_mix64.restype = ctypes.c_uint64
        L.or_mix64.argtypes = [ctypes.c_uint64]
        L.or_bag_len.restype = ctypes.c_int64
        L.or_bag_len.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_double]
        L.or_bag_index.restype = ctypes.c_int64
        L.or_bag_index.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64,
                                   ctypes.c_int64, ctypes.c_int64, ctypes.c_double]
        L.or_weight.restype = ctypes.c_float
        L.or_weight.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32]
        L.or_grad.restype = ctypes.c_float
        L.or_grad.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64]
        L.or_hot_mass.restype = ctypes.c_double
        L.or_hot_mass.argtypes = [c_vp]
        L.or_synth_batch.argtypes = [ctypes.c_int32, ctypes.c_int32, c_vp, c_vp, c_vp,
                                     ctypes.c_uint64, c_vp, c_vp, ctypes.c_int32]
        L.or_tbe_forward.argtypes = [ctypes.c_int32, c_vp, c_vp, c_vp, ctypes.c_uint64, c_vp,
                                     c_vp, c_vp, ctypes.c_int32, ctypes.c_int64,
                                     ctypes.c_int64, c_vp, ctypes.c_int64, c_vp,
                                     ctypes.c_int32]
        L.or_sorted_keys.restype = ctypes.c_int64
        L.or_sorted_keys.argtypes = [ctypes.c_int32, c_vp, c_vp, c_vp, c_vp, ctypes.c_int32,
                                     c_vp, c_vp]
        L.or_segments.restype = ctypes.c_int64
        L.or_segments.argtypes = [c_vp, ctypes.c_int64, c_vp, c_vp]
        L.or_tbe_backward_sgd.argtypes = [ctypes.c_int32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                          ctypes.c_int32, c_vp, ctypes.c_int64, c_vp,
                                          ctypes.c_float, ctypes.c_int32]
        L.or_tbe_backward_rowsums.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                              c_vp, c_vp, ctypes.c_int32, c_vp,
                                              ctypes.c_int64, ctypes.c_int64, c_vp]
        L.or_ingest.restype = ctypes.c_int32
        L.or_ingest.argtypes = [c_vp, ctypes.c_int64, c_vp, ctypes.c_int64, ctypes.c_int32,
                                ctypes.c_int32, c_vp, c_vp]
        L.or_access_count_bin.restype = ctypes.c_int32
        L.or_access_count_bin.argtypes = [ctypes.c_int64]
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def hot_mass(dist17) -> float:
    d = np.ascontiguousarray(dist17, dtype=np.float64)
    return lib().or_hot_mass(_p(d))


def synth_batch(tables, B: int, seed: int, nthreads: int = 0):
    """SURVEY §8d generator: returns (offsets int64 [T*B+1], indices int64)."""
    T = len(tables)
    pf = np.array([t["pooling_factor"] for t in tables], dtype=np.float64)
    rows = np.array([t["hash_size"] for t in tables], dtype=np.int64)
    hm = np.array([hot_mass(t["dist"]) for t in tables], dtype=np.float64)
    off = np.zeros(T * B + 1, dtype=np.int64)
    lib().or_synth_batch(T, B, _p(pf), _p(rows), _p(hm), seed, _p(off), None, nthreads)
    idx = np.zeros(int(off[-1]), dtype=np.int64)
    lib().or_synth_batch(T, B, _p(pf), _p(rows), _p(hm), seed, _p(off), _p(idx), nthreads)
    return off, idx


def weights(seed: int, t: int, rows: int, dim: int) -> np.ndarray:
    """Materialise the generator's table t (small tables only)."""
    out = np.empty((rows, dim), dtype=np.float32)
    f = lib().or_weight
    for r in range(rows):
        for c in range(dim):
            out[r, c] = f(seed, t, r, c)
    return out


def tbe_forward(dims, rows, weights_list, offsets, indices, B, tables_list=None,
                wseed=0, bag_lo=0, bag_hi=None, nthreads=0):
    """Pooled [bag_hi-bag_lo, sum dims] in global table order (fp64 accumulate)."""
    dims = np.ascontiguousarray(dims, dtype=np.int32)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    T = len(dims)
    lst = np.arange(T, dtype=np.int32) if tables_list is None else \
        np.ascontiguousarray(tables_list, dtype=np.int32)
    gcol = np.zeros(T, dtype=np.int64)
    gcol[1:] = np.cumsum(dims)[:-1]
    W = int(dims.sum())
    if bag_hi is None:
        bag_hi = B
    out = np.zeros((bag_hi - bag_lo, W), dtype=np.float32)
    if weights_list is None:
        wp = None
    else:
        arrs = [np.ascontiguousarray(w, dtype=np.float32) if w is not None else None
                for w in weights_list]
        wp = (ctypes.c_void_p * T)(*[a.ctypes.data if a is not None else None for a in arrs])
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    lib().or_tbe_forward(B, _p(dims), _p(rows), wp, wseed, _p(offsets), _p(indices),
                         _p(lst), len(lst), bag_lo, bag_hi, _p(out), W, _p(gcol), nthreads)
    return out


def sorted_keys(rows, offsets, indices, B, tables_list):
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    lst = np.ascontiguousarray(tables_list, dtype=np.int32)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    n = lib().or_sorted_keys(B, _p(rows), _p(offsets), _p(indices), _p(lst), len(lst), None, None)
    keys = np.zeros(n, dtype=np.uint32)
    bags = np.zeros(n, dtype=np.uint32)
    lib().or_sorted_keys(B, _p(rows), _p(offsets), _p(indices), _p(lst), len(lst), _p(keys),
                         _p(bags))
    heads = np.zeros(n + 1, dtype=np.uint32)
    nu = lib().or_segments(_p(keys), n, None, _p(heads))
    return keys, bags, heads[:nu]


def tbe_backward_sgd(dims, rows, weights_list, offsets, indices, B, grad, lr, tables_list):
    """Applies the row-wise SGD in place to copies of weights_list; returns them."""
    dims = np.ascontiguousarray(dims, dtype=np.int32)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    T = len(dims)
    gcol = np.zeros(T, dtype=np.int64)
    gcol[1:] = np.cumsum(dims)[:-1]
    W = int(dims.sum())
    ws = [np.array(w, dtype=np.float32, copy=True) if w is not None else None
          for w in weights_list]
    wp = (ctypes.c_void_p * T)(*[a.ctypes.data if a is not None else None for a in ws])
    g = np.ascontiguousarray(grad, dtype=np.float32).reshape(B, W)
    lst = np.ascontiguousarray(tables_list, dtype=np.int32)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    lib().or_tbe_backward_sgd(B, _p(dims), _p(rows), wp, _p(offsets), _p(indices), _p(lst),
                              len(lst), _p(g), W, _p(gcol), lr, 0)
    return ws


def tbe_backward_sgd_inplace(dims, rows, weights_list, offsets, indices, B, grad, lr,
                             tables_list, nthreads=0):
    """Row-wise SGD applied in place to weights_list (fp32 C-contiguous)."""
    dims = np.ascontiguousarray(dims, dtype=np.int32)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    T = len(dims)
    gcol = np.zeros(T, dtype=np.int64)
    gcol[1:] = np.cumsum(dims)[:-1]
    W = int(dims.sum())
    wp = (ctypes.c_void_p * T)(*[a.ctypes.data if a is not None else None
                                 for a in weights_list])
    g = np.ascontiguousarray(grad, dtype=np.float32).reshape(B, W)
    lst = np.ascontiguousarray(tables_list, dtype=np.int32)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    lib().or_tbe_backward_sgd(B, _p(dims), _p(rows), wp, _p(offsets), _p(indices), _p(lst),
                              len(lst), _p(g), W, _p(gcol), lr, nthreads)


def grad_matrix(seed: int, B: int, W: int) -> np.ndarray:
    f = lib().or_grad
    out = np.empty((B, W), dtype=np.float32)
    for b in range(B):
        for c in range(W):
            out[b, c] = f(seed, b, c)
    return out


def ingest(offsets, indices, T, B):
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    pf = np.zeros(max(T, 1))
    dist = np.zeros((max(T, 1), 17))
    rc = lib().or_ingest(_p(offsets), len(offsets), _p(indices), len(indices), T, B, _p(pf),
                         _p(dist))
    return rc, pf[:T], dist[:T]
