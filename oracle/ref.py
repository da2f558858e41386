"""ctypes face of oracle/_ref/libshardplan_ref.so — the UNMODIFIED reference
(/root/reference/proj/include/shardplan) compiled by oracle/Makefile.

TEST INFRASTRUCTURE ONLY (tests/, golden-fixture generation, bench.py's
reference arm). The product package never imports this module.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libshardplan_ref.so")

c_double_p = ctypes.POINTER(ctypes.c_double)
c_i32_p = ctypes.POINTER(ctypes.c_int32)
c_i64_p = ctypes.POINTER(ctypes.c_int64)


class Spec(ctypes.Structure):
    """sp_table_spec == shardplan::TableDesc (table.hpp:45-52)."""

    _fields_ = [
        ("id", ctypes.c_int32),
        ("dim", ctypes.c_int32),
        ("hash_size", ctypes.c_int64),
        ("pooling_factor", ctypes.c_double),
        ("table_size_gb", ctypes.c_double),
        ("dist", ctypes.c_double * 17),
    ]


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(
                f"{LIB_PATH} missing: run `make -C oracle ref` where /root/reference exists")
        L = ctypes.CDLL(LIB_PATH)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_device_comm.restype = ctypes.c_double
        L.ref_device_comm.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.ref_fusion_speedup.restype = ctypes.c_double
        L.ref_fusion_speedup.argtypes = [ctypes.c_int]
        L.ref_table_memory_gb.restype = ctypes.c_double
        L.ref_table_memory_gb.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        L.ref_access_count_bin.argtypes = [ctypes.c_int64]
        L.ref_synth_pool.argtypes = [
            ctypes.c_int, c_i32_p, c_double_p, ctypes.c_int, ctypes.c_double,
            ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
            ctypes.c_void_p, c_double_p, c_double_p]
        L.ref_ingest.argtypes = [
            c_i64_p, ctypes.c_int64, c_i64_p, ctypes.c_int64, ctypes.c_int,
            ctypes.c_int, c_i32_p, c_i64_p, ctypes.c_int, ctypes.c_void_p,
            c_double_p, c_double_p]
        L.ref_validate_batch.argtypes = [c_i64_p, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int, ctypes.c_int]
        L.ref_evaluate_placement.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
            ctypes.c_int, c_i32_p, c_double_p, c_double_p, c_double_p,
            c_double_p, c_double_p]
        L.ref_expert_placement.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
            ctypes.c_int, ctypes.c_int, c_i32_p]
        L.ref_random_placement.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
            ctypes.c_int, ctypes.c_uint64, c_i32_p]
        L.ref_rng_u01.argtypes = [ctypes.c_uint64, ctypes.c_int64, c_double_p]
        L.ref_subseed.restype = ctypes.c_uint64
        L.ref_subseed.argtypes = [ctypes.c_uint64, ctypes.c_char_p]
        L.ref_train.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_uint64, ctypes.c_char_p]
        L.ref_infer.argtypes = [
            ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
            ctypes.c_double, ctypes.c_int, c_i32_p, c_double_p, c_i32_p]
        L.ref_sampled_rollouts.argtypes = [
            ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
            ctypes.c_double, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
            c_i32_p, c_double_p]
        L.ref_costnet_overall.argtypes = [
            ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
            c_i32_p, ctypes.c_int, c_double_p, c_double_p]
        L.ref_task_features.argtypes = [
            ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int, c_double_p, c_double_p]
        L.ref_action_probs.argtypes = [
            ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
            c_i32_p, c_double_p, c_i32_p, c_double_p]
        L.ref_feature_vector.argtypes = [ctypes.c_void_p, c_double_p, c_double_p,
                                         c_double_p]
        L.ref_rng_index.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, c_i64_p]
        _cost = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, c_double_p,
                 ctypes.c_int64, ctypes.c_int, c_i32_p, c_i32_p, c_i32_p, c_double_p,
                 c_double_p]
        L.ref_costnet_loss_grad.argtypes = [c_double_p] + _cost + [c_double_p, c_double_p]
        L.ref_costnet_train_steps.argtypes = [c_double_p] + _cost + [
            ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int64, ctypes.c_uint64,
            c_double_p]
        _ep = [ctypes.c_void_p, c_double_p, ctypes.c_int, c_i32_p, c_i32_p, c_i32_p,
               c_double_p, c_i32_p, c_i32_p, c_i32_p, c_i32_p, c_i32_p, c_double_p,
               ctypes.c_double]
        L.ref_reinforce_loss_grad.argtypes = [c_double_p] + _ep + [c_double_p, c_double_p]
        L.ref_reinforce_updates.argtypes = [c_double_p] + _ep + [
            ctypes.c_int, ctypes.c_double, ctypes.c_int64, c_double_p]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


# ---- table descriptors as numpy-friendly dicts ---------------------------

def specs_to_array(tables) -> ctypes.Array:
    arr = (Spec * len(tables))()
    for i, t in enumerate(tables):
        arr[i].id = int(t["id"])
        arr[i].dim = int(t["dim"])
        arr[i].hash_size = int(t["hash_size"])
        arr[i].pooling_factor = float(t["pooling_factor"])
        arr[i].table_size_gb = float(t["table_size_gb"])
        for b in range(17):
            arr[i].dist[b] = float(t["dist"][b])
    return arr


def array_to_specs(arr) -> list:
    return [
        {"id": s.id, "dim": s.dim, "hash_size": s.hash_size,
         "pooling_factor": s.pooling_factor, "table_size_gb": s.table_size_gb,
         "dist": list(s.dist)}
        for s in arr
    ]


def synth_pool(num_tables, dim_choices, hash_log10=(4.5, 7.3), pooling_exponent=1.7,
               pooling_max=200.0, hot_fraction=(0.0, 0.8), batch=65536,
               bytes_per_param=2, seed=1):
    """synth_pool (synth.hpp:72-119)."""
    dims = np.array([d for d, _ in dim_choices], dtype=np.int32)
    ws = np.array([w for _, w in dim_choices], dtype=np.float64)
    out = (Spec * num_tables)()
    mean = np.zeros(21)
    std = np.zeros(21)
    _check(lib().ref_synth_pool(num_tables, _p(dims, ctypes.c_int32), _p(ws, ctypes.c_double),
                                len(dims), hash_log10[0], hash_log10[1], pooling_exponent,
                                pooling_max, hot_fraction[0], hot_fraction[1], batch,
                                bytes_per_param, seed, out, _p(mean, ctypes.c_double),
                                _p(std, ctypes.c_double)))
    return array_to_specs(out), mean, std


def ingest(offsets, indices, T, B, dims, hash_sizes, bytes_per_param=2):
    """ingest_lookup_batch (table.hpp:188-232)."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    dims = np.ascontiguousarray(dims, dtype=np.int32)
    hs = np.ascontiguousarray(hash_sizes, dtype=np.int64)
    out = (Spec * max(T, 1))()
    mean = np.zeros(21)
    std = np.zeros(21)
    _check(lib().ref_ingest(_p(offsets, ctypes.c_int64), len(offsets), _p(indices, ctypes.c_int64),
                            len(indices), T, B, _p(dims, ctypes.c_int32), _p(hs, ctypes.c_int64),
                            bytes_per_param, out, _p(mean, ctypes.c_double),
                            _p(std, ctypes.c_double)))
    return array_to_specs(out)[:T], mean, std


def save_lookup_batch(path, offsets, indices, T, B):
    """save_lookup_batch (table.hpp:268-281)."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    _check(lib().ref_save_lookup_batch(str(path).encode(), _p(offsets, ctypes.c_int64),
                                       len(offsets), _p(indices, ctypes.c_int64), len(indices),
                                       T, B))


def load_lookup_batch(path):
    """load_lookup_batch (table.hpp:283-305) -> (offsets, indices, T, B)."""
    n_off, n_idx = ctypes.c_int64(0), ctypes.c_int64(0)
    T, B = ctypes.c_int(0), ctypes.c_int(0)
    _check(lib().ref_load_lookup_batch(str(path).encode(), None, ctypes.byref(n_off), None,
                                       ctypes.byref(n_idx), ctypes.byref(T), ctypes.byref(B)))
    offsets = np.zeros(max(n_off.value, 1), dtype=np.int64)
    indices = np.zeros(max(n_idx.value, 1), dtype=np.int64)
    _check(lib().ref_load_lookup_batch(str(path).encode(), _p(offsets, ctypes.c_int64),
                                       ctypes.byref(n_off), _p(indices, ctypes.c_int64),
                                       ctypes.byref(n_idx), ctypes.byref(T), ctypes.byref(B)))
    return offsets[:n_off.value], indices[:n_idx.value], T.value, B.value


def evaluate_placement(tables, D, cap, B, placement):
    """CostOracle::evaluate_placement (oracle.hpp:187-240)."""
    arr = specs_to_array(tables)
    p = np.ascontiguousarray(placement, dtype=np.int32)
    fwd, bwd, comm = np.zeros(D), np.zeros(D), np.zeros(D)
    stage = np.zeros(1)
    overall = np.zeros(1)
    _check(lib().ref_evaluate_placement(arr, len(tables), D, cap, B, _p(p, ctypes.c_int32),
                                        _p(fwd, ctypes.c_double), _p(bwd, ctypes.c_double),
                                        _p(comm, ctypes.c_double), _p(stage, ctypes.c_double),
                                        _p(overall, ctypes.c_double)))
    return {"fwd_ms": fwd, "bwd_ms": bwd, "comm_ms": comm, "stage_ms": float(stage[0]),
            "overall_ms": float(overall[0])}


EXPERT = {"size": 0, "dim": 1, "lookup": 2, "size-lookup": 3}


def expert_placement(tables, D, cap, B, strategy):
    arr = specs_to_array(tables)
    out = np.zeros(len(tables), dtype=np.int32)
    _check(lib().ref_expert_placement(arr, len(tables), D, cap, B, EXPERT[strategy],
                                      _p(out, ctypes.c_int32)))
    return out


def random_placement(tables, D, cap, B, seed):
    arr = specs_to_array(tables)
    out = np.zeros(len(tables), dtype=np.int32)
    _check(lib().ref_random_placement(arr, len(tables), D, cap, B, seed, _p(out, ctypes.c_int32)))
    return out


def rng_u01(seed, n):
    out = np.zeros(n)
    lib().ref_rng_u01(seed, n, _p(out, ctypes.c_double))
    return out


def train(pool_tables, batch, num_tables, num_devices, mem_cap_gb, path, iterations=10,
          n_collect=10, n_cost=300, n_batch=64, n_rl=10, n_episode=10, seed=1):
    """harness.hpp:220 train() + checkpoint.hpp:114 save_checkpoint()."""
    arr = specs_to_array(pool_tables)
    _check(lib().ref_train(arr, len(pool_tables), batch, num_tables, num_devices, mem_cap_gb,
                           iterations, n_collect, n_cost, n_batch, n_rl, n_episode, seed,
                           path.encode()))


def infer(ckpt, tables, D, cap, B):
    """harness.hpp:332 infer(): greedy placement, predicted ms, visit order."""
    arr = specs_to_array(tables)
    M = len(tables)
    p = np.zeros(M, dtype=np.int32)
    order = np.zeros(M, dtype=np.int32)
    pred = np.zeros(1)
    _check(lib().ref_infer(ckpt.encode(), arr, M, D, cap, B, _p(p, ctypes.c_int32),
                           _p(pred, ctypes.c_double), _p(order, ctypes.c_int32)))
    return p, float(pred[0]), order


def sampled_rollouts(ckpt, tables, D, cap, B, seed, n):
    arr = specs_to_array(tables)
    M = len(tables)
    p = np.zeros((n, M), dtype=np.int32)
    overall = np.zeros(n)
    _check(lib().ref_sampled_rollouts(ckpt.encode(), arr, M, D, cap, B, seed, n,
                                      _p(p, ctypes.c_int32), _p(overall, ctypes.c_double)))
    return p, overall


def costnet_overall(ckpt, tables, D, placements):
    arr = specs_to_array(tables)
    placements = np.ascontiguousarray(placements, dtype=np.int32)
    n, M = placements.shape
    overall = np.zeros(n)
    q = np.zeros((n, D, 3))
    _check(lib().ref_costnet_overall(ckpt.encode(), arr, M, D, _p(placements, ctypes.c_int32), n,
                                     _p(overall, ctypes.c_double), _p(q, ctypes.c_double)))
    return overall, q


def task_features(ckpt, tables):
    arr = specs_to_array(tables)
    M = len(tables)
    rows = np.zeros((M, 21))
    single = np.zeros(M)
    _check(lib().ref_task_features(ckpt.encode(), arr, M, _p(rows, ctypes.c_double),
                                   _p(single, ctypes.c_double)))
    return rows, single


def action_probs(ckpt, tables, D, partial, q, legal):
    arr = specs_to_array(tables)
    partial = np.ascontiguousarray(partial, dtype=np.int32)
    q = np.ascontiguousarray(q, dtype=np.float64)
    legal = np.ascontiguousarray(legal, dtype=np.int32)
    probs = np.zeros(D)
    _check(lib().ref_action_probs(ckpt.encode(), arr, len(tables), D, _p(partial, ctypes.c_int32),
                                  _p(q, ctypes.c_double), _p(legal, ctypes.c_int32),
                                  _p(probs, ctypes.c_double)))
    return probs


def rng_index(seed, n, bound):
    """n draws of Rng(seed).index(bound) (rng.hpp:48-54)."""
    out = np.zeros(n, dtype=np.int64)
    lib().ref_rng_index(seed, n, bound, _p(out, ctypes.c_int64))
    return out


def _cost_args(batch, features, mask, red_tables, red_devices, table_relu):
    f = np.ascontiguousarray(features, dtype=np.float64)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.float64)
    return [red_tables, red_devices, table_relu,
            None if m is None else m.ctypes.data_as(ctypes.c_void_p),
            _p(f, ctypes.c_double), f.shape[0], batch["n"],
            _p(np.ascontiguousarray(batch["dev_off"], dtype=np.int32), ctypes.c_int32), _p(np.ascontiguousarray(batch["tab_off"], dtype=np.int32), ctypes.c_int32),
            _p(np.ascontiguousarray(batch["tab_row"], dtype=np.int32), ctypes.c_int32), _p(np.ascontiguousarray(batch["target_q"], dtype=np.float64), ctypes.c_double),
            _p(np.ascontiguousarray(batch["target_overall"], dtype=np.float64), ctypes.c_double)], (f, m)


def costnet_loss_grad(params, batch, features, mask=None, red_tables=0, red_devices=2,
                      table_relu=0):
    """costnet_loss_and_grad (costnet.hpp:349-427) of the reference."""
    p = np.ascontiguousarray(params, dtype=np.float64)
    args, keep = _cost_args(batch, features, mask, red_tables, red_devices, table_relu)
    grad = np.zeros_like(p)
    loss = np.zeros(1)
    _check(lib().ref_costnet_loss_grad(_p(p, ctypes.c_double), *args, _p(grad, ctypes.c_double),
                                       _p(loss, ctypes.c_double)))
    return float(loss[0]), grad


def costnet_train_steps(params, batch, features, n_steps, n_batch, lr, total_steps, seed,
                        mask=None, red_tables=0, red_devices=2, table_relu=0):
    """costnet_train_steps (costnet.hpp:431-446), batches from Rng(seed)."""
    p = np.array(params, dtype=np.float64, copy=True)
    args, keep = _cost_args(batch, features, mask, red_tables, red_devices, table_relu)
    ml = np.zeros(1)
    _check(lib().ref_costnet_train_steps(_p(p, ctypes.c_double), *args, n_steps, n_batch, lr,
                                         total_steps, seed, _p(ml, ctypes.c_double)))
    return p, float(ml[0])


_EP_INT = ("row0", "ntab", "step_off")
_EP_INT2 = ("dev_off", "action", "tab_off", "tab_id", "legal")


def _ep_args(eps, features, mask, w_entropy):
    f = np.ascontiguousarray(features, dtype=np.float64)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.float64)
    ints = {k: np.ascontiguousarray(eps[k], dtype=np.int32) for k in _EP_INT + _EP_INT2}
    rew = np.ascontiguousarray(eps["reward"], dtype=np.float64)
    q = np.ascontiguousarray(eps["q"], dtype=np.float64)
    args = [None if m is None else m.ctypes.data_as(ctypes.c_void_p), _p(f, ctypes.c_double),
            int(eps["n"])] + [_p(ints[k], ctypes.c_int32) for k in _EP_INT] + [
            _p(rew, ctypes.c_double)] + [_p(ints[k], ctypes.c_int32) for k in _EP_INT2] + [
            _p(q, ctypes.c_double), w_entropy]
    return args, (f, m, ints, rew, q)


def reinforce_loss_grad(params, eps, features, w_entropy, mask=None):
    """reinforce_loss_and_grad (policy.hpp:203-283) of the reference."""
    p = np.ascontiguousarray(params, dtype=np.float64)
    args, keep = _ep_args(eps, features, mask, w_entropy)
    grad = np.zeros_like(p)
    obj = np.zeros(1)
    _check(lib().ref_reinforce_loss_grad(_p(p, ctypes.c_double), *args,
                                         _p(grad, ctypes.c_double), _p(obj, ctypes.c_double)))
    return float(obj[0]), grad


def reinforce_updates(params, eps, features, w_entropy, n_updates, lr, total_steps, mask=None):
    p = np.array(params, dtype=np.float64, copy=True)
    args, keep = _ep_args(eps, features, mask, w_entropy)
    objs = np.zeros(n_updates)
    _check(lib().ref_reinforce_updates(_p(p, ctypes.c_double), *args, n_updates, lr,
                                       total_steps, _p(objs, ctypes.c_double)))
    return p, objs
