"""ctypes binding of the in-tree CUDA library `_shardplan_b200.so`.

Loading fails loudly: there is no CPU fallback anywhere in this package.
The ABI is declared in include/shardplan_b200.h.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SP_LIBRARY") or os.path.join(HERE, "_shardplan_b200.so")  # SP_LIBRARY: A/B builds

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_f32 = ctypes.c_float
c_f64 = ctypes.c_double
c_vp = ctypes.c_void_p
P = ctypes.POINTER

ABI_VERSION = 2  # SP_ABI_VERSION of include/shardplan_b200.h

# Every function the header declares, with (restype, argtypes).
SIGNATURES = {
    "sp_abi_version": (c_i32, []),
    "sp_last_error": (ctypes.c_char_p, []),
    "sp_kernel_launches": (c_u64, []),
    "sp_nccl_unique_id": (c_i32, [c_vp]),
    "sp_ctx_create": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_i32, c_f64, c_f32, c_i32,
                              c_i32, c_vp, c_i32, P(c_vp)]),
    "sp_ctx_create_ex": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_i32, c_f64, c_f32, c_i32,
                                 c_i32, c_vp, c_i32, c_i32, P(c_vp)]),
    "sp_ctx_destroy": (None, [c_vp]),
    "sp_ctx_stream": (c_i32, [c_vp, P(c_vp)]),
    "sp_ctx_device_bytes": (c_i32, [c_vp, P(c_u64)]),
    "sp_ctx_local_tables": (c_i32, [c_vp, c_vp, P(c_i32)]),
    "sp_init_tables": (c_i32, [c_vp, c_u64]),
    "sp_set_table": (c_i32, [c_vp, c_i32, c_vp]),
    "sp_get_table": (c_i32, [c_vp, c_i32, c_vp]),
    "sp_upload_batch": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_i64]),
    "sp_upload_batch_file": (c_i32, [c_vp, ctypes.c_char_p]),
    "sp_synth_batch": (c_i32, [c_vp, c_u64]),
    "sp_batch_nnz": (c_i32, [c_vp, P(c_i64)]),
    "sp_synth_lookup_batch": (c_i32, [c_vp, c_i32, c_i32, c_u64, c_i32, c_vp, c_vp, P(c_i64)]),
    "sp_exchange_plan": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp,
                                 c_vp, c_vp]),
    "sp_forward": (c_i32, [c_vp]),
    "sp_a2a_forward": (c_i32, [c_vp]),
    "sp_a2a_backward": (c_i32, [c_vp]),
    "sp_backward_sgd": (c_i32, [c_vp]),
    "sp_set_grad": (c_i32, [c_vp, c_vp]),
    "sp_synth_grad": (c_i32, [c_vp, c_u64]),
    "sp_get_pooled": (c_i32, [c_vp, c_vp]),
    "sp_get_local_pooled": (c_i32, [c_vp, c_i32, c_vp]),
    "sp_get_sorted": (c_i32, [c_vp, c_i32, c_vp, c_vp, P(c_i64), c_vp, P(c_i64)]),
    "sp_run_iteration": (c_i32, [c_vp, c_vp]),
    "sp_run_local": (c_i32, [c_vp, c_vp]),
    "sp_run_batch": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "sp_run_batches": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sp_enqueue_iteration": (c_i32, [c_vp]),
    "sp_graph_replay": (c_i32, [c_vp, c_i32, P(c_i32)]),
    "sp_ctx_algorithmic_bytes": (c_i32, [c_vp, P(c_f64)]),
    "sp_ctx_set_comm_model": (c_i32, [c_vp, c_i32]),
    "sp_comm_model": (c_i32, [c_i32, c_i64, c_i64, c_i32, P(c_f64)]),
    "sp_ctx_set_profiling": (c_i32, [c_vp, c_i32]),
    "sp_ctx_set_overlap": (c_i32, [c_vp, c_i32]),
    "sp_ctx_set_sort_target": (c_i32, [c_vp, c_i64]),
    "sp_ctx_set_upload_chunk": (c_i32, [c_vp, c_i64]),
    "sp_costnet_trainer_create": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i32, c_i32, c_i32,
                                          c_f64, c_i64, c_i32, P(c_vp)]),
    "sp_costnet_trainer_destroy": (None, [c_vp]),
    "sp_costnet_loss_grad": (c_i32, [c_vp, c_vp, P(c_f64), c_vp]),
    "sp_costnet_train_step": (c_i32, [c_vp, c_vp, P(c_f64)]),
    "sp_costnet_trainer_get": (c_i32, [c_vp, c_vp, c_vp, c_vp, P(c_i64)]),
    "sp_policy_trainer_create": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_vp, c_f64, c_i64, c_i32,
                                         P(c_vp)]),
    "sp_policy_trainer_destroy": (None, [c_vp]),
    "sp_reinforce_loss_grad": (c_i32, [c_vp, c_vp, c_f64, P(c_f64), c_vp]),
    "sp_reinforce_step": (c_i32, [c_vp, c_vp, c_f64, P(c_f64)]),
    "sp_policy_trainer_get": (c_i32, [c_vp, c_vp, c_vp, c_vp, P(c_i64)]),
    "sp_ipc_export": (c_i32, [c_vp, c_vp]),
    "sp_ipc_import": (c_i32, [c_vp, c_vp]),
    "sp_ctx_synchronize": (c_i32, [c_vp]),
    "sp_ctx_kernel_ms": (c_i32, [c_vp, P(c_f64), P(c_i64)]),
    "sp_host_alloc": (c_i32, [c_u64, P(c_vp)]),
    "sp_host_free": (None, [c_vp]),
    "sp_ingest_lookup_batch": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_vp, c_vp,
                                       c_i32, c_i32, c_vp]),
    "sp_ingest_batch_file": (c_i32, [ctypes.c_char_p, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp,
                                     P(c_i32), P(c_i32)]),
    "sp_evaluator_create": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_f64, c_i32, P(c_vp)]),
    "sp_evaluator_destroy": (None, [c_vp]),
    "sp_evaluator_order": (c_i32, [c_vp, c_vp]),
    "sp_eval_batch": (c_i32, [c_vp, c_vp, c_i32, c_vp, c_vp]),
    "sp_rollout_batch": (c_i32, [c_vp, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp,
                                 P(c_i32)]),
}


class SpTableSpec(ctypes.Structure):
    """sp_table_spec == shardplan::TableDesc (table.hpp:45-52)."""

    _fields_ = [
        ("id", c_i32),
        ("dim", c_i32),
        ("hash_size", c_i64),
        ("pooling_factor", c_f64),
        ("table_size_gb", c_f64),
        ("dist", c_f64 * 17),
    ]


class SpCostnetBatch(ctypes.Structure):
    """sp_costnet_batch: a CostSample list (costnet.hpp:297-304)."""

    _fields_ = [
        ("n_samples", c_i32),
        ("dev_off", c_vp),
        ("tab_off", c_vp),
        ("tab_row", c_vp),
        ("target_q", c_vp),
        ("target_overall", c_vp),
    ]


class SpReinforceBatch(ctypes.Structure):
    """sp_reinforce_batch: an Episode list (policy.hpp:189-201)."""

    _fields_ = [("n_episodes", c_i32)] + [(k, c_vp) for k in (
        "row0", "ntab", "step_off", "reward", "dev_off", "action", "tab_off", "tab_id",
        "legal", "q")]


class SpBreakdown(ctypes.Structure):
    """sp_breakdown == shardplan::CostBreakdown numbers (oracle.hpp:105-116)."""

    _fields_ = [
        ("fwd_ms", P(c_f64)),
        ("bwd_ms", P(c_f64)),
        ("comm_ms", P(c_f64)),
        ("fwd_comm_stage_ms", c_f64),
        ("bwd_comm_stage_ms", c_f64),
        ("overall_ms", c_f64),
    ]


class SpNets(ctypes.Structure):
    _fields_ = [
        ("cost_table", P(c_f64)),
        ("cost_fwd", P(c_f64)),
        ("cost_bwd", P(c_f64)),
        ("cost_comm", P(c_f64)),
        ("cost_overall", P(c_f64)),
        ("pol_table", P(c_f64)),
        ("pol_cost", P(c_f64)),
        ("pol_head", P(c_f64)),
        ("feature_mean", P(c_f64)),
        ("feature_std", P(c_f64)),
        ("feature_mask", P(c_f64)),
        ("reduction_tables", c_i32),
        ("reduction_devices", c_i32),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """The loaded library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2210_02023_b200.build`"
                " (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        L.sp_abi_version.restype = c_i32
        if L.sp_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI {L.sp_abi_version()}, this binding expects "
                              f"{ABI_VERSION}: rebuild it (python -m paper_2210_02023_b200.build)")
        for name, (res, args) in SIGNATURES.items():
            if not hasattr(L, name):
                continue  # tests/test_abi.py asserts every header symbol exists
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


# ErrorKind (error.hpp:11-22) + 1, plus device failures.
STATUS_NAMES = {
    0: "ok", 1: "infeasible", 2: "memory_violation", 3: "malformed_batch", 4: "bad_spec",
    5: "unknown_table", 6: "too_large", 7: "illegal_action", 8: "shape_mismatch",
    9: "no_legal_action", 10: "bad_input", 11: "cuda", 12: "nccl",
}


class ShardplanError(RuntimeError):
    """Mirror of shardplan::Error (error.hpp:24-45): `kind` + message.

    exit_code follows Error::exit_code(): 2 for infeasible/memory, else 3."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.kind = STATUS_NAMES.get(status, f"status{status}")
        super().__init__(f"{self.kind}: {message}")

    @property
    def exit_code(self) -> int:
        return 2 if self.kind in ("infeasible", "memory_violation") else 3


def check(status: int) -> None:
    if status != 0:
        raise ShardplanError(status, lib().sp_last_error().decode(errors="replace"))
