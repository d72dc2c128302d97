"""ctypes binding of the lsg C ABI (include/lsg.h).

The shared library is built in-tree (``make lib`` / ``__graft_entry__.build()``)
as ``paper_2211_00224_b200/libsolar_b200.so``. There is no fallback: if the
library is missing or a CUDA device is absent, every call raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsolar_b200.so")

HIT_BIT = 0x80000000
NEVER = 0xFFFFFFFE

# Reference ErrorClass codes (errors.hpp:11-18)
CONFIG, VALIDATION, CAPABILITY, CALIBRATION, STORAGE, INTERNAL = 2, 3, 4, 5, 6, 7


class LsgConfig(ctypes.Structure):
    """Field-for-field mirror of ``lsg_config`` (include/lsg.h)."""

    _fields_ = [
        ("dataset_size", ctypes.c_uint64),
        ("num_epochs", ctypes.c_uint32),
        ("num_nodes", ctypes.c_uint32),
        ("local_batch", ctypes.c_uint64),
        ("seed", ctypes.c_uint64),
        ("drop_last", ctypes.c_int32),
        ("policy", ctypes.c_int32),
        ("buffer_capacity", ctypes.c_uint64),
        ("graph_mode", ctypes.c_int32),
        ("insert_redundant", ctypes.c_int32),
        ("chunk_threshold", ctypes.c_uint64),
        ("optim_order", ctypes.c_int32),
        ("optim_remap", ctypes.c_int32),
        ("optim_balance", ctypes.c_int32),
        ("optim_chunk", ctypes.c_int32),
        ("pso_swarm", ctypes.c_uint32),
        ("pso_iters", ctypes.c_uint32),
        ("pso_stagnation", ctypes.c_uint32),
        ("pso_restart", ctypes.c_uint32),
        ("pso_p_personal", ctypes.c_double),
        ("pso_p_global", ctypes.c_double),
        ("pso_inertia", ctypes.c_double),
        ("pso_kick", ctypes.c_double),
    ]


class LsgShape(ctypes.Structure):
    _fields_ = [
        ("global_batch", ctypes.c_uint64),
        ("steps_per_epoch", ctypes.c_uint64),
        ("keep", ctypes.c_uint64),
        ("total_steps", ctypes.c_uint64),
        ("total_items", ctypes.c_uint64),
    ]


class LsgPlanOut(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "trace", "graph", "order", "cost", "hist", "iters", "items", "node_off",
        "fetch_before", "fetch_after", "read_start", "read_end", "read_count", "read_needed",
        "read_redundant")]


class LsgTraceText(ctypes.Structure):
    """Field-for-field mirror of ``lsg_trace_text`` (include/lsg.h)."""
    _fields_ = [("dataset_size", ctypes.c_uint64), ("num_epochs", ctypes.c_uint32),
                ("num_nodes", ctypes.c_uint32), ("local_batch", ctypes.c_uint64), ("seed", ctypes.c_uint64),
                ("drop_last", ctypes.c_int32), ("keep", ctypes.c_uint64)]


class LsgPlanView(ctypes.Structure):
    """Field-for-field mirror of ``lsg_plan_view`` (include/lsg.h)."""
    _fields_ = [("dataset_size", ctypes.c_uint64), ("local_batch", ctypes.c_uint64),
                ("chunk_threshold", ctypes.c_uint64), ("cost", ctypes.c_uint64),
                ("num_nodes", ctypes.c_uint32), ("num_epochs", ctypes.c_uint32),
                ("num_steps", ctypes.c_uint64), ("num_items", ctypes.c_uint64), ("num_reads", ctypes.c_uint64)] + [
        (n, ctypes.c_void_p) for n in ("order", "epoch_ids", "epoch_steps", "items", "node_off", "fetch_before",
                                       "fetch_after", "read_off", "read_start", "read_end", "read_chunk",
                                       "needed", "redundant")]


EXPORTS = [
    "lsg_version", "lsg_last_error", "lsg_shape_of", "lsg_generate_trace",
    "lsg_build_reuse_graph", "lsg_pso_order", "lsg_plan", "lsg_plan_host", "lsg_simulate",
    "lsg_store_fill", "lsg_gather", "lsg_batch_fetch", "lsg_fetch_step", "lsg_launch_count",
    "lsg_store_create", "lsg_store_open", "lsg_store_info", "lsg_store_close", "lsg_store_read",
    "lsg_store_read_rows", "lsg_fetch_step_store", "lsg_simulate_ex", "lsg_format_trace", "lsg_format_plan",
    "lsg_format_graph", "lsg_parse_trace", "lsg_parse_graph", "lsg_parse_plan", "lsg_free_plan",
    "lsg_buffer_windows", "lsg_brute_force_order", "lsg_remap_step", "lsg_balance_step", "lsg_plan_chunks",
    "lsg_buffer_create", "lsg_buffer_destroy", "lsg_buffer_access", "lsg_buffer_clear", "lsg_buffer_resident",
    "lsg_simulate_sequence", "lsg_optimal_miss_oracle", "lsg_build_reuse_graph_rows",
    "lsg_fetch_steps", "lsg_host_rows_open", "lsg_host_rows_info", "lsg_host_rows_close",
    "lsg_plan_costs", "lsg_miss_stream_create", "lsg_miss_stream_destroy", "lsg_fetch_job_create", "lsg_fetch_job_run", "lsg_fetch_job_stats", "lsg_fetch_job_destroy",
]


class LsgFetchJobDesc(ctypes.Structure):
    """Field-for-field mirror of ``lsg_fetch_job_desc`` (include/lsg.h)."""
    _fields_ = [(n, ctypes.c_void_p) for n in ("d_bufs", "d_outs", "d_items", "d_slots", "d_node_off",
                                               "h_node_off")] + [
        ("step_begin", ctypes.c_uint64), ("step_end", ctypes.c_uint64), ("N", ctypes.c_uint32),
        ("node_begin", ctypes.c_uint32), ("node_end", ctypes.c_uint32), ("sample_bytes", ctypes.c_uint64),
        ("fill_seed", ctypes.c_uint64), ("host", ctypes.c_void_p), ("ring_bytes", ctypes.c_uint64),
        ("misses", ctypes.c_void_p)]


class LsgError(RuntimeError):
    """Raised with the reference ErrorClass code of the failing call."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None


def lib() -> ctypes.CDLL:
    """Load the CUDA library (no fallback: raises if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"lsg CUDA library not built: {LIB_PATH} missing (run `make lib` or "
                "__graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        P, u64, u32, i32, dbl = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32,
                                 ctypes.c_double)
        L.lsg_version.restype = ctypes.c_int
        L.lsg_last_error.restype = ctypes.c_char_p
        L.lsg_launch_count.restype = u64
        L.lsg_shape_of.argtypes = [ctypes.POINTER(LsgConfig), ctypes.POINTER(LsgShape)]
        L.lsg_generate_trace.argtypes = [ctypes.POINTER(LsgConfig), P, P]
        L.lsg_build_reuse_graph.argtypes = [P, u32, u64, u64, u32, u64, i32, u64, i32, P, P]
        L.lsg_build_reuse_graph_rows.argtypes = [P, u32, u64, u64, u32, u64, i32, u64, i32, u32, u32, P, P]
        L.lsg_fetch_steps.argtypes = [P, P, P, P, P, P, u64, u64, u32, u32, u32, u64, u64, P]
        L.lsg_pso_order.argtypes = [P, u32, u32, u32, dbl, dbl, dbl, dbl, u32, u32, u64, P, P, P, P, P]
        L.lsg_plan.argtypes = [ctypes.POINTER(LsgConfig), ctypes.POINTER(LsgPlanOut), P]
        L.lsg_plan_host.argtypes = [ctypes.POINTER(LsgConfig), ctypes.POINTER(LsgPlanOut), P]
        L.lsg_simulate.argtypes = [P, P, u64, u32, u64, u64, i32, u32, u32, P, P, P, P]
        L.lsg_simulate_ex.argtypes = [P, P, u64, u32, u64, u64, i32, i32, P, P, P, u32, u32, P, P, P, P]
        L.lsg_format_trace.argtypes = [P, u64, u32, u32, u64, u64, i32, u64, P, u64, P, P]
        L.lsg_format_plan.argtypes = [P, P, P, P, P, P, P, P, u64, u32, u64, u32, u64, u64, u64, u64, P, u64, P, P]
        L.lsg_format_graph.argtypes = [P, u32, P, u64, P, P]
        L.lsg_parse_trace.argtypes = [ctypes.c_char_p, u64, P, P, u64]
        L.lsg_parse_graph.argtypes = [ctypes.c_char_p, u64, P, P, u64]
        L.lsg_parse_plan.argtypes = [ctypes.c_char_p, u64, P, P]
        L.lsg_free_plan.argtypes = [P]
        L.lsg_buffer_windows.argtypes = [P, u32, u64, u64, u32, u64, i32, u64, i32, P, P, P]
        L.lsg_brute_force_order.argtypes = [P, u32, P, P, P]
        L.lsg_remap_step.argtypes = [P, P, u32, P, u64, u64, i32, P, P, P]
        L.lsg_balance_step.argtypes = [P, P, u32, P, P]
        L.lsg_plan_chunks.argtypes = [P, u64, u64, P, P, P, P]
        L.lsg_buffer_create.argtypes = [i32, u64, ctypes.POINTER(ctypes.c_void_p)]
        L.lsg_buffer_destroy.argtypes = [P]
        L.lsg_buffer_destroy.restype = None
        L.lsg_buffer_access.argtypes = [P, P, P, u64, i32, P, P]
        L.lsg_buffer_clear.argtypes = [P]
        L.lsg_buffer_resident.argtypes = [P, P, u64, ctypes.POINTER(u64)]
        L.lsg_simulate_sequence.argtypes = [P, u64, u64, i32, ctypes.POINTER(u64), P]
        L.lsg_optimal_miss_oracle.argtypes = [P, u64, u64, ctypes.POINTER(u64), P]
        L.lsg_free_plan.restype = None
        L.lsg_store_fill.argtypes = [P, u64, u64, u64, P, P]
        L.lsg_gather.argtypes = [P, P, u64, u64, P, P]
        L.lsg_batch_fetch.argtypes = [P, P, P, u64, u64, u64, P, P]
        L.lsg_fetch_step.argtypes = [P, P, P, P, P, u32, u32, u64, u64, u64, P]
        L.lsg_store_create.argtypes = [ctypes.c_char_p, u64, u64, u64, u64, P]
        L.lsg_store_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.lsg_store_info.argtypes = [P, ctypes.POINTER(u64), ctypes.POINTER(u64)]
        L.lsg_store_close.argtypes = [P]
        L.lsg_store_close.restype = None
        L.lsg_store_read.argtypes = [P, u64, u64, P]
        L.lsg_store_read_rows.argtypes = [P, P, u64, u64, P, P]
        L.lsg_fetch_step_store.argtypes = [P, P, P, P, P, P, P, P, u32, u32, u64, u64, P]
        L.lsg_plan_costs.argtypes = [P, P, P, P, P, P, u64, u32, dbl, dbl, ctypes.POINTER(dbl), ctypes.POINTER(dbl), P]
        L.lsg_host_rows_open.argtypes = [ctypes.c_char_p, u64, u64, u64, i32, ctypes.POINTER(ctypes.c_void_p)]
        L.lsg_host_rows_info.argtypes = [P, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(ctypes.c_void_p)]
        L.lsg_host_rows_close.argtypes = [P]
        L.lsg_host_rows_close.restype = None
        L.lsg_miss_stream_create.argtypes = [u64, u64, ctypes.POINTER(ctypes.c_void_p)]
        L.lsg_miss_stream_destroy.argtypes = [P]
        L.lsg_miss_stream_destroy.restype = None
        L.lsg_fetch_job_create.argtypes = [ctypes.POINTER(LsgFetchJobDesc), ctypes.POINTER(ctypes.c_void_p), P]
        L.lsg_fetch_job_run.argtypes = [P, P]
        L.lsg_fetch_job_stats.argtypes = [P, ctypes.POINTER(u64), P]
        L.lsg_fetch_job_destroy.argtypes = [P, P]
        L.lsg_fetch_job_destroy.restype = None
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise LsgError(rc, lib().lsg_last_error().decode())
