"""ctypes binding of libedx.so (include/edx.h).

The shared library is built in-tree (paper_2512_21615_b200/libedx.so) by
__graft_entry__.build() / `make -C paper_2512_21615_b200/csrc`.  There is no
fallback: importing the package without the library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libedx.so")

EDX_OK, EDX_INVALID_ARGUMENT, EDX_LOGIC_ERROR, EDX_RUNTIME_ERROR, EDX_CUDA_ERROR = range(5)
EDX_NUM_PHASES = 6


class EdxError(RuntimeError):
    """Base of the errors raised through the C ABI."""


class InvalidArgument(EdxError, ValueError):
    """std::invalid_argument in the reference."""


class LogicError(EdxError):
    """std::logic_error in the reference."""


class EdxRuntimeError(EdxError):
    """std::runtime_error in the reference."""


class CudaError(EdxError):
    """Device failure (no reference counterpart)."""


_EXC = {EDX_INVALID_ARGUMENT: InvalidArgument, EDX_LOGIC_ERROR: LogicError,
        EDX_RUNTIME_ERROR: EdxRuntimeError, EDX_CUDA_ERROR: CudaError}


class ClusterConfigC(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("bandwidths_bps", C.POINTER(C.c_double)),
                ("n_bandwidths", C.c_int32), ("reserved", C.c_int32),
                ("d_tran_bytes", C.c_uint64), ("cache_capacity", C.c_uint64),
                ("alpha", C.c_double)]


class ReportC(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("miss_pull", C.c_uint64),
                ("update_push", C.c_uint64), ("evict_push", C.c_uint64),
                ("hits", C.c_uint64), ("lookups", C.c_uint64), ("cost_s", C.c_double),
                ("miss_pull_w", C.POINTER(C.c_uint64)), ("update_push_w", C.POINTER(C.c_uint64)),
                ("evict_push_w", C.POINTER(C.c_uint64)), ("cost_w", C.POINTER(C.c_double))]


class EngineOptionsC(C.Structure):
    _fields_ = [("device", C.c_int32), ("reserved0", C.c_int32), ("id_space", C.c_uint64),
                ("max_batch_ids", C.c_uint64), ("rank", C.c_int32), ("world_size", C.c_int32),
                ("nccl_unique_id", C.c_void_p)]


# edx_transport callbacks: (ctx, buf, bytes, peer/root) -> 0 on success
SEND_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32)
RECV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32)
BCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32)


class TransportC(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("send", SEND_FN), ("recv", RECV_FN),
                ("broadcast", BCAST_FN)]


# (name, restype, argtypes) for every symbol include/edx.h declares
def _sigs():
    vp, u64, i32, dbl, cint = C.c_void_p, C.c_uint64, C.c_int32, C.c_double, C.c_int
    P = C.POINTER
    u32p, u64p, i32p, dblp = P(C.c_uint32), P(C.c_uint64), P(C.c_int32), P(C.c_double)
    cfgp = P(ClusterConfigC)
    return [
        ("edx_last_error", C.c_char_p, []),
        ("edx_abi_version", cint, []),
        ("edx_validate_config", cint, [cfgp, u64]),
        ("edx_unit_costs", cint, [cfgp, dblp]),
        ("edx_nccl_unique_id", cint, [vp, u64]),
        ("edx_shard_rows", cint, [u64, i32, u64p, u64p]),
        ("edx_exchange_gather_rows", cint, [P(TransportC), dblp, u64, i32, i32, i32, i32]),
        ("edx_exchange_broadcast_decision", cint, [P(TransportC), i32p, u64, i32]),
        ("edx_engine_create", cint, [cfgp, P(EngineOptionsC), P(vp)]),
        ("edx_engine_destroy", None, [vp]),
        ("edx_engine_load_batch", cint, [vp, vp, vp, u64, cint]),
        ("edx_engine_load_device_batch", cint, [vp, vp, vp, u64, u64]),
        ("edx_engine_build", cint, [vp, dblp]),
        ("edx_engine_dispatch", cint, [vp, dbl, i32p, dblp]),
        ("edx_engine_dispatch_hitgreedy", cint, [vp, i32p]),
        ("edx_engine_step", cint, [vp, i32p, P(ReportC)]),
        ("edx_engine_iterate", cint, [vp, vp, vp, u64, cint, i32p, dblp, P(ReportC)]),
        ("edx_engine_iterate_device", cint, [vp, vp, vp, u64, u64, i32p, dblp, P(ReportC)]),
        ("edx_engine_prefetch", cint, [vp, vp, vp, u64]),
        ("edx_engine_iterate_prefetch", cint, [vp, vp, vp, u64, vp, vp, u64, i32p, dblp,
                                                P(ReportC)]),
        ("edx_engine_stream", cint, [vp, P(vp)]),
        ("edx_engine_seed_entry", cint, [vp, C.c_uint32, i32, cint, cint]),
        ("edx_engine_state_of", cint, [vp, C.c_uint32, u64p, u64p, u64p]),
        ("edx_engine_validate_consistency", cint, [vp]),
        ("edx_engine_clock", u64, [vp]),
        ("edx_engine_state_version", u64, [vp]),
        ("edx_engine_synchronize", cint, [vp]),
        ("edx_engine_expected_cost", cint, [vp, dblp]),
        ("edx_engine_export_global", cint, [vp, u32p, u64p, u64p, u64p, u64, u64p]),
        ("edx_engine_cache_size", cint, [vp, i32, u64p]),
        ("edx_engine_export_cache", cint, [vp, i32, u32p, P(C.c_uint8), u32p, u32p, u64p]),
        ("edx_engine_cache_marks", cint, [vp, i32, u32p, u64p]),
        ("edx_engine_import_snapshot", cint, [vp, u32p, u64p, u64p, u64p, u64]),
        ("edx_engine_import_state", cint, [vp, u64, u64, u32p, u64p, u64p, u64p, u64p, u32p,
                                           P(C.c_uint8), u32p, u32p, u64p, u32p, u64p]),
        ("edx_engine_last_kernels", cint, [vp, P(C.c_char_p), P(C.c_char_p), P(C.c_char_p)]),
        ("edx_engine_set_profiling", cint, [vp, cint]),
        ("edx_engine_phase_times", cint, [vp, dblp, u64p, cint]),
        ("edx_solver_stats", cint, [vp, u64p]),
        ("edx_build_matrix", cint, [cfgp, u32p, u64p, u64p, u64p, u64, u32p, u64p, u64, dblp]),
        ("edx_hitgreedy", cint, [cfgp, u32p, u64p, u64p, u64, u32p, u64p, u64, i32p]),
        ("edx_expected_costs", cint, [cfgp, u32p, u64p, u64p, u64, u32p, u64p, u64, dblp]),
        ("edx_build_matrix_sized", cint, [cfgp, u32p, u64p, u64p, u64, u32p, u64p, u64, u64p, dblp]),
        ("edx_expected_costs_sized", cint, [cfgp, u32p, u64p, u64p, u64, u32p, u64p, u64, u64p,
                                            dblp]),
        ("edx_cache_create", cint, [u64, cint, cint, P(vp)]),
        ("edx_cache_destroy", None, [vp]),
        ("edx_cache_touch", cint, [vp, C.c_uint32, cint, u64, C.c_double]),
        ("edx_cache_set_version", cint, [vp, C.c_uint32, cint]),
        ("edx_cache_erase", cint, [vp, C.c_uint32]),
        ("edx_cache_find", cint, [vp, C.c_uint32, P(cint), P(cint), u32p, u32p, u64p]),
        ("edx_cache_select_victim", cint, [vp, u32p]),
        ("edx_cache_evict_for", cint, [vp, u64, u32p, u64, u32p, u64p]),
        ("edx_cache_info", cint, [vp, u64p, u32p, u64p]),
        ("edx_cache_export", cint, [vp, u32p, P(C.c_uint8), u32p, u32p, u64p, u64, u64p]),
        ("edx_row_gap_key", cint, [u64, u64, dblp, u64, dblp]),
        ("edx_rows_by_gap", cint, [u64, u64, dblp, u64p]),
        ("edx_hungarian", cint, [u64, dblp, u64p, dblp]),
        ("edx_hungarian_blocks", cint, [u64, u64, dblp, u64p, i32, u64p, dblp]),
        ("edx_greedy_dispatch", cint, [u64, u64, dblp, u64p, u64, i32p, u64p, i32p]),
        ("edx_ecomix", cint, [cfgp, u64, u64, dblp, u64p, i32p]),
        ("edx_decision_cost", cint, [u64, u64, dblp, i32p, dblp]),
        ("edx_zipf_create", cint, [u64, u64, dbl, u64, u64, u64, P(vp)]),
        ("edx_zipf_next", cint, [vp, u32p]),
        ("edx_zipf_reset", None, [vp]),
        ("edx_zipf_sampler_create", cint, [u64, dbl, u64, P(vp)]),
        ("edx_zipf_draw", cint, [vp, u64, u32p]),
        ("edx_zipf_destroy", None, [vp]),
        ("edx_trace_load", cint, [C.c_char_p, u64, u64p, P(C.c_char_p), u64, u64, u64, P(vp)]),
        ("edx_trace_info", None, [vp, u64p, u64p, u64p, u64p]),
        ("edx_trace_iteration", cint, [vp, u64, P(u32p), P(u64p), u64p]),
        ("edx_trace_destroy", None, [vp]),
    ]


SIGNATURES = _sigs()
_lib = None


def lib():
    """Load libedx.so (once); raise if it is missing — there is no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != EDX_OK:
        msg = lib().edx_last_error().decode(errors="replace")
        raise _EXC.get(rc, EdxError)(msg)
