"""ctypes binding of libimpact_b200.so (include/impact_b200.h).

The library is built in-tree by `_build.build()` (nvcc, sm_100a).  There is
no fallback: if the library is missing or no CUDA device is present, every
product entry point raises instead of computing on the CPU.
"""

import ctypes
import os
import threading

import numpy as np

from .errors import (AbstractionError, ConvergenceError, ImpactError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IMP_LIB_PATH") or os.path.join(HERE, "libimpact_b200.so")

IMP_OK, IMP_E_ARG, IMP_E_CUDA, IMP_E_ABSTRACTION, IMP_E_NONFINITE, \
    IMP_E_CONVERGENCE, IMP_E_MONOTONE, IMP_E_BRACKET, IMP_E_JIT, \
    IMP_E_NOMEM = range(10)
SPEC_REACH, SPEC_SAFETY = 0, 1
LP_MIN, LP_MAX = 0, 1
MODE_PHASE, MODE_DIAGNOSE = 0, 1

c_i32, c_i64, c_dbl, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_double,
                             ctypes.c_void_p)
P_i32 = ctypes.POINTER(c_i32)
P_i64 = ctypes.POINTER(c_i64)
P_dbl = ctypes.POINTER(c_dbl)


class ImdpInfo(ctypes.Structure):
    _fields_ = [("n_rows", c_i64), ("row_begin", c_i64), ("nnz", c_i64),
                ("n_s", c_i32), ("n_u", c_i32), ("n_w", c_i32),
                ("k_begin", c_i32), ("k_count", c_i32), ("max_row", c_i32),
                ("device", c_i32)]


class BuildDesc(ctypes.Structure):
    _fields_ = [("device", c_i32), ("n", c_i32), ("m", c_i32), ("p", c_i32),
                ("n_u", c_i32), ("n_w", c_i32), ("separable", c_i32),
                ("counts", P_i32), ("eta", P_dbl), ("sigma", P_dbl),
                ("edges", P_dbl), ("cover_lo", P_dbl), ("cover_hi", P_dbl),
                ("n_s", c_i32), ("n_t", c_i32), ("n_a", c_i32),
                ("safe_multi", P_i32), ("target_multi", P_i32),
                ("avoid_multi", P_i32), ("src_lo", P_dbl), ("src_hi", P_dbl),
                ("dyn_source", ctypes.c_char_p), ("n_consts", c_i32),
                ("consts", P_dbl), ("deps", P_i32), ("n_deps", P_i32),
                ("zero_cutoff", c_dbl), ("tol", c_dbl), ("low_cost", c_i32),
                ("max_evals_per_dim", c_i32), ("multistart", c_i32),
                ("k_begin", c_i32), ("k_count", c_i32),
                ("mc", c_i32), ("mc_samples", c_i32),
                ("mc_seed", ctypes.c_uint64), ("mc_norm", c_dbl),
                ("inv_cov", P_dbl), ("dim_lo", P_dbl), ("dim_hi", P_dbl),
                ("exact", c_i32), ("state_cost", P_i64)]


class BuildStats(ctypes.Structure):
    _fields_ = [("ms_total", c_dbl), ("ms_mean_ranges", c_dbl),
                ("ms_outer", c_dbl), ("ms_refine", c_dbl),
                ("ms_assemble", c_dbl), ("nnz", c_i64),
                ("nm_instances", c_i64), ("nm_evals", c_i64),
                ("nm_lane_slots", c_i64), ("nm_evals_shared", c_i64),
                ("nnz_live", c_i64), ("nm_evals_mean", c_i64)]


class PhaseDesc(ctypes.Structure):
    _fields_ = [("spec", c_i32), ("lp", c_i32), ("u_max", c_i32),
                ("mode", c_i32), ("eps", c_dbl), ("horizon", c_i64),
                ("max_iterations", c_i64), ("fixed_policy", P_i64)]


class SimDesc(ctypes.Structure):
    _fields_ = [("rollouts", c_i32), ("steps", c_i32),
                ("seed", ctypes.c_uint64), ("reach_like", c_i32),
                ("n_starts", c_i32), ("starts", P_i32), ("n_ctrl", c_i32),
                ("coords", P_dbl), ("slot_input", P_i32), ("total", c_i64),
                ("slot_of", P_i32), ("kind", ctypes.POINTER(ctypes.c_uint8)),
                ("lb", P_dbl), ("ub", P_dbl)]


class PhaseOut(ctypes.Structure):
    _fields_ = [("v0", P_dbl), ("v1", P_dbl), ("policy", P_i64),
                ("iterations", c_i64), ("k0", c_i64), ("k1", c_i64),
                ("fallback", c_i32), ("gap", c_dbl), ("ms_device", c_dbl),
                ("sweeps", c_i64), ("ms_sweep", c_dbl),
                ("gap_log", P_dbl), ("gap_log_cap", c_i64),
                ("gap_log_n", c_i64)]


_lib = None
_lock = threading.Lock()


def _declare(lib):
    lib.imp_last_error.restype = ctypes.c_size_t
    lib.imp_last_error.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
    lib.imp_version.restype = ctypes.c_char_p
    lib.imp_device_query.argtypes = [c_i32, P_i32, P_i32, P_i32]
    lib.imp_imdp_import.argtypes = [c_i32, c_i32, c_i32, c_i32, c_i32, c_i64,
                                    P_i64, P_i32, P_dbl, P_dbl, P_dbl, P_dbl,
                                    P_dbl, P_dbl, ctypes.POINTER(c_vp)]
    lib.imp_imdp_info_get.argtypes = [c_vp, ctypes.POINTER(ImdpInfo)]
    lib.imp_imdp_export.argtypes = [c_vp, P_i64, P_i32, P_dbl, P_dbl, P_dbl,
                                    P_dbl, P_dbl, P_dbl]
    lib.imp_imdp_validate.argtypes = [c_vp, c_dbl]
    lib.imp_imdp_free.argtypes = [c_vp]
    lib.imp_imdp_free.restype = None
    lib.imp_build.argtypes = [ctypes.POINTER(BuildDesc), ctypes.POINTER(c_vp),
                              ctypes.POINTER(BuildStats)]
    lib.imp_run_phase.argtypes = [c_vp, ctypes.POINTER(PhaseDesc),
                                  ctypes.POINTER(PhaseOut)]
    lib.imp_bellman_step.argtypes = [c_vp, P_dbl, c_i32, c_i32, c_i32, P_i64,
                                     P_dbl, P_i64]
    lib.imp_row_values.argtypes = [c_vp, P_dbl, c_i32, P_dbl, c_i32]
    lib.imp_shard_sweep.argtypes = [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32,
                                    c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]
    lib.imp_fp64_peak.argtypes = [c_i32, P_dbl]
    lib.imp_ndtr_eval.argtypes = [ctypes.POINTER(BuildDesc), P_dbl, P_dbl,
                                  c_i64, c_i32]
    lib.imp_shard_loop_begin.argtypes = [c_vp, ctypes.POINTER(PhaseDesc),
                                         P_i64, c_i32, c_vp, c_vp, c_i64,
                                         c_vp, c_vp, ctypes.POINTER(c_vp)]
    lib.imp_shard_loop_sweep.argtypes = [c_vp, c_vp]
    lib.imp_shard_loop_control.argtypes = [c_vp, c_vp]
    lib.imp_shard_loop_poll.argtypes = [c_vp, ctypes.POINTER(PhaseOut),
                                        P_i32, c_vp]
    lib.imp_shard_loop_free.argtypes = [c_vp]
    lib.imp_shard_loop_free.restype = None
    lib.imp_jit_compile.argtypes = [ctypes.POINTER(BuildDesc),
                                    ctypes.c_char_p]
    lib.imp_export_text_rows.argtypes = [c_vp, c_i32, c_i64, c_i64,
                                         ctypes.c_char_p, c_i64, P_i64]
    lib.imp_format_values.argtypes = [P_dbl, c_i64, c_i64, c_i32,
                                      ctypes.c_char_p, c_i64, P_i64]
    lib.imp_simulate.argtypes = [ctypes.POINTER(BuildDesc),
                                 ctypes.POINTER(SimDesc), P_dbl, P_i32,
                                 P_i32]
    lib.imp_time_sweep.argtypes = [c_vp, c_i32, c_i32, c_i32, P_dbl]
    lib.imp_time_sweep.restype = c_i32
    lib.imp_launch_count.argtypes = [ctypes.POINTER(ctypes.c_ulonglong),
                                     ctypes.POINTER(ctypes.c_ulonglong)]
    lib.imp_launch_count.restype = None
    for name in ("imp_device_query", "imp_imdp_import", "imp_imdp_info_get",
                 "imp_imdp_export", "imp_imdp_validate", "imp_build",
                 "imp_jit_compile",
                 "imp_run_phase", "imp_bellman_step", "imp_row_values",
                 "imp_shard_sweep", "imp_fp64_peak"):
        getattr(lib, name).restype = c_i32


EXPORTED = ("imp_last_error", "imp_version", "imp_device_query",
            "imp_imdp_import", "imp_imdp_info_get", "imp_imdp_export",
            "imp_imdp_validate", "imp_imdp_free", "imp_build",
            "imp_jit_compile",
            "imp_run_phase", "imp_bellman_step", "imp_row_values",
            "imp_shard_sweep", "imp_fp64_peak", "imp_time_sweep",
            "imp_launch_count", "imp_export_text_rows",
            "imp_format_values", "imp_simulate", "imp_ndtr_eval",
            "imp_shard_loop_begin", "imp_shard_loop_sweep",
            "imp_shard_loop_control", "imp_shard_loop_poll",
            "imp_shard_loop_free")


def launch_count():
    """(our kernels, CUB primitive calls) launched so far by the library."""
    a, b = ctypes.c_ulonglong(0), ctypes.c_ulonglong(0)
    load().imp_launch_count(ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def load(build_if_missing=True):
    """Load (building first if needed) the CUDA library; raise if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH) and build_if_missing:
                from . import _build
                _build.build()
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: run "
                    "`python -m paper_2401_03555_b200._build` (no CPU "
                    "fallback exists)")
            lib = ctypes.CDLL(LIB_PATH)
            _declare(lib)
            _lib = lib
    return _lib


def last_error():
    lib = load()
    buf = ctypes.create_string_buffer(4096)
    lib.imp_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(status, k0=None, k1=None):
    """Map an imp_status onto the reference's exception contract."""
    if status == IMP_OK:
        return
    msg = last_error()
    if status == IMP_E_ARG:
        raise ValueError(msg)
    if status in (IMP_E_ABSTRACTION,):
        raise AbstractionError(msg)
    if status == IMP_E_NONFINITE:
        raise AbstractionError("non-finite objective value encountered; "
                               + msg)
    if status == IMP_E_CONVERGENCE:
        raise ConvergenceError(msg, k0=k0, k1=k1)
    if status in (IMP_E_MONOTONE, IMP_E_BRACKET):
        raise ImpactError(msg)
    if status == IMP_E_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"impact_b200 status {status}: {msg}")


def ptr(a, ctype):
    """ctypes pointer to a contiguous numpy array (None passes NULL)."""
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def fp64_peak_gflops(device=0):
    lib = load()
    out = c_dbl(0)
    check(lib.imp_fp64_peak(device, ctypes.byref(out)))
    return out.value


def as_i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def as_i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def as_f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)
