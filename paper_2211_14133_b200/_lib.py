"""ctypes binding of the C-ABI library ``_lib/libpf_b200.so``.

The library is the product: host scheduler (include/pf_sched.h) and the
sm_100a K-FAC kernels (include/pf_kfac.h).  There is no fallback — if the
shared object is missing, importing this module raises, and GPU entry points
raise if no sm_100 device is visible.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PF_LIB_PATH") or os.path.join(_HERE, "_lib", "libpf_b200.so")

# pf_status (include/pf_sched.h)
PF_OK, PF_BAD_SHAPE, PF_NOT_PD, PF_CUDA_ERROR, PF_BAD_ARG, PF_INFEASIBLE = 0, 1, 2, 3, 4, 5
PF_LOGIC_ERROR, PF_LENGTH_ERROR, PF_NO_DEVICE = 6, 7, 8


class PfConfig(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "method", "stages", "micro_batches", "micro_batch_size", "replicas", "devices",
        "layers_per_stage", "seq_len", "recompute")]


class PfCosts(C.Structure):
    _fields_ = ([(n, C.c_double) for n in ("t_f", "t_b", "t_curv", "t_inv", "t_prec")]
                + [(n, C.c_int64) for n in ("m_theta", "m_act", "m_err_peak", "m_err_save", "m_curv")]
                + [(n, C.c_double) for n in ("comm_alpha", "comm_beta", "p2p_latency")])


class PfItem(C.Structure):
    _fields_ = ([(n, C.c_int32) for n in ("kind", "stage", "micro_batch", "layer", "factor", "device")]
                + [("start", C.c_double), ("duration", C.c_double), ("step", C.c_int32),
                   ("reserved", C.c_int32)])


class PfWork(C.Structure):
    _fields_ = ([(n, C.c_int32) for n in ("kind", "stage", "layer", "factor", "micro_batch", "device")]
                + [("duration", C.c_double), ("base_anchor", C.c_int32), ("n_preds", C.c_int32)])


class PfInterval(C.Structure):
    _fields_ = [("begin", C.c_double), ("end", C.c_double)]


class PfStaleness(C.Structure):
    _fields_ = [("stage", C.c_int32), ("layer", C.c_int32), ("staleness_steps", C.c_int32)]


class PfSyrkProblem(C.Structure):
    _fields_ = [("x", C.c_void_p), ("f", C.c_void_p), ("d", C.c_int32), ("n", C.c_int32),
                ("ldx", C.c_int32), ("ldf", C.c_int32), ("scale", C.c_float),
                ("accumulate", C.c_int32), ("layout", C.c_int32)]


class PfInverseProblem(C.Structure):
    _fields_ = [("m", C.c_void_p), ("minv", C.c_void_p), ("minv_sliced", C.c_void_p),
                ("d", C.c_int32), ("ldm", C.c_int32), ("ldinv", C.c_int32),
                ("damping", C.c_float), ("workspace", C.c_void_p), ("d_info", C.c_void_p)]


class PfPreconditionProblem(C.Structure):
    _fields_ = [("b_inv_sliced", C.c_void_p), ("grad", C.c_void_p), ("a_inv_sliced", C.c_void_p),
                ("w", C.c_void_p), ("p_out", C.c_void_p), ("d_out", C.c_int32),
                ("d_in", C.c_int32), ("eta", C.c_float), ("workspace", C.c_void_p)]


P = C.POINTER
_SIGNATURES = {
    # pf_sched.h
    "pf_last_error": (C.c_char_p, []),
    "pf_version": (C.c_char_p, []),
    "pf_validate_config": (C.c_int, [P(PfConfig), C.c_char_p, C.c_size_t, P(C.c_int)]),
    "pf_effective_devices": (C.c_int, [P(PfConfig), P(C.c_int)]),
    "pf_build_schedule": (C.c_int, [P(PfConfig), P(PfCosts), C.c_int, P(C.c_void_p)]),
    "pf_schedule_free": (None, [C.c_void_p]),
    "pf_schedule_info": (C.c_int, [C.c_void_p, P(C.c_int), P(C.c_double), P(C.c_int), P(C.c_int),
                                   P(C.c_double), P(C.c_int), P(C.c_double)]),
    "pf_schedule_timeline": (C.c_int, [C.c_void_p, C.c_int, P(PfItem), C.c_int, P(C.c_int)]),
    "pf_schedule_staleness": (C.c_int, [C.c_void_p, P(PfStaleness), C.c_int, P(C.c_int)]),
    "pf_extract_bubbles": (C.c_int, [C.c_void_p, C.c_int, P(PfInterval), C.c_int, P(C.c_int),
                                     P(C.c_double)]),
    "pf_schedule_metrics": (C.c_int, [C.c_void_p, P(C.c_double), P(C.c_double), P(C.c_double)]),
    "pf_validate_schedule": (C.c_int, [C.c_void_p, P(PfConfig), C.c_char_p, C.c_size_t,
                                       P(C.c_int)]),
    "pf_model_collective": (C.c_int, [C.c_double, C.c_int, C.c_double, C.c_double,
                                      P(C.c_double)]),
    "pf_enumerate_kfac_works": (C.c_int, [P(PfConfig), P(PfCosts), P(C.c_void_p)]),
    "pf_queue_new": (C.c_void_p, []),
    "pf_queue_free": (None, [C.c_void_p]),
    "pf_queue_size": (C.c_int, [C.c_void_p, P(C.c_int)]),
    "pf_queue_get": (C.c_int, [C.c_void_p, C.c_int, P(PfWork), P(C.c_int32), C.c_int]),
    "pf_queue_push": (C.c_int, [C.c_void_p, P(PfWork), P(C.c_int32)]),
    "pf_queue_set_duration": (C.c_int, [C.c_void_p, C.c_int, C.c_double]),
    "pf_assign_works": (C.c_int, [C.c_void_p, P(PfConfig), P(PfCosts), C.c_void_p, C.c_int,
                                  C.c_int, P(C.c_void_p)]),
    "pf_infeasible_payload": (C.c_int, [C.c_void_p, P(C.c_double), P(C.c_int)]),
    "pf_infeasible_item": (C.c_int, [C.c_void_p, C.c_int, P(PfWork)]),
    "pf_staleness_report": (C.c_int, [C.c_void_p, P(PfStaleness), C.c_int, P(C.c_int)]),
    # pf_kfac.h
    "pf_curvature_syrk": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int,
                                    C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "pf_curvature_syrk_grouped": (C.c_int, [P(PfSyrkProblem), C.c_int, C.c_int, C.c_void_p]),
    "pf_damped_inverse_workspace": (C.c_int, [C.c_int, P(C.c_size_t)]),
    "pf_damped_inverse": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_float, C.c_void_p,
                                    C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                    C.c_void_p]),
    "pf_cholesky_factor": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_int,
                                     C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "pf_slice_bytes": (C.c_int, [C.c_int, C.c_int, P(C.c_size_t)]),
    "pf_slice": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "pf_damped_inverse_batched": (C.c_int, [P(PfInverseProblem), C.c_int, C.c_void_p]),
    "pf_precondition_workspace": (C.c_int, [C.c_int, C.c_int, P(C.c_size_t)]),
    "pf_precondition": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                  C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]),
    "pf_precondition_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_size_t,
                                         C.c_void_p]),
    "pf_precondition_update_sliced": (C.c_int, [P(PfPreconditionProblem), C.c_int, C.c_void_p]),
    "pf_f32_to_bf16": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "pf_kernel_launch_count": (C.c_int64, []),
    "pf_device_ok": (C.c_int, []),
    "pf_set_background": (C.c_int, [C.c_int]),
}

_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Load (once) and return the C-ABI library; raises if it was not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (make -C paper_2211_14133_b200); there is no fallback path")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES)


class PfError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def check(status: int, what: str = "") -> None:
    if status != PF_OK:
        msg = lib().pf_last_error().decode(errors="replace")
        if status in (PF_BAD_SHAPE, PF_BAD_ARG):
            raise ValueError(f"{what}: {msg}")
        raise PfError(status, f"{what}: {msg} (status {status})")
