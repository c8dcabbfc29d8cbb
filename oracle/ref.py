"""TEST INFRASTRUCTURE ONLY — ctypes access to the compiled reference
(oracle/_ref/libpipefill_ref.so, built by oracle/Makefile from the unmodified
/root/reference sources) and to the C restatement (oracle/libpf_oracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  Nothing in the product does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libpipefill_ref.so")
ORACLE_LIB = os.path.join(HERE, "libpf_oracle.so")

_ref = None
_orc = None

_dp = C.POINTER(C.c_double)


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            raise FileNotFoundError(f"{REF_LIB} missing: run `make -C oracle` where /root/reference exists")
        h = C.CDLL(REF_LIB)
        h.pfref_last_error.restype = C.c_char_p
        for n in ("pfref_build_dump",):
            getattr(h, n).argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_char_p, C.c_size_t,
                                      C.POINTER(C.c_size_t)]
        h.pfref_queue_dump.argtypes = [C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t,
                                       C.POINTER(C.c_size_t)]
        h.pfref_assign_dump.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_char_p,
                                        C.c_size_t, C.POINTER(C.c_size_t)]
        h.pfref_model_collective.argtypes = [C.c_double, C.c_int, C.c_double, C.c_double, _dp]
        h.pfref_curvature_factors.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_int, _dp, _dp]
        h.pfref_cholesky_spd_inverse.argtypes = [_dp, C.c_int, C.c_double, _dp]
        h.pfref_cholesky_factor.argtypes = [_dp, C.c_int, _dp]
        h.pfref_precondition.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, _dp]
        h.pfref_ngd_step.argtypes = [_dp, _dp, C.c_int, C.c_int, _dp, _dp, C.c_double,
                                     C.POINTER(C.c_int)]
        h.pfref_splitmix_symmetric.argtypes = [C.c_ulonglong, _dp, C.c_longlong]
        h.pfref_splitmix_symmetric.restype = None
        h.pfref_train_toy.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, _dp]
        _ref = h
    return _ref


def oracle() -> C.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_LIB):
            raise FileNotFoundError(f"{ORACLE_LIB} missing: run `make -C oracle oracle`")
        h = C.CDLL(ORACLE_LIB)
        h.orc_fill_symmetric.argtypes = [C.c_uint64, C.c_double, _dp, C.c_int64]
        h.orc_fill_symmetric.restype = None
        h.orc_matmul.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, _dp]
        h.orc_matmul.restype = None
        h.orc_curvature_factor.argtypes = [_dp, C.c_int, C.c_int, _dp]
        h.orc_curvature_factor.restype = None
        h.orc_cholesky_factor.argtypes = [_dp, C.c_int, _dp]
        h.orc_cholesky_spd_inverse.argtypes = [_dp, C.c_int, C.c_double, _dp]
        h.orc_precondition.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, _dp]
        h.orc_precondition.restype = None
        h.orc_ngd_update.argtypes = [_dp, _dp, C.c_int64, C.c_double]
        h.orc_ngd_update.restype = None
        h.orc_max_abs_residual.argtypes = [_dp, _dp, C.c_int, C.c_double]
        h.orc_max_abs_residual.restype = C.c_double
        h.orc_rel_frobenius.argtypes = [_dp, _dp, C.c_int64]
        h.orc_rel_frobenius.restype = C.c_double
        _orc = h
    return _orc


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


# ------------------------------------------------------------------ numerics
class DomainError(ArithmeticError):
    """std::domain_error: Cholesky pivot failed."""


def _ref_call(rc: int):
    if rc == 2:
        raise DomainError(ref().pfref_last_error().decode())
    if rc != 0:
        raise ValueError(ref().pfref_last_error().decode())


def ref_curvature_factors(a: np.ndarray, e: np.ndarray):
    """kfac::curvature_factors on a BatchTape with one layer (a: d_in x B, e: d_out x B)."""
    a = np.ascontiguousarray(a, np.float64)
    e = np.ascontiguousarray(e, np.float64)
    A = np.zeros((a.shape[0], a.shape[0]))
    B = np.zeros((e.shape[0], e.shape[0]))
    _ref_call(ref().pfref_curvature_factors(_ptr(a), a.shape[0], _ptr(e), e.shape[0], a.shape[1],
                                            _ptr(A), _ptr(B)))
    return A, B


def ref_cholesky_spd_inverse(m: np.ndarray, damping: float) -> np.ndarray:
    m = np.ascontiguousarray(m, np.float64)
    out = np.zeros_like(m)
    _ref_call(ref().pfref_cholesky_spd_inverse(_ptr(m), m.shape[0], damping, _ptr(out)))
    return out


def ref_precondition(grad, a_inv, b_inv) -> np.ndarray:
    g = np.ascontiguousarray(grad, np.float64)
    ai = np.ascontiguousarray(a_inv, np.float64)
    bi = np.ascontiguousarray(b_inv, np.float64)
    out = np.zeros_like(g)
    _ref_call(ref().pfref_precondition(_ptr(g), g.shape[0], g.shape[1], _ptr(ai), _ptr(bi),
                                       _ptr(out)))
    return out


def ref_ngd_step(weight, grad, a_inv, b_inv, eta):
    w = np.ascontiguousarray(weight, np.float64).copy()
    g = np.ascontiguousarray(grad, np.float64)
    plain = C.c_int()
    ai = None if a_inv is None else np.ascontiguousarray(a_inv, np.float64)
    bi = None if b_inv is None else np.ascontiguousarray(b_inv, np.float64)
    _ref_call(ref().pfref_ngd_step(_ptr(w), _ptr(g), g.shape[0], g.shape[1],
                                   None if ai is None else _ptr(ai),
                                   None if bi is None else _ptr(bi), eta, C.byref(plain)))
    return w, bool(plain.value)


def ref_splitmix(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    ref().pfref_splitmix_symmetric(seed, _ptr(out), n)
    return out


def ref_train_toy(steps=60, lr=1e-3, damping=1e-3, refresh=1, kfac=True) -> np.ndarray:
    out = np.zeros(steps)
    n = ref().pfref_train_toy(steps, lr, damping, refresh, int(kfac), _ptr(out))
    return out[:n]


# the C restatement (same calls, oracle/kfac_oracle.c)
def orc_symmetric(seed: int, shape, scale: float = 1.0) -> np.ndarray:
    out = np.zeros(int(np.prod(shape)))
    oracle().orc_fill_symmetric(seed, scale, _ptr(out), out.size)
    return out.reshape(shape)


def orc_curvature_factor(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros((x.shape[0], x.shape[0]))
    oracle().orc_curvature_factor(_ptr(x), x.shape[0], x.shape[1], _ptr(out))
    return out


def orc_cholesky_spd_inverse(m: np.ndarray, damping: float) -> np.ndarray:
    m = np.ascontiguousarray(m, np.float64)
    out = np.zeros_like(m)
    bad = oracle().orc_cholesky_spd_inverse(_ptr(m), m.shape[0], damping, _ptr(out))
    if bad:
        raise DomainError(f"cholesky: matrix not positive definite (column {bad})")
    return out


def orc_cholesky_factor(m: np.ndarray) -> np.ndarray:
    m = np.ascontiguousarray(m, np.float64)
    out = np.zeros_like(m)
    bad = oracle().orc_cholesky_factor(_ptr(m), m.shape[0], _ptr(out))
    if bad:
        raise DomainError(f"cholesky: matrix not positive definite (column {bad})")
    return out


def orc_precondition(grad, a_inv, b_inv) -> np.ndarray:
    g = np.ascontiguousarray(grad, np.float64)
    out = np.zeros_like(g)
    oracle().orc_precondition(_ptr(g), g.shape[0], g.shape[1],
                              _ptr(np.ascontiguousarray(a_inv, np.float64)),
                              _ptr(np.ascontiguousarray(b_inv, np.float64)), _ptr(out))
    return out


def orc_ngd_update(w, direction, eta) -> np.ndarray:
    w = np.ascontiguousarray(w, np.float64).copy()
    oracle().orc_ngd_update(_ptr(w), _ptr(np.ascontiguousarray(direction, np.float64)), w.size, eta)
    return w


def orc_residual(m, inv, damping) -> float:
    """max |(M + damping I) X - I| (reference test_kfac.cpp:150-155 norm)."""
    return oracle().orc_max_abs_residual(_ptr(np.ascontiguousarray(m, np.float64)),
                                         _ptr(np.ascontiguousarray(inv, np.float64)),
                                         m.shape[0], damping)


# ------------------------------------------------------------------ schedules
@dataclass
class Dump:
    """Canonical, bit-exact image of one scheduler result."""
    header: tuple = ()
    items: List[tuple] = field(default_factory=list)      # (dev, kind, stage, micro, layer, factor, start, dur, step)
    staleness: List[tuple] = field(default_factory=list)
    metrics: tuple = ()
    bubbles: List[tuple] = field(default_factory=list)
    violations: List[str] = field(default_factory=list)
    infeasible: Optional[tuple] = None                     # (deficit, n, message)
    unplaced: List[tuple] = field(default_factory=list)
    queue: List[tuple] = field(default_factory=list)


def _call_dump(fn, *args) -> str:
    need = C.c_size_t()
    rc = fn(*args, None, 0, C.byref(need))
    if rc not in (0, 9):
        raise ValueError(ref().pfref_last_error().decode())
    buf = C.create_string_buffer(need.value)
    rc = fn(*args, buf, need.value, C.byref(need))
    if rc != 0:
        raise ValueError(ref().pfref_last_error().decode())
    return buf.value.decode()


def _parse(text: str) -> Dump:
    d = Dump()
    for line in text.splitlines():
        tag, *f = line.split(" ")
        if tag == "H":
            d.header = (float(f[0]), int(f[1]), int(f[2]), int(f[3]))
        elif tag == "F":
            d.header = (float(f[0]), float(f[1]), int(f[2]), int(f[3]), int(f[4]))
        elif tag == "I":
            d.items.append((int(f[0]), int(f[1]), int(f[2]), int(f[3]), int(f[4]), int(f[5]),
                            float(f[6]), float(f[7]), int(f[8])))
        elif tag == "S":
            d.staleness.append(tuple(int(x) for x in f))
        elif tag == "M":
            d.metrics = (float(f[0]), float(f[1]))
        elif tag == "T":
            d.bubbles.append(("T", int(f[0]), float(f[1])))
        elif tag == "G":
            d.bubbles.append(("G", int(f[0]), float(f[1]), float(f[2])))
        elif tag == "V":
            d.violations.append(" ".join(f))
        elif tag == "X":
            d.infeasible = (float(f[0]), int(f[1]))
        elif tag == "W":
            d.infeasible = d.infeasible + (" ".join(f),)
        elif tag in ("U", "Q"):
            rec = (int(f[0]), int(f[1]), int(f[2]), int(f[3]), int(f[4]), int(f[5]), float(f[6]),
                   int(f[7]), tuple(int(x) for x in f[8:]))
            (d.unplaced if tag == "U" else d.queue).append(rec)
    return d


class _RefConfig(C.Structure):  # oracle/ref_shim.cpp RefConfig
    _fields_ = [(n, C.c_int) for n in ("method", "stages", "micro_batches", "micro_batch_size",
                                       "replicas", "devices", "layers_per_stage", "seq_len",
                                       "recompute")]


class _RefCosts(C.Structure):  # oracle/ref_shim.cpp RefCosts
    _fields_ = ([(n, C.c_double) for n in ("t_f", "t_b", "t_curv", "t_inv", "t_prec")]
                + [(n, C.c_longlong) for n in ("m_theta", "m_act", "m_err_peak", "m_err_save",
                                               "m_curv")]
                + [(n, C.c_double) for n in ("comm_alpha", "comm_beta", "p2p_latency")])


def _structs(cfg, costs):
    """Any objects carrying the PipelineConfig / CostTable attribute names."""
    c = _RefConfig(*(int(getattr(cfg, n)) for n, _ in _RefConfig._fields_))
    t = _RefCosts(*((int if ty is C.c_longlong else float)(getattr(costs, n))
                    for n, ty in _RefCosts._fields_))
    return c, t


def ref_build_dump(cfg, costs, horizon: int = 1) -> Dump:
    c, t = _structs(cfg, costs)
    return _parse(_call_dump(ref().pfref_build_dump, C.byref(c), C.byref(t), horizon))


def ref_queue_dump(cfg, costs) -> Dump:
    c, t = _structs(cfg, costs)
    return _parse(_call_dump(ref().pfref_queue_dump, C.byref(c), C.byref(t)))


def ref_assign_dump(cfg, costs, inversion_parallel=False, horizon_cap=10) -> Dump:
    c, t = _structs(cfg, costs)
    return _parse(_call_dump(ref().pfref_assign_dump, C.byref(c), C.byref(t),
                             int(inversion_parallel), horizon_cap))


def ref_assign_trace(cfg, costs, inversion_parallel=False, horizon_cap=10, devices_per_group=0) -> str:
    """io::trace_to_json (proj/src/io/trace.cpp:38-63) of the reference's
    assign_works schedule (oracle/_ref built with nlohmann json)."""
    c, t = _structs(cfg, costs)
    return _call_dump(ref().pfref_assign_trace, C.byref(c), C.byref(t), int(inversion_parallel), horizon_cap,
                      devices_per_group)


def ref_block_diag_split(m: np.ndarray, k: int):
    """kfac::block_diag_split_factor + inversion_flops (proj/src/kfac/kfac.cpp:203-226)."""
    m = np.ascontiguousarray(m, dtype=np.float64)
    d = m.shape[0]
    b = d // k
    out = np.zeros((k, b, b))
    ff, fb = C.c_double(), C.c_double()
    _ref_call(ref().pfref_block_diag_split(_ptr(m), d, k, _ptr(out), C.byref(ff), C.byref(fb)))
    return list(out), ff.value, fb.value
