"""Python mirror of the reference K-FAC API (``pipefill::kfac`` in
/root/reference/proj/include/pipefill/kfac/{kfac,matrix}.hpp) running on the
B200 kernels through the C-ABI (include/pf_kfac.h).

Tensors are CUDA torch tensors (torch is plumbing: allocation and streams).
Layout follows the reference: a BatchTape holds a_l (d_in x batch) and e_l
(d_out x batch) with examples as columns — on the device in bf16, which is
exactly the K-major operand the tcgen05 SYRK consumes.  Factors, inverses,
gradients and weights are fp32, row-major.

Errors follow the reference: shape mismatches raise ``ValueError``
(std::invalid_argument), a failed Cholesky pivot raises
:class:`NotPositiveDefinite` (std::domain_error), raised after the stream
is synchronised.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from . import _lib as L


class NotPositiveDefinite(ArithmeticError):
    """std::domain_error("cholesky: matrix not positive definite")."""

    def __init__(self, column: int):
        super().__init__(f"cholesky: matrix not positive definite (damping too small?) "
                         f"at column {column}")
        self.column = column


def _require_device(t: torch.Tensor, what: str):
    if not t.is_cuda:
        raise ValueError(f"{what}: expected a CUDA tensor (no CPU path exists)")


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def device_ok() -> bool:
    return bool(L.lib().pf_device_ok())


def kernel_launches() -> int:
    """Kernels launched by libpf_b200.so since load (host-side counter)."""
    return int(L.lib().pf_kernel_launch_count())


class background:
    """Context manager: calls issued inside run in background mode on this
    host thread (pf_set_background): least launch priority, no persistent
    GEMM CTAs -- for work placed on a second stream under a latency-bound
    inversion chain.  Results are bit-identical to a normal call."""

    def __enter__(self):
        self._was = L.lib().pf_set_background(1)
        return self

    def __exit__(self, *exc):
        L.lib().pf_set_background(self._was)
        return False


class _Workspaces:
    """Scratch arena per (device, tag, stream): grows, never shrinks; hot calls
    allocate nothing.  Keyed by the launching stream because calls on
    different streams run concurrently (the K-FAC stream's inversions beside
    the compute stream's preconditioning, one stream set per virtual device in
    vdev.py); calls on one stream are ordered, so they can share."""

    def __init__(self):
        self._bufs: Dict[Tuple[int, str, int], torch.Tensor] = {}
        # buffers replaced by a bigger one stay allocated: a CUDA graph
        # captured while one was current still reads and writes it at every
        # replay (freeing it crashed such a replay)
        self._retired: List[torch.Tensor] = []

    def get(self, nbytes: int, device: torch.device, tag: str = "ws") -> torch.Tensor:
        key = (device.index or 0, tag, torch.cuda.current_stream(device).cuda_stream)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if buf is not None:
                self._retired.append(buf)
            buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
            self._bufs[key] = buf
        return buf


_WS = _Workspaces()


def to_tape_layout(x: torch.Tensor) -> torch.Tensor:
    """bf16, contiguous, column count padded to a multiple of 8 (16-byte rows
    for TMA); zero columns do not change X X^T."""
    _require_device(x, "tape")
    if x.dim() != 2:
        raise ValueError("tape matrices are 2-D (features x examples)")
    d, n = x.shape
    n8 = (n + 7) // 8 * 8
    if x.dtype == torch.bfloat16 and x.is_contiguous() and n8 == n:
        return x
    out = torch.zeros((d, n8), dtype=torch.bfloat16, device=x.device)
    out[:, :n] = x
    return out


# ------------------------------------------------------------------ curvature
def syrk(problems: Sequence[Tuple], fill_upper: bool = True) -> None:
    """Grouped F = scale * X X^T (+F).  problems: (x_bf16, f_fp32 [d x d],
    scale, accumulate[, token_major]).  x is [d x n] (examples contiguous,
    the BatchTape layout) or, with token_major=True, [n x d] -- a layer's
    activations / output gradients as produced (features contiguous), read
    in place by the tensor cores (MN-major operand), no transposed copy."""
    arr = (L.PfSyrkProblem * len(problems))()
    for i, prob in enumerate(problems):
        x, f, scale, acc = prob[:4]
        tm = bool(prob[4]) if len(prob) > 4 else False
        _require_device(x, "syrk x")
        _require_device(f, "syrk f")
        if x.dtype != torch.bfloat16 or f.dtype != torch.float32:
            raise ValueError("syrk: x must be bf16 and f fp32")
        if x.dim() != 2 or x.stride(1) != 1 or f.stride(1) != 1:
            raise ValueError("syrk: x and f need contiguous rows")
        d, n = (x.shape[1], x.shape[0]) if tm else (x.shape[0], x.shape[1])
        if f.shape != (d, d):
            raise ValueError("syrk: shape mismatch")
        arr[i] = L.PfSyrkProblem(x.data_ptr(), f.data_ptr(), d, n, x.stride(0), f.stride(0), float(scale),
                                 int(bool(acc)), 1 if tm else 0)
    L.check(L.lib().pf_curvature_syrk_grouped(arr, len(problems), int(fill_upper), _stream()),
            "curvature_syrk")


@dataclass
class BatchTape:  # kfac.hpp:33-37
    layer_inputs: List[torch.Tensor] = field(default_factory=list)   # a_l: d_in x batch
    layer_errors: List[torch.Tensor] = field(default_factory=list)   # e_l: d_out x batch
    batch_size: int = 0


def curvature_factors(tape: BatchTape, layer: int) -> Tuple[torch.Tensor, torch.Tensor]:
    """A = (1/bs) a a^T, B = (1/bs) e e^T (kfac.cpp:125-131), one grouped launch."""
    a = to_tape_layout(tape.layer_inputs[layer])
    e = to_tape_layout(tape.layer_errors[layer])
    if tape.batch_size < 1:
        raise ValueError("batch is empty")
    A = torch.empty((a.shape[0], a.shape[0]), dtype=torch.float32, device=a.device)
    B = torch.empty((e.shape[0], e.shape[0]), dtype=torch.float32, device=e.device)
    inv_b = 1.0 / tape.batch_size
    syrk([(a, A, inv_b, False), (e, B, inv_b, False)])
    return A, B


# ------------------------------------------------------------------ inverse
def inverse_workspace_bytes(d: int) -> int:
    n = C.c_size_t()
    L.check(L.lib().pf_damped_inverse_workspace(d, n), "inverse workspace")
    return n.value


def slice_bytes(rows: int, k: int) -> int:
    n = C.c_size_t()
    L.check(L.lib().pf_slice_bytes(rows, k, n), "slice bytes")
    return n.value


@dataclass
class SlicedMatrix:
    """Digit form of an fp32 matrix (pf_slice): what the tensor-core
    preconditioner consumes.  ``fp32`` keeps the plain inverse."""
    fp32: torch.Tensor
    digits: torch.Tensor  # uint8 buffer of slice_bytes(rows, k)


def slice_matrix(x: torch.Tensor) -> SlicedMatrix:
    _require_device(x, "slice")
    if x.dtype != torch.float32 or x.stride(1) != 1:
        raise ValueError("slice: expects row-major fp32")
    buf = torch.empty(slice_bytes(x.shape[0], x.shape[1]), dtype=torch.uint8, device=x.device)
    L.check(L.lib().pf_slice(x.data_ptr(), x.shape[0], x.shape[1], x.stride(0), buf.data_ptr(),
                             _stream()), "slice")
    return SlicedMatrix(x, buf)


def damped_inverse_batched(mats: Sequence[torch.Tensor], damping: float,
                           outs: Optional[Sequence[torch.Tensor]] = None,
                           digits: Optional[Sequence[torch.Tensor]] = None,
                           check: bool = True) -> List[torch.Tensor]:
    """(M_i + damping I)^-1 for every M_i in one batched launch sequence.
    With ``digits`` (uint8 buffers of slice_bytes(d, d)) the digit form of each
    inverse is written as well."""
    if not mats:
        return []
    dev = mats[0].device
    sizes = [inverse_workspace_bytes(m.shape[0]) for m in mats]
    offs, total = [], 0
    for s in sizes:
        offs.append(total)
        total += (s + 255) // 256 * 256
    ws = _WS.get(total, dev, "inverse")
    info = _WS.get(4 * len(mats), dev, "info").view(torch.int32)[: len(mats)]
    outs = list(outs) if outs is not None else [torch.empty_like(m, dtype=torch.float32) for m in mats]
    arr = (L.PfInverseProblem * len(mats))()
    for i, m in enumerate(mats):
        _require_device(m, "cholesky_spd_inverse")
        if m.dim() != 2 or m.shape[0] != m.shape[1]:
            raise ValueError("cholesky_spd_inverse: matrix not square")
        if m.dtype != torch.float32 or m.stride(1) != 1:
            raise ValueError("cholesky_spd_inverse: expects row-major fp32")
        dg = None if digits is None else digits[i]
        arr[i] = L.PfInverseProblem(m.data_ptr(), outs[i].data_ptr(), _ptr(dg), m.shape[0],
                                    m.stride(0), outs[i].stride(0), float(damping),
                                    ws.data_ptr() + offs[i], info[i:].data_ptr())
    L.check(L.lib().pf_damped_inverse_batched(arr, len(mats), _stream()), "damped_inverse")
    if check:
        bad = info.cpu()
        for i in range(len(mats)):
            if int(bad[i]) != 0:
                raise NotPositiveDefinite(int(bad[i]))
    return outs


def cholesky_factor(m: torch.Tensor, damping: float = 0.0, out: Optional[torch.Tensor] = None,
                    check: bool = True) -> torch.Tensor:
    """matrix.cpp:117-134: lower L with L L^T = M (+ damping I), zeros above,
    on the GPU (pf_cholesky_factor: the damped inverse's factorisation).  Reads
    the lower triangle of M.  A non-positive or non-finite pivot raises
    NotPositiveDefinite with its 1-based column (the reference's
    std::domain_error)."""
    _require_device(m, "cholesky_factor")
    if m.dim() != 2 or m.shape[0] != m.shape[1]:
        raise ValueError("cholesky_factor: matrix not square")
    if m.dtype != torch.float32 or m.stride(1) != 1:
        raise ValueError("cholesky_factor: expects row-major fp32")
    d = m.shape[0]
    if out is None:
        out = torch.empty((d, d), dtype=torch.float32, device=m.device)
    elif out.shape != m.shape or out.dtype != torch.float32 or out.stride(1) != 1 or out.device != m.device:
        raise ValueError("cholesky_factor: bad output buffer")
    if d == 0:
        return out
    ws_bytes = inverse_workspace_bytes(d)
    ws = _WS.get(ws_bytes, m.device, "inverse")
    info = _WS.get(4, m.device, "info").view(torch.int32)[:1]
    L.check(L.lib().pf_cholesky_factor(m.data_ptr(), d, m.stride(0), float(damping), out.data_ptr(),
                                       out.stride(0), ws.data_ptr(), ws_bytes, info.data_ptr(), _stream()),
            "cholesky_factor")
    if check:
        bad = int(info.cpu()[0])
        if bad != 0:
            raise NotPositiveDefinite(bad)
    return out


def block_diag_split_factor(m: torch.Tensor, k: int) -> List[torch.Tensor]:
    """kfac.cpp:203-218: the K diagonal blocks of a square factor (copies)."""
    if m.dim() != 2 or m.shape[0] != m.shape[1]:
        raise ValueError("factor must be square")
    d = m.shape[0]
    if k < 1 or d % k != 0:
        raise ValueError("K must divide the factor dimension")
    b = d // k
    return [m[i * b:(i + 1) * b, i * b:(i + 1) * b].clone() for i in range(k)]


def inversion_flops(dim: int) -> float:
    """kfac.cpp:220-222 (the reference cost model's (2/3) d^3)."""
    return (2.0 / 3.0) * float(dim) * dim * dim


def block_diag_inversion_flops(dim: int, k: int) -> float:
    """kfac.cpp:224-227."""
    if k < 1 or dim % k != 0:
        raise ValueError("K must divide the dimension")
    return k * inversion_flops(dim // k)


def damped_inverse_block_diag(mats: Sequence[torch.Tensor], damping: float, k: int,
                              outs: Optional[Sequence[torch.Tensor]] = None,
                              digits: Optional[Sequence[torch.Tensor]] = None,
                              check: bool = True) -> List[torch.Tensor]:
    """Block-diagonal K-FAC for large factors (§A, kfac.cpp:203-226):
    each factor is replaced by its K diagonal blocks, so its inversion costs
    d^3 / K^2.  The damped inverses of every block of every factor run as ONE
    batched call, reading and writing views of the full matrices (no copies);
    the off-diagonal blocks of the inverse are zero.  With ``digits`` the digit
    form of the assembled block-diagonal inverse is written for the
    preconditioner."""
    outs = list(outs) if outs is not None else [torch.empty_like(m, dtype=torch.float32) for m in mats]
    blocks_in, blocks_out = [], []
    for m, o in zip(mats, outs):
        d = m.shape[0]
        if k < 1 or d % k != 0:
            raise ValueError("K must divide the factor dimension")
        b = d // k
        o.zero_()
        for i in range(k):
            blocks_in.append(m[i * b:(i + 1) * b, i * b:(i + 1) * b])
            blocks_out.append(o[i * b:(i + 1) * b, i * b:(i + 1) * b])
    damped_inverse_batched(blocks_in, damping, blocks_out, None, check=check)
    if digits is not None:
        for o, dg in zip(outs, digits):
            L.check(L.lib().pf_slice(o.data_ptr(), o.shape[0], o.shape[1], o.stride(0), dg.data_ptr(),
                                     _stream()), "slice")
    return outs


def cholesky_spd_inverse(m: torch.Tensor, damping: float) -> torch.Tensor:
    """matrix.hpp:58 — (M + damping I)^-1 via Cholesky (fp32-accurate)."""
    return damped_inverse_batched([m], damping)[0]


# ------------------------------------------------------------------ precondition
def precondition_workspace_bytes(d_out: int, d_in: int) -> int:
    n = C.c_size_t()
    L.check(L.lib().pf_precondition_workspace(d_out, d_in, n), "precondition workspace")
    return n.value


def _check_prec(grad, a_inv, b_inv):
    for t, n in ((grad, "grad"), (a_inv, "a_inv"), (b_inv, "b_inv")):
        _require_device(t, n)
        if t.dtype != torch.float32 or not t.is_contiguous():
            raise ValueError(f"precondition: {n} must be contiguous fp32")
    if b_inv.shape[1] != grad.shape[0] or grad.shape[1] != a_inv.shape[0]:
        raise ValueError("precondition: shape mismatch")


def precondition(grad: torch.Tensor, a_inv: torch.Tensor, b_inv: torch.Tensor) -> torch.Tensor:
    """kfac.hpp:51 — B^-1 G A^-1 (two chained fp32-accurate int8-digit tensor-core GEMMs)."""
    _check_prec(grad, a_inv, b_inv)
    d_out, d_in = grad.shape
    out = torch.empty_like(grad)
    nb = precondition_workspace_bytes(d_out, d_in)
    ws = _WS.get(nb, grad.device, "prec")
    L.check(L.lib().pf_precondition(b_inv.data_ptr(), grad.data_ptr(), a_inv.data_ptr(),
                                    out.data_ptr(), d_out, d_in, ws.data_ptr(), nb, _stream()),
            "precondition")
    return out


def precondition_update(weight: torch.Tensor, grad: torch.Tensor, a_inv: torch.Tensor,
                        b_inv: torch.Tensor, eta: float) -> None:
    """W -= eta * B^-1 G A^-1, update fused into the second GEMM's epilogue."""
    _check_prec(grad, a_inv, b_inv)
    if weight.shape != grad.shape or not weight.is_contiguous() or weight.dtype != torch.float32:
        raise ValueError("precondition_update: weight shape mismatch")
    d_out, d_in = grad.shape
    nb = precondition_workspace_bytes(d_out, d_in)
    ws = _WS.get(nb, grad.device, "prec")
    L.check(L.lib().pf_precondition_update(b_inv.data_ptr(), grad.data_ptr(), a_inv.data_ptr(),
                                           weight.data_ptr(), d_out, d_in, float(eta),
                                           ws.data_ptr(), nb, _stream()),
            "precondition_update")


def _check_f32_2d(t: torch.Tensor, what: str, dev: torch.device) -> None:
    _require_device(t, what)
    if t.dim() != 2 or t.dtype != torch.float32 or not t.is_contiguous() or t.device != dev:
        raise ValueError(f"precondition: {what} must be a contiguous 2-D fp32 tensor on {dev}")


def precondition_update_sliced(items: Sequence[Tuple[Optional[torch.Tensor], torch.Tensor,
                                                     SlicedMatrix, SlicedMatrix, float]],
                               p_out: Optional[Sequence[torch.Tensor]] = None) -> None:
    """Grouped W_i -= eta_i B_i^-1 G_i A_i^-1 with inverses in digit form.
    items: (weight or None, grad, a_inv, b_inv, eta); p_out receives P instead."""
    if not items:
        return
    dev = items[0][1].device
    sizes = [precondition_workspace_bytes(g.shape[0], g.shape[1]) for _, g, _, _, _ in items]
    offs, total = [], 0
    for s in sizes:
        offs.append(total)
        total += (s + 255) // 256 * 256
    ws = _WS.get(total, dev, "prec_sliced")
    arr = (L.PfPreconditionProblem * len(items))()
    for i, (w, g, ai, bi, eta) in enumerate(items):
        _check_f32_2d(g, "grad", dev)
        d_out, d_in = g.shape
        if w is not None:
            _check_f32_2d(w, "weight", dev)
            if w.shape != g.shape:
                raise ValueError("precondition: weight shape mismatch")
        if p_out is not None:
            _check_f32_2d(p_out[i], "p_out", dev)
            if p_out[i].shape != g.shape:
                raise ValueError("precondition: p_out shape mismatch")
        if w is None and p_out is None:
            raise ValueError("precondition: need a weight or p_out")
        if ai.fp32.shape != (d_in, d_in) or bi.fp32.shape != (d_out, d_out):
            raise ValueError("precondition: shape mismatch")
        for sm, d in ((ai, d_in), (bi, d_out)):
            if (sm.digits.device != dev or sm.digits.dtype != torch.uint8
                    or sm.digits.numel() < slice_bytes(d, d) or not sm.digits.is_contiguous()):
                raise ValueError("precondition: digit-form inverse has the wrong size or device")
        arr[i] = L.PfPreconditionProblem(bi.digits.data_ptr(), g.data_ptr(), ai.digits.data_ptr(),
                                         _ptr(w), None if p_out is None else p_out[i].data_ptr(),
                                         d_out, d_in, float(eta), ws.data_ptr() + offs[i])
    L.check(L.lib().pf_precondition_update_sliced(arr, len(items), _stream()),
            "precondition_update_sliced")


# ------------------------------------------------------------------ state / step
class KfacState:
    """kfac.hpp:60-73: per-layer factors, damped inverses (fp32 + digit form), staleness."""

    def __init__(self, layers: int = 0, damping: float = 0.0, learning_rate: float = 0.0,
                 block_diag_k: int = 1):
        self.factor_a: List[Optional[torch.Tensor]] = [None] * layers
        self.factor_b: List[Optional[torch.Tensor]] = [None] * layers
        self.inv_a: List[Optional[SlicedMatrix]] = [None] * layers
        self.inv_b: List[Optional[SlicedMatrix]] = [None] * layers
        self.staleness = [0] * layers
        self.refreshed_this_step = [False] * layers
        self.damping = damping
        self.learning_rate = learning_rate
        # > 1: factors whose dimension K divides are inverted block-diagonally
        # (kfac.cpp:203-226); the others in full
        self.block_diag_k = block_diag_k

    def has_inverses(self, layer: int) -> bool:
        return self.inv_a[layer] is not None and self.inv_b[layer] is not None

    def update_factors(self, tape: BatchTape) -> None:
        """Overwrites the factors (no EMA), all layers in one grouped launch."""
        probs = []
        inv_b = 1.0 / tape.batch_size
        for l in range(len(self.factor_a)):
            a = to_tape_layout(tape.layer_inputs[l])
            e = to_tape_layout(tape.layer_errors[l])
            if self.factor_a[l] is None or self.factor_a[l].shape[0] != a.shape[0]:
                self.factor_a[l] = torch.empty((a.shape[0],) * 2, dtype=torch.float32, device=a.device)
            if self.factor_b[l] is None or self.factor_b[l].shape[0] != e.shape[0]:
                self.factor_b[l] = torch.empty((e.shape[0],) * 2, dtype=torch.float32, device=e.device)
            probs += [(a, self.factor_a[l], inv_b, False), (e, self.factor_b[l], inv_b, False)]
        syrk(probs, fill_upper=False)  # inversion reads the lower triangle only

    def refresh_inverses(self) -> None:
        """Invert every layer's damped factors (batched); resets staleness."""
        mats, slots = [], []
        for l in range(len(self.factor_a)):
            if self.factor_a[l] is None:
                continue
            mats += [self.factor_a[l], self.factor_b[l]]
            slots += [(l, 0), (l, 1)]
        if not mats:
            return
        outs = [torch.empty_like(m) for m in mats]
        digits = [torch.empty(slice_bytes(m.shape[0], m.shape[0]), dtype=torch.uint8,
                              device=m.device) for m in mats]
        k = self.block_diag_k
        bd = [i for i, m in enumerate(mats) if k > 1 and m.shape[0] % k == 0]
        full = [i for i in range(len(mats)) if i not in set(bd)]
        if full:
            damped_inverse_batched([mats[i] for i in full], self.damping, [outs[i] for i in full],
                                   [digits[i] for i in full])
        if bd:
            damped_inverse_block_diag([mats[i] for i in bd], self.damping, k, [outs[i] for i in bd],
                                      [digits[i] for i in bd])
        for (l, which), o, dg in zip(slots, outs, digits):
            (self.inv_a if which == 0 else self.inv_b)[l] = SlicedMatrix(o, dg)
            self.staleness[l] = 0
            self.refreshed_this_step[l] = True


@dataclass
class NgdStepResult:
    used_plain_gradient: bool = False


def ngd_step(weights: List[torch.Tensor], state: KfacState,
             gradients: List[torch.Tensor]) -> NgdStepResult:
    """kfac.cpp:186-201: theta_l -= eta * B^-1 G_l A^-1 (grouped, fused update);
    layers without inverses take the plain gradient and set the flag."""
    if len(gradients) != len(weights):
        raise ValueError("one gradient per layer required")
    out = NgdStepResult()
    items = []
    for l, (w, g) in enumerate(zip(weights, gradients)):
        if state.has_inverses(l):
            items.append((w, g, state.inv_a[l], state.inv_b[l], state.learning_rate))
        else:
            out.used_plain_gradient = True
            w.sub_(g * state.learning_rate)
        state.staleness[l] = (0 if state.refreshed_this_step[l] else state.staleness[l]) + 1
        state.refreshed_this_step[l] = False
    precondition_update_sliced(items)
    return out
