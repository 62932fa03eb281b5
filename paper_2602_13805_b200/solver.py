"""Method-of-moments forward solve on the GPU.

`solve_fields_gpu` runs the library's batched BiCGStab (pdf_solve_total_field,
csrc/pdf_solver.cu) on (I - G_D chi) E = E_inc for every view of S scenes at
once, with the reference's restart clause and NoConvergenceError
(forward.py:193-248); `operators.solve_total_field(method="fft")` and
`simulate()` reach it for grids above 1024 cells, as the reference picks its
FFT/Krylov path there (forward.py:263-264, 367-369).
"""
from __future__ import annotations

import ctypes as ct

import numpy as np
import torch

from . import _native as N


class _SolverDevice:
    """A float64 context over the operators (only its G_D is used) + workspace."""

    def __init__(self, ops):
        from dataclasses import replace
        from .engine import DeviceProblem
        M = ops.m1
        gs1 = ops.gs_matrix[:1]
        gs1 = gs1.contiguous() if isinstance(gs1, torch.Tensor) else np.ascontiguousarray(gs1)
        one_rx = replace(ops, gs_matrix=gs1)   # views / receivers unused (host or device operators)
        self.dev = DeviceProblem(one_rx, np.ones((1, M, M), complex), np.ones((1, 1), complex), mf=1, beta=6.0,
                                 lambdas=(0, 0, 0), tau_b=0.5)
        self.ws = None

    def workspace(self, views: int) -> torch.Tensor:
        need = N.lib().pdf_solver_workspace_bytes(self.dev.ctx, int(views))
        if need == 0:
            raise ValueError(N.lib().pdf_last_error().decode())
        if self.ws is None or self.ws.numel() < need:
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.dev.device)
        return self.ws


_CACHE: list = []


def _solver_device(ops) -> _SolverDevice:
    for o, sd in _CACHE:
        if o is ops:
            return sd
    sd = _SolverDevice(ops)
    _CACHE.append((ops, sd))
    if len(_CACHE) > 2:
        _CACHE.pop(0)
    return sd


def solve_fields_gpu(chi, e_inc, ops, tol: float = 1e-8, maxiter: int = 2000):
    """Total fields E (S, n, M, M) complex128 on the device and the relative
    residuals ||E - E_inc - G_D(chi E)|| / ||E_inc|| (S, n) for contrasts chi
    (S, M, M) or (M, M) and incident fields e_inc (n, M, M) shared or
    (S, n, M, M) per scene (host arrays or device tensors).  Raises
    NoConvergenceError (the reference's message) when a view has not converged."""
    from .operators import NoConvergenceError
    if not torch.cuda.is_available():
        raise RuntimeError("the forward solve runs on the GPU (no CPU fallback)")
    dev_ = torch.device("cuda")
    chi_t = torch.as_tensor(chi, dtype=torch.complex128, device=dev_)
    b_t = torch.as_tensor(e_inc, dtype=torch.complex128, device=dev_)
    if chi_t.dim() == 2:
        chi_t = chi_t[None]
    chi_t = chi_t.contiguous()
    S, M = chi_t.shape[0], chi_t.shape[-1]
    n = b_t.shape[-3]
    if b_t.dim() == 4 and b_t.shape[0] != S:
        raise ValueError("per-scene incident fields and contrasts disagree in the scene count")
    if chi_t.shape[-2:] != b_t.shape[-2:]:
        raise ValueError("contrast grid and incident views disagree in shape")
    b_t = b_t.contiguous()
    sd = _solver_device(ops)
    ws = sd.workspace(S * n)
    x = torch.empty((S, n, M, M), dtype=torch.complex128, device=dev_)
    res = torch.empty((S, n), dtype=torch.float64, device=dev_)
    iters = ct.c_int32(0)
    stride = n * M * M if b_t.dim() == 4 else 0
    rc = N.lib().pdf_solve_total_field(sd.dev.ctx, ct.c_void_p(chi_t.data_ptr()), ct.c_void_p(b_t.data_ptr()), stride,
                                       ct.c_void_p(x.data_ptr()), S, n, float(tol), int(maxiter),
                                       ct.c_void_p(ws.data_ptr()), ws.numel(), ct.c_void_p(res.data_ptr()),
                                       ct.byref(iters), ct.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc == N.PDF_ENOCONV:
        raise NoConvergenceError(N.lib().pdf_last_error().decode())
    N.check(rc)
    return x, res, int(iters.value)
