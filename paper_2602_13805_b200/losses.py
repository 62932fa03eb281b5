"""Composite-loss terms (reference losses.py), GPU underneath.

  loss_data / loss_state                  losses.py:86-112  -> pdf_expand, pdf_gs_forward,
                                                               pdf_masked_residual / cie_state_residual
  loss_bound / loss_tv / loss_bridge      losses.py:115-137 -> pdf_regularizers (values)
  bound / tv / bridge_chi_grad,           losses.py:152-196 -> pdf_regularizers (gradients)
  regularizer_chi_grad
  LossContext ... grad_alpha              losses.py:36-312  -> api (fused pdf_loss_value / pdf_loss_grad)

Host arrays in, host arrays out.
"""
from __future__ import annotations

import ctypes as ct

import numpy as np
import torch

from . import _native as N
from .api import (EPS_TV, LossBreakdown, LossContext, PipelineState, grad_alpha, loss_total,  # noqa: F401
                  pipeline_backward, pipeline_forward)
from .cie import _c, _p, _st, cie_state_residual, masked_residual_dev
from .errors import ZeroDataError


def _regs(chi, tau_b: float = 0.5, eps_tv: float = EPS_TV, lambdas=(0.0, 0.0, 0.0), values: bool = False,
          grads: tuple = ()):
    x = _c(chi)
    if x.dim() != 2:
        raise ValueError("the regularisers take one 2-D contrast image")
    m1, m2 = x.shape
    vals = torch.empty(3, dtype=torch.float64, device=x.device) if values else None
    outs = {k: torch.empty_like(x) for k in grads}
    l1, l2, l3 = (float(v) for v in lambdas)
    N.check(N.lib().pdf_regularizers(_p(x), m1, m2, 1, float(tau_b), float(eps_tv), l1, l2, l3, _p(vals),
                                     _p(outs.get("bound")), _p(outs.get("tv")), _p(outs.get("bridge")),
                                     _p(outs.get("total")), _st()))
    return vals, outs


def loss_bound(chi) -> float:
    """Squared hinge on negative real contrast."""
    return float(_regs(chi, values=True)[0][0].item())


def loss_tv(chi, eps_tv: float = EPS_TV) -> float:
    """Smoothed isotropic total variation, forward differences (zero on the last row / column)."""
    return float(_regs(chi, eps_tv=eps_tv, values=True)[0][1].item())


def loss_bridge(chi, tau_b: float) -> float:
    """sum sigmoid((|chi| - tau_b) / tau_b) exp(-|grad |chi||^2)."""
    return float(_regs(chi, tau_b=tau_b, values=True)[0][2].item())


def bound_chi_grad(chi) -> np.ndarray:
    return _regs(chi, grads=("bound",))[1]["bound"].cpu().numpy()


def tv_chi_grad(chi, eps_tv: float = EPS_TV) -> np.ndarray:
    return _regs(chi, eps_tv=eps_tv, grads=("tv",))[1]["tv"].cpu().numpy()


def bridge_chi_grad(chi, tau_b: float) -> np.ndarray:
    return _regs(chi, tau_b=tau_b, grads=("bridge",))[1]["bridge"].cpu().numpy()


def regularizer_chi_grad(chi, lambdas: tuple[float, float, float], tau_b: float) -> np.ndarray:
    """l1 bound + l2 tv + l3 bridge gradients (zero weights skipped), dL/dRe + i dL/dIm."""
    return _regs(chi, tau_b=tau_b, lambdas=lambdas, grads=("total",))[1]["total"].cpu().numpy()


def _power(x: torch.Tensor) -> float:
    return float(torch.sum((x.conj() * x).real).item())


def loss_data(alpha, data, ops, basis, normalizer: float | None = None) -> float:
    """||G_S J - E_sca||^2 / ||E_sca||^2 over the views (mask applied to both)."""
    from .api import _basis_device, _ops_device
    alpha = np.atleast_2d(np.asarray(alpha, dtype=np.complex128))
    j = _basis_device(basis).expand(_c(alpha))
    rows = _ops_device(ops).gs_forward(j)
    mat = _c(data.matrix)
    mask = None if data.mask is None else torch.as_tensor(np.asarray(data.mask), device=mat.device)
    res = masked_residual_dev(rows, mat, mask)
    if normalizer is None:
        c = _power(mat if mask is None else mat * mask)
    else:
        c = float(normalizer)
    if c <= 0:
        raise ZeroDataError("measured scattered power is zero")
    return _power(res) / c


def loss_state(alpha, r_hat, e_inc, ops, basis, beta, normalizer: float | None = None) -> float:
    """Contraction-form state residual power over incident power."""
    res = cie_state_residual(alpha, r_hat, e_inc, ops, basis, beta)
    if normalizer is None:
        c = _power(_c(e_inc))
    else:
        c = float(normalizer)
    if c <= 0:
        raise ZeroDataError("incident power is zero")
    return _power(_c(res)) / c
