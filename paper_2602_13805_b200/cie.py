"""Contrast-integral-equation algebra (reference cie.py), GPU underneath.

  chi_to_r / r_to_chi     cie.py:24-39   -> pdf_chi_to_r (PoleError below 1e-14)
  default_eps_reg         cie.py:42-50   -> pdf_default_eps_reg
  pixel_least_squares     cie.py:66-80   -> pdf_pixel_ls
  recover_contrast        cie.py:83-99   -> api.recover_contrast
  cie_state_residual      cie.py:102-114 -> pdf_expand, pdf_apply_gd, pdf_cie_fields

Host arrays in, host arrays out, like the reference.  The *_dev helpers take
and return complex128 CUDA tensors; the solver API builds its intermediates
from them (api._recovery_dev, api.pipeline_forward).  Inside the training
step the same algebra is fused into the view / pixel kernels.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import PoleError


@dataclass
class ContrastRecovery:
    """recover_contrast with its reusable intermediates (cie.py:53-63)."""
    chi: np.ndarray           # (m1, m2)
    j_views: np.ndarray       # (n, m1, m2) currents expand(alpha)
    e_views: np.ndarray       # (n, m1, m2) total fields E_inc + G_D J
    numerator: np.ndarray     # (m1, m2) sum_i J_i conj(E_i)
    denominator: np.ndarray   # (m1, m2) real, sum_i |E_i|^2 + eps_reg
    eps_reg: float
    degenerate: np.ndarray    # (m1, m2) bool, denominator <= 10 eps_reg


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("the CIE algebra runs on the GPU (no CPU fallback)")
    return torch.device("cuda")


def _st():
    return ct.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t: torch.Tensor | None):
    return ct.c_void_p(0 if t is None else t.data_ptr())


def _c(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=_dev(), dtype=torch.complex128).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.complex128), device=_dev())


def _beta(beta) -> tuple[float, float]:
    b = complex(beta)
    return b.real, b.imag


# ---------------------------------------------------------------------------- device forms
def chi_to_r_dev(x: torch.Tensor, beta, inverse: bool = False, check: bool = True):
    """R = beta chi / (beta chi + 1) (or its inverse) on the device; with check=False
    the pole count stays a device scalar (second return value)."""
    x = _c(x)
    y = torch.empty_like(x)
    poles = torch.zeros(1, dtype=torch.int32, device=x.device)
    br, bi = _beta(beta)
    N.check(N.lib().pdf_chi_to_r(_p(x), _p(y), x.numel(), br, bi, int(inverse), _p(poles), _st()))
    if check:
        if int(poles.item()):
            raise PoleError("1 - R vanishes at some pixel" if inverse else "beta*chi + 1 vanishes at some pixel")
        return y
    return y, poles


def default_eps_reg_dev(e: torch.Tensor) -> torch.Tensor:
    """1e-10 max_v ||E_v||^2 / n_pix as a 0-d device tensor (views = all leading dims)."""
    e = _c(e)
    npix = e.shape[-1] * e.shape[-2]
    eps = torch.empty((), dtype=torch.float64, device=e.device)
    N.check(N.lib().pdf_default_eps_reg(_p(e), e.numel() // npix, npix, _p(eps), _st()))
    return eps


def pixel_ls_dev(j: torch.Tensor, e: torch.Tensor, eps: torch.Tensor):
    """(num, den, chi, degenerate) device tensors for views (n, m1, m2)."""
    j, e = _c(j), _c(e)
    if j.shape != e.shape or j.dim() != 3:
        raise ValueError("current and field views must share an (n, m1, m2) shape")
    n, m1, m2 = j.shape
    num = torch.empty((m1, m2), dtype=torch.complex128, device=j.device)
    chi = torch.empty_like(num)
    den = torch.empty((m1, m2), dtype=torch.float64, device=j.device)
    deg = torch.empty((m1, m2), dtype=torch.uint8, device=j.device)
    eps = eps.to(device=j.device, dtype=torch.float64).reshape(()).contiguous()
    N.check(N.lib().pdf_pixel_ls(_p(j), _p(e), n, m1 * m2, _p(eps), _p(num), _p(den), _p(chi), _p(deg), _st()))
    return num, den, chi, deg.bool()


def cie_fields_dev(j, e_in, beta=0.0, gdj=None, r_hat=None, want=("e",)):
    """E = e_in + gdj, P = E + beta J, res = r_hat P - beta J for views (n, m1, m2);
    e_in (n, m1, m2) or one shared (m1, m2) image.  Returns the requested tensors."""
    j = _c(j)
    n, m1, m2 = j.shape
    npix = m1 * m2
    e_in = _c(e_in)
    stride = 0 if e_in.dim() == 2 else npix
    gdj = None if gdj is None else _c(gdj)
    r_hat = None if r_hat is None else _c(r_hat)
    out = {k: torch.empty_like(j) for k in want}
    br, bi = _beta(beta)
    N.check(N.lib().pdf_cie_fields(_p(j), _p(gdj), _p(e_in), stride, _p(r_hat), br, bi, n, npix, _p(out.get("e")),
                                   _p(out.get("p")), _p(out.get("res")), _st()))
    return tuple(out[k] for k in want)


def masked_residual_dev(a: torch.Tensor, b: torch.Tensor, mask: torch.Tensor | None):
    a, b = _c(a), _c(b)
    out = torch.empty_like(a)
    mk = None if mask is None else mask.to(device=a.device, dtype=torch.float64).expand(a.shape).contiguous()
    N.check(N.lib().pdf_masked_residual(_p(a), _p(b), _p(mk), _p(out), a.numel(), _st()))
    return out


# ---------------------------------------------------------------------------- reference signatures
def chi_to_r(chi, beta) -> np.ndarray:
    """Modified contrast R = beta chi / (beta chi + 1) (cie.py:24-30)."""
    chi = np.asarray(chi, dtype=np.complex128)
    return chi_to_r_dev(chi, beta).cpu().numpy().reshape(chi.shape)


def r_to_chi(r, beta) -> np.ndarray:
    """Inverse mapping chi = R / (beta (1 - R)) (cie.py:33-39)."""
    r = np.asarray(r, dtype=np.complex128)
    return chi_to_r_dev(r, beta, inverse=True).cpu().numpy().reshape(r.shape)


def default_eps_reg(e_views) -> float:
    """Regulariser floor 1e-10 max_view ||E||^2 / n_cells (cie.py:42-50)."""
    return float(default_eps_reg_dev(e_views).item())


def pixel_least_squares(j_views, e_views, eps_reg: float | None = None) -> ContrastRecovery:
    """Per-pixel LS contrast chi = sum_i J_i conj(E_i) / (sum_i |E_i|^2 + eps_reg) (cie.py:66-80)."""
    jh, eh = np.asarray(j_views), np.asarray(e_views)
    j, e = _c(jh), _c(eh)
    eps = default_eps_reg_dev(e) if eps_reg is None else torch.tensor(float(eps_reg), dtype=torch.float64,
                                                                      device=j.device)
    num, den, chi, deg = pixel_ls_dev(j, e, eps)
    return ContrastRecovery(chi=chi.cpu().numpy(), j_views=jh, e_views=eh, numerator=num.cpu().numpy(),
                            denominator=den.cpu().numpy(), eps_reg=float(eps.item()), degenerate=deg.cpu().numpy())


def cie_state_residual(alpha, r_hat, e_inc, ops, basis, beta) -> np.ndarray:
    """R (E_inc + G_D J + beta J) - beta J per view, J = expand(alpha) (cie.py:102-114)."""
    from .api import _basis_device, _ops_device
    alpha = np.atleast_2d(np.asarray(alpha, dtype=np.complex128))
    j = _basis_device(basis).expand(_c(alpha))
    gdj = _ops_device(ops).apply_gd(j)
    n = alpha.shape[0]
    e_inc, r_hat = np.asarray(e_inc), np.asarray(r_hat)
    if e_inc.ndim == 3 and e_inc.shape[0] not in (1, n):
        raise ValueError(f"{e_inc.shape[0]} incident views for {n} coefficient vectors")
    e_in = e_inc[0] if e_inc.ndim == 3 and e_inc.shape[0] == 1 else e_inc
    if r_hat.ndim == 2:
        (res,) = cie_fields_dev(j, e_in, beta, gdj=gdj, r_hat=r_hat, want=("res",))
    else:       # one modified contrast per view
        if r_hat.shape[0] != n:
            raise ValueError("r_hat must be (m1, m2) or one image per view")
        res = torch.cat([cie_fields_dev(j[v:v + 1], e_in if e_in.ndim == 2 else e_in[v:v + 1], beta,
                                        gdj=gdj[v:v + 1], r_hat=r_hat[v], want=("res",))[0] for v in range(n)])
    return res.cpu().numpy()


def __getattr__(name):
    if name == "recover_contrast":
        from .api import recover_contrast
        return recover_contrast
    raise AttributeError(name)
