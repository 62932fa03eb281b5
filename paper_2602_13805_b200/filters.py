"""Windowed means, the guided filter and contrast compensation (reference
filters.py), GPU underneath, for images of any m1 x m2:

  box_mean       filters.py:16-33 -> pdf_box_mean
  guided_filter  filters.py:36-53 -> pdf_guided_filter
  apply_cco      filters.py:56-67 -> pdf_cco_image

Host arrays in, host arrays out.  The batched reconstruction applies CCO to
its scenes with the context entry pdf_apply_cco instead.
"""
from __future__ import annotations

import ctypes as ct

import numpy as np
import torch

from . import _native as N
from .config import CcoParams


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("the filters run on the GPU (no CPU fallback)")
    return torch.device("cuda")


def _st():
    return ct.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t: torch.Tensor):
    return ct.c_void_p(t.data_ptr())


def _real(x) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=_dev())


def box_mean(img, radius: int) -> np.ndarray:
    """Mean over (2r+1)^2 windows with edge-replicate padding, same shape."""
    if radius < 1:
        raise ValueError("radius must be >= 1")
    img = np.asarray(img)
    if img.ndim != 2:
        raise ValueError("box_mean expects a 2-D array")
    if np.iscomplexobj(img):
        return box_mean(img.real, radius) + 1j * box_mean(img.imag, radius)
    x = _real(img)
    out = torch.empty_like(x)
    N.check(N.lib().pdf_box_mean(_p(x), _p(out), img.shape[0], img.shape[1], int(radius), 1, _st()))
    return out.cpu().numpy()


def guided_filter(inp, guide, radius: int, eps_gf: float) -> np.ndarray:
    """Local-linear-model filter of a real image steered by a real guide."""
    inp, guide = np.asarray(inp), np.asarray(guide)
    if inp.shape != guide.shape:
        raise ValueError("input and guide must share a shape")
    if radius < 1:
        raise ValueError("radius must be >= 1")
    if inp.ndim != 2:
        raise ValueError("guided_filter expects 2-D images")
    p, g = _real(inp), _real(guide)
    out = torch.empty_like(p)
    scratch = torch.empty((2,) + p.shape, dtype=torch.float64, device=p.device)
    N.check(N.lib().pdf_guided_filter(_p(p), _p(g), _p(out), inp.shape[0], inp.shape[1], int(radius),
                                      float(eps_gf), 1, _p(scratch), _st()))
    return out.cpu().numpy()


def apply_cco_dev(chi: torch.Tensor, params: CcoParams) -> torch.Tensor:
    """apply_cco on (..., m1, m2) complex128 device images."""
    if params.gf_radius < 1:
        raise ValueError("radius must be >= 1")
    chi = chi.to(device=_dev(), dtype=torch.complex128).contiguous()
    m1, m2 = chi.shape[-2:]
    count = chi.numel() // (m1 * m2)
    out = torch.empty_like(chi)
    scratch = torch.empty((count, 4, m1, m2), dtype=torch.float64, device=chi.device)
    N.check(N.lib().pdf_cco_image(_p(chi), _p(out), m1, m2, count, float(params.tau), float(params.eta_max),
                                  float(params.delta), int(params.gf_radius), float(params.gf_eps), _p(scratch),
                                  _st()))
    return out


def apply_cco(chi, params: CcoParams) -> np.ndarray:
    """(1 + eta) G(chi|chi) + eta chi, eta = eta_max sig((|chi| - tau) / delta),
    G the self-guided filter on Re and Im separately."""
    chi = np.asarray(chi, dtype=np.complex128)
    if chi.ndim != 2:
        raise ValueError("apply_cco expects a 2-D contrast image")
    return apply_cco_dev(torch.as_tensor(chi, device=_dev()), params).cpu().numpy()
