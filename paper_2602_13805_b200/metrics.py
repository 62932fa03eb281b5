"""Reconstruction metrics on the GPU (reference reconstruct.py:243-254).

    relative_error(eps_hat, eps_true)      ||Re eps_hat - Re eps_true||_F / ||Re eps_true||_F
    count_components(eps_map, threshold)   4-connected components of {Re eps > threshold}

Both run in libpdfb200.so (pdf_relative_error: one fixed-order reduction per
image; pdf_count_components: union-find labelling, integer root count, equal
to scipy.ndimage.label's count).  The *_dev forms take device tensors of
shape (..., m1, m2), float64 or complex128, and return one value per image;
`offset` is added to every real part (eps = chi + 1 from contrast images).
"""
from __future__ import annotations

import ctypes as ct

import numpy as np
import torch

from . import _native as N


def _real_view(x: torch.Tensor):
    if x.dtype == torch.complex128:
        return torch.view_as_real(x.contiguous()), 2
    if x.dtype == torch.float64:
        return x.contiguous(), 1
    raise TypeError(f"metrics need float64 or complex128 images, got {x.dtype}")


def _st():
    return ct.c_void_p(torch.cuda.current_stream().cuda_stream)


def relative_error_dev(eps_hat: torch.Tensor, eps_true: torch.Tensor, offset: float = 0.0) -> torch.Tensor:
    if eps_hat.shape != eps_true.shape or eps_hat.dim() < 2:
        raise ValueError(f"image shapes differ: {tuple(eps_hat.shape)} vs {tuple(eps_true.shape)}")
    a, sa = _real_view(eps_hat)
    b, sb = _real_view(eps_true)
    if sa != sb:     # one complex, one real: compare real parts of like layouts
        a = a[..., 0].contiguous() if sa == 2 else a
        b = b[..., 0].contiguous() if sb == 2 else b
        sa = sb = 1
    m1, m2 = eps_hat.shape[-2:]
    count = int(np.prod(eps_hat.shape[:-2], dtype=np.int64)) if eps_hat.dim() > 2 else 1
    out = torch.empty(count, dtype=torch.float64, device=eps_hat.device)
    N.check(N.lib().pdf_relative_error(ct.c_void_p(a.data_ptr()), ct.c_void_p(b.data_ptr()), sa, m1 * m2, count,
                                       float(offset), ct.c_void_p(out.data_ptr()), _st()))
    return out


def count_components_dev(eps_map: torch.Tensor, threshold: float, offset: float = 0.0) -> torch.Tensor:
    if eps_map.dim() < 2:
        raise ValueError("count_components needs a 2-D image (or a stack of them)")
    x, s = _real_view(eps_map)
    m1, m2 = eps_map.shape[-2:]
    count = int(np.prod(eps_map.shape[:-2], dtype=np.int64)) if eps_map.dim() > 2 else 1
    labels = torch.empty(count * m1 * m2, dtype=torch.int32, device=eps_map.device)
    out = torch.empty(count, dtype=torch.int32, device=eps_map.device)
    N.check(N.lib().pdf_count_components(ct.c_void_p(x.data_ptr()), s, m1, m2, count, float(offset),
                                         float(threshold), ct.c_void_p(labels.data_ptr()),
                                         ct.c_void_p(out.data_ptr()), _st()))
    return out


def _dev_image(x) -> torch.Tensor:
    x = np.asarray(x)
    if not torch.cuda.is_available():
        raise RuntimeError("the metrics run on the GPU (no CPU fallback)")
    dt = np.complex128 if np.iscomplexobj(x) else np.float64
    return torch.as_tensor(np.ascontiguousarray(x, dtype=dt), device="cuda")


def relative_error(eps_hat, eps_true) -> float:
    """Frobenius-norm relative error between real permittivity maps (reconstruct.py:243-247)."""
    a, b = np.asarray(eps_hat), np.asarray(eps_true)
    if a.shape != b.shape or a.ndim != 2:
        raise ValueError(f"need two images of one shape, got {a.shape} and {b.shape}")
    return float(relative_error_dev(_dev_image(a), _dev_image(b))[0].item())


def count_components(eps_map, threshold: float) -> int:
    """4-connected components of {Re(eps) > threshold} (reconstruct.py:250-254)."""
    x = np.asarray(eps_map)
    if x.ndim != 2:
        raise ValueError(f"need a 2-D image, got shape {x.shape}")
    return int(count_components_dev(_dev_image(x), threshold)[0].item())
