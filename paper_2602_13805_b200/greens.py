"""Operator construction on the GPU.

Drop-ins for the reference's one-time setup, computed by libpdfb200.so
(csrc/pdf_greens.cu):

  bessel_j0 / j1 / y0 / y1, hankel1_0 / 1   special.py:64-106      -> pdf_bessel
  build_greens                              forward.py:101-137     -> pdf_build_greens
  incident_fields (unit line sources)       forward.py:174-181     -> pdf_incident_fields(kind 0)
  plane-wave incident fields                         -> pdf_incident_fields(kind 1)

The *_device forms keep the results in HBM (torch CUDA tensors) for the
reconstruction engine; the *_gpu forms return host numpy arrays with the
reference's types (GreensOperators, FieldSet).
"""
from __future__ import annotations

import ctypes as ct
import math

import numpy as np
import torch

from . import _native as N
from .config import ImagingConfig
from .geometry import AntennaArray, GridGeometry
from .operators import FieldSet, GeometryError, GreensOperators


def _st():
    return ct.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t: torch.Tensor):
    return ct.c_void_p(t.data_ptr())


def _need_gpu():
    if not torch.cuda.is_available():
        raise RuntimeError("the operator build runs on the GPU (no CPU fallback)")
    return torch.device("cuda")


def _check(rc: int) -> None:
    if rc == N.PDF_EGEOMETRY:
        raise GeometryError(N.lib().pdf_last_error().decode())
    N.check(rc)


def _coords(grid: GridGeometry, dev):
    xs = np.ascontiguousarray(grid.centers[: grid.m2, 0])
    ys = np.ascontiguousarray(grid.centers[:: grid.m2, 1])
    return torch.as_tensor(xs, device=dev), torch.as_tensor(ys, device=dev)


# ---------------------------------------------------------------------------- special functions
def _bessel(order: int, x):
    dev = _need_gpu()
    xa = np.asarray(x, dtype=np.float64)
    xt = torch.as_tensor(np.ascontiguousarray(xa.ravel()), device=dev)
    j, y = torch.empty_like(xt), torch.empty_like(xt)
    N.check(N.lib().pdf_bessel(order, _p(xt), _p(j), _p(y), xt.numel(), _st()))
    return j.cpu().numpy().reshape(xa.shape), y.cpu().numpy().reshape(xa.shape)


def bessel_j0(x):
    return _bessel(0, x)[0]


def bessel_j1(x):
    return _bessel(1, x)[0]


def bessel_y0(x):
    if (np.asarray(x) < 0).any():
        raise ValueError("bessel_y0 requires x >= 0")
    return _bessel(0, x)[1]


def bessel_y1(x):
    if (np.asarray(x) < 0).any():
        raise ValueError("bessel_y1 requires x >= 0")
    return _bessel(1, x)[1]


def hankel1_0(x):
    if (np.asarray(x) < 0).any():
        raise ValueError("hankel1_0 requires x >= 0")
    j, y = _bessel(0, x)
    return j + 1j * y


def hankel1_1(x):
    if (np.asarray(x) < 0).any():
        raise ValueError("hankel1_1 requires x >= 0")
    j, y = _bessel(1, x)
    return j + 1j * y


# ---------------------------------------------------------------------------- operators
def build_greens_device(config: ImagingConfig, array: AntennaArray, grid: GridGeometry) -> GreensOperators:
    """GreensOperators whose arrays are complex128 CUDA tensors (kernel, fft2, G_S)."""
    config.validate()
    dev = _need_gpu()
    m1, m2, R = grid.m1, grid.m2, array.n_rx
    xs, ys = _coords(grid, dev)
    rx = torch.as_tensor(np.ascontiguousarray(array.rx_positions, dtype=np.float64), device=dev)
    ker = torch.empty((2 * m1, 2 * m2), dtype=torch.complex128, device=dev)
    hat = torch.empty_like(ker)
    gs = torch.empty((R, m1 * m2), dtype=torch.complex128, device=dev)
    diag = (ct.c_double * 2)()
    _check(N.lib().pdf_build_greens(float(config.wavenumber), float(grid.cell_size), m1, m2, _p(xs), _p(ys), _p(rx), R,
                                    _p(ker), _p(hat), _p(gs), diag, _st()))
    return GreensOperators(gd_kernel=ker, gd_kernel_hat=hat, gd_diag=complex(diag[0], diag[1]), gs_matrix=gs,
                           k0=float(config.wavenumber), m1=m1, m2=m2, cell_size=float(grid.cell_size))


def build_greens_gpu(config: ImagingConfig, array: AntennaArray, grid: GridGeometry) -> GreensOperators:
    """build_greens (forward.py:101-137) computed on the GPU, host arrays returned."""
    o = build_greens_device(config, array, grid)
    return GreensOperators(gd_kernel=o.gd_kernel.cpu().numpy(), gd_kernel_hat=o.gd_kernel_hat.cpu().numpy(),
                           gd_diag=o.gd_diag, gs_matrix=o.gs_matrix.cpu().numpy(), k0=o.k0, m1=o.m1, m2=o.m2,
                           cell_size=o.cell_size)


def incident_fields_device(config: ImagingConfig, array: AntennaArray | None, grid: GridGeometry,
                           kind: str = "line", n: int | None = None) -> torch.Tensor:
    """(n, m1, m2) complex128 CUDA tensor: unit line sources at the transmitters
    (kind 'line', forward.py:174-181) or plane waves at angles 2 pi k / n ('plane')."""
    config.validate()
    dev = _need_gpu()
    xs, ys = _coords(grid, dev)
    if kind == "line":
        src = np.ascontiguousarray(array.tx_positions, dtype=np.float64)
        k = 0
    elif kind == "plane":
        nn = config.n_tx if n is None else n
        src = 2.0 * math.pi * np.arange(nn) / nn
        k = 1
    else:
        raise ValueError(f"unknown incidence {kind!r}")
    nv = src.shape[0]
    st = torch.as_tensor(src, device=dev)
    out = torch.empty((nv, grid.m1, grid.m2), dtype=torch.complex128, device=dev)
    _check(N.lib().pdf_incident_fields(k, float(config.wavenumber), grid.m1, grid.m2, _p(xs), _p(ys), _p(st), nv,
                                       _p(out), _st()))
    return out


def incident_fields_gpu(config: ImagingConfig, array: AntennaArray, grid: GridGeometry) -> FieldSet:
    return FieldSet(views=incident_fields_device(config, array, grid, "line").cpu().numpy(), role="incident")


def plane_wave_fields_gpu(config: ImagingConfig, grid: GridGeometry, n: int | None = None) -> FieldSet:
    return FieldSet(views=incident_fields_device(config, None, grid, "plane", n).cpu().numpy(), role="incident")
