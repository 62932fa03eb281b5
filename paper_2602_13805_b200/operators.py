"""Operator construction and the fixture forward model (host, one-time setup).

Out of the per-iteration hot path (SURVEY 2.1 marks these one-time): the
Green's operators are assembled once per geometry in float64 (host scipy here,
or on the GPU by greens.build_greens_gpu) and uploaded; synthetic
measurements come from a method-of-moments solve (dense LU on the host up to
1024 cells, the library's batched BiCGStab on the GPU above, as the
reference's 'auto' choice).

Physics follows the reference exactly (forward.py:1-374): time convention
exp(-i w t), first-kind Hankel H0^(1), equal-area-disk cell quadrature
(radius a = h / sqrt(pi)), off-diagonal (i pi k0 a/2) J1(k0 a) H0(k0 rho),
self term (i pi k0 a/2) H1(k0 a) - 1, wrap-indexed (2 m1, 2 m2) kernel with
row m1 / column m2 zeroed.  Bessel functions come from scipy.special here (the
reference's own Chebyshev fits agree with it to ~1e-15; the operators are
pinned against the reference's golden K^ / G_S in tests/test_oracle.py and
tests/test_host.py).
"""
from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, replace as dc_replace

import numpy as np
import scipy.special as sps

from .config import ImagingConfig
from .geometry import AntennaArray, ComplexGrid, GridGeometry, build_array, build_grid
from .scenes import Scene, rasterize


class GeometryError(ValueError):
    pass


class NoConvergenceError(RuntimeError):
    pass


class SingularSystemError(RuntimeError):
    """Unrecoverable Krylov breakdown (forward.py:35-36).  Declared for import
    compatibility: like the reference's BiCGStab, the GPU solver restarts on
    breakdown and reports NoConvergenceError at the iteration cap instead."""


@dataclass
class FieldSet:
    views: np.ndarray
    role: str
    residuals: np.ndarray | None = None

    @property
    def n_views(self) -> int:
        return self.views.shape[0]


@dataclass
class ScatteredData:
    matrix: np.ndarray
    snr_db: float | None = None
    mask: np.ndarray | None = None


@dataclass(frozen=True)
class GreensOperators:
    gd_kernel: np.ndarray
    gd_kernel_hat: np.ndarray
    gd_diag: complex
    gs_matrix: np.ndarray
    k0: float
    m1: int
    m2: int
    cell_size: float

    @property
    def n_cells(self) -> int:
        return self.m1 * self.m2

    @property
    def n_rx(self) -> int:
        return self.gs_matrix.shape[0]


def _cell_weights(k0: float, h: float) -> tuple[complex, complex]:
    a = h / math.sqrt(math.pi)
    pref = 0.5j * math.pi * k0 * a
    return complex(pref * sps.jv(1, k0 * a)), complex(pref * sps.hankel1(1, k0 * a) - 1.0)


def build_greens(config: ImagingConfig, array: AntennaArray, grid: GridGeometry) -> GreensOperators:
    config.validate()
    k0, h = config.wavenumber, grid.cell_size
    m1, m2 = grid.m1, grid.m2
    w_off, diag = _cell_weights(k0, h)
    # signed displacement of every doubled-grid index (circular convolution)
    si = np.fft.fftfreq(2 * m1, d=1.0 / (2 * m1))
    sj = np.fft.fftfreq(2 * m2, d=1.0 / (2 * m2))
    rho = h * np.hypot(si[:, None], sj[None, :])
    ker = np.where(rho > 0, w_off * sps.hankel1(0, k0 * np.where(rho > 0, rho, 1.0)), 0.0)
    ker = ker.astype(np.complex128)
    ker[0, 0] = diag
    ker[m1, :] = 0.0
    ker[:, m2] = 0.0
    drx = np.hypot(array.rx_positions[:, None, 0] - grid.centers[None, :, 0],
                   array.rx_positions[:, None, 1] - grid.centers[None, :, 1])
    if np.any(drx < h / 2.0):
        raise GeometryError("a receiver lies inside the pixel grid")
    gs = w_off * sps.hankel1(0, k0 * drx)
    return GreensOperators(gd_kernel=ker, gd_kernel_hat=np.fft.fft2(ker), gd_diag=diag, gs_matrix=gs,
                           k0=k0, m1=m1, m2=m2, cell_size=h)


def incident_fields(config: ImagingConfig, array: AntennaArray, grid: GridGeometry) -> FieldSet:
    """Unit line sources (i/4) H0^(1)(k0 |r - r_tx|) (reference forward.py:174-181)."""
    d = np.hypot(array.tx_positions[:, None, 0] - grid.centers[None, :, 0],
                 array.tx_positions[:, None, 1] - grid.centers[None, :, 1])
    if np.any(d <= 0):
        raise GeometryError("a transmitter coincides with a cell center")
    v = 0.25j * sps.hankel1(0, config.wavenumber * d)
    return FieldSet(views=v.reshape(array.n_tx, grid.m1, grid.m2), role="incident")


def plane_wave_fields(config: ImagingConfig, grid: GridGeometry, n: int | None = None) -> FieldSet:
    """Unit plane waves exp(i k0 (x cos phi + y sin phi)), phi = 2 pi k / n.

    The BASELINE configs use plane-wave incidence; the reference's loss path
    takes any e_inc array (losses.py:57), so this is a drop-in composition."""
    n = config.n_tx if n is None else n
    phi = 2.0 * np.pi * np.arange(n) / n
    x, y = grid.centers[:, 0], grid.centers[:, 1]
    v = np.exp(1j * config.wavenumber * (np.cos(phi)[:, None] * x[None, :] + np.sin(phi)[:, None] * y[None, :]))
    return FieldSet(views=v.reshape(n, grid.m1, grid.m2), role="incident")


def apply_gd_host(ops: GreensOperators, x: np.ndarray) -> np.ndarray:
    """Host FFT application of G_D (fixture synthesis only)."""
    m1, m2 = ops.m1, ops.m2
    y = np.fft.ifft2(np.fft.fft2(x, s=(2 * m1, 2 * m2)) * ops.gd_kernel_hat)
    return y[..., :m1, :m2]


def solve_total_field(chi: ComplexGrid, e_inc: FieldSet, ops: GreensOperators, tol: float = 1e-8,
                      maxiter: int = 2000, method: str = "auto") -> FieldSet:
    """E = E_inc + G_D (chi E) for every view (reference forward.py:251-275).

    method 'dense' LU-solves the explicit operator on the host (small grids),
    'fft' runs the batched BiCGStab on the GPU (raises NoConvergenceError),
    'auto' picks dense up to 1024 cells, as the reference does."""
    c = chi.values
    b = e_inc.views
    if c.shape != b.shape[-2:]:
        raise ValueError("contrast grid and incident views disagree in shape")
    if method == "auto":
        method = "dense" if c.size <= 1024 else "fft"
    if method == "dense":
        m = c.size
        # dense G_D from the displacement kernel (Toeplitz gather)
        ii, jj = np.divmod(np.arange(m), ops.m2)
        di = (ii[:, None] - ii[None, :]) % (2 * ops.m1)
        dj = (jj[:, None] - jj[None, :]) % (2 * ops.m2)
        G = ops.gd_kernel[di, dj]
        x = np.linalg.solve(np.eye(m) - G * c.ravel()[None, :], b.reshape(-1, m).T).T.reshape(b.shape)
        num = x - b - apply_gd_host(ops, c * x)
        nb = np.sqrt(np.sum(np.abs(b) ** 2, axis=(1, 2)))
        res = np.sqrt(np.sum(np.abs(num) ** 2, axis=(1, 2))) / np.where(nb > 0, nb, 1.0)
    elif method == "fft":
        # batched BiCGStab on the GPU (solver.py, csrc/pdf_solver.cu; forward.py:193-248)
        from .solver import solve_fields_gpu
        xd, rd, _ = solve_fields_gpu(c, b, ops, tol=tol, maxiter=maxiter)
        x, res = xd[0].cpu().numpy(), rd[0].cpu().numpy()
    else:
        raise ValueError(f"unknown method {method!r}")
    return FieldSet(views=x, role="total", residuals=res)


def synthesize_scattered(chi: ComplexGrid, e_tot: FieldSet, ops: GreensOperators) -> ScatteredData:
    j = (chi.values * e_tot.views).reshape(e_tot.n_views, -1)
    return ScatteredData(matrix=j @ ops.gs_matrix.T)


def add_awgn(data: ScatteredData, snr_db: float, rng: np.random.Generator) -> ScatteredData:
    """Circular AWGN at the stated total SNR (reference forward.py:309-322)."""
    if np.isinf(snr_db):
        return ScatteredData(matrix=data.matrix.copy(), snr_db=float("inf"), mask=data.mask)
    p = float(np.vdot(data.matrix, data.matrix).real)
    sd = math.sqrt(p / (data.matrix.size * 10.0 ** (snr_db / 10.0)) / 2.0)
    noise = rng.normal(0.0, sd, data.matrix.shape) + 1j * rng.normal(0.0, sd, data.matrix.shape)
    return ScatteredData(matrix=data.matrix + noise, snr_db=snr_db, mask=data.mask)


@dataclass
class SimulationResult:
    data: ScatteredData
    chi_true: ComplexGrid


def simulate(config: ImagingConfig, scene: Scene, snr_db: float = float("inf"),
             rng: np.random.Generator | None = None, array: AntennaArray | None = None,
             incidence: str = "line") -> SimulationResult:
    """Rasterise, solve, measure, add noise (reference forward.py:335-374).

    ``incidence='plane'`` synthesises with plane waves (BASELINE configs)."""
    config.validate()
    rng = np.random.default_rng(config.rng_seed) if rng is None else rng
    array = build_array(config) if array is None else array
    grid = build_grid(config)
    chi_true = rasterize(scene, grid)
    cfg, g, chi_sim = config, grid, chi_true
    if config.fine_forward:
        cfg = dc_replace(config, m1=2 * config.m1, m2=2 * config.m2, ring_radius=config.radius,
                         fine_forward=False)
        g = build_grid(cfg)
        chi_sim = rasterize(scene, g)
    ops = build_greens(cfg, array, g)
    e_inc = plane_wave_fields(cfg, g) if incidence == "plane" else incident_fields(cfg, array, g)
    e_tot = solve_total_field(chi_sim, e_inc, ops, tol=cfg.solver_tol, maxiter=cfg.solver_maxiter,
                              method="fft" if chi_sim.values.size > 1024 else "dense")
    data = synthesize_scattered(chi_sim, e_tot, ops)
    if float(e_tot.residuals.max()) > cfg.solver_tol * 10:
        warnings.warn(f"forward residual {float(e_tot.residuals.max()):.2e} above tolerance")
    return SimulationResult(data=add_awgn(data, snr_db, rng), chi_true=chi_true)
