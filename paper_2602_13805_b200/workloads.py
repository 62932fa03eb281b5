"""BASELINE.json workloads: configs, seeded synthetic scenes, data synthesis.

Synthetic inputs stand in for the paper's scenes (BASELINE.json configs):
plane-wave incidences, lambda = 1 m (frequency = C0), m_f mapped from the
"N x N modes" wording as m_f = (N+1)/2.  Measurements are
synthesised by a method-of-moments solve of E = E_inc + G_D(chi E) -- the
library's batched BiCGStab on the GPU (pdf_solve_total_field) -- then G_S(chi E) plus circular
AWGN drawn with numpy's generator exactly as the reference's add_awgn.
Fixture synthesis is out of the timed hot path.
"""
from __future__ import annotations

import math

import numpy as np

from .config import C0, ImagingConfig
from .geometry import build_array, build_grid
from .operators import build_greens, plane_wave_fields
from .scenes import Scene, Shape, ellipse, rasterize

SNR_5PCT = 20.0 * math.log10(100.0 / 5.0)
SNR_10PCT = 20.0


def baseline_config(i: int, k_iters: int | None = None) -> ImagingConfig:
    base = dict(frequency=C0, doi_side=2.0, ring_radius=3.0)
    if i == 1:
        c = ImagingConfig(m1=32, m2=32, n_tx=16, n_rx=32, m_f=5, k_iters=200, rng_seed=0, **base)
    elif i == 2:
        c = ImagingConfig(m1=64, m2=64, n_tx=16, n_rx=32, m_f=8, k_iters=500, rng_seed=1, **base)
    elif i == 3:
        c = ImagingConfig(m1=64, m2=64, n_tx=36, n_rx=36, m_f=8, k_iters=500, rng_seed=2, **base)
    elif i == 4:
        c = ImagingConfig(m1=64, m2=64, n_tx=16, n_rx=32, m_f=8, k_iters=500, rng_seed=0, **base)
    elif i == 5:
        c = ImagingConfig(frequency=C0, doi_side=4.0, ring_radius=5.0, m1=256, m2=256, n_tx=72, n_rx=72, m_f=16,
                          k_iters=300, rng_seed=3)
    else:
        raise ValueError(f"no BASELINE config {i}")
    if k_iters is not None:
        from dataclasses import replace
        c = replace(c, k_iters=k_iters)
    return c.validate()


def cfg4_scene(idx: int) -> tuple[Scene, np.random.Generator]:
    """1-4 non-overlapping random ellipses (256-vertex polygons), semi-axes
    U[0.15, 0.5], centre inside the domain, rotation U[0, pi), chi U[0.5, 3];
    rng = default_rng(idx), which then also draws the AWGN."""
    rng = np.random.default_rng(idx)
    k = int(rng.integers(1, 5))
    shapes, placed, tries = [], [], 0
    while len(shapes) < k and tries < 200:
        tries += 1
        a, b = rng.uniform(0.15, 0.5, 2)
        r = max(a, b)
        cx, cy = rng.uniform(-1.0 + r, 1.0 - r, 2)
        ang = rng.uniform(0.0, np.pi)
        if any(math.hypot(cx - px, cy - py) < r + pr for px, py, pr in placed):
            continue
        chi = rng.uniform(0.5, 3.0)
        placed.append((cx, cy, r))
        shapes.append(ellipse((cx, cy), a, b, ang, 1.0 + chi))
    return Scene(tuple(shapes)), rng


def cfg5_scene(seed: int = 3) -> tuple[Scene, np.random.Generator]:
    """BASELINE config 5: 6 non-overlapping random ellipses on [-2, 2], semi-axes
    U[0.2, 0.6], chi = U[0.5, 2.5] + i U[0, 0.5]; rng = default_rng(3), which
    then also draws the AWGN (same draw order as tests/golden/make_golden.py)."""
    rng = np.random.default_rng(seed)
    shapes, placed, tries = [], [], 0
    while len(shapes) < 6 and tries < 1000:
        tries += 1
        a, b = rng.uniform(0.2, 0.6, 2)
        r = max(a, b)
        cx, cy = rng.uniform(-2.0 + r, 2.0 - r, 2)
        ang = rng.uniform(0.0, np.pi)
        if any(math.hypot(cx - px, cy - py) < r + pr for px, py, pr in placed):
            continue
        chi = rng.uniform(0.5, 2.5) + 1j * rng.uniform(0.0, 0.5)
        placed.append((cx, cy, r))
        shapes.append(ellipse((cx, cy), a, b, ang, 1.0 + chi))
    return Scene(tuple(shapes)), rng


def baseline_scene(i: int, idx: int = 0) -> tuple[Scene, np.random.Generator, float]:
    """(scene, noise rng, snr_db) of BASELINE config i (scene idx for config 4)."""
    if i == 1:
        return Scene((Shape(kind="disk", eps_r=2.0, center=(0.0, 0.0), radius=0.4),)), np.random.default_rng(0), SNR_5PCT
    if i == 2:
        return Scene((Shape(kind="disk", eps_r=3.0, center=(-0.35, 0.0), radius=0.3),
                      Shape(kind="disk", eps_r=3.0, center=(0.35, 0.0), radius=0.3))), np.random.default_rng(1), SNR_5PCT
    if i == 3:
        return Scene((Shape(kind="annulus", eps_r=4.0 + 0.5j, center=(0.0, 0.0), r_inner=0.3, r_outer=0.5),
                      Shape(kind="disk", eps_r=2.5, center=(0.6, 0.6), radius=0.15))), np.random.default_rng(2), SNR_10PCT
    if i == 4:
        s, rng = cfg4_scene(idx)
        return s, rng, SNR_5PCT
    if i == 5:
        s, rng = cfg5_scene(3)
        return s, rng, SNR_5PCT
    raise ValueError(i)


def awgn(mat: np.ndarray, snr_db: float, rng: np.random.Generator) -> np.ndarray:
    p = float(np.vdot(mat, mat).real)
    sd = math.sqrt(p / (mat.size * 10.0 ** (snr_db / 10.0)) / 2.0)
    return mat + (rng.normal(0.0, sd, mat.shape) + 1j * rng.normal(0.0, sd, mat.shape))


def synthesize_gpu(config: ImagingConfig, scenes, rngs, snr_db: float, tol: float = 1e-8, maxiter: int = 2000):
    """Plane-wave measurements for S scenes sharing one geometry, on the GPU.

    Returns (data (S, n, R) complex128 host, chi_true (S, M, M) host)."""
    import torch
    from .engine import DeviceProblem
    grid, arr = build_grid(config), build_array(config)
    ops = build_greens(config, arr, grid)
    e_inc = plane_wave_fields(config, grid).views
    S, n = len(scenes), e_inc.shape[0]
    chis = np.stack([rasterize(s, grid).values for s in scenes])
    from .solver import solve_fields_gpu
    x, _, _ = solve_fields_gpu(chis, e_inc, ops, tol=tol, maxiter=maxiter)    # batched BiCGStab (pdf_solver.cu)
    dev = DeviceProblem(ops, e_inc, np.ones((S, n, arr.n_rx), complex), mf=1, beta=config.beta,
                        lambdas=(0, 0, 0), tau_b=0.5)
    chi = torch.as_tensor(chis, device=dev.device)[:, None]
    rows = dev.gs_forward((chi * x).contiguous()).cpu().numpy()
    data = np.stack([awgn(rows[s], snr_db, rngs[s]) for s in range(S)])
    return data, chis
