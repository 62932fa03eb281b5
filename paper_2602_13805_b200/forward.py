"""Forward model (reference forward.py), B200 forms of its public functions:

  build_greens / incident_fields   forward.py:101-137, 174-181 -> pdf_build_greens / pdf_incident_fields
  apply_gd(_adjoint), apply_gs_adjoint forward.py:140-151, 303-306 -> pdf_apply_gd / pdf_gs_adjoint
  dense_gd_matrix                  forward.py:154-171 (explicit operator, small grids; pdf_bessel)
  solve_total_field                forward.py:251-275 (dense LU up to 1024 cells, GPU BiCGStab above)
  synthesize_scattered, add_awgn, simulate, and the result / error types
"""
from __future__ import annotations

import numpy as np

from .api import apply_gd, apply_gd_adjoint, apply_gs_adjoint  # noqa: F401
from .geometry import GridGeometry
from .greens import bessel_j1, build_greens_gpu as build_greens, hankel1_0  # noqa: F401
from .greens import incident_fields_gpu as incident_fields  # noqa: F401
from .operators import (FieldSet, GeometryError, GreensOperators, NoConvergenceError, ScatteredData,  # noqa: F401
                        SimulationResult, SingularSystemError, add_awgn, plane_wave_fields, simulate,
                        solve_total_field, synthesize_scattered)


def dense_gd_matrix(ops: GreensOperators, grid: GridGeometry) -> np.ndarray:
    """Explicit (M, M) domain operator for small grids (tests, LU solves)."""
    m = grid.n_cells
    if m > 4096:
        raise ValueError("dense G_D limited to grids of at most 4096 cells")
    diff = grid.centers[:, None, :] - grid.centers[None, :, :]
    rho = np.hypot(diff[..., 0], diff[..., 1])
    a = grid.cell_size / np.sqrt(np.pi)
    w = 0.5j * np.pi * ops.k0 * a * float(bessel_j1(np.array([ops.k0 * a]))[0])
    off = rho > 0
    out = np.empty((m, m), dtype=np.complex128)
    out[off] = w * hankel1_0(ops.k0 * rho[off])
    np.fill_diagonal(out, ops.gd_diag)
    return out
