"""Reconstruction driver (reference reconstruct.py), GPU underneath:
reconstruct (the batched engine, pdf_train), bp_initialize / init_alpha
(library primitives), the exact-line-search objective CsiObjective, and the
metrics relative_error / count_components (pdf_relative_error,
pdf_count_components)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .api import (ReconstructionResult, SpectralBasis, _basis_device, _cdev, _ops_device,  # noqa: F401
                  bp_initialize, init_alpha, reconstruct)
from .cie import masked_residual_dev
from .metrics import count_components, relative_error  # noqa: F401
from .operators import GreensOperators, ScatteredData


@dataclass
class CsiObjective:
    """Data + state quadratic in the coefficients with the modified contrast
    frozen at r0 (reconstruct.py:74-136), evaluated on the GPU."""
    r0: np.ndarray
    e_inc: np.ndarray
    data: ScatteredData
    ops: GreensOperators
    basis: SpectralBasis
    beta: float
    c_inc: float = 0.0
    c_sca: float = 0.0

    def __post_init__(self):
        self._b = _basis_device(self.basis)
        self._o = _ops_device(self.ops)
        d = self._o
        self._r0 = torch.as_tensor(np.asarray(self.r0), dtype=torch.complex128, device=d.device)
        self._einc = torch.as_tensor(np.asarray(self.e_inc), dtype=torch.complex128, device=d.device)
        self._mat = torch.as_tensor(np.asarray(self.data.matrix), dtype=torch.complex128, device=d.device)
        self._mask = (None if self.data.mask is None else
                      torch.as_tensor(np.asarray(self.data.mask), dtype=torch.float64, device=d.device))
        mat = self._mat if self._mask is None else self._mat * self._mask
        self.c_sca = float(torch.sum((mat.conj() * mat).real).item())
        self.c_inc = float(torch.sum((self._einc.conj() * self._einc).real).item())

    def _dev_alpha(self, alpha):
        return torch.as_tensor(np.atleast_2d(np.asarray(alpha)), dtype=torch.complex128, device=self._r0.device)

    def _residuals(self, a: torch.Tensor):
        j = self._b.expand(a)
        sres = self._r0 * (self._einc + self._o.apply_gd(j)) + self.beta * (self._r0 - 1.0) * j
        rows = masked_residual_dev(self._o.gs_forward(j), self._mat, self._mask)
        return j, sres, rows

    @staticmethod
    def _pw(x):
        return float(torch.sum((x.conj() * x).real).item())

    def value_parts(self, alpha) -> tuple[float, float]:
        _, sres, rows = self._residuals(self._dev_alpha(alpha))
        return self._pw(sres) / self.c_inc, self._pw(rows) / self.c_sca

    def grad(self, alpha) -> np.ndarray:
        _, sres, rows = self._residuals(self._dev_alpha(alpha))
        gs_r = (2.0 / self.c_inc) * sres
        rc = self._r0.conj()
        g_j = self._o.apply_gd(rc * gs_r, adjoint=True) + self.beta * (rc - 1.0) * gs_r
        g_rows = (2.0 / self.c_sca) * rows
        if self._mask is not None:
            g_rows = g_rows * self._mask
        g_j = g_j + self._o.gs_adjoint(g_rows)
        return (self._b.truncate(g_j) / (self.basis.m1 * self.basis.m2)).cpu().numpy()

    def curvature(self, direction) -> float:
        """||A d||^2 in the normalised residual metric (homogeneous part)."""
        j = self._b.expand(self._dev_alpha(direction))
        s_lin = self._r0 * self._o.apply_gd(j) + self.beta * (self._r0 - 1.0) * j
        rows = self._o.gs_forward(j)
        if self._mask is not None:
            rows = rows * self._mask
        return self._pw(s_lin) / self.c_inc + self._pw(rows) / self.c_sca

    def exact_step(self, grad) -> float:
        """Minimiser of the objective along -grad."""
        q = self.curvature(grad)
        g = np.asarray(grad)
        gnorm2 = float(np.vdot(g, g).real)
        if q <= 0 or gnorm2 <= 0:
            return 0.0
        return gnorm2 / (2.0 * q)
