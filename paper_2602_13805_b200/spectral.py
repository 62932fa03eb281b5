"""Truncated Fourier basis of the induced currents (reference spectral.py):
SpectralBasis, and truncate / expand / truncate_adjoint_scale on the GPU
(pdf_truncate, pdf_expand)."""
from .api import SpectralBasis, expand, truncate, truncate_adjoint_scale  # noqa: F401
