"""Cylinder functions (reference special.py:64-106) on the GPU (pdf_bessel):
J0, J1, Y0, Y1 and the first-kind Hankel functions H^(1)_0, H^(1)_1."""
from .greens import bessel_j0, bessel_j1, bessel_y0, bessel_y1, hankel1_0, hankel1_1  # noqa: F401
