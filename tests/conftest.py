"""Shared fixtures.  `gpu`-marked tests need a CUDA device; everything else
runs on CPU (oracle vs golden vectors, setup-code parity, ABI load checks)."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def golden(name: str):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name}.npz not generated")
    return dict(np.load(path))


@pytest.fixture(scope="session")
def g_tiny():
    return golden("tiny")


@pytest.fixture(scope="session")
def g_cfg1():
    return golden("cfg1")


# -------------------------------------------------------------- problem specs
def cfg_tiny():
    from paper_2602_13805_b200.config import ImagingConfig
    return ImagingConfig(m1=16, m2=16, m_f=3, n_tx=8, n_rx=8, k_iters=30).validate()


def cfg_baseline(i: int):
    """BASELINE.json configs 1-5 (SURVEY 8(d) mapping: m_f 5/8/8/8, lambda = 1 m)."""
    from paper_2602_13805_b200.config import C0, ImagingConfig
    if i == 1:
        return ImagingConfig(frequency=C0, doi_side=2.0, m1=32, m2=32, n_tx=16, n_rx=32, ring_radius=3.0,
                             m_f=5, k_iters=200, rng_seed=0).validate()
    if i in (2, 4):
        return ImagingConfig(frequency=C0, doi_side=2.0, m1=64, m2=64, n_tx=16, n_rx=32, ring_radius=3.0,
                             m_f=8, k_iters=500, rng_seed=1 if i == 2 else 0).validate()
    if i == 3:
        return ImagingConfig(frequency=C0, doi_side=2.0, m1=64, m2=64, n_tx=36, n_rx=36, ring_radius=3.0,
                             m_f=8, k_iters=500, rng_seed=2).validate()
    if i == 5:
        return ImagingConfig(frequency=C0, doi_side=4.0, m1=256, m2=256, n_tx=72, n_rx=72, ring_radius=5.0,
                             m_f=16, k_iters=300, rng_seed=3).validate()
    raise ValueError(i)


class Setup:
    """Package-side geometry/operators/incident fields for a config."""

    def __init__(self, cfg, plane: bool):
        from paper_2602_13805_b200 import (build_array, build_grid, build_greens, incident_fields,
                                           plane_wave_fields)
        self.cfg = cfg
        self.grid = build_grid(cfg)
        self.array = build_array(cfg)
        self.ops = build_greens(cfg, self.array, self.grid)
        fs = plane_wave_fields(cfg, self.grid) if plane else incident_fields(cfg, self.array, self.grid)
        self.e_inc = fs.views


@pytest.fixture(scope="session")
def tiny_setup():
    return Setup(cfg_tiny(), plane=False)


@pytest.fixture(scope="session")
def cfg1_setup():
    return Setup(cfg_baseline(1), plane=True)


def oracle_ops(setup):
    from oracle import pdf_oracle as O
    return O.build_operators(setup.cfg.wavenumber, setup.cfg.doi_side, setup.cfg.m1, setup.cfg.m2,
                             setup.array.rx_positions)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(np.asarray(b).ravel()), 1e-300))
