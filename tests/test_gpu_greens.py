"""Operator construction on the GPU (csrc/pdf_greens.cu, greens.py; SURVEY
8(f) rank 4) against the reference's own outputs: its Chebyshev cylinder
functions (special.py:64-106, golden `special`), build_greens K^ / G_S
(forward.py:101-137, goldens `tiny`, `cfg1`, `cfg5` checksums) and
incident_fields (forward.py:174-181)."""
import numpy as np
import pytest

from conftest import Setup, cfg_baseline, cfg_tiny, golden, rel

pytestmark = pytest.mark.gpu


def test_cylinder_functions_match_reference():
    from paper_2602_13805_b200 import greens as G
    g = golden("special")
    x = g["x"]
    for name, f in (("j0", G.bessel_j0), ("j1", G.bessel_j1), ("y0", G.bessel_y0), ("y1", G.bessel_y1)):
        got = f(x)
        err = np.abs(got - g[name]) / np.maximum(1.0, np.abs(g[name]))
        assert err.max() < 1e-14, (name, float(err.max()), float(x[np.argmax(err)]))   # both ~1e-15 from exact
    np.testing.assert_allclose(G.bessel_j0(g["xneg"]), g["j0neg"], rtol=0, atol=5e-15)
    np.testing.assert_allclose(G.bessel_j1(g["xneg"]), g["j1neg"], rtol=0, atol=5e-15)
    h = G.hankel1_0(x[:100])
    np.testing.assert_allclose(h.real, g["j0"][:100], atol=5e-15)
    with pytest.raises(ValueError):
        G.bessel_y0(np.array([-1.0]))


def test_build_greens_tiny_matches_reference(tiny_setup, g_tiny):
    from paper_2602_13805_b200.greens import build_greens_gpu, incident_fields_gpu
    s = tiny_setup
    ops = build_greens_gpu(s.cfg, s.array, s.grid)
    assert rel(ops.gd_kernel_hat, g_tiny["khat"]) < 1e-13
    assert rel(ops.gs_matrix, g_tiny["gs"]) < 1e-13
    assert abs(ops.gd_diag - s.ops.gd_diag) < 1e-14 * abs(s.ops.gd_diag)
    assert rel(ops.gd_kernel, s.ops.gd_kernel) < 1e-13
    assert rel(incident_fields_gpu(s.cfg, s.array, s.grid).views, g_tiny["e_inc"]) < 1e-13


def test_build_greens_cfg1_and_cfg5(g_cfg1):
    from paper_2602_13805_b200.greens import build_greens_device, incident_fields_device
    st = Setup(cfg_baseline(1), plane=True)
    o = build_greens_device(st.cfg, st.array, st.grid)
    assert rel(o.gd_kernel_hat.cpu().numpy(), g_cfg1["khat"]) < 1e-13
    assert rel(o.gs_matrix.cpu().numpy(), g_cfg1["gs"]) < 1e-13
    assert rel(incident_fields_device(st.cfg, None, st.grid, "plane").cpu().numpy(), st.e_inc) < 1e-14
    g5 = golden("cfg5")
    st5 = Setup(cfg_baseline(5), plane=True)
    o5 = build_greens_device(st5.cfg, st5.array, st5.grid)
    kh, gs = o5.gd_kernel_hat.cpu().numpy(), o5.gs_matrix.cpu().numpy()
    np.testing.assert_allclose([kh.sum(), np.abs(kh).sum()], g5["khat_checksum"], rtol=1e-12)
    np.testing.assert_allclose([gs.sum(), np.abs(gs).sum()], g5["gs_checksum"], rtol=1e-12)
    assert rel(kh, st5.ops.gd_kernel_hat) < 1e-13 and rel(gs, st5.ops.gs_matrix) < 1e-13


def test_geometry_errors():
    from paper_2602_13805_b200 import GeometryError
    from paper_2602_13805_b200.geometry import AntennaArray, build_array, build_grid
    from paper_2602_13805_b200.greens import build_greens_gpu, incident_fields_gpu
    cfg = cfg_tiny()
    grid, arr = build_grid(cfg), build_array(cfg)
    inside = AntennaArray(arr.tx_positions, np.vstack([arr.rx_positions[:-1], grid.centers[5][None]]))
    with pytest.raises(GeometryError):
        build_greens_gpu(cfg, inside, grid)
    on_centre = AntennaArray(np.vstack([arr.tx_positions[:-1], grid.centers[7][None]]), arr.rx_positions)
    with pytest.raises(GeometryError):
        incident_fields_gpu(cfg, on_centre, grid)


def test_reconstruct_on_device_built_operators(g_tiny):
    """The engine runs on operators and incident fields that never left HBM."""
    from paper_2602_13805_b200.api import BatchReconstructor
    from paper_2602_13805_b200.greens import incident_fields_device
    cfg = cfg_tiny()
    ref = BatchReconstructor(cfg, 1).run([g_tiny["data"]], chi_trues=[g_tiny["chi_true"]])[0]
    dev = BatchReconstructor(cfg, 1, device_ops=True).run([g_tiny["data"]], chi_trues=[g_tiny["chi_true"]])[0]
    np.testing.assert_allclose([b.total for b in dev.trace], [b.total for b in ref.trace], rtol=1e-9)
    assert abs(dev.rel_error - float(g_tiny["rec_rel"])) < 1e-8
    assert incident_fields_device(cfg, BatchReconstructor(cfg, 1).array, BatchReconstructor(cfg, 1).grid).is_cuda
