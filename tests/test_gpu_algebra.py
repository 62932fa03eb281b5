"""Module-level CIE algebra, regularisers, filters and loss terms on the GPU
against vectors produced by the unmodified reference (tests/golden/algebra.npz,
make_golden.py:make_algebra), plus the behaviours the reference's own tests
check for them (tests/test_cie.py, test_filters.py, test_losses.py,
test_reconstruct.py).  Shapes are deliberately odd (40 x 40, 12 x 20, 7 x 9,
20 x 28): these entry points take any m1 x m2.

Tolerances: the elementwise maps (chi_to_r, r_to_chi) follow numpy's float64
operation order and match bit for bit; sums over views or
pixels differ by summation order only (1e-13); the transcendental terms
(hypot / exp inside TV and the bridge) 1e-12.
"""
import numpy as np
import pytest

from conftest import golden, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    return golden("algebra")


def test_chi_to_r_and_back(g):
    from paper_2602_13805_b200 import chi_to_r, r_to_chi
    chi = g["ctr_chi"]
    r = chi_to_r(chi, 6.0)
    assert r.shape == chi.shape and r.dtype == np.complex128
    # bit for bit: numpy's operation order (Smith division, FMA complex multiply)
    assert np.array_equal(r, g["ctr_r"])
    assert np.array_equal(r_to_chi(g["ctr_r"], 6.0), g["ctr_back"])
    assert np.array_equal(chi_to_r(chi, 6.0 + 1.5j), g["ctr_rc"])
    assert np.array_equal(r_to_chi(g["ctr_rc"], 6.0 + 1.5j), g["ctr_rc_back"])
    # reference tests/test_cie.py:15-33
    assert (np.abs(r_to_chi(r, 6.0) - chi) / (1.0 + np.abs(chi))).max() < 1e-13
    assert np.abs(r).max() < 1.0
    assert np.array_equal(chi_to_r(np.zeros(4), 6.0), np.zeros(4))
    from paper_2602_13805_b200 import PoleError
    with pytest.raises(PoleError):
        chi_to_r(np.array([-1.0 / 6.0]), 6.0)
    with pytest.raises(PoleError):
        r_to_chi(np.array([1.0]), 6.0)


def test_pixel_least_squares(g):
    from paper_2602_13805_b200 import default_eps_reg, pixel_least_squares
    rec = pixel_least_squares(g["pls_j"], g["pls_e"])
    assert abs(rec.eps_reg - float(g["pls_eps"])) <= 1e-14 * float(g["pls_eps"])
    assert abs(default_eps_reg(g["pls_e"]) - float(g["pls_eps_default"])) <= 1e-14 * float(g["pls_eps_default"])
    assert rel(rec.numerator, g["pls_num"]) < 1e-14
    assert rel(rec.denominator, g["pls_den"]) < 1e-14
    assert rel(rec.chi, g["pls_chi"]) < 1e-14
    assert np.array_equal(rec.degenerate, g["pls_deg"]) and rec.degenerate[2, 7]
    assert rec.chi[2, 7] == 0.0
    rec2 = pixel_least_squares(g["pls_j"], g["pls_e"], eps_reg=0.25)
    assert rel(rec2.chi, g["pls2_chi"]) < 1e-14 and rec2.eps_reg == 0.25
    assert np.array_equal(rec2.degenerate, g["pls2_deg"])
    # consistent contrast is recovered (reference tests/test_cie.py:36-44)
    rng = np.random.default_rng(1)
    chi = (rng.uniform(0, 9, 64) + 1j * rng.uniform(0, 2, 64)).reshape(8, 8)
    e = rng.standard_normal((5, 8, 8)) + 1j * rng.standard_normal((5, 8, 8))
    r = pixel_least_squares(chi[None] * e, e)
    assert np.abs(r.chi - chi).max() < 1e-8 and not r.degenerate.any() and r.eps_reg > 0


def test_regularisers(g):
    from paper_2602_13805_b200 import losses as L
    c = g["reg_chi"]
    assert abs(L.loss_bound(c) - float(g["reg_bound"])) <= 1e-13 * float(g["reg_bound"])
    assert abs(L.loss_tv(c) - float(g["reg_tv"])) <= 1e-12 * float(g["reg_tv"])
    assert abs(L.loss_bridge(c, 0.5) - float(g["reg_bridge"])) <= 1e-12 * float(g["reg_bridge"])
    assert rel(L.bound_chi_grad(c), g["reg_gb"]) < 1e-15
    assert rel(L.tv_chi_grad(c), g["reg_gt"]) < 1e-12
    assert rel(L.bridge_chi_grad(c, 0.5), g["reg_gr"]) < 1e-12
    assert rel(L.regularizer_chi_grad(c, (1e-3, 1e-5, 1e-5), 0.5), g["reg_g"]) < 1e-12
    assert rel(L.regularizer_chi_grad(c, (0, 1, 0), 0.5), g["reg_g_l2"]) < 1e-12
    assert np.array_equal(L.regularizer_chi_grad(c, (0, 0, 0), 0.5), np.zeros_like(c))


def test_regulariser_gradients_match_finite_differences():
    """Central differences of each term along Re and Im of random pixels
    (reference tests/test_losses.py:77-103)."""
    from paper_2602_13805_b200 import losses as L
    rng = np.random.default_rng(9)
    c = rng.standard_normal((9, 11)) + 1j * rng.standard_normal((9, 11))
    terms = [(L.loss_bound, L.bound_chi_grad), (L.loss_tv, L.tv_chi_grad),
             (lambda x: L.loss_bridge(x, 0.5), lambda x: L.bridge_chi_grad(x, 0.5))]
    h = 1e-6
    for f, gf in terms:
        gr = gf(c)
        for (y, x) in [(0, 0), (4, 5), (8, 10), (3, 9)]:
            for d, part in ((1.0, "re"), (1j, "im")):
                cp, cm = c.copy(), c.copy()
                cp[y, x] += h * d
                cm[y, x] -= h * d
                fd = (f(cp) - f(cm)) / (2 * h)
                an = gr[y, x].real if part == "re" else gr[y, x].imag
                assert abs(fd - an) < 1e-6 * max(1.0, abs(an)), (f, y, x, part, fd, an)


def test_box_mean_and_guided_filter(g):
    from paper_2602_13805_b200 import box_mean, guided_filter
    for k in range(4):
        out = box_mean(g[f"box{k}_img"], int(g[f"box{k}_r"]))
        assert np.abs(out - g[f"box{k}_out"]).max() < 1e-13
    assert np.abs(box_mean(np.full((9, 9), 3.5), 3) - 3.5).max() < 1e-12
    with pytest.raises(ValueError):
        box_mean(np.zeros((4, 4)), 0)
    with pytest.raises(ValueError):
        box_mean(np.zeros(16), 1)
    assert np.abs(guided_filter(g["gf_inp"], g["gf_guide"], 2, 1e-3) - g["gf_out"]).max() < 1e-12
    with pytest.raises(ValueError):
        guided_filter(np.zeros((4, 4)), np.zeros((4, 5)), 2, 1e-3)
    # large eps: a -> 0, output -> box mean applied twice (reference tests/test_filters.py:48-55)
    img = np.random.default_rng(3).standard_normal((12, 12))
    assert np.abs(guided_filter(img, img, 2, 1e9) - box_mean(box_mean(img, 2), 2)).max() < 1e-6


def test_apply_cco_any_shape(g):
    from paper_2602_13805_b200 import CcoParams, apply_cco
    p = CcoParams(tau=3.0, eta_max=0.1, delta=0.5, gf_radius=2, gf_eps=1e-3)
    assert rel(apply_cco(g["cco_small"], p), g["cco_small_out"]) < 1e-13
    plateau = np.zeros((16, 16), dtype=complex)
    plateau[4:12, 4:12] = 7.0
    out = apply_cco(plateau, p)
    assert rel(out, g["cco_plateau_out"]) < 1e-13
    assert np.all(out[7:9, 7:9].real > 7.0 * 1.15) and np.all(out[7:9, 7:9].real < 7.0 * 1.2 + 1e-6)
    assert rel(apply_cco(g["cco_big"], CcoParams()), g["cco_big_out"]) < 1e-13
    z = apply_cco(np.zeros((8, 8), dtype=complex), CcoParams())
    assert z.shape == (8, 8) and z.dtype == np.complex128 and np.abs(z).max() == 0.0


def _tiny():
    from conftest import Setup, cfg_tiny
    from paper_2602_13805_b200 import SpectralBasis
    st = Setup(cfg_tiny(), plane=False)
    return st, SpectralBasis(16, 16, 3)


def test_state_and_data_terms(g):
    from paper_2602_13805_b200 import ScatteredData, cie_state_residual
    from paper_2602_13805_b200 import losses as L
    st, basis = _tiny()
    res = cie_state_residual(g["st_alpha"], g["st_rhat"], st.e_inc, st.ops, basis, 6.0)
    assert rel(res, g["st_res"]) < 1e-12
    ls = L.loss_state(g["st_alpha"], g["st_rhat"], st.e_inc, st.ops, basis, 6.0)
    assert abs(ls - float(g["st_loss"])) <= 1e-12 * float(g["st_loss"])
    mat, mask = g["dt_mat"], g["dt_mask"]
    ld = L.loss_data(g["st_alpha"], ScatteredData(matrix=mat * mask, mask=mask), st.ops, basis)
    assert abs(ld - float(g["dt_loss"])) <= 1e-12 * float(g["dt_loss"])
    ld = L.loss_data(g["st_alpha"], ScatteredData(matrix=mat), st.ops, basis)
    assert abs(ld - float(g["dt_loss_plain"])) <= 1e-12 * float(g["dt_loss_plain"])
    with pytest.raises(L.ZeroDataError):
        L.loss_data(g["st_alpha"], ScatteredData(matrix=np.zeros_like(mat)), st.ops, basis)


def test_csi_objective_reproduces_init_alpha(g_tiny):
    """One exact line-search step from zero with CsiObjective equals the
    reference's init_alpha output (reconstruct.py:139-153); the step is the
    exact minimiser along -g, so the objective decreases."""
    from paper_2602_13805_b200 import CsiObjective, ScatteredData
    st, basis = _tiny()
    obj = CsiObjective(r0=g_tiny["r0"], e_inc=st.e_inc, data=ScatteredData(matrix=g_tiny["data"]), ops=st.ops,
                       basis=basis, beta=6.0)
    zero = np.zeros((8, basis.m0), dtype=np.complex128)
    gz = obj.grad(zero)
    t = obj.exact_step(gz)
    assert rel(-t * gz, g_tiny["alpha0"]) < 1e-12
    v0 = sum(obj.value_parts(zero))
    v1 = sum(obj.value_parts(-t * gz))
    vp = sum(obj.value_parts(-1.1 * t * gz))
    assert v1 < v0 and v1 < vp
