"""Pin the CPU oracle (oracle/pdf_oracle.py) against golden vectors produced by
the unmodified reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import oracle_ops, rel
from oracle import pdf_oracle as O

LAM = (1e-3, 1e-5, 1e-5)


def _ctx(setup, g, mask=None, r_fixed=None, data=None):
    return O.Context(g["data"] if data is None else data, setup.e_inc, oracle_ops(setup), setup.cfg.m_f,
                     setup.cfg.beta, LAM, setup.cfg.tau_b, mask=mask, r_fixed=r_fixed)


def test_operators_match_reference(tiny_setup, g_tiny):
    ops = oracle_ops(tiny_setup)
    assert rel(ops.k_hat, g_tiny["khat"]) < 1e-13
    assert rel(ops.gs, g_tiny["gs"]) < 1e-13
    e = O.line_source_fields(tiny_setup.cfg.wavenumber, tiny_setup.array.tx_positions, 1.5, 16, 16)
    assert rel(e, g_tiny["e_inc"]) < 1e-14


def test_primitives(tiny_setup, g_tiny):
    ops = oracle_ops(tiny_setup)
    assert rel(O.apply_gd(ops, g_tiny["x"]), g_tiny["gd_x"]) < 1e-13
    assert rel(O.apply_gd_adj(ops, g_tiny["x"]), g_tiny["gdh_x"]) < 1e-13
    assert rel(O.apply_gs_adj(ops, g_tiny["rows"]), g_tiny["gsh_rows"]) < 1e-13
    assert rel(O.expand(g_tiny["alpha"], 16, 16, 3), g_tiny["exp_alpha"]) < 1e-14
    assert rel(O.truncate(g_tiny["x"], 3), g_tiny["trunc_x"]) < 1e-14


@pytest.mark.parametrize("variant", ["plain", "frozen", "mask"])
def test_grad_alpha(tiny_setup, g_tiny, variant):
    g = g_tiny
    if variant == "plain":
        ctx, want, bd = _ctx(tiny_setup, g), g["g_alpha"], g["bd"]
    elif variant == "frozen":
        ctx, want, bd = _ctx(tiny_setup, g, r_fixed=g["r0"]), g["g_frozen"], g["bd_frozen"]
    else:
        ctx = _ctx(tiny_setup, g, mask=g["mask"], data=g["data"] * g["mask"])
        want, bd = g["g_mask"], g["bd_mask"]
    got, parts = O.grad_alpha(g["alpha"], ctx)
    assert rel(got, want) < 1e-12
    row = [parts[k] for k in ("state", "data", "bound", "tv", "bridge", "total")]
    np.testing.assert_allclose(row, bd, rtol=1e-12)


def test_init_and_network(tiny_setup, g_tiny):
    g = g_tiny
    ops = oracle_ops(tiny_setup)
    chi0, r0 = O.bp_initialize(g["data"], tiny_setup.e_inc, ops, 6.0)
    assert rel(chi0, g["chi0"]) < 1e-12
    a0 = O.init_alpha(r0, g["data"], tiny_setup.e_inc, ops, 3, 6.0)
    assert rel(a0, g["alpha0"]) < 1e-12
    like = O.init_net(36, np.random.default_rng(6))
    params = O.unflat(g["net_flat"], like)
    grad, _ = O.grad_loss(params, g["alpha0"], _ctx(tiny_setup, g))
    assert rel(grad, g["grad_flat"]) < 1e-12
    assert rel(O.delta_alpha(params, g["alpha0"]), g["dalpha"]) < 1e-12


def test_adam_sequence(g_tiny):
    x = g_tiny["adam_p0"].copy()
    st = O.Adam(m=np.zeros_like(x), v=np.zeros_like(x), lr=1e-2)
    for gr in g_tiny["adam_grads"]:
        x = O.adam_update(st, x, gr)
    assert np.abs(x - g_tiny["adam_p5"]).max() < 1e-14


def test_reconstruct_trajectory_tiny(tiny_setup, g_tiny):
    """30 iterations of the reference's own reconstruct() (line sources)."""
    g = g_tiny
    out = O.reconstruct_loop(_ctx(tiny_setup, g), g["alpha0"], 30, seed=0)
    tr = np.array([[p[k] for k in ("state", "data", "bound", "tv", "bridge", "total")] for p in out["trace"]])
    np.testing.assert_allclose(tr, g["rec_trace"], rtol=1e-9)
    assert rel(out["chi_cco"], g["rec_chi_cco"]) < 1e-9
    r = O.relative_error(out["chi_cco"].real + 1, g["chi_true"].real + 1)
    assert abs(r - float(g["rec_rel"])) < 1e-10


def test_cfg1_step_and_trajectory(cfg1_setup, g_cfg1):
    """BASELINE config 1 (plane waves): one step and the full 200-iteration run."""
    g = g_cfg1
    ops = oracle_ops(cfg1_setup)
    assert rel(ops.k_hat, g["khat"]) < 1e-13 and rel(ops.gs, g["gs"]) < 1e-13
    ctx = O.Context(g["data"], cfg1_setup.e_inc, ops, 5, 6.0, LAM, 0.5)
    chi0, r0 = O.bp_initialize(g["data"], cfg1_setup.e_inc, ops, 6.0)
    a0 = O.init_alpha(r0, g["data"], cfg1_setup.e_inc, ops, 5, 6.0)
    assert rel(a0, g["alpha0"]) < 1e-11
    ga, parts = O.grad_alpha(g["alpha0"], ctx)
    assert rel(ga, g["g_alpha0"]) < 1e-11
    out = O.reconstruct_loop(ctx, g["alpha0"], 200, seed=0)
    tot = np.array([p["total"] for p in out["trace"]])
    np.testing.assert_allclose(tot, g["trace"][:, 5], rtol=1e-7)
    r = O.relative_error(out["chi_cco"].real + 1, g["chi_true"].real + 1)
    assert abs(r - float(g["rel_error"])) < 1e-8


# ------------------------------------------------------------------ edge cases the reference's tests pin
@pytest.fixture(scope="module")
def g_edges():
    from conftest import golden
    return golden("edges")


def _pole_ctx(setup, g):
    from dataclasses import replace
    ops0 = replace(oracle_ops(setup), k_hat=np.zeros((32, 32), complex))
    return O.Context(g["data1"], np.ones((1, 16, 16), complex), ops0, 3, 6.0, LAM, 0.5)


def test_edges_pole(tiny_setup, g_edges):
    """cie.py:24-30 (tests/test_cie.py:29): beta chi + 1 = 0 at a pixel raises."""
    ctx = _pole_ctx(tiny_setup, g_edges)
    with pytest.raises(O.OraclePoleError):
        O.grad_alpha(g_edges["alpha_pole"], ctx)
    got, parts = O.grad_alpha(g_edges["alpha_near"], ctx)
    assert rel(got, g_edges["g_near"]) < 1e-12


def test_edges_state_zero_and_masked_data(tiny_setup, g_tiny, g_edges):
    """tests/test_losses.py:128-133 (state = 0 at R = 0) and :105-119 (masked data = 1 at alpha = 0)."""
    g = g_edges
    zero = np.zeros((8, 36), complex)
    got, parts = O.grad_alpha(zero, _ctx(tiny_setup, g_tiny, r_fixed=np.zeros((16, 16), complex)))
    assert parts["state"] == 0.0 and g["bd_r0"][0] == 0.0
    assert rel(got, g["g_r0"]) < 1e-12
    got, parts = O.grad_alpha(zero, _ctx(tiny_setup, g_tiny, mask=g["mask"]))
    assert parts["data"] == pytest.approx(1.0, rel=1e-14) and g["bd_mk0"][1] == pytest.approx(1.0, rel=1e-14)
    assert rel(got, g["g_mk0"]) < 1e-12


def test_edges_whitening_floor_and_zero_rms(tiny_setup, g_tiny, g_edges):
    """network.py:88-104 (tests/test_network.py:63-70): a dead mode hits the floor; rms 0 gives unit scales."""
    g = g_edges
    like = O.init_net(36, np.random.default_rng(5))
    params = O.unflat(g["net_flat"], like)
    ctx = _ctx(tiny_setup, g_tiny)
    for a, da, gr in (("alpha_dead", "dalpha_dead", "grad_dead"), ("alpha_zero", None, "grad_zero")):
        alpha = g[a] if a in g else np.zeros((8, 36), complex)
        want_da = g[da] if da else g["dalpha_zero"]
        assert rel(O.delta_alpha(params, alpha), want_da) < 1e-12
        grad, _ = O.grad_loss(params, alpha, ctx)
        assert rel(grad, g[gr]) < 1e-12


def test_metrics_match_reference():
    """relative_error / count_components (reconstruct.py:243-254) against the reference's outputs."""
    from conftest import golden
    g = golden("metrics")
    thr = float(g["thr"])
    for k, want in enumerate(g["counts"]):
        assert O.count_components(g[f"img{k}"] + 1.0, thr) == want, k
    for k, want in enumerate(g["extra_counts"]):
        assert O.count_components(g[f"extra{k}"] + 1.0, thr) == want, k
    for k, want in enumerate(g["rels"]):
        assert abs(O.relative_error(g["rel_a"][k].real + 1.0, g["rel_b"][k].real + 1.0) - want) < 1e-15


# ------------------------------------------------------------------ regularisers and filters (losses.py:115-196,
# filters.py:16-67) on odd shapes, golden algebra.npz
def test_oracle_regularisers_and_filters_match_reference():
    from conftest import golden
    g = golden("algebra")
    c = g["reg_chi"]
    b, t, r = O.reg_values(c, 0.5)
    assert abs(b - g["reg_bound"]) <= 1e-14 * abs(g["reg_bound"])
    assert abs(t - g["reg_tv"]) <= 1e-13 * abs(g["reg_tv"])
    assert abs(r - g["reg_bridge"]) <= 1e-13 * abs(g["reg_bridge"])
    assert rel(O.reg_grad(c, (1e-3, 1e-5, 1e-5), 0.5), g["reg_g"]) < 1e-13
    assert rel(O.reg_grad(c, (0, 1, 0), 0.5), g["reg_gt"]) < 1e-13
    assert rel(O.reg_grad(c, (0, 0, 1), 0.5), g["reg_gr"]) < 1e-13
    for k in range(4):
        assert rel(O.box_mean(g[f"box{k}_img"], int(g[f"box{k}_r"])), g[f"box{k}_out"]) < 1e-14
    assert rel(O.guided(g["gf_inp"], g["gf_guide"], 2, 1e-3), g["gf_out"]) < 1e-13
    assert rel(O.cco(g["cco_small"]), g["cco_small_out"]) < 1e-13
    assert rel(O.cco(g["cco_big"]), g["cco_big_out"]) < 1e-13
