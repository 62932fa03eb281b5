"""CUDA path (libpdfb200.so through the C-ABI) vs the golden vectors and the
oracle.  Tolerances: the default product path computes in float64 /
complex128, so single-step results must agree with the reference to ~1e-10
relative (summation order only); trajectories within the north-star gate
(final relative contrast error within 1e-3 absolute) and in practice far
tighter."""
import numpy as np
import pytest
import torch

from conftest import Setup, cfg_baseline, golden, oracle_ops, rel

pytestmark = pytest.mark.gpu
LAM = (1e-3, 1e-5, 1e-5)


def _dev(setup, data, mask=None, r_fixed=None, S=1, dtype="f64"):
    from paper_2602_13805_b200.engine import DeviceProblem
    d = np.asarray(data)
    if d.ndim == 2 and S > 1:
        d = np.broadcast_to(d, (S,) + d.shape).copy()
    return DeviceProblem(setup.ops, setup.e_inc, d, mf=setup.cfg.m_f, beta=setup.cfg.beta, lambdas=LAM,
                         tau_b=setup.cfg.tau_b, mask=mask, r_fixed=r_fixed, dtype=dtype)


def _t(x, dev):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dev.cdt, device=dev.device)


# ------------------------------------------------------------------ primitives
def test_primitives_tiny(tiny_setup, g_tiny):
    g = g_tiny
    dev = _dev(tiny_setup, g["data"])
    x = _t(g["x"], dev)
    assert rel(dev.apply_gd(x).cpu().numpy(), g["gd_x"]) < 1e-12
    assert rel(dev.apply_gd(x, adjoint=True).cpu().numpy(), g["gdh_x"]) < 1e-12
    assert rel(dev.gs_adjoint(_t(g["rows"], dev)).cpu().numpy(), g["gsh_rows"]) < 1e-12
    assert rel(dev.expand(_t(g["alpha"], dev)).cpu().numpy(), g["exp_alpha"]) < 1e-12
    assert rel(dev.truncate(x).cpu().numpy(), g["trunc_x"]) < 1e-12


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_apply_gd_sizes(cfg_id):
    from oracle import pdf_oracle as O
    st = Setup(cfg_baseline(cfg_id), plane=True)
    ops = oracle_ops(st)
    rng = np.random.default_rng(cfg_id)
    M = st.cfg.m1
    x = rng.standard_normal((5, M, M)) + 1j * rng.standard_normal((5, M, M))
    dev = _dev(st, np.ones((st.cfg.n_tx, st.cfg.n_rx), complex))
    got = dev.apply_gd(_t(x, dev)).cpu().numpy()
    assert rel(got, O.apply_gd(ops, x)) < 1e-12
    got = dev.apply_gd(_t(x, dev), adjoint=True).cpu().numpy()
    assert rel(got, O.apply_gd_adj(ops, x)) < 1e-12
    rows = dev.gs_forward(_t(x, dev)).cpu().numpy()
    assert rel(rows, x.reshape(5, -1) @ ops.gs.T) < 1e-12


# ------------------------------------------------------------------ one step
@pytest.mark.parametrize("variant", ["plain", "frozen", "mask"])
def test_grad_alpha_tiny(tiny_setup, g_tiny, variant):
    g = g_tiny
    if variant == "plain":
        dev, want, bd = _dev(tiny_setup, g["data"]), g["g_alpha"], g["bd"]
    elif variant == "frozen":
        dev, want, bd = _dev(tiny_setup, g["data"], r_fixed=g["r0"]), g["g_frozen"], g["bd_frozen"]
    else:
        dev = _dev(tiny_setup, g["data"] * g["mask"], mask=g["mask"])
        want, bd = g["g_mask"], g["bd_mask"]
    ga, bdd = dev.loss_grad(_t(g["alpha"][None], dev))
    dev.check_errors()
    assert rel(ga[0].cpu().numpy(), want) < 1e-10
    np.testing.assert_allclose(bdd[0].cpu().numpy(), bd, rtol=1e-10)


@pytest.mark.parametrize("variant", ["plain", "frozen", "mask"])
def test_grad_alpha_tiny_batch_streaming_pixel_path(tiny_setup, g_tiny, variant):
    """40 copies of the tiny scene in one batch: enough image rows for the
    streaming per-pixel kernels (pdf_pixel_stream.cuh: view sums, closed-form
    state term / R-chain, one gradient pass) -- same goldens, same tolerance."""
    g, S = g_tiny, 40
    rep = lambda x: np.repeat(np.asarray(x)[None], S, axis=0)
    if variant == "plain":
        dev, want, bd = _dev(tiny_setup, rep(g["data"])), g["g_alpha"], g["bd"]
    elif variant == "frozen":
        dev, want, bd = _dev(tiny_setup, rep(g["data"]), r_fixed=rep(g["r0"])), g["g_frozen"], g["bd_frozen"]
    else:
        dev = _dev(tiny_setup, rep(g["data"] * g["mask"]), mask=rep(g["mask"]))
        want, bd = g["g_mask"], g["bd_mask"]
    ga, bdd = dev.loss_grad(_t(rep(g["alpha"]), dev))
    dev.check_errors()
    for i in (0, 17, 39):
        assert rel(ga[i].cpu().numpy(), want) < 1e-10
        np.testing.assert_allclose(bdd[i].cpu().numpy(), bd, rtol=1e-10)
    # loss-only entry (no gradient pass) and chi
    bd2, chi = dev.loss_value(_t(rep(g["alpha"]), dev), want_chi=True)
    np.testing.assert_allclose(bd2[39].cpu().numpy(), bd, rtol=1e-10)
    assert torch.equal(chi[0], chi[39])


def test_grad_alpha_cfg1(cfg1_setup, g_cfg1):
    g = g_cfg1
    dev = _dev(cfg1_setup, g["data"])
    ga, bd = dev.loss_grad(_t(g["alpha0"][None], dev))
    dev.check_errors()
    assert rel(ga[0].cpu().numpy(), g["g_alpha0"]) < 1e-10
    np.testing.assert_allclose(bd[0].cpu().numpy(), g["bd0"], rtol=1e-10)


def test_grad_alpha_cfg2_vs_oracle():
    from oracle import pdf_oracle as O
    g = golden("cfg2")
    st = Setup(cfg_baseline(2), plane=True)
    ctx = O.Context(g["data"], st.e_inc, oracle_ops(st), 8, 6.0, LAM, 0.5)
    rng = np.random.default_rng(3)
    alpha = g["alpha0"] * (1 + 0.1 * rng.standard_normal(g["alpha0"].shape))
    want, parts = O.grad_alpha(alpha, ctx)
    dev = _dev(st, g["data"])
    ga, bd = dev.loss_grad(_t(alpha[None], dev))
    dev.check_errors()
    assert rel(ga[0].cpu().numpy(), want) < 1e-10
    row = [parts[k] for k in ("state", "data", "bound", "tv", "bridge", "total")]
    np.testing.assert_allclose(bd[0].cpu().numpy(), row, rtol=1e-10)
    ga0, bd0 = dev.loss_grad(_t(g["alpha0"][None], dev))
    assert rel(ga0[0].cpu().numpy(), g["g_alpha0"]) < 1e-10
    np.testing.assert_allclose(bd0[0].cpu().numpy(), g["bd0"], rtol=1e-10)


# ------------------------------------------------------------------ network + Adam
def test_grad_loss_tiny(tiny_setup, g_tiny):
    g = g_tiny
    dev = _dev(tiny_setup, g["data"])
    dev.net_setup(_t(g["alpha0"][None], dev))
    theta = torch.as_tensor(g["net_flat"][None], dtype=torch.float64, device="cuda").contiguous()
    grad, bd = dev.grad_loss(theta)
    dev.check_errors()
    assert rel(grad[0].cpu().numpy(), g["grad_flat"]) < 1e-10
    np.testing.assert_allclose(bd[0].cpu().numpy(), g["bd_net"], rtol=1e-10)
    out = dev.net_forward(theta)
    assert rel((out[0].cpu().numpy() - g["alpha0"]), g["dalpha"]) < 1e-10


def test_grad_loss_cfg1(cfg1_setup, g_cfg1):
    from oracle import pdf_oracle as O
    g = g_cfg1
    dev = _dev(cfg1_setup, g["data"])
    dev.net_setup(_t(g["alpha0"][None], dev))
    flat = O.flat(O.init_net(100, np.random.default_rng(0)))
    flat = flat + 0.02 * np.random.default_rng(123).standard_normal(flat.size)
    theta = torch.as_tensor(flat[None], dtype=torch.float64, device="cuda").contiguous()
    grad, bd = dev.grad_loss(theta)
    dev.check_errors()
    gr = grad[0].cpu().numpy()
    assert rel(gr[g["grad_idx"]], g["grad_sub"]) < 1e-10
    assert abs(np.linalg.norm(gr) / g["grad_norms"][0] - 1) < 1e-10
    np.testing.assert_allclose(bd[0].cpu().numpy(), g["bd_net"], rtol=1e-10)


def test_adam_matches_reference(g_tiny):
    from paper_2602_13805_b200.api import _adam_device
    dev = _adam_device(1e-2)
    p = torch.as_tensor(g_tiny["adam_p0"], device="cuda").clone()
    m, v = torch.zeros_like(p), torch.zeros_like(p)
    for t, gr in enumerate(g_tiny["adam_grads"], start=1):
        dev.adam_step(p, m, v, torch.as_tensor(gr, device="cuda"), t)
    assert np.abs(p.cpu().numpy() - g_tiny["adam_p5"]).max() < 1e-14
    assert np.abs(m.cpu().numpy() - g_tiny["adam_m5"]).max() < 1e-14


# ------------------------------------------------------------------ trajectories
def test_reconstruct_tiny_matches_reference(g_tiny):
    """The reference's own reconstruct() (line sources), 30 iterations."""
    from paper_2602_13805_b200 import ScatteredData
    from paper_2602_13805_b200.api import reconstruct
    from paper_2602_13805_b200.geometry import ComplexGrid
    g = g_tiny
    cfg = __import__("conftest").cfg_tiny()
    res = reconstruct(cfg, ScatteredData(matrix=g["data"]), chi_true=ComplexGrid(g["chi_true"], 1.5 / 16))
    tr = np.array([b.as_row() for b in res.trace])
    np.testing.assert_allclose(tr, g["rec_trace"], rtol=1e-8)
    assert rel(res.chi_hat.values, g["rec_chi_hat"]) < 1e-8
    assert rel(res.chi_cco.values, g["rec_chi_cco"]) < 1e-8
    assert rel(res.chi0.values, g["rec_chi0"]) < 1e-10
    assert abs(res.rel_error - float(g["rec_rel"])) < 1e-8


@pytest.mark.parametrize("use_graph", [True, False])
def test_cfg1_trajectory(cfg1_setup, g_cfg1, use_graph):
    """BASELINE config 1, 200 iterations, plane waves: final rel_error gate 1e-3."""
    from paper_2602_13805_b200.api import BatchReconstructor
    g = g_cfg1
    rec = BatchReconstructor(cfg1_setup.cfg, 1, e_inc=cfg1_setup.e_inc, use_graph=use_graph)
    res = rec.run([g["data"]], seeds=[0], chi_trues=[g["chi_true"]])[0]
    assert rel(res.chi0.values, g["chi0"]) < 1e-10
    tot = np.array([b.total for b in res.trace])
    np.testing.assert_allclose(tot, g["trace"][:, 5], rtol=1e-6)
    assert abs(res.rel_error - float(g["rel_error"])) < 1e-3
    assert abs(res.rel_error - float(g["rel_error"])) < 1e-7


def test_batched_equals_single(cfg1_setup, g_cfg1):
    """S scenes in one launch == S separate single-scene runs.  Kernel shapes
    (and so float64 summation orders) are chosen per batch size, so the
    comparison is to 1e-9 relative; rerun determinism is bitwise (below)."""
    from paper_2602_13805_b200.api import BatchReconstructor
    g = g_cfg1
    rng = np.random.default_rng(0)
    datas = [g["data"] * (1 + 0.05 * rng.standard_normal(g["data"].shape)) for _ in range(3)]
    seeds = [0, 1, 2]
    rb = BatchReconstructor(cfg1_setup.cfg, 3, e_inc=cfg1_setup.e_inc)
    batch = rb.run(datas, seeds=seeds, k_iters=20)
    r1 = BatchReconstructor(cfg1_setup.cfg, 1, e_inc=cfg1_setup.e_inc)
    for s in range(3):
        one = r1.run([datas[s]], seeds=[seeds[s]], k_iters=20)[0]
        np.testing.assert_allclose(one.chi_cco.values, batch[s].chi_cco.values, rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose([b.total for b in one.trace], [b.total for b in batch[s].trace], rtol=1e-9)


def test_deterministic_rerun(cfg1_setup, g_cfg1):
    from paper_2602_13805_b200.api import BatchReconstructor
    rb = BatchReconstructor(cfg1_setup.cfg, 1, e_inc=cfg1_setup.e_inc)
    a = rb.run([g_cfg1["data"]], k_iters=25)[0]
    b = rb.run([g_cfg1["data"]], k_iters=25)[0]
    assert np.array_equal(a.chi_cco.values, b.chi_cco.values)


# ------------------------------------------------------------------ errors
def test_zero_data_rejected(tiny_setup):
    from paper_2602_13805_b200.errors import ZeroDataError
    with pytest.raises(ZeroDataError):
        _dev(tiny_setup, np.zeros((8, 8), complex))


def test_nonfinite_gradient_raises(tiny_setup, g_tiny):
    g = g_tiny
    dev = _dev(tiny_setup, g["data"])
    dev.net_setup(_t(g["alpha0"][None], dev))
    flat = g["net_flat"].copy()
    flat[0] = np.nan
    theta = torch.as_tensor(flat[None], device="cuda").contiguous()
    dev.grad_loss(theta)
    with pytest.raises(FloatingPointError):
        dev.check_errors()


def test_nonfinite_loss_terms_named(tiny_setup, g_tiny):
    g = g_tiny
    dev = _dev(tiny_setup, g["data"])
    alpha = g["alpha"].copy()
    alpha[0, 0] = np.inf
    dev.loss_grad(_t(alpha[None], dev))
    with pytest.raises(FloatingPointError, match="nonfinite loss term"):
        dev.check_errors()


def test_physics_loss_autograd_function():
    """PhysicsLoss: torch autograd through the fused physics reproduces the
    reference gradient, and chains into torch-side parameters (finite difference)."""
    from paper_2602_13805_b200.api import PhysicsLoss
    from paper_2602_13805_b200.engine import DeviceProblem
    from conftest import Setup, cfg_baseline
    g = golden("cfg2")
    st = Setup(cfg_baseline(2), plane=True)
    c = st.cfg
    dev = DeviceProblem(st.ops, st.e_inc, g["data"], mf=c.m_f, beta=c.beta, lambdas=(1e-3, 1e-5, 1e-5),
                        tau_b=c.tau_b)
    a = torch.as_tensor(g["alpha0"][None], device="cuda").clone().requires_grad_(True)
    loss = PhysicsLoss.apply(a, dev)
    loss.sum().backward()
    assert rel(a.grad[0].cpu().numpy(), g["g_alpha0"]) < 1e-10
    assert abs(loss.item() - float(g["bd0"][5])) < 1e-10 * abs(float(g["bd0"][5]))
    # chain rule into a torch-side real scale s: alpha_hat = alpha0 * (1 + s)
    a0 = torch.as_tensor(g["alpha0"][None], device="cuda")
    s = torch.zeros(1, dtype=torch.float64, device="cuda", requires_grad=True)
    PhysicsLoss.apply(a0 * (1 + s), dev).sum().backward()
    h = 1e-6
    lp = dev.loss_value(a0 * (1 + h))[0][0, 5].item()
    lm = dev.loss_value(a0 * (1 - h))[0][0, 5].item()
    fd = (lp - lm) / (2 * h)
    assert abs(s.grad.item() - fd) < 1e-6 * max(1.0, abs(fd)), (s.grad.item(), fd)


def test_module_level_operator_drop_ins(tiny_setup, g_tiny, cfg1_setup):
    """forward.apply_gd / apply_gd_adjoint / apply_gs_adjoint and
    spectral.truncate / expand as module-level functions (reference signatures,
    host arrays in and out), on the golden vectors and with extra leading dims."""
    from oracle import pdf_oracle as O
    from paper_2602_13805_b200 import (SpectralBasis, apply_gd, apply_gd_adjoint, apply_gs_adjoint, expand,
                                       truncate, truncate_adjoint_scale)
    g, ops, c = g_tiny, tiny_setup.ops, tiny_setup.cfg
    basis = SpectralBasis(c.m1, c.m2, c.m_f)
    assert rel(apply_gd(ops, g["x"]), g["gd_x"]) < 1e-12
    assert rel(apply_gd_adjoint(ops, g["x"]), g["gdh_x"]) < 1e-12
    assert rel(apply_gs_adjoint(ops, g["rows"]), g["gsh_rows"]) < 1e-12
    assert rel(expand(basis, g["alpha"]), g["exp_alpha"]) < 1e-12
    assert rel(truncate(basis, g["x"]), g["trunc_x"]) < 1e-12
    # (2, 3, m1, m2) leading dims, cfg1 sizes, against the oracle
    st = cfg1_setup
    oo = oracle_ops(st)
    M, mf = st.cfg.m1, st.cfg.m_f
    rng = np.random.default_rng(7)
    x = rng.standard_normal((2, 3, M, M)) + 1j * rng.standard_normal((2, 3, M, M))
    assert apply_gd(st.ops, x).shape == x.shape
    assert rel(apply_gd(st.ops, x), O.apply_gd(oo, x)) < 1e-12
    assert rel(apply_gd_adjoint(st.ops, x), O.apply_gd_adj(oo, x)) < 1e-12
    rows = rng.standard_normal((2, 3, st.cfg.n_rx)) + 0j
    assert rel(apply_gs_adjoint(st.ops, rows), O.apply_gs_adj(oo, rows)) < 1e-12
    b = SpectralBasis(M, M, mf)
    a = truncate(b, x)
    assert a.shape == (2, 3, b.m0) and rel(a, O.truncate(x, mf)) < 1e-12
    assert rel(truncate(b, expand(b, a)), a) < 1e-12
    # <expand(a), y> = c <a, truncate(y)>
    lhs = np.vdot(expand(b, a[0, 0]), x[1, 2])
    rhs = truncate_adjoint_scale(b) * np.vdot(a[0, 0], truncate(b, x[1, 2]))
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)
    with pytest.raises(ValueError):
        truncate(b, x[..., :-1])
    with pytest.raises(ValueError):
        expand(b, a[..., :-1])
    with pytest.raises(ValueError):
        apply_gd(st.ops, x[..., :-1, :])
