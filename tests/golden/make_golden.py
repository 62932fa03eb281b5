"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [tiny cfg1 cfg2 cfg3 cfg4]

Every array below comes from `pdfisp` itself (/root/reference/pkg/src), in
float64 / complex128.  Plane-wave configs compose the reference's public
functions in the order of reconstruct.py:194-236 with a plane-wave e_inc,
exactly as SURVEY 8(c) prescribes.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from pdfisp.config import C0, ImagingConfig  # noqa: E402
from pdfisp.forward import (FieldSet, ScatteredData, add_awgn, apply_gd, apply_gd_adjoint,  # noqa: E402
                            apply_gs_adjoint, build_greens, incident_fields, simulate,
                            solve_total_field, synthesize_scattered)
from pdfisp.filters import apply_cco  # noqa: E402
from pdfisp.geometry import build_array, build_grid  # noqa: E402
from pdfisp.losses import LossContext, grad_alpha  # noqa: E402
from pdfisp import network  # noqa: E402
from pdfisp.reconstruct import bp_initialize, init_alpha, reconstruct, relative_error  # noqa: E402
from pdfisp.cie import recover_contrast  # noqa: E402
from pdfisp.scenes import Scene, Shape, builtin_scene, rasterize  # noqa: E402
from pdfisp.spectral import SpectralBasis, expand, truncate  # noqa: E402
from pdfisp.losses import loss_total  # noqa: E402


def plane_views(cfg, grid):
    phi = 2.0 * np.pi * np.arange(cfg.n_tx) / cfg.n_tx
    x, y = grid.centers[:, 0], grid.centers[:, 1]
    v = np.exp(1j * cfg.wavenumber * (np.cos(phi)[:, None] * x + np.sin(phi)[:, None] * y))
    return v.reshape(cfg.n_tx, cfg.m1, cfg.m2)


def ellipse_poly(cx, cy, a, b, ang, eps, nv=256):
    t = 2.0 * np.pi * np.arange(nv) / nv
    ca, sa = np.cos(ang), np.sin(ang)
    xs, ys = a * np.cos(t), b * np.sin(t)
    return Shape(kind="polygon", eps_r=eps,
                 vertices=tuple((float(cx + ca * u - sa * w), float(cy + sa * u + ca * w)) for u, w in zip(xs, ys)))


def cfg4_scene(idx: int):
    """1-4 non-overlapping ellipses, semi-axes U[0.15,0.5], chi U[0.5,3] (BASELINE cfg4)."""
    rng = np.random.default_rng(idx)
    k = int(rng.integers(1, 5))
    shapes, placed = [], []
    tries = 0
    while len(shapes) < k and tries < 200:
        tries += 1
        a, b = rng.uniform(0.15, 0.5, 2)
        cx, cy = rng.uniform(-1.0 + max(a, b), 1.0 - max(a, b), 2)
        ang = rng.uniform(0.0, np.pi)
        r = max(a, b)
        if any(np.hypot(cx - px, cy - py) < r + pr for px, py, pr in placed):
            continue
        chi = rng.uniform(0.5, 3.0)
        placed.append((cx, cy, r))
        shapes.append(ellipse_poly(cx, cy, a, b, ang, 1.0 + chi))
    return Scene(tuple(shapes)), rng


def cfg5_scene(seed: int = 3):
    """6 non-overlapping ellipses on [-2,2], semi-axes U[0.2,0.6], chi = U[0.5,2.5] + i U[0,0.5] (BASELINE cfg5)."""
    rng = np.random.default_rng(seed)
    shapes, placed, tries = [], [], 0
    while len(shapes) < 6 and tries < 1000:
        tries += 1
        a, b = rng.uniform(0.2, 0.6, 2)
        r = max(a, b)
        cx, cy = rng.uniform(-2.0 + r, 2.0 - r, 2)
        ang = rng.uniform(0.0, np.pi)
        if any(np.hypot(cx - px, cy - py) < r + pr for px, py, pr in placed):
            continue
        chi = rng.uniform(0.5, 2.5) + 1j * rng.uniform(0.0, 0.5)
        placed.append((cx, cy, r))
        shapes.append(ellipse_poly(cx, cy, a, b, ang, 1.0 + chi))
    return Scene(tuple(shapes)), rng


def plane_problem(cfg, scene, snr_db, rng):
    grid, arr = build_grid(cfg), build_array(cfg)
    ops = build_greens(cfg, arr, grid)
    views = plane_views(cfg, grid)
    chi = rasterize(scene, grid)
    e_tot = solve_total_field(chi, FieldSet(views, "incident"), ops,
                              method="dense" if chi.values.size <= 1024 else "fft")
    data = add_awgn(synthesize_scattered(chi, e_tot, ops), snr_db, rng)
    return grid, arr, ops, views, chi, data


def composed_reconstruct(cfg, data, views, ops, chi_true, k):
    """reconstruct.py:194-236 with plane-wave e_inc."""
    basis = SpectralBasis(cfg.m1, cfg.m2, cfg.m_f)
    fs = FieldSet(views, "incident")
    chi0, r0 = bp_initialize(data, fs, ops, cfg.beta)
    alpha0 = init_alpha(r0, data, fs, ops, basis, cfg.beta)
    net = network.init_network(basis.m0, np.random.default_rng(cfg.rng_seed))
    adam = network.AdamState.for_params(net, lr=cfg.learn_rate)
    ctx = LossContext(data=data, e_inc=views, ops=ops, basis=basis, beta=cfg.beta,
                      lambdas=(cfg.lambda1, cfg.lambda2, cfg.lambda3), tau_b=cfg.tau_b)
    trace = []
    for _ in range(k):
        g, bd = network.grad_loss(net, alpha0, ctx)
        trace.append(bd.as_row())
        net, adam = network.adam_step(adam, net, g)
    ahat = alpha0 + network.forward_net(net, alpha0)
    final = loss_total(ahat, ctx).as_row()
    chi_hat = recover_contrast(ahat, views, ops, basis)
    chi_cco = apply_cco(chi_hat, cfg.cco)
    rel = relative_error(chi_cco.real + 1.0, chi_true.values.real + 1.0)
    return dict(chi0=chi0, r0=r0, alpha0=alpha0, trace=np.array(trace), final=np.array(final),
                chi_hat=chi_hat, chi_cco=chi_cco, rel_error=rel, ctx=ctx)


def save(name, **arrs):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrs)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)", flush=True)


def make_tiny():
    """reference tests/conftest.py:43-57 setup: 16x16, m_f=3, 8 tx / 8 rx, austria eps 2."""
    cfg = ImagingConfig(m1=16, m2=16, m_f=3, n_tx=8, n_rx=8, k_iters=30).validate()
    grid, arr = build_grid(cfg), build_array(cfg)
    ops = build_greens(cfg, arr, grid)
    einc = incident_fields(cfg, arr, grid)
    basis = SpectralBasis(16, 16, 3)
    sim = simulate(cfg, builtin_scene("austria", 2.0, scale=0.9))
    ctx = LossContext(data=sim.data, e_inc=einc.views, ops=ops, basis=basis, beta=6.0,
                      lambdas=(1e-3, 1e-5, 1e-5), tau_b=0.5)
    rng = np.random.default_rng(7)
    n, m0 = 8, basis.m0
    alpha = 0.1 * (rng.standard_normal((n, m0)) + 1j * rng.standard_normal((n, m0)))
    g, bd = grad_alpha(alpha, ctx)
    chi0, r0 = bp_initialize(sim.data, einc, ops, 6.0)
    alpha0 = init_alpha(r0, sim.data, einc, ops, basis, 6.0)
    g0, bd0 = grad_alpha(alpha0, ctx)
    ctx_fr = LossContext(data=sim.data, e_inc=einc.views, ops=ops, basis=basis, beta=6.0,
                         lambdas=(1e-3, 1e-5, 1e-5), tau_b=0.5, r_fixed=r0)
    g_fr, bd_fr = grad_alpha(alpha, ctx_fr)
    mask = (np.random.default_rng(11).random((n, 8)) > 0.3).astype(float)
    dmask = ScatteredData(matrix=sim.data.matrix * mask, mask=mask)
    ctx_mk = LossContext(data=dmask, e_inc=einc.views, ops=ops, basis=basis, beta=6.0,
                         lambdas=(1e-3, 1e-5, 1e-5), tau_b=0.5)
    g_mk, bd_mk = grad_alpha(alpha, ctx_mk)
    # network gradient at perturbed parameters (reference tests/test_network.py:73-94)
    net = network.init_network(m0, np.random.default_rng(6))
    flat = network.flatten_params(net)
    flat = flat + 0.05 * np.random.default_rng(6).standard_normal(flat.size)
    net = network.unflatten_params(flat, net)
    gflat, bdn = network.grad_loss(net, alpha0, ctx)
    dalpha = network.forward_net(net, alpha0)
    # Adam sequence (reference tests/test_network.py:111-123)
    rs = np.random.default_rng(9)
    p_adam = network.init_network(16, rs)
    st = network.AdamState.for_params(p_adam, lr=1e-2)
    flat_a0 = network.flatten_params(p_adam)
    grads = [rs.standard_normal(flat_a0.size) for _ in range(5)]
    p = p_adam
    for gg in grads:
        p, st = network.adam_step(st, p, gg)
    # primitives
    rr = np.random.default_rng(12)
    x = rr.standard_normal((3, 16, 16)) + 1j * rr.standard_normal((3, 16, 16))
    rows = rr.standard_normal((3, 8)) + 1j * rr.standard_normal((3, 8))
    # 30-iteration reference reconstruct (line sources, the reference's own entry point)
    res = reconstruct(cfg, sim.data, chi_true=sim.chi_true)
    save("tiny", data=sim.data.matrix, chi_true=sim.chi_true.values, e_inc=einc.views, khat=ops.gd_kernel_hat,
         gs=ops.gs_matrix, alpha=alpha, g_alpha=g, bd=np.array(bd.as_row()), chi0=chi0, r0=r0, alpha0=alpha0,
         g_alpha0=g0, bd0=np.array(bd0.as_row()), g_frozen=g_fr, bd_frozen=np.array(bd_fr.as_row()),
         mask=mask, g_mask=g_mk, bd_mask=np.array(bd_mk.as_row()), net_flat=flat, grad_flat=gflat,
         bd_net=np.array(bdn.as_row()), dalpha=dalpha, adam_p0=flat_a0, adam_grads=np.array(grads),
         adam_p5=network.flatten_params(p), adam_m5=st.m, adam_v5=st.v,
         x=x, gd_x=apply_gd(ops, x), gdh_x=apply_gd_adjoint(ops, x), rows=rows, gsh_rows=apply_gs_adjoint(ops, rows),
         exp_alpha=expand(basis, alpha), trunc_x=truncate(basis, x),
         rec_trace=np.array([b.as_row() for b in res.trace]), rec_final=np.array(res.final_loss.as_row()),
         rec_chi_hat=res.chi_hat.values, rec_chi_cco=res.chi_cco.values, rec_chi0=res.chi0.values,
         rec_rel=np.array(res.rel_error))


def plane_case(name, cfg, scene, snr_db, noise_seed, k, store_ops=False):
    t0 = time.time()
    grid, arr, ops, views, chi, data = plane_problem(cfg, scene, snr_db, np.random.default_rng(noise_seed))
    out = composed_reconstruct(cfg, data, views, ops, chi, k)
    ctx = out["ctx"]
    g0, bd0 = grad_alpha(out["alpha0"], ctx)
    net = network.init_network(ctx.basis.m0, np.random.default_rng(cfg.rng_seed))
    flat = network.flatten_params(net)
    flat = flat + 0.02 * np.random.default_rng(123).standard_normal(flat.size)
    gflat, bdn = network.grad_loss(network.unflatten_params(flat, net), out["alpha0"], ctx)
    idx = np.sort(np.random.default_rng(5).choice(flat.size, size=min(4096, flat.size), replace=False))
    extra = dict(khat=ops.gd_kernel_hat, gs=ops.gs_matrix) if store_ops else {}
    save(name, data=data.matrix, chi_true=chi.values, chi0=out["chi0"], alpha0=out["alpha0"],
         g_alpha0=g0, bd0=np.array(bd0.as_row()), grad_idx=idx, grad_sub=gflat[idx],
         grad_norms=np.array([np.linalg.norm(gflat), np.abs(gflat).max()]), bd_net=np.array(bdn.as_row()),
         trace=out["trace"], final=out["final"], chi_hat=out["chi_hat"], chi_cco=out["chi_cco"],
         rel_error=np.array(out["rel_error"]), einc_checksum=np.array([views.sum(), np.abs(views).sum()]),
         gs_checksum=np.array([ops.gs_matrix.sum(), np.abs(ops.gs_matrix).sum()]),
         khat_checksum=np.array([ops.gd_kernel_hat.sum(), np.abs(ops.gd_kernel_hat).sum()]), **extra)
    print(f"{name}: rel_error {out['rel_error']:.6f}  ({time.time() - t0:.1f}s)", flush=True)


def make_cfg1():
    cfg = ImagingConfig(frequency=C0, doi_side=2.0, m1=32, m2=32, n_tx=16, n_rx=32, ring_radius=3.0, m_f=5,
                        k_iters=200, rng_seed=0).validate()
    scene = Scene((Shape(kind="disk", eps_r=2.0, center=(0.0, 0.0), radius=0.4),))
    plane_case("cfg1", cfg, scene, 20 * np.log10(100 / 5), 0, 200, store_ops=True)


def make_cfg2():
    cfg = ImagingConfig(frequency=C0, doi_side=2.0, m1=64, m2=64, n_tx=16, n_rx=32, ring_radius=3.0, m_f=8,
                        k_iters=500, rng_seed=1).validate()
    scene = Scene((Shape(kind="disk", eps_r=3.0, center=(-0.35, 0.0), radius=0.3),
                   Shape(kind="disk", eps_r=3.0, center=(0.35, 0.0), radius=0.3)))
    plane_case("cfg2", cfg, scene, 20 * np.log10(100 / 5), 1, 500)


def make_cfg3():
    cfg = ImagingConfig(frequency=C0, doi_side=2.0, m1=64, m2=64, n_tx=36, n_rx=36, ring_radius=3.0, m_f=8,
                        k_iters=500, rng_seed=2).validate()
    scene = Scene((Shape(kind="annulus", eps_r=4.0 + 0.5j, center=(0.0, 0.0), r_inner=0.3, r_outer=0.5),
                   Shape(kind="disk", eps_r=2.5, center=(0.6, 0.6), radius=0.15)))
    plane_case("cfg3", cfg, scene, 20.0, 2, 500)


def make_cfg4(n_scenes=2, k=500, first=0):
    for idx in range(first, first + n_scenes):
        cfg = ImagingConfig(frequency=C0, doi_side=2.0, m1=64, m2=64, n_tx=16, n_rx=32, ring_radius=3.0, m_f=8,
                            k_iters=k, rng_seed=idx).validate()
        scene, rng = cfg4_scene(idx)
        grid, arr, ops, views, chi, data = plane_problem(cfg, scene, 20 * np.log10(100 / 5), rng)
        out = composed_reconstruct(cfg, data, views, ops, chi, k)
        save(f"cfg4_s{idx}", data=data.matrix, chi_true=chi.values, alpha0=out["alpha0"], trace=out["trace"],
             final=out["final"], chi_cco=out["chi_cco"], rel_error=np.array(out["rel_error"]))
        print(f"cfg4 scene {idx}: rel_error {out['rel_error']:.6f}", flush=True)


def make_cfg5(k=300):
    """BASELINE cfg5: one large scene, 256x256 on [-2,2], 72 tx / 72 rx at 5 lambda, m_f=16, 300 iterations."""
    cfg = ImagingConfig(frequency=C0, doi_side=4.0, m1=256, m2=256, n_tx=72, n_rx=72, ring_radius=5.0, m_f=16,
                        k_iters=k, rng_seed=3).validate()
    scene, rng = cfg5_scene(3)
    t0 = time.time()
    grid, arr, ops, views, chi, data = plane_problem(cfg, scene, 20 * np.log10(100 / 5), rng)
    print(f"cfg5 data ({time.time() - t0:.0f}s)", flush=True)
    basis = SpectralBasis(cfg.m1, cfg.m2, cfg.m_f)
    fs = FieldSet(views, "incident")
    chi0, r0 = bp_initialize(data, fs, ops, cfg.beta)
    alpha0 = init_alpha(r0, data, fs, ops, basis, cfg.beta)
    ctx = LossContext(data=data, e_inc=views, ops=ops, basis=basis, beta=cfg.beta,
                      lambdas=(cfg.lambda1, cfg.lambda2, cfg.lambda3), tau_b=cfg.tau_b)
    g0, bd0 = grad_alpha(alpha0, ctx)
    net = network.init_network(basis.m0, np.random.default_rng(cfg.rng_seed))
    flat = network.flatten_params(net)
    flat = flat + 0.02 * np.random.default_rng(123).standard_normal(flat.size)
    gflat, bdn = network.grad_loss(network.unflatten_params(flat, net), alpha0, ctx)
    idx = np.sort(np.random.default_rng(5).choice(flat.size, size=4096, replace=False))
    common = dict(data=data.matrix, chi_true=chi.values, chi0=chi0, alpha0=alpha0, g_alpha0=g0,
                  bd0=np.array(bd0.as_row()), grad_idx=idx, grad_sub=gflat[idx],
                  grad_norms=np.array([np.linalg.norm(gflat), np.abs(gflat).max()]), bd_net=np.array(bdn.as_row()),
                  einc_checksum=np.array([views.sum(), np.abs(views).sum()]),
                  gs_checksum=np.array([ops.gs_matrix.sum(), np.abs(ops.gs_matrix).sum()]),
                  khat_checksum=np.array([ops.gd_kernel_hat.sum(), np.abs(ops.gd_kernel_hat).sum()]))
    save("cfg5", **common)
    print(f"cfg5 single-step part ({time.time() - t0:.0f}s)", flush=True)
    out = composed_reconstruct(cfg, data, views, ops, chi, k)
    save("cfg5", trace=out["trace"], final=out["final"], rel_error=np.array(out["rel_error"]), **common)
    print(f"cfg5: rel_error {out['rel_error']:.6f}  ({time.time() - t0:.1f}s)", flush=True)


def make_edges():
    """Edge cases the reference's own tests pin, on its tiny setup (tests/conftest.py:43-57):
    pole (cie.py:24-30, tests/test_cie.py:29), state = 0 at R = 0 (tests/test_losses.py:128-133),
    masked data = 1 at alpha = 0 (tests/test_losses.py:105-119), dead-mode whitening floor and
    the global-rms = 0 branch (network.py:88-104, tests/test_network.py:63-70)."""
    from dataclasses import replace
    from pdfisp.cie import PoleError
    from pdfisp.losses import pipeline_forward
    cfg = ImagingConfig(m1=16, m2=16, m_f=3, n_tx=8, n_rx=8, k_iters=30).validate()
    grid, arr = build_grid(cfg), build_array(cfg)
    ops = build_greens(cfg, arr, grid)
    einc = incident_fields(cfg, arr, grid)
    basis = SpectralBasis(16, 16, 3)
    sim = simulate(cfg, builtin_scene("austria", 2.0, scale=0.9))
    lam = (1e-3, 1e-5, 1e-5)
    ctx = LossContext(data=sim.data, e_inc=einc.views, ops=ops, basis=basis, beta=6.0, lambdas=lam, tau_b=0.5)
    n, m0 = 8, basis.m0
    # pole: G_D switched off (K^ = 0), one unit incident view, a constant current J = c with
    # c = -(1 + eps_reg) / beta, so chi = J conj(E) / (|E|^2 + eps_reg) = -1 / beta to rounding
    ops0 = replace(ops, gd_kernel_hat=np.zeros_like(ops.gd_kernel_hat))
    e1 = np.ones((1, 16, 16), complex)
    d1 = ScatteredData(matrix=sim.data.matrix[:1])
    ctx_pole = LossContext(data=d1, e_inc=e1, ops=ops0, basis=basis, beta=6.0, lambdas=lam, tau_b=0.5)
    c = -(1.0 + 1e-10) / 6.0
    alpha_pole = np.zeros((1, m0), complex)
    alpha_pole[0, 0] = c * 256.0          # slot 0 = DC: expand gives c at every pixel
    try:
        pipeline_forward(alpha_pole, ctx_pole)
        raise SystemExit("the reference did not raise PoleError")
    except PoleError:
        pass
    # a nearby non-pole point evaluates (the device must not flag it)
    alpha_near = alpha_pole * 1.001
    g_near, bd_near = grad_alpha(alpha_near, ctx_pole)
    # state term 0 at R = 0 (frozen R = 0, alpha = 0)
    ctx_r0 = LossContext(data=sim.data, e_inc=einc.views, ops=ops, basis=basis, beta=6.0, lambdas=lam, tau_b=0.5,
                         r_fixed=np.zeros((16, 16), complex))
    g_r0, bd_r0 = grad_alpha(np.zeros((n, m0), complex), ctx_r0)
    assert bd_r0.state == 0.0
    # masked data term = 1 at alpha = 0
    mask = np.zeros((n, 8))
    mask[:, :4] = 1.0
    ctx_mk = LossContext(data=ScatteredData(matrix=sim.data.matrix, mask=mask), e_inc=einc.views, ops=ops,
                         basis=basis, beta=6.0, lambdas=lam, tau_b=0.5)
    g_mk0, bd_mk0 = grad_alpha(np.zeros((n, m0), complex), ctx_mk)
    # whitening floor (a dead mode) and the global-rms = 0 branch
    chi0, r0 = bp_initialize(sim.data, einc, ops, 6.0)
    alpha0 = init_alpha(r0, sim.data, einc, ops, basis, 6.0)
    alpha_dead = alpha0.copy()
    alpha_dead[:, 0] = 0.0
    params = network.init_network(m0, np.random.default_rng(5))
    flat = network.flatten_params(params)
    flat = flat + 0.05 * np.random.default_rng(5).standard_normal(flat.size)
    params = network.unflatten_params(flat, params)
    dalpha_dead = network.forward_net(params, alpha_dead)
    grad_dead, bd_dead = network.grad_loss(params, alpha_dead, ctx)
    alpha_zero = np.zeros((n, m0), complex)
    dalpha_zero = network.forward_net(params, alpha_zero)
    grad_zero, bd_zero = network.grad_loss(params, alpha_zero, ctx)
    save("edges", alpha_pole=alpha_pole, data1=d1.matrix, alpha_near=alpha_near, g_near=g_near,
         bd_near=np.array(bd_near.as_row()), g_r0=g_r0, bd_r0=np.array(bd_r0.as_row()), mask=mask,
         g_mk0=g_mk0, bd_mk0=np.array(bd_mk0.as_row()), alpha0=alpha0, alpha_dead=alpha_dead, net_flat=flat,
         dalpha_dead=dalpha_dead, grad_dead=grad_dead, bd_dead=np.array(bd_dead.as_row()),
         dalpha_zero=dalpha_zero, grad_zero=grad_zero, bd_zero=np.array(bd_zero.as_row()))


def make_metrics():
    """relative_error / count_components (reconstruct.py:243-254) on images of many shapes."""
    from pdfisp.reconstruct import count_components as cc_ref, relative_error as re_ref
    from pdfisp.scenes import austria_preset
    rng = np.random.default_rng(21)
    shapes = [(6, 6), (12, 10), (9, 31), (32, 48), (64, 64), (256, 256), (1, 17), (17, 1)]
    imgs, counts, thr = [], [], 1.5
    for sh in shapes:
        for dens in (0.2, 0.45, 0.59, 0.8):
            img = np.where(rng.random(sh) < dens, 2.0, 1.0)
            imgs.append(img)
            counts.append(cc_ref(img, thr))
    # a one-pixel-wide serpentine (one component of 64 x 64 / 2 pixels, long union chains)
    snake = np.ones((64, 64))
    snake[::2, :] = 2.0
    for r in range(1, 64, 2):
        snake[r, 63 if (r // 2) % 2 == 0 else 0] = 2.0
    chk = np.indices((32, 32)).sum(0) % 2 + 1.0     # checkerboard: 4-connectivity isolates every cell
    grid = build_grid(ImagingConfig())
    aus = rasterize(austria_preset(2.0), grid).values.real + 1.0
    extra = [snake, chk * 1.6 / 1.5, aus, np.zeros((8, 8)), np.full((8, 8), 2.0)]
    ex_counts = [cc_ref(x, thr) for x in extra]
    a = rng.standard_normal((3, 32, 32)) + 1j * rng.standard_normal((3, 32, 32))
    b = rng.standard_normal((3, 32, 32)) + 1j * rng.standard_normal((3, 32, 32))
    rels = [re_ref(a[k].real + 1.0, b[k].real + 1.0) for k in range(3)]
    # images are stored as uint8 masks of {Re eps > 1.5} scaled back to eps in {1, 2} by the tests
    arrs = {f"img{k}": (x > thr).astype(np.uint8) for k, x in enumerate(imgs)}
    arrs.update({f"extra{k}": (x > thr).astype(np.uint8) for k, x in enumerate(extra)})
    save("metrics", counts=np.array(counts), extra_counts=np.array(ex_counts), rel_a=a, rel_b=b,
         rels=np.array(rels), thr=np.array(thr), **arrs)
    print("counts", counts, ex_counts)


def make_solver():
    """Forward solves of the reference (forward.py:193-275, 335-374): BiCGStab on a 32 x 32
    and a 64 x 64 grid, its dense-LU answer, NoConvergenceError at a small maxiter, and
    simulate() on a 64 x 64 grid (line sources, noise-free)."""
    from pdfisp.forward import NoConvergenceError
    out = {}
    for m in (32, 64):
        cfg = ImagingConfig(m1=m, m2=m, m_f=3, n_tx=8, n_rx=8).validate()
        grid, arr = build_grid(cfg), build_array(cfg)
        ops = build_greens(cfg, arr, grid)
        einc = incident_fields(cfg, arr, grid)
        chi = rasterize(builtin_scene("austria", 3.0, scale=0.9), grid)
        fs = solve_total_field(chi, einc, ops, method="fft")
        out[f"x{m}"], out[f"res{m}"] = fs.views, fs.residuals
        if m == 32:
            out["x32_dense"] = solve_total_field(chi, einc, ops, method="dense").views
        try:
            solve_total_field(chi, einc, ops, maxiter=3, method="fft")
            raise SystemExit("expected NoConvergenceError")
        except NoConvergenceError as ex:
            out[f"noconv_msg{m}"] = np.array(str(ex))
    cfg = ImagingConfig(m1=64, m2=64, m_f=3, n_tx=8, n_rx=8).validate()
    sim = simulate(cfg, builtin_scene("austria", 3.0, scale=0.9))
    out["sim64_data"] = sim.data.matrix
    save("solver", **out)
    print({k: v for k, v in out.items() if "msg" in k})


def make_special():
    """The reference's cylinder functions (special.py:64-106) on a grid spanning both regions."""
    from pdfisp import special as sp
    rng = np.random.default_rng(17)
    x = np.concatenate([np.linspace(1e-4, 60.0, 2401), rng.uniform(0.0, 300.0, 600), [8.0, 17.0, 0.5, 1e-6]])
    save("special", x=x, j0=sp.bessel_j0(x), j1=sp.bessel_j1(x), y0=sp.bessel_y0(x), y1=sp.bessel_y1(x),
         xneg=-x[:50], j0neg=sp.bessel_j0(-x[:50]), j1neg=sp.bessel_j1(-x[:50]))


def cfg4_sensitivity(idx: int, k: int = 500, eps=(1e-15, -1e-15)):
    """The reference's own rounding sensitivity on config-4 scene idx: its final relative
    error after k iterations when the measured data are scaled by (1 + eps), eps ~ 1 ulp.
    The loss passes a chaotic transient in its first iterations, so scenes whose reference
    output moves by ~1e-3 under 1e-15 input changes cannot be reproduced closer than that
    by any other summation order."""
    cfg = ImagingConfig(frequency=C0, doi_side=2.0, m1=64, m2=64, n_tx=16, n_rx=32, ring_radius=3.0, m_f=8,
                        k_iters=k, rng_seed=idx).validate()
    scene, rng = cfg4_scene(idx)
    grid, arr, ops, views, chi, data = plane_problem(cfg, scene, 20 * np.log10(100 / 5), rng)
    out = []
    for e in eps:
        d2 = ScatteredData(matrix=data.matrix * (1.0 + e))
        out.append(composed_reconstruct(cfg, d2, views, ops, chi, k)["rel_error"])
    return np.array(out)


def make_cfg4sens():
    """Per-scene sensitivity records for config-4 scenes given in $SCENES (default 0-9)."""
    scenes = [int(x) for x in os.environ.get("SCENES", "0,1,2,3,4,5,6,7,8,9").split(",")]
    for idx in scenes:
        rel = cfg4_sensitivity(idx)
        save(f"cfg4_sens_s{idx}", rel_perturbed=rel, eps=np.array([1e-15, -1e-15]))
        print(f"cfg4 scene {idx}: perturbed rel_error {rel}", flush=True)


def make_files():
    """.emsca / .grid files written by the reference (fileio.py:98-145)."""
    from pdfisp.fileio import save_dataset, save_grid
    from pdfisp.geometry import ComplexGrid
    rng = np.random.default_rng(31)
    mat = rng.standard_normal((8, 12)) + 1j * rng.standard_normal((8, 12))
    mask = rng.random((8, 12)) > 0.25
    save_dataset(os.path.join(HERE, "ref_masked.emsca"), ScatteredData(matrix=mat * mask, snr_db=26.02, mask=mask),
                 meta={"scene": "random", "seed": 31})
    save_dataset(os.path.join(HERE, "ref_plain.emsca"), ScatteredData(matrix=mat))
    img = rng.standard_normal((16, 16)) + 1j * rng.standard_normal((16, 16))
    save_grid(os.path.join(HERE, "ref.grid"), ComplexGrid(values=img, cell_size=0.09375), config_hash="abc123")
    save("files", mat=mat, mask=mask, img=img)


def make_cfg4more():
    """Eight more config-4 scenes (indices 2-9), 500 iterations each."""
    make_cfg4(n_scenes=8, first=2)


def make_algebra():
    """Module-level CIE algebra, regularisers and filters (cie.py, losses.py:86-196,
    filters.py) on odd shapes, and the state / data terms on the tiny setup."""
    from pdfisp import cie, filters, losses
    from pdfisp.config import CcoParams
    rng = np.random.default_rng(41)
    out = {}
    chi = rng.uniform(0.0, 9.0, (40, 40)) + 1j * rng.uniform(0.0, 2.0, (40, 40))
    chi[3, 4] = 0.0
    out.update(ctr_chi=chi, ctr_r=cie.chi_to_r(chi, 6.0), ctr_back=cie.r_to_chi(cie.chi_to_r(chi, 6.0), 6.0),
               ctr_rc=cie.chi_to_r(chi, 6.0 + 1.5j), ctr_rc_back=cie.r_to_chi(cie.chi_to_r(chi, 6.0 + 1.5j), 6.0 + 1.5j))
    j = rng.standard_normal((5, 12, 20)) + 1j * rng.standard_normal((5, 12, 20))
    e = rng.standard_normal((5, 12, 20)) + 1j * rng.standard_normal((5, 12, 20))
    e[:, 2, 7] = 0.0
    rec = cie.pixel_least_squares(j, e)
    out.update(pls_j=j, pls_e=e, pls_chi=rec.chi, pls_num=rec.numerator, pls_den=rec.denominator,
               pls_eps=np.array(rec.eps_reg), pls_deg=rec.degenerate, pls_eps_default=np.array(cie.default_eps_reg(e)))
    rec2 = cie.pixel_least_squares(j, e, eps_reg=0.25)
    out.update(pls2_chi=rec2.chi, pls2_den=rec2.denominator, pls2_deg=rec2.degenerate)
    rc = rng.standard_normal((20, 28)) + 1j * rng.standard_normal((20, 28))
    rc[5, 5] = 0.0
    rc[6:9, 10:14] = 1.7 + 0.2j          # a flat bright patch for the bridge term
    lam = (1e-3, 1e-5, 1e-5)
    out.update(reg_chi=rc, reg_bound=np.array(losses.loss_bound(rc)), reg_tv=np.array(losses.loss_tv(rc)),
               reg_bridge=np.array(losses.loss_bridge(rc, 0.5)), reg_gb=losses.bound_chi_grad(rc),
               reg_gt=losses.tv_chi_grad(rc), reg_gr=losses.bridge_chi_grad(rc, 0.5),
               reg_g=losses.regularizer_chi_grad(rc, lam, 0.5), reg_g_l2=losses.regularizer_chi_grad(rc, (0, 1, 0), 0.5))
    for k, (shape, r) in enumerate([((7, 9), 1), ((12, 5), 2), ((6, 6), 4), ((64, 48), 2)]):
        img = rng.standard_normal(shape)
        out[f"box{k}_img"], out[f"box{k}_r"], out[f"box{k}_out"] = img, np.array(r), filters.box_mean(img, r)
    gi, gg = rng.standard_normal((10, 11)), rng.standard_normal((10, 11))
    out.update(gf_inp=gi, gf_guide=gg, gf_out=filters.guided_filter(gi, gg, 2, 1e-3))
    cc = 0.05 * (rng.standard_normal((12, 12)) + 1j * rng.standard_normal((12, 12)))
    plateau = np.zeros((16, 16), dtype=complex)
    plateau[4:12, 4:12] = 7.0
    big = rng.uniform(0, 4, (30, 50)) + 1j * rng.uniform(0, 1, (30, 50))
    p = CcoParams(tau=3.0, eta_max=0.1, delta=0.5, gf_radius=2, gf_eps=1e-3)
    out.update(cco_small=cc, cco_small_out=filters.apply_cco(cc, p), cco_plateau_out=filters.apply_cco(plateau, p),
               cco_big=big, cco_big_out=filters.apply_cco(big, CcoParams()))
    # state / data terms on the tiny setup (reference tests/conftest.py:43-57)
    cfg = ImagingConfig(m1=16, m2=16, m_f=3, n_tx=8, n_rx=8).validate()
    grid, arr = build_grid(cfg), build_array(cfg)
    ops = build_greens(cfg, arr, grid)
    e_inc = incident_fields(cfg, arr, grid)
    basis = SpectralBasis(16, 16, 3)
    alpha = rng.standard_normal((8, basis.m0)) + 1j * rng.standard_normal((8, basis.m0))
    r_hat = cie.chi_to_r(0.3 * (rng.random((16, 16)) + 1j * rng.random((16, 16))), 6.0)
    mat = rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8))
    mask = rng.random((8, 8)) > 0.3
    data = ScatteredData(matrix=mat * mask, mask=mask)
    out.update(st_alpha=alpha, st_rhat=r_hat,
               st_res=cie.cie_state_residual(alpha, r_hat, e_inc.views, ops, basis, 6.0),
               st_loss=np.array(losses.loss_state(alpha, r_hat, e_inc.views, ops, basis, 6.0)),
               dt_mat=mat, dt_mask=mask, dt_loss=np.array(losses.loss_data(alpha, data, ops, basis)),
               dt_loss_plain=np.array(losses.loss_data(alpha, ScatteredData(matrix=mat), ops, basis)))
    save("algebra", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tiny", "cfg1", "cfg2", "cfg3", "cfg4"]
    for w in which:
        globals()[f"make_{w}"]()
