"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the PDF (physics-driven Fourier-spectral) solver's
per-iteration hot path as the reference package `pdfisp` defines it.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may
import this module; the CUDA product path never calls it.

Parity pinning: every function here is checked against golden vectors that
were produced by importing the unmodified reference (`/root/reference/pkg/src`)
in the build container (``tests/golden/make_golden.py``, fixtures in
``tests/golden/*.npz``).  Citations are ``file:line`` relative to
``/root/reference/pkg/src/pdfisp/``.

Conventions (reference): time dependence exp(-i w t), first-kind Hankel
H0^(1) (forward.py:10-11); forward DFT unnormalised, inverse DFT carries
1/(M1*M2) (spectral.py:1-12); complex gradients g = dL/dRe + i dL/dIm
(losses.py:255-264).

The ``cdtype`` switch (complex128 default) lets the precision study replay the
same algorithm in complex64 / float32.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.special as sps

C0 = 299792458.0
EPS_TV = 1e-12           # losses.py:29
SCALE_MIX = 0.7          # network.py:83
SCALE_FLOOR = 0.1        # network.py:84
OUTPUT_GAIN = 8.0        # network.py:85


class OraclePoleError(ValueError):
    pass


# ----------------------------------------------------------------------------
# geometry / operators (one-time setup; geometry.py:72-100, forward.py:101-137)

def grid_centers(doi_side: float, m1: int, m2: int) -> tuple[np.ndarray, float]:
    """Row-major cell centres, y grows with the row index (geometry.py:72-84)."""
    cs = doi_side / m1
    xs = -doi_side / 2 + cs * (np.arange(m2) + 0.5)
    ys = -doi_side / 2 + cs * (np.arange(m1) + 0.5)
    xx = np.broadcast_to(xs[None, :], (m1, m2))
    yy = np.broadcast_to(ys[:, None], (m1, m2))
    return np.stack([xx.ravel(), yy.ravel()], axis=1), cs


def ring(n: int, radius: float) -> np.ndarray:
    """Antennas at angles 2*pi*k/n (geometry.py:87-100)."""
    th = 2.0 * np.pi * np.arange(n) / n
    return radius * np.column_stack([np.cos(th), np.sin(th)])


@dataclass
class Operators:
    k_hat: np.ndarray        # (2m1, 2m2) FFT of the wrap-indexed displacement kernel
    gs: np.ndarray           # (R, m1*m2)
    m1: int
    m2: int
    k0: float
    cell: float


def build_operators(k0: float, doi_side: float, m1: int, m2: int,
                    rx: np.ndarray) -> Operators:
    """Equal-area-disk cell quadrature (forward.py:101-137).

    off-diagonal  (i pi k0 a / 2) J1(k0 a) H0^(1)(k0 rho)
    self term     (i pi k0 a / 2) H1^(1)(k0 a) - 1
    Row m1 and column m2 of the doubled-grid kernel are never reached and are 0.
    """
    centers, cs = grid_centers(doi_side, m1, m2)
    a = cs / math.sqrt(math.pi)
    pref = 0.5j * math.pi * k0 * a
    off_w = pref * sps.jv(1, k0 * a)
    di = np.arange(2 * m1)
    di = np.where(di < m1, di, di - 2 * m1)
    dj = np.arange(2 * m2)
    dj = np.where(dj < m2, dj, dj - 2 * m2)
    rho = cs * np.sqrt(di[:, None] ** 2 + dj[None, :] ** 2.0)
    ker = np.zeros((2 * m1, 2 * m2), dtype=np.complex128)
    nz = rho > 0
    ker[nz] = off_w * sps.hankel1(0, k0 * rho[nz])
    ker[0, 0] = pref * sps.hankel1(1, k0 * a) - 1.0
    ker[m1, :] = 0
    ker[:, m2] = 0
    d = np.sqrt(((rx[:, None, :] - centers[None, :, :]) ** 2).sum(-1))
    gs = off_w * sps.hankel1(0, k0 * d)
    return Operators(k_hat=np.fft.fft2(ker), gs=gs, m1=m1, m2=m2, k0=k0, cell=cs)


def line_source_fields(k0: float, tx: np.ndarray, doi_side: float, m1: int, m2: int) -> np.ndarray:
    """(i/4) H0^(1)(k0 |r - r_tx|) per transmitter (forward.py:174-181)."""
    centers, _ = grid_centers(doi_side, m1, m2)
    d = np.sqrt(((tx[:, None, :] - centers[None, :, :]) ** 2).sum(-1))
    return (0.25j * sps.hankel1(0, k0 * d)).reshape(len(tx), m1, m2)


def plane_wave_fields(k0: float, n: int, doi_side: float, m1: int, m2: int) -> np.ndarray:
    """exp(i k0 (x cos phi + y sin phi)), phi = 2 pi k / n."""
    centers, _ = grid_centers(doi_side, m1, m2)
    phi = 2.0 * np.pi * np.arange(n) / n
    ph = np.outer(np.cos(phi), centers[:, 0]) + np.outer(np.sin(phi), centers[:, 1])
    return np.exp(1j * k0 * ph).reshape(n, m1, m2)


# ----------------------------------------------------------------------------
# truncated Fourier basis (spectral.py:21-87)

def corner_index(m1: int, m2: int, mf: int) -> tuple[np.ndarray, np.ndarray]:
    """Corner blocks TL, TR, BL, BR; row-major inside each (spectral.py:29-44)."""
    lo_r, hi_r = np.arange(mf), np.arange(m1 - mf, m1)
    lo_c, hi_c = np.arange(mf), np.arange(m2 - mf, m2)
    rr, cc = [], []
    for rb in (lo_r, hi_r):
        for cb in (lo_c, hi_c):
            rr.append(np.repeat(rb, mf))
            cc.append(np.tile(cb, mf))
    return np.concatenate(rr), np.concatenate(cc)


def expand(alpha: np.ndarray, m1: int, m2: int, mf: int, cdtype=np.complex128) -> np.ndarray:
    """Scatter into the corners, inverse 2-D DFT with 1/(m1 m2) (spectral.py:68-79)."""
    r, c = corner_index(m1, m2, mf)
    spec = np.zeros(alpha.shape[:-1] + (m1, m2), dtype=cdtype)
    spec[..., r, c] = alpha
    return np.fft.ifft2(spec).astype(cdtype)


def truncate(img: np.ndarray, mf: int, cdtype=np.complex128) -> np.ndarray:
    """Forward 2-D DFT, gather the corners (spectral.py:56-65)."""
    m1, m2 = img.shape[-2:]
    r, c = corner_index(m1, m2, mf)
    return np.fft.fft2(img)[..., r, c].astype(cdtype)


# ----------------------------------------------------------------------------
# operators applied (forward.py:140-151, 303-306)

def apply_gd(ops: Operators, x: np.ndarray, cdtype=np.complex128) -> np.ndarray:
    m1, m2 = ops.m1, ops.m2
    big = np.zeros(x.shape[:-2] + (2 * m1, 2 * m2), dtype=cdtype)
    big[..., :m1, :m2] = x
    y = np.fft.ifft2(np.fft.fft2(big) * ops.k_hat.astype(cdtype))
    return y[..., :m1, :m2].astype(cdtype)


def apply_gd_adj(ops: Operators, x: np.ndarray, cdtype=np.complex128) -> np.ndarray:
    """Complex-symmetric kernel: G_D^H = conj o G_D o conj (forward.py:149-151)."""
    return np.conj(apply_gd(ops, np.conj(x), cdtype))


def apply_gs_adj(ops: Operators, rows: np.ndarray, cdtype=np.complex128) -> np.ndarray:
    out = rows @ np.conj(ops.gs).astype(cdtype)
    return out.reshape(rows.shape[:-1] + (ops.m1, ops.m2))


# ----------------------------------------------------------------------------
# loss context and the composite loss (losses.py:52-306, cie.py:24-80)

@dataclass
class Context:
    data: np.ndarray              # (n, R) measured scattered field
    e_inc: np.ndarray             # (n, m1, m2)
    ops: Operators
    mf: int
    beta: float
    lambdas: tuple
    tau_b: float
    mask: np.ndarray | None = None
    r_fixed: np.ndarray | None = None
    cdtype: type = np.complex128
    c_sca: float = field(init=False)
    c_inc: float = field(init=False)

    def __post_init__(self):
        d = self.data if self.mask is None else self.data * self.mask
        self.c_sca = float(np.sum(np.abs(d) ** 2))           # losses.py:71
        self.c_inc = float(np.sum(np.abs(self.e_inc) ** 2))  # losses.py:72
        if self.c_sca <= 0 or self.c_inc <= 0:
            raise ValueError("zero normaliser")


def _fdiff(img):
    dx = np.zeros_like(img)
    dy = np.zeros_like(img)
    dx[:, :-1] = np.diff(img, axis=1)
    dy[:-1, :] = np.diff(img, axis=0)
    return dx, dy


def _sig(z):
    return sps.expit(z)


def reg_values(chi: np.ndarray, tau: float) -> tuple[float, float, float]:
    """bound, tv, bridge (losses.py:115-144)."""
    bound = float(np.sum(np.minimum(chi.real, 0.0) ** 2))
    dx, dy = _fdiff(chi)
    tv = float(np.sum(np.sqrt(np.abs(dx) ** 2 + np.abs(dy) ** 2 + EPS_TV)))
    a = np.abs(chi)
    gx, gy = _fdiff(a)
    bridge = float(np.sum(_sig((a - tau) / tau) * np.exp(-(gx ** 2 + gy ** 2))))
    return bound, tv, bridge


def _scatter_adj(wx, wy):
    """Adjoint of the forward-difference pair (losses.py:160-165)."""
    g = np.zeros_like(wx)
    g[:, 1:] += wx[:, :-1]
    g[:, :-1] -= wx[:, :-1]
    g[1:, :] += wy[:-1, :]
    g[:-1, :] -= wy[:-1, :]
    return g


def reg_grad(chi: np.ndarray, lambdas, tau: float) -> np.ndarray:
    """lambda-weighted chi-gradients of bound/tv/bridge (losses.py:152-195)."""
    l1, l2, l3 = lambdas
    g = np.zeros_like(chi)
    if l1:
        g = g + l1 * (2.0 * np.minimum(chi.real, 0.0))
    if l2:
        dx, dy = _fdiff(chi)
        s = np.sqrt(np.abs(dx) ** 2 + np.abs(dy) ** 2 + EPS_TV)
        g = g + l2 * _scatter_adj(dx / s, dy / s)
    if l3:
        a = np.abs(chi)
        gx, gy = _fdiff(a)
        sg = _sig((a - tau) / tau)
        damp = np.exp(-(gx ** 2 + gy ** 2))
        ga = sg * (1.0 - sg) / tau * damp + _scatter_adj(-2.0 * sg * damp * gx,
                                                         -2.0 * sg * damp * gy)
        safe = np.where(a > 0, a, 1.0)
        phase = np.where(a > 0, chi / safe, 0.0)
        g = g + l3 * ga * phase
    return g


@dataclass
class StepState:
    j: np.ndarray
    e: np.ndarray
    chi: np.ndarray
    den: np.ndarray
    r: np.ndarray
    p: np.ndarray
    sres: np.ndarray
    dres: np.ndarray
    eps_reg: float
    parts: dict


def forward(alpha: np.ndarray, ctx: Context) -> StepState:
    """pipeline_forward (losses.py:215-247) with pixel LS (cie.py:42-80)."""
    ct = ctx.cdtype
    ops = ctx.ops
    m1, m2 = ops.m1, ops.m2
    alpha = np.atleast_2d(alpha).astype(ct)
    n = alpha.shape[0]
    j = expand(alpha, m1, m2, ctx.mf, ct)
    e = (ctx.e_inc.astype(ct) + apply_gd(ops, j, ct)).astype(ct)
    pw = np.sum(np.abs(e) ** 2, axis=(1, 2))
    eps_reg = 1e-10 * float(pw.max()) / (m1 * m2)                       # cie.py:49-50
    num = np.sum(j * np.conj(e), axis=0)
    den = np.sum(np.abs(e) ** 2, axis=0) + eps_reg
    chi = num / den
    if ctx.r_fixed is not None:
        r = ctx.r_fixed.astype(ct)
    else:
        q = ctx.beta * chi + 1.0
        if np.any(np.abs(q) < 1e-14):                                      # cie.py:27-29
            raise OraclePoleError("beta*chi + 1 vanishes")
        r = ctx.beta * chi / q
    p = e + ctx.beta * j
    sres = r * p - ctx.beta * j
    dres = j.reshape(n, -1) @ ops.gs.T.astype(ct) - ctx.data.astype(ct)
    if ctx.mask is not None:
        dres = dres * ctx.mask
    state = float(np.sum(np.abs(sres) ** 2)) / ctx.c_inc
    data = float(np.sum(np.abs(dres) ** 2)) / ctx.c_sca
    bound, tv, bridge = reg_values(chi, ctx.tau_b)
    l1, l2, l3 = ctx.lambdas
    total = state + data + l1 * bound + l2 * tv + l3 * bridge
    parts = dict(state=state, data=data, bound=bound, tv=tv, bridge=bridge, total=total)
    if not np.isfinite(total):
        bad = [k for k, v in parts.items() if k != "total" and not np.isfinite(v)]
        raise FloatingPointError(f"nonfinite loss term(s): {bad}")
    return StepState(j, e, chi, den, r, p, sres, dres, eps_reg, parts)


def backward(st: StepState, ctx: Context) -> np.ndarray:
    """pipeline_backward (losses.py:267-306); eps_reg held constant."""
    ct = ctx.cdtype
    ops = ctx.ops
    b = ctx.beta
    g_s = (2.0 / ctx.c_inc) * st.sres
    g_p = np.conj(st.r) * g_s
    g_j = b * (g_p - g_s)
    g_e = g_p
    g_rows = (2.0 / ctx.c_sca) * st.dres
    if ctx.mask is not None:
        g_rows = g_rows * ctx.mask
    g_j = g_j + apply_gs_adj(ops, g_rows.astype(ct), ct)
    g_chi = reg_grad(st.chi, ctx.lambdas, ctx.tau_b)
    if ctx.r_fixed is None:
        g_r = np.sum(np.conj(st.p) * g_s, axis=0)
        g_chi = g_chi + np.conj(b / (b * st.chi + 1.0) ** 2) * g_r
    g_num = g_chi / st.den
    g_den = -np.real(np.conj(g_chi) * st.chi) / st.den
    g_j = g_j + st.e * g_num
    g_e = g_e + np.conj(g_num) * st.j + 2.0 * g_den * st.e
    g_j = g_j + apply_gd_adj(ops, g_e.astype(ct), ct)
    return (truncate(g_j, ctx.mf, ct) / (ops.m1 * ops.m2)).astype(ct)


def grad_alpha(alpha, ctx):
    st = forward(alpha, ctx)
    return backward(st, ctx), st.parts


# ----------------------------------------------------------------------------
# corrective network + Adam (network.py:53-264)

def init_net(m0: int, rng: np.random.Generator) -> list[np.ndarray]:
    """[w1, b1, w2, b2, w3, b3]; N(0, 1/fan_in), zero last layer (network.py:53-71)."""
    dims = [2 * m0, 4 * m0, 4 * m0, 2 * m0]
    out = []
    for li in range(3):
        fi, fo = dims[li], dims[li + 1]
        w = np.zeros((fo, fi)) if li == 2 else rng.normal(0.0, math.sqrt(1.0 / fi), (fo, fi))
        out += [w, np.zeros(fo)]
    return out


def flat(params) -> np.ndarray:
    return np.concatenate([p.ravel() for p in params])


def unflat(v: np.ndarray, like) -> list[np.ndarray]:
    out, k = [], 0
    for p in like:
        out.append(v[k:k + p.size].reshape(p.shape).copy())
        k += p.size
    if k != v.size:
        raise ValueError("flat parameter vector has the wrong length")
    return out


def feature_scales(alpha0: np.ndarray, joint: bool) -> np.ndarray:
    """Per-mode whitening (network.py:88-104)."""
    a2 = np.abs(alpha0) ** 2
    mode = np.sqrt(a2.mean(axis=0))
    glob = float(np.sqrt(a2.mean()))
    if glob == 0.0:
        return np.ones(2 * (alpha0.size if joint else alpha0.shape[1]))
    s = np.maximum(mode ** SCALE_MIX * glob ** (1.0 - SCALE_MIX), SCALE_FLOOR * glob)
    if joint:
        s = np.tile(s, alpha0.shape[0])
    return np.concatenate([s, s])


def net_rows(alpha0: np.ndarray, joint: bool) -> np.ndarray:
    a = alpha0.reshape(1, -1) if joint else alpha0
    return np.concatenate([a.real, a.imag], axis=1)


def net_merge(y: np.ndarray, n: int, m0: int, joint: bool) -> np.ndarray:
    h = y.shape[1] // 2
    z = y[:, :h] + 1j * y[:, h:]
    return z.reshape(n, m0)


def net_forward(params, x, s, rdtype=np.float64):
    w1, b1, w2, b2, w3, b3 = [p.astype(rdtype) for p in params]
    x0 = (x / s).astype(rdtype)
    h1 = np.tanh(x0 @ w1.T + b1)
    h2 = np.tanh(h1 @ w2.T + b2)
    gain = (OUTPUT_GAIN * s / math.sqrt(w3.shape[1])).astype(rdtype)
    return (h2 @ w3.T + b3) * gain, (x0, h1, h2, gain)


def delta_alpha(params, alpha0, joint=False, rdtype=np.float64):
    alpha0 = np.atleast_2d(alpha0)
    y, _ = net_forward(params, net_rows(alpha0, joint), feature_scales(alpha0, joint), rdtype)
    return net_merge(y, *alpha0.shape, joint)


def grad_loss(params, alpha0, ctx: Context, joint=False, rdtype=np.float64):
    """Flat gradient in order w1,b1,w2,b2,w3,b3 (network.py:183-223)."""
    alpha0 = np.atleast_2d(alpha0)
    n, m0 = alpha0.shape
    s = feature_scales(alpha0, joint)
    y, (x0, h1, h2, gain) = net_forward(params, net_rows(alpha0, joint), s, rdtype)
    ahat = alpha0 + net_merge(y, n, m0, joint)
    st = forward(ahat, ctx)
    ga = backward(st, ctx)
    gy = net_rows(ga, joint).astype(rdtype) * gain
    w1, _, w2, _, w3, _ = [p.astype(rdtype) for p in params]
    gz2 = (gy @ w3) * (1 - h2 * h2)
    gz1 = (gz2 @ w2) * (1 - h1 * h1)
    g = np.concatenate([(gz1.T @ x0).ravel(), gz1.sum(0), (gz2.T @ h1).ravel(), gz2.sum(0),
                        (gy.T @ h2).ravel(), gy.sum(0)])
    if not np.all(np.isfinite(g)):
        raise FloatingPointError("nonfinite parameter gradient")
    return g, st.parts


@dataclass
class Adam:
    m: np.ndarray
    v: np.ndarray
    t: int = 0
    lr: float = 1e-2
    b1: float = 0.9
    b2: float = 0.999
    eps: float = 1e-8


def adam_update(st: Adam, theta: np.ndarray, g: np.ndarray, rdtype=np.float64) -> np.ndarray:
    """Bias-corrected Adam, updates st in place, returns new theta (network.py:248-264)."""
    st.t += 1
    st.m = (st.b1 * st.m + (1.0 - st.b1) * g).astype(rdtype)
    st.v = (st.b2 * st.v + (1.0 - st.b2) * g * g).astype(rdtype)
    mh = st.m / (1.0 - st.b1 ** st.t)
    vh = st.v / (1.0 - st.b2 ** st.t)
    out = (theta - st.lr * mh / (np.sqrt(vh) + st.eps)).astype(rdtype)
    if not np.all(np.isfinite(out)):
        raise FloatingPointError("nonfinite parameters after optimizer step")
    return out


# ----------------------------------------------------------------------------
# initialisation (reconstruct.py:52-153) and epilogue (cie.py:83-99, filters.py)

def bp_initialize(data, e_inc, ops: Operators, beta, mask=None):
    d = data if mask is None else data * mask
    b = apply_gs_adj(ops, d)
    w = b.reshape(d.shape[0], -1) @ ops.gs.T
    if mask is not None:
        w = w * mask
    num = np.sum(np.conj(w) * d, axis=1)
    den = np.sum(np.abs(w) ** 2, axis=1)
    gamma = np.where(den > 0, num / np.where(den > 0, den, 1.0), 0.0)
    j = gamma[:, None, None] * b
    e = e_inc + apply_gd(ops, j)
    pw = np.sum(np.abs(e) ** 2, axis=(1, 2))
    eps = 1e-10 * pw.max() / (ops.m1 * ops.m2)
    chi0 = np.sum(j * np.conj(e), axis=0) / (np.sum(np.abs(e) ** 2, axis=0) + eps)
    q = beta * chi0 + 1.0
    if np.any(np.abs(q) < 1e-14):
        raise OraclePoleError("beta*chi + 1 vanishes")
    return chi0, beta * chi0 / q


def init_alpha(r0, data, e_inc, ops: Operators, mf, beta, mask=None):
    """One exact line-search step of the frozen-R quadratic from zero."""
    m1, m2 = ops.m1, ops.m2
    d = data if mask is None else data * mask
    c_sca = float(np.sum(np.abs(d) ** 2))
    c_inc = float(np.sum(np.abs(e_inc) ** 2))
    n = e_inc.shape[0]
    sres = r0 * e_inc
    rows = -data if mask is None else -data * mask
    gs_r = (2.0 / c_inc) * sres
    g_j = apply_gd_adj(ops, np.conj(r0) * gs_r) + beta * (np.conj(r0) - 1.0) * gs_r
    g_rows = (2.0 / c_sca) * rows
    if mask is not None:
        g_rows = g_rows * mask
    g_j = g_j + apply_gs_adj(ops, g_rows)
    g = truncate(g_j, mf) / (m1 * m2)
    jd = expand(g, m1, m2, mf)
    s_lin = r0 * apply_gd(ops, jd) + beta * (r0 - 1.0) * jd
    rr = jd.reshape(n, -1) @ ops.gs.T
    if mask is not None:
        rr = rr * mask
    q = float(np.sum(np.abs(s_lin) ** 2)) / c_inc + float(np.sum(np.abs(rr) ** 2)) / c_sca
    g2 = float(np.sum(np.abs(g) ** 2))
    if q <= 0 or g2 <= 0:
        return np.zeros_like(g)
    return -(g2 / (2.0 * q)) * g


def recover_chi(alpha, e_inc, ops: Operators, mf):
    j = expand(np.atleast_2d(alpha), ops.m1, ops.m2, mf)
    e = e_inc + apply_gd(ops, j)
    eps = 1e-10 * np.sum(np.abs(e) ** 2, axis=(1, 2)).max() / (ops.m1 * ops.m2)
    return np.sum(j * np.conj(e), axis=0) / (np.sum(np.abs(e) ** 2, axis=0) + eps)


def box_mean(img, r):
    """Edge-replicate (2r+1)^2 window mean via a summed-area table (filters.py:16-33)."""
    w = 2 * r + 1
    pad = np.pad(img, r, mode="edge")
    sat = np.zeros((pad.shape[0] + 1, pad.shape[1] + 1))
    sat[1:, 1:] = pad.cumsum(0).cumsum(1)
    m1, m2 = img.shape
    return (sat[w:w + m1, w:w + m2] - sat[:m1, w:w + m2] - sat[w:w + m1, :m2]
            + sat[:m1, :m2]) / (w * w)


def guided(p, i, r, eps):
    mi, mp = box_mean(i, r), box_mean(p, r)
    a = (box_mean(i * p, r) - mi * mp) / (box_mean(i * i, r) - mi * mi + eps)
    b = mp - a * mi
    return box_mean(a, r) * i + box_mean(b, r)


def cco(chi, tau=3.0, eta_max=0.1, delta=0.5, radius=2, eps_gf=1e-3):
    """(1+eta) G(chi|chi) + eta chi per channel (filters.py:56-67)."""
    eta = eta_max * _sig((np.abs(chi) - tau) / delta)
    sm = guided(chi.real, chi.real, radius, eps_gf) + 1j * guided(chi.imag, chi.imag, radius, eps_gf)
    return (1.0 + eta) * sm + eta * chi


def relative_error(eps_hat, eps_true):
    return float(np.linalg.norm(np.real(eps_hat) - np.real(eps_true))
                 / np.linalg.norm(np.real(eps_true)))


def count_components(eps_map, threshold) -> int:
    """4-connected components of {Re eps > threshold} (reconstruct.py:250-254),
    restated as an explicit-stack flood fill (the reference calls scipy.ndimage.label)."""
    fgm = np.real(np.asarray(eps_map)) > threshold
    m1, m2 = fgm.shape
    seen = np.zeros_like(fgm)
    n = 0
    for r0, c0 in zip(*np.nonzero(fgm)):
        if seen[r0, c0]:
            continue
        n += 1
        seen[r0, c0] = True
        stack = [(r0, c0)]
        while stack:
            r, c = stack.pop()
            for rr, cc in ((r - 1, c), (r + 1, c), (r, c - 1), (r, c + 1)):
                if 0 <= rr < m1 and 0 <= cc < m2 and fgm[rr, cc] and not seen[rr, cc]:
                    seen[rr, cc] = True
                    stack.append((rr, cc))
    return n


def reconstruct_loop(ctx: Context, alpha0, k_iters, lr=1e-2, seed=0, joint=False,
                     rdtype=np.float64, use_cco=True, cco_kw=None):
    """The reference's k-loop plus epilogue (reconstruct.py:208-226)."""
    n, m0 = alpha0.shape
    params = init_net(m0 * (n if joint else 1), np.random.default_rng(seed))
    theta = flat(params).astype(rdtype)
    adam = Adam(m=np.zeros_like(theta), v=np.zeros_like(theta), lr=lr)
    trace = []
    for _ in range(k_iters):
        g, parts = grad_loss(unflat(theta, params), alpha0, ctx, joint, rdtype)
        trace.append(parts)
        theta = adam_update(adam, theta, g.astype(rdtype), rdtype)
    net = unflat(theta.astype(np.float64), params)
    ahat = alpha0 + delta_alpha(net, alpha0, joint)
    final = forward(ahat, ctx).parts
    chi_hat = recover_chi(ahat, ctx.e_inc, ctx.ops, ctx.mf)
    chi_cco = cco(chi_hat, **(cco_kw or {})) if use_cco else chi_hat.copy()
    return dict(trace=trace, final=final, chi_hat=chi_hat, chi_cco=chi_cco, theta=theta,
                alpha_hat=ahat)
