"""Reference-shaped solver API, GPU underneath.

Same names, argument meaning and error behaviour as the reference's hot-path
functions (citations relative to /root/reference/pkg/src/pdfisp/):

  LossContext, LossBreakdown          losses.py:36-80
  pipeline_forward / pipeline_backward losses.py:215-306
  grad_alpha, loss_total              losses.py:250-252, 309-312
  NetworkParams, init_network         network.py:53-71
  forward_net, flatten/unflatten      network.py:143-176
  grad_loss                           network.py:183-223
  AdamState, adam_step                network.py:230-264
  truncate, expand                    spectral.py:56-87
  apply_gd(_adjoint), apply_gs_adjoint forward.py:140-151, 303-306
  bp_initialize, init_alpha           reconstruct.py:52-153
  recover_contrast                    cie.py:83-99
  apply_cco                           filters.py:56-67
  reconstruct, ReconstructionResult   reconstruct.py:32-236

Host arrays in, host arrays out (numpy complex128 / float64), like the
reference.  Every numerical step runs in libpdfb200.so on the GPU.
"""
from __future__ import annotations

import os
import time
import warnings
from concurrent.futures import ThreadPoolExecutor
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np
import torch

from . import cie as _cie
from .cie import ContrastRecovery
from .filters import apply_cco  # noqa: F401  (filters.py:56-67, pdf_cco_image)
from .config import CcoParams, ImagingConfig
from .engine import DeviceProblem, check_config_supported
from .errors import PoleError, ZeroDataError  # noqa: F401  (re-exported)
from .geometry import AntennaArray, ComplexGrid, build_array, build_grid
from .metrics import count_components, relative_error, relative_error_dev  # noqa: F401  (GPU, reconstruct.py:243-254)
from .operators import GreensOperators, ScatteredData, build_greens, incident_fields

EPS_TV = 1e-12
SCALE_MIX, SCALE_FLOOR, OUTPUT_GAIN = 0.7, 0.1, 8.0


# ---------------------------------------------------------------------------- basis
@dataclass(frozen=True)
class SpectralBasis:
    """Corner-block index sets, TL/TR/BL/BR row-major (spectral.py:21-53)."""
    m1: int
    m2: int
    m_f: int
    rows: np.ndarray = field(init=False)
    cols: np.ndarray = field(init=False)

    def __post_init__(self):
        f = self.m_f
        if f < 1 or 2 * f > min(self.m1, self.m2):
            raise ValueError("corner blocks must not overlap: need 2*m_f <= min(m1, m2)")
        rsets = (np.arange(f), np.arange(self.m1 - f, self.m1))
        csets = (np.arange(f), np.arange(self.m2 - f, self.m2))
        r = np.concatenate([np.repeat(a, f) for a in rsets for _ in csets])
        c = np.concatenate([np.tile(b, f) for _ in rsets for b in csets])
        object.__setattr__(self, "rows", r)
        object.__setattr__(self, "cols", c)

    @property
    def m0(self) -> int:
        return 4 * self.m_f * self.m_f

    @property
    def n_cells(self) -> int:
        return self.m1 * self.m2


_BASIS_DEVS: dict = {}


def _basis_device(basis: SpectralBasis) -> DeviceProblem:
    """A geometry-free context for the spectral transforms of one basis."""
    from .engine import GRID_SIZES
    if basis.m1 != basis.m2 or basis.m1 not in GRID_SIZES:
        raise ValueError(f"the GPU transforms need a square grid with edge in {GRID_SIZES}, "
                         f"got ({basis.m1}, {basis.m2})")
    key = (basis.m1, basis.m_f)
    if key not in _BASIS_DEVS:
        M = basis.m1
        cfg = ImagingConfig(m1=M, m2=M, m_f=basis.m_f, n_tx=1, n_rx=1).validate()
        ops = build_greens(cfg, build_array(cfg), build_grid(cfg))
        _BASIS_DEVS[key] = DeviceProblem(ops, np.ones((1, M, M), complex), np.ones((1, 1), complex),
                                         mf=basis.m_f, beta=6.0, lambdas=(0, 0, 0), tau_b=0.5)
    return _BASIS_DEVS[key]


def truncate(basis: SpectralBasis, j_view) -> np.ndarray:
    """Corner-block DFT coefficients, (..., m1, m2) -> (..., m0), forward DFT
    unnormalised (spectral.py:56-65); computed by pdf_truncate."""
    j_view = np.asarray(j_view)
    if j_view.shape[-2:] != (basis.m1, basis.m2):
        raise ValueError(f"expected trailing dims ({basis.m1}, {basis.m2})")
    dev = _basis_device(basis)
    return dev.truncate(_cdev(j_view, dev)).cpu().numpy()


def expand(basis: SpectralBasis, alpha) -> np.ndarray:
    """Image(s) whose DFT is alpha on the corner blocks, zero elsewhere, inverse
    DFT carrying 1/(m1 m2) (spectral.py:68-79); computed by pdf_expand."""
    alpha = np.asarray(alpha, dtype=np.complex128)
    if alpha.shape[-1] != basis.m0:
        raise ValueError(f"expected trailing dim {basis.m0}")
    dev = _basis_device(basis)
    return dev.expand(_cdev(alpha, dev)).cpu().numpy()


def truncate_adjoint_scale(basis: SpectralBasis) -> float:
    """<expand(a), x> = c <a, truncate(x)> with c = 1/(m1 m2) (spectral.py:82-87)."""
    return 1.0 / (basis.m1 * basis.m2)


def _ops_device(ops: GreensOperators) -> DeviceProblem:
    views = np.ones((1, ops.m1, ops.m2), complex)
    return _ONE_SHOT.get(("ops", id(ops)), (ops,),
                         lambda: DeviceProblem(ops, views, np.ones((1, ops.n_rx), complex), mf=1, beta=6.0,
                                               lambdas=(0, 0, 0), tau_b=0.5))


def apply_gd(ops: GreensOperators, x) -> np.ndarray:
    """G_D on (..., m1, m2) images (forward.py:140-146): pdf_apply_gd, one
    zero-padded FFT convolution per image."""
    x = np.asarray(x)
    if x.shape[-2:] != (ops.m1, ops.m2):
        raise ValueError(f"expected trailing dims ({ops.m1}, {ops.m2})")
    dev = _ops_device(ops)
    return dev.apply_gd(_cdev(x, dev)).cpu().numpy()


def apply_gd_adjoint(ops: GreensOperators, x) -> np.ndarray:
    """G_D^H (forward.py:149-151)."""
    x = np.asarray(x)
    if x.shape[-2:] != (ops.m1, ops.m2):
        raise ValueError(f"expected trailing dims ({ops.m1}, {ops.m2})")
    dev = _ops_device(ops)
    return dev.apply_gd(_cdev(x, dev), adjoint=True).cpu().numpy()


def apply_gs_adjoint(ops: GreensOperators, rows) -> np.ndarray:
    """G_S^H on receiver vectors, (..., n_rx) -> (..., m1, m2) (forward.py:303-306)."""
    rows = np.asarray(rows)
    if rows.shape[-1] != ops.n_rx:
        raise ValueError(f"expected trailing dim {ops.n_rx}")
    dev = _ops_device(ops)
    return dev.gs_adjoint(_cdev(rows, dev)).cpu().numpy()


# ---------------------------------------------------------------------------- losses
@dataclass(frozen=True)
class LossBreakdown:
    total: float
    state: float
    data: float
    bound: float
    tv: float
    bridge: float
    weights: tuple

    def as_row(self) -> tuple:
        return (self.state, self.data, self.bound, self.tv, self.bridge, self.total)

    @classmethod
    def from_row(cls, row, weights) -> "LossBreakdown":
        st, da, bo, tv, br, tot = (float(x) for x in row)
        return cls(total=tot, state=st, data=da, bound=bo, tv=tv, bridge=br, weights=tuple(weights))


class LossTrace(Sequence):
    """Per-iteration LossBreakdown rows (reconstruct.py:217-220) backed by the
    float64 trace array copied from the device; entries are built on access,
    so a 500-iteration result costs no Python objects until it is read."""

    def __init__(self, rows: np.ndarray, weights):
        self._rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 6)
        self._w = tuple(weights)

    def __len__(self) -> int:
        return self._rows.shape[0]

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        st, da, bo, tv, br, tot = self._rows[i].tolist()
        return LossBreakdown(total=tot, state=st, data=da, bound=bo, tv=tv, bridge=br, weights=self._w)

    def __eq__(self, other) -> bool:
        return list(self) == list(other)

    def as_array(self) -> np.ndarray:
        """[k][6] rows in as_row() order (state, data, bound, tv, bridge, total)."""
        return self._rows.copy()


@dataclass
class LossContext:
    """Everything a loss evaluation needs besides the coefficients (losses.py:52-80).

    The first GPU call uploads operators and data into a cached DeviceProblem."""
    data: ScatteredData
    e_inc: np.ndarray
    ops: GreensOperators
    basis: SpectralBasis
    beta: float
    lambdas: tuple
    tau_b: float
    r_fixed: np.ndarray | None = None
    c_sca: float = 0.0
    c_inc: float = 0.0

    def __post_init__(self):
        mat = self.data.matrix if self.data.mask is None else self.data.matrix * self.data.mask
        self.c_sca = float(np.vdot(mat, mat).real)
        self.c_inc = float(np.vdot(self.e_inc, self.e_inc).real)
        if self.c_sca <= 0:
            raise ZeroDataError("measured scattered power is zero")
        if self.c_inc <= 0:
            raise ZeroDataError("incident power is zero")
        self._dev = {}

    @property
    def n_views(self) -> int:
        return self.e_inc.shape[0]

    def device(self, joint: bool = False) -> DeviceProblem:
        key = bool(joint)
        if key not in self._dev:
            self._dev[key] = DeviceProblem(
                self.ops, self.e_inc, self.data.matrix, mf=self.basis.m_f, beta=self.beta,
                lambdas=self.lambdas, tau_b=self.tau_b, mask=self.data.mask, r_fixed=self.r_fixed,
                joint=joint)
        return self._dev[key]


@dataclass
class PipelineState:
    """Intermediates of one composite-loss evaluation (losses.py:200-212), same fields.

    The loss itself comes from the fused library kernels (pdf_loss_value); the
    intermediates are assembled on the device from the library's operator
    primitives (expand, G_D, G_S) and copied to the host once."""
    alpha_hat: np.ndarray      # (n, m0)
    rec: ContrastRecovery
    r_hat: np.ndarray          # (m1, m2)
    p_views: np.ndarray        # (n, m1, m2) E + beta J
    state_res: np.ndarray      # (n, m1, m2)
    data_res: np.ndarray       # (n, n_rx), masked
    breakdown: LossBreakdown

    @property
    def chi(self) -> np.ndarray:
        return self.rec.chi


def _cdev(x, dev: DeviceProblem):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dev.cdt, device=dev.device)


def _recovery_dev(dev: DeviceProblem, alpha_d: torch.Tensor, eps_reg: float | None = None):
    """(J, E, num, den, eps, chi) of cie.py:66-99 on the device for one scene's views
    (alpha_d: (n, m0)): the library's expand and G_D, then pdf_cie_fields,
    pdf_default_eps_reg and pdf_pixel_ls."""
    j = dev.expand(alpha_d)
    einc = dev.e_inc if dev.e_inc.dim() == 3 else dev.e_inc[0]
    (e,) = _cie.cie_fields_dev(j, einc, gdj=dev.apply_gd(j), want=("e",))
    eps = _cie.default_eps_reg_dev(e) if eps_reg is None else torch.tensor(float(eps_reg), dtype=dev.rdt,
                                                                            device=dev.device)
    num, den, chi, _ = _cie.pixel_ls_dev(j, e, eps)
    return j, e, num, den, eps, chi


def _recovery_host(j, e, num, den, eps, chi) -> ContrastRecovery:
    epsf = float(eps)
    den_h = den.cpu().numpy()
    return ContrastRecovery(chi=chi.cpu().numpy(), j_views=j.cpu().numpy(), e_views=e.cpu().numpy(),
                            numerator=num.cpu().numpy(), denominator=den_h, eps_reg=epsf,
                            degenerate=den_h <= 10.0 * epsf)


def pipeline_forward(alpha_hat: np.ndarray, ctx: LossContext) -> PipelineState:
    alpha_hat = np.atleast_2d(np.asarray(alpha_hat, dtype=np.complex128))
    if alpha_hat.shape != (ctx.n_views, ctx.basis.m0):
        raise ValueError("need one coefficient vector per incidence view")
    dev = ctx.device()
    a = _cdev(alpha_hat[None], dev)
    bd, _ = dev.loss_value(a)
    dev.check_errors()           # PoleError / FloatingPointError (named terms) as the reference raises them
    j, e, num, den, eps, chi = _recovery_dev(dev, a[0])
    beta = ctx.beta
    r_hat = dev.r_fixed[0] if dev.r_fixed is not None else _cie.chi_to_r_dev(chi, beta)
    p, sres = _cie.cie_fields_dev(j, e, beta, r_hat=r_hat, want=("p", "res"))
    dres = _cie.masked_residual_dev(dev.gs_forward(j), dev.data[0], None if dev.mask is None else dev.mask[0])
    return PipelineState(alpha_hat=alpha_hat, rec=_recovery_host(j, e, num, den, eps, chi),
                         r_hat=r_hat.cpu().numpy(), p_views=p.cpu().numpy(), state_res=sres.cpu().numpy(),
                         data_res=dres.cpu().numpy(),
                         breakdown=LossBreakdown.from_row(bd[0].cpu().numpy(), ctx.lambdas))


def pipeline_backward(state: PipelineState, ctx: LossContext) -> np.ndarray:
    """g_alpha at state.alpha_hat (losses.py:267-306).  The library's fused
    kernels run the forward and the hand adjoint in one pass (the forward
    intermediates never leave the SM), so the state only supplies alpha_hat."""
    g, _ = grad_alpha(state.alpha_hat, ctx)
    return g


def grad_alpha(alpha: np.ndarray, ctx: LossContext) -> tuple[np.ndarray, LossBreakdown]:
    alpha = np.atleast_2d(np.asarray(alpha, dtype=np.complex128))
    if alpha.shape != (ctx.n_views, ctx.basis.m0):
        raise ValueError("need one coefficient vector per incidence view")
    dev = ctx.device()
    g, bd = dev.loss_grad(_cdev(alpha[None], dev))
    dev.check_errors()
    return g[0].cpu().numpy(), LossBreakdown.from_row(bd[0].cpu().numpy(), ctx.lambdas)


def loss_total(alpha: np.ndarray, ctx: LossContext) -> LossBreakdown:
    return pipeline_forward(alpha, ctx).breakdown


# ---------------------------------------------------------------------------- network
class PhysicsLoss(torch.autograd.Function):
    """The PDF physics loss as a differentiable torch op: the
    per-scene total of losses.py:215-247 for spectral coefficients alpha_hat
    (S, n, M0) complex on a DeviceProblem, with the hand adjoint of
    losses.py:267-306 as its backward.  The fused kernel computes loss and
    gradient in one pass, so the gradient is produced eagerly in forward and
    scaled by the incoming gradient in backward.  torch's complex gradient
    convention (dL/dRe + i dL/dIm) is the reference's (losses.py:255-264).

        loss = PhysicsLoss.apply(alpha_hat, dev)   # (S,) float64
        loss.sum().backward()                       # -> alpha_hat.grad
    """

    @staticmethod
    def forward(ctx, alpha_hat, dev):
        g, bd = dev.loss_grad(alpha_hat.detach())
        dev.check_errors()
        ctx.save_for_backward(g.clone())
        return bd[:, 5].clone()

    @staticmethod
    def backward(ctx, grad_out):
        (g,) = ctx.saved_tensors
        return g * grad_out.to(g.real.dtype)[:, None, None], None


@dataclass
class NetworkParams:
    weights: list
    biases: list

    @property
    def in_dim(self) -> int:
        return self.weights[0].shape[1]

    def n_params(self) -> int:
        return sum(w.size for w in self.weights) + sum(b.size for b in self.biases)


def init_network(m0: int, rng: np.random.Generator) -> NetworkParams:
    """Same draws as the reference (network.py:53-71): N(0, 1/fan_in), zero output layer."""
    if m0 < 1:
        raise ValueError("m0 must be >= 1")
    dims = (2 * m0, 4 * m0, 4 * m0, 2 * m0)
    ws, bs = [], []
    for li, (fi, fo) in enumerate(zip(dims[:-1], dims[1:])):
        ws.append(np.zeros((fo, fi)) if li == 2 else rng.normal(0.0, np.sqrt(1.0 / fi), (fo, fi)))
        bs.append(np.zeros(fo))
    return NetworkParams(weights=ws, biases=bs)


def flatten_params(params: NetworkParams) -> np.ndarray:
    return np.concatenate([a.ravel() for w, b in zip(params.weights, params.biases) for a in (w, b)])


def unflatten_params(flat: np.ndarray, like: NetworkParams) -> NetworkParams:
    ws, bs, k = [], [], 0
    for w, b in zip(like.weights, like.biases):
        ws.append(flat[k:k + w.size].reshape(w.shape).copy())
        k += w.size
        bs.append(flat[k:k + b.size].copy())
        k += b.size
    if k != flat.size:
        raise ValueError("flat parameter vector has the wrong length")
    return NetworkParams(weights=ws, biases=bs)


_NET_DEVS: dict = {}


def _net_device(n: int, m_f: int, joint: bool) -> DeviceProblem:
    """A geometry-free context just large enough to run the network kernels."""
    key = (n, m_f, joint)
    if key not in _NET_DEVS:
        M = 16
        while M < 2 * m_f:
            M *= 2
        cfg = ImagingConfig(m1=M, m2=M, m_f=m_f, n_tx=n, n_rx=1).validate()
        grid, arr = build_grid(cfg), build_array(cfg)
        ops = build_greens(cfg, arr, grid)
        _NET_DEVS[key] = DeviceProblem(ops, np.ones((n, M, M), complex), np.ones((n, 1), complex), mf=m_f,
                                       beta=cfg.beta, lambdas=(0, 0, 0), tau_b=0.5, joint=joint)
    return _NET_DEVS[key]


def _net_device_lr(n: int, m_f: int, lr: float) -> DeviceProblem:
    """As _net_device (non-joint), with the learning rate its Adam applies."""
    key = (n, m_f, False, float(lr))
    if key not in _NET_DEVS:
        M = 16
        while M < 2 * m_f:
            M *= 2
        cfg = ImagingConfig(m1=M, m2=M, m_f=m_f, n_tx=n, n_rx=1).validate()
        ops = build_greens(cfg, build_array(cfg), build_grid(cfg))
        _NET_DEVS[key] = DeviceProblem(ops, np.ones((n, M, M), complex), np.ones((n, 1), complex), mf=m_f,
                                       beta=cfg.beta, lambdas=(0, 0, 0), tau_b=0.5, lr=float(lr))
    return _NET_DEVS[key]


def _theta(params: NetworkParams, dev: DeviceProblem) -> torch.Tensor:
    return torch.as_tensor(flatten_params(params), dtype=dev.rdt, device=dev.device)[None].contiguous()


def forward_net(params: NetworkParams, alpha0: np.ndarray, joint: bool = False) -> np.ndarray:
    """Corrective update delta-alpha (network.py:143-150), on the GPU."""
    alpha0 = np.atleast_2d(np.asarray(alpha0, dtype=np.complex128))
    n, m0 = alpha0.shape
    width = 2 * (alpha0.size if joint else m0)
    if params.in_dim != width:
        raise ValueError(f"network expects input width {params.in_dim}, got {width}")
    mf = int(round(np.sqrt(m0 / 4)))
    if 4 * mf * mf != m0:
        raise ValueError("coefficient length must be 4*m_f**2")
    dev = _net_device(n, mf, joint)
    a0 = _cdev(alpha0[None], dev)
    dev.net_setup(a0)
    out = dev.net_forward(_theta(params, dev))
    return (out - a0)[0].cpu().numpy()


def grad_loss(params: NetworkParams, alpha0: np.ndarray, ctx: LossContext,
              joint: bool = False) -> tuple[np.ndarray, LossBreakdown]:
    """Exact gradient over the flat parameters (network.py:183-223)."""
    alpha0 = np.atleast_2d(np.asarray(alpha0, dtype=np.complex128))
    width = 2 * (alpha0.size if joint else alpha0.shape[1])
    if params.in_dim != width:
        raise ValueError(f"network expects input width {params.in_dim}, got {width}")
    dev = ctx.device(joint)
    dev.net_setup(_cdev(alpha0[None], dev))
    g, bd = dev.grad_loss(_theta(params, dev))
    dev.check_errors()
    return g[0].cpu().numpy().astype(np.float64), LossBreakdown.from_row(bd[0].cpu().numpy(), ctx.lambdas)


@dataclass
class AdamState:
    m: np.ndarray
    v: np.ndarray
    step: int = 0
    lr: float = 1e-2
    b1: float = 0.9
    b2: float = 0.999
    eps: float = 1e-8

    @classmethod
    def for_params(cls, params: NetworkParams, lr: float = 1e-2) -> "AdamState":
        n = params.n_params()
        return cls(m=np.zeros(n), v=np.zeros(n), lr=lr)


def adam_step(state: AdamState, params: NetworkParams, grad: np.ndarray) -> tuple[NetworkParams, AdamState]:
    """One bias-corrected Adam update on the GPU (network.py:248-264)."""
    flat = flatten_params(params)
    if grad.shape != flat.shape:
        raise ValueError("gradient length does not match parameter count")
    dev = _adam_device(state.lr, state.b1, state.b2, state.eps)
    t = state.step + 1
    to = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev.device).clone()  # noqa
    p, m, v, g = to(flat), to(state.m), to(state.v), to(grad)
    dev.adam_step(p, m, v, g, t)
    dev.check_errors()
    new = AdamState(m=m.cpu().numpy(), v=v.cpu().numpy(), step=t, lr=state.lr, b1=state.b1, b2=state.b2,
                    eps=state.eps)
    return unflatten_params(p.cpu().numpy(), params), new


_ADAM_DEVS: dict = {}


def _adam_device(lr: float, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8) -> DeviceProblem:
    key = (float(lr), float(b1), float(b2), float(eps))
    if key not in _ADAM_DEVS:
        cfg = ImagingConfig(m1=16, m2=16, m_f=1, n_tx=1, n_rx=1, learn_rate=lr).validate()
        ops = build_greens(cfg, build_array(cfg), build_grid(cfg))
        _ADAM_DEVS[key] = DeviceProblem(ops, np.ones((1, 16, 16), complex), np.ones((1, 1), complex), mf=1,
                                        beta=6.0, lambdas=(0, 0, 0), tau_b=0.5, lr=lr, adam_b1=b1, adam_b2=b2,
                                        adam_eps=eps)
    return _ADAM_DEVS[key]


# ---------------------------------------------------------------------------- pipeline
@dataclass
class ReconstructionResult:
    chi_hat: ComplexGrid
    chi_cco: ComplexGrid
    chi0: ComplexGrid
    trace: list
    final_loss: LossBreakdown
    wall_time: float
    rel_error: float | None = None

    @property
    def eps_r(self) -> np.ndarray:
        return self.chi_cco.values + 1.0


def _theta0(seeds, m0_eff: int) -> np.ndarray:
    """Reference-identical initial weights per scene (numpy PCG64 draws on the host cores)."""
    out = np.empty((len(seeds), _flat_size(m0_eff)))
    for f in _theta0_async(seeds, m0_eff, out):
        f.result()
    return out


_THETA_POOL = None


def _flat_size(m0_eff: int) -> int:
    d0 = 2 * m0_eff
    h = 2 * d0
    return h * d0 + h + h * h + h + d0 * h + d0


def init_flat_into(row: np.ndarray, m0_eff: int, seed: int) -> None:
    """flatten_params(init_network(m0_eff, default_rng(seed))) written straight
    into `row` (network.py:53-71): Generator.normal(0, s) is s * standard_normal
    draw for draw, so the standard normals are drawn into the weight slices in
    the reference's order (w1, then w2; w3 and the biases are zero)."""
    rng = np.random.default_rng(int(seed))
    d0 = 2 * m0_eff
    h = 2 * d0
    o = 0
    for fi, fo, zero in ((d0, h, False), (h, h, False), (h, d0, True)):
        w = row[o:o + fo * fi].reshape(fo, fi)
        if zero:
            w.fill(0.0)
        else:
            rng.standard_normal(out=w)
            w *= np.sqrt(1.0 / fi)
        o += fo * fi
        row[o:o + fo] = 0.0
        o += fo


def _theta0_async(seeds, m0_eff: int, out: np.ndarray, workers: int | None = None):
    """Start the per-scene draws of _theta0 into `out` rows (all host cores); returns futures."""
    global _THETA_POOL
    if _THETA_POOL is None:
        _THETA_POOL = ThreadPoolExecutor(max_workers=workers or min(32, os.cpu_count() or 8))
    return [_THETA_POOL.submit(init_flat_into, out[i], m0_eff, s) for i, s in enumerate(seeds)]


class BatchReconstructor:
    """Reconstruct S scenes that share one geometry, all resident on one GPU.

    This is the B200 form of the reference's reconstruct() (reconstruct.py:186-236):
    bp_initialize + init_alpha, then k fused {grad_loss, trace, Adam} iterations
    replayed from a CUDA graph, then forward_net + loss_total + recover_contrast
    + apply_cco.  Scenes are independent (config 4 shards them over GPUs).
    """

    def __init__(self, config: ImagingConfig, S: int, e_inc: np.ndarray | None = None,
                 array: AntennaArray | None = None, mask=None, dtype: str = "f64", use_graph: bool = True,
                 theta_cache: bool = True, device_ops: bool = True):
        config.validate()
        check_config_supported(config)
        self.config = config
        self.array = build_array(config) if array is None else array
        self.grid = build_grid(config)
        if device_ops:
            # operators and incident fields built in HBM by the library (greens.py)
            from .greens import build_greens_device, incident_fields_device
            self.ops = build_greens_device(config, self.array, self.grid)
            self.e_inc = (incident_fields_device(config, self.array, self.grid, "line") if e_inc is None
                          else np.asarray(e_inc))
        else:
            self.ops = build_greens(config, self.array, self.grid)
            self.e_inc = incident_fields(config, self.array, self.grid).views if e_inc is None else np.asarray(e_inc)
        self.basis = SpectralBasis(config.m1, config.m2, config.m_f)
        self.S = S
        self.use_graph = use_graph
        # initial weights are a pure function of (seed, width) -- the reference
        # redraws the same numbers from default_rng(config.rng_seed) on every
        # call -- so they are memoised per seed tuple like the operators
        self.theta_cache = theta_cache
        self._theta0 = {}
        self.mask = mask
        self.lambdas = (config.lambda1, config.lambda2, config.lambda3)
        placeholder = np.ones((S, self.e_inc.shape[0], self.array.n_rx), complex)
        self.dev = DeviceProblem(self.ops, self.e_inc, placeholder, mf=config.m_f, beta=config.beta,
                                 lambdas=self.lambdas, tau_b=config.tau_b, mask=mask, joint=config.joint_views,
                                 lr=config.learn_rate, dtype=dtype)
        self.m0_eff = self.basis.m0 * (self.e_inc.shape[0] if config.joint_views else 1)

    def _initialise(self):
        """bp_initialize + init_alpha + net_setup (reconstruct.py:52-153, network.py:88-104)
        on the current data: ~70 small launches, replayed from a CUDA graph
        captured on the first call (the data and normalisers are updated in
        place by set_data, so the graph stays valid)."""
        dev = self.dev
        if not self.use_graph:
            chi0, r0 = dev.bp_initialize(check=False)
            alpha0 = dev.init_alpha(r0, check=False)
            dev.net_setup(alpha0)
            return chi0, alpha0
        if getattr(self, "_init_graph", None) is None:
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):            # warm-up outside the capture
                chi0, r0 = dev.bp_initialize(check=False)
                dev.net_setup(dev.init_alpha(r0, check=False))
            torch.cuda.current_stream().wait_stream(st)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                chi0, r0 = dev.bp_initialize(check=False)
                alpha0 = dev.init_alpha(r0, check=False)
                dev.net_setup(alpha0)
            self._init_graph, self._init_out = g, (chi0, alpha0)
        self._init_graph.replay()
        return self._init_out

    def _pinned(self, slot: int) -> torch.Tensor:
        """Two page-locked host buffers for the initial weights, reused across runs."""
        bufs = self.__dict__.setdefault("_host_bufs", [None, None])
        if bufs[slot] is None:
            bufs[slot] = torch.empty((self.S, _flat_size(self.m0_eff)), dtype=torch.float64, pin_memory=True)
        return bufs[slot]

    def run(self, datas, seeds=None, chi_trues=None, k_iters: int | None = None, prefetch_seeds=None,
            check_init: bool = False) -> list:
        """Reconstruct the S scenes of `datas` (see the class docstring).

        prefetch_seeds: seeds of the NEXT batch; its reference-identical
        initial weights are drawn on the host cores while this batch trains on
        the GPU (a batch pipeline pays the draws only once, up front).
        check_init: raise the initialisation's PoleError before the training
        loop starts, as the reference does (one host synchronisation);
        otherwise it is raised after the loop (no synchronisation before it)."""
        cfg = self.config
        t0 = time.perf_counter()
        mats = np.stack([np.asarray(d.matrix if isinstance(d, ScatteredData) else d) for d in datas])
        if mats.shape != (self.S, self.e_inc.shape[0], self.array.n_rx):
            raise ValueError("data matrix does not match the antenna array")
        seeds = [cfg.rng_seed] * self.S if seeds is None else list(seeds)
        k = cfg.k_iters if k_iters is None else k_iters
        dev = self.dev
        if cfg.freeze_r:
            raise NotImplementedError("freeze_r with BatchReconstructor: build DeviceProblem(r_fixed=...)")
        key = tuple(int(x) for x in seeds)
        theta0 = self._theta0.get(key)
        pending = None
        pre = getattr(self, "_prefetch", None)
        self._prefetch = None
        if pre is not None and pre[0] != key:      # stale prefetch: let it finish before its buffer is reused
            for f in pre[2]:
                f.result()
        if theta0 is None:
            # the reference-identical initial weights are host RNG draws: fill a
            # pinned buffer on worker threads while the GPU runs the initialisation
            # (or use the draws a previous run started for these seeds)
            if pre is not None and pre[0] == key:
                _, slot, pending = pre
            else:
                slot = 0 if pre is None else 1 - pre[1]
                pending = _theta0_async(seeds, self.m0_eff, self._pinned(slot).numpy())
        # persistent device state (theta, Adam moments, trace) for this batch shape
        bufs = self.__dict__.get("_dev_bufs")
        if bufs is None or bufs[3].shape[0] < max(k, 1):
            n_par = _flat_size(self.m0_eff)
            # theta, m, v in one allocation: the library keeps that window L2-resident
            flat = torch.empty((3, self.S, n_par), dtype=dev.rdt, device=dev.device)
            bufs = [flat[0], flat[1], flat[2]]
            bufs.append(torch.empty((max(k, 1), self.S, 6), dtype=torch.float64, device=dev.device))
            self._dev_bufs = bufs
        theta, m, v, trace_buf = bufs
        trace = trace_buf[:max(k, 1)]
        # initial weights already drawn (a prefetch): their upload runs on a copy stream
        # while the GPU runs the initialisation
        early = pending is not None and all(f.done() for f in pending)
        if early:
            cs = self.__dict__.setdefault("_copy_stream", torch.cuda.Stream(device=dev.device))
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                theta.copy_(self._pinned(slot), non_blocking=True)
            up_done = torch.cuda.Event()
            up_done.record(cs)
        dev.set_data(mats)
        chi0, alpha0 = self._initialise()
        if check_init and bool(dev.pole_flag):
            for f in pending or ():
                f.result()       # the pinned buffer must be idle before a later run reuses it
            raise PoleError("beta*chi + 1 vanishes at some pixel")
        if pending is not None:
            if early:
                torch.cuda.current_stream().wait_event(up_done)
            else:
                for f in pending:
                    f.result()
                theta.copy_(self._pinned(slot), non_blocking=True)
            if self.theta_cache:
                self._theta0 = {key: theta.clone()}
        else:
            theta.copy_(theta0)
        m.zero_()
        v.zero_()
        trace.zero_()
        if k:
            dev.train(theta, m, v, 0, k, trace, use_graph=self.use_graph)
        if prefetch_seeds is not None and len(prefetch_seeds) == self.S:
            nkey = tuple(int(x) for x in prefetch_seeds)
            if nkey not in self._theta0:
                nslot = 1 - slot if pending is not None else 0
                self._prefetch = (nkey, nslot, _theta0_async(list(nkey), self.m0_eff, self._pinned(nslot).numpy()))
        ahat = dev.net_forward(theta)
        bd, chi = dev.loss_value(ahat, want_chi=True)
        chi_cco = dev.apply_cco(chi, cfg.cco) if cfg.use_cco else chi.clone()
        rels = None
        if chi_trues is not None and any(c is not None for c in chi_trues):
            # relative_error(chi_cco.real + 1, chi_true.real + 1) of every scene in one device reduction
            tr_h = np.zeros((self.S, self.config.m1, self.config.m2), complex)
            for s_, c in enumerate(chi_trues):
                if c is not None:
                    tr_h[s_] = c.values if isinstance(c, ComplexGrid) else c
            rels = relative_error_dev(chi_cco, torch.as_tensor(tr_h, device=dev.device), offset=1.0)
        if bool(dev.pole_flag):     # deferred checks of the initialisation (no host sync before the loop)
            raise PoleError("beta*chi + 1 vanishes at some pixel")
        if bool(dev.zero_grad_flag):
            warnings.warn("zero initial gradient; starting from zero coefficients")
        dev.check_errors()
        chi0_h, chi_h, cco_h = chi0.cpu().numpy(), chi.cpu().numpy(), chi_cco.cpu().numpy()
        tr_h, bd_h = trace.cpu().numpy(), bd.cpu().numpy()
        rel_h = rels.cpu().numpy() if rels is not None else None
        wall = time.perf_counter() - t0
        out = []
        cs = self.grid.cell_size
        for s in range(self.S):
            rel = None
            if rel_h is not None and chi_trues[s] is not None:
                rel = float(rel_h[s])
            out.append(ReconstructionResult(
                chi_hat=ComplexGrid(chi_h[s], cs), chi_cco=ComplexGrid(cco_h[s], cs),
                chi0=ComplexGrid(chi0_h[s], cs),
                trace=LossTrace(tr_h[:k, s], self.lambdas),
                final_loss=LossBreakdown.from_row(bd_h[s], self.lambdas), wall_time=wall, rel_error=rel))
        return out


def reconstruct(config: ImagingConfig, data: ScatteredData, array: AntennaArray | None = None,
                chi_true: ComplexGrid | None = None, *, e_inc: np.ndarray | None = None,
                dtype: str = "f64") -> ReconstructionResult:
    """Full pipeline from measured data to a permittivity map (reconstruct.py:186-236).

    ``e_inc`` overrides the reference's line-source illumination (e.g. plane
    waves for the BASELINE configs); everything else follows the reference."""
    config.validate()
    check_config_supported(config)
    t0 = time.perf_counter()
    if config.freeze_r:
        return _reconstruct_frozen(config, data, array, chi_true, e_inc, dtype, t0)
    rec = BatchReconstructor(config, 1, e_inc=e_inc, array=array, mask=data.mask, dtype=dtype)
    res = rec.run([data], chi_trues=[chi_true], check_init=True)[0]
    res.wall_time = time.perf_counter() - t0
    return res


def _reconstruct_frozen(config, data, array, chi_true, e_inc, dtype, t0):
    array = build_array(config) if array is None else array
    grid = build_grid(config)
    ops = build_greens(config, array, grid)
    e_inc = incident_fields(config, array, grid).views if e_inc is None else np.asarray(e_inc)
    lambdas = (config.lambda1, config.lambda2, config.lambda3)
    probe = DeviceProblem(ops, e_inc, data.matrix, mf=config.m_f, beta=config.beta, lambdas=lambdas,
                          tau_b=config.tau_b, mask=data.mask, lr=config.learn_rate, dtype=dtype)
    chi0, r0 = probe.bp_initialize()
    alpha0 = probe.init_alpha(r0)
    dev = DeviceProblem(ops, e_inc, data.matrix, mf=config.m_f, beta=config.beta, lambdas=lambdas,
                        tau_b=config.tau_b, mask=data.mask, r_fixed=r0[0].cpu().numpy(),
                        joint=config.joint_views, lr=config.learn_rate, dtype=dtype)
    dev.net_setup(alpha0)
    m0_eff = 4 * config.m_f ** 2 * (e_inc.shape[0] if config.joint_views else 1)
    theta = torch.as_tensor(_theta0([config.rng_seed], m0_eff), dtype=dev.rdt, device=dev.device).contiguous()
    m, v = torch.zeros_like(theta), torch.zeros_like(theta)
    k = config.k_iters
    trace = torch.zeros(max(k, 1), 1, 6, dtype=torch.float64, device=dev.device)
    if k:
        dev.train(theta, m, v, 0, k, trace)
    ahat = dev.net_forward(theta)
    bd, _ = dev.loss_value(ahat)
    # recover_contrast is evaluated with the (non-frozen) LS map, as the reference does
    _, chi = probe.loss_value(ahat, want_chi=True)
    chi_cco = probe.apply_cco(chi, config.cco) if config.use_cco else chi.clone()
    dev.check_errors()
    lam = lambdas
    cs = grid.cell_size
    rel = None
    cco_h = chi_cco[0].cpu().numpy()
    if chi_true is not None:
        rel = float(relative_error_dev(chi_cco[0], torch.as_tensor(chi_true.values, device=dev.device),
                                       offset=1.0)[0].item())
    tr = trace.cpu().numpy()
    return ReconstructionResult(chi_hat=ComplexGrid(chi[0].cpu().numpy(), cs), chi_cco=ComplexGrid(cco_h, cs),
                                chi0=ComplexGrid(chi0[0].cpu().numpy(), cs),
                                trace=LossTrace(tr[:k, 0], lam),
                                final_loss=LossBreakdown.from_row(bd[0].cpu().numpy(), lam),
                                wall_time=time.perf_counter() - t0, rel_error=rel)


class _DevCache:
    """Small LRU of DeviceProblems for the one-shot API functions (bp_initialize,
    init_alpha, recover_contrast, apply_cco): operators and workspace are
    uploaded once per (operators, incident fields, data) identity.  The cache
    holds references to the keyed host arrays, so an id is never reused while
    its entry lives; like the reference's functions it treats inputs as
    immutable."""

    def __init__(self, size: int = 4):
        self.size = size
        self.items: list = []

    def get(self, key, objs, make):
        for i, (k, o, dev) in enumerate(self.items):
            if k == key and all(a is b for a, b in zip(o, objs)):
                self.items.append(self.items.pop(i))
                return dev
        dev = make()
        self.items.append((key, objs, dev))
        if len(self.items) > self.size:
            self.items.pop(0)
        return dev


_ONE_SHOT = _DevCache()


def _one_shot_device(ops: GreensOperators, views, data: ScatteredData | None, m_f: int, beta: float,
                     n_rx: int | None = None) -> DeviceProblem:
    views = np.asarray(views)
    mat = data.matrix if data is not None else None
    mask = data.mask if data is not None else None
    key = (id(ops), id(views), id(mat), id(mask), m_f, float(beta))

    def make():
        d = mat if mat is not None else np.ones((views.shape[0], ops.n_rx if n_rx is None else n_rx), complex)
        return DeviceProblem(ops, views, d, mf=m_f, beta=beta, lambdas=(0, 0, 0), tau_b=0.5, mask=mask)
    return _ONE_SHOT.get(key, (ops, views, mat, mask), make)


def bp_initialize(data: ScatteredData, e_inc, ops: GreensOperators, beta: float):
    """Backprojection (reconstruct.py:52-71) on the GPU; returns host (chi0, r0)."""
    views = e_inc.views if hasattr(e_inc, "views") else np.asarray(e_inc)
    dev = _one_shot_device(ops, views, data, 1, beta)
    chi0, r0 = dev.bp_initialize()
    return chi0[0].cpu().numpy(), r0[0].cpu().numpy()


def init_alpha(r0, data: ScatteredData, e_inc, ops: GreensOperators, basis: SpectralBasis, beta: float):
    """Exact line-search initial coefficients (reconstruct.py:139-153) on the GPU."""
    views = e_inc.views if hasattr(e_inc, "views") else np.asarray(e_inc)
    dev = _one_shot_device(ops, views, data, basis.m_f, beta)
    a0 = dev.init_alpha(torch.as_tensor(np.asarray(r0)[None], dtype=dev.cdt, device=dev.device))
    return a0[0].cpu().numpy()


def recover_contrast(alpha, e_inc, ops: GreensOperators, basis: SpectralBasis, eps_reg: float | None = None,
                     full: bool = False):
    """Contrast implied by spectral coefficients (cie.py:83-99) on the GPU.

    full=True returns the ContrastRecovery record; eps_reg overrides the
    default floor 1e-10 max_i ||E_i||^2 / M^2 (cie.py:42-50)."""
    alpha = np.atleast_2d(np.asarray(alpha, dtype=np.complex128))
    views = e_inc.views if hasattr(e_inc, "views") else np.asarray(e_inc)
    if alpha.shape[0] != views.shape[0]:
        raise ValueError("need one coefficient vector per incidence view")
    dev = _one_shot_device(ops, views, None, basis.m_f, 6.0)
    a = _cdev(alpha[None], dev)
    if eps_reg is None and not full:
        _, chi = dev.loss_value(a, want_chi=True)     # the fused library path
        return chi[0].cpu().numpy()
    parts = _recovery_dev(dev, a[0], eps_reg)
    return _recovery_host(*parts) if full else parts[-1].cpu().numpy()


