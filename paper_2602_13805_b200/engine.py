"""Device-resident PDF problem: one geometry, S scenes, one C-ABI context.

PyTorch only provides device memory and the CUDA stream; every operator on
the hot path runs in libpdfb200.so through ``_native``.  The one-time
initialisation (bp_initialize / init_alpha, reconstruct.py:52-153) composes
the library's operator primitives with a few torch reductions on the device.
"""
from __future__ import annotations

import ctypes as ct
import warnings

import numpy as np
import torch

from . import _native as N
from .errors import PoleError, raise_for_bits


def _ptr(t: torch.Tensor | None):
    return None if t is None else ct.c_void_p(t.data_ptr())


def _stream():
    return ct.c_void_p(torch.cuda.current_stream().cuda_stream)


GRID_SIZES = (16, 32, 64, 128, 256)
MAX_VIEWS = 80
MAX_RECEIVERS = 80


def _shape(x) -> tuple:
    return tuple(x.shape) if hasattr(x, "shape") else tuple(np.shape(x))


def check_supported(ops, e_inc, data: np.ndarray, mf: int, joint: bool = False) -> None:
    """Reject, before any pointer reaches the C ABI, the problems the sm_100a
    kernels do not cover ('Supported shapes'): the grid
    must be square with a power-of-two edge in [16, 256], at most 80
    incidences and 80 receivers, and every operator must have the shape the
    grid implies.  The reference accepts any m1 x m2; there is no host path
    here, so an unsupported shape is a ValueError naming the limit."""
    if e_inc.ndim not in (3, 4):
        raise ValueError(f"e_inc must be (n, m1, m2) or (S, n, m1, m2), got shape {e_inc.shape}")
    m1, m2 = e_inc.shape[-2], e_inc.shape[-1]
    if m1 != m2:
        raise ValueError(f"unsupported grid {m1}x{m2}: the GPU path needs a square grid (m1 == m2)")
    M = m1
    if M not in GRID_SIZES:
        raise ValueError(f"unsupported grid {M}x{M}: the edge must be one of {GRID_SIZES}")
    if (ops.m1, ops.m2) != (M, M):
        raise ValueError(f"operators were built for a {ops.m1}x{ops.m2} grid, e_inc is {M}x{M}")
    if _shape(ops.gd_kernel_hat) != (2 * M, 2 * M):
        raise ValueError(f"gd_kernel_hat must be ({2 * M}, {2 * M}), got {_shape(ops.gd_kernel_hat)}")
    S, n, R = data.shape
    if _shape(ops.gs_matrix) != (R, M * M):
        raise ValueError(f"gs_matrix must be ({R}, {M * M}) for {R} receivers, got {_shape(ops.gs_matrix)}")
    if e_inc.shape[-3] != n:
        raise ValueError(f"e_inc has {e_inc.shape[-3]} views, the data {n}")
    if e_inc.ndim == 4 and e_inc.shape[0] != S:
        raise ValueError(f"per-scene e_inc has {e_inc.shape[0]} scenes, the data {S}")
    if n > MAX_VIEWS:
        raise ValueError(f"{n} incidences: the GPU path supports at most {MAX_VIEWS}")
    if R > MAX_RECEIVERS:
        raise ValueError(f"{R} receivers: the GPU path supports at most {MAX_RECEIVERS}")
    if mf < 1 or 2 * mf > M:
        raise ValueError(f"m_f = {mf}: need 1 <= m_f and 2 m_f <= {M}")


def check_config_supported(config) -> None:
    """check_supported() on an ImagingConfig, before any operator is built."""
    if config.m1 != config.m2:
        raise ValueError(f"unsupported grid {config.m1}x{config.m2}: the GPU path needs a square grid (m1 == m2)")
    if config.m1 not in GRID_SIZES:
        raise ValueError(f"unsupported grid {config.m1}x{config.m2}: the edge must be one of {GRID_SIZES}")
    if config.n_tx > MAX_VIEWS:
        raise ValueError(f"{config.n_tx} incidences: the GPU path supports at most {MAX_VIEWS}")
    if config.n_rx > MAX_RECEIVERS:
        raise ValueError(f"{config.n_rx} receivers: the GPU path supports at most {MAX_RECEIVERS}")


class DeviceProblem:
    """S scenes sharing one geometry, resident in HBM.

    e_inc: (n, M, M) shared or (S, n, M, M) per scene; data: (S, n, R);
    mask: (S, n, R) or None; r_fixed: (S, M, M) or None.
    """

    def __init__(self, ops, e_inc, data, *, mf: int, beta: float, lambdas, tau_b: float, mask=None,
                 r_fixed=None, joint: bool = False, lr: float = 1e-2, dtype: str = "f64",
                 device: str | torch.device = "cuda", adam_b1: float = 0.9, adam_b2: float = 0.999,
                 adam_eps: float = 1e-8):
        data = np.asarray(data)
        if data.ndim == 2:
            data = data[None]
        S, n, R = data.shape
        if not isinstance(e_inc, torch.Tensor):      # host array, or a device tensor (greens.py)
            e_inc = np.asarray(e_inc)
        shared = e_inc.ndim == 3
        M = e_inc.shape[-1]
        check_supported(ops, e_inc, data, mf, joint)    # before any device work
        if not torch.cuda.is_available():
            raise RuntimeError("the PDF hot path needs a CUDA device (no CPU fallback)")
        self.lib = N.lib()
        self.device = torch.device(device)
        self.rdt = torch.float64 if dtype == "f64" else torch.float32
        self.cdt = torch.complex128 if dtype == "f64" else torch.complex64
        self.S, self.n, self.R, self.M, self.mf = S, n, R, M, mf
        self.m0 = 4 * mf * mf
        self.beta, self.lambdas, self.tau_b = float(beta), tuple(float(x) for x in lambdas), float(tau_b)
        self.joint = bool(joint)
        dev = self.device
        cd = self.cdt
        self.e_inc = torch.as_tensor(e_inc, dtype=cd, device=dev).contiguous()
        self.khat = torch.as_tensor(ops.gd_kernel_hat, dtype=cd, device=dev).contiguous()
        self.gs = torch.as_tensor(ops.gs_matrix, dtype=cd, device=dev).contiguous()
        self.data = torch.as_tensor(data, dtype=cd, device=dev).contiguous()
        self.mask = None
        if mask is not None:
            mk = np.array(np.broadcast_to(np.asarray(mask, dtype=float), data.shape))
            self.mask = torch.as_tensor(mk, dtype=self.rdt, device=dev).contiguous()
        self.r_fixed = None
        if r_fixed is not None:
            rf = np.asarray(r_fixed)
            rf = np.array(np.broadcast_to(rf, (S, M, M)) if rf.ndim == 2 else rf)
            self.r_fixed = torch.as_tensor(rf, dtype=cd, device=dev).contiguous()
        # normalisers in float64 on the host, exactly as losses.py:67-76
        dm = data if mask is None else data * np.broadcast_to(np.asarray(mask, dtype=float), data.shape)
        self.c_sca = np.array([float(np.vdot(dm[s], dm[s]).real) for s in range(S)])
        if isinstance(e_inc, torch.Tensor):
            p2 = (self.e_inc.conj() * self.e_inc).real
            self.c_inc = np.full(S, float(p2.sum())) if shared else p2.reshape(S, -1).sum(-1).cpu().numpy()
        elif shared:
            ci = float(np.vdot(e_inc, e_inc).real)
            self.c_inc = np.full(S, ci)
        else:
            self.c_inc = np.array([float(np.vdot(e_inc[s], e_inc[s]).real) for s in range(S)])
        from .errors import ZeroDataError
        if np.any(self.c_sca <= 0):
            raise ZeroDataError("measured scattered power is zero")
        if np.any(self.c_inc <= 0):
            raise ZeroDataError("incident power is zero")
        self._c_inc_h = (ct.c_double * S)(*self.c_inc)
        self._c_sca_h = (ct.c_double * S)(*self.c_sca)
        d = N.PdfDesc()
        d.abi_version = N.ABI_VERSION
        d.dtype = N.PDF_F64 if dtype == "f64" else N.PDF_F32
        d.S, d.n, d.m1, d.m2, d.R, d.mf = S, n, M, M, R, mf
        d.joint, d.freeze_r = int(joint), int(r_fixed is not None)
        d.beta = self.beta
        d.lambda1, d.lambda2, d.lambda3 = self.lambdas
        d.tau_b = self.tau_b
        d.lr, d.adam_b1, d.adam_b2, d.adam_eps = float(lr), float(adam_b1), float(adam_b2), float(adam_eps)
        d.e_inc = self.e_inc.data_ptr()
        d.e_inc_scene_stride = 0 if shared else n * M * M
        d.gd_kernel_hat = self.khat.data_ptr()
        d.gs_matrix = self.gs.data_ptr()
        d.data = self.data.data_ptr()
        d.mask = self.mask.data_ptr() if self.mask is not None else None
        d.r_fixed = self.r_fixed.data_ptr() if self.r_fixed is not None else None
        d.c_inc = ct.cast(self._c_inc_h, ct.POINTER(ct.c_double))
        d.c_sca = ct.cast(self._c_sca_h, ct.POINTER(ct.c_double))
        self.desc = d
        nbytes = self.lib.pdf_workspace_bytes(ct.byref(d))
        if nbytes == 0:
            raise ValueError(f"unsupported problem: {self.lib.pdf_last_error().decode()}")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        h = ct.c_void_p()
        N.check(self.lib.pdf_ctx_create(ct.byref(d), _ptr(self.workspace), nbytes, _stream(), ct.byref(h)))
        self.ctx = h
        rows, d0, hid, npar = ct.c_int32(), ct.c_int32(), ct.c_int32(), ct.c_int64()
        N.check(self.lib.pdf_net_dims(self.ctx, ct.byref(rows), ct.byref(d0), ct.byref(hid), ct.byref(npar)))
        self.rows, self.d0, self.hidden, self.n_params = rows.value, d0.value, hid.value, npar.value
        self.c_inc_d = torch.as_tensor(np.asarray(self.c_inc, float), device=dev)
        self.c_sca_d = torch.as_tensor(np.asarray(self.c_sca, float), device=dev)
        paths = ct.c_int32()
        if hasattr(self.lib, "pdf_ctx_paths"):
            N.check(self.lib.pdf_ctx_paths(self.ctx, ct.byref(paths)))
        self.large_grid, self.data_gemm, self.split_bwd = (bool(paths.value & b) for b in (1, 2, 4))
        self.view_cluster = (paths.value >> 8) & 15   # CTAs per view of the cluster path (0: large-grid path)
        self.bd = torch.zeros(S, 6, dtype=torch.float64, device=dev)

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                self.lib.pdf_ctx_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    def paths(self) -> dict:
        """Kernel paths the library chose for this problem (pdf_ctx_paths)."""
        return {"large_grid": self.large_grid, "data_gemm": self.data_gemm, "split_bwd": self.split_bwd,
                "view_cluster": self.view_cluster}

    # ------------------------------------------------------------------ helpers
    def cplx(self, *shape):
        return torch.empty(*shape, dtype=self.cdt, device=self.device)

    def check_errors(self) -> None:
        err = (ct.c_int32 * self.S)()
        N.check(self.lib.pdf_get_error(self.ctx, err, _stream()))
        bits = [int(x) for x in err]
        if any(bits):
            raise_for_bits(bits)

    # ------------------------------------------------------------------ physics
    def loss_grad(self, alpha: torch.Tensor, g_alpha: torch.Tensor | None = None):
        alpha = alpha.to(self.cdt).contiguous()
        g = self.cplx(self.S, self.n, self.m0) if g_alpha is None else g_alpha
        N.check(self.lib.pdf_loss_grad(self.ctx, _ptr(alpha), _ptr(g), _ptr(self.bd), _stream()))
        return g, self.bd

    def loss_value(self, alpha: torch.Tensor, want_chi: bool = False):
        alpha = alpha.to(self.cdt).contiguous()
        chi = self.cplx(self.S, self.M, self.M) if want_chi else None
        N.check(self.lib.pdf_loss_value(self.ctx, _ptr(alpha), _ptr(self.bd), _ptr(chi), _stream()))
        return self.bd, chi

    # ------------------------------------------------------------------ network
    def net_setup(self, alpha0: torch.Tensor) -> None:
        self.alpha0 = alpha0.to(self.cdt).contiguous()
        N.check(self.lib.pdf_net_setup(self.ctx, _ptr(self.alpha0), _stream()))

    def net_forward(self, theta: torch.Tensor) -> torch.Tensor:
        out = self.cplx(self.S, self.n, self.m0)
        N.check(self.lib.pdf_net_forward(self.ctx, _ptr(theta), _ptr(out), _stream()))
        return out

    def grad_loss(self, theta: torch.Tensor, grad: torch.Tensor | None = None):
        g = torch.empty_like(theta) if grad is None else grad
        N.check(self.lib.pdf_grad_loss(self.ctx, _ptr(theta), _ptr(g), _ptr(self.bd), _stream()))
        return g, self.bd

    def adam_step(self, theta, m, v, grad, t: int) -> None:
        N.check(self.lib.pdf_adam_step(self.ctx, _ptr(theta), _ptr(m), _ptr(v), _ptr(grad), theta.numel(),
                                       int(t), _stream()))

    def set_data(self, data, mask=None) -> None:
        """Replace the measured data of all S scenes in place (new batch, same geometry)."""
        data = np.asarray(data)
        data = data[None] if data.ndim == 2 else data
        self.data.copy_(torch.as_tensor(data, dtype=self.cdt), non_blocking=True)
        dm = data if self.mask is None else data * self.mask.cpu().numpy()
        self.c_sca = np.array([float(np.vdot(dm[s], dm[s]).real) for s in range(self.S)])
        self.set_norms(self.c_inc, self.c_sca)

    def set_norms(self, c_inc, c_sca) -> None:
        from .errors import ZeroDataError
        if np.any(np.asarray(c_sca) <= 0) or np.any(np.asarray(c_inc) <= 0):
            raise ZeroDataError("measured scattered / incident power is zero")
        self.c_inc, self.c_sca = np.asarray(c_inc, float), np.asarray(c_sca, float)
        # device copies (read by init_alpha; updated in place so a captured graph sees new values)
        if getattr(self, "c_inc_d", None) is None:
            self.c_inc_d = torch.empty(self.S, dtype=torch.float64, device=self.device)
            self.c_sca_d = torch.empty(self.S, dtype=torch.float64, device=self.device)
        self.c_inc_d.copy_(torch.as_tensor(self.c_inc))
        self.c_sca_d.copy_(torch.as_tensor(self.c_sca))
        ci = (ct.c_double * self.S)(*self.c_inc)
        cs = (ct.c_double * self.S)(*self.c_sca)
        N.check(self.lib.pdf_set_norms(self.ctx, ci, cs, _stream()))

    def alloc_state(self, theta0: torch.Tensor):
        """(theta, m, v) for train(): one allocation (the library keeps that
        window L2-resident in the captured loop), theta = theta0, m = v = 0."""
        flat = torch.zeros((3,) + tuple(theta0.shape), dtype=self.rdt, device=self.device)
        flat[0].copy_(theta0)
        return flat[0], flat[1], flat[2]

    def train(self, theta, m, v, t0: int, k: int, trace: torch.Tensor | None = None, use_graph: bool = True):
        N.check(self.lib.pdf_train(self.ctx, _ptr(theta), _ptr(m), _ptr(v), int(t0), int(k), _ptr(trace),
                                   int(use_graph), _stream()))

    def profile_phases(self, theta, m, v, t0: int, iters: int) -> dict:
        ms = (ct.c_float * len(N.PHASES))()
        N.check(self.lib.pdf_profile_train(self.ctx, _ptr(theta), _ptr(m), _ptr(v), int(t0), int(iters), ms,
                                           _stream()))
        return {name: float(ms[i]) for i, name in enumerate(N.PHASES)}

    def timeline(self, theta, m, v, t0: int = 0) -> list:
        """One replay of the 10-iteration training graph with per-kernel
        globaltimer stamps: [(iteration, phase, entry_ns, waited_ns, exit_ns)]
        relative to the first entry (measurement only)."""
        st = _stream()
        N.check(self.lib.pdf_timeline_reset(self.ctx, 1, st))
        self.train(theta, m, v, t0, 10)          # capture with slots + one replay
        torch.cuda.synchronize()
        N.check(self.lib.pdf_timeline_reset(self.ctx, 2, st))   # clear the stamps, keep the graph
        self.train(theta, m, v, t0 + 10, 10)
        torch.cuda.synchronize()
        buf = (ct.c_uint64 * (128 * 3 + 128 * 8))()
        N.check(self.lib.pdf_timeline_read(buf, st))
        N.check(self.lib.pdf_timeline_reset(self.ctx, 0, st))
        rows = []
        for sl in range(128):
            e, w, x = buf[3 * sl], buf[3 * sl + 1], buf[3 * sl + 2]
            if x == 0:
                continue
            stages = [buf[384 + 8 * sl + k] for k in range(8)]
            rows.append((sl // len(N.PHASES), sl % len(N.PHASES), e, w, x, stages))
        t0ns = min(r[2] for r in rows) if rows else 0
        return [(i, N.PHASES[p], e - t0ns, w - t0ns, x - t0ns, [s - t0ns if s else None for s in st_])
                for i, p, e, w, x, st_ in rows]

    # ------------------------------------------------------------------ primitives
    def apply_gd(self, x: torch.Tensor, adjoint: bool = False) -> torch.Tensor:
        x = x.to(self.cdt).contiguous()
        cnt = x.numel() // (self.M * self.M)
        y = torch.empty_like(x)
        N.check(self.lib.pdf_apply_gd(self.ctx, _ptr(x), _ptr(y), cnt, int(adjoint), _stream()))
        return y

    def gs_forward(self, img: torch.Tensor) -> torch.Tensor:
        img = img.to(self.cdt).contiguous()
        cnt = img.numel() // (self.M * self.M)
        rows = self.cplx(*img.shape[:-2], self.R)
        N.check(self.lib.pdf_gs_forward(self.ctx, _ptr(img), _ptr(rows), cnt, _stream()))
        return rows

    def gs_adjoint(self, rows: torch.Tensor) -> torch.Tensor:
        rows = rows.to(self.cdt).contiguous()
        cnt = rows.numel() // self.R
        img = self.cplx(*rows.shape[:-1], self.M, self.M)
        N.check(self.lib.pdf_gs_adjoint(self.ctx, _ptr(rows), _ptr(img), cnt, _stream()))
        return img

    def expand(self, alpha: torch.Tensor) -> torch.Tensor:
        alpha = alpha.to(self.cdt).contiguous()
        cnt = alpha.numel() // self.m0
        img = self.cplx(*alpha.shape[:-1], self.M, self.M)
        N.check(self.lib.pdf_expand(self.ctx, _ptr(alpha), _ptr(img), cnt, _stream()))
        return img

    def truncate(self, img: torch.Tensor) -> torch.Tensor:
        img = img.to(self.cdt).contiguous()
        cnt = img.numel() // (self.M * self.M)
        out = self.cplx(*img.shape[:-2], self.m0)
        N.check(self.lib.pdf_truncate(self.ctx, _ptr(img), _ptr(out), cnt, _stream()))
        return out

    def apply_cco(self, chi: torch.Tensor, cco) -> torch.Tensor:
        chi = chi.to(self.cdt).contiguous()
        cnt = chi.numel() // (self.M * self.M)
        out = torch.empty_like(chi)
        N.check(self.lib.pdf_apply_cco(self.ctx, _ptr(chi), _ptr(out), cnt, float(cco.tau), float(cco.eta_max),
                                       float(cco.delta), int(cco.gf_radius), float(cco.gf_eps), _stream()))
        return out

    # ------------------------------------------------------------------ init (reconstruct.py:52-153)
    def _einc_b(self):
        return self.e_inc if self.e_inc.dim() == 4 else self.e_inc.unsqueeze(0).expand(self.S, -1, -1, -1)

    def _masked(self, rows):
        return rows if self.mask is None else rows * self.mask

    def bp_initialize(self, check: bool = True):
        """Backprojection chi0 and R0 per scene (reconstruct.py:52-71).  check=False
        leaves the pole test as a device flag (`self.pole_flag`, raised later
        by the caller) so the sequence has no host synchronisation."""
        d = self._masked(self.data)
        b = self.gs_adjoint(d)
        w = self._masked(self.gs_forward(b))
        num = torch.sum(torch.conj(w) * d, dim=-1)
        den = torch.sum((w.conj() * w).real, dim=-1)
        gamma = torch.where(den > 0, num / torch.where(den > 0, den, torch.ones_like(den)),
                            torch.zeros_like(num))
        j = gamma[..., None, None] * b
        e = self._einc_b() + self.apply_gd(j)
        chi0 = self._pixel_ls(j, e)
        q = self.beta * chi0 + 1.0
        self.pole_flag = (q.abs() < 1e-14).any()
        if check and bool(self.pole_flag):
            raise PoleError("beta*chi + 1 vanishes at some pixel")
        return chi0, self.beta * chi0 / q

    def _pixel_ls(self, j, e):
        M2 = self.M * self.M
        pw = torch.sum((e.conj() * e).real, dim=(-1, -2))            # (S, n)
        eps = 1e-10 * pw.max(dim=-1).values / M2                      # cie.py:49-50
        num = torch.sum(j * e.conj(), dim=1)
        den = torch.sum((e.conj() * e).real, dim=1) + eps[:, None, None]
        return num / den

    def init_alpha(self, r0: torch.Tensor, check: bool = True) -> torch.Tensor:
        """One exact line-search step of the frozen-R quadratic (reconstruct.py:74-153).
        check=False leaves the zero-gradient test as `self.zero_grad_flag`."""
        M2 = self.M * self.M
        beta = self.beta
        c_inc = self.c_inc_d[:, None, None, None]
        c_sca = self.c_sca_d[:, None, None]
        r0b = r0[:, None]
        einc = self._einc_b()
        gs_r = (2.0 / c_inc) * (r0b * einc)
        rows = -self._masked(self.data)
        g_rows = self._masked((2.0 / c_sca) * rows)
        g_j = self.apply_gd(torch.conj(r0b) * gs_r, adjoint=True) + beta * (torch.conj(r0b) - 1.0) * gs_r
        g_j = g_j + self.gs_adjoint(g_rows)
        g = self.truncate(g_j) / M2
        jd = self.expand(g)
        s_lin = r0b * self.apply_gd(jd) + beta * (r0b - 1.0) * jd
        rr = self._masked(self.gs_forward(jd))
        q = (torch.sum((s_lin.conj() * s_lin).real, dim=(1, 2, 3)) / c_inc.view(-1)
             + torch.sum((rr.conj() * rr).real, dim=(1, 2)) / c_sca.view(-1))
        g2 = torch.sum((g.conj() * g).real, dim=(1, 2))
        ok = (q > 0) & (g2 > 0)
        self.zero_grad_flag = ~ok.all()
        if check and bool(self.zero_grad_flag):
            warnings.warn("zero initial gradient; starting from zero coefficients")
        t = torch.where(ok, g2 / (2.0 * torch.where(ok, q, torch.ones_like(q))), torch.zeros_like(q))
        return -t[:, None, None] * g
