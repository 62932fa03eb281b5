"""Incidence sharding for one large scene (BASELINE config 5).

The views of a scene are split over ranks (`shard.shard_range`).  Every rank
holds the full network (replicated parameters and Adam state) and runs the
physics for its own views only.  One PDF iteration then needs three
reductions, which the library exposes as float64 device buffers and the
caller performs (NCCL over NVLink through torch.distributed on the B200 box):

  red1 : per-pixel sum_i J_i conj(E_i), sum_i |E_i|^2 (SUM) and the max view
         power for eps_reg (MAX)                     -- cie.py:42-80
  red2 : per-pixel g_R = sum_i conj(P_i) g_S_i and the state / data loss sums
         (SUM)                                       -- losses.py:227,232,293
  grad : the flat network gradient (SUM), after which every rank applies the
         same Adam step                              -- network.py:220, 248-264

The one-time initialisation (bp_initialize, init_alpha) is replicated on
every rank over all views.  `LocalShards` runs several shards in one process
(the reductions become plain sums) so a single GPU can check the sharded
algebra against the unsharded path; `TorchDistReducer` is the multi-GPU form.
"""
from __future__ import annotations

import ctypes as ct

import numpy as np
import torch

from . import _native as N
from .engine import DeviceProblem, _ptr, _stream
from .shard import shard_range


class IncidenceShard:
    """This rank's slice of the views of one scene, resident on the GPU."""

    def __init__(self, ops, e_inc_all, data_all, *, mf, beta, lambdas, tau_b, rank, world, mask=None,
                 lr=1e-2, dtype="f64"):
        e_inc_all = np.asarray(e_inc_all)
        data_all = np.asarray(data_all)
        self.n_all = e_inc_all.shape[0]
        own = shard_range(self.n_all, rank, world)
        if len(own) == 0:
            raise ValueError("more ranks than incidences")
        self.own = own
        kw = dict(mf=mf, beta=beta, lambdas=lambdas, tau_b=tau_b, lr=lr, dtype=dtype)
        mk = None if mask is None else np.asarray(mask)
        # one-time initialisation over all views (replicated)
        full = DeviceProblem(ops, e_inc_all, data_all, mask=mk, **kw)
        self.chi0, r0 = full.bp_initialize()
        self.alpha0_all = full.init_alpha(r0)
        c_inc, c_sca = full.c_inc, full.c_sca
        del full
        sl = slice(own.start, own.stop)
        self.dev = DeviceProblem(ops, np.ascontiguousarray(e_inc_all[sl]), np.ascontiguousarray(data_all[sl]),
                                 mask=None if mk is None else np.ascontiguousarray(mk[sl]), **kw)
        self.dev.set_norms(c_inc, c_sca)          # normalisers over ALL views (losses.py:67-76)
        N.check(self.dev.lib.pdf_net_setup_sharded(self.dev.ctx, _ptr(self.alpha0_all), self.n_all, own.start,
                                                   _stream()))
        r1, r2 = ct.c_int64(), ct.c_int64()
        N.check(self.dev.lib.pdf_shard_buffer_sizes(self.dev.ctx, ct.byref(r1), ct.byref(r2)))
        dd = self.dev.device
        self.red1 = torch.zeros(r1.value, dtype=torch.float64, device=dd)
        self.red2 = torch.zeros(r2.value, dtype=torch.float64, device=dd)
        self.img = self.dev.M * self.dev.M
        self.bd = torch.zeros(1, 6, dtype=torch.float64, device=dd)

    # the three segments of one iteration
    def step_a(self, theta):
        N.check(self.dev.lib.pdf_shard_step_a(self.dev.ctx, _ptr(theta), _ptr(self.red1), _stream()))

    def step_b(self, chi_out=None):
        N.check(self.dev.lib.pdf_shard_step_b(self.dev.ctx, _ptr(self.red1), _ptr(self.red2), _ptr(chi_out),
                                              _stream()))

    def step_c(self, theta, grad):
        N.check(self.dev.lib.pdf_shard_step_c(self.dev.ctx, _ptr(theta), _ptr(self.red2), _ptr(grad),
                                              _ptr(self.bd), _stream()))

    def red1_sum_max(self):
        """(slice reduced with SUM, slice reduced with MAX) of red1."""
        return self.red1[: 3 * self.img], self.red1[3 * self.img:]


class TorchDistReducer:
    """Reductions over a torch.distributed group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def __call__(self, shards, what):
        d = self.dist
        (s,) = shards
        if what == "red1":
            a, b = s.red1_sum_max()
            d.all_reduce(a, op=d.ReduceOp.SUM, group=self.group)
            d.all_reduce(b, op=d.ReduceOp.MAX, group=self.group)
        elif what == "red2":
            d.all_reduce(s.red2, op=d.ReduceOp.SUM, group=self.group)
        else:
            d.all_reduce(what, op=d.ReduceOp.SUM, group=self.group)


class LocalShards:
    """All shards of a scene in one process; reductions are fixed-order sums."""

    def __call__(self, shards, what):
        if what == "red1":
            a = sum(s.red1_sum_max()[0] for s in shards)
            b = torch.stack([s.red1_sum_max()[1] for s in shards]).max(dim=0).values
            for s in shards:
                s.red1[: 3 * s.img] = a
                s.red1[3 * s.img:] = b
        elif what == "red2":
            t = sum(s.red2 for s in shards)
            for s in shards:
                s.red2.copy_(t)
        else:   # list of gradient tensors, one per shard
            t = sum(what)
            for g in what:
                g.copy_(t)


def run_sharded(shards, reduce, theta0, k_iters: int, lr: float = 1e-2, trace_on_device: bool = False):
    """k incidence-sharded Adam iterations for the given (local) shards.

    Returns (thetas per shard, trace [k][6]).  Every shard keeps its own copy
    of the replicated parameters and Adam state.  trace_on_device keeps the
    breakdown rows on the GPU (no per-iteration host synchronisation) and
    returns them as a tensor."""
    thetas = [theta0.clone() for _ in shards]
    ms = [torch.zeros_like(theta0) for _ in shards]
    vs = [torch.zeros_like(theta0) for _ in shards]
    grads = [torch.zeros_like(theta0) for _ in shards]
    trace = []
    dtrace = torch.zeros(k_iters, 6, dtype=torch.float64, device=shards[0].bd.device) if trace_on_device else None
    for t in range(1, k_iters + 1):
        for s, th in zip(shards, thetas):
            s.step_a(th)
        reduce(shards, "red1")
        for s in shards:
            s.step_b()
        reduce(shards, "red2")
        for s, th, g in zip(shards, thetas, grads):
            s.step_c(th, g)
        if isinstance(reduce, LocalShards):
            reduce(shards, grads)
        else:
            for g in grads:
                reduce(shards, g)
        if dtrace is not None:
            dtrace[t - 1].copy_(shards[0].bd[0])
        else:
            trace.append(shards[0].bd[0].cpu().numpy().copy())
        for s, th, m, v, g in zip(shards, thetas, ms, vs, grads):
            s.dev.adam_step(th, m, v, g, t)
    for s in shards:
        s.dev.check_errors()
    return thetas, (dtrace if dtrace is not None else np.array(trace))


def sharded_chi(shards, reduce, thetas):
    """Recovered contrast at the current parameters (cie.py:83-99) via the sharded forward."""
    for s, th in zip(shards, thetas):
        s.step_a(th)
    reduce(shards, "red1")
    chi = torch.empty(1, shards[0].dev.M, shards[0].dev.M, dtype=shards[0].dev.cdt, device=shards[0].dev.device)
    shards[0].step_b(chi)
    return chi[0]


# ---------------------------------------------------------------------------- ZeRO-1 form
def bucket_plan(offs, world: int) -> list[dict]:
    """Gradient buckets of the flat parameter vector, one per layer in the order
    the backward produces them (3, 2, 1): bucket L = [W_L | b_L], flat slice
    [offs[2L-2], offs[2L]) (offs = pdf_net_offsets: w1 b1 w2 b2 w3 b3 Np),
    padded to a multiple of `world` so a reduce-scatter hands rank r the
    contiguous shard [r s, (r + 1) s) of s = padded / world entries."""
    out = []
    for L in (3, 2, 1):
        lo, hi = int(offs[2 * L - 2]), int(offs[2 * L])
        n = hi - lo
        npad = -(-n // world) * world
        out.append({"layer": L, "lo": lo, "n": n, "npad": npad, "shard": npad // world})
    return out


class ShardedTrainer:
    """Incidence-sharded training of one large scene with sharded optimizer state
    (the alternative to replicated Adam VERDICT r01 asked for).

    One iteration on every rank:
      step_a (network forward, own views' physics)  -> all-reduce red1 (SUM, MAX)
      step_b (per-pixel chi / R / regularisers)     -> all-reduce red2 (SUM)
      step_c in layer parts 3, 2, 1: each layer's gradient bucket is
        reduce-scattered on a communication stream while the next layer's
        backward runs (bucketed overlap, NCCL over NVLink);
      Adam on this rank's 1/W shard of every bucket only (m, v hold 1/W of the
        parameters; step counter on the device);
      all-gather of the updated shards back into the replicated parameters.
    graph=True captures `graph_iters` such iterations -- library kernels and
    NCCL collectives -- in one CUDA graph and replays it."""

    def __init__(self, shard: IncidenceShard, theta0: torch.Tensor, group=None, graph: bool = True,
                 graph_iters: int = 10):
        import torch.distributed as dist
        self.dist, self.group, self.s = dist, group, shard
        self.W = dist.get_world_size(group)
        self.r = dist.get_rank(group)
        dev = shard.dev
        self.lib = dev.lib
        offs = (ct.c_int64 * 7)()
        N.check(self.lib.pdf_net_offsets(dev.ctx, offs))
        self.offs = [int(x) for x in offs]
        if self.offs[6] != theta0.numel():
            raise ValueError("theta0 does not match the network of this shard")
        self.plan = bucket_plan(self.offs, self.W)
        dd, rdt = dev.device, dev.rdt
        self.theta = theta0.detach().to(dd, rdt).reshape(-1).clone()
        self.gbuf, self.gshard, self.pown, self.m, self.v, self.pfull = {}, {}, {}, {}, {}, {}
        for b in self.plan:
            L, lo, n, npad, sh = b["layer"], b["lo"], b["n"], b["npad"], b["shard"]
            self.gbuf[L] = torch.zeros(npad, dtype=rdt, device=dd)
            self.gshard[L] = torch.zeros(sh, dtype=rdt, device=dd)
            full = torch.zeros(npad, dtype=rdt, device=dd)
            full[:n] = self.theta[lo:lo + n]
            self.pown[L] = full[self.r * sh:(self.r + 1) * sh].clone()
            self.m[L] = torch.zeros(sh, dtype=rdt, device=dd)
            self.v[L] = torch.zeros(sh, dtype=rdt, device=dd)
            # all-gather straight into theta when the bucket needs no padding
            self.pfull[L] = self.theta[lo:lo + n] if npad == n else full
        self.t_dev = torch.zeros(1, dtype=torch.int32, device=dd)
        self.comm = torch.cuda.Stream(device=dd)
        self.ev = {L: torch.cuda.Event() for L in (1, 2, 3)}
        self.graph_on, self.G = graph, max(1, int(graph_iters))
        self.graph = None
        self.gtrace = torch.zeros(self.G, 6, dtype=torch.float64, device=dd)

    def _red(self, t, op):
        self.dist.all_reduce(t, op=op, group=self.group)

    def iteration(self, trace_row: torch.Tensor | None = None):
        s, d = self.s, self.dist
        s.step_a(self.theta)
        a, b = s.red1_sum_max()
        self._red(a, d.ReduceOp.SUM)
        self._red(b, d.ReduceOp.MAX)
        s.step_b()
        self._red(s.red2, d.ReduceOp.SUM)
        main = torch.cuda.current_stream()
        for bk in self.plan:
            L = bk["layer"]
            N.check(self.lib.pdf_shard_step_c_part(s.dev.ctx, _ptr(self.theta), _ptr(s.red2), _ptr(self.gbuf[L]), L,
                                                   _ptr(s.bd), _stream()))
            self.ev[L].record(main)
            self.comm.wait_event(self.ev[L])
            with torch.cuda.stream(self.comm):
                d.reduce_scatter_tensor(self.gshard[L], self.gbuf[L], op=d.ReduceOp.SUM, group=self.group)
        main.wait_stream(self.comm)
        if trace_row is not None:
            trace_row.copy_(s.bd[0])
        self.t_dev += 1
        for bk in self.plan:
            L = bk["layer"]
            N.check(self.lib.pdf_adam_step_dev(s.dev.ctx, _ptr(self.pown[L]), _ptr(self.m[L]), _ptr(self.v[L]),
                                               _ptr(self.gshard[L]), bk["shard"], _ptr(self.t_dev), _stream()))
        for bk in self.plan:
            L, lo, n, npad = bk["layer"], bk["lo"], bk["n"], bk["npad"]
            d.all_gather_into_tensor(self.pfull[L], self.pown[L], group=self.group)
            if npad != n:
                self.theta[lo:lo + n].copy_(self.pfull[L][:n])

    def _capture(self):
        st = torch.cuda.Stream(device=self.theta.device)
        st.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(self.G):
                self.iteration(self.gtrace[i])
        self.graph = g

    def train(self, k: int) -> torch.Tensor:
        """k iterations; returns the device trace [k][6] (state, data, bound, tv, bridge, total)."""
        trace = torch.zeros(k, 6, dtype=torch.float64, device=self.theta.device)
        done = 0
        if self.graph_on and k >= self.G:
            if self.graph is None:
                # warm the collectives (communicator setup) outside the capture: two eager iterations
                # from a saved state, then restore it
                saved = [x.clone() for x in (self.theta, self.t_dev, *self.pown.values(), *self.m.values(),
                                             *self.v.values())]
                for _ in range(2):
                    self.iteration()
                torch.cuda.synchronize()
                for x, y in zip((self.theta, self.t_dev, *self.pown.values(), *self.m.values(), *self.v.values()),
                                saved):
                    x.copy_(y)
                self._capture()
            while done + self.G <= k:
                self.graph.replay()
                trace[done:done + self.G].copy_(self.gtrace)
                done += self.G
        while done < k:
            self.iteration(trace[done])
            done += 1
        return trace

    def check_errors(self):
        self.s.dev.check_errors()


# ---------------------------------------------------------------------------- peer-memory form
def peer_shard_len(n_params: int, world: int) -> int:
    """Per-rank shard of the flat parameters for the peer-scatter layout: even
    (16-byte g_W pairs never straddle two owners) and world * shard >= n_params."""
    s = -(-n_params // world)
    return s + (s & 1)


class PeerTrainer:
    """Incidence sharding with the gradient reduce-scatter fused into the
    backward kernels (the prompt's compute -> collective fusion).

    Every rank runs step_a / red1 / step_b / red2 as `ShardedTrainer` does;
    then `pdf_shard_step_c_scatter` (layers 3, 2, 1) stores each g_W / g_b
    entry, in the epilogue of the DMMA kernel that computes it, straight into
    the owner rank's receive buffer (peer stores over NVLink); after a
    barrier `pdf_adam_gather` on every rank sums its shard over the source
    ranks in rank order, applies Adam and writes the updated parameters into
    every rank's parameter vector (the all-gather, again as peer stores), and
    a second barrier closes the iteration.  No NCCL call moves gradient or
    parameter bytes.

    `shards` are either the ranks of one process emulated on one GPU (a list
    of IncidenceShard over all views, `group=None`: the "peer" buffers are
    local and the barriers are stream order -- no kernel waits for another)
    or this rank's single shard on a multi-GPU node (`group` given): the
    receive and parameter buffers are torch symmetric memory and their
    peer-mapped addresses are exchanged once (`rendezvous`)."""

    def __init__(self, shards, theta0: torch.Tensor, group=None, graph: bool = False, graph_iters: int = 10):
        self.shards = list(shards)
        self.group = group
        self.graph_on, self.G, self.graph = graph, max(1, int(graph_iters)), None
        dev0 = self.shards[0].dev
        self.lib = dev0.lib
        dd, rdt = dev0.device, dev0.rdt
        if rdt != torch.float64:
            raise ValueError("the peer-scatter path is float64")
        np_ = theta0.numel()
        if group is None:
            self.world, self.ranks = len(self.shards), list(range(len(self.shards)))
        else:
            import torch.distributed as dist
            self.world, self.ranks = dist.get_world_size(group), [dist.get_rank(group)]
            if len(self.shards) != 1:
                raise ValueError("one shard per process on a multi-GPU node")
        W = self.world
        self.np = np_
        self.shard = peer_shard_len(np_, W)
        n_pad = W * self.shard
        if group is None:
            self.recv = [torch.zeros(n_pad, dtype=rdt, device=dd) for _ in self.shards]
            self.theta = [torch.zeros(n_pad, dtype=rdt, device=dd) for _ in self.shards]
            recv_ptrs = [t.data_ptr() for t in self.recv]
            th_ptrs = [t.data_ptr() for t in self.theta]
        else:
            import torch.distributed._symmetric_memory as symm
            self.recv = [symm.empty(n_pad, dtype=rdt, device=dd)]
            self.theta = [symm.empty(n_pad, dtype=rdt, device=dd)]
            self.recv[0].zero_()
            self.theta[0].zero_()
            h_recv = symm.rendezvous(self.recv[0], group)
            h_th = symm.rendezvous(self.theta[0], group)
            recv_ptrs, th_ptrs = list(h_recv.buffer_ptrs), list(h_th.buffer_ptrs)
            self._handles = (h_recv, h_th)
        self.recv_peers = torch.tensor(recv_ptrs, dtype=torch.int64, device=dd)
        self.theta_peers = torch.tensor(th_ptrs, dtype=torch.int64, device=dd)
        for th in self.theta:
            th[:np_].copy_(theta0.reshape(-1))
        self.m = [torch.zeros(self.shard, dtype=rdt, device=dd) for _ in self.shards]
        self.v = [torch.zeros(self.shard, dtype=rdt, device=dd) for _ in self.shards]
        self.t_dev = torch.zeros(1, dtype=torch.int32, device=dd)
        self._bar = torch.zeros(1, dtype=torch.float64, device=dd)
        if group is not None:
            self._barrier()

    def _barrier(self):
        if self.group is not None:          # stream-ordered: every rank's earlier kernels are done
            import torch.distributed as dist
            dist.all_reduce(self._bar, group=self.group)

    def _reduce(self, what):
        if self.group is None:
            LocalShards()(self.shards, what)
        else:
            TorchDistReducer(self.group)(self.shards, what)

    def iteration(self, trace_row: torch.Tensor | None = None):
        for s, th in zip(self.shards, self.theta):
            s.step_a(th)
        self._reduce("red1")
        for s in self.shards:
            s.step_b()
        self._reduce("red2")
        for s, th, r in zip(self.shards, self.theta, self.ranks):
            for L in (3, 2, 1):
                N.check(self.lib.pdf_shard_step_c_scatter(
                    s.dev.ctx, _ptr(th), _ptr(s.red2), _ptr(self.recv_peers), self.world, r, self.shard, L,
                    _ptr(s.bd), _stream()))
        if trace_row is not None:
            trace_row.copy_(self.shards[0].bd[0])
        self._barrier()
        self.t_dev += 1
        for s, rv, m, v, r in zip(self.shards, self.recv, self.m, self.v, self.ranks):
            N.check(self.lib.pdf_adam_gather(s.dev.ctx, _ptr(rv), _ptr(self.theta_peers), _ptr(m), _ptr(v),
                                             self.world, r, self.shard, _ptr(self.t_dev), _stream()))
        self._barrier()

    def _state(self):
        return [*self.theta, *self.m, *self.v, self.t_dev]

    def train(self, k: int) -> torch.Tensor:
        """k iterations (graph=True: replayed from a CUDA graph of graph_iters
        iterations that holds the library kernels and the NCCL barriers)."""
        dd = self.theta[0].device
        trace = torch.zeros(k, 6, dtype=torch.float64, device=dd)
        done = 0
        if self.graph_on and k >= self.G:
            if self.graph is None:
                saved = [x.clone() for x in self._state()]
                for _ in range(2):                 # warm the collectives outside the capture
                    self.iteration()
                torch.cuda.synchronize()
                for x, y in zip(self._state(), saved):
                    x.copy_(y)
                self._barrier()
                self.gtrace = torch.zeros(self.G, 6, dtype=torch.float64, device=dd)
                st = torch.cuda.Stream(device=dd)
                st.wait_stream(torch.cuda.current_stream())
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for i in range(self.G):
                        self.iteration(self.gtrace[i])
                self.graph = g
            while done + self.G <= k:
                self.graph.replay()
                trace[done:done + self.G].copy_(self.gtrace)
                done += self.G
        while done < k:
            self.iteration(trace[done])
            done += 1
        return trace

    def params(self, rank: int = 0) -> torch.Tensor:
        return self.theta[rank][: self.np]

    def check_errors(self):
        for s in self.shards:
            s.dev.check_errors()


# ---------------------------------------------------------------------------- tensor-parallel network
def tp_split(total: int, world: int) -> tuple[int, list[tuple[int, int]]]:
    """Block size and (start, size) of every rank's slice of `total` units:
    blocks of ceil(total / world) rounded up to even (16-byte rows), the last
    one shorter.  Raises when a rank would get nothing."""
    blk = -(-total // world)
    blk += blk & 1
    parts = [(min(r * blk, total), min((r + 1) * blk, total) - min(r * blk, total)) for r in range(world)]
    if any(n <= 0 for _, n in parts):
        raise ValueError(f"{world} ranks leave some rank without a slice of {total} units")
    return blk, parts


def tp_full_offsets(H: int, D0: int) -> list[int]:
    """Offsets of W1, b1, W2, b2, W3, b3 and the end in the flat parameter vector
    (network.py:158-166 order; W_L stored [out][in])."""
    o = [0, H * D0]
    o.append(o[-1] + H)
    o.append(o[-1] + H * H)
    o.append(o[-1] + H)
    o.append(o[-1] + D0 * H)
    o.append(o[-1] + D0)
    return o


def tp_local_offsets(H: int, D0: int, hr: int, dr: int) -> list[int]:
    """Offsets of one rank's W1 rows [hr][D0], b1 slice, W2 columns [H][hr], b2 [H],
    W3 rows [dr][H], b3 slice, and the end."""
    o = [0, hr * D0]
    o.append(o[-1] + hr)
    o.append(o[-1] + H * hr)
    o.append(o[-1] + H)
    o.append(o[-1] + dr * H)
    o.append(o[-1] + dr)
    return o


def tp_local_params(th: torch.Tensor, H: int, D0: int, hpart, dpart) -> torch.Tensor:
    """One rank's parameters in the local layout, cut from the full flat vector."""
    (h0, hr), (c0, dr) = hpart, dpart
    f = tp_full_offsets(H, D0)
    W1, W2, W3 = th[f[0]:f[1]].view(H, D0), th[f[2]:f[3]].view(H, H), th[f[4]:f[5]].view(D0, H)
    return torch.cat([W1[h0:h0 + hr].reshape(-1), th[f[1] + h0:f[1] + h0 + hr], W2[:, h0:h0 + hr].reshape(-1),
                      th[f[3]:f[4]], W3[c0:c0 + dr].reshape(-1), th[f[5] + c0:f[5] + c0 + dr]])


def tp_assemble(locals_, H: int, D0: int, hparts, dparts) -> torch.Tensor:
    """The full flat vector from every rank's local vector (b2 taken from rank 0)."""
    f = tp_full_offsets(H, D0)
    th = torch.zeros(f[6], dtype=locals_[0].dtype, device=locals_[0].device)
    W1, W2, W3 = th[f[0]:f[1]].view(H, D0), th[f[2]:f[3]].view(H, H), th[f[4]:f[5]].view(D0, H)
    for r in reversed(range(len(locals_))):
        (h0, hr), (c0, dr), p = hparts[r], dparts[r], locals_[r]
        lo = tp_local_offsets(H, D0, hr, dr)
        W1[h0:h0 + hr] = p[lo[0]:lo[1]].view(hr, D0)
        th[f[1] + h0:f[1] + h0 + hr] = p[lo[1]:lo[2]]
        W2[:, h0:h0 + hr] = p[lo[2]:lo[3]].view(H, hr)
        th[f[3]:f[4]] = p[lo[3]:lo[4]]
        W3[c0:c0 + dr] = p[lo[4]:lo[5]].view(dr, H)
        th[f[5] + c0:f[5] + c0 + dr] = p[lo[5]:lo[6]]
    return th


def tp_to_blocks(y: torch.Tensor, blk: int, world: int) -> torch.Tensor:
    """(rows, D0) -> the column-block layout Y[w][rows][N_w] (flat, world * rows * blk
    entries) that pdf_shard_tp_a reads and pdf_shard_tp_c writes."""
    rows, D0 = y.shape
    out = torch.zeros(world * rows * blk, dtype=y.dtype, device=y.device)
    for w in range(world):
        c0 = w * blk
        nw = min(blk, D0 - c0)
        if nw > 0:
            out[w * rows * blk:w * rows * blk + rows * nw] = y[:, c0:c0 + nw].reshape(-1)
    return out


def tp_from_blocks(Y: torch.Tensor, rows: int, D0: int, blk: int) -> torch.Tensor:
    """Inverse of tp_to_blocks."""
    y = torch.empty(rows, D0, dtype=Y.dtype, device=Y.device)
    for w in range(-(-D0 // blk)):
        c0 = w * blk
        nw = min(blk, D0 - c0)
        y[:, c0:c0 + nw] = Y[w * rows * blk:w * rows * blk + rows * nw].view(rows, nw)
    return y


class TensorParallelTrainer:
    """Incidence sharding with a tensor-parallel network (SURVEY 8(e)'s
    alternative to exchanging the network gradient).

    The widths are [D0, H, H, D0] (network.py:61; W_L stored [out][in]).  Rank
    r holds rows h_r of W1 / b1 (column-parallel), columns h_r of W2 with all
    of b2 (row-parallel), rows d_r of W3 / b3, and their Adam state: 1/W of
    the parameters, updated locally.  One iteration, for all views of the
    scene on every rank's network slice and its own views' physics:

      h1_r = tanh(x0 W1_r^T + b1_r)           local
      z2   = sum_r h1_r W2_r^T                all-reduce (rows x H)
      h2   = tanh(z2 + b2)                    local (replicated)
      Y_r  = h2 W3_r^T + b3_r                 all-reduce of the column blocks (rows x D0)
      physics of own views (tp_a, red1, step_b, red2, tp_c) -> the gradient rows of Y
      GY                                       all-reduce of the row blocks (rows x D0)
      g_W3_r, g_b3_r; g_z2 = sum_r (GY_r W3_r)(1 - h2^2)   all-reduce (rows x H)
      g_W2_r, g_b2, g_z1_r = (g_z2 W2_r)(1 - h1_r^2)       local
      g_W1_r, g_b1_r                                        local
      Adam on this rank's slices

    Per iteration and rank the collectives move 2 (rows x H) + 2 (rows x D0)
    doubles plus the physics' red1 / red2 (at config 5: 2.4 + 2.4 + 1.2 + 1.2
    MB + 2.6 MB), instead of the 268 MB gradient reduce-scatter and the 268 MB
    parameter all-gather of the ZeRO-1 forms; weights, Adam state and network
    FLOPs are 1/W per rank.  All network arithmetic runs in the library's DMMA
    layer kernels (pdf_net_layer_fwd / _bwd).

    `shards` are all ranks of one process emulated on one GPU (a list of
    IncidenceShard over all views, `group=None`: the collectives become
    rank-order sums; no kernel waits for another) or this rank's single shard
    with a torch.distributed `group` (NCCL)."""

    def __init__(self, shards, theta0: torch.Tensor, group=None, graph: bool = False, graph_iters: int = 10,
                 lr: float = 1e-2):
        from .api import _net_device_lr
        self.shards = list(shards)
        self.group = group
        self.graph_on, self.G, self.graph = graph, max(1, int(graph_iters)), None
        s0 = self.shards[0]
        if s0.dev.rdt != torch.float64:
            raise ValueError("the tensor-parallel network is float64")
        if group is None:
            self.world, self.ranks = len(self.shards), list(range(len(self.shards)))
        else:
            import torch.distributed as dist
            self.world, self.ranks = dist.get_world_size(group), [dist.get_rank(group)]
            if len(self.shards) != 1:
                raise ValueError("one shard per process on a multi-GPU node")
        W = self.world
        self.rows = s0.n_all
        # a geometry-free context that runs the network kernels over all views of the scene
        self.net = _net_device_lr(self.rows, s0.dev.mf, lr)
        lib, nc = self.net.lib, self.net.ctx
        self.lib = lib
        rows, d0, hid, np_ = ct.c_int32(), ct.c_int32(), ct.c_int32(), ct.c_int64()
        N.check(lib.pdf_net_dims(nc, ct.byref(rows), ct.byref(d0), ct.byref(hid), ct.byref(np_)))
        self.D0, self.H, self.np = d0.value, hid.value, np_.value
        if theta0.numel() != self.np:
            raise ValueError("theta0 does not match the network of this scene")
        dd = s0.dev.device
        N.check(lib.pdf_net_setup(nc, _ptr(s0.alpha0_all), _stream()))
        self.x0 = torch.empty(self.rows, self.D0, dtype=torch.float64, device=dd)
        N.check(lib.pdf_net_features(nc, _ptr(self.x0), None, _stream()))
        self.hblk, self.hparts = tp_split(self.H, W)
        self.dblk, self.dparts = tp_split(self.D0, W)
        th = theta0.detach().to(dd, torch.float64).reshape(-1)
        self.st = [self._rank_state(th, r, dd) for r in self.ranks]
        self.t_dev = torch.zeros(1, dtype=torch.int32, device=dd)

    # ------------------------------------------------------------------ layout
    def _rank_state(self, th, r, dd):
        hr, dr = self.hparts[r][1], self.dparts[r][1]
        p = tp_local_params(th, self.H, self.D0, self.hparts[r], self.dparts[r]).contiguous()
        z = lambda *shape: torch.zeros(*shape, dtype=torch.float64, device=dd)   # noqa: E731
        W, R = self.world, self.rows
        return {"r": r, "hr": hr, "dr": dr, "off": tp_local_offsets(self.H, self.D0, hr, dr), "theta": p,
                "m": z(p.numel()), "v": z(p.numel()), "grad": z(p.numel()), "h1": z(R, hr), "z2": z(R, self.H),
                "Y": z(W * R * self.dblk), "GY": z(W * R * self.dblk), "gz2": z(R, self.H), "gz1": z(R, hr)}

    def params(self) -> torch.Tensor:
        """The full flat parameter vector (emulated ranks: assembled from every rank's slices)."""
        if self.group is not None:
            raise NotImplementedError("assemble with an all-gather on a multi-GPU node")
        return tp_assemble([s["theta"] for s in self.st], self.H, self.D0, self.hparts, self.dparts)

    # ------------------------------------------------------------------ collectives
    def _sum(self, key):
        """All-reduce (SUM) of every rank's buffer `key`."""
        if self.group is None:
            t = self.st[0][key].clone()
            for s in self.st[1:]:
                t += s[key]
            for s in self.st:
                s[key].copy_(t)
        else:
            import torch.distributed as dist
            dist.all_reduce(self.st[0][key], op=dist.ReduceOp.SUM, group=self.group)

    def _reduce_phys(self, what):
        if self.group is None:
            LocalShards()(self.shards, what)
        else:
            TorchDistReducer(self.group)(self.shards, what)

    # ------------------------------------------------------------------ one iteration
    def _fwd(self, s, inp, K, Nn, w, b, out, mode):
        N.check(self.lib.pdf_net_layer_fwd(self.net.ctx, _ptr(inp), K, Nn, _ptr(s["theta"]), w, b, _ptr(out), mode,
                                           _stream()))

    def _bwd(self, s, gz, hin, K, Nn, w, b, gin):
        N.check(self.lib.pdf_net_layer_bwd(self.net.ctx, _ptr(gz), _ptr(hin), K, Nn, _ptr(s["theta"]), w, b,
                                           _ptr(s["grad"]), None if gin is None else _ptr(gin), _stream()))

    def iteration(self, trace_row: torch.Tensor | None = None):
        R, H, D0 = self.rows, self.H, self.D0
        for s in self.st:
            o = s["off"]
            self._fwd(s, self.x0, D0, s["hr"], o[0], o[1], s["h1"], 0)
            self._fwd(s, s["h1"], s["hr"], H, o[2], -1, s["z2"], 3)
        self._sum("z2")
        for s in self.st:
            o = s["off"]
            N.check(self.lib.pdf_bias_tanh(_ptr(s["z2"]), _ptr(s["theta"][o[3]:]), R, H, _stream()))   # z2 -> h2
            s["Y"].zero_()
            yb = s["Y"][s["r"] * R * self.dblk:]
            self._fwd(s, s["z2"], H, s["dr"], o[4], o[5], yb, 2)
        self._sum("Y")
        for sh, s in zip(self.shards, self.st):
            N.check(self.lib.pdf_shard_tp_a(sh.dev.ctx, _ptr(s["Y"]), self.dblk, R, sh.own.start, _ptr(sh.red1),
                                            _stream()))
        self._reduce_phys("red1")
        for sh in self.shards:
            sh.step_b()
        self._reduce_phys("red2")
        for sh, s in zip(self.shards, self.st):
            s["GY"].zero_()
            N.check(self.lib.pdf_shard_tp_c(sh.dev.ctx, _ptr(sh.red2), _ptr(s["GY"]), self.dblk, R, sh.own.start,
                                            _ptr(sh.bd), _stream()))
        if trace_row is not None:
            trace_row.copy_(self.shards[0].bd[0])
        self._sum("GY")
        for s in self.st:
            o = s["off"]
            gy = s["GY"][s["r"] * R * self.dblk:]
            self._bwd(s, gy, s["z2"], H, s["dr"], o[4], o[5], s["gz2"])
        self._sum("gz2")
        self.t_dev += 1
        for s in self.st:
            o = s["off"]
            self._bwd(s, s["gz2"], s["h1"], s["hr"], H, o[2], o[3], s["gz1"])
            self._bwd(s, s["gz1"], self.x0, D0, s["hr"], o[0], o[1], None)
            N.check(self.lib.pdf_adam_step_dev(self.net.ctx, _ptr(s["theta"]), _ptr(s["m"]), _ptr(s["v"]),
                                               _ptr(s["grad"]), s["theta"].numel(), _ptr(self.t_dev), _stream()))

    def _state(self):
        return [x for s in self.st for x in (s["theta"], s["m"], s["v"])] + [self.t_dev]

    def train(self, k: int) -> torch.Tensor:
        """k iterations (graph=True: replayed from a CUDA graph of graph_iters iterations
        holding the library kernels and the collectives); returns the trace [k][6]."""
        dd = self.x0.device
        trace = torch.zeros(k, 6, dtype=torch.float64, device=dd)
        done = 0
        if self.graph_on and k >= self.G:
            if self.graph is None:
                saved = [x.clone() for x in self._state()]
                for _ in range(2):                 # warm the collectives outside the capture
                    self.iteration()
                torch.cuda.synchronize()
                for x, y in zip(self._state(), saved):
                    x.copy_(y)
                self.gtrace = torch.zeros(self.G, 6, dtype=torch.float64, device=dd)
                st = torch.cuda.Stream(device=dd)
                st.wait_stream(torch.cuda.current_stream())
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for i in range(self.G):
                        self.iteration(self.gtrace[i])
                self.graph = g
            while done + self.G <= k:
                self.graph.replay()
                trace[done:done + self.G].copy_(self.gtrace)
                done += self.G
        while done < k:
            self.iteration(trace[done])
            done += 1
        return trace

    def check_errors(self):
        for s in self.shards:
            s.dev.check_errors()
        self.net.check_errors()
