"""Config 5 with the tensor-parallel network, W ranks emulated on one GPU.

    python tools/tp_emulate.py [W] [iters]

Prints the emulated iteration time (all W ranks' work, sequential on one GPU)
and, per segment, the slowest rank's time; their sum is the compute part of
one rank's iteration on a W-GPU node (the collectives, ~10 MB of all-reduces
per iteration at config 5, come on top).  Also checks the trace of the timed
iterations against the unsharded run (rtol 1e-9)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_13805_b200 import _native as N  # noqa: E402
from paper_2602_13805_b200 import build_grid, plane_wave_fields  # noqa: E402
from paper_2602_13805_b200.api import BatchReconstructor, _theta0  # noqa: E402
from paper_2602_13805_b200.engine import _ptr, _stream  # noqa: E402
from paper_2602_13805_b200.sharded import IncidenceShard, TensorParallelTrainer  # noqa: E402
from paper_2602_13805_b200.workloads import baseline_config, baseline_scene, synthesize_gpu  # noqa: E402


class Timed(TensorParallelTrainer):
    """iteration() with CUDA events around every rank's share of each segment."""

    def seg(self, name, r, fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        self.ev.append((name, r, e0, e1))

    def iteration(self, trace_row=None):
        R, H, D0 = self.rows, self.H, self.D0
        for s in self.st:
            o = s["off"]
            self.seg("net_fwd_12", s["r"], lambda: (self._fwd(s, self.x0, D0, s["hr"], o[0], o[1], s["h1"], 0),
                                                    self._fwd(s, s["h1"], s["hr"], H, o[2], -1, s["z2"], 3)))
        self._sum("z2")
        for s in self.st:
            o = s["off"]

            def f3():
                N.check(self.lib.pdf_bias_tanh(_ptr(s["z2"]), _ptr(s["theta"][o[3]:]), R, H, _stream()))
                s["Y"].zero_()
                self._fwd(s, s["z2"], H, s["dr"], o[4], o[5], s["Y"][s["r"] * R * self.dblk:], 2)
            self.seg("net_fwd_3", s["r"], f3)
        self._sum("Y")
        for sh, s in zip(self.shards, self.st):
            self.seg("phys_a", s["r"], lambda: N.check(self.lib.pdf_shard_tp_a(
                sh.dev.ctx, _ptr(s["Y"]), self.dblk, R, sh.own.start, _ptr(sh.red1), _stream())))
        self._reduce_phys("red1")
        for sh, s in zip(self.shards, self.st):
            self.seg("phys_b", s["r"], sh.step_b)
        self._reduce_phys("red2")
        for sh, s in zip(self.shards, self.st):
            def fc():
                s["GY"].zero_()
                N.check(self.lib.pdf_shard_tp_c(sh.dev.ctx, _ptr(sh.red2), _ptr(s["GY"]), self.dblk, R,
                                                sh.own.start, _ptr(sh.bd), _stream()))
            self.seg("phys_c", s["r"], fc)
        if trace_row is not None:
            trace_row.copy_(self.shards[0].bd[0])
        self._sum("GY")
        for s in self.st:
            o = s["off"]
            self.seg("net_bwd_3", s["r"], lambda: self._bwd(s, s["GY"][s["r"] * R * self.dblk:], s["z2"], H,
                                                            s["dr"], o[4], o[5], s["gz2"]))
        self._sum("gz2")
        self.t_dev += 1
        for s in self.st:
            o = s["off"]

            def fb():
                self._bwd(s, s["gz2"], s["h1"], s["hr"], H, o[2], o[3], s["gz1"])
                self._bwd(s, s["gz1"], self.x0, D0, s["hr"], o[0], o[1], None)
                N.check(self.lib.pdf_adam_step_dev(self.net.ctx, _ptr(s["theta"]), _ptr(s["m"]), _ptr(s["v"]),
                                                   _ptr(s["grad"]), s["theta"].numel(), _ptr(self.t_dev), _stream()))
            self.seg("net_bwd_21_adam", s["r"], fb)


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    cfg = baseline_config(5, k_iters=k)
    scene, rng, snr = baseline_scene(5)
    data, _ = synthesize_gpu(cfg, [scene], [rng], snr)
    e_inc = plane_wave_fields(cfg, build_grid(cfg)).views
    rec = BatchReconstructor(cfg, 1, e_inc=e_inc)
    theta0 = torch.as_tensor(_theta0([cfg.rng_seed], rec.m0_eff), device="cuda")
    ref = rec.run([data[0]], seeds=[cfg.rng_seed], k_iters=k)[0]
    shards = [IncidenceShard(rec.ops, e_inc, data[0], mf=cfg.m_f, beta=cfg.beta, lambdas=rec.lambdas,
                             tau_b=cfg.tau_b, rank=r, world=W) for r in range(W)]
    tr = Timed(shards, theta0, graph=False, lr=cfg.learn_rate)     # warm-up instance
    tr.ev = []
    tr.train(2)
    del tr
    tr2 = Timed(shards, theta0, graph=False, lr=cfg.learn_rate)
    tr2.ev = []
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    trace = tr2.train(k).cpu().numpy()
    e1.record()
    torch.cuda.synchronize()
    tr2.check_errors()
    err = float(np.max(np.abs(trace - np.array([b.as_row() for b in ref.trace])) /
                       np.abs(np.array([b.as_row() for b in ref.trace]))))
    seg = {}
    for name, r, a, b in tr2.ev:
        seg.setdefault(name, {}).setdefault(r, []).append(a.elapsed_time(b))
    per = {n: {"max_rank_ms": max(float(np.mean(v)) for v in d.values()),
               "sum_ranks_ms": float(sum(np.mean(v) for v in d.values()))} for n, d in seg.items()}
    out = {"world_emulated": W, "iters": k, "emulated_ms_per_iter": e0.elapsed_time(e1) / k,
           "segments": per, "rank_compute_ms_per_iter": sum(p["max_rank_ms"] for p in per.values()),
           "trace_max_rel_err_vs_unsharded": err}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
