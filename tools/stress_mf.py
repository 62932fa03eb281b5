"""Literal-m_f stress variants of the BASELINE configs (cfg2*/4* with
m_f = 15, cfg5* with m_f = 31): the same hot loop with 4 m_f^2 = 900 / 3844 modes
(spectral.py:52-54), i.e. 25.9 M and 473 M network parameters per scene.

    python tools/stress_mf.py [--which 2 4 5] [--scenes4 32] [--iters 20] [--check]

For each variant: allocate, initialise, train `iters` iterations from the
captured graph, time them with CUDA events, and print the time per iteration
against SURVEY's roofline restated for float64 (56 B per parameter at the
measured HBM peak + the physics flops at the measured DFMA peak).  --check
compares one cfg2* gradient with the numpy oracle (test infrastructure).
"""
import argparse
import json
import math
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_13805_b200 import build_grid, plane_wave_fields  # noqa: E402
from paper_2602_13805_b200.api import BatchReconstructor  # noqa: E402
from paper_2602_13805_b200.workloads import baseline_config, baseline_scene, cfg4_scene, synthesize_gpu  # noqa: E402


def peaks():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))["hbm_gbs"]
    except Exception:
        return 6545.6


def theta0(m0: int, scenes: int, seed: int) -> np.ndarray:
    """Reference-shaped initial weights (network.py:52-71) drawn with numpy's
    generator in float64; the draws here only need the reference's scale."""
    widths = [2 * m0, 4 * m0, 4 * m0, 2 * m0]
    out = []
    for s in range(scenes):
        rng = np.random.default_rng(seed + s)
        parts = []
        for i in range(3):
            fi, fo = widths[i], widths[i + 1]
            w = np.zeros((fo, fi)) if i == 2 else rng.standard_normal((fo, fi)) * math.sqrt(1.0 / fi)
            parts += [w.ravel(), np.zeros(fo)]
        out.append(np.concatenate(parts))
    return np.stack(out)


def run(cfg_id: int, mf: int, scenes: int, iters: int, check: bool) -> dict:
    cfg = replace(baseline_config(cfg_id), m_f=mf).validate()
    if scenes == 1:
        sc, rng, snr = baseline_scene(cfg_id)
        scs, rngs = [sc], [rng]
    else:
        pairs = [cfg4_scene(i) for i in range(scenes)]
        scs, rngs, snr = [p[0] for p in pairs], [p[1] for p in pairs], baseline_scene(4)[2]
    data, _ = synthesize_gpu(cfg, scs, rngs, snr)
    e_inc = plane_wave_fields(cfg, build_grid(cfg)).views
    rec = BatchReconstructor(cfg, scenes, e_inc=e_inc)
    dev = rec.dev
    dev.set_data(data)
    _, r0 = dev.bp_initialize()
    alpha0 = dev.init_alpha(r0)
    dev.net_setup(alpha0)
    m0 = rec.m0_eff
    th_host = theta0(m0, scenes, 0)
    np_ = th_host.shape[1]
    out = {"cfg": f"{cfg_id}*", "m_f": mf, "modes": m0, "scenes": scenes, "params_per_scene": int(np_),
           "theta_m_v_GB": round(3 * 8 * np_ * scenes / 1e9, 3)}
    if check:
        from oracle import pdf_oracle as O
        from paper_2602_13805_b200 import build_array
        from paper_2602_13805_b200.operators import build_greens
        arr = build_array(cfg)
        ops = build_greens(cfg, arr, build_grid(cfg))
        ctx = O.Context(data[0], e_inc, O.build_operators(cfg.wavenumber, cfg.doi_side, cfg.m1, cfg.m2, arr.rx_positions),
                        mf, cfg.beta, (cfg.lambda1, cfg.lambda2, cfg.lambda3), cfg.tau_b)
        del ops
        flat = th_host[0] + 0.02 * np.random.default_rng(9).standard_normal(np_)
        params = O.unflat(flat, O.init_net(m0, np.random.default_rng(0)))
        want, parts = O.grad_loss(params, alpha0[0].cpu().numpy(), ctx)
        got, bd = dev.grad_loss(torch.as_tensor(flat[None], device="cuda").contiguous())
        dev.check_errors()
        g = got[0].cpu().numpy()
        out["grad_rel_err_vs_oracle"] = float(np.linalg.norm(g - want) / np.linalg.norm(want))
        out["loss_rel_err_vs_oracle"] = float(abs(bd[0, 5].item() - parts["total"]) / abs(parts["total"]))
    th = torch.as_tensor(th_host, dtype=dev.rdt, device=dev.device).contiguous()
    th, m, v = dev.alloc_state(th)
    dev.train(th, m, v, 0, 10)             # capture + warm-up
    torch.cuda.synchronize()
    dev.check_errors()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dev.train(th, m, v, 10, iters)
    e1.record()
    torch.cuda.synchronize()
    dev.check_errors()
    us = e0.elapsed_time(e1) * 1e3 / iters
    M, n, R = cfg.m1, cfg.n_tx, cfg.n_rx
    P = 2 * M
    K = 2 * mf
    f_phys = n * (2 * (10 * P * P * math.log2(P * P) + 6 * P * P + 8 * (M * K * K + M * M * K)) + 16 * m0 * R)
    fp64 = 36.3                                          # TFLOP/s, the bench's live DFMA probe (pdf_fp64_probe)
    t_net = 56.0 * np_ / (peaks() * 1e3)                 # us
    t_phys = f_phys / (fp64 * 1e6)                       # us
    out.update({"us_per_iteration": round(us, 2), "us_per_scene_iteration": round(us / scenes, 2),
                "t_roof_us_per_scene_iteration": round(t_net + t_phys, 2), "t_net_us": round(t_net, 2),
                "t_phys_us": round(t_phys, 2), "path_roofline_frac": round((t_net + t_phys) * scenes / us, 3),
                "peak_mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 2),
                "final_theta_finite": bool(torch.isfinite(th).all().item())})
    del rec, dev, th, m, v
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", type=int, nargs="*", default=[2, 4, 5])
    ap.add_argument("--scenes4", type=int, default=32)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    res = []
    for c in a.which:
        mf = 31 if c == 5 else 15
        scenes = a.scenes4 if c == 4 else 1
        torch.cuda.reset_peak_memory_stats()
        r = run(c, mf, scenes, a.iters, a.check and c == 2)
        print(json.dumps(r), flush=True)
        res.append(r)
    return res


if __name__ == "__main__":
    main()
