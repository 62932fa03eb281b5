"""Profiling driver: set up one BASELINE workload and run a few un-graphed
fused iterations (for ncu / compute-sanitizer).  Not a benchmark.

    python tools/prof_step.py [--cfg 2] [--scenes 1] [--iters 3] [--dtype f64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_13805_b200 import build_grid, plane_wave_fields  # noqa: E402
from paper_2602_13805_b200.api import BatchReconstructor, _theta0  # noqa: E402
from paper_2602_13805_b200.workloads import baseline_config, baseline_scene, cfg4_scene, synthesize_gpu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--scenes", type=int, default=1)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--graph", action="store_true")
    a = ap.parse_args()
    cfg = baseline_config(a.cfg)
    if a.scenes == 1:
        sc, rng, snr = baseline_scene(a.cfg)
        scenes, rngs = [sc], [rng]
    else:
        pairs = [cfg4_scene(i) for i in range(a.scenes)]
        scenes, rngs, snr = [p[0] for p in pairs], [p[1] for p in pairs], baseline_scene(4)[2]
    data, _ = synthesize_gpu(cfg, scenes, rngs, snr)
    e_inc = plane_wave_fields(cfg, build_grid(cfg)).views
    rec = BatchReconstructor(cfg, a.scenes, e_inc=e_inc, dtype=a.dtype)
    dev = rec.dev
    dev.set_data(data)
    _, r0 = dev.bp_initialize()
    dev.net_setup(dev.init_alpha(r0))
    th = torch.as_tensor(_theta0(list(range(a.scenes)), rec.m0_eff), dtype=dev.rdt, device=dev.device).contiguous()
    m, v = torch.zeros_like(th), torch.zeros_like(th)
    trace = torch.zeros(a.iters, a.scenes, 6, dtype=torch.float64, device=dev.device)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("iters")
    dev.train(th, m, v, 0, a.iters, trace, use_graph=a.graph)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    dev.check_errors()
    print("ok", trace[-1, 0].cpu().numpy())


if __name__ == "__main__":
    main()
