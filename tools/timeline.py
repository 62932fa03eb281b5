"""Kernel timeline of one replay of the 10-iteration training graph (measurement only).

    python tools/timeline.py [--cfg 2] [--scenes 1]
Prints per phase (mean over iterations 2-9): start offset within the iteration,
dependency-wait release, exit, and the gap to the previous kernel's exit.
"""
import argparse
import json
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
    rec = BatchReconstructor(cfg, a.scenes, e_inc=e_inc)
    dev = rec.dev
    dev.set_data(data)
    _, r0 = dev.bp_initialize()
    dev.net_setup(dev.init_alpha(r0))
    th = torch.as_tensor(_theta0(list(range(a.scenes)), rec.m0_eff), dtype=dev.rdt, device=dev.device).contiguous()
    th, m, v = dev.alloc_state(th)
    dev.train(th, m, v, 0, 20)
    rows = dev.timeline(th, m, v, 20)
    dev.check_errors()
    it0 = {}
    for i, p, e, w, x, _ in rows:
        it0.setdefault(i, e)
    per, stg = {}, {}
    prev_exit = {}
    for i, p, e, w, x, st in sorted(rows, key=lambda r: (r[0], r[2])):
        if 2 <= i <= 9:
            base = it0[i]
            gap = (w - prev_exit[i]) if i in prev_exit else float("nan")
            per.setdefault(p, []).append(((e - base) / 1e3, (w - base) / 1e3, (x - base) / 1e3, gap / 1e3,
                                          (x - w) / 1e3))
            if any(s is not None for s in st):
                stg.setdefault(p, []).append([(s - w) / 1e3 if s is not None else np.nan for s in st])
        prev_exit[i] = x
    iters = sorted(it0)
    period = np.diff([it0[i] for i in iters]).mean() / 1e3 if len(iters) > 1 else float("nan")
    print(f"iteration period {period:.2f} us (entry of fwd_l1 to the next)")
    print(f"{'phase':9s} {'entry':>8s} {'waited':>8s} {'exit':>8s} {'wait-prevexit':>14s} {'exit-waited':>12s}")
    out = {"period_us": period}
    for p, vals in per.items():
        mv = np.nanmean(np.array(vals), axis=0)
        print(f"{p:9s} {mv[0]:8.2f} {mv[1]:8.2f} {mv[2]:8.2f} {mv[3]:14.2f} {mv[4]:12.2f}")
        out[p] = [round(float(x), 2) for x in mv]
    for p, vals in stg.items():
        mv = np.nanmean(np.array(vals, dtype=float), axis=0)
        print(f"{p:9s} stages (us after the wait release, last CTA): " + " ".join(f"{v:6.2f}" for v in mv))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
