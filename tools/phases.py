"""Per-kernel live timing of one fused iteration (events between kernels), and
the graph-replayed per-iteration time, for a BASELINE workload.

    python tools/phases.py [--cfg 2] [--scenes 1] [--iters 20]
Environment knobs read by the library (experiments only): PDF_NET_CLUSTER,
PDF_VIEW_CLUSTER.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2602_13805_b200 import build_grid, plane_wave_fields  # noqa: E402
from paper_2602_13805_b200.api import BatchReconstructor, _theta0  # noqa: E402
from paper_2602_13805_b200.workloads import baseline_config, baseline_scene, cfg4_scene, synthesize_gpu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--scenes", type=int, default=1)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--dtype", default="f64")
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
    th0 = torch.as_tensor(_theta0(list(range(a.scenes)), rec.m0_eff), dtype=dev.rdt, device=dev.device).contiguous()
    th, m, v = dev.alloc_state(th0)
    ph = dev.profile_phases(th, m, v, 0, a.iters)
    th.copy_(th0); m.zero_(); v.zero_()
    tr = torch.zeros(200, a.scenes, 6, dtype=torch.float64, device=dev.device)
    dev.train(th, m, v, 0, 50, tr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th.copy_(th0); m.zero_(); v.zero_()
    e0.record()
    dev.train(th, m, v, 0, 200, tr)
    e1.record()
    torch.cuda.synchronize()
    dev.check_errors()
    out = {"env": {k: os.environ.get(k) for k in ("PDF_NET_CLUSTER", "PDF_VIEW_CLUSTER")},
           "scenes": a.scenes, "graph_us_per_iter": 1e3 * e0.elapsed_time(e1) / 200,
           "phases_us": {k: round(1e3 * t, 2) for k, t in ph.items()},
           "sum_us": round(1e3 * sum(ph.values()), 1), "final_total": float(tr[-1, 0, 5])}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
