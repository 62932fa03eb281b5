"""Host-side breakdown of one BatchReconstructor.run (measurement only).

    python tools/e2e_breakdown.py [--cfg 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_13805_b200 import build_grid, plane_wave_fields  # noqa: E402
from paper_2602_13805_b200.api import BatchReconstructor  # noqa: E402
from paper_2602_13805_b200.workloads import baseline_config, baseline_scene, synthesize_gpu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    a = ap.parse_args()
    cfg = baseline_config(a.cfg)
    sc, rng, snr = baseline_scene(a.cfg)
    data, _ = synthesize_gpu(cfg, [sc], [rng], snr)
    e_inc = plane_wave_fields(cfg, build_grid(cfg)).views
    rec = BatchReconstructor(cfg, 1, e_inc=e_inc)
    for _ in range(3):
        rec.run([data[0]])
    dev = rec.dev
    orig = {}
    times = {}

    def wrap(obj, name):
        f = getattr(obj, name)
        orig[name] = f

        def g(*args, **kw):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = f(*args, **kw)
            torch.cuda.synchronize()
            times[name] = times.get(name, 0.0) + time.perf_counter() - t
            return r
        setattr(obj, name, g)

    for nm in ("set_data", "bp_initialize", "init_alpha", "net_setup", "train", "net_forward", "loss_value",
               "apply_cco", "check_errors"):
        wrap(dev, nm)
    reps = 5
    t = time.perf_counter()
    for _ in range(reps):
        rec.run([data[0]])
    tot = (time.perf_counter() - t) / reps
    print(f"run total {1e3 * tot:.2f} ms")
    for k, v in times.items():
        print(f"  {k:14s} {1e3 * v / reps:8.3f} ms")
    print(f"  other (host)   {1e3 * (tot - sum(times.values()) / reps):8.3f} ms")


if __name__ == "__main__":
    main()
