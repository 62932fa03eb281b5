"""Timings of the one-time components around the hot loop:
GPU operator build vs host scipy build, GPU forward solve (batched
BiCGStab) for one cfg5 scene and for the 256-scene cfg4 batch, GPU metrics.

    python tools/bench_setup.py            (prints one JSON line)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best, out


def main():
    from paper_2602_13805_b200 import build_array, build_grid, build_greens, plane_wave_fields
    from paper_2602_13805_b200.greens import build_greens_device, incident_fields_device
    from paper_2602_13805_b200.metrics import count_components_dev, relative_error_dev
    from paper_2602_13805_b200.scenes import rasterize
    from paper_2602_13805_b200.solver import solve_fields_gpu
    from paper_2602_13805_b200.workloads import baseline_config, baseline_scene, cfg4_scene
    out = {}
    cfg5 = baseline_config(5)
    g5, a5 = build_grid(cfg5), build_array(cfg5)
    t_gpu, _ = timed(lambda: build_greens_device(cfg5, a5, g5))
    t0 = time.perf_counter()
    build_greens(cfg5, a5, g5)
    t_host = time.perf_counter() - t0
    t_inc, _ = timed(lambda: incident_fields_device(cfg5, a5, g5, "plane"))
    out["operator_build_cfg5"] = {"gpu_s": t_gpu, "host_scipy_s": t_host, "incident_fields_gpu_s": t_inc}
    ops5 = build_greens_device(cfg5, a5, g5)
    e5 = incident_fields_device(cfg5, a5, g5, "plane")
    chi5 = rasterize(baseline_scene(5)[0], g5).values
    t_s5, (x, res, it) = timed(lambda: solve_fields_gpu(chi5, e5, ops5), reps=2)
    out["forward_solve_cfg5"] = {"gpu_s": t_s5, "iterations": it, "max_residual": float(res.max()),
                                 "reference_cpu_s_survey": 109.0}
    cfg4 = baseline_config(4)
    g4, a4 = build_grid(cfg4), build_array(cfg4)
    ops4 = build_greens_device(cfg4, a4, g4)
    e4 = plane_wave_fields(cfg4, g4).views
    chis = np.stack([rasterize(cfg4_scene(i)[0], g4).values for i in range(256)])
    t_s4, (x4, res4, it4) = timed(lambda: solve_fields_gpu(chis, e4, ops4), reps=2)
    out["forward_solve_cfg4_256_scenes"] = {"gpu_s": t_s4, "per_scene_ms": 1e3 * t_s4 / 256, "iterations": it4,
                                            "max_residual": float(res4.max()), "reference_cpu_s_per_scene_survey": 0.6}
    imgs = torch.as_tensor(chis, device="cuda")
    t_m, _ = timed(lambda: (relative_error_dev(imgs, imgs.flip(0), offset=1.0), count_components_dev(imgs, 1.5, 1.0)))
    out["metrics_256_images"] = {"gpu_s": t_m}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
