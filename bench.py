#!/usr/bin/env python
"""PDF solver hot-path benchmark on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json metric, config 2): one 64x64 scene, 16 plane-wave
incidences, 32 receivers, m_f = 8 (15x15 modes), 500 Adam iterations.
A STEP is one full 500-iteration optimisation loop of that scene with its
inputs (data, alpha0, operators) resident in HBM; L2 is flushed between
steps.  value = whole-job iterations/s (N GPUs each run their own scene,
weak scaling, no collective).  e2e = the same metric through the public
API (BatchReconstructor.run on HOST data: H2D, bp_initialize, init_alpha,
the initial-weight draws, the loop, forward_net + loss_total +
recover_contrast + CCO + relative_error, D2H).
`batched` adds the config-4 form: S scenes per GPU reconstructed together
(scenes/s); `large` the config-5 form (one 256x256 scene).  Every leg
carries a roofline block computed from the kernels' IN-GRAPH durations
(globaltimer stamps inside the replayed CUDA graph, pdf_timeline).
--impl reference times the CPU oracle port of the reference algorithm on
the host cores on the same workload.  --gpus N without torchrun re-launches
itself under torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "PDF solver iter/s (fwd+bwd) and scenes/s at 64x64, 16 inc; % of roofline"
WORKLOAD = ("cfg2: 64x64 grid on [-1,1] lambda, 16 plane-wave incidences, 32 receivers at 3 lambda, "
            "m_f=8 (15x15 modes), beta=6, CIE+bridge loss, 500 Adam iterations per reconstruction")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--iters", type=int, default=500)
    ap.add_argument("--batch", type=int, default=256, help="scenes for the batched (config 4) leg; 0 = skip")
    ap.add_argument("--batch-steps", type=int, default=2)
    ap.add_argument("--cpu-sample-iters", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--large-iters", type=int, default=300, help="iterations of the config-5 leg; 0 = skip")
    ap.add_argument("--no-timeline", action="store_true", help="skip the in-graph kernel timing (ncu runs)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the config-5 leg through the multi-GPU (incidence-sharded) code path even on one "
                         "rank (a one-rank NCCL group; path validation on a one-GPU box)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- dist
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def spawn(args) -> int:
    """`--gpus N` outside torchrun: re-launch this script with N ranks (one per GPU)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


class Dist:
    def __init__(self, gpus, force: bool = False):
        self.rank, self.world, self.local = dist_env()
        self.pg = None
        if force and self.world == 1:
            os.environ.setdefault("MASTER_PORT", "29555")
        if self.world > 1 or force:
            import torch
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if torch.cuda.is_available():
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local), rank=self.rank,
                                        world_size=self.world)
            else:        # CPU-only host: the reference arm still runs (rank 0), the ranks meet over gloo
                dist.init_process_group("gloo")
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.th = None

    def _nvml(self):
        """NVML handle for fast sampling (a query takes well under a millisecond, so the
        ~0.2 s headline region gets tens of samples); None: fall back to nvidia-smi."""
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = self.index
            if vis:
                ids = [x.strip() for x in vis.split(",") if x.strip()]
                if self.index < len(ids) and ids[self.index].isdigit():
                    idx = int(ids[self.index])
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)
        except Exception:
            return None

    def _run(self):
        nv = self._nvml()
        if nv is not None:
            pynvml, h = nv
            bits = ((0x8, 3), (0x40, 4), (0x20, 5), (0x4, 6))   # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            try:
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            except Exception:
                mx = 0
            while not self.stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    try:
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except Exception:
                        rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    row = [str(sm), str(mx), "", "", "", "", ""]
                    for bit, pos in bits:
                        row[pos] = "Active" if rs & bit else "Not Active"
                    self.samples.append(row)
                except Exception:
                    pass
                self.stop.wait(0.005)
            return
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- host description
def host_info() -> dict:
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    import scipy
    return {"cpu_model": model, "nproc": os.cpu_count(), "numpy": np.__version__, "scipy": scipy.__version__,
            "python": platform.python_version()}


def pdf_env() -> dict:
    """Every PDF_* variable set for this run (library knobs; all unset in the driver's runs)."""
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("PDF_")}


# ----------------------------------------------------------------------------- CPU oracle
def _oracle_problem(cfg_id: int, scene_idx: int = 0):
    from oracle import pdf_oracle as O
    from paper_2602_13805_b200 import build_array, build_grid, plane_wave_fields
    from paper_2602_13805_b200.scenes import rasterize
    from paper_2602_13805_b200.workloads import baseline_config, baseline_scene
    cfg = baseline_config(cfg_id)
    grid, arr = build_grid(cfg), build_array(cfg)
    e_inc = plane_wave_fields(cfg, grid).views
    ops = O.build_operators(cfg.wavenumber, cfg.doi_side, cfg.m1, cfg.m2, arr.rx_positions)
    scene = baseline_scene(cfg_id, scene_idx)[0]
    chi = rasterize(scene, grid).values
    jt = chi * e_inc   # Born-level current: the step cost does not depend on the data values
    data = jt.reshape(cfg.n_tx, -1) @ ops.gs.T
    ctx = O.Context(data, e_inc, ops, cfg.m_f, cfg.beta, (cfg.lambda1, cfg.lambda2, cfg.lambda3), cfg.tau_b)
    return cfg, O, ops, e_inc, data, ctx


def cpu_oracle_rate(iters: int, threads: int | None):
    """Iterations/s of the oracle port of the reference loop (grad_loss + Adam) on host cores."""
    from threadpoolctl import threadpool_limits
    cfg, O, ops, e_inc, data, ctx = _oracle_problem(2)
    chi0, r0 = O.bp_initialize(data, e_inc, ops, cfg.beta)
    a0 = O.init_alpha(r0, data, e_inc, ops, cfg.m_f, cfg.beta)
    params = O.init_net(4 * cfg.m_f ** 2, np.random.default_rng(cfg.rng_seed))
    theta = O.flat(params)
    adam = O.Adam(m=np.zeros_like(theta), v=np.zeros_like(theta), lr=cfg.learn_rate)
    with threadpool_limits(limits=threads):
        g, _ = O.grad_loss(O.unflat(theta, params), a0, ctx)   # warm
        t0 = time.perf_counter()
        for _ in range(iters):
            g, _ = O.grad_loss(O.unflat(theta, params), a0, ctx)
            theta = O.adam_update(adam, theta, g)
        dt = time.perf_counter() - t0
    return iters / dt, dt


def cpu_baseline(iters: int):
    ncores = os.cpu_count() or 1
    best = None
    for th in (1, ncores):
        rate, dt = cpu_oracle_rate(iters, th)
        if best is None or rate > best[0]:
            best = (rate, dt, th)
    return {"value": best[0], "unit": "iter/s", "cores": best[2], "kind": "port",
            "sample": f"{iters} iterations of the cfg2 loop (grad_loss + Adam, oracle/pdf_oracle.py numpy port), "
                      f"best of 1 and {ncores} BLAS threads, {best[1]:.2f} s",
            "host": host_info()}


def _pool_scene(args):
    """One worker of the config-4 process-pool baseline: one scene, single-threaded BLAS."""
    idx, iters = args
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        cfg, O, ops, e_inc, data, ctx = _oracle_problem(4, idx)
        t1 = time.perf_counter()
        chi0, r0 = O.bp_initialize(data, e_inc, ops, cfg.beta)
        a0 = O.init_alpha(r0, data, e_inc, ops, cfg.m_f, cfg.beta)
        params = O.init_net(4 * cfg.m_f ** 2, np.random.default_rng(idx))
        theta = O.flat(params)
        adam = O.Adam(m=np.zeros_like(theta), v=np.zeros_like(theta), lr=cfg.learn_rate)
        t2 = time.perf_counter()
        for _ in range(iters):
            g, _ = O.grad_loss(O.unflat(theta, params), a0, ctx)
            theta = O.adam_update(adam, theta, g)
        t3 = time.perf_counter()
    return t1 - t0, t2 - t1, t3 - t2


def cpu_pool_baseline(iters: int, k_full: int = 500) -> dict:
    """Config-4 CPU baseline as the reference runs many scenes (studies.py:271-275):
    a process pool, one scene per core, each timing initialisation (bp_initialize
    + init_alpha + init_network) and `iters` loop iterations; scenes/s for the
    full k-iteration reconstruction extrapolated from the per-iteration rate.
    Operator build and data synthesis are excluded, as SURVEY 8(d) specifies."""
    from concurrent.futures import ProcessPoolExecutor
    ncores = os.cpu_count() or 1
    with ProcessPoolExecutor(max_workers=ncores) as ex:
        t0 = time.perf_counter()
        res = list(ex.map(_pool_scene, [(i, iters) for i in range(ncores)]))
        wall = time.perf_counter() - t0
    init = float(np.mean([r[1] for r in res]))
    per_it = float(np.mean([r[2] for r in res])) / iters
    per_scene = init + k_full * per_it
    return {"value": ncores / per_scene, "unit": "scenes/s", "cores": ncores, "kind": "port",
            "sample": f"{ncores} config-4 scenes in a {ncores}-process pool (one per core, 1 BLAS thread), "
                      f"init + {iters} iterations each ({wall:.1f} s wall); per scene {init * 1e3:.0f} ms init + "
                      f"{k_full} x {per_it * 1e3:.1f} ms",
            "host": host_info()}


def run_reference(args, d: Dist):
    if d.rank != 0:
        return
    k = args.cpu_sample_iters
    for _ in range(args.warmup):
        cpu_oracle_rate(1, None)
    rates, times = [], []
    ncores = os.cpu_count() or 1
    for _ in range(args.steps):
        r, dt = cpu_oracle_rate(k, ncores)
        r1, dt1 = cpu_oracle_rate(k, 1)
        rates.append(max(r, r1))
        times.append(min(dt, dt1))
    v = float(np.median(rates))
    line = {"metric": METRIC, "value": v, "unit": "iter/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.median(times)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128/f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "sample_iters_per_step": k},
            "cpu_baseline": {"value": v, "unit": "iter/s", "cores": ncores, "kind": "port",
                             "sample": f"{k} iterations per step of the cfg2 loop, numpy oracle port "
                                       f"(reference is pure Python; best of 1 / {ncores} BLAS threads)",
                             "host": host_info()},
            "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- roofline
def algorithmic_work(dev, phase: str, in_graph: bool = False, fp64_tflops: float = 36.2, hbm_gbs: float = 6453.4):
    """(bound, work) per launch: algorithmic bytes of an HBM-bound kernel or FP64
    flops of a compute-bound one.  The network layers
    carry both (W / m / v bytes and 2 rows N K DMMA flops per product); the
    binding one -- the larger of bytes / HBM peak and flops / FP64 peak -- is
    reported (HBM at 16 rows, FP64 from ~40 rows on: config 5's 72 rows).
    in_graph: the split-backward layout of the captured single-scene graph,
    where bwd_l1 is layer 1's g_W + Adam only (layers 3 / 2 on a side branch)."""
    M, P, n, R, S = dev.M, 2 * dev.M, dev.n, dev.R, dev.S
    K = 2 * dev.mf
    rows, D0, H = dev.rows, dev.d0, dev.hidden
    es = 8 if dev.rdt.itemsize == 8 else 4
    cs = 2 * es
    lg = np.log2(P * P)
    if phase in ("view_fwd", "view_bwd"):
        fft = 2 * 5 * P * P * lg + 6 * P * P                  # forward + inverse padded 2-D FFT, x K^
        spec = 8 * (M * K * K + M * M * K)                     # corner-sparse DFT contraction
        data = 8 * K * K * R                                   # D = alpha H^T row / g_rows conj(H) (H = G_S o expand)
        return "fp64", S * n * (fft + spec + data)
    if phase == "pixel":
        return "hbm", S * 4 * n * M * M * cs                   # J, E read; g_J, g_E written
    layer = {"fwd_l1": (H, D0), "fwd_l2": (H, H), "fwd_l3": (D0, H),
             "bwd_l1": (H, D0), "bwd_l2": (H, H), "bwd_l3": (D0, H)}.get(phase)
    if layer is None:
        return None, 0
    N_, K_ = layer
    if phase.startswith("fwd"):
        b, f = S * es * (N_ * K_ + rows * K_ + rows * N_), S * 2.0 * rows * N_ * K_
    elif getattr(dev, "split_bwd", False):
        # split backward: bwd_l3 / bwd_l2 = g_h kernels (W_old read, g_z and h read,
        # g_z' written); bwd_l1 = g_W + Adam (W, m, v read + written)
        if phase in ("bwd_l3", "bwd_l2"):
            b, f = S * es * (N_ * K_ + rows * (N_ + 2 * K_)), S * 2.0 * rows * N_ * K_
        elif in_graph and graph_fork(dev):
            b, f = S * es * (6 * (H * D0 + H) + rows * (H + D0)), S * 2.0 * rows * H * D0
        else:
            weights = H * D0 + H * H + D0 * H
            b, f = S * es * (6 * (weights + 2 * H + D0) + rows * (2 * H + D0) * 2), S * 2.0 * rows * weights
    else:
        b, f = S * es * (6 * N_ * K_ + rows * (K_ + 2 * N_)), S * 4.0 * rows * N_ * K_
    if f / (fp64_tflops * 1e12) > b / (hbm_gbs * 1e9):
        return "fp64", f
    return "hbm", b


def graph_fork(dev) -> bool:
    """The captured graph of this context runs layers 3 / 2 of Adam on a side branch."""
    return bool(dev.split_bwd and dev.rows <= 16 and dev.hidden <= 1024 and dev.d0 <= 1024 and dev.rdt.itemsize == 8)


def graph_phases(dev, theta, m, v) -> tuple[dict, float]:
    """Per-phase kernel durations INSIDE the replayed CUDA graph (mean over
    iterations 1-9 of one 10-iteration replay: last CTA exit minus the first
    CTA past the dependency wait, globaltimer stamps) and the iteration period
    (entry of one iteration's first kernel to the next), both in microseconds."""
    rows = dev.timeline(theta, m, v, 0)
    per, entry = {}, {}
    for i, p, e, w, x, _ in rows:
        entry[i] = min(entry.get(i, e), e)
        if i >= 1:
            per.setdefault(p, []).append((x - w) / 1e3)
    its = sorted(entry)
    period = float(np.mean(np.diff([entry[i] for i in its]))) / 1e3 if len(its) > 1 else float("nan")
    return {p: float(np.mean(vs)) for p, vs in per.items()}, period


def roofline_table(dev, phases_us: dict, period_us: float, fp64_tflops: float, hbm_gbs: float,
                   in_graph: bool = True) -> dict:
    out = {}
    for p, us in phases_us.items():
        bound, work = algorithmic_work(dev, p, in_graph, fp64_tflops, hbm_gbs)
        if bound is None or us <= 0:
            continue
        if bound == "hbm":
            ach, peak, unit = work / (us * 1e-6) / 1e9, hbm_gbs, "GB/s"
        else:
            ach, peak, unit = work / (us * 1e-6) / 1e12, fp64_tflops, "TFLOP/s"
        out[p] = {"bound": bound, "us": us, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                  "algorithmic_per_launch": work, "share_of_step": us / period_us if period_us else None}
    return out


def dominant_roofline(table: dict, peak_notes: dict, traffic=None) -> dict:
    dom = max(table, key=lambda p: table[p]["us"])
    t = table[dom]
    r = {"bound": t["bound"], "achieved": t["achieved"], "peak": t["peak"], "unit": t["unit"], "frac": t["frac"],
         "traffic": traffic, "kernel": dom, "algorithmic_per_launch": t["algorithmic_per_launch"],
         "launch_ms": t["us"] / 1e3, "share_of_step": t["share_of_step"],
         "timing": "in-graph: globaltimer stamps of the replayed CUDA graph (last CTA exit - first CTA past the "
                   "dependency wait), mean over 9 iterations",
         "peak_source": peak_notes[t["bound"]]}
    return r


PHASE_REGEX = {"view_fwd": r"view_kernel<double, \d+, 0,", "view_bwd": r"view_kernel<double, \d+, 1,",
               "pixel": r"pixel_kernel<double, 1"}


def ncu_traffic(phase: str, tag: str) -> dict | None:
    """Mean DRAM bytes (read + write) per launch of the phase's kernel from the
    committed ncu launch list of this bench leg (profiles/*_launches_<tag>.csv.gz),
    else None.  ncu flushes caches before each launch (cold), and writes still
    in L2 when a kernel ends are not counted."""
    import csv
    import glob
    import gzip
    import re
    files = sorted(glob.glob(os.path.join(HERE, "profiles", f"*_launches_{tag}.csv.gz")))
    rx = PHASE_REGEX.get(phase)
    if not files or not rx:
        return None
    try:
        rows = list(csv.reader(gzip.open(files[-1], "rt")))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hi]
        ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
        ui = h.index("Metric Unit")
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        per = {}
        for r in rows[hi + 1:]:
            if re.search(rx, r[ki]) and r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                per[int(r[idi])] = per.get(int(r[idi]), 0.0) + float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        vals = list(per.values())
        return {"bytes_per_launch": float(np.mean(vals)), "launches": len(vals),
                "source": os.path.relpath(files[-1], HERE)} if vals else None
    except Exception:
        return None


def path_roofline(M: int, n: int, R: int, np_params: int, fp64_tflops: float, hbm_gbs: float,
                  m0: int | None = None) -> dict:
    """SURVEY 8(d) path roofline per scene-iteration, restated for float64:
    F_phys = n [20 P^2 log2 P^2 + 12 P^2 + 10 M^2 log2 M^2 + 16 M^2 R] flop at the
    FP64 peak, B_net = 56 Np bytes (W read forward, W/m/v read + written by the
    fused backward/Adam) at the HBM peak.  This implementation contracts the
    data term over the M0 spectral coefficients (H = G_S o expand),
    so the bound of the work it executes replaces 16 M^2 R by 16 M0 R; `frac`
    uses that (smaller, stricter) bound, F_phys_reference_flop is SURVEY's."""
    P = 2 * M
    base = 20 * P * P * np.log2(P * P) + 12 * P * P + 10 * M * M * np.log2(M * M)
    f_ref = n * (base + 16 * M * M * R)
    f = n * (base + 16 * (m0 if m0 else M * M) * R)
    b = 56.0 * np_params
    t_phys = f / (fp64_tflops * 1e12)
    t_net = b / (hbm_gbs * 1e9)
    return {"F_phys_flop": float(f), "F_phys_reference_flop": float(f_ref), "B_net_bytes": b,
            "t_phys_us": 1e6 * t_phys, "t_net_us": 1e6 * t_net, "t_roof_us_per_scene_iter": 1e6 * (t_phys + t_net)}


def leg_rooflines(dev, theta0, fp64, hbm, notes, args) -> dict:
    """In-graph per-kernel roofline table of a context + its dominant kernel."""
    if args.no_timeline:
        return {}
    th, m, v = dev.alloc_state(theta0)
    ph, period = graph_phases(dev, th, m, v)
    dev.check_errors()
    table = roofline_table(dev, ph, period, fp64, hbm)
    return {"dominant": dominant_roofline(table, notes), "kernels": table, "iteration_period_us": period}


# ----------------------------------------------------------------------------- legs
def large_leg(args, d: Dist, fp64, hbm, notes):
    """BASELINE config 5: one 256x256 scene, 72 incidences / receivers, m_f = 16.
    N = 1: the whole scene on one GPU (CUDA-graph replay).  N > 1: incidences
    sharded over the ranks (sharded.py), timed in three forms (peer-scatter,
    zero1-nccl, tensor-parallel); the fastest is the headline."""
    import torch
    from paper_2602_13805_b200 import build_grid, plane_wave_fields
    from paper_2602_13805_b200.api import BatchReconstructor, _theta0
    from paper_2602_13805_b200.sharded import (IncidenceShard, PeerTrainer, ShardedTrainer, TensorParallelTrainer,
                                               TorchDistReducer, run_sharded)
    from paper_2602_13805_b200.workloads import baseline_config, baseline_scene, synthesize_gpu
    k = args.large_iters
    cfg = baseline_config(5, k_iters=k)
    scene, rng, snr = baseline_scene(5)
    data, chi_true = synthesize_gpu(cfg, [scene], [rng], snr)
    e_inc = plane_wave_fields(cfg, build_grid(cfg)).views
    rec = BatchReconstructor(cfg, 1, e_inc=e_inc, dtype=args.dtype)
    theta0 = torch.as_tensor(_theta0([cfg.rng_seed], rec.m0_eff), dtype=rec.dev.rdt, device=rec.dev.device)
    out = {"workload": "cfg5: 256x256 on [-2,2] lambda, 72 plane-wave incidences, 72 receivers at 5 lambda, "
                       f"m_f=16 (31x31 modes, 33.6 M network parameters), {k} Adam iterations; scene: 6 "
                       "non-overlapping ellipses, semi-axes U[0.2,0.6] lambda, chi = U[0.5,2.5] + i U[0,0.5], seed 3"}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if d.world == 1 and not args.force_sharded:
        dev = rec.dev
        dev.set_data(data)
        _, r0 = dev.bp_initialize()
        dev.net_setup(dev.init_alpha(r0))
        th, m, v = dev.alloc_state(theta0)
        tr = torch.zeros(k, 1, 6, dtype=torch.float64, device=dev.device)
        dev.train(th, m, v, 0, 20, tr)
        th.copy_(theta0); m.zero_(); v.zero_()
        torch.cuda.synchronize()
        e0.record()
        dev.train(th, m, v, 0, k, tr)
        e1.record()
        torch.cuda.synchronize()
        dev.check_errors()
        secs = e0.elapsed_time(e1) / 1e3
        th.copy_(theta0); m.zero_(); v.zero_()
        out.update({"mode": "single GPU, CUDA graph", "phases_ms_events": dev.profile_phases(th, m, v, 0, 5),
                    "final_loss_total": float(tr[-1, 0, 5])})
        pr = path_roofline(dev.M, dev.n, dev.R, int(dev.n_params), fp64, hbm, m0=4 * dev.mf ** 2)
        pr["frac"] = pr["t_roof_us_per_scene_iter"] * k / (1e6 * secs)
        out["path_roofline"] = pr
        out["roofline"] = leg_rooflines(dev, theta0, fp64, hbm, notes, args)
        del dev
    else:
        c = cfg
        err = None
        try:
            sh = IncidenceShard(rec.ops, e_inc, data[0], mf=c.m_f, beta=c.beta, lambdas=rec.lambdas, tau_b=c.tau_b,
                                rank=d.rank, world=d.world)
        except Exception as ex:      # every rank must agree before the first collective of the loop
            err = f"{type(ex).__name__}: {ex}"
        if d.max(1.0 if err else 0.0) > 0:
            raise RuntimeError(err or "incidence-shard setup failed on another rank")
        # three multi-GPU forms, each timed over the same k iterations (CUDA-graph replay):
        #   peer-scatter: the gradient reduce-scatter fused into the backward kernels (g_W / g_b
        #     stored by the DMMA epilogue into the owner rank's symmetric-memory receive buffer over
        #     NVLink), owner-side Adam with the parameter all-gather as peer stores
        #   zero1-nccl: per-layer reduce-scatter (NCCL) on a comm stream overlapping the next
        #     layer's backward, sharded Adam, NCCL all-gather
        #   tensor-parallel: W1 / W3 rows and W2 columns per rank with their Adam state; four
        #     activation-sized all-reduces instead of any gradient / parameter exchange
        # every rank takes the same branches (the collective sequences must match)
        import torch.distributed as tdist
        forms = {}
        makers = (("peer-scatter", lambda: PeerTrainer([sh], theta0, group=tdist.group.WORLD, graph=True)),
                  ("zero1-nccl", lambda: ShardedTrainer(sh, theta0, graph=True)),
                  ("tensor-parallel", lambda: TensorParallelTrainer([sh], theta0, group=tdist.group.WORLD, graph=True,
                                                                    lr=c.learn_rate)))
        tr = None
        for name, make in makers:
            try:
                trn = make()
                trn.train(10)
                torch.cuda.synchronize()
                bad = None
            except Exception as ex:      # noqa: BLE001 -- reported in the line
                bad, trn = f"{type(ex).__name__}: {ex}", None
            if d.max(1.0 if bad else 0.0) > 0:
                forms[name] = {"error": bad or "failed on another rank"}
                continue
            d.barrier()
            e0.record()
            tr_k = trn.train(k)
            e1.record()
            torch.cuda.synchronize()
            s_k = d.max(e0.elapsed_time(e1) / 1e3)
            forms[name] = {"ms_per_iter": 1e3 * s_k / k, "iter_per_s": k / s_k,
                           "final_loss_total": float(tr_k[-1, 5])}
            if tr is None or s_k < secs:
                tr, secs, best = tr_k, s_k, name
            del trn
            torch.cuda.empty_cache()
        if tr is None:      # neither form ran: replicated Adam, eager NCCL loop
            red = TorchDistReducer()
            d.barrier()
            e0.record()
            _, tr = run_sharded([sh], red, theta0, k, trace_on_device=True)
            e1.record()
            torch.cuda.synchronize()
            secs, best = d.max(e0.elapsed_time(e1) / 1e3), "replicated-eager"
        out.update({"mode": f"incidence-sharded over {d.world} GPUs ({len(sh.own)} views on rank {d.rank}); "
                            f"headline form: {best}", "forms": forms, "final_loss_total": float(tr[-1, 5])})
    out.update({"iter_per_s": k / secs, "ms_per_iter": 1e3 * secs / k, "s_per_reconstruction": secs,
                "scaling": "strong (one scene, incidences split over the GPUs)"})
    return out


def batched_leg(args, d: Dist, e_inc, fp64, hbm, notes):
    """BASELINE config 4 form: S scenes per GPU reconstructed together."""
    import torch
    from paper_2602_13805_b200.api import BatchReconstructor, _theta0
    from paper_2602_13805_b200.workloads import SNR_5PCT, baseline_config, cfg4_scene, synthesize_gpu
    k = args.iters
    S = max(1, args.batch // d.world)
    cfg4 = baseline_config(4, k_iters=k)
    idx = list(range(d.rank * S, (d.rank + 1) * S))
    sc = [cfg4_scene(i) for i in idx]
    datab, chib = synthesize_gpu(cfg4, [s for s, _ in sc], [r for _, r in sc], SNR_5PCT)
    rb = BatchReconstructor(cfg4, S, e_inc=e_inc, dtype=args.dtype, theta_cache=False)
    # batch pipeline: each run draws the NEXT batch's reference-identical
    # initial weights on the host cores while its own batch trains (the
    # next batch here is the same seeds again; weights are never cached)
    rb.run(list(datab), seeds=idx, k_iters=k, prefetch_seeds=idx)          # warm-up
    torch.cuda.synchronize()
    d.barrier()
    tb0 = time.perf_counter()
    for _ in range(args.batch_steps):
        outb = rb.run(list(datab), seeds=idx, chi_trues=list(chib), k_iters=k, prefetch_seeds=idx)
    torch.cuda.synchronize()
    tb = d.max((time.perf_counter() - tb0) / args.batch_steps)
    # device-resident batched loop only
    devb = rb.dev
    th0 = torch.as_tensor(_theta0(idx, rb.m0_eff), dtype=devb.rdt, device=devb.device)
    thb, mb, vb = devb.alloc_state(th0)
    trb = torch.zeros(k, S, 6, dtype=torch.float64, device=devb.device)
    devb.train(thb, mb, vb, 0, k, trb)
    torch.cuda.synchronize()
    eb0, eb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    thb.copy_(th0); mb.zero_(); vb.zero_()
    eb0.record()
    devb.train(thb, mb, vb, 0, k, trb)
    eb1.record()
    torch.cuda.synchronize()
    tdev = d.max(eb0.elapsed_time(eb1) / 1e3)
    thb.copy_(th0); mb.zero_(); vb.zero_()
    phb = devb.profile_phases(thb, mb, vb, 0, 3)
    devb.check_errors()
    rels = [o.rel_error for o in outb]
    proof_b = path_roofline(devb.M, devb.n, devb.R, int(devb.n_params), fp64, hbm, m0=4 * devb.mf ** 2)
    proof_b["frac"] = proof_b["t_roof_us_per_scene_iter"] * S * k / (1e6 * tdev)
    out = {"workload": f"cfg4: {S * d.world} scenes of 1-4 random ellipses (semi-axes U[0.15,0.5] lambda, "
                       f"chi U[0.5,3], seed = scene index), {S} per GPU, {k} iterations each",
           "scenes_per_s": d.world * S / tdev, "iter_per_s": d.world * S * k / tdev,
           "e2e_scenes_per_s": d.world * S / tb, "s_per_batch": tdev, "e2e_s_per_batch": tb,
           "e2e_pipeline": "BatchReconstructor.run(host data, prefetch_seeds=next batch): the next "
                           "batch's initial-weight draws overlap this batch's GPU work",
           "median_rel_error": float(np.median(rels)), "phases_ms_events": phb, "path_roofline": proof_b,
           "scaling": "strong (256 scenes split over the GPUs)"}
    out["roofline"] = leg_rooflines(devb, th0, fp64, hbm, notes, args)
    if d.rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_pool_baseline(args.cpu_sample_iters)
    return out


def run_ours(args, d: Dist):
    import ctypes as ct

    import torch
    from paper_2602_13805_b200 import _native as N
    from paper_2602_13805_b200 import build_grid, plane_wave_fields
    from paper_2602_13805_b200.api import BatchReconstructor, _theta0
    from paper_2602_13805_b200.workloads import baseline_config, baseline_scene, cfg4_scene, synthesize_gpu

    torch.cuda.set_device(d.local)
    k = args.iters
    cfg = baseline_config(2, k_iters=k)
    # each rank reconstructs its own scene: config-2 geometry, scene/noise seeds offset by rank
    scene, rng, snr = baseline_scene(2)
    if d.rank:
        scene, rng = cfg4_scene(d.rank)[0], np.random.default_rng(1000 + d.rank)
    data, chi_true = synthesize_gpu(cfg, [scene], [rng], snr)
    e_inc = plane_wave_fields(cfg, build_grid(cfg)).views
    rec = BatchReconstructor(cfg, 1, e_inc=e_inc, dtype=args.dtype, theta_cache=False)
    dev = rec.dev
    dev.set_data(data)
    chi0, r0 = dev.bp_initialize()
    alpha0 = dev.init_alpha(r0)
    dev.net_setup(alpha0)
    theta0 = torch.as_tensor(_theta0([cfg.rng_seed], rec.m0_eff), dtype=dev.rdt, device=dev.device).contiguous()
    theta, m, v = dev.alloc_state(theta0)
    trace = torch.zeros(k, 1, 6, dtype=torch.float64, device=dev.device)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev.device)

    def step():
        theta.copy_(theta0)
        m.zero_()
        v.zero_()
        dev.train(theta, m, v, 0, k, trace, use_graph=True)

    for _ in range(max(args.warmup, 3)):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    dev.check_errors()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d.barrier()
    torch.cuda.synchronize()
    with ClockSampler(d.local) as clk:
        e0.record(st)
        for _ in range(args.steps):
            flush.fill_(1)      # L2 flush between steps (256 MiB write > 126 MB L2)
            step()
        e1.record(st)
        torch.cuda.synchronize()
    d.barrier()
    ms_total = d.max(e0.elapsed_time(e1))
    ms_step = ms_total / args.steps
    value = d.world * k / (ms_step / 1e3)
    dev.check_errors()
    final_total = float(trace[-1, 0, 5].item())

    # kernels per fused iteration of the captured graph: 3 forward layers,
    # view_fwd, pixel, view_bwd (loss finalize fused), then either 3 fused
    # backward layers with Adam, or (split backward, <= 16 rows, widths <= 1024)
    # g_h3, g_h2, Adam layer 1 on the main chain plus the side branch's data
    # GEMM, its reduce, gad and the Adam of layers 3 / 2
    fork = graph_fork(dev)
    launches_per_iter = 14 if fork else 9 + (2 if dev.data_gemm else 0)

    # ---- peaks: HBM from MEASURED_PEAKS.json; FP64 (not in that file) from a live DFMA probe
    g = ct.c_double()
    N.check(N.lib().pdf_fp64_probe(ct.byref(g), ct.c_void_p(torch.cuda.current_stream().cuda_stream)))
    fp64 = g.value / 1e3
    mp = os.path.join(HERE, "MEASURED_PEAKS.json")
    hbm = json.load(open(mp))["hbm_gbs"] if os.path.exists(mp) else 6650.0
    notes = {"hbm": "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)" if os.path.exists(mp) else
             "B200_PROFILING.md fallback",
             "fp64": "live DFMA probe (pdf_fp64_probe; MEASURED_PEAKS.json has no FP64 entry)"}

    # ---- per-kernel roofline from the kernels' in-graph durations
    theta.copy_(theta0); m.zero_(); v.zero_()
    phases_ev = dev.profile_phases(theta, m, v, 0, 20)      # un-graphed, event-bracketed (secondary)
    dev.check_errors()
    legroof = leg_rooflines(dev, theta0, fp64, hbm, notes, args)
    if legroof:
        roof = dict(legroof["dominant"])
        tr_info = ncu_traffic(roof["kernel"], "cfg2")
        roof["traffic"] = tr_info["bytes_per_launch"] if tr_info else None
        roof["traffic_source"] = tr_info
    else:
        roof = None
    proof = path_roofline(dev.M, dev.n, dev.R, int(dev.n_params), fp64, hbm, m0=4 * dev.mf ** 2)
    proof["frac"] = proof["t_roof_us_per_scene_iter"] / (1e3 * ms_step / k)

    # ---- e2e through the public API with host buffers (per step: H2D data and
    # chi_true, the reference-identical initial-weight draws for the run (drawn
    # for the NEXT run while this one trains: prefetch_seeds), D2H results)
    res = rec.run([data[0]], seeds=[cfg.rng_seed], chi_trues=[chi_true[0]], prefetch_seeds=[cfg.rng_seed])
    for _ in range(2):
        rec.run([data[0]], seeds=[cfg.rng_seed], chi_trues=[chi_true[0]], prefetch_seeds=[cfg.rng_seed])
    torch.cuda.synchronize()
    d.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = rec.run([data[0]], seeds=[cfg.rng_seed], chi_trues=[chi_true[0]], prefetch_seeds=[cfg.rng_seed])
    torch.cuda.synchronize()
    e2e_s = d.max((time.perf_counter() - t0) / args.steps)
    M = cfg.m1
    h2d = data[0].nbytes + M * M * 16 + int(dev.n_params) * 8     # data, chi_true, the run's initial weights
    d2h = 3 * M * M * 16 + k * 6 * 8 + 6 * 8 + 8

    # the other legs' timed regions are sampled as well: `clocks` is the headline
    # region, `clocks.by_leg` the batched and large legs (the 256-scene batch runs
    # into the software power cap)
    with ClockSampler(d.local) as clk_b:
        batched = batched_leg(args, d, e_inc, fp64, hbm, notes) if args.batch else None

    large = None
    with ClockSampler(d.local) as clk_l:
        if args.large_iters:
            try:
                large = large_leg(args, d, fp64, hbm, notes)
            except Exception as ex:   # reported, never fatal for the headline line
                large = {"error": f"{type(ex).__name__}: {ex}"}
    by_leg = {"batched": clk_b.summary() if args.batch else None,
              "large": clk_l.summary() if args.large_iters else None}

    cpu = None
    if d.rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_sample_iters)

    line = {"metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": d.world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128/f64" if args.dtype == "f64" else "c64/f32",
            "data": "synthetic (seeded BASELINE cfg2 scene, GPU MoM forward solve + 5% AWGN)",
            "config": {"workload": WORKLOAD, "k_iters": k, "scenes_per_gpu": 1,
                       "parallelism": f"scene-sharded x{d.world} (no collective)",
                       "l2": "flushed between steps (256 MiB write)", "graph": "CUDA graph of 10 iterations",
                       "final_loss_total": final_total, "env": pdf_env()},
            "e2e": {"value": d.world * k / e2e_s, "unit": "iter/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "s_per_reconstruction": e2e_s,
                    "api": "BatchReconstructor.run(host data, theta_cache=False, prefetch_seeds=next run) -> "
                           "ReconstructionResult",
                    "rel_error": res[0].rel_error},
            "roofline": roof, "kernels_in_graph": legroof.get("kernels") if legroof else None,
            "iteration_period_us": legroof.get("iteration_period_us") if legroof else None,
            "path_roofline": proof, "phases_ms_events": phases_ev, "fp64_peak_tflops_measured": fp64,
            "cpu_baseline": cpu,
            "clocks": dict(clk.summary(), by_leg=by_leg),
            "gpu_launches": args.steps * (1 + launches_per_iter * k), "batched": batched, "large": large}
    if d.rank == 0:
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    d = Dist(args.gpus, force=args.force_sharded and args.impl == "ours")
    try:
        if args.impl == "reference":
            run_reference(args, d)
        else:
            run_ours(args, d)
    finally:
        d.close()


if __name__ == "__main__":
    main()
