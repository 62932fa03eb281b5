"""Experiment: two independent half-batches (S scenes each) trained concurrently on two streams."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2602_13805_b200 import build_grid, plane_wave_fields
from paper_2602_13805_b200.api import BatchReconstructor, _theta0
from paper_2602_13805_b200.workloads import baseline_config, baseline_scene, cfg4_scene, synthesize_gpu

S = int(sys.argv[1]) if len(sys.argv) > 1 else 128
k = 50
cfg = baseline_config(4, k_iters=k)
e_inc = plane_wave_fields(cfg, build_grid(cfg)).views
devs, states = [], []
for h in range(2):
    pairs = [cfg4_scene(h * S + i) for i in range(S)]
    data, _ = synthesize_gpu(cfg, [p[0] for p in pairs], [p[1] for p in pairs], baseline_scene(4)[2])
    rec = BatchReconstructor(cfg, S, e_inc=e_inc)
    dev = rec.dev
    dev.set_data(data)
    _, r0 = dev.bp_initialize()
    dev.net_setup(dev.init_alpha(r0))
    th0 = torch.as_tensor(_theta0(list(range(h * S, h * S + S)), rec.m0_eff), dtype=dev.rdt, device=dev.device)
    th, m, v = dev.alloc_state(th0)
    tr = torch.zeros(k, S, 6, dtype=torch.float64, device=dev.device)
    devs.append(dev); states.append((th, m, v, tr))
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
for h in range(2):      # warm (graph capture per stream)
    with torch.cuda.stream(streams[h]):
        devs[h].train(*states[h][:3], 0, 10, states[h][3])
torch.cuda.synchronize()
t = time.perf_counter()
for h in range(2):
    with torch.cuda.stream(streams[0]):
        devs[h].train(*states[h][:3], 0, k, states[h][3])
torch.cuda.synchronize()
seq = time.perf_counter() - t
t = time.perf_counter()
for h in range(2):
    with torch.cuda.stream(streams[h]):
        devs[h].train(*states[h][:3], 0, k, states[h][3])
torch.cuda.synchronize()
con = time.perf_counter() - t
print(f"S={S} x2, {k} its: sequential {1e3*seq:.1f} ms, concurrent {1e3*con:.1f} ms ({seq/con:.2f}x)")
