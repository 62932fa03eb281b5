import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from conftest import Setup, cfg_baseline, golden, rel
from paper_2602_13805_b200.engine import DeviceProblem
LAM = (1e-3, 1e-5, 1e-5)
def run(cfg_id, stream):
    os.environ["PDF_PIX_STREAM"] = str(stream)
    if cfg_id == 5:
        g = golden("cfg5"); st = Setup(cfg_baseline(5), plane=True)
        data, a0 = g["data"][None], g["alpha0"][None]
    else:
        gs = [golden(f"cfg4_s{i % 10}") for i in range(40)]; st = Setup(cfg_baseline(4), plane=True)
        data, a0 = np.stack([x["data"] for x in gs]), np.stack([x["alpha0"] for x in gs])
    c = st.cfg
    dev = DeviceProblem(st.ops, st.e_inc, data, mf=c.m_f, beta=c.beta, lambdas=LAM, tau_b=c.tau_b)
    ga, bd = dev.loss_grad(torch.as_tensor(a0, device="cuda"))
    return ga.cpu().numpy().copy(), bd.cpu().numpy().copy()
for cfg_id in (4, 5):
    # NOTE: PDF_PIX_STREAM is read once per process (static); run both in subprocesses
    pass
if __name__ == "__main__":
    cfg_id, stream = int(sys.argv[1]), int(sys.argv[2])
    ga, bd = run(cfg_id, stream)
    np.savez(f"/tmp/pix_{cfg_id}_{stream}.npz", ga=ga, bd=bd)
