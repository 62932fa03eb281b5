"""Size-independent properties of the CUDA path at the BASELINE configs'
full sizes (config 5: 256 x 256, 72 views / receivers, m_f = 16; config 4's
batch shape), where the oracle would take too long per case:

  adjoint identities  <G_D x, y> = <x, G_D^H y>, <G_S x, r> = <x, G_S^H r>
                      (reference tests/test_forward.py:52-65)
  linearity           G_D(a x + b y) = a G_D x + b G_D y
  round trip          truncate(expand(alpha)) = alpha (tests/test_spectral.py:35-40)
  gradient            central differences of the composite loss along random
                      directions match Re <g_alpha, d> (tests/test_losses.py:140-160)
"""
import numpy as np
import pytest
import torch

from conftest import Setup, cfg_baseline, golden, rel

pytestmark = pytest.mark.gpu
LAM = (1e-3, 1e-5, 1e-5)


@pytest.fixture(scope="module")
def dev5():
    from paper_2602_13805_b200.engine import DeviceProblem
    g = golden("cfg5")
    st = Setup(cfg_baseline(5), plane=True)
    c = st.cfg
    return DeviceProblem(st.ops, st.e_inc, g["data"], mf=c.m_f, beta=c.beta, lambdas=LAM, tau_b=c.tau_b), g


def _rand(shape, seed):
    r = np.random.default_rng(seed)
    return torch.as_tensor(r.standard_normal(shape) + 1j * r.standard_normal(shape), device="cuda")


def _ip(a, b):
    return complex(torch.sum(a.conj() * b).item())


def test_gd_adjoint_and_linearity_full_size(dev5):
    dev, _ = dev5
    M = dev.M
    x, y = _rand((3, M, M), 1), _rand((3, M, M), 2)
    gx = dev.apply_gd(x)
    ghy = dev.apply_gd(y, adjoint=True)
    lhs, rhs = _ip(gx, y), _ip(x, ghy)
    assert abs(lhs - rhs) / (torch.linalg.norm(gx).item() * torch.linalg.norm(y).item()) < 1e-12
    a, b = 0.7 - 0.2j, -1.3 + 0.5j
    lin = dev.apply_gd(a * x + b * y)
    assert rel(lin.cpu().numpy(), (a * gx + b * dev.apply_gd(y)).cpu().numpy()) < 1e-12


def test_gs_adjoint_full_size(dev5):
    dev, _ = dev5
    x, r = _rand((4, dev.M, dev.M), 3), _rand((4, dev.R), 4)
    gx, ghr = dev.gs_forward(x), dev.gs_adjoint(r)
    lhs, rhs = _ip(gx, r), _ip(x, ghr)
    assert abs(lhs - rhs) / (torch.linalg.norm(gx).item() * torch.linalg.norm(r).item()) < 1e-12


def test_expand_truncate_round_trip_full_size(dev5):
    dev, _ = dev5
    alpha = _rand((5, dev.m0), 5)
    back = dev.truncate(dev.expand(alpha))
    assert rel(back.cpu().numpy(), alpha.cpu().numpy()) < 1e-13


@pytest.mark.parametrize("which", ["cfg5", "cfg4"])
def test_loss_gradient_directional_derivative(dev5, which):
    """Central differences of the float64 composite loss along three random
    directions agree with Re <g_alpha, d> to 1e-6 relative (the reference's
    finite-difference gate is 1e-5, tests/test_losses.py:140-160)."""
    from paper_2602_13805_b200.engine import DeviceProblem
    if which == "cfg5":
        dev, g = dev5
        a0 = torch.as_tensor(g["alpha0"][None], device="cuda")
    else:
        gs = [golden(f"cfg4_s{i}") for i in range(4)]
        st = Setup(cfg_baseline(4), plane=True)
        c = st.cfg
        dev = DeviceProblem(st.ops, st.e_inc, np.stack([x["data"] for x in gs]), mf=c.m_f, beta=c.beta,
                            lambdas=LAM, tau_b=c.tau_b)
        a0 = torch.as_tensor(np.stack([x["alpha0"] for x in gs]), device="cuda")
    ga, _ = dev.loss_grad(a0)
    ga = ga.clone()
    dev.check_errors()
    for k in range(3):
        d = _rand(tuple(a0.shape), 10 + k)
        d = d / torch.linalg.norm(d) * torch.linalg.norm(a0) * 1e-3
        h = 1e-4
        lp = dev.loss_value(a0 + h * d)[0][:, 5].clone()
        lm = dev.loss_value(a0 - h * d)[0][:, 5].clone()
        fd = ((lp - lm) / (2 * h)).cpu().numpy()
        an = torch.sum((ga.conj() * d).real, dim=(1, 2)).cpu().numpy()
        err = np.abs(fd - an) / np.maximum(np.abs(an), 1e-300)
        assert err.max() < 1e-6, (which, k, err)
