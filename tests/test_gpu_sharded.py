"""Incidence sharding: views split over shards with the three
per-iteration reductions must reproduce the unsharded iteration.  The shards
run in one process on one GPU (LocalShards: the reductions are plain sums),
which checks the sharded algebra exactly as the survey prescribes; the
multi-process plumbing is covered on CPU by tests/test_host.py (gloo)."""
import numpy as np
import pytest
import torch

from conftest import Setup, cfg_baseline, golden, rel

pytestmark = pytest.mark.gpu
LAM = (1e-3, 1e-5, 1e-5)


@pytest.mark.parametrize("cfg_id,world", [(1, 2), (1, 3), (3, 3)])
def test_sharded_matches_unsharded(cfg_id, world):
    from paper_2602_13805_b200.api import BatchReconstructor, _theta0
    from paper_2602_13805_b200.sharded import IncidenceShard, LocalShards, run_sharded, sharded_chi
    g = golden(f"cfg{cfg_id}")
    st = Setup(cfg_baseline(cfg_id), plane=True)
    cfg = st.cfg
    k = 12
    ref = BatchReconstructor(cfg, 1, e_inc=st.e_inc).run([g["data"]], seeds=[cfg.rng_seed], k_iters=k)[0]
    shards = [IncidenceShard(st.ops, st.e_inc, g["data"], mf=cfg.m_f, beta=cfg.beta, lambdas=LAM, tau_b=cfg.tau_b,
                             rank=r, world=world) for r in range(world)]
    theta0 = torch.as_tensor(_theta0([cfg.rng_seed], 4 * cfg.m_f ** 2), device="cuda")
    thetas, trace = run_sharded(shards, LocalShards(), theta0, k)
    ref_tr = np.array([b.as_row() for b in ref.trace])
    np.testing.assert_allclose(trace, ref_tr, rtol=1e-9)
    # replicated parameters stay identical on every shard
    for th in thetas[1:]:
        assert torch.equal(th, thetas[0])
    chi = sharded_chi(shards, LocalShards(), thetas).cpu().numpy()
    assert rel(chi, ref.chi_hat.values) < 1e-9


@pytest.mark.parametrize("graph", [False, True])
def test_zero1_trainer_single_rank_nccl(graph):
    """ShardedTrainer (per-layer gradient buckets reduce-scattered on a comm
    stream, Adam on the owned shard with a device step counter, all-gather; the
    whole iteration optionally captured in a CUDA graph WITH its NCCL
    collectives) on a one-rank NCCL group reproduces the unsharded run."""
    import torch.distributed as dist
    from paper_2602_13805_b200.api import BatchReconstructor, _theta0
    from paper_2602_13805_b200.sharded import IncidenceShard, ShardedTrainer
    g = golden("cfg1")
    st = Setup(cfg_baseline(1), plane=True)
    cfg = st.cfg
    k = 20
    ref = BatchReconstructor(cfg, 1, e_inc=st.e_inc).run([g["data"]], seeds=[cfg.rng_seed], k_iters=k)[0]
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        sh = IncidenceShard(st.ops, st.e_inc, g["data"], mf=cfg.m_f, beta=cfg.beta, lambdas=LAM, tau_b=cfg.tau_b,
                            rank=0, world=1)
        theta0 = torch.as_tensor(_theta0([cfg.rng_seed], 4 * cfg.m_f ** 2), device="cuda")
        tr = ShardedTrainer(sh, theta0, graph=graph, graph_iters=10)
        trace = tr.train(k).cpu().numpy()
        tr.check_errors()
    finally:
        if own:
            dist.destroy_process_group()
    ref_tr = np.array([b.as_row() for b in ref.trace])
    np.testing.assert_allclose(trace, ref_tr, rtol=1e-9)


@pytest.mark.parametrize("cfg_id,world,graph", [(1, 2, False), (1, 3, False), (3, 2, False), (1, 2, True)])
def test_peer_scatter_emulated_ranks(cfg_id, world, graph):
    """Reduce-scatter fused into the backward (pdf_shard_step_c_scatter: every
    g_W / g_b entry stored by the kernel that computes it into its owner's
    receive buffer) + owner-side Adam with the parameter all-gather as stores
    (pdf_adam_gather), with `world` ranks emulated in one process on one GPU
    (local buffers stand in for the peer-mapped ones, stream order for the
    barriers): the iteration trace matches the unsharded run and every rank
    ends with the same parameters."""
    from paper_2602_13805_b200.api import BatchReconstructor, _theta0
    from paper_2602_13805_b200.sharded import IncidenceShard, PeerTrainer
    g = golden(f"cfg{cfg_id}")
    st = Setup(cfg_baseline(cfg_id), plane=True)
    cfg = st.cfg
    k = 12
    ref = BatchReconstructor(cfg, 1, e_inc=st.e_inc).run([g["data"]], seeds=[cfg.rng_seed], k_iters=k)[0]
    shards = [IncidenceShard(st.ops, st.e_inc, g["data"], mf=cfg.m_f, beta=cfg.beta, lambdas=LAM, tau_b=cfg.tau_b,
                             rank=r, world=world) for r in range(world)]
    theta0 = torch.as_tensor(_theta0([cfg.rng_seed], 4 * cfg.m_f ** 2), device="cuda")
    tr = PeerTrainer(shards, theta0, graph=graph, graph_iters=5)
    trace = tr.train(k).cpu().numpy()
    tr.check_errors()
    np.testing.assert_allclose(trace, np.array([b.as_row() for b in ref.trace]), rtol=1e-9)
    for r in range(1, world):
        assert torch.equal(tr.params(r), tr.params(0))


def test_peer_scatter_symmetric_memory_single_rank():
    """The multi-GPU form of PeerTrainer -- torch symmetric memory buffers,
    rendezvous of their peer addresses, NCCL barriers -- on a one-rank group."""
    import torch.distributed as dist
    from paper_2602_13805_b200.api import BatchReconstructor, _theta0
    from paper_2602_13805_b200.sharded import IncidenceShard, PeerTrainer
    g = golden("cfg1")
    st = Setup(cfg_baseline(1), plane=True)
    cfg = st.cfg
    k = 8
    ref = BatchReconstructor(cfg, 1, e_inc=st.e_inc).run([g["data"]], seeds=[cfg.rng_seed], k_iters=k)[0]
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        sh = IncidenceShard(st.ops, st.e_inc, g["data"], mf=cfg.m_f, beta=cfg.beta, lambdas=LAM, tau_b=cfg.tau_b,
                            rank=0, world=1)
        theta0 = torch.as_tensor(_theta0([cfg.rng_seed], 4 * cfg.m_f ** 2), device="cuda")
        tr = PeerTrainer([sh], theta0, group=dist.group.WORLD, graph=True, graph_iters=4)
        trace = tr.train(k).cpu().numpy()
        tr.check_errors()
    finally:
        if own:
            dist.destroy_process_group()
    np.testing.assert_allclose(trace, np.array([b.as_row() for b in ref.trace]), rtol=1e-9)


@pytest.mark.parametrize("cfg_id,world,graph", [(1, 2, False), (1, 3, False), (3, 2, False), (1, 2, True)])
def test_tensor_parallel_emulated_ranks(cfg_id, world, graph):
    """Tensor-parallel network (W1 / W3 rows, W2 columns per rank; SURVEY 8(e)'s
    alternative) with incidence-sharded physics, `world` ranks emulated in one
    process on one GPU: the iteration trace matches the unsharded run and the
    assembled parameters match the one-rank tensor-parallel run."""
    from paper_2602_13805_b200.api import BatchReconstructor, _theta0
    from paper_2602_13805_b200.sharded import IncidenceShard, TensorParallelTrainer
    g = golden(f"cfg{cfg_id}")
    st = Setup(cfg_baseline(cfg_id), plane=True)
    cfg = st.cfg
    k = 12
    ref = BatchReconstructor(cfg, 1, e_inc=st.e_inc).run([g["data"]], seeds=[cfg.rng_seed], k_iters=k)[0]
    theta0 = torch.as_tensor(_theta0([cfg.rng_seed], 4 * cfg.m_f ** 2), device="cuda")

    def run(w):
        shards = [IncidenceShard(st.ops, st.e_inc, g["data"], mf=cfg.m_f, beta=cfg.beta, lambdas=LAM,
                                 tau_b=cfg.tau_b, rank=r, world=w) for r in range(w)]
        tr = TensorParallelTrainer(shards, theta0, graph=graph, graph_iters=4, lr=cfg.learn_rate)
        trace = tr.train(k).cpu().numpy()
        tr.check_errors()
        return trace, tr.params()

    trace, params = run(world)
    np.testing.assert_allclose(trace, np.array([b.as_row() for b in ref.trace]), rtol=1e-9)
    _, params1 = run(1)
    assert float(torch.max(torch.abs(params - params1))) < 1e-9 * float(torch.max(torch.abs(params1)))


def test_tensor_parallel_single_rank_nccl():
    """The torch.distributed form (NCCL all-reduces, CUDA-graph captured) on a one-rank group."""
    import torch.distributed as dist
    from paper_2602_13805_b200.api import BatchReconstructor, _theta0
    from paper_2602_13805_b200.sharded import IncidenceShard, TensorParallelTrainer
    g = golden("cfg1")
    st = Setup(cfg_baseline(1), plane=True)
    cfg = st.cfg
    k = 8
    ref = BatchReconstructor(cfg, 1, e_inc=st.e_inc).run([g["data"]], seeds=[cfg.rng_seed], k_iters=k)[0]
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        sh = IncidenceShard(st.ops, st.e_inc, g["data"], mf=cfg.m_f, beta=cfg.beta, lambdas=LAM, tau_b=cfg.tau_b,
                            rank=0, world=1)
        theta0 = torch.as_tensor(_theta0([cfg.rng_seed], 4 * cfg.m_f ** 2), device="cuda")
        tr = TensorParallelTrainer([sh], theta0, group=dist.group.WORLD, graph=True, graph_iters=4, lr=cfg.learn_rate)
        trace = tr.train(k).cpu().numpy()
        tr.check_errors()
    finally:
        if own:
            dist.destroy_process_group()
    np.testing.assert_allclose(trace, np.array([b.as_row() for b in ref.trace]), rtol=1e-9)
