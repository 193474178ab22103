"""GPU: the pole-sharded stepper (distributed.ShardedStepper: per-rank native
plan, segmented all-to-all of the double-double partials, rank-order combine,
all-gather) gives the single-plan step bit for bit.  Two ranks share GPU 0
over gloo -- a functional check of the multi-rank code path (the NCCL
collectives themselves need one GPU per rank)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, q, exchange="auto"):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import torch.distributed as dist
    from conftest import load_golden
    from paper_1912_03312_b200.distributed import ShardedStepper
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, sysm, ap = load_golden(name)
        torch.cuda.set_device(0)
        sh = ShardedStepper(sysm, ap, float(d["tau"]), rank=rank, world=world, device=0, refine=1,
                            exchange=exchange)
        u = torch.from_numpy(d["u0"]).cuda()
        out = torch.empty_like(u)
        sh.step(u, out)
        torch.cuda.synchronize()
        q.put((rank, out.cpu().numpy()))
        sh.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["segmented", "allgather"])
@pytest.mark.parametrize("name", ["cfg1_k32", "p1_2d_m16", "fem_p2"])
def test_sharded_step_equals_single_plan(name, exchange):
    """both exchanges (one all-gather collective, or all-to-all + all-gather of
    segments) give the single plan's bits, on the direct 1D, COCG and band
    paths"""
    import torch.multiprocessing as mp
    from conftest import load_golden
    from paper_1912_03312_b200 import rexi_prepare, rexi_step
    d, sysm, ap = load_golden(name)
    stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True,
                       refine=1)
    single = rexi_step(stp, d["u0"])
    stp.close()
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for _, u in outs:
        assert np.array_equal(u, single)


def test_partial_step_graph_cache_many_buffers():
    """rexi_plan_step_partial replays a captured graph per (u, partial)
    buffer pair (at most 4 kept): six distinct input buffers, each result
    equal bit for bit to the plan's own step"""
    import torch
    from paper_1912_03312_b200 import _native, fixtures
    from paper_1912_03312_b200._pattern import shared_pattern
    cfg = fixtures.config2(m=20_000, k=16)
    ip, ix, ar, ai, br = shared_pattern(cfg.system.A, cfg.system.B)
    s = torch.cuda.Stream()
    p = _native.NativePlan(ip, ix, ar, br, cfg.approx.shifts, cfg.approx.weights, cfg.tau, a_imag=ai,
                           device=0, refine=1, stream=s.cuda_stream)
    n = cfg.system.n_dof
    part = torch.empty((4, n), dtype=torch.float64, device="cuda")
    for q in range(6):
        u = torch.from_numpy(cfg.u0 * np.exp(0.3j * q)).cuda()
        ref = torch.empty_like(u)
        p.step_device(u.data_ptr(), ref.data_ptr(), 1)
        for _ in range(2):                       # capture, then replay
            p.step_partial(u.data_ptr(), part.data_ptr())
            out = torch.empty_like(u)
            _native.combine_partials(part.data_ptr(), 1, n, out.data_ptr(), s.cuda_stream)
            s.synchronize()
            assert torch.equal(out, ref), q
