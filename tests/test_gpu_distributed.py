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


def _worker(rank, world, port, name, q):
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
        sh = ShardedStepper(sysm, ap, float(d["tau"]), rank=rank, world=world, device=0, refine=1)
        u = torch.from_numpy(d["u0"]).cuda()
        out = torch.empty_like(u)
        sh.step(u, out)
        torch.cuda.synchronize()
        q.put((rank, out.cpu().numpy()))
        sh.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg1_k32", "p1_2d_m16"])
def test_sharded_step_equals_single_plan(name):
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
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for _, u in outs:
        assert np.array_equal(u, single)
