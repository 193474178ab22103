"""Pole-parallel ("time-parallel") REXI across GPUs, one process per GPU.

The reference splits the K shifted solves over a thread pool in contiguous
chunks and reduces on the coordinating thread in fixed ascending-j order
(``integrate.py:114-120, 196-198, 215-224``); the paper runs the same split
over MPI ranks with one reduce per step (``PAPER.md:112-129, 1133-1137``).

Here each rank owns a shard of the shifts (one native plan on its GPU),
produces the double-double partial sum of its shard, and one collective per
step -- ``all_gather`` of the (hi, lo) partials over NCCL/NVLink -- is
followed by a fixed-rank-order double-double combine on every rank.  Because
the partials are double-double and combined in a fixed order, the result is
independent of the number of GPUs to ~1e-30 relative (the reference's
worker-count determinism contract, ``test_integrate.py:268-274``), which a
plain fp64 ``all_reduce`` would not give (the weights reach 1.7e7 and the
terms cancel to O(1)).
"""

from __future__ import annotations

import numpy as np

from . import _native
from ._pattern import shared_pattern


def shard_indices(k: int, world: int, cost=None):
    """Shift indices per rank.

    Without a cost model: contiguous, balanced chunks (``np.array_split``,
    the reference's chunking, ``integrate.py:117``) -- right for the direct
    1D solver whose cost is identical per shift.  With per-shift costs
    (e.g. measured COCG iteration counts): longest-processing-time-first
    assignment, each rank's list sorted ascending.
    """
    if world < 1:
        raise ValueError(f"world size must be >= 1, got {world}")
    if cost is None:
        return [list(map(int, c)) for c in np.array_split(np.arange(k), world)]
    cost = np.asarray(cost, dtype=float)
    order = np.argsort(-cost, kind="stable")
    load = np.zeros(world)
    out = [[] for _ in range(world)]
    for j in order:
        r = int(np.argmin(load))
        out[r].append(int(j))
        load[r] += cost[j]
    return [sorted(o) for o in out]


def dd_combine_host(parts: np.ndarray) -> np.ndarray:
    """Reference (host, numpy) semantics of ``rexi_combine_partials`` for the
    CPU tests of the multi-rank logic: parts (G, 4, n) -> complex128 (n,)."""
    def two_sum(a, b):
        s = a + b
        bb = s - a
        return s, (a - (s - bb)) + (b - bb)

    def dd_add(ah, al, bh, bl):
        sh, sl = two_sum(ah, bh)
        th, tl = two_sum(al, bl)
        sl = sl + th
        s2 = sh + sl
        sl = sl - (s2 - sh)
        sh = s2
        sl = sl + tl
        s3 = sh + sl
        return s3, sl - (s3 - sh)

    n = parts.shape[2]
    rh = np.zeros(n); rl = np.zeros(n); ih = np.zeros(n); il = np.zeros(n)
    for g in range(parts.shape[0]):
        rh, rl = dd_add(rh, rl, parts[g, 0], parts[g, 1])
        ih, il = dd_add(ih, il, parts[g, 2], parts[g, 3])
    return (rh + rl) + 1j * (ih + il)


def shard_partial_host(terms: np.ndarray) -> np.ndarray:
    """Double-double partial (4, n) of a shard's fp64 complex terms (k, n),
    summed in ascending j with TwoSum -- host statement of what the level-0
    kernels accumulate per shard (used by the CPU tests of the collective)."""
    n = terms.shape[1]
    out = np.zeros((4, n))
    for comp, (hi_i, lo_i) in enumerate([(0, 1), (2, 3)]):
        hi = np.zeros(n)
        lo = np.zeros(n)
        part = terms.real if comp == 0 else terms.imag
        for t in part:
            s = hi + t
            bb = s - hi
            e = (hi - (s - bb)) + (t - bb)
            hi, lo = s, lo + e
        out[hi_i], out[lo_i] = hi, lo
    return out


def allgather_partials(mine, world: int, group=None, out=None):
    """All ranks' (4, n) float64 partials -> (world, 4, n), rank order.
    NCCL: one all_gather_into_tensor over NVLink; other backends (gloo, used
    by the CPU tests) fall back to all_gather of a tensor list."""
    import torch
    import torch.distributed as dist
    if out is None:
        out = torch.empty((world,) + tuple(mine.shape), dtype=mine.dtype, device=mine.device)
    if world == 1:
        out[0].copy_(mine)
        return out
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out.view(-1), mine.contiguous().view(-1), group=group)
    elif mine.is_cuda:
        # gloo gathers host tensors only (functional multi-rank checks)
        parts = [torch.empty(tuple(mine.shape), dtype=mine.dtype) for _ in range(world)]
        dist.all_gather(parts, mine.detach().cpu(), group=group)
        out.copy_(torch.stack(parts))
    else:
        dist.all_gather(list(out.unbind(0)), mine.contiguous(), group=group)
    return out


def exchange_segments(mine, send, recv, world: int, seg: int, group=None):
    """All-to-all of row segments of the (4, n) partials: afterwards
    recv[g] = rows [r*seg, (r+1)*seg) of rank g's partial (r = this rank),
    zero-padded past n.  NCCL: one all_to_all_single; gloo (functional
    checks): host tensors."""
    import torch
    import torch.distributed as dist
    n = mine.shape[1]
    npad = seg * world
    src = mine
    if npad != n:
        src = torch.zeros((4, npad), dtype=mine.dtype, device=mine.device)
        src[:, :n] = mine
    send.copy_(src.view(4, world, seg).transpose(0, 1))
    if dist.get_backend(group) == "nccl":
        dist.all_to_all_single(recv.view(-1), send.view(-1), group=group)
        return
    # gloo has no all_to_all: gather every rank's segments, keep this rank's
    rank = dist.get_rank(group)
    allp = [torch.empty(tuple(send.shape), dtype=send.dtype) for _ in range(world)]
    dist.all_gather(allp, send.detach().cpu(), group=group)
    recv.copy_(torch.stack([allp[g][rank] for g in range(world)]))


def gather_segments(useg, uall, world: int, group=None):
    """All-gather of the rounded complex128 segments into uall (world*seg)."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(torch.view_as_real(uall).view(-1), torch.view_as_real(useg).view(-1),
                                    group=group)
    else:
        parts = [torch.empty(useg.shape, dtype=useg.dtype) for _ in range(world)]
        dist.all_gather(parts, useg.detach().cpu(), group=group)
        uall.copy_(torch.cat(parts))


class ShardedStepper:
    """This rank's shard of one REXI step.  ``step(u, out)`` takes and writes
    device tensors (complex128, length n) on this rank's GPU.

    ``stream`` (a cudaStream_t as int) defaults to torch's current stream on
    ``device``, so the step is ordered with the torch ops that produce u and
    consume out.  A rank whose shard is empty (world > K) contributes a zero
    partial.  ``reshard(cost)`` re-splits the shifts by per-shift costs
    (``measure_costs()``: the COCG iterations of the last step, gathered from
    every rank), longest-processing-time first."""

    def __init__(self, sysm, approx, tau, *, rank: int, world: int, device: int,
                 refine: int = -1, solver: int = _native.SOLVER_AUTO, cost=None, group=None,
                 stream=None, tol: float = 0.0, max_iters: int = 0, exchange: str = "auto"):
        import torch
        self.rank, self.world, self.group = rank, world, group
        self.shifts = np.asarray(approx.shifts, dtype=complex)
        self.weights = np.asarray(approx.weights, dtype=complex)
        self.k = len(self.shifts)
        self.pattern = shared_pattern(sysm.A, sysm.B)
        self.tau = tau
        self.device = device
        self.n = int(sysm.n_dof)
        dev = torch.device("cuda", device)
        if stream is None:
            stream = torch.cuda.current_stream(dev).cuda_stream
        self.stream = stream
        self._opts = dict(device=device, solver=solver, refine=refine, stream=stream, tol=tol,
                          max_iters=max_iters, weight_ref=float(np.mean(np.abs(self.weights))))
        self.plan = None
        self._build(shard_indices(self.k, world, cost))
        # exchange of the partials: "allgather" = ONE collective per step (all
        # ranks' (hi, lo) partials, then the rank-order combine of the whole
        # vector everywhere; (world-1) x 32 B/row per rank), "segmented" = an
        # all-to-all of row segments + an all-gather of the rounded segments
        # (48 B/row per rank).  auto: one collective where a step is long
        # (COCG, >= 0.1 s: the extra bytes cost microseconds), segmented for
        # the direct solvers (a 1D step is ~0.2-1.6 ms per rank)
        if exchange not in ("auto", "allgather", "segmented"):
            raise ValueError(f"unknown exchange {exchange!r}")
        if exchange == "auto":
            iterative = self.plan is not None and int(self.plan.info.solver) == _native.SOLVER_COCG
            exchange = "allgather" if iterative or world == 1 else "segmented"
        self.exchange = exchange
        self.parts = torch.empty((world, 4, self.n), dtype=torch.float64, device=dev)
        self.mine = torch.zeros((4, self.n), dtype=torch.float64, device=dev)
        # segmented exchange buffers: row segments of seg rows per rank
        self.seg = -(-self.n // world)
        npad = self.seg * world
        self.send = torch.zeros((world, 4, self.seg), dtype=torch.float64, device=dev)
        self.recv = torch.empty((world, 4, self.seg), dtype=torch.float64, device=dev)
        self.useg = torch.empty(self.seg, dtype=torch.complex128, device=dev)
        self.uall = torch.empty(npad, dtype=torch.complex128, device=dev)

    def _build(self, shards):
        if self.plan is not None:
            self.plan.close()
            self.plan = None
        self.shards = shards
        idx = shards[self.rank]
        if idx:
            indptr, indices, a_re, a_im, b_re = self.pattern
            ids = np.asarray(idx, dtype=np.int64)
            self.plan = _native.NativePlan(indptr, indices, a_re, b_re, self.shifts[ids],
                                           self.weights[ids], self.tau, a_imag=a_im,
                                           shift_offset=int(idx[0]), shift_ids=ids, **self._opts)

    def measure_costs(self):
        """Per-shift COCG iterations of the last step, all K, on every rank
        (one small all_reduce of an int tensor: each rank fills its shifts)."""
        import torch
        import torch.distributed as dist
        c = np.zeros(self.k, dtype=np.int64)
        if self.plan is not None:
            c[self.shards[self.rank]] = self.plan.shift_iters()
        t = torch.from_numpy(c)
        if self.world > 1:
            if dist.get_backend(self.group) == "nccl":
                t = t.to(f"cuda:{self.device}")
            dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def reshard(self, cost):
        """Rebuild this rank's plan for the LPT split by ``cost`` (same on
        every rank, e.g. from measure_costs()).  Returns the new shards."""
        self._build(shard_indices(self.k, self.world, np.asarray(cost, dtype=float) + 1.0))
        return self.shards

    def step(self, u, out):
        """u1 = sum over all shards of beta_j x_j.  Each rank computes its
        shard's double-double partial.  exchange "allgather": one all-gather
        of the partials and the rank-order combine on every rank (one
        collective per step).  exchange "segmented": an all-to-all hands rank
        r the row segment r of every partial; rank r combines it in rank order
        (the same per-row double-double operations as combining everything
        everywhere) and rounds; an all-gather assembles u1 -- 48 B/row per
        rank instead of (world-1) x 32 B/row.  Both give the same bits."""
        if self.plan is not None:
            self.plan.step_partial(u.data_ptr(), self.mine.data_ptr())
        else:
            self.mine.zero_()
        if self.world == 1:
            _native.combine_partials(self.mine.data_ptr(), 1, self.n, out.data_ptr(), self.stream)
            return
        if self.exchange == "allgather":
            allgather_partials(self.mine, self.world, self.group, out=self.parts)
            _native.combine_partials(self.parts.data_ptr(), self.world, self.n, out.data_ptr(), self.stream)
            return
        exchange_segments(self.mine, self.send, self.recv, self.world, self.seg, self.group)
        _native.combine_partials(self.recv.data_ptr(), self.world, self.seg, self.useg.data_ptr(),
                                 self.stream)
        gather_segments(self.useg, self.uall, self.world, self.group)
        out.copy_(self.uall[:self.n])

    def close(self):
        if self.plan is not None:
            self.plan.close()
            self.plan = None
