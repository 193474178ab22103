#!/usr/bin/env python
"""bench.py -- REXI steps/s on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One "step" is one full REXI time step u1 = sum_j beta_j S_j^{-1}(iB u0) over
the whole workload.  Default workload = BASELINE.json configs[1] (the metric's
"1M DOF, K=64" case): 1D P1, n = 2^20 nodes (1,048,574 DOF), K = 64, tau = 0.5,
with the parity-correct setting (one double-double refinement round, which
brings the GPU result to the truth oracle; the reference's own fp64 path sits
2.4e-7 away from it).  Synthetic inputs: seeded fixtures (paper_1912_03312_b200/
fixtures.py), poles frozen from the reference's generator.

N > 1 (torchrun, one rank per GPU): the K shifts are sharded across ranks;
each step every rank computes its double-double partial sum and one NCCL
all_gather + fixed-order combine produces u1 on every rank (strong scaling:
the work per step is fixed).

--impl reference: the reference's CPU algorithm (the C restatement in oracle/
of zgbtrf/zgbtrs + fl(beta x) + Kahan, all host threads) on the same config;
rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "REXI steps/s (1M DOF, K=64)"
UNIT = "steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--refine", type=int, default=-1, help="-1: rexi_prepare's default")
    ap.add_argument("--secondary", type=int, default=-1,
                    help="also time this config's steps in a 'secondary' block (default: cfg 3 when "
                         "the main config is 2 and N = 1; 0 = off)")
    ap.add_argument("--secondary-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0: same as --steps")
    return ap.parse_args()


def acceptance_config():
    """--config 6: the reference's own acceptance workload (tests/golden/
    acceptance_p2.npz, made by tests/golden/make_acceptance.py from the
    reference: test_acceptance.py:60-65,95-121) -- the 7,999-DOF P2
    tunneling system (pentadiagonal), the flagship K = 16 poles, dt = 2e-4."""
    import numpy as np
    from scipy.sparse import csr_matrix
    from paper_1912_03312_b200 import fixtures
    from paper_1912_03312_b200.types import PartialFractionApproximation, SystemMatrices
    d = np.load(os.path.join(ROOT, "tests", "golden", "acceptance_p2.npz"))

    def csr(p):
        return csr_matrix((d[p + "_data"], d[p + "_indices"], d[p + "_indptr"]), shape=tuple(d[p + "_shape"]))
    sysm = SystemMatrices(csr("A"), csr("B"), int(d["A_shape"][0]))
    ap = PartialFractionApproximation(d["shifts"], d["weights"], float(d["R1"]), 0.0)
    mesh = fixtures.StructuredMesh(1, 4000, np.array([-120.0]), 240.0 / 4000)
    return fixtures.Config(name="acceptance_p2 (reference test_acceptance.py workload, P2)", system=sysm,
                           u0=d["u0"], approx=ap, tau=float(d["tau"]), n_steps=1000, sr=float(d["sr"]),
                           mesh=mesh)


def build_cfg(idx):
    from paper_1912_03312_b200 import fixtures
    return acceptance_config() if idx == 6 else fixtures.build_config(idx)


def workload_name(cfg):
    """The same string in both arms (the refinement setting is a separate
    config key: it is how an arm computes, not what the workload is)."""
    n, k = cfg.system.n_dof, cfg.approx.K
    dims = {1: "1D", 2: "2D", 3: "3D"}[cfg.mesh.d]
    fem = "P2" if cfg.name.startswith("acceptance") else "P1"
    return (f"{cfg.name}: {dims} {fem} Schroedinger REXI step, {n} DOF, nnz {cfg.system.A.nnz}, "
            f"K={k}, tau={cfg.tau}")


def api_refine(cfg):
    """rexi_prepare's default refinement for this config (integrate.default_refine)."""
    from paper_1912_03312_b200._pattern import shared_pattern
    from paper_1912_03312_b200.integrate import default_refine
    ip, ix = shared_pattern(cfg.system.A, cfg.system.B)[:2]
    return default_refine(ip, ix, cfg.tau, cfg.sr)


def cocg_8d_bytes(prof, n, nnz, k, steps):
    """SURVEY.md 8(d)'s algorithmic bytes of a COCG step: per lockstep
    iteration (20 nnz + 4 (N+1)) + 160 K_act N, plus 16 N (2 + 3K) for the
    prologue / epilogue; the refinement's dd-residual SpMVs count as extra
    iterations with K_act = K.  sum(K_act) over the iterations comes from the
    spmv hooks' own byte counts (112 B per live row-shift + the CSR bytes)."""
    csr_impl = 28.0 * nnz + 4.0 * (n + 1)
    csr_8d = 20.0 * nnz + 4.0 * (n + 1)
    total, iters, kact_n = 0.0, 0, 0.0
    for name, (cnt, _t, b) in prof.items():
        if name.startswith("cg_spmv"):
            kact_n += max(0.0, (b - cnt * csr_impl) / 112.0)
            iters += cnt
        elif name.startswith("cg_residual"):
            kact_n += cnt * k * n
            iters += cnt
    total = iters * csr_8d + 160.0 * kact_n + steps * 16.0 * n * (2 + 3 * k)
    return total / steps, iters / steps, kact_n / max(iters, 1) / n


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled every 200 ms."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def kernel_bytes(name, n, k, m=16):
    """Algorithmic HBM bytes per launch of the level-0 kernels (DESIGN.md
    "Roofline"): 16 B per (row, shift) for every per-shift complex array the
    kernel must read or write (inverse pivots, stored residual), the shared
    per-row inputs once (rhs 16 B, 8 B per A/B coefficient array), the
    per-block interface values (16 or 32 B per (block, shift), blocks = n/m)
    and the row outputs (rounded 16 B or the double-double partial 32 B)."""
    kb = k * n / m
    table = {
        # per-shift complex arrays, shared row bytes, per-(block,shift) bytes
        "l0_s1": (1, 16 + 48, 32),
        "l0_s3acc": (1, 16 + 48 + 16, 32),
        "l0_k2": (2, 16 + 72 + 32, 16 * 2 + 48),       # pivots in (16 B), complex64 residual out and pivots in (8 + 8 B); interface halves 2 x 24 B
        "l0_k3": (1, 48 + 32 + 16, 32),                # complex64 pivots + residual in (8 + 8 B)
    }
    if name == "rhs":
        return (16 + 16 + 24) * n
    if name not in table:
        return None
    per_shift, shared, per_block = table[name]
    return int(per_shift * 16 * n * k + shared * n + per_block * kb)


def l2_note(n, k):
    work = 16 * n * max(k, 1)
    if work > 126e6:
        return f"inputs larger than L2: one per-shift array is {work / 1e9:.2f} GB (L2 126 MB), no flush"
    return (f"per-shift arrays ({work / 1e6:.1f} MB) fit in L2; not flushed -- a latency-bound "
            "small config, reported as such")


def fp64_peak():
    """Measured FP64 issue peak (profiles/r01_fp64_peak.json, written by
    scripts/micro/dfma_peak.cu on a B200 of this pool)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


def load_traffic(name):
    """ncu evidence for a kernel (profiles/ncu_traffic.json, from one
    `ncu --set full` capture): DRAM bytes per launch and FP64-pipe use."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(name) or {}
    except Exception:
        return {}


def cpu_baseline_cocg(cfg, shifts=4, refine=1, repeats=1):
    """2D/3D: the reference cannot run (dense-LU fallback, solvers.py:108-115);
    time the C/OpenMP Jacobi-COCG restatement (oracle/cocg_oracle.c, same
    stopping rule, refinement as the GPU arm) on a bounded sample of
    `shifts` of the K shifts, `repeats` times, and scale to a full step."""
    import numpy as np
    from oracle.oracle import cocg_step
    from paper_1912_03312_b200.types import PartialFractionApproximation
    cores = os.cpu_count() or 1
    k = cfg.approx.K
    idx = np.linspace(0, k - 1, shifts).round().astype(int)
    sub = PartialFractionApproximation(cfg.approx.shifts[idx], cfg.approx.weights[idx],
                                       cfg.approx.domain_radius, 0.0)
    t0 = time.perf_counter()
    for _ in range(repeats):
        cocg_step(cfg.system, sub, cfg.tau, cfg.u0, tol=1e-10, refine=refine, tol_refine=1e-6,
                  nthreads=cores)
    steps_eq = repeats * shifts / k
    dt = (time.perf_counter() - t0) / steps_eq
    return {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "port", "steps_equivalent": steps_eq,
            "sample": f"{repeats} x {shifts} of {k} shifts (evenly spaced) of step 1 of {cfg.name} through "
                      f"oracle/cocg_oracle.c (Jacobi-COCG 1e-10, refine={refine}: dd-residual correction "
                      f"1e-6), OpenMP over shifts on {cores} threads; value = full steps/s, the sample "
                      f"time scaled by K/{shifts}"}


def cpu_baseline(cfg, steps=2):
    """The reference algorithm restated in C (oracle/, kind "port"), timed on
    this host's cores: factor once (not timed), then `steps` full steps."""
    if cfg.mesh.d > 1:
        return cpu_baseline_cocg(cfg, refine=api_refine(cfg))
    from oracle.oracle import OraclePlan
    cores = os.cpu_count() or 1
    orc = OraclePlan(cfg.system, cfg.approx, cfg.tau, nthreads=cores)
    u = cfg.u0
    orc.step(u)                                    # warm
    t0 = time.perf_counter()
    for _ in range(steps):
        u = orc.step(u)
    dt = time.perf_counter() - t0
    orc.close()
    return {"value": steps / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{steps} full {cfg.name} steps (all {cfg.approx.K} shifts, {cfg.system.n_dof} DOF) "
                      "through oracle/rexi_oracle.c (zgbtf2/zgbtrs restated, fl(beta x), Kahan), "
                      f"OpenMP over shifts on {cores} threads"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_1912_03312_b200 import fixtures
    from oracle.oracle import OraclePlan
    cfg = build_cfg(args.config)
    cores = os.cpu_count() or 1
    refine = api_refine(cfg)
    if cfg.mesh.d > 1:
        # 2D/3D: the reference cannot run (dense-LU fallback); one full CPU
        # step takes minutes, so the arm times a bounded sample (4 of the K
        # shifts) and reports what it ran: `steps` is the number of full-step
        # equivalents actually computed (samples x 4/K), `ms_per_step` the
        # measured time per full-step equivalent
        samples = max(1, min(args.steps, 2))
        cb = cpu_baseline_cocg(cfg, refine=refine, repeats=samples)
        v = cb["value"]
        steps_done = cb["steps_equivalent"]
        dt = steps_done / v
        sample = cb["sample"]
    else:
        orc = OraclePlan(cfg.system, cfg.approx, cfg.tau, nthreads=cores)
        u = cfg.u0
        for _ in range(args.warmup):
            u = orc.step(u)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            u = orc.step(u)
        dt = time.perf_counter() - t0
        v = args.steps / dt
        steps_done = args.steps
        sample = (f"{args.steps} full steps, reference algorithm restated in C "
                  "(oracle/rexi_oracle.c: zgbtrf/zgbtrs, fl(beta x), Kahan), OpenMP over shifts")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": steps_done, "warmup": args.warmup, "ms_per_step": 1e3 * dt / steps_done,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "complex128",
            "data": "synthetic (seeded fixtures, poles frozen from the reference generator)",
            "config": {"workload": workload_name(cfg), "refine": "n/a (direct LU)" if cfg.mesh.d == 1 else refine,
                       "parallelism": "host threads"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def secondary(c, steps, local, peak):
    """The 2D north_star target on the same run: device-timed steps of
    config c (default cfg 3: 2D, 1M DOF, K = 64) at rexi_prepare's default
    refinement, one warm-up step, then `steps` consecutive steps (2..steps+1
    of the trajectory) timed with CUDA events on the plan's stream, and a
    second pass over the same steps with per-kernel profiling for the
    SURVEY.md 8(d) step bytes.  The per-shift arrays (1 GB each) exceed L2."""
    import torch
    from paper_1912_03312_b200 import fixtures, _native
    from paper_1912_03312_b200._pattern import shared_pattern
    t_build = time.perf_counter()
    cfg = fixtures.build_config(c)
    n, k, nnz = cfg.system.n_dof, cfg.approx.K, cfg.system.A.nnz
    refine = api_refine(cfg)
    stream = torch.cuda.current_stream()
    ip, ix, ar, ai, br = shared_pattern(cfg.system.A, cfg.system.B)
    plan = _native.NativePlan(ip, ix, ar, br, cfg.approx.shifts, cfg.approx.weights, cfg.tau, a_imag=ai,
                              device=local, refine=refine, stream=stream.cuda_stream)
    t_build = time.perf_counter() - t_build
    u0 = torch.from_numpy(cfg.u0).to(f"cuda:{local}")
    u1 = torch.empty_like(u0)
    bufs = [torch.empty_like(u0), torch.empty_like(u0)]
    st = _native.RexiStats()
    plan.step_device(u0.data_ptr(), u1.data_ptr(), 1, st)         # warm-up = step 1
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local) as clk:
        e0.record(stream)
        src = u1
        for s in range(steps):
            st = _native.RexiStats()
            plan.step_device(src.data_ptr(), bufs[s % 2].data_ptr(), 1, st)
            launches += int(st.launches)
            src = bufs[s % 2]
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    plan.profile(True)
    src = u1
    iters = []
    for s in range(steps):
        plan.step_device(src.data_ptr(), bufs[s % 2].data_ptr(), 1, _native.RexiStats())
        iters.append(int(plan.shift_iters().max()))
        src = bufs[s % 2]
    torch.cuda.synchronize()
    prof = plan.profile_report()
    plan.profile(False)
    plan.close()
    step_bytes, it_step, kact = cocg_8d_bytes(prof, n, nnz, k, steps)
    ms_step = ms / steps
    ach = step_bytes / (ms_step / 1e3) / 1e9
    dom = max(prof.items(), key=lambda kv: kv[1][1])
    return {
        "workload": workload_name(cfg), "refine": refine, "steps": steps, "warmup": 1,
        "timed": f"steps 2..{steps + 1} of the trajectory from u0, device-resident state, CUDA events "
                 "on the plan's stream",
        "value": steps / (ms / 1e3), "unit": UNIT, "ms_per_step": ms_step, "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "algorithmic_bytes_per_step": step_bytes,
                     "bytes": "SURVEY.md 8(d): per lockstep iteration (20 nnz + 4(N+1)) + 160 K_act N, plus "
                              "16 N (2 + 3K) per step; dd-residual SpMVs count as iterations with K_act = K",
                     "lockstep_iterations_per_step": it_step, "mean_live_lanes": kact,
                     "max_shift_iterations": iters},
        "dominant_kernel": {"name": dom[0], "share_of_step": dom[1][1] / sum(v[1] for v in prof.values())},
        "kernels": {kname: {"launches": cnt, "total_ms": t} for kname, (cnt, t, _b) in prof.items()},
        "clocks": clk.summary(), "setup_s": t_build,
    }


def max_over_ranks(x, backend, local):
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}" if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_step
    from paper_1912_03312_b200.distributed import ShardedStepper
    from paper_1912_03312_b200 import _native

    # one rank per GPU; REXI_DIST_BACKEND=gloo (functional checks on a box with
    # fewer GPUs than ranks) maps ranks onto the visible devices round-robin
    backend = os.environ.get("REXI_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = build_cfg(args.config)
    n, k = cfg.system.n_dof, cfg.approx.K
    sec_cfg = args.secondary if args.secondary >= 0 else (3 if args.config == 2 and world == 1 else 0)
    if world > 1 or sec_cfg == args.config:
        sec_cfg = 0
    refine = args.refine
    if refine < 0:
        refine = api_refine(cfg)      # what rexi_prepare does by default
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    u0 = torch.from_numpy(cfg.u0).to(f"cuda:{local}")
    ua = u0.clone()
    ub = torch.empty_like(u0)

    def barrier():
        if world > 1:
            dist.barrier()

    if world == 1:
        from paper_1912_03312_b200._pattern import shared_pattern
        ip, ix, ar, ai, br = shared_pattern(cfg.system.A, cfg.system.B)
        plan = _native.NativePlan(ip, ix, ar, br, cfg.approx.shifts, cfg.approx.weights, cfg.tau,
                                  a_imag=ai, device=local, refine=refine, stream=sptr)

        def run(nsteps, src, dst):
            st = _native.RexiStats()
            plan.step_device(src.data_ptr(), dst.data_ptr(), nsteps, st)
            return int(st.launches)
    else:
        sh = ShardedStepper(cfg.system, cfg.approx, cfg.tau, rank=rank, world=world, device=local,
                            refine=refine, stream=sptr)
        plan = sh.plan

        def run(nsteps, src, dst):
            a, b = src, dst
            for s in range(nsteps):
                sh.step(a, b)
                a, b = b, a
            if nsteps % 2 == 0:
                dst.copy_(a)
            return int(nsteps * 0)  # counted below from the profile pass

    # warm-up
    run(args.warmup, ua, ub)
    torch.cuda.synchronize()
    if world > 1 and cfg.mesh.d > 1:
        # COCG: balance the pole shards by the per-shift iterations of the
        # last warm-up step (longest processing time first),
        # then warm the re-built plans once
        sh.reshard(sh.measure_costs())
        plan = sh.plan
        run(1, ua, ub)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        launches = run(args.steps, ua, ub)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        persistent = world == 1 and int(getattr(plan.info, "persistent", 0)) > 0
        if persistent:
            # one launch runs every step (tridiag_persist.cu): that launch is the kernel
            prof = {"k_persist": (1, ms, float(80 * n + 32 * k * n) * args.steps)}
        else:
            # profiled pass (same K steps): per-kernel device time for the roofline
            plan.profile(True)
            run(args.steps, ua, ub)
            torch.cuda.synchronize()
            prof = plan.profile_report()
            plan.profile(False)
    if world > 1:
        ms = max_over_ranks(ms, backend, local)
    launches = sum(v[0] for v in prof.values()) if launches == 0 else launches
    value = args.steps / (ms / 1e3)

    # end-to-end through the public API, host (pinned) buffers, H2D + D2H every step
    e2e = None
    if world == 1:
        stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr,
                           override_admissibility=True, device=local, refine=refine)
        pin_in = torch.from_numpy(cfg.u0).pin_memory()
        u_host = pin_in.numpy()
        ke = args.e2e_steps or args.steps
        rexi_step(stp, u_host)
        torch.cuda.synchronize()
        import gc
        trials = []
        gc.disable()
        try:
            # the median of up to 3 trials of ke steps (one when a trial takes
            # over 5 s): host wall-clock timing of short calls is noisy
            while len(trials) < 3:
                u_host = pin_in.numpy()                  # every trial steps from u0, like the device pass
                t0 = time.perf_counter()
                for _ in range(ke):
                    u_host = rexi_step(stp, u_host)      # H2D of u, one step, D2H of u1
                trials.append(time.perf_counter() - t0)
                if trials[-1] > 5.0:
                    break
        finally:
            gc.enable()
        dt = statistics.median(trials)
        stp.close()
        e2e = {"value": ke / dt, "unit": UNIT, "h2d_bytes_per_step": 16 * n,
               "d2h_bytes_per_step": 16 * n, "api": "paper_1912_03312_b200.rexi_step(numpy)",
               "timing": f"host wall clock around synchronous calls, median of {len(trials)} trials of {ke} steps",
               "transfer": "page-locked numpy buffers: the state crosses PCIe every step, read inside the "
                           "first kernel (1D) or copied in (COCG), and written by the last kernel"}
    else:
        # multi-GPU public API (distributed.ShardedStepper): every rank holds the
        # state on the host (pinned), copies it in, steps its shard (all-gather
        # of the dd partials over NCCL) and copies the result back
        pin_a = torch.from_numpy(cfg.u0.copy()).pin_memory()
        pin_b = torch.empty_like(pin_a).pin_memory()
        ud, od = torch.empty_like(u0), torch.empty_like(u0)
        ke = args.e2e_steps or args.steps
        ud.copy_(pin_a)
        sh.step(ud, od)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            ud.copy_(pin_a, non_blocking=True)
            sh.step(ud, od)
            pin_b.copy_(od, non_blocking=True)
            torch.cuda.synchronize()
            pin_a, pin_b = pin_b, pin_a
        dt = time.perf_counter() - t0
        dt = max_over_ranks(dt, backend, local)
        e2e = {"value": ke / dt, "unit": UNIT, "h2d_bytes_per_step": 16 * n * world,
               "d2h_bytes_per_step": 16 * n * world,
               "api": "paper_1912_03312_b200.distributed.ShardedStepper.step (host state on every rank)",
               "timing": "host wall clock, max over ranks"}

    # roofline of the dominant kernel
    peak, peak_src = measured_peak()
    dom = max(prof.items(), key=lambda kv: kv[1][1]) if prof else None
    roof = None
    if dom is not None:
        name, (cnt, tot, tot_bytes) = dom
        kshard = len(sh.shards[rank]) if world > 1 else k
        # bytes per launch: the kernel's own algorithmic count (COCG: live shifts
        # only, varies per launch) or the closed form of kernel_bytes()
        b = tot_bytes / max(cnt, 1) if tot_bytes > 0 else kernel_bytes(name, n, kshard)
        avg_ms = tot / max(cnt, 1)
        ach = (b / (avg_ms / 1e3)) / 1e9 if b else None
        ev = load_traffic(name)
        if ev.get("config") not in (None, args.config):
            ev = {}           # an ncu capture of another config is not this kernel's traffic
        roof = {"bound": "hbm", "kernel": name, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": (ach / peak) if ach else None, "traffic": ev.get("dram_bytes"),
                "algorithmic_bytes_per_launch": b, "avg_launch_ms": avg_ms,
                "share_of_step": tot / sum(v[1] for v in prof.values()), "peak_source": peak_src}
        if ev.get("fp64_pipe_pct") is not None:
            # the double-double kernels are FP64-issue bound, not HBM bound
            roof["fp64_pipe_pct"] = ev["fp64_pipe_pct"]
            roof["ncu_capture"] = ev.get("capture")
        fp = fp64_peak()
        if ev.get("fp64_inst_per_row_shift") and fp and not name.startswith("cg"):
            # t_roof = max(B_alg / HBM peak, F_alg / FP64 peak); FP64
            # work as thread-level DADD/DMUL/DFMA instructions (ncu counts of one
            # cfg 2 launch, per row-shift) against the measured DFMA issue rate
            inst = ev["fp64_inst_per_row_shift"] * n * kshard
            t_hbm = b / (peak * 1e9) * 1e3 if b else 0.0
            t_fp = inst / fp["dfma_per_s"] * 1e3
            roof["fp64"] = {"inst_per_launch": inst, "achieved_inst_per_s": inst / (avg_ms / 1e3),
                            "peak_inst_per_s": fp["dfma_per_s"], "frac": (inst / (avg_ms / 1e3)) / fp["dfma_per_s"],
                            "peak_source": "profiles/r01_fp64_peak.json (scripts/micro/dfma_peak.cu)",
                            "count_source": ev.get("fp64_inst_src")}
            roof["t_roof_ms"] = max(t_hbm, t_fp)
            roof["t_roof_bound"] = "fp64" if t_fp > t_hbm else "hbm"
            roof["t_roof_frac"] = max(t_hbm, t_fp) / avg_ms

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                cpu = cpu_baseline(cfg)
            except Exception as exc:  # the baseline must not kill the bench line
                cpu = {"error": str(exc)}
        # algorithmic bytes of one step: the kernels' own counts where the
        # profile carries them (COCG: live shifts per iteration), else SURVEY
        # 8(d)'s closed form for the direct 1D step
        kshard_ = len(sh.shards[rank]) if world > 1 else k
        prof_bytes = 0.0
        for kname, (cnt_, _t, b_) in prof.items():
            kb = kernel_bytes(kname, n, kshard_) if b_ <= 0 else None
            prof_bytes += b_ if b_ > 0 else (kb or 0) * cnt_
        step_bytes = prof_bytes / args.steps if prof_bytes > 0 else 80 * n + 32 * k * n
        bytes_note = "the kernels' own algorithmic byte counts (bench.kernel_bytes / the COCG hooks)"
        cg_iters = cg_kact = None
        if cfg.mesh.d > 1:
            step_bytes, cg_iters, cg_kact = cocg_8d_bytes(prof, n, cfg.system.A.nnz, kshard_, args.steps)
            bytes_note = ("SURVEY.md 8(d): per lockstep iteration (20 nnz + 4(N+1)) + 160 K_act N, plus "
                          "16 N (2 + 3K) per step; dd-residual SpMVs count as iterations with K_act = K")
        prof_ms = sum(v[1] for v in prof.values())
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "complex128",
            "data": "synthetic (seeded fixtures, poles frozen from the reference generator)",
            "config": {"workload": workload_name(cfg), "n_dof": n, "K": k, "tau": cfg.tau,
                       "refine": refine, "parallelism": f"pole-shard x{world}" if world > 1 else "1 GPU",
                       "l2": l2_note(n, k)},
            "e2e": e2e,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "kernels": {kname: {"launches": c, "total_ms": t, "GBps": (bt / (t / 1e3) / 1e9 if bt else None)}
                        for kname, (c, t, bt) in prof.items()},
            "step_algorithmic_GBps": step_bytes / (ms / args.steps / 1e3) / 1e9,
            "step_roofline": {
                "algorithmic_bytes_per_step": step_bytes,
                "achieved_GBps": step_bytes / (ms / args.steps / 1e3) / 1e9,
                "frac": step_bytes / (ms / args.steps / 1e3) / 1e9 / peak,
                "kernel_time_frac": (prof_ms / ms) if prof_ms and not persistent else None,
                "bytes": bytes_note,
                "cocg_iterations_per_step": cg_iters, "cocg_mean_live_lanes": cg_kact,
                "note": "whole step (all kernels, launch gaps and host polls included) against the "
                        "measured HBM peak"},
        }
        if sec_cfg:
            line["secondary"] = secondary(sec_cfg, args.secondary_steps, local, peak)
        print(json.dumps(line), flush=True)
    if world > 1:
        sh.close()
        dist.destroy_process_group()
    else:
        plan.close()


if __name__ == "__main__":
    main()
