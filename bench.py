#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for libsvk.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl svk|reference]

Workload (BASELINE.json configs[2]): 2D Stokes, Q2-Q1 Taylor-Hood on a 4096 x 4096
structured mesh (151,035,907 DOFs), the paper's manufactured solution
as synthetic input.  One STEP = one FGMRES solve to 1e-10 right-preconditioned by
one V(1,1) cycle with additive Vanka relaxation per iteration, which runs
every row of the hot path: residual, Vanka sweep, restriction, prolongation,
level-0 solve, V-cycle, FGMRES.  The hierarchy + patch setup (svk_create) runs once
per context, as the paper precomputes its patch inverses; its time is
reported as `setup_s`.

value  = DOFs solved per second (whole job).
sweep  = the finest-level Vanka sweeps inside the timed solves (CUDA events on the
         sweep stream, svk_set_profiling): DOF/s, algorithmic HBM GB/s, roofline.
e2e    = the same solve from pinned HOST buffers through svk_solve_host_batch: a
         stream of >= 4 problems, every step's H2D of b and x0 and D2H of x inside
         the timed region, the copies of steps k+1 / k-1 overlapping the solve of
         step k; e2e.serial = one svk_solve_host call per step (nothing overlapped).
--impl reference  times the CPU oracle (oracle/, C++ + OpenMP, fp64) on a bounded
         sample of the same workload (a 512^2 solve per step, the cpu_baseline's size) on the host cores.
Multi-GPU (N > 1): one process per GPU under torchrun (bench.py relaunches itself
under torch.distributed.run when WORLD_SIZE is unset): `--mode slabs` (default) splits the ONE 4096^2
problem into N row slabs (libsvk multi-GPU mode over NCCL: halo exchanges,
coarse-level agglomeration, all-reduced Krylov dots; strong scaling);
`--mode replicas` solves an independent 4096^2 problem per rank (weak scaling).
Time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Vanka sweep DOF/s + HBM GB/s vs peak; FGMRES-MG time-to-solve at 1/2/4/8 B200"
# Algorithmic work per pressure node (= per patch) of one fused sweep; see
# DESIGN.md "Roofline accounting".  Bytes: read x, read b, write x_out = 3 x 8 B
# per DOF.  FP64 flops of the parity-blocked Schur patch solve + stencil residual.
FLOPS_PER_NODE = 1316
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2: guide's SM count x DFMA/clk x max clock
L2_BYTES = 126e6


def n_dof(N: int) -> int:
    return 2 * (2 * N + 1) ** 2 + (N + 1) ** 2


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def measured_dfma_tflops():
    try:
        with open(os.path.join(ROOT, "profiles", "r2_fp64_peak.json")) as f:
            return float(json.load(f)["fp64_fma_tflops"])
    except (OSError, ValueError, KeyError):
        return None


def ncu_traffic():
    """dram__bytes_read.sum + write.sum per fused-sweep launch from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if p[5 + k].lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    """Reference arm: the CPU oracle on a bounded sample, rank 0 only."""
    world, rank, local = dist_setup(args)
    if rank != 0:
        return 0
    import oracle
    N = args.ref_n
    o = oracle.Oracle(N)
    b, x0 = o.problem(oracle.MMS_PAPER)
    for _ in range(args.warmup):
        o.fgmres(b, x0, rtol=args.rtol)
    t = []
    its = 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, its, _, _, _ = o.fgmres(b, x0, rtol=args.rtol)
        t.append(time.perf_counter() - t0)
    tot = sum(t)
    value = n_dof(N) * args.steps / tot
    cores = oracle.max_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong" if world > 1 and args.mode == "slabs" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(config_dict(args, world, n=N),
                       bounded_sample_of=config_dict(args, world)["workload"],
                       sample_note="the CPU oracle solves the N=%d instance of the same workload per step (a 4096^2 "
                                   "oracle solve takes tens of minutes); value is its DOF/s" % N),
        "iterations": its,
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": cores, "kind": "oracle",
                         "sample": "FGMRES+V(1,1)-Vanka solve of the %d^2 MMS problem per step (oracle C++/OpenMP, "
                                   "setup excluded)" % N},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


RELAX_NAMES = {"vanka": "Vanka", "bs": "Braess-Sarazin", "su": "Schur-Uzawa"}


def config_dict(args, world=1, n=None):
    relax = getattr(args, "relax", "vanka")
    if n is not None:  # the size actually run (reference arm: the oracle's bounded sample)
        args = argparse.Namespace(**dict(vars(args), n=n))
    if getattr(args, "precond", "mg") == "bt":
        wl = ("configs[4] comparator: 2D Stokes Q2-Q1, %dx%d structured mesh, paper MMS, FGMRES(1e-10) + block-triangular "
              "preconditioner (3 V(3,3) Jacobi cycles per block)" % (args.n, args.n))
        relax = "block-triangular"
    elif relax == "vanka":
        tag = {4096: "configs[2]: ", 8192: "configs[3] size: "}.get(args.n, "")
        wl = "%s2D Stokes Q2-Q1, %dx%d structured mesh, paper MMS, FGMRES(1e-10)+V(1,1)-Vanka" % (tag, args.n, args.n)
    else:
        wl = ("configs[4] comparator: 2D Stokes Q2-Q1, %dx%d structured mesh, paper MMS, FGMRES(1e-10)+V(1,1)-%s"
              % (args.n, args.n, RELAX_NAMES[relax]))
    if getattr(args, "low_memory", False):
        wl += " (low-memory Krylov: V only, x = x0 + M sum y_j V_j)"
    return {"workload": wl, "relaxation": relax,
            "N": args.n, "levels_to": 4, "dofs": n_dof(args.n), "omega_v": 0.8, "weighting": "multiplicity",
            "sweep_impl": args.sweep, "l2": "inputs exceed L2 (%.2f GB per vector vs 126 MB L2)"
            % (n_dof(args.n) * 8 / 1e9),
            "parallelism": ("slabs%d" % world) if world > 1 and args.mode == "slabs" else "replicas%d" % world,
            "agglom_rows": args.agglom}


def cpu_baseline(args):
    import oracle
    N = args.cpu_n
    o = oracle.Oracle(N)
    b, x0 = o.problem(oracle.MMS_PAPER)
    # repeat the solve until about 10 s of CPU work (at most 5 solves)
    t, nsolve = 0.0, 0
    while nsolve < 5 and (nsolve == 0 or t < 10.0):
        t0 = time.perf_counter()
        _, its, _, _, _ = o.fgmres(b, x0, rtol=args.rtol)
        t += time.perf_counter() - t0
        nsolve += 1
    # context: the oracle's one full-size solve, recorded by tests/test_gpu_iterations_large.py
    # (SVK_LARGE_ORACLE=4096) on a GPU box's 16 host cores -- not re-timed in this run
    at_size = None
    try:
        with open(os.path.join(ROOT, "profiles", "r2_iteration_parity.jsonl")) as f:
            for ln in f:
                if ln.startswith("{"):
                    r = json.loads(ln)
                    if r["N"] == args.n and r["kind"] == "mms_paper":
                        at_size = {"N": r["N"], "solve_s": r["solve_s"], "setup_s": r["setup_s"],
                                   "dof_per_s": n_dof(r["N"]) / r["solve_s"], "cores": r["threads"],
                                   "iterations": r["iterations"],
                                   "source": "profiles/r2_iteration_parity.jsonl (recorded run, not re-timed here)"}
    except (OSError, ValueError, KeyError):
        pass
    return {"value": nsolve * n_dof(N) / t, "unit": "DOF/s", "cores": oracle.max_threads(), "kind": "oracle",
            "oracle_at_benched_size": at_size,
            "sample": "%d FGMRES+V(1,1)-Vanka solve(s) of the %d^2 MMS problem to %g (%d iterations each, %.1f s "
                      "in total; oracle C++/OpenMP, setup excluded)" % (nsolve, N, args.rtol, its, t)}


def run_svk(args):
    import numpy as np
    import torch
    from paper_2401_06277_b200 import Solver

    world, rank, local = dist_setup(args)
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)
    N = args.n
    slabs = world > 1 and args.mode == "slabs"
    t0 = time.perf_counter()
    if slabs:
        from paper_2401_06277_b200 import svk
        nid = svk.nccl_id_broadcast()
        S = Solver(N, sweep=args.sweep, device=dev, rank=rank, nranks=world, transport="nccl",
                   agglom_rows=args.agglom, nccl_id=nid, low_memory=args.low_memory)
    else:
        S = Solver(N, sweep=args.sweep, device=dev, relax=args.relax, precond=args.precond,
                   low_memory=args.low_memory)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    b, x0 = S.set_problem("mms_paper")
    x = S.new_vector()

    def step():
        x.copy_(x0)
        return S.fgmres(b, x, rtol=args.rtol, maxit=args.maxit)

    # profiling on before the warm-up: the V-cycle graphs with the sweep-timing
    # events are captured there, not in the timed region
    S.set_profiling(True)
    for _ in range(args.warmup):
        rep, _ = step()
    S.sweep_stats()  # reset
    clocks = ClockSampler(dev)
    clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = S.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record()
    ev[0].record()
    reps = []
    for k in range(args.steps):
        rep, _ = step()
        reps.append(rep)
        ev[k + 1].record()
    e1.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    launches = S.launch_count - launches0
    nsw, sw_ms = S.sweep_stats()
    S.set_profiling(False)
    t = e0.elapsed_time(e1) / 1e3
    step_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    if dist:
        tt = torch.tensor([t], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    ms_step = 1e3 * t / args.steps
    jobs = 1 if slabs else world  # problems solved per step by the whole job
    value = jobs * n_dof(N) * args.steps / t
    its = [r["iterations"] for r in reps]

    # sweep roofline (dominant kernel); comparator runs have no Vanka sweep to time
    if nsw == 0:
        nsw, sw_ms = 1, float("nan")
    t_sweep = sw_ms / 1e3 / max(nsw, 1)
    r0, r1, _ = S.owned_rows()
    share = (r1 - r0) / (N + 1)  # this rank's slab of the sweep (1 on a single GPU)
    nodes = (N + 1) ** 2 * share
    bytes_alg = 3 * 8 * n_dof(N) * share
    hbm_peak, hbm_src = measured_peaks()
    sweep_gbs = bytes_alg / t_sweep / 1e9
    flops = FLOPS_PER_NODE * nodes
    achieved_tf = flops / t_sweep / 1e12
    traffic = ncu_traffic()
    roofline = {"bound": "alu", "achieved": achieved_tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved_tf / FP64_PEAK_TFLOPS,
                "traffic": traffic.get("bytes_per_launch") if traffic else None,
                "kernel": "k_vanka_fused, finest level (timed window opens after the sweep's k_boundary_patches "
                          "launch: the O(N) boundary patches, 0.2% of the patches, are solved there)",
                "launches": nsw, "avg_ms": 1e3 * t_sweep,
                "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (B200_PROFILING.md counts)",
                "hbm": {"achieved": sweep_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": sweep_gbs / hbm_peak,
                        "peak_source": hbm_src, "algorithmic_bytes": bytes_alg}}
    # the combined roofline time max(bytes/BW, flops/FP64 peak) over the measured time,
    # the fraction of the measured DFMA-loop rate (tools/fp64_peak), and the paper-equivalent rate
    # (dense 51x51 patch apply, 5202 flop/patch, tab:rwf) for comparison with P:640
    t_roof = max(bytes_alg / (hbm_peak * 1e9), flops / (FP64_PEAK_TFLOPS * 1e12))
    roofline["roofline_time_frac"] = t_roof / t_sweep
    dfma = measured_dfma_tflops()
    if dfma:
        roofline["frac_of_measured_dfma"] = {"value": achieved_tf / dfma, "measured_tflops": dfma,
                                             "source": "profiles/r2_fp64_peak.json (tools/fp64_peak.cu)"}
    roofline["paper_equivalent_tflops"] = 5202 * nodes / t_sweep / 1e12

    # second roofline entry: the FGMRES orthogonalisation (mat-vec + Gram-Schmidt
    # multi-dot / multi-update kernels), HBM-bound.  Algorithmic vectors streamed
    # per iteration j (m = j+1 basis vectors): mat-vec 2 (read z, write w),
    # dots m+1 (V_0..V_j, w), update m+2 (V_0..V_j, w read; w' written); a
    # second Gram-Schmidt pass adds m + (m+2).  Vector = owned rows incl. padding.
    rep_last = reps[-1]
    k_its, n_re = rep_last["iterations"], rep_last.get("n_reorth", 0)
    lat = 2 * N + 1
    vec_bytes = 8.0 * (2 * lat * ((lat + 7) // 8 * 8) + (N + 1) * ((N + 2 + 6) // 8 * 8)) * share
    nvec = sum(2 + (j + 2) + (j + 3) for j in range(k_its))
    # adaptive second passes: their iterations are not reported; charge them at the average m
    nvec += n_re * (2 * ((k_its + 1) / 2) + 2)
    orth_bytes = nvec * vec_bytes
    t_orth = rep_last["t_orth_s"]
    roofline_orth = {"bound": "hbm", "kernels": "k_residual_strip (mat-vec), k_cgs_dots, k_cgs_update, k_reduce_partials",
                     "achieved": orth_bytes / t_orth / 1e9, "peak": hbm_peak, "unit": "GB/s",
                     "frac": orth_bytes / t_orth / 1e9 / hbm_peak, "algorithmic_bytes": orth_bytes,
                     "vectors_streamed": nvec, "t_s": t_orth, "peak_source": hbm_src,
                     "traffic": "profiles/r2_krylov_ncu.json (DRAM bytes = algorithmic per launch)"}

    # end to end through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        bh = S.to_compact(b).cpu().pin_memory()
        x0h = S.to_compact(x0).cpu().pin_memory()
        xh = torch.empty_like(bh).pin_memory()
        bn, x0n, xn = bh.numpy(), x0h.numpy(), xh.numpy()
        S.solve_host(bn, x0n, rtol=args.rtol, x_host=xn)  # warm

        def tmax_of(t):
            if dist:
                tt = torch.tensor([t], device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t = float(tt.item())
            return t

        # (1) one svk_solve_host call per step: copies in, solve, copy out, serially
        if dist:
            dist.barrier()
        te = []
        for _ in range(args.e2e_steps):
            t1 = time.perf_counter()
            _, repe = S.solve_host(bn, x0n, rtol=args.rtol, x_host=xn)
            te.append(time.perf_counter() - t1)
        t_serial = tmax_of(sum(te))
        # (2) svk_solve_host_batch over the steps as a stream of problems (own pinned
        # input / output arrays per step): every step's H2D and D2H are made, the
        # copies of steps k+1 / k-1 overlapping the solve of step k
        kb = max(args.e2e_steps, 8)
        bl = [torch.empty_like(bh).pin_memory().numpy() for _ in range(kb)]
        x0l = [torch.empty_like(bh).pin_memory().numpy() for _ in range(kb)]
        xl = [torch.empty_like(bh).pin_memory().numpy() for _ in range(kb)]
        for a, c in zip(bl, x0l):
            a[:] = bn
            c[:] = x0n
        S.solve_host_batch(bl[:2], x0l[:2], rtol=args.rtol, x_hosts=xl[:2])  # warm: staging buffers, copy streams
        if dist:
            dist.barrier()
        t1 = time.perf_counter()
        _, repb, _ = S.solve_host_batch(bl, x0l, rtol=args.rtol, x_hosts=xl)
        t_batch = tmax_of(time.perf_counter() - t1)
        assert all(r["iterations"] == repe["iterations"] for r in repb) and np.array_equal(xl[-1], xn)
        e2e = {"value": jobs * n_dof(N) * kb / t_batch, "unit": "DOF/s",
               "h2d_bytes_per_step": world * 2 * n_dof(N) * 8, "d2h_bytes_per_step": world * n_dof(N) * 8,
               "steps": kb, "ms_per_step": 1e3 * t_batch / kb,
               "api": "svk_solve_host_batch (a stream of %d problems from pinned compact host arrays; the H2D of "
                      "step k+1 and the D2H of step k-1 overlap the solve of step k on two copy streams)" % kb,
               "serial": {"value": jobs * n_dof(N) * args.e2e_steps / t_serial, "steps": args.e2e_steps,
                          "ms_per_step": 1e3 * t_serial / args.e2e_steps,
                          "api": "svk_solve_host per step (copies in, solve, copy out, nothing overlapped)"}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if slabs else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (paper manufactured solution, P:76-81)",
            "config": config_dict(args, world),
            "time_to_solve_s": ms_step / 1e3, "iterations": its[-1], "iterations_all": its, "step_ms": step_ms,
            "rel_residual": reps[-1]["rel_residual"], "setup_s": setup_s, "t_setup_s": reps[-1]["t_setup_s"],
            "t_vcycle_s": reps[-1]["t_vcycle_s"], "t_orth_s": reps[-1]["t_orth_s"],
            "sweep": {"dof_per_s": n_dof(N) * share / t_sweep, "slab_share": share, "ms": 1e3 * t_sweep, "hbm_gbs_alg": sweep_gbs,
                      "hbm_frac": sweep_gbs / hbm_peak, "gflops_alg": achieved_tf * 1e3},
            "roofline": roofline, "roofline_orth": roofline_orth, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": launches,
        }
        if args.relax != "vanka" or args.precond != "mg":  # comparator line: no Vanka sweep in it
            line["sweep"] = line["roofline"] = line["roofline_orth"] = None
        elif args.sweep != "fused":  # comparator line: the roofline accounting is the fused kernel's
            line["roofline"] = None
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_emulated(args):
    """--emulate: args.gpus logical ranks in threads on cuda:0 through the EMULATED
    transport (row slabs, halo exchanges, agglomeration all-gather, all-reduced
    dots; only the byte mover differs from NCCL).  A logic check of the
    multi-GPU path at full size, not a multi-GPU measurement.  Every rank holds
    full-size b and x (as each GPU would), so P ranks on one GPU need P of them:
    4096^2 with 8 ranks fits one B200, 8192^2 does not.  A failing rank ends the
    process (the others would wait at the next emulated barrier)."""
    import threading
    import torch
    from paper_2401_06277_b200 import Solver
    P, N = args.gpus, args.n
    Ss = [Solver(N, rank=r, nranks=P, transport="emulated", agglom_rows=args.agglom, emul_group=4242,
                 low_memory=args.low_memory) for r in range(P)]
    res = [None] * P

    def body(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                S = Ss[r]
                b, x0 = S.set_problem("mms_paper")
                x = S.new_vector()
                for _ in range(args.warmup):
                    x.copy_(x0)
                    S.fgmres(b, x, rtol=args.rtol, maxit=args.maxit)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                its = []
                for _ in range(args.steps):
                    x.copy_(x0)
                    rep, _ = S.fgmres(b, x, rtol=args.rtol, maxit=args.maxit)
                    its.append(rep["iterations"])
                e1.record(st)
                st.synchronize()
                res[r] = (e0.elapsed_time(e1) / 1e3, its, rep["rel_residual"], S.device_bytes)
        except BaseException as e:  # noqa: BLE001 - the other ranks would wait at the next emulated barrier
            sys.stderr.write("emulated rank %d failed: %r\n" % (r, e))
            sys.stderr.flush()
            os._exit(1)

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    t = max(q[0] for q in res)
    line = {"metric": METRIC, "value": n_dof(N) * args.steps / t, "unit": "DOF/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (paper manufactured solution, P:76-81)",
            "emulated": "%d logical ranks on one GPU (emulated transport): a logic check of the slab path, "
                        "not a multi-GPU measurement" % P,
            "config": dict(config_dict(args, P), parallelism="slabs%d-emulated" % P),
            "iterations": res[0][1][-1], "iterations_per_rank": [q[1][-1] for q in res],
            "rel_residual": res[0][2], "device_bytes_per_rank": [q[3] for q in res]}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["svk", "reference"], default="svk")
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--rtol", type=float, default=1e-10)
    ap.add_argument("--maxit", type=int, default=60,
                    help="FGMRES iteration cap (no restart: 2 vectors of 1.2 GB per iteration at 4096^2)")
    ap.add_argument("--sweep", choices=["fused", "unfused", "simple"], default="fused",
                    help="unfused / simple (per-patch stored inverses, N <= 2048): the paper's split kernels, comparators")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-n", type=int, default=512)
    ap.add_argument("--ref-n", type=int, default=512)
    ap.add_argument("--mode", choices=["slabs", "replicas"], default="slabs")
    ap.add_argument("--agglom", type=int, default=64)
    ap.add_argument("--low-memory", action="store_true",
                    help="keep only the Arnoldi basis V (right-preconditioned GMRES with the fixed V-cycle, one "
                         "extra V-cycle at the end): halves the Krylov memory, e.g. 8192^2 on one B200")
    ap.add_argument("--emulate", action="store_true",
                    help="--gpus N logical ranks on one GPU through the emulated transport (logic check)")
    ap.add_argument("--relax", choices=["vanka", "bs", "su"], default="vanka",
                    help="V-cycle relaxation; bs / su are the paper's same-run comparators (configs[4], 1 GPU)")
    ap.add_argument("--precond", choices=["mg", "bt"], default="mg",
                    help="FGMRES preconditioner; bt = the paper's block-triangular comparator (configs[4], 1 GPU)")
    args = ap.parse_args()
    if args.precond != "mg" and (args.gpus > 1 or args.impl == "reference"):
        ap.error("--precond bt: single-GPU comparator runs of the svk arm only")
    if args.relax != "vanka" and (args.gpus > 1 or args.impl == "reference"):
        ap.error("--relax bs/su: single-GPU comparator runs of the svk arm only")
    if args.warmup < 3:
        args.warmup = 3
    if args.emulate:
        return run_emulated(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this script under torchrun (the driver's own launch sets WORLD_SIZE)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_svk(args)


if __name__ == "__main__":
    sys.exit(main())
