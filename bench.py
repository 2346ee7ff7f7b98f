#!/usr/bin/env python
"""bench.py — condensed DoFs/s solved to rtol 1e-8 (FGMRES + p-MG V-cycle).

Workload (default): BASELINE.json config 2(a) — unit square, 256x256 cells
split into triangles, interior vertices jittered by 0.2h (SplitMix64 seed 0),
HHO-dp (hybrid velocity, discontinuous pressure) with element velocity
condensed, k = 3, p-levels 3 -> 2 -> 1 -> 0, V(2,2) with the reference's
ILU(0)-GMRES smoother, ILU-GMRES coarse solve (rtol 1e-3, maxit 400),
FGMRES(30) to rtol 1e-8, sin/cos manufactured data, FP64.

One step = one reference `t_solve` (plevels.hpp:217-235): hierarchy setup
(operator inheritance, ILU(0) factorisations, sweep schedules) + FGMRES on
the condensed system resident in HBM. value = dofs x n_gpus / step time
(replicas: the 2D path does not shard). e2e = the same through the one-call
C ABI (pscu_solve_system) from host buffers, copies inside the timed region.

--impl reference times the reference's own solver (oracle/_ref, the
unmodified headers) on the host cores: every core (bounded by memory) runs
the same bounded sample of the workload concurrently — for config 2 the
recipe at 128x128, one FGMRES iteration per step, extrapolated to the full
solve as t_setup + its x t_iteration (see reference_timed).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "config1": dict(tri=False, n=16, jitter=0.0, seed=0, k=1, strategy="v-cond", degrees=[1, 0],
                    coarse="lu", name="2D unit square 16x16 quads, HHO-dp v-cond, k=1, levels 1-0",
                    ref_sample_n=16, outer_its=None),
    "config2a": dict(tri=True, n=256, jitter=0.2, seed=0, k=3, strategy="v-cond",
                     degrees=[3, 2, 1, 0], coarse="gmres-ilu",
                     name="2D unit square 256x256x2 jittered tris (0.2h, seed 0), HHO-dp v-cond, "
                          "k=3, levels 3-2-1-0",
                     ref_sample_n=128, outer_its=45),
    "config2b": dict(tri=True, n=256, jitter=0.2, seed=0, k=3, strategy="vp-cond",
                     degrees=[3, 2, 1, 0], coarse="gmres-ilu",
                     name="2D unit square 256x256x2 jittered tris (0.2h, seed 0), HHO-dp vp-cond, "
                          "k=3, levels 3-2-1-0",
                     ref_sample_n=128, outer_its=None),
}
# 3D (BASELINE.json configs 3 and 5): HHO-hp vp-cond on jittered hexahedra,
# face-block operators, block-Jacobi-smoothed V-cycles, ILU-GMRES coarse.
# The reference is 2D only: the CPU side is the oracle restatement ("port").
CONFIGS3 = {
    "config3": dict(dim=3, n=32, jitter=0.15, seed=1, fseed=2, k=2, degrees=[2, 1, 0], smooth=3,
                    name="3D unit cube 32^3 hexahedra (jitter 0.15h, seed 1), HHO-hp vp-cond, k=2, "
                         "levels 2-1-0, V(3,3) block-Jacobi, random modal f (seed 2)",
                    ref_sample_n=8),
    "config5": dict(dim=3, n=64, jitter=0.1, seed=4, fseed=5, k=2, degrees=[2, 1, 0], smooth=2,
                    name="3D unit cube 64^3 hexahedra (jitter 0.1h, seed 4), HHO-hp vp-cond, k=2, "
                         "levels 2-1-0, V(2,2) block-Jacobi, random modal f (seed 5)",
                    ref_sample_n=8),
    # config 4: the reference's DG (BR2, assemble.hpp:177-346) in 3D; levels
    # 3-2-1 because DG needs a coarsest degree >= 1 (plevels.hpp:137-139,
    # SURVEY.md §0 finding 7)
    "config4": dict(dim=3, scheme="dg", n=32, jitter=0.0, seed=0, fseed=3, k=3,
                    degrees=[3, 2, 1], smooth=2,
                    name="3D unit cube 32^3 uniform hexahedra, DG (BR2) k=3 equal order "
                         "(80x80 element blocks, DG block storage), levels 3-2-1, V(2,2) "
                         "block-Jacobi, random modal f (seed 3)",
                    ref_sample_n=4),
}
CONFIGS.update(CONFIGS3)
METRIC = "condensed DoFs/s solved to rtol 1e-8 (FGMRES+p-MG V-cycle)"
RTOL = 1e-8
RESTART = 30


from paper_2009_13840_b200.replicas import Replicas, dist_env  # noqa: E402


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_record(cls: str, config: str):
    """dram bytes per launch of the dominant kernel class on this config from
    the committed `ncu --set full` capture summary (profiles/ncu_summary.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        return d.get("traffic_bytes_per_launch", {}).get(config, {}).get(cls)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# reference arm / CPU baseline (oracle/_ref, test infrastructure)
# ---------------------------------------------------------------------------

def _ref_worker(args):
    """One reference process: assemble the sample (untimed, like the
    reference's own t_solve), then time hierarchy setup + FGMRES."""
    cfg, n, mode, rounds, maxit = args
    # sampled mode runs exactly `maxit` FGMRES iterations (rtol 0: the
    # reference's fixed-iteration convention, gmres.hpp:103-139), so the
    # per-iteration stamps exist for any --warmup/--steps; full mode solves
    # to the workload's rtol.
    rtol = RTOL if mode == "full" else 0.0
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ref as O

    s = O.RefSystem(mesh="unit-tri" if cfg["tri"] else "unit-quad", n=n, seed=cfg["seed"],
                    jitter=cfg["jitter"], side="top", scheme="hho-dp", strategy=cfg["strategy"],
                    k=cfg["k"], data="sincos")
    out = []
    for _ in range(rounds):
        t_setup, stamps = s.solve_timed(cfg["degrees"], maxit, coarse=cfg["coarse"], rtol=rtol,
                                        restart=RESTART)
        if mode != "full" and len(stamps) < maxit:
            raise RuntimeError(f"reference sample stopped after {len(stamps)} of {maxit} "
                               "fixed FGMRES iterations (breakdown)")
        out.append((t_setup, stamps.tolist()))
    return s.n, out


def _ref_procs(n_cells: int) -> int:
    """All host cores, bounded by memory (~2 GB per 128^2 k=3 sample)."""
    procs = os.cpu_count() or 1
    try:
        import psutil

        per = max(0.25e9, 2.5e9 * (n_cells / 128.0) ** 2)
        procs = max(1, min(procs, int(psutil.virtual_memory().available * 0.8 // per)))
    except Exception:
        pass
    return procs


def reference_timed(cfg: dict, n: int, procs: int, warmup: int, steps: int):
    """Reference solver timing on the host cores (oracle/_ref: the unmodified
    reference headers). `procs` processes each run the same sample.

    full mode (sample == workload size): every step is one complete solve,
    t_solve = setup + all FGMRES iterations (the reference's own t_solve).
    sampled mode (sample smaller than the workload): every step is one FGMRES
    iteration (one V-cycle + Arnoldi step) of the sample; the solve time is
    t_setup + its * t_iteration with `its` the workload's FGMRES iteration
    count, i.e. the sample's per-DoF cost of a setup and an iteration applied
    to the full solve (both scale linearly with the DoFs at fixed levels).
    Returns (per-step DoF/s values, sample DoFs, description)."""
    import multiprocessing as mp

    full = n == cfg["n"]
    if full:
        job = (cfg, n, "full", warmup + steps, 1000)
    else:
        job = (cfg, n, "sampled", 1, warmup + steps)
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_ref_worker, [job] * procs)
    dofs = res[0][0]
    vals = []
    if full:
        for r in range(warmup + steps):
            t = max(w[1][r][0] + w[1][r][1][-1] for w in res)  # slowest process
            vals.append(dofs * procs / t)
        its = len(res[0][1][0][1])
        desc = (f"reference solve_system recipe at {n}x{n} ({dofs} DoFs, {its} FGMRES its), "
                f"{procs} concurrent single-threaded processes, one solve per step")
        return vals[warmup:], dofs, desc, None
    its_full = cfg["outer_its"]
    t_setup = max(w[1][0][0] for w in res)
    for k in range(warmup, warmup + steps):
        t_it = max((w[1][0][1][k] - (w[1][0][1][k - 1] if k else 0.0)) for w in res)
        vals.append(dofs * procs / (t_setup + its_full * t_it))
    desc = (f"reference hierarchy setup + FGMRES iterations of the recipe at {n}x{n} "
            f"({dofs} DoFs), {procs} concurrent single-threaded processes; one step = one "
            f"FGMRES iteration, solve time = t_setup + {its_full} x t_iteration "
            f"({its_full} = the workload's FGMRES iteration count)")
    return vals, dofs, desc, t_setup


def _port3_worker(args):
    """One oracle-restatement process (3D has no reference): host local blocks
    + port condensation/assembly (untimed), then `rounds` timed solves
    (hierarchy setup + FGMRES, the reference's t_solve)."""
    cfg, n, rounds = args
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ref as O
    from paper_2009_13840_b200 import host

    m = host.Mesh3(n, jitter=cfg["jitter"], seed=cfg["seed"])
    if cfg.get("scheme") == "dg":
        D = host.DgLocal3(cfg["k"])
        lay = O.po_layout(2, 0, cfg["k"], m.n_faces, m.n_elements, dim=3)
        a, b = O.port_dg_assemble(lay, m.faces(), *D.local_terms(m, data="random",
                                                                 seed=cfg["fseed"], nthreads=1))
        return _port3_solves(O, a, b, lay, cfg, rounds)
    L = host.HpLocal3(cfg["k"])
    mats, rhs = L.local_blocks(m, 0, m.n_elements, data="random", seed=cfg["fseed"], nthreads=1)
    brp, bcols = m.block_pattern()
    rp, cols = O.bsr_to_csr_pattern(brp, bcols, L.face_block)
    lay = O.po_layout(1, 2, cfg["k"], m.n_faces, m.n_elements, dim=3)
    a, b = O.port_condense_assemble(mats, rhs, L.n_local, L.elim, L.kept_global(m.element_faces()),
                                    lay, rp, cols)
    del mats
    return _port3_solves(O, a, b, lay, cfg, rounds)


def _port3_solves(O, a, b, lay, cfg, rounds):
    out = []
    for _ in range(rounds):
        t0 = time.perf_counter()
        h = O.PortHierarchy(a, lay, cfg["degrees"], smoother_iters=cfg["smooth"], smoother=1)
        r = h.solve(b, rtol=RTOL, maxit=1000, restart=RESTART)
        out.append(time.perf_counter() - t0)
        del h
    return a.n, out, r["its"]


def reference3_timed(cfg, n, procs, warmup, steps):
    import multiprocessing as mp

    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_port3_worker, [(cfg, n, warmup + steps)] * procs)
    dofs, its = res[0][0], res[0][2]
    vals = [dofs * procs / max(w[1][r] for w in res) for r in range(warmup, warmup + steps)]
    desc = (f"oracle restatement (oracle/pstokes_oracle.c; the reference has no 3D) solving the "
            f"recipe at {n}^3 ({dofs} DoFs, {its} FGMRES its), {procs} concurrent single-threaded "
            f"processes, one solve (hierarchy setup + FGMRES) per step")
    return vals, dofs, desc


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    if cfg.get("dim") == 3:
        n = args.ref_sample_n or cfg["ref_sample_n"]
        procs = os.cpu_count() or 1
        vals, dofs, desc = reference3_timed(cfg, n, procs, args.warmup, args.steps)
        v = statistics.mean(vals)
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": "DoF/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dofs * procs / v,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (random modal body force)",
            "config": {"workload": cfg["name"], "sample": f"{n}^3", "sample_dofs": dofs,
                       "solver": "oracle restatement LevelHierarchy + FGMRES(30)",
                       "parallelism": f"{procs} concurrent single-threaded processes"},
            "cpu_baseline": {"value": v, "unit": "DoF/s", "cores": procs, "kind": "port",
                             "sample": desc},
            "e2e": {"value": v, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    n = args.ref_sample_n or cfg["ref_sample_n"]
    procs = _ref_procs(n)
    vals, dofs, desc, _ = reference_timed(cfg, n, procs, args.warmup, args.steps)
    v = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "DoF/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dofs * procs / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (manufactured sin/cos field)",
        "config": {"workload": cfg["name"], "sample": f"{n}x{n}", "sample_dofs": dofs,
                   "solver": "reference LevelHierarchy + FGMRES(30)",
                   "parallelism": f"{procs} concurrent single-threaded processes"},
        "cpu_baseline": {"value": v, "unit": "DoF/s", "cores": procs, "kind": "reference",
                         "sample": desc},
        "e2e": {"value": v, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours3(args, cfg):
    """3D configs: host local blocks -> streamed device condensation into
    face-block storage (untimed, like the reference's t_assembly), then one
    step = hierarchy setup + FGMRES on the device-resident operator."""
    ws, rank, local = dist_env()
    import numpy as np

    rep_group = Replicas("nccl")
    barrier, max_over_ranks = rep_group.barrier, rep_group.max_over_ranks
    from paper_2009_13840_b200 import host
    from paper_2009_13840_b200 import solver as S

    n = args.n or cfg["n"]
    ctx = S.Context(local)
    t0 = time.time()
    mesh = host.Mesh3(n, jitter=cfg["jitter"], seed=cfg["seed"])
    dg = cfg.get("scheme") == "dg"
    if dg:
        A, b, lay, info = host.assemble_dg3(mesh, cfg["k"], data="random", seed=cfg["fseed"],
                                            ctx=ctx)
        info.update(t_local_s=info["t_assembly_s"], t_condense_s=0.0)
    else:
        A, b, lay, info = host.assemble_stokes3(mesh, cfg["k"], data="random", seed=cfg["fseed"],
                                                ctx=ctx)
    t_asm = time.time() - t0
    lcfg = S.LevelConfig(degrees=cfg["degrees"], smoother_iters=cfg["smooth"], coarse="gmres-ilu",
                         smoother="bjacobi", outer_rtol=RTOL, restart=RESTART)
    dofs = A.n
    setup_s = []

    def step():
        t_h = time.perf_counter()
        h = S.LevelHierarchy(A, lay, lcfg)
        setup_s.append(time.perf_counter() - t_h)
        x, hist, rep = h.solve(b)
        del h
        return rep

    reps = [step() for _ in range(args.warmup)]
    barrier()
    ctx.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.launches()
    ctx.profile(True)
    times = []
    for _ in range(args.steps):
        ctx.timer_start()
        reps.append(step())
        times.append(ctx.timer_stop() / 1e3)
    ctx.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    launches = ctx.launches() - launches0
    barrier()
    clk = clocks.stop()
    t_step = max_over_ranks(statistics.mean(times))
    rep = reps[-1]
    # e2e through the one-call C ABI from pinned host buffers (block pattern,
    # values, load): the 40 GB of block values cross PCIe/C2C every step
    from paper_2009_13840_b200 import _native as N
    pinned = N.PinnedArray(A.nnz)
    brp, bcols, bvals = A.download_blocks(vals_out=pinned.a)
    bh = np.array(b)
    bs = A.block_size
    e2e_times = []
    for _ in range(max(1, args.e2e_steps)):
        ctx.timer_start()
        if dg:
            x, hist, r2 = S.solve_system_dgb(brp, bcols, bvals, A.dg_modes, bh, lay, lcfg, ctx=ctx)
        else:
            x, hist, r2 = S.solve_system_bsr(brp, bcols, bvals, bs, bh, lay, lcfg, ctx=ctx)
        e2e_times.append(ctx.timer_stop() / 1e3)
    t_e2e = max_over_ranks(statistics.mean(e2e_times))
    h2d = brp.nbytes + bcols.nbytes + bvals.nbytes + bh.nbytes
    d2h = x.nbytes
    del bvals, pinned
    if rank != 0:
        return
    peak, peak_src = peaks()
    dom = max(prof, key=lambda k: prof[k][1])
    cnt, ms, byt = prof[dom]
    achieved = (byt / (ms / 1e3)) / 1e9 if ms > 0 else 0.0
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        try:
            sn = args.ref_sample_n or cfg["ref_sample_n"]
            vals, sdofs, desc = reference3_timed(cfg, sn, 1, 0, 1)
            cpu = {"value": vals[0], "unit": "DoF/s", "cores": 1, "kind": "port", "sample": desc}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "DoF/s", "cores": 1, "kind": "port",
                   "sample": f"unavailable: {e}"}
    t_cond = info["t_condense_s"]
    line = {
        "metric": METRIC, "value": dofs * ws / t_step, "unit": "DoF/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (random modal body force, BASELINE.json config recipe)",
        "config": {
            "workload": cfg["name"] + (f" [n={n}]" if n != cfg["n"] else ""),
            "dofs": dofs, "nnz": A.nnz, "fgmres_its": rep.outer_its,
            "coarse_its_per_vcycle": rep.coarse_its / max(rep.vcycles, 1),
            "converged": rep.converged, "rel_residual": rep.rel_residual,
            "smoother": (f"block-Jacobi ({A.block_size}x{A.block_size} "
                         f"{'element' if dg else 'face'} blocks) GMRES "
                         f"V({cfg['smooth']},{cfg['smooth']})"),
            "coarse": "ILU-GMRES rtol 1e-3 maxit 400", "restart": RESTART,
            "step": "hierarchy setup + FGMRES (reference t_solve)",
            "l2": "inputs larger than L2 (fine operator %.2f GB)" % (8 * A.nnz / 1e9),
            "assembly_s_untimed": round(t_asm, 3),
            "local_blocks_host_s": round(info["t_local_s"], 3),
            "condense_device_s": round(t_cond, 3) if not dg else None,
            "dofs_per_s_incl_condense": dofs * ws / (t_step + t_cond),
            "parallelism": f"replicas x{ws}",
            "hierarchy_setup_s_in_step": round(setup_s[-1], 3),
        },
        "e2e": {"value": dofs * ws / t_e2e, "unit": "DoF/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches // max(args.steps, 1)),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic_record(dom, args.config),
                     "peak_source": peak_src, "launch_groups": cnt, "avg_ms": ms / max(cnt, 1),
                     "share_of_step": (ms / 1e3) / (sum(times))},
        "kernel_classes": {k: {"launch_groups": v[0], "ms": v[1],
                               "GBps": (v[2] / (v[1] / 1e3)) / 1e9 if v[1] > 0 else 0.0}
                           for k, v in prof.items()},
        "clocks": clk, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def run_ours3_zslab(args, cfg):
    """3D configs sharded by z-slab over the ranks (SURVEY.md §8(e),
    paper_2009_13840_b200/zslab.py): each rank assembles its face shard on
    its GPU; one step = shard setup (inheritance, block-Jacobi, gathered
    coarse operator + ILU(0)) + the sharded FGMRES(30) solve with ghost
    exchanges and dot allreduces over NCCL; the coarse ILU-GMRES is
    replicated. Strong scaling (the problem is fixed as N grows)."""
    ws, rank, local = dist_env()
    import torch

    rep_group = Replicas("nccl")
    barrier, max_over_ranks = rep_group.barrier, rep_group.max_over_ranks
    from paper_2009_13840_b200 import host, zslab
    from paper_2009_13840_b200 import solver as S

    n = args.n or cfg["n"]
    ctx = S.Context(local)
    mesh = host.Mesh3(n, jitter=cfg["jitter"], seed=cfg["seed"])
    part = zslab.SlabPartition(mesh, ws)
    v = part.view(rank)
    t0 = time.time()
    A, b = zslab.assemble_local(mesh, v, cfg["k"], data="random", seed=cfg["fseed"], ctx=ctx)
    t_asm = time.time() - t0
    bt = torch.as_tensor(b, device=torch.device("cuda", local))
    dofs = mesh.n_faces * A.block_size

    def step():
        ops = zslab.GpuOps(v, A, cfg["k"], part, ctx)
        solver = zslab.ZSlabSolver(ops, zslab.Dist(), len(cfg["degrees"]),
                                   smoother_iters=cfg["smooth"])
        x, hist, its, conv = solver.solve(bt, rtol=RTOL, maxit=1000, restart=RESTART)
        return its, conv, solver

    for _ in range(args.warmup):
        step()
    barrier()
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        # CUDA events on the current stream; every library call in between
        # completes on its own stream before returning, so the end event
        # follows all of the step's device work
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        its, conv, solver = step()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    barrier()
    t_step = max_over_ranks(statistics.mean(times))
    if rank != 0:
        return
    print(json.dumps({
        "metric": METRIC, "value": dofs / t_step, "unit": "DoF/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (random modal body force, BASELINE.json config recipe)",
        "config": {"workload": cfg["name"] + (f" [n={n}]" if n != cfg["n"] else ""),
                   "dofs": dofs, "fgmres_its": its, "converged": conv,
                   "coarse_its_per_vcycle": solver.coarse_its / max(solver.vcycles, 1),
                   "parallelism": f"z-slab x{ws} (faces by z-layer slab, NCCL ghost exchange + "
                                  "dot allreduce, replicated coarse)",
                   "assembly_s_untimed": round(t_asm, 3),
                   "timing": "CUDA events per step, max over ranks"},
    }), flush=True)


def run_ours(args, cfg):
    if cfg.get("dim") == 3 and args.shard == "zslab":
        return run_ours3_zslab(args, cfg)
    if cfg.get("dim") == 3:
        return run_ours3(args, cfg)
    ws, rank, local = dist_env()
    import numpy as np

    rep_group = Replicas("nccl")
    barrier, max_over_ranks = rep_group.barrier, rep_group.max_over_ranks
    from paper_2009_13840_b200 import host
    from paper_2009_13840_b200 import solver as S

    n = args.n or cfg["n"]
    ctx = S.Context(local)
    t0 = time.time()
    mesh = host.Mesh.unit_square(n, tri=cfg["tri"], jitter=cfg["jitter"], seed=cfg["seed"],
                                 neumann="top")
    loc = host.LocalSystem(mesh, "hho-dp", cfg["strategy"], cfg["k"], data="sincos")
    A, b = host.assemble_stokes(loc, ctx=ctx)
    t_asm = time.time() - t0
    lay = loc.layout()
    lcfg = S.LevelConfig(degrees=cfg["degrees"], coarse=cfg["coarse"], outer_rtol=RTOL,
                         restart=RESTART)
    dofs = A.n

    setup_s = []

    def step():
        t_h = time.perf_counter()
        h = S.LevelHierarchy(A, lay, lcfg)
        setup_s.append(time.perf_counter() - t_h)
        x, hist, rep = h.solve(b)
        del h
        return rep

    reps = []
    for _ in range(args.warmup):
        reps.append(step())
    barrier()
    ctx.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.launches()
    ctx.profile(True)
    times = []
    for _ in range(args.steps):
        ctx.timer_start()
        reps.append(step())
        times.append(ctx.timer_stop() / 1e3)
    ctx.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    launches = ctx.launches() - launches0
    barrier()
    clk = clocks.stop()
    t_step = max_over_ranks(statistics.mean(times))
    rep = reps[-1]

    # e2e through the one-call C ABI from host buffers
    rp, cl, vl = A.download()
    bh = np.array(b)
    e2e_times = []
    for _ in range(max(1, args.e2e_steps)):
        ctx.timer_start()
        x, hist, r2 = S.solve_system(rp, cl, vl, bh, lay, lcfg, ctx=ctx)
        e2e_times.append(ctx.timer_stop() / 1e3)
    t_e2e = max_over_ranks(statistics.mean(e2e_times))
    h2d = rp.nbytes + cl.nbytes + vl.nbytes + bh.nbytes
    d2h = x.nbytes

    if rank != 0:
        return
    # dominant kernel class and its roofline
    peak, peak_src = peaks()
    dom = max(prof, key=lambda k: prof[k][1])
    cnt, ms, byt = prof[dom]
    achieved = (byt / (ms / 1e3)) / 1e9 if ms > 0 else 0.0
    traffic = traffic_record(dom, args.config)
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        try:
            sn = args.ref_sample_n or cfg["ref_sample_n"]
            vals, sdofs, desc, _ = reference_timed(cfg, sn, 1, 0, 1)
            cpu = {"value": vals[0], "unit": "DoF/s", "cores": 1, "kind": "reference",
                   "sample": desc}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "DoF/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    line = {
        "metric": METRIC,
        "value": dofs * ws / t_step,
        "unit": "DoF/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_step * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (manufactured sin/cos field, BASELINE.json config recipe)",
        "config": {
            "workload": cfg["name"] + (f" [n={n}]" if n != cfg["n"] else ""),
            "dofs": dofs, "nnz": A.nnz, "fgmres_its": rep.outer_its,
            "coarse_its_per_vcycle": rep.coarse_its / max(rep.vcycles, 1),
            "converged": rep.converged, "rel_residual": rep.rel_residual,
            "smoother": "ILU(0)-GMRES V(2,2) (reference smoother)",
            "coarse": "ILU-GMRES rtol 1e-3 maxit 400" if cfg["coarse"] != "lu" else "dense LU",
            "restart": RESTART, "step": "hierarchy setup + FGMRES (reference t_solve)",
            "l2": "inputs larger than L2 (fine operator %.2f GB)" % ((12 * A.nnz) / 1e9),
            "assembly_s_untimed": round(t_asm, 3), "parallelism": f"replicas x{ws}",
            "hierarchy_setup_s_in_step": round(setup_s[-1], 3),
        },
        "e2e": {"value": dofs * ws / t_e2e, "unit": "DoF/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches // max(args.steps, 1)),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src, "launch_groups": cnt,
                     "avg_ms": ms / max(cnt, 1),
                     "share_of_step": (ms / 1e3) / (sum(times))},
        "kernel_classes": {k: {"launch_groups": v[0], "ms": v[1],
                               "GBps": (v[2] / (v[1] / 1e3)) / 1e9 if v[1] > 0 else 0.0}
                           for k, v in prof.items()},
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config5", choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=0, help="override the mesh size (testing)")
    ap.add_argument("--ref-sample-n", type=int, default=0,
                    help="mesh size of the reference / cpu_baseline sample (default per config)")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="replicas", choices=["replicas", "zslab"],
                    help="3D multi-GPU mode: independent replicas (weak scaling, default) or "
                         "the z-slab sharded solve (strong scaling)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
