#!/usr/bin/env python
"""bench.py -- BASELINE.json's metric on B200:
"GDSW-GMRES solve s & iters to 1e-7, 3D Laplace 2M dof/GPU; apply HBM GB/s".

One step = one complete right-preconditioned single-reduce GMRES(30) solve
of A x = b to rtol 1e-7 (x0 = 0) on config C2 (BASELINE.json configs[1]):
3D 7-point Laplace 128^3 = 2,097,152 dof per GPU, 4x4x4 = 64 subdomains
batched per GPU, overlap 1, rGDSW coarse space, FastILU(0, 3 sweeps) +
FastSpTRSV(5 iterates) local solves, natural ordering, fp64.

* value / ms_per_step: device time of K solves (CUDA events on the solve
  stream, barrier + synchronize on both sides, max over ranks), inputs
  resident in HBM.
* e2e: the same solve through the public API with the right-hand side in
  pinned host memory and the solution read back every step.
* roofline: the dominant kernel's algorithmic bytes / its average launch
  time (CUDA events recorded by libgdsw on the launching stream during the
  timed region) against MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline: the oracle (plain-C restatement of the reference's
  sequential kernels + numpy GMRES): one full solve on 1 core.

--impl reference: the reference's CPU path (the oracle port with the
reference's setup restated in oracle/reference_setup.py, entirely on the
host) on the same workload: full solves on every host thread.
Multi-GPU (--gpus N self-launches torchrun; weak scaling): ONE global system
of N x 2M dof (128 x 128 x 128N grid, 4 x 4 x 4N boxes) sharded in z-slabs,
64 subdomains per GPU, every rank building only its own z-window
(paper_2304_04876_b200.slab); halos, the coarse right-hand side and the
GMRES block go through libgdsw's peer-memory collectives
(paper_2304_04876_b200.dist).
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import time
import types
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GDSW-GMRES solve s & iters to 1e-7, 3D Laplace 2M dof/GPU; apply HBM GB/s"
# iterations of the reference on C2 (measured by running it)
APPLY_PHASES = ("restrict_panels", "restrict_columns", "coarse_solve", "gather",
                "gather_jacobi_lower", "jacobi_lower", "jacobi_lower_diag", "diag_solve", "jacobi_upper", "jacobi_flow", "levelset",
                "prolong", "scatter")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="native", choices=("native", "reference"))
    # (not --n / --parts: torchrun's parser would claim those prefixes)
    p.add_argument("--grid", dest="n", type=int, default=128,
                   help="grid nodes per axis (per GPU)")
    p.add_argument("--boxes", dest="parts", type=int, default=4,
                   help="subdomain boxes per axis (per GPU)")
    p.add_argument("--solver", default="fast_ilu(0,3,5)")
    p.add_argument("--ordering", default="natural")
    p.add_argument("--precision", default="double")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-sample-iters", type=int, default=5)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--ref-budget", type=float, default=150.0,
                   help="--impl reference: seconds of timed full solves (at least one)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--sharded", action="store_true",
                   help="run the sharded (multi-GPU) code path even at one rank")
    p.add_argument("--profile-region", action="store_true",
                   help="cudaProfilerStart/Stop around the timed region (ncu --profile-from-start off)")
    return p.parse_args()


def solver_tuple(token: str):
    """(method, fill_level, factor_sweeps, trisolve_iters) of a solver token
    (no product import: the reference arm parses it too)."""
    name = token.split("(")[0]
    args = [int(x) for x in token[token.index("(") + 1:-1].split(",")] if "(" in token else []
    if name == "exact_lu":
        return ("exact_lu", 0, 3, 5)
    if name == "ilu_k":
        return ("ilu_k", (args[:1] or [0])[0], 3, 5)
    fill, sweeps, iters = (args + [0, 3, 5][len(args):])[:3]
    return ("fast_ilu", fill, sweeps, iters)


def solver_spec(token: str):
    from paper_2304_04876_b200.local_solvers import SolverSpec
    name = token.split("(")[0]
    args = [int(x) for x in token[token.index("(") + 1:-1].split(",")] if "(" in token else []
    if name == "exact_lu":
        return SolverSpec("exact_lu")
    if name == "ilu_k":
        return SolverSpec("ilu_k", *(args[:1] or [0]))
    fill, sweeps, iters = (args + [0, 3, 5][len(args):])[:3]
    return SolverSpec("fast_ilu", fill, sweeps, iters)


def build_problem_config(args):
    from paper_2304_04876_b200.schwarz import SchwarzConfig
    return SchwarzConfig(local=solver_spec(args.solver), ordering=args.ordering,
                         precision=args.precision)


def build_problem(args):
    from paper_2304_04876_b200.decomposition import box_partition, decompose
    from paper_2304_04876_b200.model_problems import Grid3D, assemble_laplace3d
    prob = assemble_laplace3d(Grid3D(args.n, args.n, args.n))
    part = box_partition(prob.grid, args.parts, args.parts, args.parts)
    dec = decompose(prob.a, part, 1, "rgdsw")
    return prob, dec, build_problem_config(args)


def workload(args, world: int = 1, sharded: bool = False) -> dict:
    n = args.n ** 3
    if world > 1 or sharded:
        par = (f"sharded x{world}: z-slabs of {args.parts ** 3} subdomains per GPU, global "
               f"{args.n}x{args.n}x{args.n * world} grid / {args.parts}x{args.parts}x"
               f"{args.parts * world} boxes; halos, coarse rhs and the GMRES block over "
               "libgdsw peer-memory collectives (CUDA IPC, NVLink)")
    else:
        par = "single GPU"
    if os.environ.get("GDSW_SAME_DEVICE") == "1" and world > 1:
        par += " -- every rank on cuda:0 (functional check; times are not a scaling measurement)"
    return {"workload": (f"C2: 3D Laplace 7-pt {args.n}^3 ({n:,} dof per GPU), "
                         f"{args.parts}x{args.parts}x{args.parts}={args.parts ** 3} subdomains "
                         f"per GPU, overlap 1, rGDSW, {args.solver} local solves, "
                         f"{args.ordering} ordering, {args.precision} preconditioner, "
                         "single-reduce GMRES(30) to rtol 1e-7, x0=0"),
            "dof_per_gpu": n, "subdomains_per_gpu": args.parts ** 3,
            "parallelism": par,
            "l2": "no flush: per-solve working set (A, factors, Phi panels, 2x30 Krylov "
                  "vectors ~1.9 GB) >> 126 MB L2"}


PHASE_KERNEL = {"jacobi_upper": "k_jacobi_upper", "jacobi_lower": "k_jacobi_lower",
                "sr_update": "k_sr_update", "block_dot": "k_block_dot_rg",
                "restrict_panels": "k_restrict_chunks", "prolong": "k_prolong",
                "spmv": "k_sell_spmv", "jacobi_fused": "k_jacobi_cluster"}


def ncu_traffic(phase: str):
    """DRAM read+write bytes per launch of the phase's kernel from the
    committed `ncu --set full` capture summary (profiles/*_ncu_summary.json),
    or None when no capture of that kernel exists."""
    kern = PHASE_KERNEL.get(phase)
    for f in sorted((ROOT / "profiles").glob("*_ncu_summary.json"), reverse=True):
        for c in json.loads(f.read_text()).get("captures", []):
            if c.get("kernel") == kern and c.get("traffic_bytes"):
                return {"bytes": c["traffic_bytes"], "source": f"profiles/{f.name}:{c['capture']}"}
    return None


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampled during the timed region."""

    def __init__(self, index: int):
        self.fh = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.fh.seek(0)
        rows = [r.split(",") for r in self.fh.read().strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for name, v in zip(names, r[5:9]):
                if v.strip() == "Active":
                    reasons.add(name)
        load = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": float(rows[0][2]),
                "reasons": sorted(reasons), "samples": len(rows)}


# ---------------------------------------------------------------------------
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def native(args):
    import torch
    import torch.distributed as tdist

    from paper_2304_04876_b200 import device
    from paper_2304_04876_b200.krylov import KrylovConfig, gmres
    from paper_2304_04876_b200.schwarz import setup_numeric, setup_symbolic

    world, rank, local = dist_setup()
    # GDSW_SAME_DEVICE=1: every rank on cuda:0 (functional check of the
    # sharded path on a single-GPU box; timings are then meaningless)
    if os.environ.get("GDSW_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    sharded = world > 1 or args.sharded
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "MASTER_PORT" not in os.environ:
            os.environ["MASTER_PORT"] = str(_free_port())
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        # bootstrap only (IPC handles, dense A0 partials, timing max); the data
        # path uses libgdsw's own peer-memory collectives
        tdist.init_process_group("gloo")

    def barrier():
        if sharded:
            tdist.barrier()

    def max_over_ranks(v: float) -> float:
        if not sharded:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    kcfg = KrylovConfig(variant="single_reduce")
    t0 = time.perf_counter()
    if not sharded:
        prob, dec, cfg = build_problem(args)
        n = prob.a.nrows
        x_star = np.random.default_rng(0).standard_normal(n)
        b = prob.a @ x_star
    else:
        # every rank builds only its z-window (slab.py): per-rank setup
        # independent of the number of GPUs
        from paper_2304_04876_b200.slab import build_slab_problem
        sp = build_slab_problem(args.n, args.n, args.parts, args.parts, world, rank)
        cfg = build_problem_config(args)
        n = sp.n_global
        x_star = np.random.default_rng(0).standard_normal(n)
        b = sp.a @ x_star[sp.offset:sp.offset + sp.a.nrows]   # window rows (owned ones exact)
    t_inputs = time.perf_counter() - t0
    t0 = time.perf_counter()
    if not sharded:
        skel = setup_symbolic(prob.a, dec, cfg)
        t_sym = time.perf_counter() - t0
        t0 = time.perf_counter()
        pre = setup_numeric(skel, prob.a, prob.nullspace)
        g0, g1 = 0, n

        def solve(bd):
            return gmres(prob.a, pre, bd, kcfg)
    else:
        from paper_2304_04876_b200.dist import DistPreconditioner, plan_slab_shard
        sh = plan_slab_shard(sp, world, rank)
        t_sym = time.perf_counter() - t0
        t0 = time.perf_counter()
        dpre = DistPreconditioner(sp.a, sp.dec, cfg, sp.nullspace, sh, slab=sp)
        g0, g1 = sh.g0, sh.g1

        def solve(bd):
            bd = bd if bd.is_cuda else bd.to("cuda", non_blocking=True)
            x, out = dpre.solve(bd, kcfg)
            return x, types.SimpleNamespace(iterations=out["iterations"],
                                            converged=out["converged"])
    torch.cuda.synchronize()
    t_num = time.perf_counter() - t0
    b_dev = torch.from_numpy(b[g0:g1].copy()).cuda()

    for _ in range(args.warmup):
        x, rep = solve(b_dev)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    l0 = device.launch_count()
    barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    if args.profile_region:
        torch.cuda.profiler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    reps = []
    for _ in range(args.steps):
        x, rep = solve(b_dev)
        reps.append(rep)
    e1.record(stream)
    torch.cuda.synchronize()
    if args.profile_region:
        torch.cuda.profiler.stop()
    barrier()
    clk = clocks.stop()
    launches = device.launch_count() - l0
    ms_step = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    # per-kernel roofline: an identical K-solve pass with libgdsw's CUDA-event
    # instrumentation on (events on the launching stream around every kernel;
    # kept out of the timed pass above because each record costs ~1 us)
    # The side-stream overlap of the coarse restriction is switched off for
    # this pass so that every kernel's event interval is its own (the timed
    # pass above runs with the overlap).
    os.environ["GDSW_NO_OVERLAP"] = "1"
    device.prof_reset()
    device.prof_enable(True)
    for _ in range(args.steps):
        solve(b_dev)
    torch.cuda.synchronize()
    device.prof_enable(False)
    del os.environ["GDSW_NO_OVERLAP"]
    phases = device.prof_read()
    its = reps[-1].iterations
    xh = x.cpu().numpy()
    if sharded:
        pieces = [None] * world
        tdist.all_gather_object(pieces, xh)
        xh = np.concatenate(pieces)
        res = (b - sp.a @ xh[sp.offset:sp.offset + sp.a.nrows])[g0:g1]
        sq = torch.tensor([float(res @ res), float(b[g0:g1] @ b[g0:g1])], dtype=torch.float64)
        tdist.all_reduce(sq)
        true_res = float(np.sqrt(sq[0].item() / sq[1].item()))
    else:
        true_res = float(np.linalg.norm(b - prob.a @ xh) / np.linalg.norm(b))
    true_err = float(np.linalg.norm(xh - x_star) / np.linalg.norm(x_star))

    peak, peak_kind = peaks()
    # per-phase achieved bandwidth; dominant = most device time
    table = {}
    for name, ph in phases.items():
        if ph["launches"] == 0 or ph["ms"] <= 0:
            continue
        table[name] = dict(ms_total=ph["ms"], launches=ph["launches"],
                           us_per_launch=1e3 * ph["ms"] / ph["launches"],
                           bytes_per_launch=ph["bytes"] / ph["launches"],
                           gbs=ph["bytes"] / (ph["ms"] * 1e-3) / 1e9)
    dom = max((k for k in table if table[k]["bytes_per_launch"] > 0),
              key=lambda k: table[k]["ms_total"])
    d = table[dom]
    app_ms = sum(table[k]["ms_total"] for k in APPLY_PHASES if k in table)
    app_bytes = sum(phases[k]["bytes"] for k in APPLY_PHASES if k in table)
    n_apply = max(1, max(phases.get(k, {}).get("launches", 0) for k in ("prolong", "scatter")))
    # one apply's wall time on the device (the coarse restriction overlaps
    # the local solves on a side stream, so the phase sum overstates it)
    apply_ms = app_ms / n_apply
    if not sharded:
        r_dev = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).cuda()
        z_dev = torch.empty_like(r_dev)
        for _ in range(3):
            pre._dev.apply(r_dev, z_dev)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(20):
            pre._dev.apply(r_dev, z_dev)
        a1.record(stream)
        torch.cuda.synchronize()
        apply_ms = a0.elapsed_time(a1) / 20
    apply_gbs = (app_bytes / n_apply) / (apply_ms * 1e-3) / 1e9 if apply_ms else None
    solve_ms = e0.elapsed_time(e1) / args.steps
    step_bytes = sum(ph["bytes"] for ph in phases.values()) / args.steps
    comm_ms = sum(table[k]["ms_total"] for k in ("halo_fwd", "halo_rev", "block_allreduce",
                                                 "coarse_allreduce") if k in table) / args.steps
    result = {
        "metric": METRIC, "value": ms_step / 1e3, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference generators (assemble_laplace3d), x*=default_rng(0)."
                "standard_normal(n), b=A x*",
        "config": workload(args, world, sharded),
        "iterations": its, "converged": bool(reps[-1].converged),
        "ms_per_iteration": ms_step / max(its, 1),
        "true_rel_residual": true_res, "true_error": true_err,
        "apply_gbs": apply_gbs, "apply_frac_of_hbm": apply_gbs / peak if apply_gbs else None,
        "apply_ms": apply_ms,
        "solve_gbs": step_bytes / (solve_ms * 1e-3) / 1e9,
        "comm_ms_per_solve": comm_ms,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": d["gbs"], "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": d["gbs"] / peak,
                     "traffic": (ncu_traffic(dom) or {}).get("bytes"),
                     "traffic_source": (ncu_traffic(dom) or {}).get("source"),
                     "us_per_launch": d["us_per_launch"],
                     "bytes_per_launch": d["bytes_per_launch"],
                     "timing": "libgdsw CUDA events on the launching stream, K-solve pass "
                               "identical to the timed one"},
        "phases": {k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in table.items()},
        "gpu_launches": launches,
        "clocks": clk,
        "setup_s": {"inputs": t_inputs, "symbolic_host": t_sym, "numeric": t_num},
    }
    if not args.no_e2e:
        bh = torch.from_numpy(b[g0:g1].copy()).pin_memory()
        if not sharded:
            def solve_host(bh):
                return gmres(prob.a, pre, bh, kcfg)
        else:
            def solve_host(bh):
                x, r = solve(bh.to("cuda", non_blocking=True))
                return x.cpu(), r
        # two warm calls: the returned solutions come from torch's caching
        # pinned allocator, whose blocks are populated by then
        for _ in range(2):
            xe, _ = solve_host(bh)
        torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            xe, repe = solve_host(bh)
        f1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = max_over_ranks(f0.elapsed_time(f1) / args.e2e_steps)
        nb = (g1 - g0) * 8
        result["e2e"] = {"value": e2e_ms / 1e3, "unit": "s", "h2d_bytes_per_step": nb * world,
                         "d2h_bytes_per_step": (nb + 8 * 2 * 31 * repe.iterations) * world,
                         "api": ("paper_2304_04876_b200.krylov.gmres(A, M, pinned host b)"
                                 if not sharded else
                                 "paper_2304_04876_b200.dist.DistPreconditioner.solve "
                                 "(pinned host b -> device, x -> host)")}
    if rank == 0 and not sharded and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args, prob, dec, cfg, skel, pre, b, its)
    if sharded:
        tdist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def _oracle_sample(ore, prob, b, sample_iters: int):
    from oracle import oracle as O
    t0 = time.perf_counter()
    _, rep = O.gmres(lambda v: O.csr_spmv(prob.a, v), ore.apply, b, max_iters=sample_iters)
    return (time.perf_counter() - t0) / max(rep["iterations"], 1)


def cpu_baseline(args, prob, dec, cfg, skel, pre, b, iterations):
    """Oracle port on 1 core (subdomain solves and BLAS on one thread): ONE
    full solve of the same system from x0 = 0 to rtol 1e-7 (the coarse basis
    taken from the GPU setup, local factors from the oracle's own FastILU)."""
    from oracle import oracle as O
    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(1)
    except Exception:
        limiter = None
    ore = O.OracleSchwarz(prob.a, dec, cfg, None, symbolics=skel.local_symbolics, threads=1,
                          coarse_parts=(pre.coarse.phi, pre.coarse.a0))
    t0 = time.perf_counter()
    _, rep = O.gmres(lambda v: O.csr_spmv(prob.a, v), ore.apply, b)
    value = time.perf_counter() - t0
    if limiter is not None and hasattr(limiter, "unregister"):
        limiter.unregister()
    return {"value": value, "unit": "s", "cores": 1, "kind": "port",
            "per_iteration_s": value / max(rep["iterations"], 1), "iterations": rep["iterations"],
            "cpu_model": cpu_model(),
            "sample": f"one full oracle single-reduce GMRES solve of the same system on 1 core "
                      f"(BLAS 1 thread): {rep['iterations']} iterations (GPU {iterations}); "
                      "oracle FastILU factors, coarse basis from the GPU setup"}


def _loaded_libraries() -> list:
    """Shared objects mapped into this process (/proc/self/maps)."""
    try:
        return sorted({line.split()[-1] for line in open("/proc/self/maps")
                       if line.rstrip().endswith(".so") and "/repo" in line})
    except OSError:
        return []


def cpu_model() -> str:
    """`lscpu`'s model name (BASELINE.md section 2 asks for it)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def reference(args):
    """The reference's CPU implementation of the path (oracle port) on this
    host: full CPU setup (FastILU, exact-LU harmonic extension), then FULL
    GMRES solves of the same system (x0 = 0 to rtol 1e-7), subdomain solves
    and BLAS on every host thread. Warm-up steps are short samples; the timed
    steps are whole solves, as many of the K requested as fit the time budget
    (--ref-budget seconds, at least one)."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    try:  # numpy BLAS (GMRES vector work) on every host thread as well
        from threadpoolctl import threadpool_limits
        threadpool_limits(cores)
    except Exception:
        pass
    method, fill, sweeps, iters = solver_tuple(args.solver)
    t0 = time.perf_counter()
    if (method == "fast_ilu" and fill == 0 and args.ordering == "natural"
            and args.precision == "double"):
        # the reference's setup restated inside the oracle (numpy + scipy +
        # liboracle): nothing of the product is loaded on this arm
        from oracle.reference_setup import IndependentSchwarz
        ore = IndependentSchwarz(args.n, args.n, args.n, args.parts, args.parts, args.parts,
                                 sweeps, iters, threads=cores)
        prob = types.SimpleNamespace(a=ore.a)
        setup_kind = "oracle/reference_setup.py (independent of the product)"
    else:
        prob, dec, cfg = build_problem(args)
        ore = O.OracleSchwarz(prob.a, dec, cfg, prob.nullspace, threads=cores)
        setup_kind = "product host layer for index sets (configuration outside reference_setup)"
    t_setup = time.perf_counter() - t0
    x_star = np.random.default_rng(0).standard_normal(prob.a.nrows)
    b = prob.a @ x_star
    for _ in range(args.warmup):
        _oracle_sample(ore, prob, b, args.cpu_sample_iters)
    times, iters, true_rel = [], None, None
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t1 = time.perf_counter()
        x, rep = O.gmres(lambda v: O.csr_spmv(prob.a, v), ore.apply, b)
        times.append(time.perf_counter() - t1)
        iters = rep["iterations"]
        if time.perf_counter() - t_all + times[-1] > args.ref_budget:
            break
    true_rel = float(np.linalg.norm(b - prob.a @ x) / np.linalg.norm(b))
    value = float(np.mean(times))
    sample = (f"oracle port of the reference path (plain-C sequential kernels + numpy "
              f"single-reduce GMRES): {len(times)} full solve(s) of the {workload(args)['workload']} "
              f"system from x0 = 0 to rtol 1e-7 ({iters} iterations, true relative residual "
              f"{true_rel:.2e}), subdomain solves on {cores} threads (the reference's `threads` "
              f"option) and BLAS on {cores} threads; {args.warmup} warm-up samples of "
              f"{args.cpu_sample_iters} iterations; setup {t_setup:.1f}s not timed, built by "
              f"{setup_kind}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": world,
        "steps": len(times), "steps_requested": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * value, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference generators, x*=default_rng(0).standard_normal(n), b=A x*",
        "config": workload(args), "iterations": iters, "ms_per_iteration": 1e3 * value / iters,
        "true_relative_residual": true_rel,
        "cpu_baseline": {"value": value, "unit": "s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "loaded_native": sorted({Path(p).name for p in _loaded_libraries()}),
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int | None:
    """`bench.py --gpus N` (N > 1) outside torchrun: re-exec this script
    under torch.distributed.run with N ranks, one per GPU (the driver's own
    launch form), so the sharded solve runs instead of a silent 1-GPU one.
    Returns the exit code, or None when no launch is needed."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if args.impl == "reference":
        return None      # rank 0's host work only: nothing to spread
    if os.environ.get("GDSW_SAME_DEVICE") != "1":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"metric": METRIC, "n_gpus": args.gpus,
                              "error": f"--gpus {args.gpus} but {have} CUDA device(s) visible "
                                       "(GDSW_SAME_DEVICE=1 runs every rank on cuda:0 as a "
                                       "functional check)"}), flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    code = self_launch(args)
    if code is not None:
        sys.exit(code)
    if args.impl == "reference":
        reference(args)
    else:
        native(args)


if __name__ == "__main__":
    main()
