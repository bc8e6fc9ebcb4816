"""Run harness over the CUDA path.

The reference's benchmark contract (schwarzdd/bench.py): flat dotted-key
configs with command-line overrides (bench.py:45-73, 115-175, 273-286), the
compact local-solver tokens (227-270), `run_single` / `run_sweep` with
failures turned into records (307-418), the fixed CSV column order and the
JSON record form, both readable back (37-40, 420-527), and the `solve` /
`sweep` CLI with exit codes 0 / 1 / 2 (575-626). Every run here goes
through the public GPU API (`setup_symbolic`, `setup_numeric`, `gmres`).

Added on top of the reference's record: a `gpu` section in the JSON form --
device-timed solve and apply (CUDA events on the launching stream, after a
warm solve), the apply's algorithmic bytes from libgdsw's per-kernel
counters, its GB/s and fraction of the measured HBM peak
(MEASURED_PEAKS.json), the dominant solve kernel's roofline, and the number
of libgdsw launches of the solve. The CSV columns are unchanged, so reports
stay byte-compatible with the reference's readers.

The `devices` key is the reference's reporting label (subdomains grouped
per device, numerics untouched) in a single process. Under torchrun with
WORLD_SIZE == devices it is real: the run is the sharded solve of
`paper_2304_04876_b200.dist` (z-slabs of subdomains, one rank per GPU,
peer-memory collectives), `device_subdomains` lists the actual slabs, and
rank 0 prints and writes the report.
"""

from __future__ import annotations

import argparse
import csv
import dataclasses
import json
import os
import re
import sys
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .decomposition import box_partition, decompose
from .krylov import KrylovConfig, gmres
from .local_solvers import SolverSpec
from .model_problems import Grid3D, assemble_elasticity3d, assemble_laplace3d
from .schwarz import SchwarzConfig, setup_numeric, setup_symbolic

PROBLEM_KINDS = ("laplace3d", "elasticity3d")
COARSE_MODES = ("none", "gdsw", "rgdsw")
SWEEP_AXES = ("subdomains", "ilu_level", "overlap", "precision", "local_solver", "devices")
CSV_COLUMNS = ("problem", "n", "px", "py", "pz", "overlap", "coarse", "local_solver", "ordering",
               "precision", "n_coarse", "iterations", "converged", "t_symbolic", "t_numeric",
               "t_solve", "true_error", "error_msg")
_INT_COLUMNS = frozenset(("n", "px", "py", "pz", "overlap", "n_coarse", "iterations"))
_FLOAT_COLUMNS = frozenset(("t_symbolic", "t_numeric", "t_solve", "true_error"))

# dotted key -> (default text, attribute path in RunConfig, value type)
_SCHEMA = {
    "problem.kind": ("laplace3d", "kind", str),
    "problem.nx": ("9", "nx", int),
    "problem.ny": ("9", "ny", int),
    "problem.nz": ("9", "nz", int),
    "problem.boundary": ("dirichlet", "boundary", str),
    "problem.e": ("1.0", "e_mod", float),
    "problem.nu": ("0.3", "nu", float),
    "partition.px": ("2", "px", int),
    "partition.py": ("2", "py", int),
    "partition.pz": ("2", "pz", int),
    "overlap": ("1", "overlap", int),
    "coarse": ("rgdsw", "coarse", str),
    "local_solver.method": ("exact_lu", "solver.method", str),
    "local_solver.fill_level": ("0", "solver.fill_level", int),
    "local_solver.factor_sweeps": ("3", "solver.factor_sweeps", int),
    "local_solver.trisolve_iters": ("5", "solver.trisolve_iters", int),
    "local_solver.diag_shift": ("0.0", "solver.diag_shift", float),
    "ordering": ("nested_dissection", "ordering", str),
    "precision": ("double", "precision", str),
    "krylov.restart": ("30", "krylov.restart", int),
    "krylov.rel_tol": ("1e-7", "krylov.rel_tol", float),
    "krylov.max_iters": ("500", "krylov.max_iters", int),
    "krylov.variant": ("classic", "krylov.variant", str),
    "krylov.orthogonalization": ("mgs", "krylov.orthogonalization", str),
    "devices": ("1", "devices", int),
    "threads": ("1", "threads", int),
    "seed": ("0", "seed", int),
}


def _one_line(err: BaseException) -> str:
    return f"{type(err).__name__}: " + " ".join(str(err).split())


@dataclass(frozen=True)
class RunConfig:
    kind: str = "laplace3d"
    nx: int = 9
    ny: int = 9
    nz: int = 9
    boundary: str = "dirichlet"
    e_mod: float = 1.0
    nu: float = 0.3
    px: int = 2
    py: int = 2
    pz: int = 2
    overlap: int = 1
    coarse: str = "rgdsw"
    solver: SolverSpec = SolverSpec()
    ordering: str = "nested_dissection"
    precision: str = "double"
    krylov: KrylovConfig = KrylovConfig()
    devices: int = 1
    threads: int = 1
    seed: int = 0

    def __post_init__(self):
        if self.kind not in PROBLEM_KINDS:
            raise ValueError(f"unknown problem kind {self.kind!r}")
        if self.coarse not in COARSE_MODES:
            raise ValueError(f"unknown coarse mode {self.coarse!r}")
        bad = [k for k in ("px", "py", "pz", "devices", "threads") if getattr(self, k) < 1]
        if bad:
            raise ValueError(f"{bad[0]} must be positive")
        if self.overlap < 0:
            raise ValueError("overlap must be nonnegative")
        if self.coarse == "rgdsw" and sum(p > 1 for p in (self.px, self.py, self.pz)) < 2:
            raise ValueError("rgdsw needs at least 2 subdomains per axis in at least 2 axes; "
                             "use gdsw for slab partitions")

    @classmethod
    def from_keys(cls, keys: dict) -> "RunConfig":
        text = {k: v[0] for k, v in _SCHEMA.items()}
        for raw_key, value in keys.items():
            key = raw_key.strip()
            if key == "local_solver":      # compact token, e.g. fast_ilu(0,3,5)
                spec = parse_solver_token(str(value), SolverSpec())
                for name in ("method", "fill_level", "factor_sweeps", "trisolve_iters"):
                    text[f"local_solver.{name}"] = str(getattr(spec, name))
                continue
            if key not in _SCHEMA:
                raise ValueError(f"unknown config key {key!r}")
            text[key] = str(value)
        flat, groups = {}, {"solver": {}, "krylov": {}}
        for key, (_, path, typ) in _SCHEMA.items():
            try:
                val = typ(text[key])
            except ValueError:
                what = "an integer" if typ is int else "a number"
                raise ValueError(f"config key {key} needs {what}, got {text[key]!r}") from None
            head, _, tail = path.partition(".")
            if tail:
                groups[head][tail] = val
            else:
                flat[head] = val
        return cls(solver=SolverSpec(**groups["solver"]), krylov=KrylovConfig(**groups["krylov"]),
                   **flat)

    def to_keys(self) -> dict:
        """Flat dotted keys with native value types."""
        out = {}
        for key, (_, path, _) in _SCHEMA.items():
            obj = self
            for part in path.split("."):
                obj = getattr(obj, part)
            out[key] = obj
        return out


@dataclass
class RunRecord:
    config: RunConfig
    n: int = 0
    n_interface: int = 0
    n_coarse: int = 0
    iterations: int = 0
    converged: bool = False
    t_symbolic: float = 0.0
    t_numeric: float = 0.0
    t_solve: float = 0.0
    peak_factor_nnz: int = 0
    max_local_size: int = 0
    device_subdomains: list = field(default_factory=list)
    true_error: float | None = None
    error_msg: str = ""
    solution: np.ndarray | None = field(default=None, repr=False, compare=False)
    gpu: dict = field(default_factory=dict)


# ---------------------------------------------------------------------------
# local-solver tokens and config files
# ---------------------------------------------------------------------------
_TOKEN = re.compile(r"^\s*([A-Za-z_]+)\s*(?:\((.*)\))?\s*$")
_ARITY = {"exact_lu": 0, "ilu_k": 1, "fast_ilu": 3}
_ARITY_MSG = {"exact_lu": "exact_lu takes no arguments",
              "ilu_k": "ilu_k takes at most one argument (fill level)",
              "fast_ilu": "fast_ilu takes at most (fill, sweeps, trisolve_iters)"}


def parse_solver_token(token: str, base: SolverSpec) -> SolverSpec:
    """exact_lu | ilu_k(k) | fast_ilu(k, sweeps, iters); omitted arguments
    keep `base`'s values."""
    token = token.strip()
    m = _TOKEN.match(token)
    if m is None or ("(" in token and not token.endswith(")")):
        raise ValueError(f"malformed local solver {token!r}")
    name, inner = m.group(1), m.group(2)
    try:
        args = [int(a) for a in inner.split(",")] if inner and inner.strip() else []
    except ValueError:
        raise ValueError(f"malformed local solver {token!r}") from None
    if name not in _ARITY:
        raise ValueError(f"unknown local solver {name!r}")
    if len(args) > _ARITY[name]:
        raise ValueError(_ARITY_MSG[name])
    fields = ("fill_level", "factor_sweeps", "trisolve_iters")[:len(args)]
    return dataclasses.replace(base, method=name, **dict(zip(fields, args)))


def format_solver(spec: SolverSpec) -> str:
    return {"exact_lu": "exact_lu",
            "ilu_k": f"ilu_k({spec.fill_level})",
            "fast_ilu": f"fast_ilu({spec.fill_level},{spec.factor_sweeps},{spec.trisolve_iters})"
            }[spec.method]


def parse_config_file(path: str) -> dict:
    keys = {}
    with open(path) as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            key, eq, value = line.partition("=")
            if not eq:
                raise ValueError(f"{path}:{lineno}: expected 'key = value', got {raw.strip()!r}")
            keys[key.strip()] = value.strip()
    return keys


def split_values(text: str) -> list:
    """Comma split that keeps parenthesised solver arguments together."""
    out, depth, start = [], 0, 0
    for i, ch in enumerate(text + ","):
        depth += (ch == "(") - (ch == ")")
        if ch == "," and depth == 0:
            out.append(text[start:i].strip())
            start = i + 1
    return [t for t in out if t]


def _parse_overrides(extra: list) -> dict:
    out = {}
    for i in range(0, len(extra), 2):
        tok = extra[i]
        if not tok.startswith("--") or len(tok) <= 2:
            raise ValueError(f"expected --key value pairs, got {tok!r}")
        if i + 1 >= len(extra):
            raise ValueError(f"override {tok!r} is missing a value")
        out[tok[2:]] = extra[i + 1]
    return out


# ---------------------------------------------------------------------------
# runs
# ---------------------------------------------------------------------------
def assemble_problem(cfg: RunConfig):
    grid = Grid3D(cfg.nx, cfg.ny, cfg.nz)
    if cfg.kind == "laplace3d":
        return assemble_laplace3d(grid, boundary=cfg.boundary)
    return assemble_elasticity3d(grid, e_mod=cfg.e_mod, nu=cfg.nu, boundary=cfg.boundary)


def device_groups(cfg: RunConfig) -> list:
    """Subdomains per device label: as even as possible, larger groups first."""
    q, r = divmod(cfg.px * cfg.py * cfg.pz, cfg.devices)
    return [q + (d < r) for d in range(cfg.devices)]


def _sharded_world(cfg: RunConfig) -> int:
    """World size when this run is a real sharded solve, else 1."""
    if cfg.devices < 2:
        return 1
    try:
        import torch.distributed as tdist
    except ImportError:
        return 1
    if tdist.is_available() and tdist.is_initialized() and tdist.get_world_size() == cfg.devices:
        return cfg.devices
    return 1


def _symbolic_nnz(sym) -> int:
    return int(sym.l_idx.size + sym.u_idx.size)


def _peak_gbs():
    f = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    if f.exists():
        return float(json.loads(f.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _timed(fn, reps: int = 1) -> float:
    """Device milliseconds per call: CUDA events on the current stream."""
    from . import device
    t = device.torch()
    s = t.cuda.current_stream()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    t.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    t.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def _profiled(fn) -> dict:
    """libgdsw's per-kernel event counters around one call."""
    from . import device
    t = device.torch()
    t.cuda.synchronize()
    device.prof_reset()
    device.prof_enable(True)
    try:
        fn()
        t.cuda.synchronize()
    finally:
        device.prof_enable(False)
    return device.prof_read()


def _gpu_section(prob, pre, b: np.ndarray, kcfg: KrylovConfig, launches: int) -> dict:
    from . import device
    t = device.torch()
    peak, kind = _peak_gbs()
    bd = t.from_numpy(b).cuda()
    gmres(prob.a, pre, bd, kcfg)                     # warm: graphs captured
    its = []
    solve_ms = _timed(lambda: its.append(gmres(prob.a, pre, bd, kcfg)[1].iterations))
    phases = _profiled(lambda: gmres(prob.a, pre, bd, kcfg))
    live = {k: v for k, v in phases.items() if v["launches"] and v["ms"] > 0 and v["bytes"] > 0}
    dom = max(live, key=lambda k: live[k]["ms"]) if live else None
    r = t.from_numpy(np.random.default_rng(1).standard_normal(prob.a.nrows)).cuda()
    z = t.empty_like(r)
    for _ in range(3):
        pre.apply_device(r, z)
    apply_ms = _timed(lambda: pre.apply_device(r, z), reps=10)
    apply_bytes = sum(v["bytes"] for v in _profiled(lambda: pre.apply_device(r, z)).values())
    apply_gbs = apply_bytes / (apply_ms * 1e-3) / 1e9 if apply_ms > 0 else None
    out = {"device": t.cuda.get_device_name(), "devices_used": 1,
           "solve_ms": solve_ms, "ms_per_iteration": solve_ms / max(its[0], 1),
           "gpu_launches": launches, "apply_ms": apply_ms, "apply_bytes": apply_bytes,
           "apply_gbs": apply_gbs, "hbm_peak_gbs": peak, "peak_kind": kind,
           "apply_frac_of_hbm": apply_gbs / peak if apply_gbs else None, "roofline": None}
    if dom is not None:
        ph = live[dom]
        gbs = ph["bytes"] / (ph["ms"] * 1e-3) / 1e9
        out["roofline"] = {"bound": "hbm", "kernel": dom, "launches": ph["launches"],
                           "us_per_launch": 1e3 * ph["ms"] / ph["launches"],
                           "bytes_per_launch": ph["bytes"] / ph["launches"],
                           "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak}
    return out


def _run_local(rec: RunRecord, cfg: RunConfig, prob, dec, scfg: SchwarzConfig, mode,
               keep_solution: bool, measure: bool):
    from . import device
    t = device.torch()
    t0 = time.perf_counter()
    skel = setup_symbolic(prob.a, dec, scfg)
    rec.t_symbolic = time.perf_counter() - t0
    t0 = time.perf_counter()
    pre = setup_numeric(skel, prob.a, prob.nullspace if mode else None)
    t.cuda.synchronize()
    rec.t_numeric = time.perf_counter() - t0
    nnz = [_symbolic_nnz(s) for s in skel.local_symbolics]
    if pre.coarse is not None:
        rec.n_coarse = pre.coarse.a0.nrows
        nnz.append(_symbolic_nnz(pre.coarse.a0_factorization.symbolic))
    rec.peak_factor_nnz = max(nnz)
    x_star = np.random.default_rng(cfg.seed).standard_normal(rec.n)
    b = prob.a @ x_star
    l0 = device.launch_count()
    x, rep = gmres(prob.a, pre, b, cfg.krylov)
    launches = device.launch_count() - l0
    rec.iterations, rec.converged, rec.t_solve = rep.iterations, rep.converged, rep.timings.solve
    rec.true_error = float(np.linalg.norm(x - x_star) / np.linalg.norm(x_star))
    if keep_solution:
        rec.solution = x
    if measure:
        rec.gpu = _gpu_section(prob, pre, b, cfg.krylov, launches)


def _run_sharded(rec: RunRecord, cfg: RunConfig, prob, dec, scfg: SchwarzConfig, mode, world: int,
                 keep_solution: bool):
    """One rank's share of the sharded solve (dist.py); every rank ends with
    the same record (timings = max over ranks)."""
    import torch.distributed as tdist

    from . import device
    from .dist import DistPreconditioner, plan_shards
    t = device.torch()
    rank = tdist.get_rank()

    def wall_max(v):
        vs = [None] * world
        tdist.all_gather_object(vs, v)
        return max(vs)

    tdist.barrier()
    t0 = time.perf_counter()
    shards = plan_shards(prob.a, dec, world)
    rec.t_symbolic = wall_max(time.perf_counter() - t0)
    sh = shards[rank]
    rec.device_subdomains = [int(s.subs.size) for s in shards]
    t0 = time.perf_counter()
    dpre = DistPreconditioner(prob.a, dec, scfg, prob.nullspace if mode else None, sh)
    t.cuda.synchronize()
    rec.t_numeric = wall_max(time.perf_counter() - t0)
    rec.n_coarse = dpre.coarse_n
    nnz = [_symbolic_nnz(s) for s in dpre.local_symbolics]
    if dpre.coarse_n:
        nnz.append(_symbolic_nnz(dpre.a0_factorization.symbolic))
    rec.peak_factor_nnz = wall_max(max(nnz))
    x_star = np.random.default_rng(cfg.seed).standard_normal(rec.n)
    b = prob.a @ x_star
    tdist.barrier()
    l0 = device.launch_count()
    t0 = time.perf_counter()
    x_own, out = dpre.solve(t.from_numpy(b[sh.g0:sh.g1].copy()).cuda(), cfg.krylov)
    xh = x_own.cpu().numpy()
    rec.t_solve = wall_max(time.perf_counter() - t0)
    launches = device.launch_count() - l0
    pieces = [None] * world
    tdist.all_gather_object(pieces, xh)
    x = np.concatenate(pieces)
    rec.iterations, rec.converged = int(out["iterations"]), bool(out["converged"])
    rec.true_error = float(np.linalg.norm(x - x_star) / np.linalg.norm(x_star))
    if keep_solution:
        rec.solution = x
    rec.gpu = {"device": t.cuda.get_device_name(), "devices_used": world,
               "solve_ms": 1e3 * rec.t_solve, "ms_per_iteration": 1e3 * rec.t_solve / max(rec.iterations, 1),
               "gpu_launches": wall_max(launches)}


def run_single(cfg: RunConfig, keep_solution: bool = False, _assembled=None,
               measure: bool = True) -> RunRecord:
    """Assemble, decompose, set up (both phases) and solve b = A x* with
    x* = default_rng(seed).standard_normal(n) on the GPU (bench.py:307-358).
    Errors become a failure record. `measure` adds the `gpu` section."""
    rec = RunRecord(config=cfg, device_subdomains=device_groups(cfg))
    try:
        prob = _assembled if _assembled is not None else assemble_problem(cfg)
        rec.n = prob.a.nrows
        mode = None if cfg.coarse == "none" else cfg.coarse
        dec = decompose(prob.a, box_partition(prob.grid, cfg.px, cfg.py, cfg.pz), cfg.overlap, mode)
        if dec.structure is not None:
            rec.n_interface = int(len(dec.structure.interface))
        rec.max_local_size = max(len(s) for s in dec.overlap.sets)
        scfg = SchwarzConfig(local=cfg.solver, use_coarse=mode is not None, precision=cfg.precision,
                             ordering=cfg.ordering, threads=cfg.threads)
        world = _sharded_world(cfg)
        if world > 1:
            _run_sharded(rec, cfg, prob, dec, scfg, mode, world, keep_solution)
        else:
            _run_local(rec, cfg, prob, dec, scfg, mode, keep_solution, measure)
    except Exception as err:  # noqa: BLE001 -- the record carries it (bench.py:352-356)
        rec.error_msg = _one_line(err)
        rec.converged = False
    return rec


def _with_axis(base: RunConfig, axis: str, value: str) -> RunConfig:
    rep = dataclasses.replace
    if axis == "subdomains":
        total = int(value)
        p = round(total ** (1.0 / 3.0))
        if p ** 3 != total:
            raise ValueError(f"subdomain count {total} is not a perfect cube")
        return rep(base, px=p, py=p, pz=p)
    if axis == "ilu_level":
        return rep(base, solver=rep(base.solver, fill_level=int(value)))
    if axis == "local_solver":
        return rep(base, solver=parse_solver_token(str(value), base.solver))
    if axis in ("overlap", "devices"):
        return rep(base, **{axis: int(value)})
    if axis == "precision":
        return rep(base, precision=str(value))
    raise ValueError(f"unknown sweep axis {axis!r}")


def run_sweep(base: RunConfig, axis: str, values: list, measure: bool = True) -> list:
    """One run per value; a bad value becomes a failure record and the sweep
    goes on. Assembly is shared while the operator is unchanged."""
    if axis not in SWEEP_AXES:
        raise ValueError(f"unknown sweep axis {axis!r}")
    if axis == "ilu_level" and base.solver.method == "exact_lu":
        raise ValueError("ilu_level sweep needs an ilu_k or fast_ilu base local solver")
    if not values:
        raise ValueError("sweep needs at least one value")
    problems, records = {}, []
    for value in values:
        try:
            cfg = _with_axis(base, axis, value)
        except (ValueError, TypeError) as err:
            rec = RunRecord(config=base, device_subdomains=device_groups(base))
            rec.error_msg = _one_line(err)
            records.append(rec)
            continue
        key = (cfg.kind, cfg.nx, cfg.ny, cfg.nz, cfg.boundary, cfg.e_mod, cfg.nu)
        if key not in problems:
            problems[key] = assemble_problem(cfg)
        records.append(run_single(cfg, _assembled=problems[key], measure=measure))
    return records


# ---------------------------------------------------------------------------
# reports
# ---------------------------------------------------------------------------
def record_row(rec: RunRecord) -> dict:
    """The CSV row of a record (CSV_COLUMNS order)."""
    c = rec.config
    vals = (c.kind, rec.n, c.px, c.py, c.pz, c.overlap, c.coarse, format_solver(c.solver),
            c.ordering, c.precision, rec.n_coarse, rec.iterations, rec.converged,
            rec.t_symbolic, rec.t_numeric, rec.t_solve, rec.true_error, rec.error_msg)
    return dict(zip(CSV_COLUMNS, vals))


def record_dict(rec: RunRecord) -> dict:
    """The JSON form: the reference's record plus the `gpu` section."""
    return {"config": rec.config.to_keys(), "n": rec.n, "n_interface": rec.n_interface,
            "n_coarse": rec.n_coarse, "iterations": rec.iterations, "converged": rec.converged,
            "timings": {"symbolic": rec.t_symbolic, "numeric": rec.t_numeric, "solve": rec.t_solve},
            "peak_factor_nnz": rec.peak_factor_nnz, "max_local_size": rec.max_local_size,
            "device_subdomains": list(rec.device_subdomains), "true_error": rec.true_error,
            "error_msg": rec.error_msg, "gpu": dict(rec.gpu)}


def _cell(col: str, value) -> str:
    if value is None:
        return ""
    if col == "converged":
        return "true" if value else "false"
    return repr(float(value)) if col in _FLOAT_COLUMNS else str(value)


def emit_report(records: list, path: str, fmt: str = "csv"):
    """Write RunRecords (or rows / dicts read back earlier) as CSV or JSON."""
    if not records:
        raise ValueError("no records to report")
    if fmt not in ("csv", "json"):
        raise ValueError(f"unknown report format {fmt!r}")
    if fmt == "json":
        payload = [r if isinstance(r, dict) else record_dict(r) for r in records]
        Path(path).write_text(json.dumps(payload, indent=2) + "\n")
        return
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(CSV_COLUMNS)
        for r in records:
            row = r if isinstance(r, dict) else record_row(r)
            w.writerow([_cell(c, row[c]) for c in CSV_COLUMNS])


def _typed(col: str, cell: str):
    if col in _INT_COLUMNS:
        return int(cell)
    if col in _FLOAT_COLUMNS:
        return float(cell) if cell != "" else None
    if col == "converged":
        return cell == "true"
    return cell


def read_csv_report(path: str) -> list:
    with open(path, newline="") as fh:
        reader = csv.DictReader(fh)
        if reader.fieldnames != list(CSV_COLUMNS):
            raise ValueError(f"unexpected CSV header in {path}")
        return [{c: _typed(c, raw[c]) for c in CSV_COLUMNS} for raw in reader]


def read_json_report(path: str) -> list:
    return json.loads(Path(path).read_text())


# ---------------------------------------------------------------------------
# CLI: python -m paper_2304_04876_b200.harness solve|sweep --config FILE ...
# ---------------------------------------------------------------------------
def summary_line(rec: RunRecord) -> str:
    c = rec.config
    head = (f"{c.kind} {c.nx}x{c.ny}x{c.nz} part={c.px}x{c.py}x{c.pz} coarse={c.coarse} "
            f"solver={format_solver(c.solver)} precision={c.precision}")
    if rec.error_msg:
        return f"{head}: FAILED {rec.error_msg}"
    err = "" if rec.true_error is None else f" true_error={rec.true_error:.3e}"
    gpu = ""
    if rec.gpu.get("apply_gbs"):
        gpu = (f" gpu_solve={rec.gpu['solve_ms']:.3f}ms apply={rec.gpu['apply_ms']:.3f}ms"
               f" ({rec.gpu['apply_gbs']:.0f} GB/s, {100 * rec.gpu['apply_frac_of_hbm']:.0f}% of HBM)")
    return (f"{head}: iterations={rec.iterations} converged={'true' if rec.converged else 'false'}"
            f"{err} t_setup={rec.t_symbolic + rec.t_numeric:.3f}s t_solve={rec.t_solve:.3f}s{gpu}")


def _init_distributed():
    """torchrun: one rank per GPU, gloo for the host bootstrap (the data
    path uses libgdsw's peer-memory collectives). Returns the rank."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world < 2:
        return 0
    import torch
    import torch.distributed as tdist
    local = 0 if os.environ.get("GDSW_SAME_DEVICE") == "1" else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if not tdist.is_initialized():
        tdist.init_process_group("gloo")
    return tdist.get_rank()


def main(argv=None) -> int:
    parser = argparse.ArgumentParser(prog="schwarzdd",
                                     description="Two-level Schwarz preconditioner benchmark harness "
                                                 "(B200)")
    sub = parser.add_subparsers(dest="command", required=True)
    for name in ("solve", "sweep"):
        p = sub.add_parser(name)
        p.add_argument("--config", required=True, help="flat key-value config file")
        p.add_argument("--output", help="report file path")
        p.add_argument("--format", choices=("csv", "json"), default="csv")
        p.add_argument("--threads", type=int)
        p.add_argument("--seed", type=int)
        if name == "sweep":
            p.add_argument("--axis", required=True, choices=SWEEP_AXES)
            p.add_argument("--values", required=True, help="comma-separated axis values")
    args, extra = parser.parse_known_args(argv)
    try:
        keys = parse_config_file(args.config)
        keys.update(_parse_overrides(extra))
        for opt in ("threads", "seed"):
            if getattr(args, opt) is not None:
                keys[opt] = str(getattr(args, opt))
        cfg = RunConfig.from_keys(keys)
        rank = _init_distributed()
        if args.command == "solve":
            records = [run_single(cfg)]
        else:
            records = run_sweep(cfg, args.axis, split_values(args.values))
    except (ValueError, TypeError, OSError) as err:
        print(f"error: {err}", file=sys.stderr)
        return 2
    if rank == 0:
        for rec in records:
            print(summary_line(rec))
        if args.output:
            emit_report(records, args.output, args.format)
    return 0 if all(r.converged for r in records) else 1


if __name__ == "__main__":
    sys.exit(main())
