"""Run harness on the GPU: the reference's run/sweep/report/CLI cases
(tests/test_bench.py:132-357) through the CUDA path, the `gpu` record
section, and the devices axis as a real sharded solve (2 ranks sharing one
GPU through the IPC mailboxes)."""

import os
import socket

import numpy as np
import pytest

from paper_2304_04876_b200.harness import (
    CSV_COLUMNS, RunConfig, emit_report, main, read_csv_report, read_json_report, record_dict,
    record_row, run_single, run_sweep,
)

pytestmark = pytest.mark.gpu


def write_config(path, lines):
    path.write_text("\n".join(lines) + "\n")
    return str(path)


def test_default_run_shape_and_gpu_section():
    rec = run_single(RunConfig())
    assert rec.error_msg == ""
    assert (rec.n, rec.n_interface, rec.n_coarse) == (729, 386, 8)
    assert rec.converged and rec.iterations == 17     # reference: 17 (acceptance criterion 1)
    assert rec.true_error < 1e-5
    assert rec.t_symbolic > 0 and rec.t_numeric > 0 and rec.t_solve > 0
    assert rec.max_local_size > 0 and rec.peak_factor_nnz > 0
    assert rec.solution is None
    g = rec.gpu
    assert g["devices_used"] == 1 and g["gpu_launches"] > 0
    assert g["solve_ms"] > 0 and g["apply_ms"] > 0 and g["apply_bytes"] > 0
    assert 0 < g["apply_frac_of_hbm"] < 1.5
    assert g["roofline"]["kernel"] and 0 < g["roofline"]["frac"] < 1.5


def test_deterministic_and_seeded():
    a = run_single(RunConfig(), keep_solution=True, measure=False)
    b = run_single(RunConfig(), keep_solution=True, measure=False)
    assert a.iterations == b.iterations and a.true_error == b.true_error
    assert np.array_equal(a.solution, b.solution)
    c = run_single(RunConfig.from_keys({"seed": 3}), keep_solution=True, measure=False)
    assert c.converged and not np.array_equal(a.solution, c.solution)


def test_coarse_level_helps_at_many_subdomains():
    base = {"problem.nx": 21, "problem.ny": 21, "problem.nz": 21,
            "partition.px": 5, "partition.py": 5, "partition.pz": 5}
    two = run_single(RunConfig.from_keys(base), measure=False)
    one = run_single(RunConfig.from_keys({**base, "coarse": "none"}), measure=False)
    assert two.converged and one.converged
    assert two.n_coarse > 0 and one.n_coarse == 0 and two.iterations < one.iterations


def test_failures_become_records():
    rec = run_single(RunConfig.from_keys({"problem.boundary": "neumann"}))
    assert not rec.converged and "coarse matrix" in rec.error_msg and "\n" not in rec.error_msg
    assert rec.n == 9 ** 3
    ok = run_single(RunConfig.from_keys({"problem.boundary": "neumann", "coarse": "none"}),
                    measure=False)
    assert ok.converged and ok.error_msg == ""


def test_sweeps():
    base = RunConfig.from_keys({"problem.nx": 13, "problem.ny": 13, "problem.nz": 13})
    recs = run_sweep(base, "subdomains", ["8", "12", "27"], measure=False)
    assert [(r.config.px, r.config.py, r.config.pz) for r in recs[::2]] == [(2, 2, 2), (3, 3, 3)]
    assert recs[0].converged and recs[2].converged
    assert "perfect cube" in recs[1].error_msg and not recs[1].converged
    counts = [r.iterations for r in run_sweep(RunConfig.from_keys({"local_solver": "ilu_k(0)"}),
                                              "ilu_level", ["0", "1", "2"], measure=False)]
    assert counts == sorted(counts, reverse=True)
    recs = run_sweep(RunConfig(), "devices", ["1", "2", "4"], measure=False)
    assert [r.device_subdomains for r in recs] == [[8], [4, 4], [2, 2, 2, 2]]
    assert len({r.iterations for r in recs}) == 1 and len({r.true_error for r in recs}) == 1
    recs = run_sweep(RunConfig(), "precision", ["double", "single"], measure=False)
    assert all(r.converged for r in recs) and recs[0].iterations == recs[1].iterations


def test_reports_from_real_runs(tmp_path):
    recs = [run_single(RunConfig()), run_single(RunConfig.from_keys({"problem.boundary": "neumann"}))]
    p1, p2 = tmp_path / "a.csv", tmp_path / "b.csv"
    emit_report(recs, str(p1), "csv")
    rows = read_csv_report(str(p1))
    emit_report(rows, str(p2), "csv")
    assert p1.read_bytes() == p2.read_bytes()
    assert rows[0]["true_error"] == recs[0].true_error and rows[1]["true_error"] is None
    assert tuple(record_row(recs[0])) == CSV_COLUMNS
    pj = tmp_path / "r.json"
    emit_report(recs, str(pj), "json")
    import json
    assert read_json_report(str(pj))[0] == json.loads(json.dumps(record_dict(recs[0])))


def test_cli(tmp_path, capsys):
    cfg = write_config(tmp_path / "run.cfg", ["problem.kind = laplace3d", "problem.nx = 7",
                                             "problem.ny = 7", "problem.nz = 7"])
    assert main(["solve", "--config", cfg]) == 0
    out = capsys.readouterr().out
    assert "converged=true" in out and "iterations=" in out and "GB/s" in out
    assert main(["solve", "--config", cfg, "--coarse", "gdsw"]) == 0
    assert "coarse=gdsw" in capsys.readouterr().out
    assert main(["solve", "--config", cfg, "--krylov.max_iters", "2"]) == 1
    report = tmp_path / "s.csv"
    assert main(["sweep", "--config", cfg, "--axis", "overlap", "--values", "0,1",
                 "--output", str(report)]) == 0
    assert [r["overlap"] for r in read_csv_report(str(report))] == [0, 1]
    assert main(["sweep", "--config", cfg, "--axis", "local_solver",
                 "--values", "exact_lu,ilu_k(1),fast_ilu(0,3,5)"]) == 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


_SHARD_KEYS = {"problem.nx": 14, "problem.ny": 14, "problem.nz": 16, "partition.px": 2,
               "partition.py": 2, "partition.pz": 4, "local_solver": "fast_ilu(0,3,5)",
               "ordering": "natural", "krylov.variant": "single_reduce"}


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rec = run_single(RunConfig.from_keys({**_SHARD_KEYS, "devices": world}), keep_solution=True)
        q.put((rank, rec.error_msg, rec.iterations, rec.converged, rec.device_subdomains,
               rec.gpu.get("devices_used"), rec.solution, rec.n_coarse))
    finally:
        tdist.destroy_process_group()


def test_devices_axis_is_real_under_a_process_group():
    import torch.multiprocessing as mp
    world = 2
    single = run_single(RunConfig.from_keys({**_SHARD_KEYS, "devices": world}), keep_solution=True,
                        measure=False)
    assert single.converged and single.device_subdomains == [8, 8]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(60)
    for rank, err, its, conv, groups, used, x, n_c in res:
        assert err == "" and conv and used == world
        assert groups == [8, 8] and n_c == single.n_coarse
        assert its == single.iterations
        np.testing.assert_allclose(x, single.solution, rtol=0, atol=1e-10 * np.abs(x).max())
