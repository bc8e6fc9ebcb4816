"""Run-harness contract on the host (the reference's tests/test_bench.py
config, token, sweep-validation, report and CLI-error cases; runs that need
the GPU are in test_gpu_harness.py)."""

import json

import pytest

from paper_2304_04876_b200.harness import (
    CSV_COLUMNS, RunConfig, RunRecord, _parse_overrides, device_groups, emit_report,
    format_solver, main, parse_config_file, parse_solver_token, read_csv_report,
    read_json_report, record_dict, record_row, run_sweep, split_values,
)
from paper_2304_04876_b200.local_solvers import SolverSpec


def write_config(path, lines):
    path.write_text("\n".join(lines) + "\n")
    return str(path)


def test_empty_keys_give_defaults():
    assert RunConfig.from_keys({}) == RunConfig()


def test_to_keys_round_trips():
    cfg = RunConfig.from_keys({"problem.kind": "elasticity3d", "problem.nx": 5,
                               "local_solver": "fast_ilu(1,4,6)", "krylov.variant": "single_reduce",
                               "precision": "single", "devices": 3, "seed": 7, "coarse": "gdsw"})
    assert RunConfig.from_keys(cfg.to_keys()) == cfg
    assert cfg.to_keys()["local_solver.trisolve_iters"] == 6
    assert isinstance(cfg.to_keys()["problem.e"], float)


def test_unknown_and_bad_keys():
    with pytest.raises(ValueError, match="unknown config key"):
        RunConfig.from_keys({"problem.size": 3})
    with pytest.raises(ValueError, match="problem.nx needs an integer"):
        RunConfig.from_keys({"problem.nx": "nine"})
    with pytest.raises(ValueError, match="krylov.rel_tol needs a number"):
        RunConfig.from_keys({"krylov.rel_tol": "tiny"})


def test_compact_local_solver_key():
    cfg = RunConfig.from_keys({"local_solver": "fast_ilu(1,4,6)"})
    assert cfg.solver == SolverSpec(method="fast_ilu", fill_level=1, factor_sweeps=4,
                                    trisolve_iters=6)
    cfg = RunConfig.from_keys({"local_solver": "ilu_k(2)"})
    assert (cfg.solver.method, cfg.solver.fill_level) == ("ilu_k", 2)


def test_validation():
    with pytest.raises(ValueError, match="rgdsw needs at least 2"):
        RunConfig(px=4, py=1, pz=1)
    RunConfig(px=4, py=1, pz=1, coarse="gdsw")
    for kw, msg in ((dict(kind="heat"), "unknown problem kind"), (dict(coarse="x"), "unknown coarse"),
                    (dict(devices=0), "devices must be positive"),
                    (dict(threads=0), "threads must be positive"),
                    (dict(overlap=-1), "overlap must be nonnegative")):
        with pytest.raises(ValueError, match=msg):
            RunConfig(**kw)


def test_parse_config_file(tmp_path):
    path = write_config(tmp_path / "a.cfg", ["# comment", "problem.nx = 11  # trailing",
                                            "", "coarse=gdsw"])
    assert parse_config_file(path) == {"problem.nx": "11", "coarse": "gdsw"}
    bad = write_config(tmp_path / "b.cfg", ["problem.nx = 3", "oops"])
    with pytest.raises(ValueError, match="b.cfg:2"):
        parse_config_file(bad)


def test_solver_tokens():
    for tok in ("exact_lu", "ilu_k(3)", "fast_ilu(0,3,5)", "fast_ilu(2,10,20)"):
        assert format_solver(parse_solver_token(tok, SolverSpec())) == tok
    base = SolverSpec(method="fast_ilu", fill_level=1, factor_sweeps=7, trisolve_iters=9)
    spec = parse_solver_token("fast_ilu(2)", base)
    assert (spec.fill_level, spec.factor_sweeps, spec.trisolve_iters) == (2, 7, 9)
    for bad, msg in (("ilu_k(1,2)", "at most one"), ("exact_lu(1)", "no arguments"),
                     ("fast_ilu(1,2,3,4)", "at most"), ("ilu_k(x)", "malformed"),
                     ("ilu_k(1", "malformed"), ("amg", "unknown local solver")):
        with pytest.raises(ValueError, match=msg):
            parse_solver_token(bad, SolverSpec())


def test_split_values_and_overrides():
    assert split_values("0, 1,2") == ["0", "1", "2"]
    assert split_values("exact_lu,ilu_k(2),fast_ilu(0,3,5)") == \
        ["exact_lu", "ilu_k(2)", "fast_ilu(0,3,5)"]
    assert _parse_overrides(["--overlap", "2", "--coarse", "gdsw"]) == {"overlap": "2",
                                                                        "coarse": "gdsw"}
    with pytest.raises(ValueError, match="missing a value"):
        _parse_overrides(["--overlap"])
    with pytest.raises(ValueError, match="--key value"):
        _parse_overrides(["overlap", "2"])


def test_device_groups():
    assert [device_groups(RunConfig(devices=d)) for d in (1, 2, 3, 4)] == \
        [[8], [4, 4], [3, 3, 2], [2, 2, 2, 2]]


def test_sweep_validation_before_any_run():
    with pytest.raises(ValueError, match="unknown sweep axis"):
        run_sweep(RunConfig(), "restart", ["10"])
    with pytest.raises(ValueError, match="at least one value"):
        run_sweep(RunConfig(), "overlap", [])
    with pytest.raises(ValueError, match="ilu_k or fast_ilu base"):
        run_sweep(RunConfig(), "ilu_level", ["0", "1"])


def _records():
    ok = RunRecord(config=RunConfig(), n=729, n_interface=386, n_coarse=8, iterations=17,
                   converged=True, t_symbolic=0.125, t_numeric=0.1 + 0.2, t_solve=1 / 3,
                   true_error=1.2345678901234567e-9, device_subdomains=[8],
                   gpu={"solve_ms": 1.5, "apply_gbs": 100.0})
    bad = RunRecord(config=RunConfig.from_keys({"problem.boundary": "neumann"}), n=729,
                    error_msg="LinAlgError: coarse matrix is singular: pivot, too small")
    return [ok, bad]


def test_csv_round_trip_is_byte_identical(tmp_path):
    recs = _records()
    p1, p2 = tmp_path / "a.csv", tmp_path / "b.csv"
    emit_report(recs, str(p1), "csv")
    rows = read_csv_report(str(p1))
    emit_report(rows, str(p2), "csv")
    assert p1.read_bytes() == p2.read_bytes()
    assert p1.read_text().splitlines()[0] == ",".join(CSV_COLUMNS)
    assert rows[0]["converged"] is True and isinstance(rows[0]["iterations"], int)
    assert rows[0]["true_error"] == recs[0].true_error and rows[0]["t_numeric"] == 0.1 + 0.2
    assert rows[1]["converged"] is False and rows[1]["true_error"] is None
    assert rows[1]["error_msg"] == recs[1].error_msg


def test_csv_header_is_enforced(tmp_path):
    path = tmp_path / "r.csv"
    path.write_text("a,b,c\n1,2,3\n")
    with pytest.raises(ValueError, match="unexpected CSV header"):
        read_csv_report(str(path))


def test_json_round_trip_with_config_echo(tmp_path):
    recs = _records()
    path = tmp_path / "r.json"
    emit_report(recs, str(path), "json")
    loaded = read_json_report(str(path))
    assert loaded[0]["config"] == recs[0].config.to_keys()
    assert loaded[0] == json.loads(json.dumps(record_dict(recs[0])))
    assert loaded[0]["gpu"]["apply_gbs"] == 100.0
    assert loaded[1]["error_msg"] == recs[1].error_msg
    assert path.read_text().endswith("\n")


def test_record_row_and_emit_validation(tmp_path):
    row = record_row(_records()[0])
    assert tuple(row) == CSV_COLUMNS and row["local_solver"] == "exact_lu"
    with pytest.raises(ValueError, match="no records"):
        emit_report([], str(tmp_path / "x.csv"))
    with pytest.raises(ValueError, match="unknown report format"):
        emit_report(_records(), str(tmp_path / "x.xml"), "xml")


def test_cli_config_errors_exit_two(tmp_path, capsys):
    cfg = write_config(tmp_path / "run.cfg", ["problem.nx = 7"])
    assert main(["solve", "--config", cfg, "--problem.size", "3"]) == 2
    assert main(["solve", "--config", str(tmp_path / "missing.cfg")]) == 2
    assert main(["solve", "--config", cfg, "--coarse"]) == 2
    assert "error:" in capsys.readouterr().err
