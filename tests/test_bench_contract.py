"""bench.py's reference arm on CPU (a small grid): the JSON line carries the
contract's keys, times FULL solves to rtol 1e-7, reports the CPU model, and
the process maps no library of the product (only liboracle.so)."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_line_and_independence():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--grid", "20", "--boxes", "2", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, check=True).stdout
    d = json.loads(out.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "s" and d["higher_is_better"] is False
    for k in ("metric", "value", "n_gpus", "steps", "warmup", "config", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["true_relative_residual"] <= 1e-7
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cpu_model"]
    assert d["loaded_native"] == ["liboracle.so"]


def test_gpus_flag_refuses_missing_devices():
    """--gpus N outside torchrun re-launches N ranks; with fewer visible
    devices it says so instead of timing one GPU."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 2 and "error" in d
