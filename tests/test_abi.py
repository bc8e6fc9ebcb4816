"""The C-ABI libraries load on a CPU-only host and export every entry point
include/*.h declares (no compute calls without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2304_04876_b200" / "_lib"


def _declared(header: Path, prefix: str):
    text = header.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(rf"\b({prefix}\w+)\s*\(", text)))


def _exports(so: Path):
    lib = ctypes.CDLL(str(so))
    return lib


@pytest.mark.parametrize("header,so,prefix", [
    ("gdsw.h", "libgdsw.so", "gdsw_"),
    ("gdsw_host.h", "libgdsw_host.so", "gh_"),
])
def test_library_exports_every_declared_symbol(header, so, prefix):
    names = _declared(ROOT / "include" / header, prefix)
    assert len(names) > 5
    lib = _exports(LIB / so)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_abi():
    from paper_2304_04876_b200 import device
    declared = set(_declared(ROOT / "include" / "gdsw.h", "gdsw_"))
    assert declared == set(device.EXPORTED)
    assert device._lib.gdsw_abi_version() == 1


def test_sm100a_code_in_the_fatbin():
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", str(LIB / "libgdsw.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
