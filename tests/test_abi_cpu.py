"""CPU-only checks of the product library: it builds for sm_100a, loads, and
exports every entry point include/gf_b200.h declares (no device calls)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2311_04648_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "gf_b200.h")).read()
    return sorted(set(re.findall(r"\b(gf_[a-z_]+)\s*\(", text)))


def test_header_declares_python_binding_exports():
    assert set(header_symbols()) == set(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = _lib.load_library()
    for name in header_symbols():
        assert hasattr(L, name), name


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_device_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("a device is present")
    import paper_2311_04648_b200 as gf
    sim = gf.Simulator(gf.Domain.cube(1.0))
    sim.load_material({"E": 1e7, "nu": 0.3, "CoR": 0.5, "mu": 0.3, "Crr": 0.0})
    with pytest.raises(gf.DeviceUnavailableError):
        sim.initialize()
