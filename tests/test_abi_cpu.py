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


def test_host_uploads_are_stream_ordered():
    """The context's streams are non-blocking: a legacy-stream cudaMemcpy /
    cudaMemset is not ordered with kernels launched on them afterwards (a
    fresh context once read its fixed-point scales before their upload
    landed).  Host -> device copies go through h2d(), memsets are async."""
    csrc = os.path.join(ROOT, "paper_2311_04648_b200", "csrc")
    bad = []
    for name in sorted(os.listdir(csrc)):
        if not name.endswith((".cu", ".cuh")):
            continue
        for no, line in enumerate(open(os.path.join(csrc, name)), 1):
            code = line.split("//")[0]
            if re.search(r"\bcudaMemset\s*\(", code) or (
                    re.search(r"\bcudaMemcpy\s*\(", code) and "DeviceToHost" not in code):
                bad.append(f"{name}:{no}: {line.strip()}")
    assert not bad, "\n".join(bad)
