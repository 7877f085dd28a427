"""ctypes binding of libgf_b200.so (include/gf_b200.h).

The product path has no CPU fallback: importing works anywhere (so the
package can be inspected on a CPU-only host), but any call that needs the
device raises ``DeviceUnavailableError`` if the shared library or a CUDA
device is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# GF_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("GF_LIB") or os.path.join(PKG_DIR, "libgf_b200.so")
CSRC_DIR = os.path.join(PKG_DIR, "csrc")  # gf_device.cuh for NVRTC user models

GF_STATE_F32 = 1


class DeviceUnavailableError(RuntimeError):
    """libgf_b200.so or a CUDA device is missing; there is no CPU fallback."""


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_D = C.c_double


class StepParams(C.Structure):
    _fields_ = [("h", _D), ("g", _D * 3), ("v_err", _D), ("sim_time", _D), ("step", _I64),
                ("write_acc", _I32), ("pad", _I32)]


class RunParams(C.Structure):
    _fields_ = [("n_steps", _I64), ("step0", _I64), ("h", _D), ("g", _D * 3), ("v_err", _D),
                ("margin", _D), ("period", _I32), ("lag", _I32), ("n_dyn", _I32),
                ("write_acc", _I32), ("dyn_spec", _P), ("dyn_vals", _P)]


class RunResult(C.Structure):
    _fields_ = [("steps_done", _I64), ("bad_owner", _I64), ("bad_step", _I64),
                ("oob_owner", _I64), ("oob_step", _I64), ("touching", _I64), ("n_acs", _I64),
                ("ca_updates", _I64), ("sum_acs", _I64), ("sum_touch_pairs", _I64), ("dt_ms", _D),
                ("kt_ms", _D), ("wall_ms", _D), ("kt_rebuilds", _I64), ("dd_trip_step", _I64)]


# every symbol include/gf_b200.h declares
EXPORTS = (
    "gf_create", "gf_destroy", "gf_last_error", "gf_device_count", "gf_set_domain",
    "gf_upload_owners", "gf_download_owners", "gf_set_owner_families", "gf_set_external_loads",
    "gf_download_accumulators", "gf_upload_geometry", "gf_upload_materials",
    "gf_upload_families", "gf_download_world", "gf_set_acs", "gf_acs_size", "gf_get_acs",
    "gf_detect", "gf_detect_snapshot", "gf_bin_ranges", "gf_adopt", "gf_dt_step", "gf_run",
    "gf_merge_history", "gf_set_profiling", "gf_kernel_times", "gf_set_force_model",
    "gf_nvrtc_compile", "gf_run_begin", "gf_step_forces", "gf_step_integrate", "gf_run_end",
    "gf_set_decomposition", "gf_halo_record_bytes", "gf_stream", "gf_pack_state", "gf_unpack_state",
    "gf_pack_forces", "gf_add_forces", "gf_trip_word", "gf_sync",
    "gf_contact_forces", "gf_eval_core", "gf_reduce", "gf_integrate_and_refresh", "gf_apply_active_boxes",
    "gf_set_persistent_wildcard", "gf_read_owners", "gf_clump_max_absv", "gf_sphere_frame",
)

_lib = None


def build(verbose: bool = False) -> str:
    """Compile libgf_b200.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
    out = None if verbose else subprocess.DEVNULL
    subprocess.run(["make", "-j4", "-C", PKG_DIR], check=True, stdout=out)
    return LIB_PATH


def load_library():
    """Load the shared library (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceUnavailableError(
            f"{LIB_PATH} is missing; build it with `make -C {PKG_DIR}` (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.gf_create.restype = _P
    L.gf_create.argtypes = [C.c_int, C.c_int, C.c_uint32]
    L.gf_destroy.argtypes = [_P]
    L.gf_acs_size.restype = _I64
    L.gf_acs_size.argtypes = [_P, C.c_int]
    L.gf_stream.restype = _P
    L.gf_stream.argtypes = [_P]
    L.gf_step_forces.argtypes = [_P, _I64]
    L.gf_step_integrate.argtypes = [_P, _I64]
    L.gf_set_decomposition.argtypes = [_P, _P, _D, C.c_int, _D]
    L.gf_trip_word.argtypes = [_P, _P, C.c_int]
    for name in ("gf_pack_state", "gf_unpack_state", "gf_pack_forces", "gf_add_forces"):
        getattr(L, name).argtypes = [_P, _P, _I64, _P]
    for name in EXPORTS:
        fn = getattr(L, name)
        if name not in ("gf_create", "gf_destroy", "gf_acs_size", "gf_stream"):
            fn.restype = C.c_int
    _lib = L
    return L


def device_count() -> int:
    try:
        return int(load_library().gf_device_count())
    except (OSError, DeviceUnavailableError):
        return 0


def ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_P)


def carr(a, dtype, shape=None):
    a = np.ascontiguousarray(a, dtype=dtype)
    if shape is not None:
        a = a.reshape(shape)
    return a


class Context:
    """Owns one gf_ctx (device buffers, streams, events)."""

    def __init__(self, device: int = 0, f32_state: bool = False, kt_device=None):
        """kt_device: None = kT as a second stream on `device`; an index =
        the paper's 2-GPU split, kT on that device (include/gf_b200.h)."""
        L = load_library()
        if L.gf_device_count() <= 0:
            raise DeviceUnavailableError("no CUDA device visible; the B200 path has no CPU fallback")
        self.L = L
        kt = -1 if kt_device is None else int(kt_device)
        self.h = L.gf_create(int(device), kt, GF_STATE_F32 if f32_state else 0)
        if not self.h:
            raise DeviceUnavailableError(f"gf_create failed on device {device} (kT device {kt})")
        self.f32_state = f32_state
        self.kt_device = kt_device

    def close(self):
        if getattr(self, "h", None):
            self.L.gf_destroy(_P(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def error(self) -> str:
        buf = C.create_string_buffer(4096)
        self.L.gf_last_error(_P(self.h), buf, C.c_size_t(4096))
        return buf.value.decode(errors="replace")

    def call(self, name, *args):
        rc = getattr(self.L, name)(_P(self.h), *args)
        if rc != 0:
            raise RuntimeError(f"{name} failed: {self.error()}")
        return rc
