"""Force-model plugin interface of the drop-in (mirrors grainforge/forces.py:
ForceModel + registry :360-440, material_pair_stack :443-460,
effective_contact_params :31-38, restitution_damping :41-44).

The contact-force arithmetic itself runs only on the device
(csrc/gf_dt_impl.cuh, hertz_mindlin); this module holds the host-side
parameter tables the kernel consumes.  A model is selected by name exactly as
in the reference (`Simulator(domain, force_model="hertz_mindlin")`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from .core import ConfigurationError, MaterialTable


def effective_contact_params(e_a: float, nu_a: float, e_b: float, nu_b: float):
    """Hertzian effective Young's and shear moduli (forces.py:31-38)."""
    e_cnt = 1.0 / ((1.0 - nu_a * nu_a) / e_a + (1.0 - nu_b * nu_b) / e_b)
    g_cnt = 1.0 / (2.0 * (2.0 - nu_a) * (1.0 + nu_a) / e_a + 2.0 * (2.0 - nu_b) * (1.0 + nu_b) / e_b)
    return e_cnt, g_cnt


def restitution_damping(cor: float) -> float:
    """beta = ln(CoR) / sqrt(ln^2(CoR) + pi^2), CoR clamped at 1e-12.

    Evaluated on the host with the same libm log the reference calls in its
    kernel (forces.py:122), then uploaded as a per-material-pair table; the
    device never evaluates a transcendental for it."""
    loge = math.log(1e-12) if cor < 1e-12 else math.log(cor)
    return loge / math.sqrt(loge * loge + math.pi * math.pi)


@dataclass(frozen=True)
class ForceModel:
    """A contact force model (forces.py:360-405).

    ``wildcards`` are the ordered per-contact history names; ``pair_props``
    the material properties stacked after E_cnt / G_cnt.

    ``cuda_src`` is the device implementation of a user model: CUDA source
    defining ``__device__ void user_core(...)`` with the reference core's
    argument list (forces.py:82-87; see include/gf_b200.h,
    gf_set_force_model).  It is compiled for sm_100a with NVRTC when a
    Simulator using the model initialises -- the paper's JIT-compiled force
    models.  ``gf::hm_default_core`` (same arguments) is available to build
    on the default law.  Without ``cuda_src`` the model is the built-in
    compiled Hertz-Mindlin kernel.

    ``flip_on_swap`` lists the wildcards that change sign when a contact's A
    and B sides swap (tangential displacement for Hertz-Mindlin).
    ``core`` / ``jit_core`` keep the reference's field names for source
    compatibility; the device path does not call them.
    """

    name: str
    wildcards: tuple
    pair_props: tuple
    device_kernel: str = "hertz_mindlin"
    core: Optional[Callable] = None
    jit_core: Optional[Callable] = None
    cuda_src: Optional[str] = None
    flip_on_swap: tuple = ()


_REGISTRY: dict = {}


def register_force_model(model: ForceModel) -> ForceModel:
    if model.name in _REGISTRY:
        raise ConfigurationError(f"force model {model.name!r} already registered")
    if model.cuda_src is None and model.device_kernel != "hertz_mindlin":
        raise ConfigurationError(
            f"force model {model.name!r}: no compiled device kernel {model.device_kernel!r}")
    _REGISTRY[model.name] = model
    return model


def get_force_model(name: str) -> ForceModel:
    try:
        return _REGISTRY[name]
    except KeyError:
        raise ConfigurationError(f"unknown force model {name!r}") from None


DEFAULT_MODEL = register_force_model(ForceModel(
    name="hertz_mindlin",
    wildcards=("delta_tan_x", "delta_tan_y", "delta_tan_z", "delta_time"),
    pair_props=("CoR", "mu", "Crr"),
    flip_on_swap=(0, 1, 2),
))


def compile_check(model: ForceModel) -> str:
    """NVRTC-compile a user model's source without a device; returns the
    compiler log, raises ConfigurationError on failure."""
    import ctypes as C
    from . import _lib
    if model.cuda_src is None:
        return ""
    L = _lib.load_library()
    log = C.create_string_buffer(1 << 16)
    rc = L.gf_nvrtc_compile(model.cuda_src.encode(), _lib.CSRC_DIR.encode(), log, C.c_size_t(1 << 16))
    text = log.value.decode(errors="replace")
    if rc != 0:
        raise ConfigurationError(f"force model {model.name!r} does not compile:\n{text}")
    return text


def material_pair_stack(materials: MaterialTable, model: ForceModel) -> np.ndarray:
    """(2 + n_props, M, M) float64: E_cnt, G_cnt, then the model's pair props."""
    n = len(materials)
    if n == 0:
        raise ConfigurationError("no materials loaded")
    e = materials.single_array("E")
    nu = materials.single_array("nu")
    stack = np.zeros((2 + len(model.pair_props), n, n), dtype=np.float64)
    for a in range(n):
        for b in range(n):
            stack[0, a, b], stack[1, a, b] = effective_contact_params(e[a], nu[a], e[b], nu[b])
    for i, prop in enumerate(model.pair_props):
        stack[2 + i] = materials.pair_matrix(prop)
    return stack


def beta_table(pair_stack: np.ndarray) -> np.ndarray:
    """Per-pair restitution damping from the CoR row of the stack."""
    cor = pair_stack[2]
    out = np.zeros_like(cor)
    for a in range(cor.shape[0]):
        for b in range(cor.shape[1]):
            out[a, b] = restitution_damping(float(cor[a, b]))
    return out
