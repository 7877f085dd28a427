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
import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .core import ConfigurationError, MaterialTable, ValidationError
from .types import REAL


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


# ---------------------------------------------------------------------------
# the device core behind ForceModel.core / jit_core
# ---------------------------------------------------------------------------

class DeviceCore:
    """A model core with the reference's scalar signature (forces.py:82-87):
    ``core(overlap, ts, sim_time, b2ax, b2ay, b2az, vx, vy, vz, wrx, wry, wrz,
    mass_eff, ra, rb, mat_a, mat_b, pair, wild, out)`` -- ``wild`` (float32
    row) updated in place, ``out[0:6]`` = force on A + torque-only force.

    Evaluated on the GPU (gf_eval_core, include/gf_b200.h): the built-in
    Hertz-Mindlin kernel or the model's NVRTC-compiled ``cuda_src``.  It is
    the same device code the step runs; there is no host implementation of
    the law.  ``batch()`` evaluates many contexts in one launch."""

    def __init__(self, model: "ForceModel"):
        self.model = model
        self._ctx = None

    def _context(self):
        if self._ctx is None:
            from . import _lib
            ctx = _lib.Context(_device())
            if self.model.cuda_src is not None:
                log = C.create_string_buffer(1 << 16)
                ctx.call("gf_set_force_model", self.model.cuda_src.encode(), _lib.CSRC_DIR.encode(),
                         C.c_int(len(self.model.wildcards)), log, C.c_size_t(1 << 16))
            self._ctx = ctx
        return self._ctx

    def batch(self, args, mats, pair, wild):
        """args (n, 15) float64, mats (n, 2) int, pair (rows, M, M), wild (n, W)
        float32 (updated in place); returns out (n, 6) float64."""
        from . import _lib
        args = _lib.carr(args, np.float64).reshape(-1, 15)
        n = args.shape[0]
        mats = _lib.carr(mats, np.int32).reshape(n, 2)
        pair = _lib.carr(pair, np.float64)
        W = len(self.model.wildcards)
        if wild.dtype != np.float32 or not wild.flags.c_contiguous:
            raise ValidationError("wildcard rows must be a C-contiguous float32 array")
        out = np.zeros((n, 6), dtype=np.float64)
        P = _lib.ptr
        self._context().call("gf_eval_core", C.c_int64(n), P(args), P(mats), C.c_int(pair.shape[1]),
                             C.c_int(pair.shape[0]), P(pair), P(wild), C.c_int(W), P(out))
        return out

    def __call__(self, overlap, ts, sim_time, b2ax, b2ay, b2az, vx, vy, vz, wrx, wry, wrz, mass_eff, ra, rb,
                 mat_a, mat_b, pair, wild, out):
        args = np.array([[overlap, ts, sim_time, b2ax, b2ay, b2az, vx, vy, vz, wrx, wry, wrz, mass_eff,
                          ra, rb]], dtype=np.float64)
        row = np.ascontiguousarray(np.asarray(wild, dtype=np.float32).reshape(1, -1))
        res = self.batch(args, [[int(mat_a), int(mat_b)]], pair, row)
        wild[:] = row[0]
        out[:6] = res[0]


def _device() -> int:
    import os
    return int(os.environ.get("GF_PLUGIN_DEVICE", "0"))


@dataclass
class ContactContext:
    """The per-contact variable bundle handed to a force model (forces.py:
    298-336).  force / torque_only_force start at zero."""

    contact_pnt: np.ndarray
    b2a: np.ndarray
    overlap_depth: float
    ts: float
    time: float
    a_owner_pos: np.ndarray
    b_owner_pos: np.ndarray
    a_ori_q: np.ndarray
    b_ori_q: np.ndarray
    a_owner_mass: float
    b_owner_mass: float
    a_radius: float
    b_radius: float
    a_mat: int
    b_mat: int
    a_lin_vel: np.ndarray
    b_lin_vel: np.ndarray
    a_rot_vel: np.ndarray            # owner-local frames
    b_rot_vel: np.ndarray
    a_owner: int = 0
    b_owner: int = 0
    a_geo: int = 0
    b_geo: int = 0
    a_family: int = 0
    b_family: int = 0
    a_owner_moi: np.ndarray = field(default_factory=lambda: np.ones(3))
    b_owner_moi: np.ndarray = field(default_factory=lambda: np.ones(3))
    loc_cpa: Optional[np.ndarray] = None
    loc_cpb: Optional[np.ndarray] = None
    body_a_pos: Optional[np.ndarray] = None
    body_b_pos: Optional[np.ndarray] = None
    wildcards: dict = field(default_factory=dict)
    force: np.ndarray = field(default_factory=lambda: np.zeros(3))
    torque_only_force: np.ndarray = field(default_factory=lambda: np.zeros(3))


@dataclass
class ContactResult:
    """Force on A in the global frame; the solver applies the reaction to B
    (forces.py:339-345)."""

    force: np.ndarray
    torque_only_force: np.ndarray
    wildcards: dict


def _quat_rot(q, v):
    """v rotated by the unit quaternion q = (w, x, y, z), the term order of
    the reference (forces.py:348-357)."""
    w, x, y, z = (float(c) for c in q)
    tx = y * v[2] - z * v[1] + w * v[0]
    ty = z * v[0] - x * v[2] + w * v[1]
    tz = x * v[1] - y * v[0] + w * v[2]
    return (v[0] + 2.0 * (y * tz - z * ty), v[1] + 2.0 * (z * tx - x * tz), v[2] + 2.0 * (x * ty - y * tx))


@dataclass(frozen=True)
class ForceModel:
    """A contact force model (forces.py:360-405), positional fields in the
    reference's order: ``ForceModel(name, core, jit_core, wildcards,
    pair_props)``.

    ``wildcards`` are the ordered per-contact history names; ``pair_props``
    the material properties stacked after E_cnt / G_cnt.

    ``cuda_src`` is the device implementation of a user model: CUDA source
    defining ``__device__ void user_core(...)`` with the reference core's
    argument list (forces.py:82-87; see include/gf_b200.h,
    gf_set_force_model), compiled for sm_100a with NVRTC when a Simulator
    using the model initialises -- the paper's JIT-compiled force models.
    ``gf::hm_default_core`` (same arguments) is available to build on the
    default law.  Without ``cuda_src`` the model is the built-in compiled
    Hertz-Mindlin kernel.

    ``core`` / ``jit_core`` default to the model's DeviceCore (the same
    device code, callable with the reference's scalar signature).  A plain
    Python core with no ``cuda_src`` is accepted by ``evaluate`` (the
    reference's host-side plugin path) but a Simulator refuses it: the step
    runs only on the device.

    ``flip_on_swap`` lists the wildcards that change sign when a contact's A
    and B sides swap (tangential displacement for Hertz-Mindlin).
    """

    name: str
    core: Optional[Callable] = None
    jit_core: Optional[Callable] = None
    wildcards: tuple = ()
    pair_props: tuple = ()
    cuda_src: Optional[str] = None
    flip_on_swap: tuple = ()
    device_kernel: Optional[str] = None

    def __post_init__(self):
        object.__setattr__(self, "wildcards", tuple(self.wildcards))
        object.__setattr__(self, "pair_props", tuple(self.pair_props))
        if self.device_kernel is None:
            object.__setattr__(self, "device_kernel", "nvrtc" if self.cuda_src is not None else
                               ("hertz_mindlin" if self.core is None else "python"))
        if self.on_device:
            dc = DeviceCore(self)
            if self.core is None:
                object.__setattr__(self, "core", dc)
            if self.jit_core is None:
                object.__setattr__(self, "jit_core", dc)

    @property
    def on_device(self) -> bool:
        """True when the step can run this model on the GPU."""
        return self.cuda_src is not None or self.device_kernel == "hertz_mindlin"

    def evaluate(self, ctx: ContactContext, pair_stack: np.ndarray) -> ContactResult:
        """The reference's generic plugin path (forces.py:375-405): pair
        kinematics from the context, then the core."""
        wa = _quat_rot(ctx.a_ori_q, np.asarray(ctx.a_rot_vel, dtype=np.float64))
        wb = _quat_rot(ctx.b_ori_q, np.asarray(ctx.b_rot_vel, dtype=np.float64))
        cp = [float(x) for x in ctx.contact_pnt]
        pa = [float(x) for x in ctx.a_owner_pos]
        pb = [float(x) for x in ctx.b_owner_pos]
        va = [float(x) for x in ctx.a_lin_vel]
        vb = [float(x) for x in ctx.b_lin_vel]
        ra_ = [cp[0] - pa[0], cp[1] - pa[1], cp[2] - pa[2]]
        rb_ = [cp[0] - pb[0], cp[1] - pb[1], cp[2] - pb[2]]
        rotax = wa[1] * ra_[2] - wa[2] * ra_[1]
        rotay = wa[2] * ra_[0] - wa[0] * ra_[2]
        rotaz = wa[0] * ra_[1] - wa[1] * ra_[0]
        rotbx = wb[1] * rb_[2] - wb[2] * rb_[1]
        rotby = wb[2] * rb_[0] - wb[0] * rb_[2]
        rotbz = wb[0] * rb_[1] - wb[1] * rb_[0]
        vx = (va[0] + rotax) - (vb[0] + rotbx)
        vy = (va[1] + rotay) - (vb[1] + rotby)
        vz = (va[2] + rotaz) - (vb[2] + rotbz)
        ma, mb = float(ctx.a_owner_mass), float(ctx.b_owner_mass)
        mass_eff = (ma * mb) / (ma + mb)
        wild = np.zeros(len(self.wildcards), dtype=REAL)
        for i, name in enumerate(self.wildcards):
            wild[i] = ctx.wildcards.get(name, 0.0)
        out = np.zeros(6, dtype=np.float64)
        self.core(float(ctx.overlap_depth), float(ctx.ts), float(ctx.time),
                  float(ctx.b2a[0]), float(ctx.b2a[1]), float(ctx.b2a[2]),
                  vx, vy, vz, rotbx - rotax, rotby - rotay, rotbz - rotaz,
                  mass_eff, float(ctx.a_radius), float(ctx.b_radius),
                  int(ctx.a_mat), int(ctx.b_mat), pair_stack, wild, out)
        return ContactResult(force=out[:3].copy(), torque_only_force=out[3:].copy(),
                             wildcards={name: float(wild[i]) for i, name in enumerate(self.wildcards)})


_REGISTRY: dict = {}


def register_force_model(model: ForceModel) -> ForceModel:
    if model.name in _REGISTRY:
        raise ConfigurationError(f"force model {model.name!r} already registered")
    if model.cuda_src is None and model.device_kernel not in ("hertz_mindlin", "python"):
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
    "hertz_mindlin", None, None,
    ("delta_tan_x", "delta_tan_y", "delta_tan_z", "delta_time"),
    ("CoR", "mu", "Crr"),
    flip_on_swap=(0, 1, 2),
))


def _registered_models():
    """BREAKAGE_MODEL and the other shipped NVRTC models (models.py)."""
    from . import models
    return models.breakage_model()


def evaluate_default_model(ctx: ContactContext, materials: MaterialTable) -> ContactResult:
    """forces.py:468-469: the built-in model on one context."""
    return DEFAULT_MODEL.evaluate(ctx, material_pair_stack(materials, DEFAULT_MODEL))


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


# ---------------------------------------------------------------------------
# the reference's per-kernel dT entry points, on the device
# ---------------------------------------------------------------------------

_PLUGIN_CTX = {}


def _plugin_context(model: Optional[ForceModel] = None):
    """A scene-less device context for the per-kernel entry points (one per
    NVRTC model; the built-in model shares one)."""
    from . import _lib
    key = model.name if (model is not None and model.cuda_src is not None) else None
    ctx = _PLUGIN_CTX.get(key)
    if ctx is None:
        ctx = _lib.Context(_device())
        if key is not None:
            log = C.create_string_buffer(1 << 16)
            ctx.call("gf_set_force_model", model.cuda_src.encode(), _lib.CSRC_DIR.encode(),
                     C.c_int(len(model.wildcards)), log, C.c_size_t(1 << 16))
        _PLUGIN_CTX[key] = ctx
    return ctx


def contact_forces(kind, slot_a, slot_b, owner_a, owner_b, mat_a, mat_b, sph_centers, sph_radii, tri_world,
                   ana_world, ana_kind, owner_pos, lin_vel, ang_vel_global, mass, pair_stack, wild, ts,
                   sim_time, out_ft, depth, cp, model: Optional[ForceModel] = None) -> int:
    """make_contact_kernel's sweep (forces.py:547-593) on the GPU
    (gf_contact_forces): the contact geometry, pair kinematics and the model
    core per ACS entry.  ``wild`` (n, W) float32, ``out_ft`` (n, 6), ``depth``
    (n,) and ``cp`` (n, 3) float64 are written in place; returns the
    touching count (2 per sphere-sphere, 1 per wall contact)."""
    from . import _lib
    model = model or DEFAULT_MODEL
    P, carr = _lib.ptr, _lib.carr
    n = int(np.asarray(kind).shape[0])
    for name, arr, dt in (("wild", wild, np.float32), ("out_ft", out_ft, np.float64),
                          ("depth", depth, np.float64), ("cp", cp, np.float64)):
        if arr.dtype != dt or not arr.flags.c_contiguous:
            raise ValidationError(f"{name} must be a C-contiguous {np.dtype(dt).name} array")
    sc = carr(sph_centers, np.float64).reshape(-1, 3)
    tw = carr(tri_world, np.float64).reshape(-1, 9)
    aw = carr(ana_world, np.float64).reshape(-1, 8)
    op = carr(owner_pos, np.float64).reshape(-1, 3)
    pair = carr(pair_stack, np.float64)
    touching = C.c_int64(0)
    _plugin_context(model).call(
        "gf_contact_forces", C.c_int64(n), P(carr(kind, np.uint8)), P(carr(slot_a, np.int64)),
        P(carr(slot_b, np.int64)), P(carr(owner_a, np.int64)), P(carr(owner_b, np.int64)),
        P(carr(mat_a, np.uint8)), P(carr(mat_b, np.uint8)), C.c_int64(sc.shape[0]), P(sc),
        P(carr(sph_radii, np.float32)), C.c_int64(tw.shape[0]), P(tw), C.c_int64(aw.shape[0]), P(aw),
        P(carr(ana_kind, np.uint8)), C.c_int64(op.shape[0]), P(op), P(carr(lin_vel, np.float64)),
        P(carr(ang_vel_global, np.float64)), P(carr(mass, np.float64)), C.c_int(pair.shape[1]),
        C.c_int(pair.shape[0]), P(pair), P(wild), C.c_int(len(model.wildcards)), C.c_double(ts),
        C.c_double(sim_time), P(out_ft), P(depth), P(cp), C.byref(touching))
    return int(touching.value)


def reduce_to_owners(owner_a, owner_b, forces, tofs, contact_points, owner_pos, mass, gravity):
    """Per-owner totals (forces.py:600-614) on the GPU (gf_reduce): force =
    m g + sum F, torque = sum (r x (F + tof)), the reaction on B at its own
    lever arm, each owner summed in the reference loop's order."""
    from . import _lib
    P, carr = _lib.ptr, _lib.carr
    op = carr(owner_pos, np.float64).reshape(-1, 3)
    n_o = op.shape[0]
    oa = carr(owner_a, np.int64).reshape(-1)
    acc_f = np.zeros((n_o, 3), dtype=np.float64)
    acc_t = np.zeros((n_o, 3), dtype=np.float64)
    _plugin_context().call(
        "gf_reduce", C.c_int64(oa.shape[0]), P(oa), P(carr(owner_b, np.int64).reshape(-1)),
        P(carr(forces, np.float64).reshape(-1, 3)), P(carr(tofs, np.float64).reshape(-1, 3)),
        P(carr(contact_points, np.float64).reshape(-1, 3)), C.c_int64(n_o), P(op),
        P(carr(mass, np.float64).reshape(-1)), P(carr(gravity, np.float64).reshape(3)), P(acc_f), P(acc_t))
    return acc_f, acc_t


BREAKAGE_MODEL = _registered_models()


def build_bonds(centers, radii, geom_ids, owner_ids, gamma_int: float):
    """Bond every sphere pair whose centre distance is below gamma_int (R_i +
    R_j) (forces.py:617-675): candidate pairs from the device detection
    (detect_contacts with margin (gamma_int - 1) 2 r_max), the exact distance
    cut, initialLength = the overlap at creation.  Returns (ContactArray with
    the breakage wildcards, stats)."""
    from . import broadphase as B
    if gamma_int <= 0.0:
        raise ValidationError(f"gamma_int must be positive, got {gamma_int}")
    centers = np.asarray(centers, dtype=np.float64).reshape(-1, 3)
    radii = np.asarray(radii, dtype=REAL).reshape(-1)
    m = centers.shape[0]
    r_max = float(radii.max()) if m else 0.0
    margin = max(0.0, (gamma_int - 1.0) * 2.0 * r_max) + 1e-12
    snap = B.DetectionSnapshot(
        sph_center=centers, sph_radius=radii, sph_geom=np.arange(m, dtype=np.int64),
        sph_owner=np.asarray(owner_ids, dtype=np.int64), sph_family=np.zeros(m, np.uint8),
        tri_world=np.zeros((0, 9)), tri_geom=np.zeros(0, np.int64), tri_owner=np.zeros(0, np.int64),
        tri_family=np.zeros(0, np.uint8), ana_world=np.zeros((0, 8)), ana_kind=np.zeros(0, np.uint8),
        ana_geom=np.zeros(0, np.int64), ana_owner=np.zeros(0, np.int64), ana_family=np.zeros(0, np.uint8),
        mask=np.ones((256, 256), dtype=bool))
    cand = B.detect_contacts(snap, margin)
    a, b = cand.geom_a, cand.geom_b
    d = np.linalg.norm(centers[a] - centers[b], axis=1)
    rsum = radii[a].astype(np.float64) + radii[b].astype(np.float64)
    keep = d < gamma_int * rsum
    a, b = a[keep], b[keep]
    overlap = rsum[keep] - d[keep]
    gid = np.asarray(geom_ids, dtype=np.int64)
    bonds = B.ContactArray(np.full(a.shape[0], B.CONTACT_SS, dtype=np.uint8), gid[a], gid[b])
    for name in BREAKAGE_MODEL.wildcards:
        bonds.wildcards[name] = np.zeros(bonds.size, dtype=REAL)
    bonds.wildcards["unbroken"][:] = 1.0
    bonds.wildcards["initialLength"][:] = overlap.astype(REAL)
    bonds = bonds.canonicalize()
    degree = np.bincount(a, minlength=m) + np.bincount(b, minlength=m)
    assigned = np.bincount(a, minlength=m)
    stats = {"count": int(a.shape[0]), "mean_degree": float(degree.mean()) if m else 0.0,
             "modal_degree": int(np.bincount(degree).argmax()) if m else 0,
             "modal_assigned": int(np.bincount(assigned).argmax()) if m else 0}
    return bonds, stats
