"""The drop-in Simulator: the reference's scene/solver API
(grainforge/engine.py:235-908) driving the B200 worker protocol.

Where the reference runs a kinematics thread and a dynamics thread that hand
off work orders and contact arrays through condition-variable slots
(engine.py:90-115, 669-906), this simulator owns one device context with two
CUDA streams (csrc/gf_context.cu, gf_run): kT detects on a snapshot while dT
keeps stepping, and the new contact array is adopted `lag` steps later with
its history remapped on the device.  The whole step loop of a do_dynamics call
is one native call; the host only evaluates prescribed-motion expressions up
front and reads back the watchdog and counters at the end.

Host mirrors: after initialize() the StateStore owner arrays, `_pos`,
`_sph_centers`, `_acs`, `_wild`, `_tri_world`, `_ana_world` are synced from
the device on access, and host edits (trackers, set_family, set_pos) are
pushed back before the next step -- the private attributes the reference's
tests and IO read stay valid.
"""

from __future__ import annotations

import ctypes as C
import math
import threading
import time as _time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import broadphase as B
from . import forces as F
from .core import (GEOM_CYLINDER, GEOM_PLANE, GEOM_SPHERE, GEOM_TRIANGLE, OWNER_CLUMP,
                   ClumpTemplate, ConfigurationError, Domain, MaterialTable, StateStore,
                   ValidationError, quat_rotate)
from .types import NUM_FAMILIES, REAL


class DivergenceError(RuntimeError):
    """The watchdog tripped: an owner exceeded the error-out velocity or left
    the domain (engine.py:42)."""


_SAFE_EVAL_NS = {"t": 0.0, "sin": math.sin, "cos": math.cos, "tan": math.tan, "sqrt": math.sqrt,
                 "exp": math.exp, "abs": abs, "pi": math.pi}


def _compile_expr(expr: str):
    """Constant or expression of t (engine.py:53-67)."""
    try:
        return float(expr), None
    except ValueError:
        pass
    try:
        code = compile(expr, "<prescription>", "eval")
        float(eval(code, {"__builtins__": {}}, dict(_SAFE_EVAL_NS)))
    except Exception as exc:
        raise ConfigurationError(f"malformed prescription expression {expr!r}: {exc}")
    return None, code


@dataclass
class SchedulerState:
    n_max: int = 2
    step_counter: int = 0
    last_wo_stamp: int = -1
    last_ca_stamp: int = -1
    dynamics_waits: int = 0
    kinematics_waits: int = 0
    ca_updates: int = 0
    timing: dict = field(default_factory=lambda: {
        "dyn_force": 0.0, "dyn_integrate": 0.0, "dyn_transfer": 0.0, "dyn_wait": 0.0,
        "kin_detect": 0.0, "kin_transfer": 0.0, "kin_wait": 0.0})
    step_time_ema: float = 0.0
    last_cd_seconds: float = 0.0


@dataclass
class ActiveBoxPolicy:
    half_extents: list
    anchors: list
    centers: list
    refresh_period: float
    frozen_family: int
    active_family: int


class Tracker:
    """Owner handle (engine.py:132-189); reads reflect the last completed step.

    While the host mirrors are stale (after a run), reads gather just this
    owner's record on the device (gf_read_owners) instead of syncing the
    whole state -- the rover co-simulation's per-wheel force readback
     costs one small copy, not an n-owner download."""

    def __init__(self, sim: "Simulator", owner: int):
        self._sim = sim
        self.owner = owner

    def _dev(self):
        """This owner's device record, or None when the host mirror is current."""
        sim = self._sim
        if sim._ctx is None or not sim._host_stale or sim.decomposition is not None:
            return None
        return sim._read_owner(self.owner)

    def pos(self) -> np.ndarray:
        r = self._dev()
        if r is not None:
            return r["pos"]
        return self._sim._pos[self.owner].copy()

    def vel(self) -> np.ndarray:
        r = self._dev()
        if r is not None:
            return r["lin_vel"]
        return self._sim.store.lin_vel[self.owner].astype(np.float64)

    def ang_vel_local(self) -> np.ndarray:
        r = self._dev()
        if r is not None:
            return r["ang_vel"]
        return self._sim.store.ang_vel[self.owner].astype(np.float64)

    def quat(self) -> np.ndarray:
        r = self._dev()
        if r is not None:
            return r["quat"]
        return self._sim.store.quat[self.owner].astype(np.float64)

    def moi(self) -> np.ndarray:
        return self._sim.store.moi[self.owner].astype(np.float64)

    def mass(self) -> float:
        return float(self._sim.store.mass[self.owner])

    def contact_force(self) -> np.ndarray:
        r = self._dev()
        if r is not None:
            return r["acc_force"]
        return self._sim.store.acc_force[self.owner].copy()

    def contact_torque(self) -> np.ndarray:
        r = self._dev()
        if r is not None:
            return r["acc_torque"]
        return self._sim.store.acc_torque[self.owner].copy()

    def contact_acc(self) -> np.ndarray:
        return self.contact_force() / self.mass()

    def contact_ang_acc_local(self) -> np.ndarray:
        q = self.quat()
        tl = quat_rotate(np.array([q[0], -q[1], -q[2], -q[3]]), self.contact_torque())
        return tl / self.moi()

    def set_pos(self, xyz) -> None:
        self._sim._set_owner_position(self.owner, xyz)

    def set_vel(self, v) -> None:
        self._sim.store.lin_vel[self.owner] = np.asarray(v, dtype=np.float64)

    def set_ang_vel_local(self, w) -> None:
        self._sim.store.ang_vel[self.owner] = np.asarray(w, dtype=np.float64)

    def set_external_force(self, f) -> None:
        self._sim.store.ext_force[self.owner] = np.asarray(f, dtype=np.float64)

    def set_external_torque(self, t) -> None:
        self._sim.store.ext_torque[self.owner] = np.asarray(t, dtype=np.float64)

    def set_family(self, family: int) -> None:
        self._sim.store.set_family(self.owner, family)


class Inspector:
    def __init__(self, sim: "Simulator", quantity: str):
        if quantity not in ("clump_max_absv", "avg_sph_contacts"):
            raise ConfigurationError(f"unknown inspector quantity {quantity!r}")
        self._sim = sim
        self.quantity = quantity

    def get_value(self) -> float:
        sim = self._sim
        if self.quantity == "clump_max_absv":
            if sim._ctx is not None and sim._host_stale and sim.decomposition is None:
                out = C.c_double(0.0)   # a device reduction, no state download
                sim._ctx.call("gf_clump_max_absv", C.byref(out))
                return float(out.value)
            s = sim.store
            n = s.n_owners
            if n == 0:
                return 0.0
            fixed = np.array([p.fixed for p in s.families.prescriptions], bool)[s.owner_family[:n]]
            sel = (s.owner_kind[:n] == OWNER_CLUMP) & ~fixed
            if not sel.any():
                return 0.0
            v = s.lin_vel[:n][sel].astype(np.float64)
            return float(np.sqrt((v * v).sum(axis=1)).max())
        n_sph = sim._sph_geom.shape[0]
        return 0.0 if n_sph == 0 else sim._last_touching / n_sph


_MIRROR_FIELDS = ("voxel", "subvoxel", "quat", "lin_vel", "ang_vel", "owner_family",
                  "acc_force", "acc_torque", "ext_force", "ext_torque")


class Simulator:
    """A discrete element simulation on one B200: build the scene,
    initialize(), then advance with do_dynamics()."""

    default_sync = False

    def __init__(self, domain: Domain, force_model: str = "hertz_mindlin", *,
                 device: int = 0, precision: str = "f64", reorder=None, decomposition=None,
                 kt_device=None):
        if precision not in ("f64", "f32"):
            raise ValidationError(f"precision must be 'f64' or 'f32', got {precision!r}")
        self.materials = MaterialTable()
        self.store = StateStore(domain, self.materials)
        self.model = F.get_force_model(force_model)
        self.gravity = np.zeros(3, dtype=np.float64)
        self.h = 1e-5
        self.v_err = 50.0
        self.scheduler = SchedulerState()
        self.margin_policy = B.MarginPolicy(v_max=self.v_err, h=self.h, n_max=2)
        self.sync_mode = bool(Simulator.default_sync)
        self.sim_time = 0.0
        self.active_box_policy = None
        self.device = int(device)
        # the paper's 2-GPU split: contact detection (kT) on
        # kt_device, forces and integration (dT) on `device`; None = both on
        # `device` as concurrent streams
        self.kt_device = None if kt_device is None else int(kt_device)
        if self.kt_device is not None and decomposition is not None:
            raise ConfigurationError("the 2-GPU kT/dT split and the slab decomposition are separate modes")
        self.precision = precision
        # device memory order: Morton order of the initial positions so contact
        # gathers hit nearby owners; the fp64 parity build keeps the reference's
        # order (its per-owner summation order is then the reference's too)
        self.reorder = (precision == "f32") if reorder is None else bool(reorder)
        self._initialized = False
        self._closed = False
        self._sph_geom = np.zeros(0, dtype=np.int64)
        self._last_touching = 0
        self._acs0 = B.ContactArray()
        self._lv_mask = np.zeros((NUM_FAMILIES, 3), dtype=np.bool_)
        self._lv_val = np.zeros((NUM_FAMILIES, 3), dtype=np.float64)
        self._av_mask = np.zeros((NUM_FAMILIES, 3), dtype=np.bool_)
        self._av_val = np.zeros((NUM_FAMILIES, 3), dtype=np.float64)
        self._fixed_flag = np.zeros(NUM_FAMILIES, dtype=np.bool_)
        self._prescribed_flag = np.zeros(NUM_FAMILIES, dtype=np.bool_)
        self._dynamic_prescriptions: list = []
        self._n_max_floor = 2
        self._calm_cycles = 0
        self._fixed_n_max = None
        self._margin_cap_steps = None
        self._ctx = None
        self._host_stale = False   # device newer than the host mirror
        self._host_dirty = False   # host mirror may hold edits for the device
        self._tables_dirty = False
        self._lock = threading.RLock()
        self._kin_delay = None     # accepted for API compatibility (engine.py:285-287)
        self._dyn_delay = None
        self.last_run = None
        # spatial slab decomposition across ranks (decomp.SlabDecomposition);
        # None = the whole scene on this device
        self.decomposition = decomposition
        if decomposition is not None and precision != "f32":
            raise ConfigurationError("a decomposed simulator needs precision='f32' (fixed-point reduction)")

    # -- scene construction ---------------------------------------------------
    def load_material(self, props: dict) -> int:
        return self.materials.load_material(props)

    def set_material_pair(self, name: str, a: int, b: int, value: float) -> None:
        self.materials.set_pair(name, a, b, value)

    def load_clump_template(self, template: ClumpTemplate) -> int:
        return self.store.register_template(template)

    def add_clumps(self, template_id: int, positions) -> list:
        self._require_setup("add_clumps")
        return self.store.add_clumps(template_id, positions)

    def add_mesh(self, triangles, material: int, family: int = 0, mass=None, moi=None,
                 position=(0, 0, 0)) -> int:
        self._require_setup("add_mesh")
        kw = {} if mass is None else {"mass": mass}
        return self.store.add_mesh(triangles, material, family=family, moi=moi, position=position, **kw)

    def add_analytic(self, components, family: int = 0, position=(0, 0, 0)) -> int:
        self._require_setup("add_analytic")
        return self.store.add_analytic(components, family=family, position=position)

    def add_box_boundaries(self, material: int, family: int = 0) -> int:
        self._require_setup("add_box_boundaries")
        o = self.store.add_box_boundaries(material, family=family)
        self.set_family_fixed(family)
        return o

    def _require_setup(self, what):
        if self._initialized:
            raise ConfigurationError(f"{what} after initialize() is not supported")

    def track(self, owner: int) -> Tracker:
        if not (0 <= owner < self.store.n_owners):
            raise ValidationError(f"unknown owner id {owner}")
        return Tracker(self, owner)

    def create_inspector(self, quantity: str) -> Inspector:
        return Inspector(self, quantity)

    # -- families ---------------------------------------------------------------
    def set_family_prescribed_lin_vel(self, family: int, vx, vy, vz) -> None:
        self.store.families.set_lin_vel(family, vx, vy, vz)
        self._compile_family(family)

    def set_family_prescribed_ang_vel(self, family: int, wx, wy, wz) -> None:
        self.store.families.set_ang_vel(family, wx, wy, wz)
        self._compile_family(family)

    def set_family_fixed(self, family: int) -> None:
        self.store.families.set_fixed(family)
        self._fixed_flag[family] = True
        self._tables_dirty = True

    def set_family_mask(self, a: int, b: int, allow: bool) -> None:
        self.store.families.set_mask(a, b, allow)
        self._tables_dirty = True

    def _compile_family(self, family: int) -> None:
        p = self.store.families.prescriptions[family]
        self._prescribed_flag[family] = True
        self._dynamic_prescriptions = [e for e in self._dynamic_prescriptions if e[0] != family]
        for table, exprs, mask, val in ((0, p.lin_vel, self._lv_mask, self._lv_val),
                                        (1, p.ang_vel, self._av_mask, self._av_val)):
            if exprs is None:
                continue
            for ax, comp in enumerate(exprs):
                if comp is None or str(comp).lower() == "none":
                    mask[family, ax] = False
                    continue
                const, code = _compile_expr(str(comp))
                mask[family, ax] = True
                if code is None:
                    val[family, ax] = const
                else:
                    self._dynamic_prescriptions.append((family, table, ax, code))
        self._tables_dirty = True

    # -- configuration ----------------------------------------------------------
    def set_gravity(self, g) -> None:
        self.gravity = np.asarray(g, dtype=np.float64)

    def set_init_time_step(self, h: float) -> None:
        if h <= 0.0:
            raise ValidationError(f"time step must be positive, got {h}")
        self.h = float(h)

    def set_error_out_velocity(self, v: float) -> None:
        if v <= 0.0:
            raise ValidationError(f"error-out velocity must be positive, got {v}")
        self.v_err = float(v)

    def set_sync_mode(self, sync: bool) -> None:
        self.sync_mode = bool(sync)

    def set_fixed_lookahead(self, n_max: int) -> None:
        n_max = int(n_max)
        if n_max < 1:
            raise ValidationError(f"n_max must be >= 1, got {n_max}")
        if n_max == 1:
            self.sync_mode = True
        else:
            self.sync_mode = False
            self.scheduler.n_max = n_max
            self.margin_policy.n_max = n_max
        self._fixed_n_max = n_max

    def set_added_margin(self, added: float) -> None:
        self.margin_policy.added = float(added)

    def set_active_box_policy(self, policy: ActiveBoxPolicy) -> None:
        self.active_box_policy = policy
        self.set_family_fixed(policy.frozen_family)
        for fam in range(NUM_FAMILIES):
            self.set_family_mask(policy.frozen_family, fam, False)

    def init_bonds(self, gamma_int: float):
        """Install bonds between nearby sphere pairs (engine.py:409-427); call
        after the scene is built and before initialize().  Requires the
        breakage force model (models.BREAKAGE_SRC, NVRTC).  Bond candidates
        come from the device detection (forces.build_bonds)."""
        if self.model.name != "breakage":
            raise ConfigurationError("init_bonds requires the breakage force model")
        if self._initialized:
            raise ConfigurationError("init_bonds must run before initialize()")
        from .core import quat_rotate_many
        s = self.store
        geom_ids = np.nonzero(s.geom_kind[:s.n_geoms] == GEOM_SPHERE)[0].astype(np.int64)
        owners = s.geom_owner[geom_ids]
        pos = s.positions()
        offsets = s.geom_params[geom_ids, :3].astype(np.float64)
        centers = pos[owners] + quat_rotate_many(s.quat[owners], offsets)
        radii = s.geom_params[geom_ids, 3].astype(REAL)
        bonds, stats = F.build_bonds(centers, radii, geom_ids, owners, gamma_int)
        r_max = float(radii.max()) if radii.size else 0.0
        self.set_added_margin(max(0.0, (gamma_int - 1.0) * 2.0 * r_max) + 0.05 * r_max)
        self._acs = bonds
        return stats

    # -- lifecycle ----------------------------------------------------------------
    def initialize(self) -> None:
        if self._initialized:
            raise ConfigurationError("already initialized")
        if len(self.materials) == 0:
            raise ConfigurationError("no materials loaded")
        if self.decomposition is not None:
            from . import decomp
            decomp.prepare(self)   # self.store becomes this rank's piece of the scene
        s = self.store
        self.pair_stack = F.material_pair_stack(self.materials, self.model)
        self._beta = F.beta_table(self.pair_stack)
        self.margin_policy = B.MarginPolicy(v_max=self.v_err, h=self.h, n_max=self.scheduler.n_max,
                                            added=self.margin_policy.added)
        n_g = s.n_geoms
        kinds = s.geom_kind[:n_g]
        self._sph_geom = np.nonzero(kinds == GEOM_SPHERE)[0].astype(np.int64)
        self._tri_geom = np.nonzero(kinds == GEOM_TRIANGLE)[0].astype(np.int64)
        self._ana_geom = np.nonzero((kinds == GEOM_PLANE) | (kinds == GEOM_CYLINDER))[0].astype(np.int64)
        self._geom_slot = np.zeros(n_g, dtype=np.int64)
        for arr in (self._sph_geom, self._tri_geom, self._ana_geom):
            self._geom_slot[arr] = np.arange(arr.shape[0])
        self._sph_radius = s.geom_params[self._sph_geom, 3].astype(REAL)
        self._sph_owner = s.geom_owner[self._sph_geom]
        self._ana_kind_arr = s.geom_kind[self._ana_geom]
        if self._sph_geom.size:
            r_min = float(self._sph_radius.min())
            self._margin_cap_steps = max(4, int(r_min / (4.0 * self.v_err * self.h)))
        else:
            self._margin_cap_steps = None
        n = s.n_owners
        self._build_permutation()
        # mass-property templates: unique (mass, moi) rows
        self._tpl_rows, self._tpl_id = self._mass_templates()

        self._ctx = _lib.Context(self.device, f32_state=(self.precision == "f32"), kt_device=self.kt_device)
        ctx, P = self._ctx, _lib.ptr
        dom = s.domain
        ctx.call("gf_set_domain", P(_lib.carr(dom.lo, np.float64)), P(_lib.carr(dom.hi, np.float64)),
                 C.c_double(dom.voxel_edge))
        if self.model.cuda_src is not None:  # NVRTC user model (the paper's JIT)
            log = C.create_string_buffer(1 << 16)
            ctx.call("gf_set_force_model", self.model.cuda_src.encode(), _lib.CSRC_DIR.encode(),
                     C.c_int(len(self.model.wildcards)), log, C.c_size_t(1 << 16))
            if "unbroken" in self.model.wildcards:   # bonds persist (engine.py:639-662)
                ctx.call("gf_set_persistent_wildcard", C.c_int(self.model.wildcards.index("unbroken")))
        self._upload_tables()
        self._upload_owners()
        gp = s.geom_params[:n_g]
        sph_dev = self._sph_geom[self._sph_d2u]  # user geometry id of each device sphere slot
        sph_params = _lib.carr(gp[sph_dev, :4], np.float32)
        tri_local = _lib.carr(gp[self._tri_geom, :9], np.float32)
        ana_local = _lib.carr(gp[self._ana_geom, :8], np.float32)
        gm = s.geom_material[:n_g]
        go = s.geom_owner[:n_g]
        u2d = self._own_u2d
        keep = [_lib.carr(u2d[go[sph_dev]], np.int64), sph_params, _lib.carr(gm[sph_dev], np.uint8),
                _lib.carr(u2d[go[self._tri_geom]], np.int64), tri_local, _lib.carr(gm[self._tri_geom], np.uint8),
                _lib.carr(u2d[go[self._ana_geom]], np.int64), _lib.carr(self._ana_kind_arr, np.uint8),
                ana_local, _lib.carr(gm[self._ana_geom], np.uint8)]
        ctx.call("gf_upload_geometry", C.c_int64(self._sph_geom.size), P(keep[0]), P(keep[1]), P(keep[2]),
                 C.c_int64(self._tri_geom.size), P(keep[3]), P(keep[4]), P(keep[5]),
                 C.c_int64(self._ana_geom.size), P(keep[6]), P(keep[7]), P(keep[8]), P(keep[9]))
        self._install_acs(self._acs0.canonicalize())
        s._sync_hook = self._sync_field
        if self.decomposition is not None:
            decomp.attach(self)
        self._initialized = True

    def close(self) -> None:
        if self._closed:
            return
        self._closed = True
        if self._ctx is not None:
            try:
                self._sync_all()
            except Exception:
                pass
            self.store._sync_hook = None
            self._ctx.close()
            self._ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    # -- host <-> device ----------------------------------------------------------
    def _mass_templates(self):
        """Unique (mass, moi) rows and each owner's row (what the device's
        template table holds).  Clump owners normally carry their clump
        template's mass properties: those are matched in one vectorised pass,
        and only the rest (boundary owners, edited masses) go through a row
        sort -- np.unique over every owner's row costs minutes at 1e8
        owners."""
        s = self.store
        n = s.n_owners
        if n == 0:
            return np.zeros((0, 4)), np.zeros(0, np.uint32)
        mass, moi = s.mass[:n], s.moi[:n]
        tpl = np.asarray(s.owner_template[:n], dtype=np.int64)
        nt = len(s.templates)
        ref = np.full((nt + 1, 4), np.nan)
        for t, ct in enumerate(s.templates):
            ref[t, 0] = ct.mass
            ref[t, 1:] = np.asarray(ct.moi, dtype=np.float64)
        k = np.where(tpl >= 0, tpl, nt)
        ok = (mass == ref[k, 0]) & np.all(moi == ref[k, 1:], axis=1)
        rest = np.nonzero(~ok)[0]
        rest_rows = np.concatenate([mass[rest, None], moi[rest]], axis=1)
        cand = np.concatenate([ref[:nt], rest_rows], axis=0)
        rows, inv = np.unique(cand, axis=0, return_inverse=True)
        inv = np.asarray(inv).reshape(-1)
        tid = np.empty(n, np.int64)
        tid[ok] = inv[k[ok]]
        tid[rest] = inv[nt + np.arange(rest.size)]
        return np.ascontiguousarray(rows, dtype=np.float64), np.ascontiguousarray(tid, dtype=np.uint32)

    def _build_permutation(self):
        s = self.store
        n = s.n_owners
        if self.reorder and n > 1:
            from .decomp import morton_order
            d2u = morton_order(s.positions())
        else:
            d2u = np.arange(n, dtype=np.int64)
        identity = not (self.reorder and n > 1)
        u2d = d2u if identity else np.empty(n, np.int64)
        if not identity:
            u2d[d2u] = np.arange(n, dtype=np.int64)
        self._own_d2u, self._own_u2d = d2u, u2d
        self._own_identity = identity
        # device sphere slots: grouped by device owner, geometry order within
        sph_owner_dev = u2d[s.geom_owner[self._sph_geom]] if self._sph_geom.size else np.zeros(0, np.int64)
        if sph_owner_dev.size == 0 or np.all(sph_owner_dev[1:] >= sph_owner_dev[:-1]):
            sd2u = np.arange(sph_owner_dev.size, dtype=np.int64)   # already grouped (no sort)
            su2d = sd2u
        else:
            sd2u = np.argsort(sph_owner_dev, kind="stable").astype(np.int64)
            su2d = np.empty(sd2u.size, np.int64)
            su2d[sd2u] = np.arange(sd2u.size, dtype=np.int64)
        self._sph_d2u, self._sph_u2d = sd2u, su2d

    def _upload_tables(self):
        ctx, P = self._ctx, _lib.ptr
        fam = self.store.families
        flags = (self._fixed_flag.astype(np.uint8) | (self._prescribed_flag.astype(np.uint8) << 1))
        bits = np.array([1, 2, 4], np.uint8)
        lvm = (self._lv_mask.astype(np.uint8) * bits).sum(axis=1).astype(np.uint8)
        avm = (self._av_mask.astype(np.uint8) * bits).sum(axis=1).astype(np.uint8)
        keep = [_lib.carr(fam.mask, np.uint8).reshape(-1), _lib.carr(flags, np.uint8), lvm, avm,
                _lib.carr(self._lv_val, np.float64), _lib.carr(self._av_val, np.float64)]
        ctx.call("gf_upload_families", *[P(a) for a in keep])
        ps = _lib.carr(self.pair_stack, np.float64)
        ctx.call("gf_upload_materials", C.c_int(ps.shape[1]), C.c_int(ps.shape[0]), P(ps),
                 P(_lib.carr(self._beta, np.float64)))
        self._tables_dirty = False

    def _upload_owners(self):
        s, ctx, P = self.store, self._ctx, _lib.ptr
        n = s.n_owners
        d = s.__dict__
        p = slice(0, n) if self._own_identity else self._own_d2u
        keep = [_lib.carr(d["_voxel"][:n][p], np.uint64), _lib.carr(d["_subvoxel"][:n][p], np.uint16),
                _lib.carr(d["_quat"][:n][p], np.float32), _lib.carr(d["_lin_vel"][:n][p], np.float64),
                _lib.carr(d["_ang_vel"][:n][p], np.float64), _lib.carr(d["_owner_family"][:n][p], np.uint8),
                _lib.carr(self._tpl_id[p], np.uint32), self._tpl_rows[:, 0].copy(),
                _lib.carr(self._tpl_rows[:, 1:], np.float64)]
        ctx.call("gf_upload_owners", C.c_int64(n), P(keep[0]), P(keep[1]), P(keep[2]), P(keep[3]),
                 P(keep[4]), P(keep[5]), P(keep[6]), C.c_int64(self._tpl_rows.shape[0]), P(keep[7]),
                 P(keep[8]))
        ef = _lib.carr(d["_ext_force"][:n][p], np.float64)
        et = _lib.carr(d["_ext_torque"][:n][p], np.float64)
        if np.any(ef != 0.0) or np.any(et != 0.0):
            ctx.call("gf_set_external_loads", P(ef), P(et))
        else:
            ctx.call("gf_set_external_loads", None, None)

    def _read_owner(self, owner: int) -> dict:
        """One owner's state straight from the device (gf_read_owners)."""
        from .core import decode_position
        d = int(self._own_u2d[int(owner)])
        out = np.zeros((1, 23), np.float64)
        with self._lock:
            self._ctx.call("gf_read_owners", C.c_int64(1), _lib.ptr(np.array([d], np.int64)), _lib.ptr(out))
        r = out[0]
        vox = np.array([r[0]], np.float64).view(np.uint64)
        sub = r[1:4].astype(np.uint16).reshape(1, 3)
        return {"pos": decode_position(vox, sub, self.store.domain)[0], "quat": r[4:8].copy(),
                "lin_vel": r[8:11].copy(), "ang_vel": r[11:14].copy(), "family": int(r[14]),
                "acc_force": r[15:18].copy(), "acc_torque": r[18:21].copy()}

    def _sync_all(self):
        """Device -> host mirror of every owner field."""
        if not self._host_stale or self._ctx is None:
            return
        s, P = self.store, _lib.ptr
        n = s.n_owners
        d = s.__dict__
        vox = np.zeros(n, np.uint64)
        sub = np.zeros((n, 3), np.uint16)
        quat = np.zeros((n, 4), np.float32)
        lv = np.zeros((n, 3))
        av = np.zeros((n, 3))
        fam = np.zeros(n, np.uint8)
        self._ctx.call("gf_download_owners", P(vox), P(sub), P(quat), P(lv), P(av), P(fam))
        af = np.zeros((n, 3))
        at = np.zeros((n, 3))
        self._ctx.call("gf_download_accumulators", P(af), P(at))
        p = slice(0, n) if self._own_identity else self._own_d2u
        d["_voxel"][:n][p] = vox
        d["_subvoxel"][:n][p] = sub
        d["_quat"][:n][p] = quat
        d["_lin_vel"][:n][p] = lv
        d["_ang_vel"][:n][p] = av
        d["_owner_family"][:n][p] = fam
        d["_acc_force"][:n][p] = af
        d["_acc_torque"][:n][p] = at
        self._host_stale = False

    def _sync_field(self, name):
        if self._host_stale:
            with self._lock:
                self._sync_all()
        if name in _MIRROR_FIELDS:
            self._host_dirty = True

    def _push_host(self):
        if self._host_dirty:
            self._upload_owners()
            self._host_dirty = False
        if self._tables_dirty:
            self._upload_tables()

    def _install_acs(self, ca: B.ContactArray) -> None:
        ca.ensure_wildcards(self.model.wildcards)
        n = ca.size
        wild = np.zeros((n, len(self.model.wildcards)), np.float32)
        for i, name in enumerate(self.model.wildcards):
            wild[:, i] = ca.wildcards[name]
        P = _lib.ptr
        kind = _lib.carr(ca.kind, np.uint8)
        sa = self._geom_slot[ca.geom_a] if n else np.zeros(0, np.int64)
        sb = self._geom_slot[ca.geom_b] if n else np.zeros(0, np.int64)
        if n:
            sa, sb, wild = self._orient(kind, self._sph_u2d[sa],
                                        np.where(kind == 0, self._sph_u2d[np.where(kind == 0, sb, 0)], sb),
                                        wild)
            order = np.lexsort((sb, sa, kind))
            kind, sa, sb, wild = kind[order], sa[order], sb[order], wild[order]
        self._ctx.call("gf_set_acs", C.c_int64(n), P(_lib.carr(kind, np.uint8)),
                       P(_lib.carr(sa, np.int64)), P(_lib.carr(sb, np.int64)),
                       P(_lib.carr(wild, np.float32)), C.c_int(len(self.model.wildcards)))

    # -- host mirrors of engine internals (read by tests / IO) -------------------
    @property
    def _pos(self) -> np.ndarray:
        return self.store.positions()

    @property
    def _sph_centers(self) -> np.ndarray:
        out = np.zeros((self._sph_geom.shape[0], 3))
        if self._ctx is not None and out.shape[0]:
            self._push_host()
            dev = np.zeros_like(out)
            self._ctx.call("gf_download_world", _lib.ptr(dev), None, None)
            out[self._sph_d2u] = dev
        return out

    @property
    def _tri_world(self) -> np.ndarray:
        out = np.zeros((self._tri_geom.shape[0], 9))
        if self._ctx is not None and out.shape[0]:
            self._push_host()
            self._ctx.call("gf_download_world", None, _lib.ptr(out), None)
        return out

    @property
    def _ana_world(self) -> np.ndarray:
        out = np.zeros((self._ana_geom.shape[0], 8))
        if self._ctx is not None and out.shape[0]:
            self._push_host()
            self._ctx.call("gf_download_world", None, None, _lib.ptr(out))
        return out

    def _acs_arrays(self):
        n = int(self._ctx.L.gf_acs_size(C.c_void_p(self._ctx.h), 0))
        kind = np.zeros(n, np.uint8)
        sa = np.zeros(n, np.int64)
        sb = np.zeros(n, np.int64)
        wild = np.zeros((n, len(self.model.wildcards)), np.float32)
        if n:
            self._ctx.call("gf_get_acs", C.c_int(0), _lib.ptr(kind), _lib.ptr(sa), _lib.ptr(sb),
                           _lib.ptr(wild))
        return kind, sa, sb, wild

    @property
    def _acs(self) -> B.ContactArray:
        if self._ctx is None:
            return self._acs0
        kind, sa, sb, wild = self._acs_arrays()
        if kind.size:
            sa, sb, wild = self._orient(kind, self._sph_d2u[sa],
                                        np.where(kind == 0, self._sph_d2u[np.where(kind == 0, sb, 0)], sb),
                                        wild)
        tabs = (self._sph_geom, self._tri_geom, self._ana_geom)
        ga = self._sph_geom[sa] if kind.size else np.zeros(0, np.int64)
        gb = np.zeros(kind.shape[0], np.int64)
        for k in range(3):
            sel = kind == k
            if sel.any():
                gb[sel] = tabs[k][sb[sel]]
        ca = B.ContactArray(kind, ga, gb)
        for i, name in enumerate(self.model.wildcards):
            ca.wildcards[name] = wild[:, i].copy()
        return ca.canonicalize() if self.reorder else ca

    def _orient(self, kind, sa, sb, wild):
        """Sphere-sphere pairs are stored as (lower slot, higher slot); when a
        slot permutation flips a pair, A and B swap roles and the model's
        orientation-dependent history (e.g. the tangential displacement of A
        relative to B, forces.py:111-118) changes sign."""
        flip = (kind == 0) & (sa > sb)
        if flip.any():
            sa, sb = np.where(flip, sb, sa), np.where(flip, sa, sb)
            wild = wild.copy()
            for col in self.model.flip_on_swap:
                wild[flip, col] = -wild[flip, col]
        return sa, sb, wild

    @_acs.setter
    def _acs(self, value):
        self._acs0 = value

    @property
    def _wild(self) -> np.ndarray:
        ca = self._acs
        if not ca.size:
            return np.zeros((0, len(self.model.wildcards)), np.float32)
        return np.stack([ca.wildcards[nm] for nm in self.model.wildcards], axis=1)

    def _refresh_world(self) -> None:
        """World geometry is derived on the device on demand."""

    def _set_owner_position(self, owner: int, xyz) -> None:
        self.store.set_position(owner, xyz)

    def _current_margin(self) -> float:
        base = B.compute_margin(self.v_err, self.h, max(1, self.scheduler.n_max))
        return 2.0 * base + self.margin_policy.added

    # -- driving --------------------------------------------------------------------
    def _adapt_n_max(self, waited_event: bool) -> None:
        """Lookahead adaptation, the reference's policy (engine.py:743-775)."""
        sch = self.scheduler
        if self.sync_mode:
            sch.n_max = 1
            return
        if self._fixed_n_max is not None:
            sch.n_max = self._fixed_n_max
            return
        if waited_event:
            self._n_max_floor = max(self._n_max_floor, sch.n_max + 1)
            self._calm_cycles = 0
        else:
            self._calm_cycles += 1
            if self._calm_cycles >= 64 and self._n_max_floor > 2:
                self._n_max_floor -= 1
                self._calm_cycles = 0
        if sch.step_time_ema <= 0.0 or sch.last_cd_seconds <= 0.0:
            return
        proposal = int(math.ceil(1.25 * sch.last_cd_seconds / sch.step_time_ema))
        if self._margin_cap_steps is not None:
            proposal = min(proposal, self._margin_cap_steps)
            self._n_max_floor = min(self._n_max_floor, self._margin_cap_steps)
        sch.n_max = min(1024, max(2, self._n_max_floor, proposal))
        self.margin_policy.n_max = sch.n_max

    def _schedule(self):
        """(period, lag) of the deterministic kT/dT schedule for the current
        n_max: snapshots every n_max // 2 steps (the reference's work-order
        throttle, engine.py:719-724), adopted one period later, so a contact
        array is never older than n_max - 1 steps (engine.py:853-855)."""
        if self.sync_mode:
            self.scheduler.n_max = 1
            return 1, 0
        n_max = max(2, int(self.scheduler.n_max))
        period = max(1, n_max // 2)
        return period, period

    def do_dynamics(self, duration: float) -> None:
        if not self._initialized:
            raise ConfigurationError("initialize() must be called first")
        if self._closed:
            raise ConfigurationError("simulator is closed")
        steps = int(math.ceil(duration / self.h - 1e-9))
        if steps <= 0:
            return
        if self.active_box_policy is not None:
            self._run_with_boxes(steps)
        else:
            self._run(steps)

    def _run_with_boxes(self, steps: int) -> None:
        done = 0
        while done < steps:
            if self.sim_time >= self._next_box_refresh():
                self._apply_active_boxes()
                self._box_next = self.sim_time + self.active_box_policy.refresh_period
            # run until the next refresh time
            nxt = self._next_box_refresh()
            chunk = max(1, min(steps - done, int(math.ceil((nxt - self.sim_time) / self.h - 1e-9))))
            self._run(chunk)
            done += chunk

    def _next_box_refresh(self) -> float:
        return getattr(self, "_box_next", 0.0)

    def _apply_active_boxes(self) -> None:
        """Family re-tagging at box refresh (engine.py:857-879), on the device
        (gf_apply_active_boxes): positions, families and velocities never
        leave HBM; the host mirrors are marked stale."""
        policy = self.active_box_policy
        nb = len(policy.half_extents)
        if nb == 0:
            return
        boxes = np.zeros((nb, 6), np.float64)
        anchors = np.full(nb, -1, np.int64)
        for b, (half, anchor, center) in enumerate(zip(policy.half_extents, policy.anchors, policy.centers)):
            boxes[b, 3:] = np.asarray(half, dtype=np.float64)
            if anchor is not None:
                anchors[b] = int(self._own_u2d[int(anchor)])
            else:
                boxes[b, :3] = np.asarray(center, dtype=np.float64)
        with self._lock:
            self._push_host()
            changed = C.c_int64(0)
            self._ctx.call("gf_apply_active_boxes", C.c_int(nb), _lib.ptr(boxes), _lib.ptr(anchors),
                           C.c_int(int(policy.active_family)), C.c_int(int(policy.frozen_family)),
                           C.byref(changed))
            if changed.value:
                self._host_stale = True
        self.box_retags = getattr(self, "box_retags", 0) + int(changed.value)

    def _run(self, steps: int) -> None:
        if self.decomposition is not None:
            from . import decomp
            decomp.run_member(self, steps)
            return
        with self._lock:
            self._push_host()
            rp, keep = self._run_params(steps)
            rr = _lib.RunResult()
            t0 = _time.perf_counter()
            self._ctx.call("gf_run", C.byref(rp), C.byref(rr))
            self._finish_run(rr, _time.perf_counter() - t0)

    def _run_params(self, steps: int):
        """gf_run_params of the next `steps` steps (+ the arrays it points to)."""
        sch = self.scheduler
        period, lag = self._schedule()
        margin = self._current_margin()
        step0 = sch.step_counter
        dyn = self._dynamic_prescriptions
        spec = np.zeros((max(1, len(dyn)), 3), np.int32)
        vals = np.zeros((steps, max(1, len(dyn))), np.float64)
        if dyn:
            ns = dict(_SAFE_EVAL_NS)
            for j, (famid, table, ax, _) in enumerate(dyn):
                spec[j] = (famid, table, ax)
            for i in range(steps):
                ns["t"] = (step0 + i) * self.h
                for j, (_, _, _, code) in enumerate(dyn):
                    vals[i, j] = float(eval(code, {"__builtins__": {}}, ns))
        rp = _lib.RunParams()
        rp.n_steps = steps
        rp.step0 = step0
        rp.h = self.h
        for a in range(3):
            rp.g[a] = float(self.gravity[a])
        rp.v_err = self.v_err
        rp.margin = margin
        rp.period = period
        rp.lag = lag
        rp.n_dyn = len(dyn)
        rp.write_acc = 1
        rp.dyn_spec = spec.ctypes.data_as(C.c_void_p)
        rp.dyn_vals = vals.ctypes.data_as(C.c_void_p)
        return rp, (spec, vals)

    def _finish_run(self, rr, wall: float, adapt: bool = True) -> None:
        """Scheduler / timing bookkeeping after a gf_run; raises on a watchdog."""
        sch = self.scheduler
        period, _ = self._schedule()
        step0 = sch.step_counter
        self.last_run = rr
        self._host_stale = True
        done = int(rr.steps_done)
        sch.step_counter = step0 + done
        self.sim_time = sch.step_counter * self.h
        sch.ca_updates = int(rr.ca_updates)
        sch.timing["dyn_force"] += rr.dt_ms * 1e-3
        sch.timing["kin_detect"] += rr.kt_ms * 1e-3
        sch.timing["dyn_transfer"] += max(0.0, wall - rr.dt_ms * 1e-3)
        sch.last_wo_stamp = step0 + done
        self._last_touching = int(rr.touching)
        if done > 0:
            sch.step_time_ema = rr.dt_ms * 1e-3 / done
        n_cd = max(1, done // max(1, period))
        sch.last_cd_seconds = rr.kt_ms * 1e-3 / n_cd
        if rr.oob_owner >= 0 or rr.bad_owner >= 0:
            self._raise_watchdog(rr)
        if adapt:
            self._adapt_n_max(waited_event=False)

    def _raise_watchdog(self, rr) -> None:
        oob_first = rr.oob_owner >= 0 and (rr.bad_owner < 0 or rr.oob_step <= rr.bad_step)
        d2u = self._own_d2u
        if oob_first:
            o = int(d2u[int(rr.oob_owner)])
            msg = (f"owner {o} left the domain at t={self.sim_time:.6g} "
                   f"(position {self._pos[o].tolist()})")
        else:
            o = int(d2u[int(rr.bad_owner)])
            v = self.store.lin_vel[o]
            msg = (f"owner {o} exceeded error-out velocity {self.v_err} m/s "
                   f"(speed {float(np.linalg.norm(v)):.3g}) at t={self.sim_time:.6g}")
        self.close()
        raise DivergenceError(msg)

    def timing_report(self) -> dict:
        sch = self.scheduler
        rep = dict(sch.timing)
        rep.update(steps=sch.step_counter, n_max=sch.n_max, dynamics_waits=sch.dynamics_waits,
                   kinematics_waits=sch.kinematics_waits, ca_updates=sch.ca_updates,
                   margin=self._current_margin())
        return rep


# ---------------------------------------------------------------------------
# samplers (setup only; engine.py:913-967)
# ---------------------------------------------------------------------------

def hcp_lattice(lo, hi, spacing: float, anchor=None) -> np.ndarray:
    if spacing <= 0.0:
        raise ValidationError(f"spacing must be positive, got {spacing}")
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    anchor = lo if anchor is None else np.asarray(anchor, dtype=np.float64)
    r = spacing / 2.0
    dy = math.sqrt(3.0) * r
    dz = 2.0 * math.sqrt(6.0) / 3.0 * r
    eps = 1e-12

    def span(a, b, step):
        return int(math.ceil(a / step - eps)), int(math.floor(b / step + eps))

    rows = []
    k0, k1 = span(lo[2] - anchor[2], hi[2] - anchor[2], dz)
    for k in range(k0, k1 + 1):
        z = anchor[2] + k * dz
        yoff = (k % 2) * dy / 3.0
        j0, j1 = span(lo[1] - anchor[1] - yoff, hi[1] - anchor[1] - yoff, dy)
        for j in range(j0, j1 + 1):
            y = anchor[1] + j * dy + yoff
            xoff = ((j + k) % 2) * r
            i0, i1 = span(lo[0] - anchor[0] - xoff, hi[0] - anchor[0] - xoff, 2.0 * r)
            if i1 < i0:
                continue
            i = np.arange(i0, i1 + 1)
            row = np.empty((i.shape[0], 3))
            row[:, 0] = anchor[0] + i * 2.0 * r + xoff
            row[:, 1] = y
            row[:, 2] = z
            rows.append(row)
    return np.concatenate(rows) if rows else np.zeros((0, 3))


def hcp_sample_cylinder(center, radius: float, half_height: float, spacing: float) -> np.ndarray:
    c = np.asarray(center, dtype=np.float64)
    pts = hcp_lattice(c - (radius, radius, half_height), c + (radius, radius, half_height), spacing,
                      anchor=c)
    if pts.shape[0] == 0:
        return pts
    keep = (((pts[:, 0] - c[0]) ** 2 + (pts[:, 1] - c[1]) ** 2 <= radius ** 2 + 1e-12)
            & (np.abs(pts[:, 2] - c[2]) <= half_height + 1e-12))
    return pts[keep]


def hcp_sample_box(center, half_extents, spacing: float) -> np.ndarray:
    c = np.asarray(center, dtype=np.float64)
    h = np.asarray(half_extents, dtype=np.float64)
    return hcp_lattice(c - h, c + h, spacing)
