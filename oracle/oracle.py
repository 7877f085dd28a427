"""CPU parity oracle for the grainforge DEM step -- TEST INFRASTRUCTURE ONLY.

ctypes front-end over ``oracle/build/liborc.so`` (gf_oracle.c, a plain-C
restatement of the reference kernels) plus the numpy glue the reference does
in numpy itself (slot -> geometry-id map and canonical sort of
broadphase.py:283-288, merge_history of broadphase.py:110-135).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.  The product path (``paper_2311_04648_b200``) never does.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
bit-for-bit against fixtures produced by the reference package itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liborc.so")
_lib = None

_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_encode_positions.restype = _I64
        L.orc_contact_forces.restype = _I64
        L.orc_detect.restype = _P
        L.orc_grid_for.restype = C.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_P) if a is not None else None


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ---------------------------------------------------------------------------
# coordinates / transforms
# ---------------------------------------------------------------------------

def encode_positions(pos, lo, hi, edge):
    pos = _c(pos, np.float64).reshape(-1, 3)
    n = pos.shape[0]
    vox = np.zeros(n, np.uint64)
    sub = np.zeros((n, 3), np.uint16)
    bad = lib().orc_encode_positions(_I64(n), _p(pos), _p(_c(lo, np.float64)),
                                     _p(_c(hi, np.float64)), _D(edge), _p(vox), _p(sub))
    return vox, sub, int(bad)


def decode_positions(vox, sub, lo, edge):
    vox = _c(vox, np.uint64)
    sub = _c(sub, np.uint16).reshape(-1, 3)
    out = np.zeros((vox.shape[0], 3), np.float64)
    lib().orc_decode_positions(_I64(vox.shape[0]), _p(vox), _p(sub),
                               _p(_c(lo, np.float64)), _D(edge), _p(out))
    return out


def sphere_world(sph_geom, geom_params, geom_owner, owner_pos, quat):
    sph_geom = _c(sph_geom, np.int64)
    out = np.zeros((sph_geom.shape[0], 3), np.float64)
    rad = np.zeros(sph_geom.shape[0], np.float32)
    lib().orc_sphere_world(_I64(sph_geom.shape[0]), _p(sph_geom),
                           _p(_c(geom_params, np.float32)), _p(_c(geom_owner, np.int64)),
                           _p(_c(owner_pos, np.float64)), _p(_c(quat, np.float32)),
                           _p(out), _p(rad))
    return out, rad


def triangle_world(tri_geom, geom_params, geom_owner, owner_pos, quat):
    tri_geom = _c(tri_geom, np.int64)
    out = np.zeros((tri_geom.shape[0], 9), np.float64)
    lib().orc_triangle_world(_I64(tri_geom.shape[0]), _p(tri_geom),
                             _p(_c(geom_params, np.float32)), _p(_c(geom_owner, np.int64)),
                             _p(_c(owner_pos, np.float64)), _p(_c(quat, np.float32)), _p(out))
    return out


def analytic_world(ana_geom, geom_params, geom_owner, owner_pos, quat):
    ana_geom = _c(ana_geom, np.int64)
    out = np.zeros((ana_geom.shape[0], 8), np.float64)
    lib().orc_analytic_world(_I64(ana_geom.shape[0]), _p(ana_geom),
                             _p(_c(geom_params, np.float32)), _p(_c(geom_owner, np.int64)),
                             _p(_c(owner_pos, np.float64)), _p(_c(quat, np.float32)), _p(out))
    return out


def angular_velocity_global(quat, w_local):
    quat = _c(quat, np.float32)
    out = np.zeros((quat.shape[0], 3), np.float64)
    lib().orc_angular_velocity_global(_I64(quat.shape[0]), _p(quat),
                                      _p(_c(w_local, np.float64)), _p(out))
    return out


def closest_point_on_triangle(p, tri):
    out = np.zeros(4, np.float64)
    lib().orc_closest_point_on_triangle(_p(_c(p, np.float64)),
                                        _p(_c(tri, np.float64).reshape(9)), _p(out))
    return out[:3], float(out[3])


# ---------------------------------------------------------------------------
# broad phase
# ---------------------------------------------------------------------------

def bin_ranges(centers, radii, margin, glo, inv_bin, nb):
    centers = _c(centers, np.float64).reshape(-1, 3)
    out = np.zeros((centers.shape[0], 6), np.int64)
    lib().orc_bin_ranges(_I64(centers.shape[0]), _p(centers), _p(_c(radii, np.float32)),
                         _D(margin), _p(_c(glo, np.float64)), _D(inv_bin),
                         _p(_c(nb, np.int64)), _p(out))
    return out


_KEY_BITS = 24


def sort_keys(kind, a, b):
    """broadphase.py:77-86 (24-bit id budget of the reference)."""
    return ((np.asarray(kind, np.uint64) << np.uint64(2 * _KEY_BITS))
            | (np.asarray(a, np.uint64) << np.uint64(_KEY_BITS))
            | np.asarray(b, np.uint64))


def detect_contacts(snap: dict, margin: float):
    """broadphase.detect_contacts over a snapshot dict with the
    DetectionSnapshot field names.  Returns dict(kind, geom_a, geom_b,
    slot_a, slot_b, glo, inv_bin, nb) in canonical order."""
    L = lib()
    c = _c(snap["sph_center"], np.float64).reshape(-1, 3)
    m = c.shape[0]
    rad = _c(snap["sph_radius"], np.float32)
    tri = _c(snap["tri_world"], np.float64).reshape(-1, 9)
    ana = _c(snap["ana_world"], np.float64).reshape(-1, 8)
    grid = np.zeros(4, np.float64)
    nb = np.zeros(3, np.int64)
    h = L.orc_detect(
        _I64(m), _p(c), _p(rad), _p(_c(snap["sph_owner"], np.int64)),
        _p(_c(snap["sph_family"], np.uint8)),
        _I64(tri.shape[0]), _p(tri), _p(_c(snap["tri_owner"], np.int64)),
        _p(_c(snap["tri_family"], np.uint8)),
        _I64(ana.shape[0]), _p(ana), _p(_c(snap["ana_kind"], np.uint8)),
        _p(_c(snap["ana_owner"], np.int64)), _p(_c(snap["ana_family"], np.uint8)),
        _p(_c(snap["mask"], np.uint8)), _D(margin), _p(grid), _p(nb))
    counts = np.zeros(3, np.int64)
    L.orc_pairs_counts(_P(h), _p(counts))
    parts = []
    geom_tabs = (snap["sph_geom"], snap["tri_geom"], snap["ana_geom"])
    for kind in range(3):
        n = int(counts[kind])
        sa = np.zeros(n, np.int64)
        sb = np.zeros(n, np.int64)
        L.orc_pairs_copy(_P(h), C.c_int(kind), _p(sa), _p(sb))
        parts.append((np.full(n, kind, np.uint8), sa, sb,
                      np.asarray(snap["sph_geom"], np.int64)[sa],
                      np.asarray(geom_tabs[kind], np.int64)[sb]))
    L.orc_pairs_free(_P(h))
    kind = np.concatenate([p[0] for p in parts])
    sa = np.concatenate([p[1] for p in parts])
    sb = np.concatenate([p[2] for p in parts])
    ga = np.concatenate([p[3] for p in parts])
    gb = np.concatenate([p[4] for p in parts])
    order = np.argsort(sort_keys(kind, ga, gb), kind="stable")
    return dict(kind=kind[order], geom_a=ga[order], geom_b=gb[order],
                slot_a=sa[order], slot_b=sb[order], glo=grid[:3].copy(),
                inv_bin=float(grid[3]), nb=nb)


def merge_history(old_keys, old_wild, new_keys):
    """broadphase.py:110-135 on canonical key arrays; wild is (n, W) f32."""
    old_keys = np.asarray(old_keys, np.uint64)
    new_keys = np.asarray(new_keys, np.uint64)
    w = old_wild.shape[1] if old_wild.ndim == 2 else 0
    out = np.zeros((new_keys.shape[0], w), np.float32)
    if old_keys.shape[0] == 0:
        return out
    pos = np.searchsorted(old_keys, new_keys)
    pos_c = np.minimum(pos, old_keys.shape[0] - 1)
    matched = old_keys[pos_c] == new_keys
    out[matched] = old_wild[pos_c[matched]]
    return out


# ---------------------------------------------------------------------------
# dynamics
# ---------------------------------------------------------------------------

def contact_forces(kind, slot_a, slot_b, owner_a, owner_b, mat_a, mat_b,
                   sph_centers, sph_radii, tri_world, ana_world, ana_kind,
                   owner_pos, lin_vel, ang_vel_global, mass, pair_stack, wild,
                   ts, sim_time, nthreads=1, model=0):
    """make_contact_kernel(hertz_mindlin_core_jit) (forces.py:547-593).
    wild (n, W) f32 is updated in place.  Returns (touching, out_ft, depth, cp)."""
    n = int(np.asarray(kind).shape[0])
    out_ft = np.zeros((n, 6), np.float64)
    depth = np.zeros(n, np.float64)
    cp = np.zeros((n, 3), np.float64)
    assert wild.dtype == np.float32 and wild.flags.c_contiguous
    pair_stack = _c(pair_stack, np.float64)
    touching = lib().orc_contact_forces(
        _I64(n), _p(_c(kind, np.uint8)), _p(_c(slot_a, np.int64)), _p(_c(slot_b, np.int64)),
        _p(_c(owner_a, np.int64)), _p(_c(owner_b, np.int64)),
        _p(_c(mat_a, np.int64)), _p(_c(mat_b, np.int64)),
        _p(_c(sph_centers, np.float64)), _p(_c(sph_radii, np.float32)),
        _p(_c(tri_world, np.float64)), _p(_c(ana_world, np.float64)),
        _p(_c(ana_kind, np.uint8)), _p(_c(owner_pos, np.float64)),
        _p(_c(lin_vel, np.float64)), _p(_c(ang_vel_global, np.float64)),
        _p(_c(mass, np.float64)), _p(pair_stack), _I64(pair_stack.shape[1]),
        _I64(wild.shape[1] if n else 4), _p(wild), _D(ts), _D(sim_time),
        _p(out_ft), _p(depth), _p(cp), C.c_int(nthreads), C.c_int(model))
    return int(touching), out_ft, depth, cp


def reduce_to_owners(owner_a, owner_b, out_ft, cps, owner_pos):
    owner_pos = _c(owner_pos, np.float64)
    n_o = owner_pos.shape[0]
    acc_f = np.zeros((n_o, 3), np.float64)
    acc_t = np.zeros((n_o, 3), np.float64)
    owner_a = _c(owner_a, np.int64)
    lib().orc_reduce_to_owners(_I64(owner_a.shape[0]), _p(owner_a), _p(_c(owner_b, np.int64)),
                               _p(_c(out_ft, np.float64)), _p(_c(cps, np.float64)),
                               _p(owner_pos), _I64(n_o), _p(acc_f), _p(acc_t))
    return acc_f, acc_t


def integrate_and_refresh(h, g, owner_pos, quat, lin_vel, ang_vel, mass, moi,
                          acc_f, acc_t, ext_f, ext_t, family, fixed_flag,
                          lv_mask, lv_val, av_mask, av_val, prescribed_flag,
                          v_err, lo, hi, edge, voxel, sub, sph_geom,
                          geom_params, geom_owner, sph_centers, nthreads=1):
    """_kernels.integrate_and_refresh; every state array is updated in place
    (must be C-contiguous with the reference dtypes).  Returns (bad, oob)."""
    for a, dt in ((owner_pos, np.float64), (quat, np.float32), (lin_vel, np.float64),
                  (ang_vel, np.float64), (voxel, np.uint64), (sub, np.uint16),
                  (sph_centers, np.float64)):
        assert a.dtype == dt and a.flags.c_contiguous, (a.dtype, dt)
    out2 = np.zeros(2, np.int64)
    n = owner_pos.shape[0]
    lib().orc_integrate_and_refresh(
        _I64(n), _D(h), _D(g[0]), _D(g[1]), _D(g[2]), _p(owner_pos), _p(quat),
        _p(lin_vel), _p(ang_vel), _p(_c(mass, np.float64)), _p(_c(moi, np.float64)),
        _p(_c(acc_f, np.float64)), _p(_c(acc_t, np.float64)),
        _p(_c(ext_f, np.float64)), _p(_c(ext_t, np.float64)),
        _p(_c(family, np.uint8)), _p(_c(fixed_flag, np.uint8)),
        _p(_c(lv_mask, np.uint8)), _p(_c(lv_val, np.float64)),
        _p(_c(av_mask, np.uint8)), _p(_c(av_val, np.float64)),
        _p(_c(prescribed_flag, np.uint8)), _D(v_err),
        _p(_c(lo, np.float64)), _p(_c(hi, np.float64)), _D(edge),
        _p(voxel), _p(sub), _I64(np.asarray(sph_geom).shape[0]),
        _p(_c(sph_geom, np.int64)), _p(_c(geom_params, np.float32)),
        _p(_c(geom_owner, np.int64)), _p(sph_centers), C.c_int(nthreads), _p(out2))
    return int(out2[0]), int(out2[1])


# ---------------------------------------------------------------------------
# step driver (engine._step_once, engine.py:785-855) on a plain scene dict
# ---------------------------------------------------------------------------

GEOM_SPHERE, GEOM_TRIANGLE, GEOM_PLANE, GEOM_CYLINDER = 0, 1, 2, 3


class OracleStepper:
    """Deterministic CPU re-run of the reference dT/kT protocol.

    scene: dict with the StateStore arrays (trimmed to n_owners / n_geoms):
      voxel, subvoxel, quat, lin_vel, ang_vel, mass, moi, owner_family,
      ext_force, ext_torque, geom_owner, geom_kind, geom_material,
      geom_params, lo, hi, edge, pair_stack, mask, fixed_flag,
      prescribed_flag, lv_mask, lv_val, av_mask, av_val, gravity, h, v_err.
    Schedule (the B200 scheduler's, csrc/gf_context.cu gf_run): the first
    detection is adopted immediately; afterwards, once no detection is in
    flight and `period` steps passed since the last snapshot, a snapshot is
    taken at the start of step s and adopted at the start of step s + lag
    (adoption precedes the next snapshot check).  lag=0, period=1 is the
    reference's sync mode (engine.py:726-741).
    """

    def __init__(self, scene: dict, margin: float, period: int = 1, lag: int = 0,
                 nthreads: int = 1, model: int = 0):
        s = {k: (np.array(v, copy=True) if isinstance(v, np.ndarray) else v)
             for k, v in scene.items()}
        self.s = s
        self.margin = float(margin)
        self.period = int(period)
        self.lag = int(lag)
        self.nthreads = int(nthreads)
        self.model = int(model)  # 0 Hertz-Mindlin, 1 models.py hertz_mindlin_cohesive
        kinds = s["geom_kind"]
        self.sph_geom = np.nonzero(kinds == GEOM_SPHERE)[0].astype(np.int64)
        self.tri_geom = np.nonzero(kinds == GEOM_TRIANGLE)[0].astype(np.int64)
        self.ana_geom = np.nonzero((kinds == GEOM_PLANE) | (kinds == GEOM_CYLINDER))[0].astype(np.int64)
        n_g = kinds.shape[0]
        self.geom_slot = np.zeros(n_g, np.int64)
        for arr in (self.sph_geom, self.tri_geom, self.ana_geom):
            self.geom_slot[arr] = np.arange(arr.shape[0])
        self.sph_radius = s["geom_params"][self.sph_geom, 3].astype(np.float32)
        self.sph_owner = s["geom_owner"][self.sph_geom]
        self.ana_kind = kinds[self.ana_geom].astype(np.uint8)
        self.pos = decode_positions(s["voxel"], s["subvoxel"], s["lo"], s["edge"])
        self.centers, _ = sphere_world(self.sph_geom, s["geom_params"], s["geom_owner"],
                                       self.pos, s["quat"])
        self.tri_world = triangle_world(self.tri_geom, s["geom_params"], s["geom_owner"],
                                        self.pos, s["quat"])
        self.ana_world = analytic_world(self.ana_geom, s["geom_params"], s["geom_owner"],
                                        self.pos, s["quat"])
        n = self.pos.shape[0]
        self.acc_f = np.zeros((n, 3))
        self.acc_t = np.zeros((n, 3))
        self.step = 0
        self.sim_time = 0.0
        self.last_touching = 0
        self.keys = np.zeros(0, np.uint64)
        self.acs = dict(kind=np.zeros(0, np.uint8), geom_a=np.zeros(0, np.int64),
                        geom_b=np.zeros(0, np.int64))
        self.wild = np.zeros((0, 4), np.float32)
        self.pending = []  # (adopt_step, acs); at most one in flight
        self.first = True
        self.last_snap = 0
        self.dyn_prescriptions = []  # (family, table_name, axis, fn(t))

    def snapshot(self):
        s = self.s
        fam = s["owner_family"]
        go = s["geom_owner"]
        return dict(
            sph_center=self.centers.copy(), sph_radius=self.sph_radius,
            sph_geom=self.sph_geom, sph_owner=self.sph_owner,
            sph_family=fam[self.sph_owner],
            tri_world=self.tri_world.copy(), tri_geom=self.tri_geom,
            tri_owner=go[self.tri_geom], tri_family=fam[go[self.tri_geom]],
            ana_world=self.ana_world.copy(), ana_kind=self.ana_kind,
            ana_geom=self.ana_geom, ana_owner=go[self.ana_geom],
            ana_family=fam[go[self.ana_geom]], mask=s["mask"])

    def adopt(self, acs):
        new_keys = sort_keys(acs["kind"], acs["geom_a"], acs["geom_b"])
        self.wild = merge_history(self.keys, self.wild, new_keys)
        self.keys = new_keys
        self.acs = acs

    def step_once(self):
        s = self.s
        while self.pending and self.pending[0][0] <= self.step:
            self.adopt(self.pending.pop(0)[1])
        if self.first or (not self.pending and self.step - self.last_snap >= self.period):
            # the first detection is waited for (engine.py:679-682)
            adopt_at = self.step if self.first else self.step + self.lag
            self.pending.append((adopt_at, detect_contacts(self.snapshot(), self.margin)))
            self.last_snap = self.step
            self.first = False
        while self.pending and self.pending[0][0] <= self.step:
            self.adopt(self.pending.pop(0)[1])
        acs = self.acs
        ga, gb = acs["geom_a"], acs["geom_b"]
        go = s["geom_owner"]
        wang = angular_velocity_global(s["quat"], s["ang_vel"])
        if ga.shape[0]:
            self.last_touching, out_ft, depth, cp = contact_forces(
                acs["kind"], self.geom_slot[ga], self.geom_slot[gb], go[ga], go[gb],
                s["geom_material"][ga].astype(np.int64), s["geom_material"][gb].astype(np.int64),
                self.centers, self.sph_radius, self.tri_world, self.ana_world,
                self.ana_kind, self.pos, s["lin_vel"], wang, s["mass"],
                s["pair_stack"], self.wild, s["h"], self.sim_time, self.nthreads, self.model)
        else:
            self.last_touching = 0
            out_ft = np.zeros((0, 6)); cp = np.zeros((0, 3)); depth = np.zeros(0)
        # the step's per-contact forces (tests normalise tolerances by them)
        self.last_force_median = (float(np.median(np.linalg.norm(out_ft[depth > 0, :3], axis=1)))
                                  if np.any(depth > 0) else 0.0)
        self.acc_f, self.acc_t = reduce_to_owners(go[ga], go[gb], out_ft, cp, self.pos)
        for fam, tab, ax, fn in self.dyn_prescriptions:
            s[tab][fam, ax] = fn(self.sim_time)
        bad, oob = integrate_and_refresh(
            s["h"], s["gravity"], self.pos, s["quat"], s["lin_vel"], s["ang_vel"],
            s["mass"], s["moi"], self.acc_f, self.acc_t, s["ext_force"], s["ext_torque"],
            s["owner_family"], s["fixed_flag"], s["lv_mask"], s["lv_val"],
            s["av_mask"], s["av_val"], s["prescribed_flag"], s["v_err"],
            s["lo"], s["hi"], s["edge"], s["voxel"], s["subvoxel"], self.sph_geom,
            s["geom_params"], s["geom_owner"], self.centers, self.nthreads)
        if oob >= 0 or bad >= 0:
            raise RuntimeError(f"oracle watchdog: bad={bad} oob={oob}")
        if self.tri_geom.shape[0] or self.ana_geom.shape[0]:
            fams = s["owner_family"][np.unique(go[np.concatenate([self.tri_geom, self.ana_geom])])]
            if np.any(~s["fixed_flag"][fams].astype(bool)):
                self.tri_world = triangle_world(self.tri_geom, s["geom_params"], go, self.pos, s["quat"])
                self.ana_world = analytic_world(self.ana_geom, s["geom_params"], go, self.pos, s["quat"])
        self.step += 1
        self.sim_time = self.step * s["h"]


def margin_for(v_err: float, h: float, n_max: int, added: float = 0.0) -> float:
    """engine._current_margin (engine.py:598-602)."""
    return 2.0 * (2.0 * v_err * h * max(1, n_max)) + added


def restitution_beta(cor: float) -> float:
    loge = math.log(1e-12) if cor < 1e-12 else math.log(cor)
    return loge / math.sqrt(loge * loge + math.pi * math.pi)
