"""Generate golden input/output fixtures from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports `grainforge` from /root/reference/pkg/src, builds small seeded
scenes, runs the reference's own kernels / Simulator on them and writes
`tests/golden/*.npz`.  The fixtures pin the C oracle (oracle/gf_oracle.c) bit
for bit (tests/test_oracle_golden.py); the GPU path is then checked against
the oracle.  Nothing under tests/ reads /root/reference at run time.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import grainforge as gf  # noqa: E402
from grainforge import _kernels as K  # noqa: E402
from grainforge import broadphase as B  # noqa: E402
from grainforge import meshes  # noqa: E402
from grainforge.core import ClumpSphere, ClumpTemplate, Domain  # noqa: E402
from grainforge.engine import Simulator, hcp_sample_box  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def snap_arrays(snap: B.DetectionSnapshot) -> dict:
    return {f"snap_{k}": np.asarray(getattr(snap, k)) for k in (
        "sph_center", "sph_radius", "sph_geom", "sph_owner", "sph_family",
        "tri_world", "tri_geom", "tri_owner", "tri_family", "ana_world",
        "ana_kind", "ana_geom", "ana_owner", "ana_family", "mask")}


def scene_arrays(sim: Simulator) -> dict:
    """StateStore + engine tables in the OracleStepper scene layout."""
    s = sim.store
    n, g = s.n_owners, s.n_geoms
    return dict(
        voxel=s.voxel[:n].copy(), subvoxel=s.subvoxel[:n].copy(),
        quat=s.quat[:n].copy(), lin_vel=s.lin_vel[:n].copy(),
        ang_vel=s.ang_vel[:n].copy(), mass=s.mass[:n].copy(), moi=s.moi[:n].copy(),
        owner_family=s.owner_family[:n].copy(), ext_force=s.ext_force[:n].copy(),
        ext_torque=s.ext_torque[:n].copy(), geom_owner=s.geom_owner[:g].copy(),
        geom_kind=s.geom_kind[:g].copy(), geom_material=s.geom_material[:g].copy(),
        geom_params=s.geom_params[:g].copy(), lo=s.domain.lo.copy(),
        hi=s.domain.hi.copy(), edge=np.float64(s.domain.voxel_edge),
        pair_stack=gf.forces.material_pair_stack(sim.materials, sim.model),
        mask=s.families.mask.astype(np.uint8),
        fixed_flag=sim._fixed_flag.astype(np.uint8),
        prescribed_flag=sim._prescribed_flag.astype(np.uint8),
        lv_mask=sim._lv_mask.astype(np.uint8), lv_val=sim._lv_val.copy(),
        av_mask=sim._av_mask.astype(np.uint8), av_val=sim._av_val.copy(),
        gravity=sim.gravity.copy(), h=np.float64(sim.h), v_err=np.float64(sim.v_err),
        owner_template=s.owner_template[:n].copy(),
    )


# ---------------------------------------------------------------------------
# scenes
# ---------------------------------------------------------------------------

def box_scene(n=2000, seed=0, crr=0.0, mu=0.3, with_mesh=False, clumps=False):
    """C1-style settling box (BASELINE.json configs[0], scaled down)."""
    rng = np.random.default_rng(seed)
    r = 0.005
    dom = Domain((-0.1, -0.1, -0.02), (0.1, 0.1, 0.3))
    sim = Simulator(dom)
    mat = sim.load_material({"E": 1e7, "nu": 0.3, "CoR": 0.6, "mu": mu, "Crr": crr})
    if clumps:
        tpl = sim.load_clump_template(ClumpTemplate(
            mass=2600 * 3 * 4 / 3 * math.pi * r**3, moi=np.array([2e-8, 3e-8, 3e-8]),
            spheres=tuple(ClumpSphere(np.array([dx, 0.0, 0.0]), r, mat)
                          for dx in (-r, 0.0, r))))
        spacing = 2 * 2 * r * 0.99
    else:
        m = 2600 * 4 / 3 * math.pi * r**3
        tpl = sim.load_clump_template(ClumpTemplate.solid_sphere(r, m, mat))
        spacing = 2 * r * 1.02
    zc = 0.14 if with_mesh else 0.08 + 1.01 * r
    half = (0.062, 0.07, 0.08) if clumps else (0.07, 0.07, 0.08)
    pts = hcp_sample_box((0, 0, zc), half, spacing)
    if with_mesh:  # keep clear of the solid column at (0.05, 0.05)
        keep = (pts[:, 0] - 0.05) ** 2 + (pts[:, 1] - 0.05) ** 2 > (0.012 + 2.5 * r) ** 2
        pts = pts[keep]
    pts = pts[:n]
    sim.add_clumps(tpl, pts)
    # walls: floor + 4 sides, fixed family 255 (C1 config)
    walls = [("plane", (0, 0, 0), (0, 0, 1), mat),
             ("plane", (-0.08, 0, 0), (1, 0, 0), mat),
             ("plane", (0.08, 0, 0), (-1, 0, 0), mat),
             ("plane", (0, -0.08, 0), (0, 1, 0), mat),
             ("plane", (0, 0.08, 0), (0, -1, 0), mat)]
    sim.add_analytic(walls, family=255)
    sim.set_family_fixed(255)
    if with_mesh:
        blades = meshes.builtin("paddle")
        mix = sim.add_mesh(blades, mat, family=10, position=(0, 0, 0.03))
        sim.store.scale_mesh(mix, (0.06, 0.06, 0.05))
        sim.set_family_prescribed_ang_vel(10, "0", "0", "6.0")
        # a cylinder column in the middle
        sim.add_analytic([("cylinder", (0.05, 0.05, 0), (0, 0, 1), 0.012, 1.0, mat)],
                         family=254)
        sim.set_family_fixed(254)
    sim.set_gravity([0, 0, -9.81])
    sim.set_init_time_step(1e-5)
    sim.set_error_out_velocity(5.0)
    # jitter velocities so tangential/rolling branches are exercised
    for o in range(sim.store.n_owners):
        if sim.store.owner_kind[o] == 0:
            sim.store.lin_vel[o] = rng.normal(scale=0.05, size=3)
            sim.store.ang_vel[o] = rng.normal(scale=2.0, size=3)
    return sim


def gen_coords():
    rng = np.random.default_rng(3)
    out = {}
    for tag, lo, hi in (("unit", (0, 0, 0), (1, 1, 1)),
                        ("hopper", (-0.13, -0.05, -0.32), (0.13, 0.05, 0.50)),
                        ("skew", (-2.0, 0.5, -1.0), (3.0, 2.5, 0.0))):
        dom = Domain(lo, hi)
        pts = rng.uniform(dom.lo, dom.hi, (5000, 3))
        vox = np.zeros(5000, np.uint64)
        sub = np.zeros((5000, 3), np.uint16)
        bad = K.encode_positions(pts, dom.lo, dom.hi, dom.voxel_edge, vox, sub)
        dec = np.zeros((5000, 3))
        K.decode_positions(vox, sub, dom.lo, dom.voxel_edge, dec)
        out.update({f"{tag}_lo": dom.lo, f"{tag}_hi": dom.hi,
                    f"{tag}_edge": np.float64(dom.voxel_edge), f"{tag}_pts": pts,
                    f"{tag}_vox": vox, f"{tag}_sub": sub, f"{tag}_dec": dec,
                    f"{tag}_bad": np.int64(bad)})
    save("coords", **out)


def sphere_snapshot(centers, radii, owners=None, families=None, mask=None):
    centers = np.asarray(centers, np.float64)
    n = centers.shape[0]
    return B.DetectionSnapshot(
        sph_center=centers, sph_radius=np.asarray(radii, np.float32),
        sph_geom=np.arange(n, dtype=np.int64),
        sph_owner=np.asarray(owners if owners is not None else np.arange(n), np.int64),
        sph_family=np.asarray(families if families is not None else np.zeros(n), np.uint8),
        tri_world=np.zeros((0, 9)), tri_geom=np.zeros(0, np.int64),
        tri_owner=np.zeros(0, np.int64), tri_family=np.zeros(0, np.uint8),
        ana_world=np.zeros((0, 8)), ana_kind=np.zeros(0, np.uint8),
        ana_geom=np.zeros(0, np.int64), ana_owner=np.zeros(0, np.int64),
        ana_family=np.zeros(0, np.uint8),
        mask=mask if mask is not None else np.ones((256, 256), dtype=bool))


def detect_record(snap, margin):
    ca = B.detect_contacts(snap, margin)
    grid = B._grid_for(snap, margin, None)
    rec = snap_arrays(snap)
    rec.update(margin=np.float64(margin), kind=ca.kind, geom_a=ca.geom_a,
               geom_b=ca.geom_b)
    if grid is not None and snap.sph_center.shape[0]:
        glo, inv_bin, nb = grid
        ranges = np.zeros((snap.sph_center.shape[0], 6), np.int64)
        K.bin_ranges(snap.sph_center, snap.sph_radius, margin, glo, inv_bin, nb, ranges)
        rec.update(glo=glo, inv_bin=np.float64(inv_bin), nb=nb, ranges=ranges)
    return rec


def gen_detect():
    rng = np.random.default_rng(11)
    centers = rng.uniform(0, 1, (500, 3))
    radii = rng.uniform(0.01, 0.05, 500)
    save("detect_random500", **detect_record(sphere_snapshot(centers, radii), 0.0))

    rng = np.random.default_rng(1234)
    n = 150
    centers = rng.uniform(-0.5, 0.5, (n, 3))
    radii = rng.uniform(0.005, 0.08, n)
    fam = rng.integers(0, 5, n)
    mask = np.ones((256, 256), bool)
    mask[1, 2] = mask[2, 1] = False
    owners = np.arange(n) // 2  # pairs of spheres share an owner
    save("detect_families", **detect_record(
        sphere_snapshot(centers, radii, owners=owners, families=fam, mask=mask), 0.021))

    # straddling registration case of test_broadphase.py:234-244
    save("detect_straddle", **detect_record(
        sphere_snapshot([[0.0, 0, 0], [0.40, 0, 0], [0.45, 0, 0]], [0.08] * 3), 0.0))

    sim = box_scene(n=1500, seed=1, with_mesh=True)
    sim.initialize()
    try:
        sim.do_dynamics(20 * sim.h)
        snap = sim._snapshot()
        save("detect_box_mesh", **detect_record(snap, sim._current_margin() * 15))
    finally:
        sim.close()

    sim = box_scene(n=600, seed=2, clumps=True)
    sim.initialize()
    try:
        sim.do_dynamics(10 * sim.h)
        snap = sim._snapshot()
        save("detect_clumps", **detect_record(snap, sim._current_margin() * 3))
    finally:
        sim.close()


def dyn_record(sim: Simulator) -> dict:
    """Inputs/outputs of one dT step's kernels, captured from a live sim."""
    s = sim.store
    n = s.n_owners
    wang = np.zeros((n, 3))
    K.angular_velocity_global(s.quat[:n], s.ang_vel[:n], wang)
    wild_in = sim._wild.copy()
    wild = sim._wild.copy()
    out_ft = np.zeros((sim._acs.size, 6))
    depth = np.zeros(sim._acs.size)
    cp = np.zeros((sim._acs.size, 3))
    touching = sim._kernel(
        sim._acs_kind, sim._acs_slot_a, sim._acs_slot_b, sim._acs_owner_a,
        sim._acs_owner_b, sim._acs_mat_a, sim._acs_mat_b, sim._sph_centers,
        sim._sph_radius, sim._tri_world, sim._ana_world, sim._ana_kind_arr,
        sim._pos, s.lin_vel[:n], wang, s.mass[:n], sim.pair_stack, wild,
        sim.h, sim.sim_time, out_ft, depth, cp)
    acc_f = np.zeros((n, 3))
    acc_t = np.zeros((n, 3))
    K.reduce_to_owners(sim._acs_owner_a, sim._acs_owner_b, out_ft[:, :3],
                       out_ft[:, 3:], cp, sim._pos, acc_f, acc_t)
    rec = scene_arrays(sim)
    rec.update(
        acs_kind=sim._acs_kind, acs_slot_a=sim._acs_slot_a, acs_slot_b=sim._acs_slot_b,
        acs_owner_a=sim._acs_owner_a, acs_owner_b=sim._acs_owner_b,
        acs_mat_a=sim._acs_mat_a, acs_mat_b=sim._acs_mat_b,
        acs_geom_a=sim._acs.geom_a, acs_geom_b=sim._acs.geom_b,
        sph_geom=sim._sph_geom, sph_centers=sim._sph_centers.copy(),
        sph_radius=sim._sph_radius, tri_world=sim._tri_world.copy(),
        ana_world=sim._ana_world.copy(), ana_kind=sim._ana_kind_arr,
        owner_pos=sim._pos.copy(), ang_vel_global=wang, wild_in=wild_in,
        sim_time=np.float64(sim.sim_time), touching=np.int64(touching),
        out_ft=out_ft, depth=depth, cp=cp, wild_out=wild, acc_f=acc_f, acc_t=acc_t)
    # integrate_and_refresh on copies of the live state
    pos = sim._pos.copy()
    quat = s.quat[:n].copy()
    lv = s.lin_vel[:n].copy()
    av = s.ang_vel[:n].copy()
    vox = s.voxel[:n].copy()
    sub = s.subvoxel[:n].copy()
    cen = sim._sph_centers.copy()
    bad, oob = K.integrate_and_refresh(
        sim.h, sim.gravity[0], sim.gravity[1], sim.gravity[2], pos, quat, lv, av,
        s.mass[:n], s.moi[:n], acc_f, acc_t, s.ext_force[:n], s.ext_torque[:n],
        s.owner_family[:n], sim._fixed_flag, sim._lv_mask, sim._lv_val,
        sim._av_mask, sim._av_val, sim._prescribed_flag, sim.v_err,
        s.domain.lo, s.domain.hi, s.domain.voxel_edge, vox, sub,
        sim._sph_geom, s.geom_params, s.geom_owner, cen)
    rec.update(int_pos=pos, int_quat=quat, int_lin_vel=lv, int_ang_vel=av,
               int_voxel=vox, int_sub=sub, int_centers=cen,
               int_bad=np.int64(bad), int_oob=np.int64(oob))
    return rec


def gen_dynamics():
    for tag, kw, steps in (("box", dict(n=2000, seed=3), 300),
                           ("box_rolling_mesh", dict(n=1200, seed=4, crr=0.05, with_mesh=True), 600),
                           ("clumps", dict(n=500, seed=5, clumps=True, mu=0.5), 200)):
        sim = box_scene(**kw)
        sim.set_fixed_lookahead(4)
        # an external load and a prescribed linear velocity family
        sim.track(3).set_external_force([0.01, -0.02, 0.005])
        sim.track(3).set_external_torque([1e-6, 0.0, -2e-6])
        sim.track(5).set_family(7)
        sim.set_family_prescribed_lin_vel(7, "0.1", "none", "-0.05")
        sim.initialize()
        try:
            sim.do_dynamics(steps * sim.h)
            save(f"dyn_{tag}", **dyn_record(sim))
        finally:
            sim.close()


def gen_merge():
    rng = np.random.default_rng(99)
    out = {}
    for t in range(5):
        def pairs(n):
            raw = rng.integers(0, 300, (n, 2))
            raw = raw[raw[:, 0] != raw[:, 1]]
            raw.sort(axis=1)
            return np.unique(raw, axis=0)
        po, pn = pairs(400), pairs(400)
        # share a fraction of pairs
        pn = np.unique(np.concatenate([pn, po[: 200]]), axis=0)
        old = B.ContactArray(np.zeros(po.shape[0], np.uint8), po[:, 0], po[:, 1])
        for i, name in enumerate(gf.forces.DEFAULT_MODEL.wildcards):
            old.wildcards[name] = rng.normal(size=po.shape[0]).astype(np.float32)
        old = old.canonicalize()
        new = B.ContactArray(np.zeros(pn.shape[0], np.uint8), pn[:, 0], pn[:, 1]).canonicalize()
        merged = B.merge_history(old, new)
        names = gf.forces.DEFAULT_MODEL.wildcards
        out[f"t{t}_old_keys"] = old.sort_keys()
        out[f"t{t}_old_wild"] = np.stack([old.wildcards[n] for n in names], 1)
        out[f"t{t}_new_keys"] = new.sort_keys()
        out[f"t{t}_merged_wild"] = np.stack([merged.wildcards[n] for n in names], 1)
    save("merge", **out)


def gen_trajectory():
    """Sync-mode (n_max = 1) runs are deterministic in the reference, so the
    whole trajectory is a golden vector."""
    for tag, kw, steps in (("box", dict(n=800, seed=6), 150),
                           ("mesh", dict(n=600, seed=7, crr=0.02, with_mesh=True), 120),
                           ("clumps", dict(n=300, seed=8, clumps=True), 120)):
        sim = box_scene(**kw)
        sim.set_sync_mode(True)
        sim.track(2).set_external_force([0.0, 0.003, 0.0])
        init = scene_arrays(sim)
        init["margin"] = np.float64(2.0 * (2.0 * sim.v_err * sim.h * 1) + sim.margin_policy.added)
        sim.initialize()
        try:
            sim.do_dynamics(steps * sim.h)
            s = sim.store
            n = s.n_owners
            rec = {f"init_{k}": v for k, v in init.items()}
            rec.update(steps=np.int64(steps), final_voxel=s.voxel[:n].copy(),
                       final_sub=s.subvoxel[:n].copy(), final_quat=s.quat[:n].copy(),
                       final_lin_vel=s.lin_vel[:n].copy(), final_ang_vel=s.ang_vel[:n].copy(),
                       final_acc_force=s.acc_force[:n].copy(),
                       final_acc_torque=s.acc_torque[:n].copy(),
                       final_wild=sim._wild.copy(), final_kind=sim._acs.kind,
                       final_geom_a=sim._acs.geom_a, final_geom_b=sim._acs.geom_b,
                       final_touching=np.int64(sim._last_touching))
            save(f"traj_{tag}", **rec)
        finally:
            sim.close()


if __name__ == "__main__":
    gen_coords()
    gen_detect()
    gen_dynamics()
    gen_merge()
    gen_trajectory()
