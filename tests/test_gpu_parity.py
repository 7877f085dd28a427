"""CUDA path vs the oracle / reference golden vectors (needs a B200).

Parity bar:
  * kT pair lists and bin ranges: bit-exact;
  * dT in the fp64-velocity build: bit-exact per step for every clump owner
    (state, history, touching count, accumulators); boundary owners with more
    than kHeavyThreshold incidences are block-reduced in a different summation
    order, so their accumulators are compared at rel 1e-12;
  * dT in the fp32-velocity build: per-step forces / state within rel 1e-5 of
    the oracle fed the same (fp32-rounded) state;
  * whole sync-mode trajectories: bit-exact against the reference Simulator.
"""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2311_04648_b200 import broadphase as B
from tests import _scene as S

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


def scene_of(g, prefix=""):
    return {k[len(prefix):]: (v if v.ndim else v[()]) for k, v in g.items() if k.startswith(prefix)}


def snapshot_of(g):
    d = {k[5:]: v for k, v in g.items() if k.startswith("snap_")}
    return B.DetectionSnapshot(**d)


@pytest.mark.parametrize("name", ["detect_random500", "detect_families", "detect_straddle",
                                  "detect_box_mesh", "detect_clumps"])
def test_detect_bit_exact(name):
    g = load(name)
    ca = B.detect_contacts(snapshot_of(g), float(g["margin"]))
    assert np.array_equal(ca.kind, g["kind"])
    assert np.array_equal(ca.geom_a, g["geom_a"])
    assert np.array_equal(ca.geom_b, g["geom_b"])
    kind, sa, sb, glo, inv_bin, nb = B.detect_contacts_raw(snapshot_of(g), float(g["margin"]))
    if "glo" in g:
        assert np.array_equal(glo, g["glo"])
        assert inv_bin == float(g["inv_bin"])
        assert np.array_equal(nb, g["nb"])
        ctx = B._util_ctx(0)
        out = np.zeros((g["snap_sph_center"].shape[0], 6), np.int64)
        ctx.call("gf_bin_ranges", S.C.c_double(float(g["margin"])), S.P(out))
        assert np.array_equal(out, g["ranges"])


def test_detect_random_vs_oracle_many():
    """Property sweep in the style of test_broadphase.py:109-125: random
    snapshots, margins, families and masks -> device == oracle, bit-exact."""
    for seed in range(25):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(2, 400))
        centers = rng.uniform(-0.5, 0.5, (n, 3))
        radii = rng.uniform(0.005, 0.08, n).astype(np.float32)
        margin = float(rng.uniform(0.0, 0.03))
        fam = rng.integers(0, 5, n).astype(np.uint8)
        owners = rng.integers(0, max(1, n // 2), n)
        mask = np.ones((256, 256), bool)
        mask[1, 2] = mask[2, 1] = False
        ana = np.array([[0, 0, -0.45, 0, 0, 1, 0, 0], [0.1, 0, 0, 0, 0, 1, 0.3, -1.0]])
        snap = dict(sph_center=centers, sph_radius=radii, sph_geom=np.arange(n), sph_owner=owners,
                    sph_family=fam, tri_world=np.zeros((0, 9)), tri_geom=np.zeros(0, np.int64),
                    tri_owner=np.zeros(0, np.int64), tri_family=np.zeros(0, np.uint8),
                    ana_world=ana, ana_kind=np.array([2, 3], np.uint8),
                    ana_geom=np.array([n, n + 1]), ana_owner=np.array([10 ** 6, 10 ** 6]),
                    ana_family=np.array([3, 4], np.uint8), mask=mask)
        want = O.detect_contacts(snap, margin)
        got = B.detect_contacts(B.DetectionSnapshot(**snap), margin)
        assert np.array_equal(got.kind, want["kind"]), seed
        assert np.array_equal(got.geom_a, want["geom_a"]), seed
        assert np.array_equal(got.geom_b, want["geom_b"]), seed


def test_detect_empty_world():
    snap = B.DetectionSnapshot(
        sph_center=np.zeros((0, 3)), sph_radius=np.zeros(0, np.float32), sph_geom=np.zeros(0, np.int64),
        sph_owner=np.zeros(0, np.int64), sph_family=np.zeros(0, np.uint8), tri_world=np.zeros((0, 9)),
        tri_geom=np.zeros(0, np.int64), tri_owner=np.zeros(0, np.int64), tri_family=np.zeros(0, np.uint8),
        ana_world=np.zeros((0, 8)), ana_kind=np.zeros(0, np.uint8), ana_geom=np.zeros(0, np.int64),
        ana_owner=np.zeros(0, np.int64), ana_family=np.zeros(0, np.uint8),
        mask=np.ones((256, 256), bool))
    assert B.detect_contacts(snap, 0.01).size == 0


def test_merge_history_bit_exact():
    g = load("merge")
    for t in range(5):
        ok, nk = g[f"t{t}_old_keys"], g[f"t{t}_new_keys"]
        def unpack(keys):
            keys = keys.astype(np.uint64)
            return ((keys >> np.uint64(48)).astype(np.uint8),
                    ((keys >> np.uint64(24)) & np.uint64(0xFFFFFF)).astype(np.int64),
                    (keys & np.uint64(0xFFFFFF)).astype(np.int64))
        k0, a0, b0 = unpack(ok)
        k1, a1, b1 = unpack(nk)
        names = ("delta_tan_x", "delta_tan_y", "delta_tan_z", "delta_time")
        old = B.ContactArray(k0, a0, b0, {n: g[f"t{t}_old_wild"][:, i] for i, n in enumerate(names)})
        new = B.ContactArray(k1, a1, b1)
        merged = B.merge_history(old, new)
        got = np.stack([merged.wildcards[n] for n in names], 1)
        assert np.array_equal(got, g[f"t{t}_merged_wild"])


def _heavy_owners(g, threshold=192):
    n = g["voxel"].shape[0]
    inc = np.bincount(np.concatenate([g["acs_owner_a"], g["acs_owner_b"]]), minlength=n)
    return inc > threshold


@pytest.mark.parametrize("name", ["dyn_box", "dyn_box_rolling_mesh", "dyn_clumps"])
def test_dt_step_f64_bit_exact(name):
    g = load(name)
    scene = scene_of(g)
    ctx = S.upload_scene(scene)
    S.set_acs(ctx, g["acs_kind"], g["acs_slot_a"], g["acs_slot_b"], g["wild_in"])
    touching, bad, oob = S.dt_step(ctx, scene, float(g["sim_time"]))
    assert (bad, oob) == (int(g["int_bad"]), int(g["int_oob"]))
    assert touching == int(g["touching"])
    _, _, _, wild = S.get_acs(ctx)
    rolling = np.any(g["out_ft"][:, 3:] != 0.0, axis=1)
    # pow(r_eff, 0.25) in the rolling gate is the only libm call left on the
    # device; history rows are bit-exact everywhere else
    assert np.array_equal(wild[~rolling], g["wild_out"][~rolling])
    np.testing.assert_allclose(wild, g["wild_out"], rtol=1e-6, atol=1e-12)
    st = S.download_state(ctx, g["voxel"].shape[0])
    heavy = _heavy_owners(g)
    light = ~heavy
    for key, ref in (("acc_f", "acc_f"), ("acc_t", "acc_t")):
        assert np.array_equal(st[key][light], g[ref][light]), key
        np.testing.assert_allclose(st[key][heavy], g[ref][heavy], rtol=1e-12, atol=1e-15)
    if not rolling.any():
        for key, ref in (("voxel", "int_voxel"), ("subvoxel", "int_sub"), ("quat", "int_quat"),
                         ("lin_vel", "int_lin_vel"), ("ang_vel", "int_ang_vel")):
            assert np.array_equal(st[key], g[ref]), key
    else:
        np.testing.assert_allclose(st["lin_vel"], g["int_lin_vel"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(st["ang_vel"], g["int_ang_vel"], rtol=1e-9, atol=1e-9)
    ctx.close()


@pytest.mark.parametrize("name", ["dyn_box", "dyn_box_rolling_mesh", "dyn_clumps"])
def test_dt_step_f32_within_tolerance(name):
    """Throughput build: velocities stored as float32.  Compare with the
    oracle fed the same float32-rounded velocities; forces within rel 1e-5 of
    the median touching force (SURVEY.md 8(c) protocol)."""
    g = load(name)
    scene = scene_of(g)
    scene["lin_vel"] = scene["lin_vel"].astype(np.float32).astype(np.float64)
    scene["ang_vel"] = scene["ang_vel"].astype(np.float32).astype(np.float64)
    ctx = S.upload_scene(scene, f32_state=True)
    S.set_acs(ctx, g["acs_kind"], g["acs_slot_a"], g["acs_slot_b"], g["wild_in"])
    touching, bad, oob = S.dt_step(ctx, scene, float(g["sim_time"]))
    st = S.download_state(ctx, g["voxel"].shape[0])
    wang = O.angular_velocity_global(scene["quat"], scene["ang_vel"])
    wild = g["wild_in"].copy()
    tch, out_ft, depth, cp = O.contact_forces(
        g["acs_kind"], g["acs_slot_a"], g["acs_slot_b"], g["acs_owner_a"], g["acs_owner_b"],
        g["acs_mat_a"], g["acs_mat_b"], g["sph_centers"], g["sph_radius"], g["tri_world"],
        g["ana_world"], g["ana_kind"], g["owner_pos"], scene["lin_vel"], wang, scene["mass"],
        scene["pair_stack"], wild, float(scene["h"]), float(g["sim_time"]))
    acc_f, acc_t = O.reduce_to_owners(g["acs_owner_a"], g["acs_owner_b"], out_ft, cp, g["owner_pos"])
    assert touching == tch
    fscale = np.median(np.linalg.norm(out_ft[depth > 0, :3], axis=1)) if (depth > 0).any() else 1.0
    assert np.max(np.abs(st["acc_f"] - acc_f)) <= 1e-5 * fscale + 1e-12
    tscale = fscale * float(np.max(g["sph_radius"]))
    assert np.max(np.abs(st["acc_t"] - acc_t)) <= 1e-5 * tscale + 1e-15
    ctx.close()


@pytest.mark.parametrize("name", ["traj_box", "traj_mesh", "traj_clumps"])
def test_sync_trajectory_bit_exact(name):
    """gf_run in sync mode replays the reference Simulator's trajectory."""
    g = load(name)
    scene = scene_of(g, "init_")
    ctx = S.upload_scene(scene)
    rr = S.run(ctx, scene, int(g["steps"]), float(scene["margin"]), period=1, lag=0)
    assert rr.bad_owner == -1 and rr.oob_owner == -1
    n = scene["voxel"].shape[0]
    st = S.download_state(ctx, n)
    kind, sa, sb, wild = S.get_acs(ctx)
    sph, tri, ana, _ = S.slots(scene)
    tabs = (sph, tri, ana)
    ga = sph[sa]
    gb = np.array([tabs[k][b] for k, b in zip(kind, sb)], np.int64)
    assert np.array_equal(ga, g["final_geom_a"])
    assert np.array_equal(gb, g["final_geom_b"])
    assert rr.touching == int(g["final_touching"])
    crr = float(np.max(scene["pair_stack"][4]))
    if crr == 0.0:
        for key, ref in (("voxel", "final_voxel"), ("subvoxel", "final_sub"), ("quat", "final_quat"),
                         ("lin_vel", "final_lin_vel"), ("ang_vel", "final_ang_vel")):
            assert np.array_equal(st[key], g[ref]), key
        assert np.array_equal(wild, g["final_wild"])
    else:
        np.testing.assert_allclose(st["lin_vel"], g["final_lin_vel"], rtol=1e-6, atol=1e-9)
    ctx.close()


def test_async_schedule_matches_oracle_stepper():
    """The deterministic async schedule (snapshot every `period`, adopt `lag`
    later) against the oracle driver running the same schedule."""
    g = load("traj_box")
    scene = scene_of(g, "init_")
    margin = O.margin_for(float(scene["v_err"]), float(scene["h"]), 4)
    st = O.OracleStepper(scene, margin, period=2, lag=2)
    for _ in range(60):
        st.step_once()
    ctx = S.upload_scene(scene)
    rr = S.run(ctx, scene, 60, margin, period=2, lag=2)
    out = S.download_state(ctx, scene["voxel"].shape[0])
    assert np.array_equal(out["voxel"], st.s["voxel"])
    assert np.array_equal(out["subvoxel"], st.s["subvoxel"])
    assert np.array_equal(out["lin_vel"], st.s["lin_vel"])
    assert rr.touching == st.last_touching
    ctx.close()


def test_detect_polydisperse_with_big_spheres_vs_oracle():
    """Spheres far above 2x the median radius take the k_big path; the pair
    list must still equal the reference's (oracle) bit for bit."""
    for seed in range(6):
        rng = np.random.default_rng(100 + seed)
        n = 3000
        centers = rng.uniform(-0.3, 0.3, (n, 3))
        radii = rng.uniform(0.008, 0.012, n)
        big = rng.choice(n, 12, replace=False)
        radii[big] = rng.uniform(0.03, 0.09, big.size)
        radii = radii.astype(np.float32)
        margin = float(rng.uniform(0.0, 0.004))
        owners = np.arange(n)
        owners[1::7] = owners[0::7][: owners[1::7].size]  # some clump-mates
        tri = rng.uniform(-0.3, 0.3, (40, 9))
        snap = dict(sph_center=centers, sph_radius=radii, sph_geom=np.arange(n), sph_owner=owners,
                    sph_family=np.zeros(n, np.uint8), tri_world=tri, tri_geom=np.arange(n, n + 40),
                    tri_owner=np.full(40, 10 ** 7), tri_family=np.zeros(40, np.uint8),
                    ana_world=np.zeros((0, 8)), ana_kind=np.zeros(0, np.uint8),
                    ana_geom=np.zeros(0, np.int64), ana_owner=np.zeros(0, np.int64),
                    ana_family=np.zeros(0, np.uint8), mask=np.ones((256, 256), bool))
        want = O.detect_contacts(snap, margin)
        got = B.detect_contacts(B.DetectionSnapshot(**snap), margin)
        assert np.array_equal(got.kind, want["kind"]), seed
        assert np.array_equal(got.geom_a, want["geom_a"]), seed
        assert np.array_equal(got.geom_b, want["geom_b"]), seed


# ---------------------------------------------------------------------------
# NVRTC user force models (forces.py:360-440 plugin contract)
# ---------------------------------------------------------------------------

def _with_coh(scene, coh=2.0e3):
    s = dict(scene)
    ps = s["pair_stack"]
    s["pair_stack"] = np.concatenate([ps, np.full((1,) + ps.shape[1:], coh)], axis=0)
    return s


def _set_model(ctx, src, W=4):
    import ctypes as C
    from paper_2311_04648_b200 import _lib
    log = C.create_string_buffer(1 << 16)
    ctx.call("gf_set_force_model", src.encode(), _lib.CSRC_DIR.encode(), C.c_int(W), log,
             C.c_size_t(1 << 16))


HM_AS_USER = r"""
__device__ void user_core(double overlap, double ts, double sim_time, double b2ax, double b2ay,
                          double b2az, double vx, double vy, double vz, double wrx, double wry,
                          double wrz, double mass_eff, double ra, double rb, int mat_a, int mat_b,
                          const double *pair, int n_mat, float *wild, double *out) {
  gf::hm_default_core(overlap, ts, sim_time, b2ax, b2ay, b2az, vx, vy, vz, wrx, wry, wrz, mass_eff,
                      ra, rb, mat_a, mat_b, pair, n_mat, wild, out);
}
"""


@pytest.mark.parametrize("name", ["dyn_box", "dyn_clumps"])
def test_user_model_equal_to_builtin(name):
    """A user model that is the default law, compiled by NVRTC, reproduces the
    built-in kernel (beta from the device log instead of the host table)."""
    g = load(name)
    scene = scene_of(g)
    outs = []
    for user in (False, True):
        ctx = S.upload_scene(scene)
        if user:
            _set_model(ctx, HM_AS_USER)
        S.set_acs(ctx, g["acs_kind"], g["acs_slot_a"], g["acs_slot_b"], g["wild_in"])
        touching, bad, oob = S.dt_step(ctx, scene, float(g["sim_time"]))
        st = S.download_state(ctx, g["voxel"].shape[0])
        outs.append((touching, st, S.get_acs(ctx)[3]))
        ctx.close()
    assert outs[0][0] == outs[1][0]
    for key in ("acc_f", "acc_t", "lin_vel", "ang_vel"):
        ref = outs[0][1][key]
        np.testing.assert_allclose(outs[1][1][key], ref, rtol=1e-12, atol=1e-12 * np.max(np.abs(ref)))
    np.testing.assert_allclose(outs[1][2], outs[0][2], rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("f32", [False, True])
def test_cohesive_user_model_vs_oracle(f32):
    """configs[3]'s cohesive contact model: NVRTC-compiled CUDA source vs the
    oracle twin (oracle/gf_oracle.c model 1) on the same state."""
    from paper_2311_04648_b200 import models
    g = load("dyn_box")
    scene = _with_coh(scene_of(g))
    if f32:
        scene["lin_vel"] = scene["lin_vel"].astype(np.float32).astype(np.float64)
        scene["ang_vel"] = scene["ang_vel"].astype(np.float32).astype(np.float64)
    ctx = S.upload_scene(scene, f32_state=f32)
    _set_model(ctx, models.COHESIVE_SRC)
    S.set_acs(ctx, g["acs_kind"], g["acs_slot_a"], g["acs_slot_b"], g["wild_in"])
    touching, bad, oob = S.dt_step(ctx, scene, float(g["sim_time"]))
    st = S.download_state(ctx, g["voxel"].shape[0])
    ctx.close()
    wang = O.angular_velocity_global(scene["quat"], scene["ang_vel"])
    wild = g["wild_in"].copy()
    tch, out_ft, depth, cp = O.contact_forces(
        g["acs_kind"], g["acs_slot_a"], g["acs_slot_b"], g["acs_owner_a"], g["acs_owner_b"],
        g["acs_mat_a"], g["acs_mat_b"], g["sph_centers"], g["sph_radius"], g["tri_world"],
        g["ana_world"], g["ana_kind"], g["owner_pos"], scene["lin_vel"], wang, scene["mass"],
        scene["pair_stack"], wild, float(scene["h"]), float(g["sim_time"]), model=1)
    acc_f, acc_t = O.reduce_to_owners(g["acs_owner_a"], g["acs_owner_b"], out_ft, cp, g["owner_pos"])
    assert touching == tch
    fscale = np.median(np.linalg.norm(out_ft[depth > 0, :3], axis=1))
    tol = 1e-5 if f32 else 1e-10
    assert np.max(np.abs(st["acc_f"] - acc_f)) <= tol * fscale
    # the cohesive pull is really there: compare with plain Hertz-Mindlin
    wild2 = g["wild_in"].copy()
    _, out_hm, _, _ = O.contact_forces(
        g["acs_kind"], g["acs_slot_a"], g["acs_slot_b"], g["acs_owner_a"], g["acs_owner_b"],
        g["acs_mat_a"], g["acs_mat_b"], g["sph_centers"], g["sph_radius"], g["tri_world"],
        g["ana_world"], g["ana_kind"], g["owner_pos"], scene["lin_vel"], wang, scene["mass"],
        scene["pair_stack"], wild2, float(scene["h"]), float(g["sim_time"]), model=0)
    assert np.max(np.abs(out_ft[:, :3] - out_hm[:, :3])) > 1e3 * tol * fscale


def test_cohesive_model_through_simulator():
    """Simulator(force_model=...) compiles the user model at initialize and
    runs a sync-mode trajectory that matches the oracle driver."""
    import paper_2311_04648_b200 as gf
    from paper_2311_04648_b200 import models, scenes
    models.cohesive_model()
    sim = gf.Simulator(gf.Domain.cube(1.0), force_model="hertz_mindlin_cohesive")
    mat = sim.load_material({"E": 1e7, "nu": 0.3, "CoR": 0.5, "mu": 0.3, "Crr": 0.0, "coh": 5e3})
    tpl = sim.load_clump_template(gf.ClumpTemplate.solid_sphere(0.01, 0.0109, mat))
    sim.add_clumps(tpl, gf.hcp_sample_box((0, 0, 0.06), (0.05, 0.05, 0.05), 0.0199))
    sim.add_analytic([("plane", (0, 0, 0), (0, 0, 1), mat)], family=255)
    sim.set_family_fixed(255)
    sim.set_gravity([0, 0, -9.81])
    sim.set_init_time_step(2e-5)
    sim.set_error_out_velocity(5.0)
    sim.set_sync_mode(True)
    scene = scenes.oracle_scene(sim)
    sim.initialize()
    with sim:
        sim.do_dynamics(100 * sim.h)
        pos = sim._pos.copy()
        v = sim.store.lin_vel[: sim.store.n_owners].copy()
    st = O.OracleStepper(scene, sim._current_margin(), period=1, lag=0, model=1)
    for _ in range(100):
        st.step_once()
    np.testing.assert_allclose(pos, st.pos, atol=1e-12)
    np.testing.assert_allclose(v, st.s["lin_vel"], rtol=1e-8, atol=1e-12)
