"""The benched throughput build (fp32 velocities, k_contacts_ss: fp64 centre
difference and R^2 - d^2, fp32 contact law, int64 fixed-point owner sums)
against the oracle, per SURVEY.md §8(c) protocol leg 2:

  * per step, from an identical state + contact array + history: touching
    count exact; updated history rows within rel 1e-5 (of the row's own
    magnitude, floor 1e-5 of the median touching row); per-owner force and
    torque within 1e-5 x the median touching force (x the largest radius for
    torque); post-step velocities within 1e-5 of the step's velocity change
    plus fp32 storage rounding; positions within a few sub-voxel quanta;
  * short multi-step trajectories (fp64 oracle vs fp32 GPU) from identical
    states, including the exact C1 10k box and a window of the settled
    1M-sphere crater bed of configs[1] (BASELINE size) continued from its
    settled contact history (installed through gf_set_acs on the GPU side);
  * the fp64 parity build bit-exact on the C1 10k box.

The oracle is fed the fp32-rounded velocities so both start identical.
"""

import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import _bulk as BK
from tests import _scene as S

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
EPS32 = float(np.finfo(np.float32).eps)

# tolerances (north star: "per-step forces within a stated relative tolerance,
# e.g. 1e-5 fp32")
REL = 1e-5
POS_QUANTA = 4          # sub-voxel quanta per step of position drift allowed


def load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


def scene_of(g, prefix=""):
    return {k[len(prefix):]: (v if v.ndim else v[()]) for k, v in g.items() if k.startswith(prefix)}


def f32_rounded(scene):
    s = dict(scene)
    s["lin_vel"] = scene["lin_vel"].astype(np.float32).astype(np.float64)
    s["ang_vel"] = scene["ang_vel"].astype(np.float32).astype(np.float64)
    return s


def positions(st, scene):
    return O.decode_positions(st["voxel"], st["subvoxel"], scene["lo"], scene["edge"])


def owner_scales(scene):
    """Per owner: mass, smallest principal moment and reach (largest
    |offset| + radius of its spheres)."""
    n = scene["voxel"].shape[0]
    sph = scene["geom_kind"] == 0
    gp = scene["geom_params"][sph].astype(np.float64)
    reach = np.zeros(n)
    np.maximum.at(reach, scene["geom_owner"][sph], np.linalg.norm(gp[:, :3], axis=1) + gp[:, 3])
    return scene["mass"], scene["moi"].min(axis=1), reach


def check_state(out, ref, scene, v0, w0, steps=1, label="", fmed=None, crr=0.0):
    """GPU fp32 state `out` vs the oracle's fp64 state `ref` (dicts of
    voxel/subvoxel/lin_vel/ang_vel) after `steps` steps from velocities
    v0 / w0.

    Tolerance: the force criterion carried through the integrator.  Contact
    forces agree to REL x the median touching force F (north star: 1e-5);
    an owner's net force is a sum of its contacts' and can cancel to far
    below F (a resting grain), so its velocity error is bounded by
    REL x steps x h x F / m (linear) and REL x steps x h x F x reach / I
    (angular), plus the fp32 storage rounding of the velocities.  The
    stricter ratio to the owner's own velocity change is reported too.

    With rolling resistance (C_rr > 0) the reference's rolling torque is
    C_rr |F_n| along v_rot / |v_rot|, v_rot = w_B x r_B - w_A x r_A
    (forces.py:132-150): a unit vector of a difference that nearly cancels
    for a grain rolling without slip, switched on and off by a time gate and
    a 1e-12 m/s floor.  Over a multi-step window the fp32 / fp64 rounding of
    the inputs turns it for a few owners by much more than 1e-5: there 99.9 %
    of the owners must meet the force bound and every owner the rolling
    torque's own scale, 2 C_rr x the force bound / REL."""
    quantum = float(scene["edge"]) / 65536.0
    h = float(scene["h"])
    dp = np.abs(positions(out, scene) - positions(ref, scene)).max()
    res = {"dp_quanta": dp / quantum}
    m, imin, reach = owner_scales(scene)
    free = ~scene["fixed_flag"].astype(bool)[scene["owner_family"]]
    for key, start, scale in (("lin_vel", v0, 1.0 / m), ("ang_vel", w0, reach / imin)):
        r = ref[key]
        own = np.linalg.norm(r - start, axis=1)
        med = float(np.median(own[own > 0])) if np.any(own > 0) else 1.0
        err = np.maximum(np.linalg.norm(out[key] - r, axis=1) - 4 * steps * EPS32 * np.linalg.norm(r, axis=1), 0.0)
        ratio = err / np.maximum(own, med)
        res[key] = {"own_change_max": float(ratio.max()), "own_change_p99": float(np.quantile(ratio, 0.99))}
        if fmed is not None:
            bound = REL * steps * h * fmed * scale
            fr = np.where(free & (err > 0), err / np.maximum(bound, 1e-300), 0.0)
            res[key]["force_scale_max"] = float(fr.max())
            res[key]["force_scale_p999"] = float(np.quantile(fr[free], 0.999))
            res[key]["worst_owner"] = int(fr.argmax())
    print(label, res)
    for key in ("lin_vel", "ang_vel"):
        if fmed is None:
            assert res[key]["own_change_max"] <= REL, (label, key, res[key])
        elif crr > 0.0 and key == "ang_vel":
            assert res[key]["force_scale_p999"] <= 1.0, (label, key, res[key])
            assert res[key]["force_scale_max"] <= 2.0 * crr / REL, (label, key, res[key])
        else:
            assert res[key]["force_scale_max"] <= 1.0, (label, key, res[key])
    # positions: quantisation of each step plus h x the velocity error
    assert dp <= POS_QUANTA * steps * quantum + steps * h * np.abs(
        out["lin_vel"] - ref["lin_vel"]).max() + 1e-300, (label, res)
    return res


def per_step_case(scene, g):
    """One fp32 step on the GPU vs the oracle from the golden (state, ACS,
    history)."""
    scene = f32_rounded(scene)
    ctx = S.upload_scene(scene, f32_state=True)
    S.set_acs(ctx, g["acs_kind"], g["acs_slot_a"], g["acs_slot_b"], g["wild_in"])
    touching, bad, oob = S.dt_step(ctx, scene, float(g["sim_time"]))
    assert (bad, oob) == (-1, -1)
    out = S.download_state(ctx, g["voxel"].shape[0])
    _, _, _, wild_gpu = S.get_acs(ctx)
    ctx.close()

    wang = O.angular_velocity_global(scene["quat"], scene["ang_vel"])
    wild = np.ascontiguousarray(g["wild_in"], np.float32).copy()
    tch, out_ft, depth, cp = O.contact_forces(
        g["acs_kind"], g["acs_slot_a"], g["acs_slot_b"], g["acs_owner_a"], g["acs_owner_b"],
        g["acs_mat_a"], g["acs_mat_b"], g["sph_centers"], g["sph_radius"], g["tri_world"],
        g["ana_world"], g["ana_kind"], g["owner_pos"], scene["lin_vel"], wang, scene["mass"],
        scene["pair_stack"], wild, float(scene["h"]), float(g["sim_time"]))
    acc_f, acc_t = O.reduce_to_owners(g["acs_owner_a"], g["acs_owner_b"], out_ft, cp, g["owner_pos"])
    assert touching == tch

    # history: every row the oracle updated (touching), rel 1e-5 of its norm
    t = depth > 0
    assert np.array_equal(wild_gpu[~t], wild[~t]), "false positives must leave history untouched"
    if t.any():
        ref_rows = wild[t].astype(np.float64)
        got = wild_gpu[t].astype(np.float64)
        # tangential displacement (xyz) and delta_time (w) separately
        dnorm = np.linalg.norm(ref_rows[:, :3], axis=1)
        # normalised like the forces: by the row's own norm, floored at the
        # median touching row (fp32 cancellation in the projection makes
        # rows much smaller than typical ill-conditioned)
        floor = np.median(dnorm) if np.median(dnorm) > 0 else 1.0
        derr = np.linalg.norm(got[:, :3] - ref_rows[:, :3], axis=1)
        ratio = derr / (REL * np.maximum(dnorm, floor))
        assert ratio.max() <= 1.0, (float(ratio.max()), float(dnorm[ratio.argmax()]), float(floor))
        np.testing.assert_allclose(got[:, 3], ref_rows[:, 3], rtol=2 * EPS32)
        print(f"history: worst error {ratio.max() * REL:.2e} of max(|row|, median |row|)")

    fscale = np.median(np.linalg.norm(out_ft[t, :3], axis=1)) if t.any() else 1.0
    assert np.max(np.abs(out["acc_f"] - acc_f)) <= REL * fscale + 1e-12
    tscale = fscale * float(np.max(g["sph_radius"]))
    assert np.max(np.abs(out["acc_t"] - acc_t)) <= REL * tscale + 1e-15

    # post-step state: the oracle's integrator on the oracle's sums
    ref = {k: np.array(scene[k], copy=True) for k in ("voxel", "subvoxel", "quat", "lin_vel", "ang_vel")}
    pos = np.ascontiguousarray(g["owner_pos"], np.float64).copy()
    sph = np.nonzero(scene["geom_kind"] == 0)[0].astype(np.int64)
    centers = np.ascontiguousarray(g["sph_centers"], np.float64).copy()
    bad, oob = O.integrate_and_refresh(
        scene["h"], scene["gravity"], pos, ref["quat"], ref["lin_vel"], ref["ang_vel"], scene["mass"],
        scene["moi"], acc_f, acc_t, scene["ext_force"], scene["ext_torque"], scene["owner_family"],
        scene["fixed_flag"], scene["lv_mask"], scene["lv_val"], scene["av_mask"], scene["av_val"],
        scene["prescribed_flag"], scene["v_err"], scene["lo"], scene["hi"], scene["edge"], ref["voxel"],
        ref["subvoxel"], sph, scene["geom_params"], scene["geom_owner"], centers)
    assert (bad, oob) == (-1, -1)
    # velocity change of this step is dominated by gravity + contact forces;
    # the contact part must agree to 1e-5 of itself: compare against the
    # force-only velocity change
    return check_state(out, ref, scene, scene["lin_vel"], scene["ang_vel"], label="per-step")


@pytest.mark.parametrize("name", ["dyn_box", "dyn_box_rolling_mesh", "dyn_clumps"])
def test_f32_step_history_and_state(name):
    g = load(name)
    per_step_case(scene_of(g), g)


def run_both(scene, steps, margin, period=1, lag=0, nthreads=1, f32=True):
    """`steps` steps of the GPU build and the oracle stepper from the same
    (fp32-rounded if f32) state with zero history."""
    sc = f32_rounded(scene) if f32 else scene
    ref = O.OracleStepper(sc, margin, period=period, lag=lag, nthreads=nthreads)
    for _ in range(steps):
        ref.step_once()
    ctx = S.upload_scene(sc, f32_state=f32)
    rr = S.run(ctx, sc, steps, margin, period=period, lag=lag)
    out = S.download_state(ctx, sc["voxel"].shape[0])
    kind, sa, sb, wild = S.get_acs(ctx)
    ctx.close()
    assert rr.bad_owner == -1 and rr.oob_owner == -1
    return sc, ref, out, rr, (kind, sa, sb, wild)


@pytest.mark.parametrize("name", ["traj_box", "traj_clumps"])
def test_f32_short_trajectory_vs_oracle(name):
    """20 sync steps of the fp32 build against the fp64 oracle stepper: the
    fp32 contact law and velocity storage stay within tolerance over a
    trajectory, not just one step."""
    g = load(name)
    scene = scene_of(g, "init_")
    steps = 20
    sc, ref, out, rr, _ = run_both(scene, steps, float(scene["margin"]))
    assert rr.touching == ref.last_touching
    check_state(out, ref.s, sc, sc["lin_vel"], sc["ang_vel"], steps=steps, label=name,
                fmed=ref.last_force_median)


# ---------------------------------------------------------------------------
# configs[0] (C1): the exact 10k monodisperse settling box
# ---------------------------------------------------------------------------

def c1_settled_scene(steps=6000):
    """The C1 box (tests/_bulk.py c1_box, exactly 10,000 spheres) after
    `steps` steps of the fp64 build (the lattice has fallen onto the floor
    and the lower layers are in contact), as an oracle scene dict."""
    import paper_2311_04648_b200 as gf
    from paper_2311_04648_b200 import scenes
    sim = BK.c1_box(gf, precision="f64")
    sim.initialize()
    sim.do_dynamics(steps * sim.h)
    scene = scenes.oracle_scene(sim)
    margin = sim._current_margin()
    sim.close()
    return scene, margin


@pytest.fixture(scope="module")
def c1_scene():
    return c1_settled_scene()


def test_c1_10k_fp64_bit_exact(c1_scene):
    scene, margin = c1_scene
    assert scene["voxel"].shape[0] == 10_000 + 1   # + the wall owner
    sc, ref, out, rr, (kind, sa, sb, wild) = run_both(scene, 5, margin, f32=False, nthreads=8)
    assert rr.touching == ref.last_touching and rr.touching > 1000
    for key in ("voxel", "subvoxel", "quat", "lin_vel", "ang_vel"):
        assert np.array_equal(out[key], ref.s[key]), key
    assert np.array_equal(wild, ref.wild)


def test_c1_10k_fp32_within_tolerance(c1_scene):
    scene, margin = c1_scene
    steps = 8
    sc, ref, out, rr, _ = run_both(scene, steps, margin, period=2, lag=2, nthreads=8)
    assert rr.touching == ref.last_touching
    check_state(out, ref.s, sc, sc["lin_vel"], sc["ang_vel"], steps=steps, label="c1",
                fmed=ref.last_force_median)


# ---------------------------------------------------------------------------
# configs[1] at BASELINE size: a window of the settled 1M-sphere crater bed
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n,crr", [(20_000, 0.01), (20_000, 0.0),
                                   pytest.param(1_000_000, 0.01, marks=pytest.mark.slow),
                                   pytest.param(1_000_000, 0.0, marks=pytest.mark.slow)])
def test_crater_window_vs_oracle(n, crr):
    """The settled 1M-sphere crater bed (bench.py's workload): three steps of
    the benched schedule (period 2, lag 2) from an identical fixed-point
    state AND the settled contact history (the Simulator's contact array,
    installed on both sides), the fp32 GPU build vs the OpenMP oracle.
    Starting from the settled history matters: with zero history every
    contact crosses the rolling-resistance collision-time gate
    (forces.py:132-143, a discontinuity) within the window, and fp32 vs fp64
    rounding of the gate decides a few of them differently."""
    from paper_2311_04648_b200 import scenes
    sim = scenes.crater_bed(n, hold_ball=True, extra_props={"Crr": crr})
    sim.initialize()
    sim.do_dynamics(12000 * sim.h)
    scenes.release_balls(sim)
    sim.do_dynamics(20 * sim.h)
    scene = scenes.oracle_scene(sim)
    ca = sim._acs
    margin = sim._current_margin()
    period, lag = sim._schedule()
    sim.close()
    wild = np.stack([ca.wildcards[k] for k in ("delta_tan_x", "delta_tan_y", "delta_tan_z", "delta_time")],
                    axis=1).astype(np.float32)
    assert np.count_nonzero(wild[:, 3]) > n   # a settled history, not zeros
    sc = f32_rounded(scene)
    steps = 3
    nthreads = os.cpu_count() or 1
    ref = O.OracleStepper(sc, margin, period=period, lag=lag, nthreads=nthreads)
    ref.keys = O.sort_keys(ca.kind, ca.geom_a, ca.geom_b)
    ref.wild = wild.copy()
    ref.acs = dict(kind=ca.kind.copy(), geom_a=ca.geom_a.copy(), geom_b=ca.geom_b.copy())
    for _ in range(steps):
        ref.step_once()
    ctx = S.upload_scene(sc, f32_state=True)
    _, _, _, slot = S.slots(sc)
    S.set_acs(ctx, ca.kind, slot[ca.geom_a], slot[ca.geom_b], wild)
    rr = S.run(ctx, sc, steps, margin, period=period, lag=lag)
    out = S.download_state(ctx, sc["voxel"].shape[0])
    ctx.close()
    assert rr.bad_owner == -1 and rr.oob_owner == -1
    assert rr.touching == ref.last_touching
    assert rr.touching > n
    check_state(out, ref.s, sc, sc["lin_vel"], sc["ang_vel"], steps=steps, label=f"crater {n} crr {crr}",
                fmed=ref.last_force_median, crr=crr)


# ---------------------------------------------------------------------------
# the fused kernel's TMA gather4 variant (GF_SS_TMA=1) reads the same centre
# records through the TMA unit: bitwise the same trajectory
# ---------------------------------------------------------------------------

def test_tma_gather_variant_bit_identical(c1_scene, monkeypatch):
    scene, margin = c1_scene
    sc = f32_rounded(scene)
    steps = 12
    runs = []
    for tma in ("0", "1"):
        monkeypatch.setenv("GF_SS_TMA", tma)   # read when the context is created
        ctx = S.upload_scene(sc, f32_state=True)
        rr = S.run(ctx, sc, steps, margin, period=2, lag=2)
        out = S.download_state(ctx, sc["voxel"].shape[0])
        kind, sa, sb, wild = S.get_acs(ctx)
        ctx.close()
        assert rr.bad_owner == -1 and rr.touching > 1000
        runs.append((rr.touching, out, wild))
    assert runs[0][0] == runs[1][0]
    for key in ("voxel", "subvoxel", "quat", "lin_vel", "ang_vel"):
        assert np.array_equal(runs[0][1][key], runs[1][1][key]), key
    assert np.array_equal(runs[0][2], runs[1][2])
