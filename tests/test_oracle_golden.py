"""Pin the C oracle to the reference: every oracle function must reproduce the
golden vectors produced by the reference implementation itself
(tests/golden/make_golden.py) BIT FOR BIT.  CPU only."""

import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


def snap_of(g):
    return {k[5:]: v for k, v in g.items() if k.startswith("snap_")}


def test_coords_bitwise():
    g = load("coords")
    for tag in ("unit", "hopper", "skew"):
        vox, sub, bad = O.encode_positions(g[f"{tag}_pts"], g[f"{tag}_lo"], g[f"{tag}_hi"],
                                           float(g[f"{tag}_edge"]))
        assert bad == int(g[f"{tag}_bad"])
        assert np.array_equal(vox, g[f"{tag}_vox"])
        assert np.array_equal(sub, g[f"{tag}_sub"])
        dec = O.decode_positions(vox, sub, g[f"{tag}_lo"], float(g[f"{tag}_edge"]))
        assert np.array_equal(dec, g[f"{tag}_dec"])


@pytest.mark.parametrize("name", ["detect_random500", "detect_families", "detect_straddle",
                                  "detect_box_mesh", "detect_clumps"])
def test_detect_bitwise(name):
    g = load(name)
    res = O.detect_contacts(snap_of(g), float(g["margin"]))
    assert np.array_equal(res["kind"], g["kind"])
    assert np.array_equal(res["geom_a"], g["geom_a"])
    assert np.array_equal(res["geom_b"], g["geom_b"])
    if "glo" in g:
        assert np.array_equal(res["glo"], g["glo"])
        assert res["inv_bin"] == float(g["inv_bin"])
        assert np.array_equal(res["nb"], g["nb"])
        rng = O.bin_ranges(g["snap_sph_center"], g["snap_sph_radius"], float(g["margin"]),
                           g["glo"], float(g["inv_bin"]), g["nb"])
        assert np.array_equal(rng, g["ranges"])


def test_detect_kinds_present():
    g = load("detect_box_mesh")
    kinds = set(np.unique(g["kind"]).tolist())
    assert kinds == {0, 1, 2}, kinds


@pytest.mark.parametrize("name", ["dyn_box", "dyn_box_rolling_mesh", "dyn_clumps"])
def test_contact_reduce_integrate_bitwise(name):
    g = load(name)
    wild = g["wild_in"].copy()
    touching, out_ft, depth, cp = O.contact_forces(
        g["acs_kind"], g["acs_slot_a"], g["acs_slot_b"], g["acs_owner_a"], g["acs_owner_b"],
        g["acs_mat_a"], g["acs_mat_b"], g["sph_centers"], g["sph_radius"], g["tri_world"],
        g["ana_world"], g["ana_kind"], g["owner_pos"], g["lin_vel"], g["ang_vel_global"],
        g["mass"], g["pair_stack"], wild, float(g["h"]), float(g["sim_time"]))
    assert touching == int(g["touching"])
    assert np.array_equal(out_ft, g["out_ft"])
    assert np.array_equal(depth, g["depth"])
    assert np.array_equal(cp, g["cp"])
    assert np.array_equal(wild, g["wild_out"])
    acc_f, acc_t = O.reduce_to_owners(g["acs_owner_a"], g["acs_owner_b"], out_ft, cp, g["owner_pos"])
    assert np.array_equal(acc_f, g["acc_f"])
    assert np.array_equal(acc_t, g["acc_t"])
    wg = O.angular_velocity_global(g["quat"], g["ang_vel"])
    assert np.array_equal(wg, g["ang_vel_global"])
    for nthreads in (1, 4):
        pos = g["owner_pos"].copy(); quat = g["quat"].copy()
        lv = g["lin_vel"].copy(); av = g["ang_vel"].copy()
        vox = g["voxel"].copy(); sub = g["subvoxel"].copy(); cen = g["sph_centers"].copy()
        bad, oob = O.integrate_and_refresh(
            float(g["h"]), g["gravity"], pos, quat, lv, av, g["mass"], g["moi"], acc_f, acc_t,
            g["ext_force"], g["ext_torque"], g["owner_family"], g["fixed_flag"], g["lv_mask"],
            g["lv_val"], g["av_mask"], g["av_val"], g["prescribed_flag"], float(g["v_err"]),
            g["lo"], g["hi"], float(g["edge"]), vox, sub, g["sph_geom"], g["geom_params"],
            g["geom_owner"], cen, nthreads=nthreads)
        assert (bad, oob) == (int(g["int_bad"]), int(g["int_oob"]))
        for a, b in ((pos, "int_pos"), (quat, "int_quat"), (lv, "int_lin_vel"),
                     (av, "int_ang_vel"), (vox, "int_voxel"), (sub, "int_sub"),
                     (cen, "int_centers")):
            assert np.array_equal(a, g[b]), b


def test_contact_branches_exercised():
    g = load("dyn_box_rolling_mesh")
    assert np.any(g["out_ft"][:, 3:] != 0.0), "rolling branch not exercised"
    assert np.any(g["depth"] <= 0.0) and np.any(g["depth"] > 0.0)
    assert {0, 1} <= set(np.unique(g["acs_kind"]).tolist())
    assert 2 in set(np.unique(load("dyn_box")["acs_kind"]).tolist())


def test_merge_bitwise():
    g = load("merge")
    for t in range(5):
        got = O.merge_history(g[f"t{t}_old_keys"], g[f"t{t}_old_wild"], g[f"t{t}_new_keys"])
        assert np.array_equal(got, g[f"t{t}_merged_wild"])


def scene_from_golden(g):
    return {k[5:]: (v if v.ndim else v[()]) for k, v in g.items() if k.startswith("init_")}


@pytest.mark.parametrize("name", ["traj_box", "traj_mesh", "traj_clumps"])
def test_sync_trajectory_bitwise(name):
    """The oracle driver in sync mode replays the reference Simulator's whole
    trajectory bit for bit (positions, velocities, history, ACS)."""
    g = load(name)
    scene = scene_from_golden(g)
    st = O.OracleStepper(scene, float(scene["margin"]), period=1, lag=0)
    for _ in range(int(g["steps"])):
        st.step_once()
    s = st.s
    assert np.array_equal(s["voxel"], g["final_voxel"])
    assert np.array_equal(s["subvoxel"], g["final_sub"])
    assert np.array_equal(s["quat"], g["final_quat"])
    assert np.array_equal(s["lin_vel"], g["final_lin_vel"])
    assert np.array_equal(s["ang_vel"], g["final_ang_vel"])
    assert np.array_equal(st.acc_f, g["final_acc_force"])
    assert np.array_equal(st.acc_t, g["final_acc_torque"])
    assert np.array_equal(st.acs["geom_a"], g["final_geom_a"])
    assert np.array_equal(st.acs["geom_b"], g["final_geom_b"])
    assert np.array_equal(st.wild, g["final_wild"])
    assert st.last_touching == int(g["final_touching"])
