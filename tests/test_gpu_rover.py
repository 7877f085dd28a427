"""configs[4]'s rover wheel: the grousered wheel mesh
with a prescribed spin (and forward speed) rolling through the GRC-1-like
clump terrain (scenes.rover_wheel).

  * moving-mesh sphere-triangle parity: the same scene stepped by the oracle
    driver (the reference's algorithm: world triangles re-derived from the
    prescribed pose every step, sphere-triangle detection, Hertz-Mindlin) and
    by the device in sync mode (fp64 build) -- bit-identical state, contact
    set and history; the fp32 throughput build within the north-star
    tolerance on velocities;
  * the wheel's contact force readback: the mesh owner's
    accumulated force after a step equals minus the sum of what its
    triangles exert on the grains (Newton's third law through the device
    reduction)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2311_04648_b200 import scenes
from tests import _scene as S

pytestmark = pytest.mark.gpu


def small_rover(precision="f64"):
    # the wheel plunges at 1 m/s while it spins, so its grousers and rim
    # reach the grains under it within the window
    sim = scenes.rover_wheel(6_000, packing="lattice", precision=precision, h=1e-5, v_err=3.0, n_max=4, sinkage=0.0,
                             wheel_radius=0.05, aspect=2.0, plunge=1.0)
    return sim


def test_rover_wheel_sync_trajectory_matches_oracle():
    sim = small_rover()
    scene = scenes.oracle_scene(sim)
    margin = O.margin_for(float(scene["v_err"]), float(scene["h"]), 1)
    steps = 400
    ref = O.OracleStepper(scene, margin, period=1, lag=0)
    for _ in range(steps):
        ref.step_once()
    ctx = S.upload_scene(scene)
    rr = S.run(ctx, scene, steps, margin, period=1, lag=0)
    assert rr.bad_owner == -1 and rr.oob_owner == -1
    out = S.download_state(ctx, scene["voxel"].shape[0])
    kind, sa, sb, wild = S.get_acs(ctx)
    ctx.close()
    assert int(np.sum(kind == 1)) > 0, "the wheel must touch the terrain"
    assert rr.touching == ref.last_touching
    for key in ("voxel", "subvoxel", "quat", "lin_vel", "ang_vel"):
        assert np.array_equal(out[key], ref.s[key]), key


def test_rover_wheel_f32_within_tolerance():
    sim = small_rover()
    scene = scenes.oracle_scene(sim)
    scene["lin_vel"] = scene["lin_vel"].astype(np.float32).astype(np.float64)
    scene["ang_vel"] = scene["ang_vel"].astype(np.float32).astype(np.float64)
    margin = O.margin_for(float(scene["v_err"]), float(scene["h"]), 1)
    steps = 400
    ref = O.OracleStepper(scene, margin, period=1, lag=0)
    for _ in range(steps):
        ref.step_once()
    ctx = S.upload_scene(scene, f32_state=True)
    rr = S.run(ctx, scene, steps, margin, period=1, lag=0)
    out = S.download_state(ctx, scene["voxel"].shape[0])
    ctx.close()
    assert rr.touching == ref.last_touching
    dv = np.abs(out["lin_vel"] - ref.s["lin_vel"])
    vscale = max(float(np.max(np.abs(ref.s["lin_vel"] - scene["lin_vel"]))), 1e-12)
    assert float(np.max(dv)) <= 1e-5 * vscale + 1e-6 * float(np.max(np.abs(ref.s["lin_vel"])))


def test_wheel_contact_force_readback():
    """Through the Simulator: after a do_dynamics call the wheel owner's
    accumulated force (acc_force, read back for passive owners on the
    reported step) balances the grains' wall-contact forces."""
    sim = scenes.rover_wheel(20_000, packing="lattice", precision="f64", h=1e-5, v_err=3.0, n_max=4, sinkage=0.0,
                             wheel_radius=0.06, aspect=2.0, plunge=1.0)
    sim.initialize()
    with sim:
        s = sim.store
        n = s.n_owners
        wheel = [o for o in range(n) if s.owner_family[o] == scenes.WHEEL_FAMILY][0]
        tr = sim.track(wheel)
        f_wheel = np.zeros(3)
        for _ in range(12):   # until the plunging wheel meets the terrain
            sim.do_dynamics(100 * sim.h)
            f_wheel = tr.contact_force()   # device read (gf_read_owners), no state download
            if np.linalg.norm(f_wheel) > 0.0:
                break
        assert sim._host_stale
        assert np.linalg.norm(f_wheel) > 0.0
        sim._sync_all()
        assert np.array_equal(np.asarray(s.acc_force)[wheel], f_wheel)
