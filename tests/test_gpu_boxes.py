"""Active boxes on the device (engine.py:857-879):
gf_apply_active_boxes re-tags clump owners between the active and the frozen
family by box membership (a box that follows a moving anchor owner and a
static box), zeroes the velocities of owners frozen now, and the frozen
owners stay put (fixed family, masked from every contact).  Each refresh is
checked against the reference's rule evaluated here on the state downloaded
just before it."""

import numpy as np
import pytest

import paper_2311_04648_b200 as gf
from paper_2311_04648_b200 import scenes

pytestmark = pytest.mark.gpu

ACTIVE, FROZEN = 0, 7


def expected_families(sim, policy):
    """The reference's rule (engine.py:857-879) on the host mirrors."""
    s = sim.store
    n = s.n_owners
    fam = np.asarray(s.owner_family[:n]).copy()
    pos = sim._pos[:n]
    managed = ((fam == policy.active_family) | (fam == policy.frozen_family)) & (np.asarray(s.owner_kind[:n]) == 0)
    inside = np.zeros(n, dtype=bool)
    for half, anchor, center in zip(policy.half_extents, policy.anchors, policy.centers):
        c = pos[anchor] if anchor is not None else np.asarray(center)
        inside |= np.all(np.abs(pos - c) <= np.asarray(half, dtype=np.float64), axis=1)
    new = np.where(inside, policy.active_family, policy.frozen_family)
    out = fam.copy()
    out[managed] = new[managed]
    return out, managed & (fam != new) & (new == policy.frozen_family)


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_moving_box_retags_on_device(precision):
    sim = scenes.crater_bed(20_000, precision=precision, n_max=4, hold_ball=False)
    ball = sim.store.n_owners - 1   # the projectile is the last owner (scenes.crater_bed)
    policy = gf.ActiveBoxPolicy(half_extents=[np.array([0.03, 0.03, 0.08]), np.array([0.02, 0.02, 0.02])],
                                anchors=[ball, None], centers=[None, np.array([0.08, 0.08, 0.02])],
                                refresh_period=1e9, frozen_family=FROZEN, active_family=ACTIVE)
    sim.set_active_box_policy(policy)
    sim.initialize()
    with sim:
        retagged = 0
        for _ in range(4):
            want, frozen_now = expected_families(sim, policy)
            sim._apply_active_boxes()
            got = np.asarray(sim.store.owner_family[:sim.store.n_owners])
            assert np.array_equal(got, want)
            n = sim.store.n_owners
            assert np.all(np.asarray(sim.store.lin_vel)[:n][frozen_now] == 0.0)
            assert np.all(np.asarray(sim.store.ang_vel)[:n][frozen_now] == 0.0)
            retagged += int(np.sum(got != ACTIVE))
            frozen = got == FROZEN
            before = sim._pos[frozen].copy()
            sim._box_next = sim.sim_time + 1e9   # no automatic refresh inside the chunk
            sim._run(200)
            # frozen owners are fixed: they do not move (beyond the re-encode
            # every owner gets each step, _kernels.py:654: sub-voxel quanta)
            assert np.max(np.abs(sim._pos[frozen] - before)) <= 1e-9
        assert retagged > 0


def test_box_follows_anchor_through_do_dynamics():
    """The automatic refresh inside do_dynamics re-tags as the anchor moves."""
    sim = scenes.crater_bed(20_000, precision="f32", n_max=4, hold_ball=False)
    ball = sim.store.n_owners - 1
    policy = gf.ActiveBoxPolicy(half_extents=[np.array([0.025, 0.025, 0.1])], anchors=[ball], centers=[None],
                                refresh_period=50 * sim.h, frozen_family=FROZEN, active_family=ACTIVE)
    sim.set_active_box_policy(policy)
    sim.initialize()
    with sim:
        sim.do_dynamics(400 * sim.h)
        fam = np.asarray(sim.store.owner_family[:sim.store.n_owners])
        assert fam[ball] == ACTIVE
        assert np.any(fam == FROZEN) and np.any(fam[:-1] == ACTIVE)
        assert sim.box_retags > 0
