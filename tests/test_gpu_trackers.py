"""Device-side trackers and inspectors (engine.py:
132-219): after a run, Tracker reads and the clump_max_absv inspector come
from the device (gf_read_owners / gf_clump_max_absv) without syncing the
owner state -- and equal what a full download gives."""

import numpy as np
import pytest

from paper_2311_04648_b200 import scenes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_tracker_reads_without_full_sync(precision):
    sim = scenes.crater_bed(20_000, precision=precision, n_max=4)
    sim.initialize()
    with sim:
        sim.do_dynamics(200 * sim.h)
        owners = [0, 17, 4321, sim.store.n_owners - 1]
        trs = [sim.track(o) for o in owners]
        got = [(t.pos(), t.vel(), t.ang_vel_local(), t.quat(), t.contact_force(), t.contact_torque()) for t in trs]
        vmax = sim.create_inspector("clump_max_absv").get_value()
        assert sim._host_stale, "tracker / inspector reads must not download the whole state"
        sim._sync_all()
        for o, g in zip(owners, got):
            assert np.array_equal(g[0], sim._pos[o])
            assert np.array_equal(g[1], sim.store.lin_vel[o].astype(np.float64))
            assert np.array_equal(g[2], sim.store.ang_vel[o].astype(np.float64))
            assert np.array_equal(g[3], sim.store.quat[o].astype(np.float64))
            assert np.array_equal(g[4], sim.store.acc_force[o])
            assert np.array_equal(g[5], sim.store.acc_torque[o])
        host = sim.create_inspector("clump_max_absv").get_value()   # host path (mirrors current)
        assert vmax == pytest.approx(host, rel=1e-12)
        assert vmax > 0.0
