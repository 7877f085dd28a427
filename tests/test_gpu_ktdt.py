"""The paper's 2-GPU kT/dT split:
contact detection (kT) on one device, forces and integration (dT) on
another, the snapshot and the contact arrays crossing over NVLink peer
access (gf_create(device, kt_device, flags)).

On a one-GPU box the split runs with kt_device == device: the same code
path (kT scratch, stream and events on the kT device, contact arrays
allocated on the dT device and written from the kT stream) on one device.
The trajectory must be bit-identical to the single-device schedule -- the
split changes where detection runs, not what it computes.  With two or more
devices the real cross-device split is checked the same way."""

import numpy as np
import pytest

import paper_2311_04648_b200 as gf
from paper_2311_04648_b200 import _lib, scenes

pytestmark = pytest.mark.gpu


def run_bed(kt_device, steps=120, n=30_000):
    sim = scenes.crater_bed(n, hold_ball=False, kt_device=kt_device, n_max=4)
    sim.initialize()
    sim.do_dynamics(steps * sim.h)
    st = {k: np.asarray(v).copy() for k, v in (("voxel", sim.store.voxel), ("sub", sim.store.subvoxel),
                                               ("quat", sim.store.quat), ("v", sim.store.lin_vel),
                                               ("w", sim.store.ang_vel))}
    rr = sim.last_run
    out = (st, int(rr.n_acs), int(rr.touching), int(sim.scheduler.ca_updates))
    sim.close()
    return out


def assert_same(a, b):
    for k in a[0]:
        assert np.array_equal(a[0][k], b[0][k]), k
    assert a[1:] == b[1:]


def test_split_on_one_device_is_bit_identical():
    ref = run_bed(None)
    split = run_bed(0)
    assert_same(ref, split)


@pytest.mark.skipif(_lib.device_count() < 2, reason="needs two GPUs")
def test_split_across_two_devices_is_bit_identical():
    ref = run_bed(None)
    split = run_bed(1)
    assert_same(ref, split)


def test_split_refuses_decomposition():
    with pytest.raises(gf.ConfigurationError):
        gf.Simulator(gf.Domain.cube(1.0), decomposition=gf.SlabDecomposition(), kt_device=0)
