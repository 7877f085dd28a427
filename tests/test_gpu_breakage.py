"""The reference's bonded breakage model (forces.py:
185-291, build_bonds :617-675, init_bonds engine.py:409-427, bond
persistence engine.py:639-662) on the device: the model is CUDA source
compiled with NVRTC (models.BREAKAGE_SRC), the paper's JIT-model showcase.
Checked against fixtures the reference itself produced
(tests/golden/make_breakage.py):

  * the core over 400 random bonded / broken contexts: forces rel 1e-9 of
    the row's force scale, the failure latch and history exactly (the
    device log() in beta is the only libm call: one-ulp level);
  * build_bonds: the bonded pair set and initialLength bit-exact;
  * a bonded granite block dropped on a plane through Simulator.init_bonds:
    every bond intact at every sample, centre-of-mass height within 0.2 mm
    of the reference's trajectory."""

import os

import numpy as np
import pytest

import paper_2311_04648_b200 as gf
from paper_2311_04648_b200 import forces as F
from tests import _bulk as BK

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load():
    g = dict(np.load(os.path.join(GOLD, "breakage.npz")))
    return {k: (v[()] if v.ndim == 0 else v) for k, v in g.items()}


def test_breakage_core_vs_reference():
    g = load()
    wild = np.ascontiguousarray(g["core_wild_in"].copy())
    out = F.BREAKAGE_MODEL.core.batch(g["core_args"], np.zeros((wild.shape[0], 2)), g["stack"], wild)
    ref = g["core_out"]
    scale = np.maximum(np.max(np.abs(ref[:, :3]), axis=1, keepdims=True), 1e-300)
    assert np.all(np.abs(out - ref) <= 1e-9 * scale + 1e-300)
    assert np.array_equal(wild[:, 4], g["core_wild_out"][:, 4])       # the latch
    assert np.array_equal(wild[:, 5], g["core_wild_out"][:, 5])       # initialLength untouched
    np.testing.assert_allclose(wild[:, :4], g["core_wild_out"][:, :4], rtol=1e-6, atol=1e-12)
    assert np.any(g["core_wild_out"][:, 4] < 0) and np.any(g["core_wild_out"][:, 4] > 0)


def test_build_bonds_vs_reference():
    g = load()
    m = g["bonds_centers"].shape[0]
    bonds, stats = F.build_bonds(g["bonds_centers"], g["bonds_radii"], np.arange(m), np.arange(m), 1.05)
    assert stats["count"] == int(g["bonds_count"])
    assert np.array_equal(bonds.geom_a, g["bonds_a"])
    assert np.array_equal(bonds.geom_b, g["bonds_b"])
    assert np.array_equal(bonds.wildcards["initialLength"], g["bonds_init"])


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_bonded_block_drop_vs_reference(precision):
    g = load()
    r = BK.run_bonded_block(gf, precision=precision)
    assert np.array_equal(r["intact"], g["block_intact"])
    assert np.max(np.abs(r["com_z"] - g["block_com_z"])) <= 2e-4


def test_init_bonds_requires_breakage_model():
    sim = gf.Simulator(gf.Domain.cube(1.0))
    with pytest.raises(gf.ConfigurationError):
        sim.init_bonds(1.01)


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_stretched_bond_persists(precision):
    """An intact bond stretched beyond the detection margin (two soft bonded
    spheres launched apart) leaves the detected set every half period; the
    device persistence rule (gf_set_persistent_wildcard, engine.py:639-662)
    re-appends it, so the bond keeps pulling the spheres back -- the gap
    history matches the reference's within 2 % of its range."""
    g = load()
    r = BK.stretched_bond(gf, precision=precision)
    assert r["gap"].max() > r["margin"], "the scenario must stretch the bond beyond the margin"
    assert np.all(r["intact"] == 1)
    ref = g["stretch_gap"]
    assert np.max(np.abs(r["gap"] - ref)) <= 0.02 * (ref.max() - ref.min())
