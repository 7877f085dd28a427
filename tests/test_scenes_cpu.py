"""Host-side scene builders and the device owner order (no GPU needed)."""

import numpy as np

from paper_2311_04648_b200 import scenes
from paper_2311_04648_b200.core import OWNER_CLUMP
from paper_2311_04648_b200.decomp import morton_order


def _naive_morton(q):
    code = np.zeros(q.shape[0], np.uint64)
    for b in range(21):
        for ax in range(3):
            code |= ((q[:, ax] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + ax)
    return code


def test_morton_order_matches_bitwise_interleave():
    rng = np.random.default_rng(3)
    pos = rng.random((5000, 3)) * np.array([3.0, 1.0, 0.2])
    lo = pos.min(axis=0)
    span = float((pos.max(axis=0) - lo).max())
    q = np.minimum((pos - lo) / span * 2097151.0, 2097151.0).astype(np.uint64)
    ref = np.argsort(_naive_morton(q), kind="stable")
    assert np.array_equal(morton_order(pos), ref)


def test_tiled_bed_replicates_state_without_overlap():
    src = scenes.crater_bed(4000, hold_ball=True)
    scenes.release_balls(src)
    n = src.store.n_owners
    sim = scenes.tiled_bed(src, 3, 2)
    s, t = src.store, sim.store
    clump_src = s.owner_kind[:n] == OWNER_CLUMP
    n_clump = int(clump_src.sum())
    assert t.n_owners == 6 * n_clump + 1            # six copies + one wall owner
    assert t.sphere_count() == 6 * s.sphere_count()
    # every copy carries the source velocities (the released ball's too)
    assert np.isclose(np.sort(t.lin_vel[: t.n_owners, 2])[:6], s.lin_vel[:n, 2].min()).all()
    # copies meet without overlap: spheres of neighbouring copies stay apart
    pos = t.positions()[t.owner_kind[: t.n_owners] == OWNER_CLUMP]
    assert pos[:, 0].max() <= 3 * 6 * 0.0254 and pos[:, 0].min() >= -3 * 6 * 0.0254
    assert pos[:, 1].max() <= 2 * 6 * 0.0254 and pos[:, 1].min() >= -2 * 6 * 0.0254
