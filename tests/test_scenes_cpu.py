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


def test_rover_dense_terrain_packed_without_overlap():
    """configs[4]'s dense GRC-1 bed (scenes.rover_wheel packing "dense"):
    the requested sphere count, every GRC-1 type present at 1M spheres is
    a real component radius, no two clumps overlap, and the bed is a packed
    layer stack (solid fraction ~0.49, a few centimetres deep) -- the
    lattice packing collapses to a monolayer (solid fraction ~1 %)."""
    from scipy.spatial import cKDTree
    from paper_2311_04648_b200 import scenes
    n = 200_000
    sim = scenes.rover_wheel(n, sinkage=0.0, bed_depth=0.02)
    bed = sim.rover_bed
    assert 0.45 < bed["solid_fraction"] < 0.55
    assert bed["layers"] >= 3 and 0.005 < bed["bed_top"] < 0.04
    sc = scenes.oracle_scene(sim)
    pos = np.asarray(sim.store.positions())
    sel = sc["geom_kind"] == 0
    assert int(sel.sum()) in (n, n + 1)
    o = sc["geom_owner"][sel]
    off = sc["geom_params"][sel][:, :3].astype(np.float64)
    r = sc["geom_params"][sel][:, 3].astype(np.float64)
    assert set(np.unique(r.astype(np.float32))) <= {np.float32(t[1]) for t in scenes.GRC1_TYPES}
    w, x, y, z = (sc["quat"][o, i].astype(np.float64) for i in range(4))
    vx, vy, vz = off[:, 0], off[:, 1], off[:, 2]
    tx, ty, tz = 2 * (y * vz - z * vy), 2 * (z * vx - x * vz), 2 * (x * vy - y * vx)
    c = pos[o] + np.stack([vx + w * tx + (y * tz - z * ty), vy + w * ty + (z * tx - x * tz),
                           vz + w * tz + (x * ty - y * tx)], axis=1)
    pairs = cKDTree(c).query_pairs(2 * r.max(), output_type="ndarray")
    inter = o[pairs[:, 0]] != o[pairs[:, 1]]
    gap = np.linalg.norm(c[pairs[:, 0]] - c[pairs[:, 1]], axis=1) - (r[pairs[:, 0]] + r[pairs[:, 1]])
    assert float(gap[inter].min()) > 0.0
    # inside the trough, above the floor
    assert float((c[:, 2] - r).min()) > 0.0
    assert float(np.abs(c[:, 0]).max() + r.max()) < bed["length"] / 2
    assert float(np.abs(c[:, 1]).max() + r.max()) < bed["width"] / 2
