"""Synthetic workloads of BASELINE.json's configs, built through the public
Simulator API only (setup code; no compute here).

crater_bed  configs[1]: projectile impact onto an n-sphere polydisperse bed.
            Geometry and materials follow the reference's crater builders
            (scenarios.py:229-307, _crater_sim / settle_crater_bed): bed
            12 D x 12 D x 8 D, D = 2.54 cm, eleven grain diameters uniform over
            the relative band [0.25, 0.35] scaled to the mean the bed volume
            implies for n grains, rho_g = 2500, E = 5e6, nu = 0.3, CoR = 0.5,
            mu = 0.3, Crr = 0.01, five fixed analytic walls, a 7.8 g/cc ball
            released just above the bed at the free-fall speed of a 20 cm drop.
            Deviations (stated in DESIGN.md): the grains start on an HCP
            lattice of pitch d_max (the reference pours and settles first,
            scenarios.py:286-291) and the step is h = 1e-5 s with v_err = 5 m/s
            (the reference's 1e-4 s / 30 m/s give a 24 mm detection margin,
            i.e. thousands of candidate pairs per grain).
settling_box configs[0]: monodisperse r = 5 mm spheres in a walled box.
clump_bed   configs[2]'s clump path: 5-sphere cylinder clumps (the reference's
            WC clump, scenarios.py:386-407: r = 2 mm, L = 8.5 mm, rho = 476)
            settling in a box, random orientations.
tiled_bed   configs[4]'s size sweep: tx x ty copies of a settled crater bed
            side by side in one box (same grains, same step), so the sphere
            count grows at fixed grain size.
"""

from __future__ import annotations

import math

import numpy as np

from .core import ClumpTemplate, Domain
from .engine import Simulator, hcp_sample_box

G = 9.81


def crater_bed(n_spheres: int = 1_000_000, *, seed: int = 7, h: float = 1e-5, v_err: float = 5.0,
               n_max: int = 4, precision: str = "f32", device: int = 0, ball: bool = True,
               drop_height: float = 0.20, ball_density: float = 7800.0, decomposition=None,
               tiles: int = 1, hold_ball: bool = False, force_model: str = "hertz_mindlin",
               extra_props: dict | None = None, kt_device=None) -> Simulator:
    rng = np.random.default_rng(seed)
    D = 0.0254
    bed_half = 12.0 * D / 2.0
    depth = 8.0 * D
    packing = 1460.0 / 2500.0
    volume = (2 * bed_half) ** 2 * depth
    d_mean = (6.0 * volume * packing / (math.pi * n_spheres)) ** (1.0 / 3.0)
    # `tiles` beds side by side along x (weak-scaling scene: one bed and one
    # projectile per rank); tiles = 1 is configs[1] itself
    tiles = max(1, int(tiles))
    half_x = bed_half * tiles
    dset = np.linspace(0.25, 0.35, 11) * (d_mean / 0.30)
    radii = dset / 2.0
    r_max = float(radii.max())
    dom = Domain((-half_x - 0.2 * bed_half, -bed_half * 1.2, -0.02),
                 (half_x + 0.2 * bed_half, bed_half * 1.2, depth * 3.0 + 0.3))
    sim = Simulator(dom, force_model, precision=precision, device=device, decomposition=decomposition,
                    kt_device=kt_device)
    grain = sim.load_material({**CRATER_MATERIAL, **(extra_props or {})})
    wall = sim.load_material({**CRATER_MATERIAL, **(extra_props or {})})
    tpls = [sim.load_clump_template(ClumpTemplate.solid_sphere(
        float(r), 2500.0 * 4.0 / 3.0 * math.pi * float(r) ** 3, grain)) for r in radii]
    # lattice pitch d_max: the largest grains touch, nobody overlaps
    pitch = 2.0 * r_max * 1.0005
    half_xy = bed_half - r_max * 1.05
    # enough layers for n grains (rows come out bottom layer first)
    per_layer = (2 * half_xy) ** 2 / (math.sqrt(3.0) / 2.0 * pitch ** 2)
    layer_dz = 2.0 * math.sqrt(6.0) / 3.0 * pitch / 2.0
    n_layers = int(math.ceil(1.15 * n_spheres / max(per_layer, 1.0))) + 2
    top = r_max * 1.05 + n_layers * layer_dz
    pts = hcp_sample_box((0.0, 0.0, (top + r_max * 1.05) / 2.0), (half_xy, half_xy, (top - r_max * 1.05) / 2.0),
                         pitch)
    if pts.shape[0] < n_spheres:
        raise RuntimeError(f"lattice holds {pts.shape[0]} < {n_spheres} grains")
    pts = pts[:n_spheres]
    offsets = [-half_x + (2 * t + 1) * bed_half for t in range(tiles)]
    for x_off in offsets:
        kinds = rng.integers(0, 11, pts.shape[0])
        for k, tpl in enumerate(tpls):
            sel = pts[kinds == k]
            if sel.shape[0]:
                sim.add_clumps(tpl, sel + np.array([x_off, 0.0, 0.0]))
    walls = [("plane", (0, 0, 0), (0, 0, 1), wall),
             ("plane", (-half_x, 0, 0), (1, 0, 0), wall),
             ("plane", (half_x, 0, 0), (-1, 0, 0), wall),
             ("plane", (0, -bed_half, 0), (0, 1, 0), wall),
             ("plane", (0, bed_half, 0), (0, -1, 0), wall)]
    sim.add_analytic(walls, family=255)
    sim.set_family_fixed(255)
    if ball:
        R = D / 2.0
        mass = ball_density * 4.0 / 3.0 * math.pi * R ** 3
        btpl = sim.load_clump_template(ClumpTemplate.solid_sphere(R, mass, grain))
        surface = float(pts[:, 2].max()) + r_max
        for x_off in offsets:
            b = sim.add_clumps(btpl, [[x_off, 0.0, surface + R + 2e-3]])[0]
            if hold_ball:   # parked (family 1, fixed) while the bed settles; see release_balls
                sim.store.owner_family[b] = 1
            else:
                sim.track(b).set_vel([0.0, 0.0, -math.sqrt(2.0 * G * drop_height)])
        if hold_ball:
            sim.set_family_fixed(1)
    sim.set_gravity([0, 0, -G])
    sim.set_init_time_step(h)
    sim.set_error_out_velocity(v_err)
    sim.set_fixed_lookahead(n_max)
    return sim


CRATER_MATERIAL = {"E": 5e6, "nu": 0.3, "CoR": 0.5, "mu": 0.3, "Crr": 0.01}


def tiled_bed(src: Simulator, tx: int, ty: int, *, precision: str = "f32", device: int = 0,
              n_max: int = 4, kt_device=None) -> Simulator:
    """tx x ty copies of the (settled, released) crater bed `src` in one box:
    owners keep their state (position, orientation, velocities), copies are
    laid out at the bed pitch 12 D, the floor and the four outer walls bound
    the whole array (inner walls removed; every grain is at least its radius
    from its old wall plane, so copies meet without overlap)."""
    from .core import OWNER_CLUMP, decode_position, encode_position
    s = src.store
    n = s.n_owners
    s.voxel  # sync the host mirror
    d = s.__dict__
    pos = decode_position(d["_voxel"][:n], d["_subvoxel"][:n], s.domain)
    clump = d["_owner_kind"][:n] == OWNER_CLUMP
    tpl = d["_owner_template"][:n]
    D = 0.0254
    bed_half = 12.0 * D / 2.0
    lo, hi = s.domain.lo, s.domain.hi
    dom = Domain((-tx * bed_half - 0.2 * bed_half, -ty * bed_half - 0.2 * bed_half, float(lo[2])),
                 (tx * bed_half + 0.2 * bed_half, ty * bed_half + 0.2 * bed_half, float(hi[2])))
    sim = Simulator(dom, precision=precision, device=device, reorder=False, kt_device=kt_device)
    grain = sim.load_material(dict(CRATER_MATERIAL))
    wall = sim.load_material(dict(CRATER_MATERIAL))
    for t in s.templates:
        sim.load_clump_template(t)
    offsets = [(-tx * bed_half + (2 * ix + 1) * bed_half, -ty * bed_half + (2 * iy + 1) * bed_half)
               for iy in range(ty) for ix in range(tx)]
    # owners tile by tile, each tile in the source's device (Morton) order:
    # the copy needs no reordering of its own (reorder=False above), and
    # every tile is a block copy of the source rows (only the positions are
    # re-encoded), so the 150M-sphere setup does no sort, permutation or
    # per-owner Python work
    order = np.asarray(getattr(src, "_own_d2u", np.arange(n)), dtype=np.int64)
    order = order[clump[order]]
    n_c = order.size
    T = len(offsets)
    ng_all = s.n_geoms
    go = d["_geom_owner"][:ng_all]
    gsort = np.argsort(go, kind="stable")
    gcnt = np.bincount(go, minlength=n)
    gstart = np.concatenate([[0], np.cumsum(gcnt)])
    kk = gcnt[order]
    gidx = gsort[np.repeat(gstart[order], kk) + (np.arange(int(kk.sum())) - np.repeat(np.cumsum(kk) - kk, kk))]
    n_g = gidx.size
    st = sim.store
    st.reserve(n_c * T + 8, n_g * T + 8)
    dd = st.__dict__
    own_rows = {name: d[name][order] for name in ("_owner_kind", "_owner_template", "_owner_family", "_quat",
                                                  "_lin_vel", "_ang_vel", "_mass", "_moi")}
    geo_rows = {name: d[name][gidx] for name in ("_geom_kind", "_geom_material", "_geom_params")}
    local_owner = np.repeat(np.arange(n_c, dtype=np.int64), kk)
    p0 = pos[order]
    for ti, (ox, oy) in enumerate(offsets):
        o0, g0 = st.n_owners, st.n_geoms
        vox, sub = encode_position(p0 + np.array([ox, oy, 0.0]), st.domain)
        osl, gsl = slice(o0, o0 + n_c), slice(g0, g0 + n_g)
        dd["_voxel"][osl] = vox
        dd["_subvoxel"][osl] = sub
        for name, rows in own_rows.items():
            dd[name][osl] = rows
        dd["_geom_owner"][gsl] = local_owner + o0
        for name, rows in geo_rows.items():
            dd[name][gsl] = rows
        st.n_owners += n_c
        st.n_geoms += n_g
    hx, hy = tx * bed_half, ty * bed_half
    walls = [("plane", (0, 0, 0), (0, 0, 1), wall),
             ("plane", (-hx, 0, 0), (1, 0, 0), wall), ("plane", (hx, 0, 0), (-1, 0, 0), wall),
             ("plane", (0, -hy, 0), (0, 1, 0), wall), ("plane", (0, hy, 0), (0, -1, 0), wall)]
    sim.add_analytic(walls, family=255)
    sim.set_family_fixed(255)
    sim.set_gravity(src.gravity)
    sim.set_init_time_step(src.h)
    sim.set_error_out_velocity(src.v_err)
    sim.set_fixed_lookahead(n_max)
    del grain
    return sim


def clump_bed(n_clumps: int = 1_000_000, *, seed: int = 11, h: float = 1e-5, v_err: float = 5.0,
              n_max: int = 4, precision: str = "f32", device: int = 0) -> Simulator:
    """configs[2]: n five-sphere cylinder clumps (r = 2 mm, L = 8.5 mm,
    rho = 476; the reference's WC clump, scenarios.py:386-407) on a cubic
    lattice with random orientations in a walled box, crater materials."""
    from .core import ClumpSphere
    rng = np.random.default_rng(seed)
    r, L, rho = 0.002, 0.0085, 476.0
    m = rho * math.pi * r * r * L
    i_ax = 0.5 * m * r * r
    i_pe = m * (3 * r * r + L * L) / 12.0
    pitch = L * 1.02
    per_side = int(math.ceil((n_clumps * 2.0) ** (1.0 / 3.0)))     # footprint side; ~half as many layers
    half = per_side * pitch / 2.0
    layers = int(math.ceil(n_clumps / per_side ** 2)) + 1
    top = layers * pitch + pitch
    dom = Domain((-half - 0.05, -half - 0.05, -0.02), (half + 0.05, half + 0.05, top + 0.1))
    sim = Simulator(dom, precision=precision, device=device)
    mat = sim.load_material(dict(CRATER_MATERIAL))
    offs = np.linspace(-(L / 2 - r), L / 2 - r, 5)
    tpl = sim.load_clump_template(ClumpTemplate(
        m, np.array([i_ax, i_pe, i_pe]),
        tuple(ClumpSphere(np.array([x, 0.0, 0.0]), r, mat) for x in offs)))
    g = (np.arange(per_side) + 0.5) * pitch - half
    gx, gy = np.meshgrid(g, g, indexing="ij")
    pts = []
    for k in range(layers):
        pts.append(np.stack([gx.ravel(), gy.ravel(), np.full(gx.size, (k + 1) * pitch)], -1))
    pts = np.concatenate(pts)[:n_clumps]
    ids = np.asarray(sim.add_clumps(tpl, pts), dtype=np.int64)
    q = rng.normal(size=(ids.size, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sim.store.__dict__["_quat"][ids] = q
    walls = [("plane", (0, 0, 0), (0, 0, 1), mat),
             ("plane", (-half, 0, 0), (1, 0, 0), mat), ("plane", (half, 0, 0), (-1, 0, 0), mat),
             ("plane", (0, -half, 0), (0, 1, 0), mat), ("plane", (0, half, 0), (0, -1, 0), mat)]
    sim.add_analytic(walls, family=255)
    sim.set_family_fixed(255)
    sim.set_gravity([0, 0, -G])
    sim.set_init_time_step(h)
    sim.set_error_out_velocity(v_err)
    sim.set_fixed_lookahead(n_max)
    return sim


def release_balls(sim: Simulator, drop_height: float = 0.20) -> list:
    """After the bed settled (crater_bed(hold_ball=True)): every parked
    projectile (family 1) moves to 2 mm above the highest grain under its
    footprint with the
    free-fall speed of a `drop_height` drop, and becomes free (family 0) --
    the reference's settle-then-drop order (scenarios.py:255-307).  Works on
    a decomposed simulator too (a global edit, decomp.update_global)."""
    from .core import GEOM_SPHERE, OWNER_CLUMP, decode_position

    def edit(store):
        n = store.n_owners
        d = store.__dict__
        pos = decode_position(d["_voxel"][:n], d["_subvoxel"][:n], store.domain)
        fam = d["_owner_family"][:n]
        kind = d["_owner_kind"][:n]
        ng = store.n_geoms
        go = d["_geom_owner"][:ng]
        sph = d["_geom_kind"][:ng] == GEOM_SPHERE
        rad = np.zeros(n)
        np.maximum.at(rad, go[sph], d["_geom_params"][:ng][sph, 3].astype(np.float64))
        balls = np.nonzero((fam == 1) & (kind == OWNER_CLUMP))[0]
        grains = (fam == 0) & (kind == OWNER_CLUMP)
        v = -math.sqrt(2.0 * G * drop_height)
        for b in balls:
            # clear the highest grain under the ball's footprint
            rho = np.hypot(pos[:, 0] - pos[b, 0], pos[:, 1] - pos[b, 1])
            near = grains & (rho < rad[b] + rad + 1e-3)
            top = float(np.max(pos[near, 2] + rad[near]))
            xyz = np.array([pos[b, 0], pos[b, 1], top + rad[b] + 2e-3])
            store.set_position(int(b), xyz)
            d["_lin_vel"][b] = (0.0, 0.0, v)
            d["_ang_vel"][b] = 0.0
            d["_owner_family"][b] = 0
        return balls.tolist()

    if sim.decomposition is not None:
        from . import decomp
        target = sim.decomposition.group if sim.decomposition.group is not None else sim
        decomp.update_global(target, edit)
        return []
    s = sim.store
    s.voxel  # sync the host mirror
    out = edit(s)
    sim._host_dirty = True
    return out


def settling_box(n_spheres: int = 10_000, *, h: float = 1e-5, v_err: float = 5.0, n_max: int = 4,
                 precision: str = "f64", device: int = 0) -> Simulator:
    """configs[0]: r = 5 mm, rho = 2600, {E 1e7, nu 0.3, CoR 0.6, mu 0.3}, floor
    + 4 side walls fixed (test_engine.py:13-18 materials)."""
    r = 0.005
    side = (n_spheres * (2 * r * 1.02) ** 3 / 0.70) ** (1.0 / 3.0)
    half = max(side / 2.0, 4 * r)
    dom = Domain((-half - 0.05, -half - 0.05, -0.02), (half + 0.05, half + 0.05, 4 * half + 0.2))
    sim = Simulator(dom, precision=precision, device=device)
    mat = sim.load_material({"E": 1e7, "nu": 0.3, "CoR": 0.6, "mu": 0.3, "Crr": 0.0})
    m = 2600.0 * 4.0 / 3.0 * math.pi * r ** 3
    tpl = sim.load_clump_template(ClumpTemplate.solid_sphere(r, m, mat))
    pts = hcp_sample_box((0, 0, 1.1 * half + 1.02 * r), (half - 1.5 * r, half - 1.5 * r, 1.1 * half),
                         2 * r * 1.02)
    if pts.shape[0] < n_spheres:
        raise RuntimeError("box too small")
    sim.add_clumps(tpl, pts[:n_spheres])
    walls = [("plane", (0, 0, 0), (0, 0, 1), mat),
             ("plane", (-half, 0, 0), (1, 0, 0), mat), ("plane", (half, 0, 0), (-1, 0, 0), mat),
             ("plane", (0, -half, 0), (0, 1, 0), mat), ("plane", (0, half, 0), (0, -1, 0), mat)]
    sim.add_analytic(walls, family=255)
    sim.set_family_fixed(255)
    sim.set_gravity([0, 0, -G])
    sim.set_init_time_step(h)
    sim.set_error_out_velocity(v_err)
    sim.set_fixed_lookahead(n_max)
    return sim


def oracle_scene(sim: Simulator) -> dict:
    """The simulator's setup state in the oracle's scene-dict layout (used by
    the bench's CPU legs and tests; reads host mirrors only)."""
    from .forces import material_pair_stack
    s = sim.store
    n, g = s.n_owners, s.n_geoms
    return dict(
        voxel=s.voxel[:n].copy(), subvoxel=s.subvoxel[:n].copy(), quat=s.quat[:n].copy(),
        lin_vel=s.lin_vel[:n].copy(), ang_vel=s.ang_vel[:n].copy(), mass=s.mass[:n].copy(),
        moi=s.moi[:n].copy(), owner_family=s.owner_family[:n].copy(),
        ext_force=s.ext_force[:n].copy(), ext_torque=s.ext_torque[:n].copy(),
        geom_owner=s.geom_owner[:g].copy(), geom_kind=s.geom_kind[:g].copy(),
        geom_material=s.geom_material[:g].copy(), geom_params=s.geom_params[:g].copy(),
        lo=s.domain.lo.copy(), hi=s.domain.hi.copy(), edge=float(s.domain.voxel_edge),
        pair_stack=material_pair_stack(sim.materials, sim.model),
        mask=s.families.mask.astype(np.uint8), fixed_flag=sim._fixed_flag.astype(np.uint8),
        prescribed_flag=sim._prescribed_flag.astype(np.uint8),
        lv_mask=sim._lv_mask.astype(np.uint8), lv_val=sim._lv_val.copy(),
        av_mask=sim._av_mask.astype(np.uint8), av_val=sim._av_val.copy(),
        gravity=sim.gravity.copy(), h=float(sim.h), v_err=float(sim.v_err))


# ---------------------------------------------------------------------------
# configs[4] rover wheel: a grousered wheel mesh with a
# prescribed spin of 0.8 rad/s rolling through a GRC-1-like terrain of
# multi-sphere clumps (table GRCDS: component radius,
# clump size, weight share; E = 1e8, nu = 0.3, mu = 0.4, CoR = 0.5), DEM step
# 2e-6 s.
# ---------------------------------------------------------------------------

# type: (clump size, component radius, weight share) -- PAPER.md:1196-1202
GRC1_TYPES = ((21.0e-3, 3.6e-3, 0.17), (11.4e-3, 1.95e-3, 0.21), (6.6e-3, 1.81e-3, 0.14),
              (4.5e-3, 1.24e-3, 0.19), (3.0e-3, 0.82e-3, 0.16), (2.75e-3, 0.75e-3, 0.05),
              (2.5e-3, 0.70e-3, 0.08))
GRC1_MATERIAL = {"E": 1e8, "nu": 0.3, "CoR": 0.5, "mu": 0.4, "Crr": 0.0}
WHEEL_FAMILY = 2


def grousered_wheel(radius: float = 0.25, width: float = 0.2, n_around: int = 96, n_grousers: int = 24,
                    grouser_h: float = 0.02) -> np.ndarray:
    """Triangles (n, 3, 3) of a wheel centred at the origin, axle along y:
    the rim (n_around quads), two side disks (fans) and n_grousers radial
    fins of height grouser_h spanning the width."""
    th = np.linspace(0.0, 2.0 * math.pi, n_around + 1)
    hw = width / 2.0
    tris = []
    for a, b in zip(th[:-1], th[1:]):
        p = lambda t, y, r=radius: (r * math.cos(t), y, r * math.sin(t))  # noqa: E731
        tris.append((p(a, -hw), p(b, -hw), p(b, hw)))
        tris.append((p(a, -hw), p(b, hw), p(a, hw)))
        for y in (-hw, hw):
            tris.append(((0.0, y, 0.0), p(a, y), p(b, y)))
    for t in np.linspace(0.0, 2.0 * math.pi, n_grousers, endpoint=False):
        c, s = math.cos(t), math.sin(t)
        r0, r1 = radius, radius + grouser_h
        q00, q10 = (r0 * c, -hw, r0 * s), (r1 * c, -hw, r1 * s)
        q01, q11 = (r0 * c, hw, r0 * s), (r1 * c, hw, r1 * s)
        tris.append((q00, q10, q11))
        tris.append((q00, q11, q01))
    return np.asarray(tris, dtype=np.float64)


def grc1_templates(sim: Simulator, material: int, density: float = 2500.0, scale: float = 1.0):
    """One clump template per GRC-1 type: ceil(size / (2 r_c)) component
    spheres of radius r_c on a line spanning the clump size; mass and
    principal MOI of the spheres (overlaps ignored)."""
    from .core import ClumpSphere
    out = []
    for size, rc, share in GRC1_TYPES:
        size, rc = size * scale, rc * scale
        k = max(2, int(math.ceil(size / (2.0 * rc))))
        span = size - 2.0 * rc
        xs = np.linspace(-span / 2.0, span / 2.0, k)
        ms = density * 4.0 / 3.0 * math.pi * rc ** 3
        m = k * ms
        i_ax = k * 0.4 * ms * rc * rc
        i_pe = i_ax + ms * float(np.sum(xs * xs))
        tpl = ClumpTemplate(m, np.array([i_ax, i_pe, i_pe]),
                            tuple(ClumpSphere(np.array([x, 0.0, 0.0]), rc, material) for x in xs))
        out.append((sim.load_clump_template(tpl), tpl, share, size, k))
    return out


def _grc1_layers(n_spheres: int, lo, hi, rng, gap: float = 0.05, tilt: float = 0.02):
    """Dense GRC-1 layers inside the box lo..hi (x, y; z from lo[2] up) until
    n_spheres component spheres: per layer one type t (probability ~ weight
    share / layer thickness, so volumes follow the weight shares), clumps
    aligned with the layer's yaw (0 or 90 degrees, alternating), spaced
    (1 + gap) x (clump size, sphere diameter), rows offset by half a pitch,
    each tilted by a random angle <= `tilt` about its horizontal normal
    (small enough for the gap).  Returns (type, centres (n, 3), quats (n, 4)
    as (w, x, y, z)) per layer."""
    size = np.array([t[0] for t in GRC1_TYPES])
    rc = np.array([t[1] for t in GRC1_TYPES])
    k_of = np.array([max(2, math.ceil(t[0] / (2 * t[1]))) for t in GRC1_TYPES])
    thick = 2.0 * rc * (1.0 + gap)
    p = np.array([t[2] for t in GRC1_TYPES]) / thick
    p /= p.sum()
    layers, total, z_top, yaw, prev_rc = [], 0, float(lo[2]), 0, 0.0
    while total < n_spheres:
        t = int(rng.choice(len(GRC1_TYPES), p=p))
        a, b = size[t] * (1.0 + gap), 2.0 * rc[t] * (1.0 + gap)
        half = 0.5 * (size[t] - 2.0 * rc[t])
        # the layer's centre plane: the previous layer's top + this one's
        # radius, with room for both tilts
        z = (z_top + rc[t] * (1.0 + gap) + half * math.sin(tilt)) if layers else float(lo[2]) + rc[t] + half * math.sin(tilt) + 1e-4
        ax_len = (hi[0] - lo[0], hi[1] - lo[1]) if yaw == 0 else (hi[1] - lo[1], hi[0] - lo[0])
        n_along = int((ax_len[0] - size[t]) // a) + 1
        n_across = int((ax_len[1] - 2.0 * rc[t]) // b) + 1
        if n_along < 1 or n_across < 1:
            raise ValueError("trough too small for the GRC-1 clumps")
        i, j = np.meshgrid(np.arange(n_along - 1), np.arange(n_across), indexing="ij")
        u = (i + 0.5 * (j % 2)) * a + 0.5 * size[t] + 0.5 * (ax_len[0] - size[t] - (n_along - 1) * a)
        v = j * b + rc[t] + 0.5 * (ax_len[1] - 2.0 * rc[t] - (n_across - 1) * b)
        u, v = u.ravel(), v.ravel()
        if yaw == 0:
            cen = np.stack([lo[0] + u, lo[1] + v, np.full(u.size, z)], axis=1)
        else:
            cen = np.stack([lo[0] + v, lo[1] + u, np.full(u.size, z)], axis=1)
        need = -(-(n_spheres - total) // int(k_of[t]))
        if cen.shape[0] > need:
            cen = cen[rng.permutation(cen.shape[0])[:need]]
        n = cen.shape[0]
        al = rng.uniform(-tilt, tilt, n)
        psi = 0.0 if yaw == 0 else 0.5 * math.pi
        cy, sy = math.cos(psi / 2), math.sin(psi / 2)
        ct, st = np.cos(al / 2), np.sin(al / 2)
        q = np.stack([cy * ct, -sy * st, cy * st, sy * ct], axis=1)   # yaw (z) * tilt (body y)
        layers.append((t, cen, q))
        total += n * int(k_of[t])
        z_top = z + rc[t] + half * math.sin(tilt)
        yaw ^= 1
    return layers, z_top


def _rover_dense(n_spheres, *, seed, h, v_err, n_max, precision, device, omega, slip, wheel_radius,
                 sinkage, aspect, plunge, kt_device, bed_depth):
    rng = np.random.default_rng(seed)
    gap = 0.05
    size = np.array([t[0] for t in GRC1_TYPES])
    rc = np.array([t[1] for t in GRC1_TYPES])
    k_of = np.array([max(2, math.ceil(t[0] / (2 * t[1]))) for t in GRC1_TYPES])
    w = np.array([t[2] for t in GRC1_TYPES])
    # solid fraction of each type's layer, volume-weighted mean
    phi_t = k_of * 4.0 / 3.0 * math.pi * rc ** 3 / (size * (2 * rc) ** 2 * (1 + gap) ** 3)
    phi = float(np.sum(w * phi_t) / np.sum(w))
    # mean component-sphere volume: spheres per unit volume of each type
    sph_vol = 4.0 / 3.0 * math.pi * rc ** 3
    share_sph = w / (k_of * sph_vol) * k_of   # spheres per unit solid volume of each type
    v_mean = float(np.sum(w) / np.sum(share_sph))
    depth = bed_depth if bed_depth is not None else (0.06 if n_spheres >= 2_000_000 else 0.03)
    area = n_spheres * v_mean / (phi * depth)
    width = max(math.sqrt(area / aspect), 1.4 * min(0.2, 2.0 * wheel_radius))
    length = max(area / width, 4.0 * wheel_radius + 0.2)
    wall_gap = 2e-3
    lo = (-length / 2 + wall_gap, -width / 2 + wall_gap, 1e-4)
    hi = (length / 2 - wall_gap, width / 2 - wall_gap, None)
    layers, top = _grc1_layers(n_spheres, lo, hi, rng, gap=gap)
    dom = Domain((-length / 2 - 0.3, -width / 2 - 0.05, -0.02),
                 (length / 2 + 0.3, width / 2 + 0.05, top + 2.5 * wheel_radius + 0.3))
    sim = Simulator(dom, precision=precision, device=device, kt_device=kt_device)
    mat = sim.load_material(dict(GRC1_MATERIAL))
    tpls = grc1_templates(sim, mat)
    for t, cen, q in layers:
        ids = np.asarray(sim.store.add_clumps_array(tpls[t][0], cen), dtype=np.int64)
        sim.store.__dict__["_quat"][ids] = q
    walls = [("plane", (0, 0, 0), (0, 0, 1), mat),
             ("plane", (-length / 2, 0, 0), (1, 0, 0), mat), ("plane", (length / 2, 0, 0), (-1, 0, 0), mat),
             ("plane", (0, -width / 2, 0), (0, 1, 0), mat), ("plane", (0, width / 2, 0), (0, -1, 0), mat)]
    sim.add_analytic(walls, family=255)
    sim.set_family_fixed(255)
    wheel_w = min(0.2, 0.6 * width)
    grouser = 0.08 * wheel_radius
    tris = grousered_wheel(radius=wheel_radius, width=wheel_w, grouser_h=grouser)
    x0 = -length / 2 + wheel_radius + grouser + 0.05
    z0 = top + wheel_radius + grouser - sinkage   # the lowest grouser tip `sinkage` into the bed top
    sim.add_mesh(tris, mat, family=WHEEL_FAMILY, position=(x0, 0.0, z0))
    sim.set_family_prescribed_lin_vel(WHEEL_FAMILY, omega * wheel_radius * (1.0 - slip), 0.0, -plunge)
    sim.set_family_prescribed_ang_vel(WHEEL_FAMILY, 0.0, omega, 0.0)
    sim.set_gravity([0, 0, -G])
    sim.set_init_time_step(h)
    sim.set_error_out_velocity(v_err)
    sim.set_fixed_lookahead(n_max)
    sim.rover_bed = {"length": length, "width": width, "bed_top": top, "solid_fraction": phi,
                     "layers": len(layers)}
    return sim


def rover_wheel(n_spheres: int = 11_000_000, *, seed: int = 3, h: float = 2e-6, v_err: float = 3.0,
                n_max: int = 8, precision: str = "f32", device: int = 0, omega: float = 0.8,
                slip: float = 0.2, wheel_radius: float = 0.25, sinkage: float = 0.005,
                aspect: float = 4.0, plunge: float = 0.0, kt_device=None,
                packing: str = "dense", bed_depth: float = None) -> Simulator:
    """A GRC-1-like terrain of about n_spheres component spheres in a walled
    trough (length = aspect x width) with the grousered wheel resting
    `sinkage` into its surface at one end, spinning at `omega` about its axle
    and moving forward at omega R (1 - slip) (family WHEEL_FAMILY, fully
    prescribed: a boundary owner whose contact force is read back).

    packing "dense" (default): horizontal layers of one GRC-1 type each
    (layer types drawn so the volume shares follow the weight shares), rows
    of clumps 5 % apart, yaw alternating 0 / 90 degrees between layers, a
    small random tilt -- a bed `bed_depth` deep (0.06 m from 2M spheres up,
    else 0.03 m) that settles by a few per cent.  packing "lattice": the
    round-2 HCP lattice of pitch = the type-2 clump size (11.4 mm, random
    types by number share, random orientations); its solid fraction is ~1 %,
    so it collapses to a grain monolayer -- kept for the small parity scenes
    in tests/."""
    if packing == "dense":
        return _rover_dense(n_spheres, seed=seed, h=h, v_err=v_err, n_max=n_max, precision=precision,
                            device=device, omega=omega, slip=slip, wheel_radius=wheel_radius,
                            sinkage=sinkage, aspect=aspect, plunge=plunge, kt_device=kt_device,
                            bed_depth=bed_depth)
    if packing != "lattice":
        raise ValueError(f"unknown packing {packing!r}")
    rng = np.random.default_rng(seed)
    pitch = GRC1_TYPES[1][0] * 1.02
    # number shares from the weight shares (w / m, m ~ k rc^3)
    w = np.array([t[2] for t in GRC1_TYPES])
    per = np.array([max(2, math.ceil(t[0] / (2 * t[1]))) * t[1] ** 3 for t in GRC1_TYPES])
    num = w / per
    num /= num.sum()
    k_of = np.array([max(2, math.ceil(t[0] / (2 * t[1]))) for t in GRC1_TYPES])
    spheres_per_site = float(np.sum(num * k_of))
    n_sites = int(n_spheres / spheres_per_site)
    site_vol = pitch ** 3 / math.sqrt(2.0)
    depth = 0.12 if n_sites > 200_000 else 0.06
    width = math.sqrt(n_sites * site_vol / (aspect * depth))
    length = aspect * width
    dom = Domain((-length / 2 - 0.3, -width / 2 - 0.05, -0.02),
                 (length / 2 + 0.3, width / 2 + 0.05, depth + 2.5 * wheel_radius + 0.3))
    sim = Simulator(dom, precision=precision, device=device, kt_device=kt_device)
    mat = sim.load_material(dict(GRC1_MATERIAL))
    tpls = grc1_templates(sim, mat)
    lift = GRC1_TYPES[0][0] / 2 + 1e-3     # the lowest (and outermost) sites clear the walls for any type
    pts = hcp_sample_box((0.0, 0.0, depth / 2 + lift), (length / 2 - lift, width / 2 - lift, depth / 2), pitch)
    pts = pts[:n_sites]
    kinds = rng.choice(len(GRC1_TYPES), size=pts.shape[0], p=num)
    # reach of each type from its centre (any orientation)
    reach = np.array([(k - 1) * 0.5 * (t[0] - 2 * t[1]) / max(k - 1, 1) + t[1]
                      for t, k in zip(GRC1_TYPES, k_of)])
    # a 21 mm type-1 clump clears every site it could touch: the others
    # within its reach + the largest other reach, other type-1 within twice
    # its reach
    big = np.nonzero(kinds == 0)[0]
    if big.size:
        from scipy.spatial import cKDTree
        keep = np.ones(pts.shape[0], dtype=bool)
        tree = cKDTree(pts)
        r_other = reach[0] + reach[1:].max() + 1e-4
        r_big = 2.0 * reach[0] + 1e-4
        for i in big:
            if keep[i]:
                for j in tree.query_ball_point(pts[i], max(r_other, r_big)):
                    if j != i and (kinds[j] == 0 or np.linalg.norm(pts[j] - pts[i]) < r_other):
                        keep[j] = False
        pts, kinds = pts[keep], kinds[keep]
    for t, (tid, tpl, _, size, k) in enumerate(tpls):
        sel = pts[kinds == t]
        if sel.shape[0] == 0:
            continue
        ids = np.asarray(sim.add_clumps(tid, sel), dtype=np.int64)
        q = rng.normal(size=(ids.size, 4))
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        sim.store.__dict__["_quat"][ids] = q
    surface = float(np.max(pts[:, 2] + reach[kinds]))   # the highest grain's top
    walls = [("plane", (0, 0, 0), (0, 0, 1), mat),
             ("plane", (-length / 2, 0, 0), (1, 0, 0), mat), ("plane", (length / 2, 0, 0), (-1, 0, 0), mat),
             ("plane", (0, -width / 2, 0), (0, 1, 0), mat), ("plane", (0, width / 2, 0), (0, -1, 0), mat)]
    sim.add_analytic(walls, family=255)
    sim.set_family_fixed(255)
    wheel_w = min(0.2, 0.6 * width)
    grouser = 0.08 * wheel_radius
    tris = grousered_wheel(radius=wheel_radius, width=wheel_w, grouser_h=grouser)
    x0 = -length / 2 + wheel_radius + grouser + 0.01
    # the terrain top under the wheel's lowest grouser (the grain reaching
    # highest within a grain size of the axle's vertical plane)
    foot = (np.abs(pts[:, 0] - x0) < 0.012) & (np.abs(pts[:, 1]) < wheel_w / 2)
    top_under = float(np.max(pts[foot, 2] + reach[kinds[foot]])) if foot.any() else surface
    z0 = top_under + wheel_radius + grouser - sinkage   # the lowest grouser tip `sinkage` into it
    sim.add_mesh(tris, mat, family=WHEEL_FAMILY, position=(x0, 0.0, z0))
    sim.set_family_prescribed_lin_vel(WHEEL_FAMILY, omega * wheel_radius * (1.0 - slip), 0.0, -plunge)
    sim.set_family_prescribed_ang_vel(WHEEL_FAMILY, 0.0, omega, 0.0)
    sim.set_gravity([0, 0, -G])
    sim.set_init_time_step(h)
    sim.set_error_out_velocity(v_err)
    sim.set_fixed_lookahead(n_max)
    return sim


# ---------------------------------------------------------------------------
# the paper's mixer timing scene (scenarios.py:752-838, `grainforge bench
# mixer`, cli.py:183-209): a cylindrical chamber, a rotating two-paddle blade
# mesh, granular fill of 1-, 3- or 6-sphere clumps above the blades.
# ---------------------------------------------------------------------------

def paddle_blades(nu: int = 6, nv: int = 1) -> np.ndarray:
    """Two crossed vertical paddles spanning x / y in [-0.9, 0.9], z in
    [-0.5, 0.5] (unit box), each an nu x nv quad grid (2 nu nv facets)."""
    tris = []
    for blade in (0, 1):
        for i in range(nu):
            for j in range(nv):
                u0, u1 = -0.9 + 1.8 * i / nu, -0.9 + 1.8 * (i + 1) / nu
                z0, z1 = -0.5 + j / nv, -0.5 + (j + 1) / nv
                pt = (lambda u, z: (u, 0.0, z)) if blade == 0 else (lambda u, z: (0.0, u, z))
                p00, p10, p01, p11 = pt(u0, z0), pt(u1, z0), pt(u0, z1), pt(u1, z1)
                tris.append((p00, p10, p11))
                tris.append((p00, p11, p01))
    return np.asarray(tris, dtype=np.float64)


def mixer(target_spheres: int, *, clump: str = "3sph", young: float = 1e7, omega: float = 2.0 * math.pi,
          precision: str = "f32", device: int = 0, h: float | None = None) -> tuple:
    """build_mixer_sim at the grain size that puts ~target_spheres in the
    fill (run_mixer_timing's sizing rule).  Returns (sim, meta)."""
    from .core import ClumpSphere
    from .engine import hcp_sample_cylinder
    per = {"spheres": 1, "3sph": 3, "6sph": 6}[clump]
    chamber_vol = math.pi * 0.25 * (1.0 / 3.0)
    n_clumps = target_spheres / per
    r = (chamber_vol * 0.42 / (n_clumps * per * 4.19)) ** (1 / 3)
    world = 1.0
    chamber_h = world / 3.0
    sim = Simulator(Domain.cube(world * 1.02), precision=precision, device=device)
    mat_mixer = sim.load_material({"E": young, "nu": 0.3, "CoR": 0.6, "mu": 0.5, "Crr": 0.0})
    mat_gran = sim.load_material({"E": young, "nu": 0.3, "CoR": 0.6, "mu": 0.2, "Crr": 0.0})
    sim.set_material_pair("mu", mat_mixer, mat_gran, 0.5)
    wall_fam, mixer_fam = 255, 10
    sim.add_analytic([("cylinder", (0, 0, 0), (0, 0, 1), world / 2, -1.0, mat_mixer),
                      ("plane", (0, 0, -world / 2), (0, 0, 1), mat_mixer),
                      ("plane", (0, 0, world / 2), (0, 0, -1), mat_mixer)], family=wall_fam)
    sim.set_family_fixed(wall_fam)
    m_id = sim.add_mesh(paddle_blades(), mat_mixer, family=mixer_fam, position=(0, 0, -world / 2 + chamber_h / 2))
    sim.store.scale_mesh(m_id, (world / 2 * 0.92, world / 2 * 0.92, chamber_h * 0.96))
    sim.set_family_prescribed_ang_vel(mixer_fam, "0", "0", f"{omega!r}")
    if clump == "spheres":
        spheres = (ClumpSphere(np.zeros(3), r, mat_gran),)
    elif clump == "3sph":
        spheres = tuple(ClumpSphere(np.array([dx, 0.0, 0.0]), r, mat_gran) for dx in (-r, 0.0, r))
    else:
        spheres = tuple(ClumpSphere(np.array(off) * r, r, mat_gran)
                        for off in ((-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)))
    density = 2.6e3
    mass = density * sum(4 / 3 * math.pi * s.radius ** 3 for s in spheres)
    span = max(np.linalg.norm(s.offset) + s.radius for s in spheres)
    tpl = ClumpTemplate(mass=mass, moi=np.array([0.4 * mass * span ** 2] * 3), spheres=spheres)
    tid = sim.load_clump_template(tpl)
    fill_bottom = -world / 2 + chamber_h
    pts = hcp_sample_cylinder((0, 0, fill_bottom + chamber_h / 2), world / 2 - 2.2 * span, chamber_h / 2 - span,
                              2.0 * span * 1.05)
    sim.add_clumps(tid, pts)
    if h is None:
        h = 0.3 / math.sqrt(2.0 * young * r * 0.02 / mass)
    sim.set_gravity([0, 0, -G])
    sim.set_init_time_step(h)
    sim.set_error_out_velocity(25.0)
    return sim, {"n_clumps": int(pts.shape[0]), "n_spheres": int(pts.shape[0]) * len(spheres), "h": h, "r": r}
