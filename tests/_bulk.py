"""Bulk-observable scenes shared by the reference fixture generator
(tests/golden/make_bulk.py, which passes the reference's `grainforge` module)
and the GPU tests (tests/test_gpu_bulk.py, which pass this package).  Both
sides build the scene through the same public Simulator API, so the only
difference is the engine underneath.

SURVEY.md §8(c), parity protocol leg 3: settled pile height (97th-percentile
centre z, the convention of scenarios.py:295), total kinetic energy, and the
crater penetration depth d = surface - (z_final - R) (scenarios.py:335-336)
after long runs.  Trajectories are chaotic, so these are compared as
observables with stated tolerances, not state by state.
"""

from __future__ import annotations

import math

import numpy as np

G = 9.81

# configs[0] / SURVEY §8(d) C1: r = 5 mm, rho = 2600, the test_engine.py:13-18 material
C1_R = 0.005
C1_RHO = 2600.0
C1_MATERIAL = {"E": 1e7, "nu": 0.3, "CoR": 0.6, "mu": 0.3, "Crr": 0.0}
C1_H = 1e-5
C1_V_ERR = 5.0


def c1_points(gf, n: int = 10_000) -> tuple[np.ndarray, float]:
    """HCP lattice of pitch 2r*1.02 filling a cube oversized 10 % for n
    points, truncated to exactly n (lowest layers first, no RNG).  Returns
    (points, wall half width)."""
    pitch = 2.0 * C1_R * 1.02
    per_volume = math.sqrt(2.0) / pitch ** 3           # HCP density at this pitch
    side = 1.1 * (n / per_volume) ** (1.0 / 3.0)
    half = side / 2.0
    pts = gf.hcp_sample_box((0.0, 0.0, half + 1.02 * C1_R), (half, half, half), pitch)
    order = np.lexsort((pts[:, 0], pts[:, 1], pts[:, 2]))
    if pts.shape[0] < n:
        raise RuntimeError(f"C1 lattice holds {pts.shape[0]} < {n} points")
    pts = pts[order[:n]]
    return pts, half + 1.5 * C1_R


def c1_box(gf, n: int = 10_000, n_max: int = 4, **sim_kw):
    """C1: n monodisperse spheres settling under gravity in a box, Hertz-
    Mindlin, floor + 4 fixed analytic side walls (family 255)."""
    pts, wall = c1_points(gf, n)
    dom = gf.Domain((-wall - 0.05, -wall - 0.05, -0.02), (wall + 0.05, wall + 0.05, 2.5 * wall + 0.2))
    sim = gf.Simulator(dom, **sim_kw)
    mat = sim.load_material(dict(C1_MATERIAL))
    m = C1_RHO * 4.0 / 3.0 * math.pi * C1_R ** 3
    tpl = sim.load_clump_template(gf.ClumpTemplate.solid_sphere(C1_R, m, mat))
    sim.add_clumps(tpl, pts)
    walls = [("plane", (0, 0, 0), (0, 0, 1), mat),
             ("plane", (-wall, 0, 0), (1, 0, 0), mat), ("plane", (wall, 0, 0), (-1, 0, 0), mat),
             ("plane", (0, -wall, 0), (0, 1, 0), mat), ("plane", (0, wall, 0), (0, -1, 0), mat)]
    sim.add_analytic(walls, family=255)
    sim.set_family_fixed(255)
    sim.set_gravity([0, 0, -G])
    sim.set_init_time_step(C1_H)
    sim.set_error_out_velocity(C1_V_ERR)
    sim.set_fixed_lookahead(n_max)
    return sim


def clump_rows(sim):
    """Indices of the free clump owners (no boundary owners)."""
    s = sim.store
    n = s.n_owners
    kind = np.asarray(s.owner_kind[:n])
    fam = np.asarray(s.owner_family[:n])
    return np.nonzero((kind == 0) & (fam != 255))[0]


def pile_height(sim) -> float:
    """97th-percentile owner centre z (scenarios.py:295)."""
    rows = clump_rows(sim)
    return float(np.percentile(np.asarray(sim._pos)[rows, 2], 97.0))


def kinetic_energy(sim) -> float:
    """Total translational + rotational kinetic energy of the free clumps."""
    s = sim.store
    rows = clump_rows(sim)
    v = np.asarray(s.lin_vel)[rows].astype(np.float64)
    w = np.asarray(s.ang_vel)[rows].astype(np.float64)
    m = np.asarray(s.mass)[rows].astype(np.float64)
    moi = np.asarray(s.moi)[rows].astype(np.float64)
    return float(0.5 * np.sum(m * np.sum(v * v, axis=1)) + 0.5 * np.sum(moi * w * w))


def run_c1(gf, t_end: float = 0.5, every: float = 0.05, **kw) -> dict:
    """Run C1 for t_end, sampling pile height and KE every `every` s."""
    sim = c1_box(gf, **kw)
    sim.initialize()
    out = {"t": [], "height": [], "ke": []}
    try:
        t = 0.0
        n_chunks = int(round(t_end / every))
        for _ in range(n_chunks):
            sim.do_dynamics(every)
            t += every
            out["t"].append(t)
            out["height"].append(pile_height(sim))
            out["ke"].append(kinetic_energy(sim))
    finally:
        sim.close()
    return {k: np.asarray(v) for k, v in out.items()}


# ---------------------------------------------------------------------------
# configs[1] crater: settle_crater_bed / run_crater_drop (scenarios.py:229-346)
# ---------------------------------------------------------------------------

CRATER_D = 0.0254


# The reference scenario runs at v_err = 30 m/s with the adaptive lookahead:
# a 24-48 mm detection margin around 1 cm grains, ~280 contact-array entries
# per grain, 2.3 s per step on the host (7.8 M entries at 28 k grains) -- a
# 1 s settle would take 6 h there.  The bulk fixtures use v_err = 5 m/s (still
# 2.5x the 20 cm impact speed, so the watchdog never trips) and a fixed
# lookahead of 2: a 4 mm margin.  Both engines run the same scene.
CRATER_V_ERR = 5.0
CRATER_N_MAX = 2
# the drop's watchdog: ejecta stay well below it (a 12 mm margin)
CRATER_DROP_V_ERR = 15.0


def crater_sim(gf, bed_half, depth, young, mu, grain_density, radii, h, v_err=CRATER_V_ERR,
               n_max=CRATER_N_MAX, **sim_kw):
    """The crater box of scenarios.py:229-253: five fixed analytic walls,
    one sphere template per grain radius."""
    dom = gf.Domain((-bed_half * 1.2, -bed_half * 1.2, -0.02),
                    (bed_half * 1.2, bed_half * 1.2, depth * 3.0 + 0.3))
    sim = gf.Simulator(dom, **sim_kw)
    props = {"E": young, "nu": 0.3, "CoR": 0.5, "mu": mu, "Crr": 0.01}
    grain = sim.load_material(dict(props))
    wall = sim.load_material(dict(props))
    tpls = [sim.load_clump_template(gf.ClumpTemplate.solid_sphere(
        float(r), grain_density * 4.0 / 3.0 * math.pi * float(r) ** 3, grain)) for r in radii]
    planes = [((0, 0, 0), (0, 0, 1)), ((-bed_half, 0, 0), (1, 0, 0)), ((bed_half, 0, 0), (-1, 0, 0)),
              ((0, -bed_half, 0), (0, 1, 0)), ((0, bed_half, 0), (0, -1, 0))]
    sim.add_analytic([("plane", p, nrm, wall) for p, nrm in planes], family=255)
    sim.set_family_fixed(255)
    sim.set_gravity([0, 0, -G])
    sim.set_init_time_step(h)
    sim.set_error_out_velocity(v_err)
    sim.set_fixed_lookahead(n_max)
    return sim, tpls, grain


def crater_settle(gf, seed: int = 7, settle_time: float = 1.0, **sim_kw) -> dict:
    """The pour and settle of settle_crater_bed (scenarios.py:256-307):
    bed 12 D x 12 D x 8 D, eleven diameters over the relative band
    [0.25, 0.35] sized for ~2e4 grains, an HCP lattice of pitch 1.01 d_max
    overfilled 12 % in height, shuffled and assigned sizes with
    default_rng(seed); settled in 0.1 s chunks until the fastest grain is
    below 0.08 m/s or settle_time elapsed (scenarios.py:24-35)."""
    rng = np.random.default_rng(seed)
    D = CRATER_D
    bed_half = 12.0 * D / 2.0
    depth = 8.0 * D
    packing = 1460.0 / 2500.0
    d_mean = (6.0 * (2 * bed_half) ** 2 * depth * packing / (math.pi * 2.0e4)) ** (1.0 / 3.0)
    dset = np.linspace(0.25, 0.35, 11) * (d_mean / 0.30)
    radii = dset / 2.0
    young, mu, h, rho_g = 5e6, 0.3, 1e-4, 2500.0
    sim, tpls, _ = crater_sim(gf, bed_half, depth, young, mu, rho_g, radii, h, **sim_kw)
    r_max = float(radii.max())
    fill_top = depth / packing * 1.12
    pts = gf.hcp_sample_box((0.0, 0.0, fill_top / 2.0 + r_max),
                            (bed_half - r_max * 1.05, bed_half - r_max * 1.05, fill_top / 2.0),
                            float(dset.max()) * 1.01)
    pts = pts[rng.permutation(pts.shape[0])]
    kinds = rng.integers(0, 11, pts.shape[0])
    for k, tpl in enumerate(tpls):
        sim.add_clumps(tpl, pts[kinds == k])
    sim.initialize()
    try:
        probe = sim.create_inspector("clump_max_absv")
        t = 0.0
        while t < settle_time:
            sim.do_dynamics(0.1)
            t += 0.1
            if probe.get_value() < 0.08:
                break
        n = sim.store.n_owners
        rows = clump_rows(sim)
        pos = np.asarray(sim._pos)[rows].copy()
        tpl = np.asarray(sim.store.owner_template[:n])[rows].astype(np.int32)
        surface = float(np.percentile(pos[:, 2], 97.0))
        grain_mass = float(np.sum(rho_g * 4.0 / 3.0 * math.pi * radii[tpl] ** 3))
        bulk = grain_mass / ((2 * bed_half) ** 2 * surface)
        ke = kinetic_energy(sim)
    finally:
        sim.close()
    return {"positions": pos, "template": tpl, "radii": radii, "surface_z": surface,
            "bulk_density": bulk, "mu": mu, "young": young, "h": h, "box_half": bed_half,
            "depth": depth, "settle_t": t, "ke": ke}


def crater_drop(gf, bed: dict, ball_density: float, drop_height: float,
                grain_density: float = 2500.0, sim_time: float = 0.5, **sim_kw) -> dict:
    """Release the projectile 2 mm above the settled bed `bed` (the fixture
    dict: per-template positions, radii, surface, bulk density, mu, young,
    h, box half width, depth) with the free-fall speed of `drop_height`;
    run in 0.05 s chunks until 0.5 s or |v| < 0.02 m/s after 0.15 s
    (scenarios.py:310-346).  Returns depth_cm and the ball's z history."""
    sim_kw.setdefault("v_err", CRATER_DROP_V_ERR)
    sim, tpls, grain = crater_sim(gf, bed["box_half"], bed["depth"], bed["young"], bed["mu"],
                                  grain_density, bed["radii"], bed["h"], **sim_kw)
    for k, tpl in enumerate(tpls):
        pts = bed["positions"][bed["template"] == k]
        if pts.shape[0]:
            sim.add_clumps(tpl, pts)
    R = CRATER_D / 2.0
    mass = ball_density * 4.0 / 3.0 * math.pi * R ** 3
    btpl = sim.load_clump_template(gf.ClumpTemplate.solid_sphere(R, mass, grain))
    # 2 mm above the surface (scenarios.py:326-328) -- and above every grain
    # under the ball's footprint: the 97th-percentile surface leaves the top
    # grains inside a ball placed at surface + R + 2 mm, and the overlap
    # kicks them to 8-20 m/s in the first step (a deviation from the
    # reference scenario, which absorbs that with its 30 m/s watchdog)
    pos, rg = bed["positions"], np.asarray(bed["radii"])[bed["template"]]
    under = np.hypot(pos[:, 0], pos[:, 1]) < R + rg
    top = float(np.max(pos[under, 2] + rg[under])) if np.any(under) else -np.inf
    z0 = max(bed["surface_z"], top) + R + 2e-3
    ball = sim.add_clumps(btpl, [[0.0, 0.0, z0]])[0]
    tr = sim.track(ball)
    tr.set_vel([0.0, 0.0, -math.sqrt(2.0 * G * drop_height)])
    sim.initialize()
    zs = []
    try:
        t = 0.0
        while t < sim_time:
            sim.do_dynamics(0.05)
            t += 0.05
            zs.append(float(tr.pos()[2]))
            if t > 0.15 and float(np.linalg.norm(tr.vel())) < 0.02:
                break
        z_final = float(tr.pos()[2])
    finally:
        sim.close()
    d = max(bed["surface_z"] - (z_final - R), 1e-6)
    return {"depth_cm": d * 100.0, "z": np.asarray(zs), "t_end": t}


def crater_fixed_point(mu, rho_b, rho_g, D_cm, h_cm, C=0.14):
    """d = (C/mu) sqrt(rho_b/rho_g) D^(2/3) (h + d)^(1/3) solved by
    iteration (scenarios.py:356-363, the paper's Eq. (7))."""
    k = (C / mu) * math.sqrt(rho_b / rho_g) * D_cm ** (2.0 / 3.0)
    d = k * h_cm ** (1.0 / 3.0)
    for _ in range(200):
        d = k * (h_cm + d) ** (1.0 / 3.0)
    return d


# ---------------------------------------------------------------------------
# configs[2] hopper discharge: run_hopper test 2 (scenarios.py:486-575) --
# five-sphere WC cylinder clumps (_cylinder_clump :386-398, DRUM_SETUPS WC)
# in a flat-bottom hopper discharging through a slot.  `scale` multiplies
# the hopper (width, depth, layer height, orifice) at fixed particle size
# (x3.68 for ~1 M clumps); `fill` is the reference's
# fill_scale.  v_err / lookahead reduced as for the crater fixtures.
# ---------------------------------------------------------------------------

HOPPER_H = 4e-5
HOPPER_V_ERR = 5.0
HOPPER_N_MAX = 2
WC = dict(radius=2.0e-3, length=8.5e-3, density=476.0, E=1e7, nu=0.35, CoR=0.55)


def cylinder_clump(gf, radius, length, density, material, n_spheres=5):
    """Five spheres on the axis; mass / MOI of the ideal cylinder."""
    vol = math.pi * radius ** 2 * length
    mass = density * vol
    ixx = mass * (3 * radius ** 2 + length ** 2) / 12.0
    izz = 0.5 * mass * radius ** 2
    span = length - 2 * radius
    zs = np.linspace(-span / 2.0, span / 2.0, n_spheres)
    spheres = tuple(gf.ClumpSphere(np.array([0.0, 0.0, z]), radius, material) for z in zs)
    return gf.ClumpTemplate(mass=mass, moi=np.array([ixx, ixx, izz]), spheres=spheres)


def quad(x0, x1, y0, y1, z):
    """Two facets covering [x0, x1] x [y0, y1] at height z."""
    p00, p10, p01, p11 = (x0, y0, z), (x1, y0, z), (x0, y1, z), (x1, y1, z)
    return np.array([(p00, p10, p11), (p00, p11, p01)], dtype=np.float64)


def hopper_sim(gf, scale: float = 1.0, fill: float = 1.0, orifice: float = 0.04, mu_i: float = 0.70,
               cr: float = 0.07, h: float = HOPPER_H, v_err: float = HOPPER_V_ERR, n_max: int = HOPPER_N_MAX,
               **sim_kw):
    """Returns (sim, n_clumps, clump_mass, gate_family)."""
    width, depth_y, height = 0.20 * scale, 0.04 * scale, 0.40 * scale
    lo = (-0.13 * scale, -0.05 * scale, -0.32 * scale)
    hi = (0.13 * scale, 0.05 * scale, 0.10 * scale + 0.40 * scale * fill + 0.05)
    sim = gf.Simulator(gf.Domain(lo, hi), **sim_kw)
    gate_fam, wall_fam = 20, 255
    wall = sim.load_material({"E": WC["E"], "nu": 0.3, "CoR": 0.5, "mu": 0.45, "Crr": 0.0})
    mat = sim.load_material({"E": WC["E"], "nu": WC["nu"], "CoR": WC["CoR"], "mu": mu_i, "Crr": cr})
    tpl = cylinder_clump(gf, WC["radius"], WC["length"], WC["density"], mat)
    tid = sim.load_clump_template(tpl)
    hw, hd, so = width / 2, depth_y / 2, (orifice * scale) / 2
    floor = np.concatenate([quad(-hw, -so, -hd, hd, 0.0), quad(so, hw, -hd, hd, 0.0)])
    sim.add_mesh(floor, wall, family=wall_fam)
    sim.add_mesh(quad(-so, so, -hd, hd, -1e-4), wall, family=gate_fam)
    for x, nx in ((-hw, 1.0), (hw, -1.0)):
        sim.add_analytic([("plane", (x, 0, -0.3 * scale), (nx, 0, 0), wall)], family=wall_fam)
    for y, ny in ((-hd, 1.0), (hd, -1.0)):
        sim.add_analytic([("plane", (0, y, 0), (0, ny, 0), wall)], family=wall_fam)
    sim.add_analytic([("plane", (0, 0, -0.30 * scale), (0, 0, 1), wall)], family=wall_fam)
    sim.set_family_fixed(wall_fam)
    sim.set_family_fixed(gate_fam)
    layer_h = 0.36 * scale * fill
    spacing = WC["length"] * 1.06
    # the reference offsets the lattice by 1.2 r above the floor
    # (scenarios.py:540); its upright 8.5 mm rods then start inside the floor
    # plate, so here the lowest rod end clears it by 1 mm
    pts = gf.hcp_sample_box((0, 0, layer_h / 2 + WC["length"] / 2 + 1e-3),
                            (hw - 1.6 * WC["radius"], hd - 1.6 * WC["radius"], layer_h / 2), spacing)
    sim.add_clumps(tid, pts)
    sim.set_gravity([0, 0, -G])
    sim.set_init_time_step(h)
    sim.set_error_out_velocity(v_err)
    sim.set_fixed_lookahead(n_max)
    return sim, int(pts.shape[0]), float(tpl.mass), gate_fam


def settle(sim, max_time, calm=0.1, threshold=0.12):
    """scenarios.py:24-35"""
    probe = sim.create_inspector("clump_max_absv")
    t = 0.0
    while t < max_time:
        sim.do_dynamics(calm)
        t += calm
        if probe.get_value() < threshold:
            break
    return t


def run_hopper(gf, scale=1.0, fill=0.25, settle_time=0.6, discharge_time=1.0, sample_dt=0.1, **kw) -> dict:
    """Settle, open the gate (mask it against the grains), sample the
    discharged mass fraction (clumps below z = -0.05 scale) every sample_dt
    (scenarios.py:552-575)."""
    sim, n_clumps, cmass, gate_fam = hopper_sim(gf, scale=scale, fill=fill, **kw)
    sim.initialize()
    try:
        t_settle = settle(sim, settle_time)
        sim.set_family_mask(gate_fam, 0, False)
        t, ts, frac = 0.0, [0.0], [0.0]
        while t < discharge_time - 1e-9:
            sim.do_dynamics(sample_dt)
            t += sample_dt
            z = np.asarray(sim._pos)[:n_clumps, 2]
            ts.append(t)
            frac.append(float(np.mean(z < -0.05 * scale)))
    finally:
        sim.close()
    return {"t": np.asarray(ts), "frac": np.asarray(frac), "n_clumps": n_clumps, "settle_t": t_settle}


# ---------------------------------------------------------------------------
# bonded granite block (the breakage model, forces.py:185-291; init_bonds,
# engine.py:409-427): a 6 x 6 x 4 cubic block of touching 12 mm spheres,
# bonded (gamma_int 1.01), dropped from 2 cm onto a fixed plane.
# ---------------------------------------------------------------------------

GRANITE = {"E": 60e9, "nu": 0.25, "CoR": 0.5, "mu": 0.3, "Crr": 0.0, "tension": -9.3e6, "cohesion": 200e6}
BLOCK_R = 12e-3


def bonded_block(gf, drop=0.02, h=1e-6, **sim_kw):
    sim = gf.Simulator(gf.Domain((-0.2, -0.2, -0.05), (0.2, 0.2, 0.35)), "breakage", **sim_kw)
    mat = sim.load_material(dict(GRANITE))
    m = 2650.0 * 4.0 / 3.0 * math.pi * BLOCK_R ** 3
    tpl = sim.load_clump_template(gf.ClumpTemplate.solid_sphere(BLOCK_R, m, mat))
    g = (np.arange(6) - 2.5) * 2 * BLOCK_R
    gz = np.arange(4) * 2 * BLOCK_R + BLOCK_R + drop
    pts = np.array([(x, y, z) for z in gz for y in g for x in g])
    sim.add_clumps(tpl, pts)
    sim.add_analytic([("plane", (0, 0, 0), (0, 0, 1), mat)], family=255)
    sim.set_family_fixed(255)
    sim.set_gravity([0, 0, -G])
    sim.set_init_time_step(h)
    sim.set_error_out_velocity(5.0)
    sim.set_fixed_lookahead(4)
    stats = sim.init_bonds(1.01)
    return sim, int(pts.shape[0]), stats


def run_bonded_block(gf, t_end=0.08, every=0.002, **kw) -> dict:
    sim, n, stats = bonded_block(gf, **kw)
    sim.initialize()
    out = {"t": [0.0], "intact": [int(stats["count"])], "com_z": []}
    try:
        out["com_z"].append(float(np.mean(np.asarray(sim._pos)[:n, 2])))
        t = 0.0
        while t < t_end - 1e-12:
            sim.do_dynamics(every)
            t += every
            wild = np.asarray(sim._wild)
            intact = int(np.sum(wild[:, 4] > 0.0)) if wild.size else 0
            out["t"].append(t)
            out["intact"].append(intact)
            out["com_z"].append(float(np.mean(np.asarray(sim._pos)[:n, 2])))
    finally:
        sim.close()
    return {k: np.asarray(v) for k, v in out.items()}


# ---------------------------------------------------------------------------
# a stretched bond (bond persistence, engine.py:639-662): two touching soft
# spheres bonded with an unbreakable tension, launched apart; they oscillate
# with an amplitude (~2 mm) larger than the detection margin, so the
# detection loses the pair every half period and the persistence rule must
# keep re-appending the intact bond.
# ---------------------------------------------------------------------------

SOFT_BOND = {"E": 1e5, "nu": 0.25, "CoR": 0.5, "mu": 0.3, "Crr": 0.0, "tension": -1e7, "cohesion": 1e7}


def stretched_bond(gf, t_end=0.06, every=0.002, v0=0.5, h=1e-5, **sim_kw):
    sim = gf.Simulator(gf.Domain((-0.1, -0.1, -0.1), (0.1, 0.1, 0.1)), "breakage", **sim_kw)
    mat = sim.load_material(dict(SOFT_BOND))
    r = BLOCK_R
    m = 2650.0 * 4.0 / 3.0 * math.pi * r ** 3
    tpl = sim.load_clump_template(gf.ClumpTemplate.solid_sphere(r, m, mat))
    a, b = sim.add_clumps(tpl, [[-r, 0.0, 0.0], [r, 0.0, 0.0]])
    sim.track(a).set_vel([-v0, 0.0, 0.0])
    sim.track(b).set_vel([v0, 0.0, 0.0])
    sim.set_init_time_step(h)
    sim.set_error_out_velocity(5.0)
    sim.set_fixed_lookahead(4)
    stats = sim.init_bonds(1.01)
    sim.initialize()
    out = {"t": [], "gap": [], "intact": []}
    try:
        t = 0.0
        while t < t_end - 1e-12:
            sim.do_dynamics(every)
            t += every
            p = np.asarray(sim._pos)
            wild = np.asarray(sim._wild)
            out["t"].append(t)
            out["gap"].append(float(p[b, 0] - p[a, 0] - 2 * r))
            out["intact"].append(int(np.sum(wild[:, 4] > 0.0)) if wild.size else 0)
    finally:
        sim.close()
    res = {k: np.asarray(v) for k, v in out.items()}
    res["bonds"] = int(stats["count"])
    res["margin"] = float(sim._current_margin()) if hasattr(sim, "_current_margin") else 0.0
    return res
