import sys, os, time, json
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
from bench_configs import rover_clearance
from paper_2311_04648_b200 import scenes
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
sim = scenes.rover_wheel(n, h=4e-6, sinkage=0.0, plunge=0.0, v_err=50.0)
fam = scenes.WHEEL_FAMILY
sim.set_family_prescribed_lin_vel(fam, 0.0, 0.0, 0.0)
sim.set_family_prescribed_ang_vel(fam, 0.0, 0.0, 0.0)
sim.initialize()
t0 = time.time()
sim.do_dynamics(60000 * sim.h)
print("settled", time.time() - t0, flush=True)
fam_of = sim.store.__dict__["_owner_family"][:sim.store.n_owners]
wheel = sim.track(int(np.nonzero(fam_of == fam)[0][0]))
cen, rad = sim._sph_centers, np.asarray(sim._sph_radius, np.float64)
print("n_sph", cen.shape, "rad min/max", rad.min(), rad.max(), "grain top z", float(np.max(cen[:, 2] + rad)),
      "p50 top", float(np.percentile(cen[:, 2] + rad, 50)), flush=True)
wp = wheel.pos()
tw = sim._tri_world.reshape(-1, 3, 3)
print("wheel pos", wp, "tri z range", float(tw[:, :, 2].min()), float(tw[:, :, 2].max()),
      "tri x", float(tw[:, :, 0].min()), float(tw[:, :, 0].max()), "tri y", float(tw[:, :, 1].min()), float(tw[:, :, 1].max()), flush=True)
wp[0] = -0.5 if n > 5e6 else wp[0] + 0.05
cl = rover_clearance(sim, wp, cen, rad)
print("clearance at", wp, cl, flush=True)
wheel.set_pos([wp[0], wp[1], wp[2] - (cl - 2e-4)])
def entries():
    a = sim._acs_arrays()
    kind = a[0]
    return int(np.sum(kind == 1))
sim.set_family_prescribed_lin_vel(fam, 0.0, 0.0, -0.2)
for i in range(40):
    e = entries()
    wpn = wheel.pos()
    tw = sim._tri_world.reshape(-1, 3, 3)
    cen, rad = sim._sph_centers, np.asarray(sim._sph_radius, np.float64)
    v = np.linalg.norm(np.asarray(sim.store.__dict__["_lin_vel"][:sim.store.n_owners]), axis=1) if False else None
    print(i, "wheel z", round(float(wpn[2]), 5), "tri zmin", round(float(tw[:, :, 2].min()), 5), "entries", e,
          "force", [round(float(x), 3) for x in wheel.contact_force()], "clear", round(rover_clearance(sim, wpn, cen, rad), 5), flush=True)
    sim.do_dynamics(0.002)
