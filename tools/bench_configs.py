"""Throughput of the other BASELINE.json configs on one GPU (their parity is
tested in tests/; bench.py times configs[1]).  Timed like bench.py: CUDA
events on the dT stream over K steps after an untimed settle + warm-up, kT
joined.  One JSON line per config on stdout.

  cohesive  configs[3]: the crater bed at 4M spheres with the NVRTC-compiled
            cohesive Hertz-Mindlin user model (models.py)
  hopper    configs[2]: the reference's hopper test 2 (five-sphere WC
            cylinder clumps, scenarios.py:486-575) scaled at fixed particle
            size to ~1M clumps (5M spheres), settled, gate opened, timed
            while discharging (tests/_bulk.py hopper_sim)
  clumps    1M five-sphere cylinder clumps settling in a box
  rover     configs[4]: the grousered wheel (prescribed 0.8 rad/s) rolling
            through an 11M-sphere GRC-1-like clump terrain at h = 2e-6
            (scenes.rover_wheel); the terrain settles first at h = 1e-5

The timed window has no per-kernel events in it; kernel times come from a
separate profiled window after it.

usage: python tools/bench_configs.py [--configs cohesive,hopper,rover] [--steps 100]
"""

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(sim, steps, warmup, prof_steps=10):
    import torch
    from paper_2311_04648_b200 import _lib
    sim.do_dynamics(warmup * sim.h)
    torch.cuda.synchronize()
    dev0 = sim.scheduler.timing["dyn_force"]
    sim.do_dynamics(steps * sim.h)
    torch.cuda.synchronize()
    dt_ms = (sim.scheduler.timing["dyn_force"] - dev0) * 1e3
    rr = sim.last_run
    # per-kernel events only in a separate window after the timed one
    sim._ctx.call("gf_set_profiling", C.c_int(1))
    sim.do_dynamics(prof_steps * sim.h)
    torch.cuda.synchronize()
    times = np.zeros(6)
    sim._ctx.call("gf_kernel_times", _lib.ptr(times))
    sim._ctx.call("gf_set_profiling", C.c_int(0))
    n_s = int(sim._sph_geom.size)
    steps_prof = max(1.0, times[4])
    return {"n_spheres": n_s, "n_owners": int(sim.store.n_owners), "steps": steps,
            "ms_per_step": dt_ms / steps,
            "M_sphere_steps_per_s": n_s * steps / (dt_ms * 1e-3) / 1e6,
            "M_owner_steps_per_s": sim.store.n_owners * steps / (dt_ms * 1e-3) / 1e6,
            "avg_acs": float(rr.sum_acs) / max(1, steps),
            "avg_touching_pairs": float(rr.sum_touch_pairs) / max(1, steps),
            "contact_phase_ms": times[0] / steps_prof, "k_integrate_ms": times[2] / steps_prof}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cohesive,hopper,rover")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--settle-steps", type=int, default=6000)
    ap.add_argument("--hopper-scale", type=float, default=5.85, help="~1M clumps at fill 1")
    ap.add_argument("--hopper-settle", type=float, default=0.6)
    ap.add_argument("--rover-spheres", type=int, default=11_000_000)
    ap.add_argument("--rover-settle-steps", type=int, default=25_000)
    ap.add_argument("--rover-settle-verr", type=float, default=20.0, help="watchdog speed while the terrain settles")
    ap.add_argument("--rover-sinkage", type=float, default=0.01, help="grouser-tip sinkage before timing (m)")
    args = ap.parse_args()
    from paper_2311_04648_b200 import models, scenes
    for name in args.configs.split(","):
        try:
            run_one(name, args, models, scenes)
        except Exception as exc:   # one config failing must not hide the others
            import traceback
            traceback.print_exc()
            print(json.dumps({"config": name, "error": f"{type(exc).__name__}: {exc}"}), flush=True)


def rover_clearance(sim, wp, cen, rad):
    """Smallest vertical gap between the wheel's lower envelope (a circle of
    the grouser-tip radius about the axle, over the wheel's width) and the
    grains under it."""
    tw = sim._tri_world.reshape(-1, 3, 3)
    ylo, yhi = float(tw[:, :, 1].min()), float(tw[:, :, 1].max())
    rg = float(wp[2] - tw[:, :, 2].min())
    sel = (cen[:, 1] > ylo) & (cen[:, 1] < yhi) & (np.abs(cen[:, 0] - wp[0]) < rg)
    dx = cen[sel, 0] - wp[0]
    bottom = wp[2] - np.sqrt(np.maximum(rg * rg - dx * dx, 0.0))
    return float(np.min(bottom - (cen[sel, 2] + rad[sel])))


def run_one(name, args, models, scenes):
    if True:
        t0 = time.perf_counter()
        if name == "cohesive":
            models.cohesive_model()
            sim = scenes.crater_bed(4_000_000, hold_ball=True, force_model="hertz_mindlin_cohesive",
                                    extra_props={"coh": 1.0e4})
            sim.initialize()
            sim.do_dynamics(args.settle_steps * sim.h)
            scenes.release_balls(sim)
            rec = {"config": "configs[3]: crater bed, 4M spheres, cohesive Hertz-Mindlin via NVRTC (coh 1e4 Pa)"}
        elif name == "hopper":
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            import _bulk as BK
            import paper_2311_04648_b200 as gf
            # discharged clumps fall up to ~1.7 m below the orifice: a 10 m/s watchdog
            # (h = 2e-5: at the scaled column height 4e-5 -- the reference's
            # step for its 0.4 m hopper -- let a clump reach 15-30 m/s)
            sim, n_clumps, _, gate = BK.hopper_sim(gf, scale=args.hopper_scale, fill=1.0, precision="f32",
                                                   v_err=10.0, h=2e-5)
            sim.initialize()
            BK.settle(sim, args.hopper_settle)
            sim.set_family_mask(gate, 0, False)
            sim.do_dynamics(0.05)   # the discharge under way
            rec = {"config": f"configs[2]: hopper test 2 scaled x{args.hopper_scale} at fixed particle size, "
                             f"{n_clumps} five-sphere WC cylinder clumps, discharging through the orifice"}
        elif name == "rover":
            # the terrain settles with the wheel held still just above it
            # (untimed input preparation at h = 4e-6), the wheel is pushed
            # down into the settled surface, then rolls: timed at h = 2e-6
            # (the dense layered bed -- scenes.rover_wheel packing "dense" --
            # closes its 5 % gaps within ~0.05 s; the settle runs with a loose
            # watchdog, 8 m/s once timed)
            sim = scenes.rover_wheel(args.rover_spheres, h=4e-6, sinkage=0.0, plunge=0.0, v_err=args.rover_settle_verr)
            fam = scenes.WHEEL_FAMILY
            sim.set_family_prescribed_lin_vel(fam, 0.0, 0.0, 0.0)
            sim.set_family_prescribed_ang_vel(fam, 0.0, 0.0, 0.0)
            sim.initialize()
            # 25k steps at 4e-6 = 0.1 s
            sim.do_dynamics(max(args.settle_steps, args.rover_settle_steps) * sim.h)
            fam_of = sim.store.__dict__["_owner_family"][:sim.store.n_owners]
            wheel = sim.track(int(np.nonzero(fam_of == fam)[0][0]))
            # the dense layered bed settles by a few per cent: move the wheel
            # down onto the settled surface, 0.2 mm above the first grain its
            # grouser-tip envelope would meet
            cen, rad = sim._sph_centers, np.asarray(sim._sph_radius, np.float64)
            wp = wheel.pos()
            t_down = rover_clearance(sim, wp, cen, rad) - 2e-4
            wheel.set_pos([wp[0], wp[1], wp[2] - t_down])
            # then down at 0.2 m/s (still at the settling step), 0.4 mm per
            # check, until the grouser tips sit `rover_sinkage` into the bed;
            # then roll at the timed step
            def wheel_entries():
                kind = sim._acs_arrays()[0]
                return int(np.sum(kind == 1))
            sim.set_family_prescribed_lin_vel(fam, 0.0, 0.0, -0.2)
            n_down, trace = 0, []
            n_checks = int(round(args.rover_sinkage / 4e-4))
            ztrace = []
            while n_down < n_checks:
                trace.append(wheel_entries())
                ztrace.append(round(float(wheel.pos()[2]), 5))
                sim.do_dynamics(0.002)
                n_down += 1
            trace.append(wheel_entries())
            sim.set_init_time_step(2e-6)
            sim.set_error_out_velocity(8.0)
            sim.set_family_prescribed_lin_vel(fam, 0.8 * 0.25 * 0.8, 0.0, -0.01)
            sim.set_family_prescribed_ang_vel(fam, 0.0, 0.8, 0.0)
            sim.do_dynamics(0.004)
            rec = {"config": f"configs[4]: grousered wheel (0.8 rad/s, 20% slip) on a {args.rover_spheres}-sphere "
                             "GRC-1-like clump terrain, h = 2e-6"}
            rec["terrain"] = {k: float(v) for k, v in sim.rover_bed.items()}
            rec["wheel_lowered_m"] = t_down
            rec["wheel_plunge_checks"] = n_down
            rec["wheel_entries_per_check"] = trace
            rec["wheel_z_per_check"] = ztrace
            rec["wheel_force_N_before_timed"] = [float(x) for x in wheel.contact_force()]
            rec["wheel_contact_entries_before_timed"] = wheel_entries()
        elif name == "clumps":
            sim = scenes.clump_bed(1_000_000)
            sim.initialize()
            sim.do_dynamics(args.settle_steps * sim.h)
            rec = {"config": "configs[2]: 1M five-sphere cylinder clumps (5M spheres) settling in a box"}
        else:
            raise SystemExit(f"unknown config {name}")
        rec["setup_and_settle_s"] = time.perf_counter() - t0
        rec["settle_steps"] = args.settle_steps
        rec.update(timed(sim, args.steps, args.warmup))
        sim.close()
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
