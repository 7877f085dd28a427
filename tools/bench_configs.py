"""Throughput of the other BASELINE.json configs on one GPU (their parity is
tested in tests/; bench.py times configs[1]).  Timed like bench.py: CUDA
events on the dT stream over K steps after an untimed settle + warm-up, kT
joined.  One JSON line per config on stdout.

  cohesive  configs[3]: the crater bed at 4M spheres with the NVRTC-compiled
            cohesive Hertz-Mindlin user model (models.py)
  clumps    configs[2]: 1M five-sphere cylinder clumps (5M spheres) settling
            in a box (the clump owner-reduction path)

usage: python tools/bench_configs.py [--configs cohesive,clumps] [--steps 100]
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


def timed(sim, steps, warmup):
    import torch
    from paper_2311_04648_b200 import _lib
    sim.do_dynamics(warmup * sim.h)
    sim._ctx.call("gf_set_profiling", C.c_int(1))
    torch.cuda.synchronize()
    dev0 = sim.scheduler.timing["dyn_force"]
    sim.do_dynamics(steps * sim.h)
    torch.cuda.synchronize()
    dt_ms = (sim.scheduler.timing["dyn_force"] - dev0) * 1e3
    times = np.zeros(6)
    sim._ctx.call("gf_kernel_times", _lib.ptr(times))
    rr = sim.last_run
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
    ap.add_argument("--configs", default="cohesive,clumps")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--settle-steps", type=int, default=6000)
    args = ap.parse_args()
    from paper_2311_04648_b200 import models, scenes
    for name in args.configs.split(","):
        t0 = time.perf_counter()
        if name == "cohesive":
            models.cohesive_model()
            sim = scenes.crater_bed(4_000_000, hold_ball=True, force_model="hertz_mindlin_cohesive",
                                    extra_props={"coh": 1.0e4})
            sim.initialize()
            sim.do_dynamics(args.settle_steps * sim.h)
            scenes.release_balls(sim)
            rec = {"config": "configs[3]: crater bed, 4M spheres, cohesive Hertz-Mindlin via NVRTC (coh 1e4 Pa)"}
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
