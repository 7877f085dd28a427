"""`grainforge bench mixer` on the B200 (cli.py:183-209, scenarios.py:
813-838): the mixer scene at several component-sphere counts, time per step
after a settle, and the scaling exponent of time per step vs N (log-log
fit).  Device time: CUDA events on the dT stream (kT joined), not wall
clock.  Writes <out>/mixer_scaling.csv and mixer_summary.json.

usage: python tools/bench_mixer.py [--n 100000 1000000 ...] [--clump 3sph] [--steps 400] [--out DIR]
"""

import argparse
import csv
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="*", default=[100_000, 1_000_000, 4_000_000, 16_000_000])
    ap.add_argument("--clump", default="3sph", choices=["spheres", "3sph", "6sph"])
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--settle-time", type=float, default=0.02)
    ap.add_argument("--out", default="gpurun_out/mixer")
    ap.add_argument("--v-err", type=float, default=10.0)
    ap.add_argument("--h-scale", type=float, default=0.1)
    args = ap.parse_args()
    import torch
    from paper_2311_04648_b200 import scenes
    rows = []
    for n in args.n:
        sim, meta = scenes.mixer(int(n), clump=args.clump)
        # the reference's step, 0.3 / sqrt(k / m) (proportional to the grain
        # size), with its 25 m/s watchdog gives a detection margin of ~17 grain
        # radii (thousands of candidate pairs per grain); here the step is
        # h_scale x the reference's (still proportional to the grain size, so
        # the margin / radius ratio -- and the work per sphere -- is the same
        # at every N) and 10 m/s (blade tips move at 2.9 m/s) with a fixed
        # lookahead of 2: a ~0.7-radius margin (documented deviation; time per
        # step vs N is the measured quantity)
        sim.set_init_time_step(meta["h"] * args.h_scale)
        meta["h"] = sim.h
        sim.set_error_out_velocity(args.v_err)
        sim.set_fixed_lookahead(2)
        sim.initialize()
        sim.do_dynamics(args.settle_time)
        torch.cuda.synchronize()
        d0 = sim.scheduler.timing["dyn_force"]
        sim.do_dynamics(args.steps * sim.h)
        torch.cuda.synchronize()
        ms = (sim.scheduler.timing["dyn_force"] - d0) * 1e3 / args.steps
        row = {"target": int(n), "n_spheres": meta["n_spheres"], "n_clumps": meta["n_clumps"], "h": meta["h"],
               "steps": args.steps, "ms_per_step": ms,
               "M_sphere_steps_per_s": meta["n_spheres"] / (ms * 1e-3) / 1e6}
        sim.close()
        rows.append(row)
        print(f"N={row['n_spheres']:9d} spheres: {ms:.3f} ms/step, {row['M_sphere_steps_per_s']:.0f} M sphere-steps/s",
              flush=True)
    exponent = float("nan")
    if len(rows) >= 2:
        x = np.log([r["n_spheres"] for r in rows])
        y = np.log([r["ms_per_step"] for r in rows])
        exponent = float(np.polyfit(x, y, 1)[0])
    os.makedirs(args.out, exist_ok=True)
    with open(os.path.join(args.out, "mixer_scaling.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)
    with open(os.path.join(args.out, "mixer_summary.json"), "w") as f:
        json.dump({"exponent": exponent, "clump": args.clump, "rows": rows}, f, indent=1)
    print(f"scaling exponent {exponent:.3f}")


if __name__ == "__main__":
    main()
