"""Size sweep on one GPU (configs[4]: "1M-150M sphere scaling sweep"): the
settled 1M-sphere crater bed of bench.py, tiled tx x ty side by side in one
box (scenes.tiled_bed), timed like bench.py (CUDA events on the dT stream,
kT joined) at each size.  One JSON line per size on stdout.

usage: python tools/sweep.py [--tiles 1,2,4,8,16,32,64,128] [--steps 40] [--warmup 10]
"""

import argparse
import ctypes as C
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def factor(t):
    """tx x ty = t, as square as possible"""
    ty = int(math.isqrt(t))
    while t % ty:
        ty -= 1
    return t // ty, ty


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", default="1,2,4,8,16,32,64,128")
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--settle-steps", type=int, default=12000)
    ap.add_argument("--n-spheres", type=int, default=1_000_000)
    args = ap.parse_args()
    import torch
    from paper_2311_04648_b200 import _lib, scenes

    src = scenes.crater_bed(args.n_spheres, hold_ball=True)
    src.initialize()
    t0 = time.perf_counter()
    src.do_dynamics(args.settle_steps * src.h)
    scenes.release_balls(src)
    src.store.voxel  # host mirror of the settled state
    settle_s = time.perf_counter() - t0
    for t in [int(x) for x in args.tiles.split(",")]:
        tx, ty = factor(t)
        rec = {"tiles": t, "layout": f"{tx}x{ty}"}
        try:
            t_b = time.perf_counter()
            sim = scenes.tiled_bed(src, tx, ty)
            sim.initialize()
            rec["setup_s"] = time.perf_counter() - t_b
            sim.do_dynamics(args.warmup * sim.h)
            ctx = sim._ctx
            ctx.call("gf_set_profiling", C.c_int(1))
            torch.cuda.synchronize()
            dev0 = sim.scheduler.timing["dyn_force"]
            sim.do_dynamics(args.steps * sim.h)
            torch.cuda.synchronize()
            dt_ms = (sim.scheduler.timing["dyn_force"] - dev0) * 1e3
            times = np.zeros(6)
            ctx.call("gf_kernel_times", _lib.ptr(times))
            free, total = torch.cuda.mem_get_info(0)
            n_s = int(sim._sph_geom.size)
            rr = sim.last_run
            steps_prof = max(1.0, times[4])
            rec.update({
                "n_spheres": n_s, "ms_per_step": dt_ms / args.steps,
                "M_sphere_steps_per_s": n_s * args.steps / (dt_ms * 1e-3) / 1e6,
                "avg_acs_per_sphere": float(rr.sum_acs) / max(1, args.steps) / n_s,
                "k_contacts_ss_ms": times[5] / steps_prof, "k_integrate_ms": times[2] / steps_prof,
                "device_mem_used_gb": (total - free) / 1e9, "device_mem_total_gb": total / 1e9,
                "bytes_per_sphere": (total - free) / n_s, "settle_s_1M": settle_s,
            })
            sim.close()
            del sim
        except Exception as e:   # e.g. out of device memory at the largest sizes
            rec["error"] = f"{type(e).__name__}: {e}"[:300]
        print(json.dumps(rec), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
