"""Timeline of the kT/dT schedule on the bench bed (diagnostics): settles the
bench.py scene, then runs a few steps with GF_TRACE=1 so gf_run_end prints
every stream mark (ms since the run's first event) and the host's waits to
stderr; this script turns them into per-step spans.

usage: python tools/trace_step.py [--steps 12] 2> trace.txt
"""

import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--settle-steps", type=int, default=12000)
    ap.add_argument("--scene", default="crater", choices=["crater", "cohesive"])
    args = ap.parse_args()
    from paper_2311_04648_b200 import models, scenes
    if args.scene == "cohesive":
        models.cohesive_model()
        sim = scenes.crater_bed(4_000_000, hold_ball=True, force_model="hertz_mindlin_cohesive",
                                extra_props={"coh": 1.0e4})
    else:
        sim = scenes.crater_bed(1_000_000, hold_ball=True)
    sim.initialize()
    sim.do_dynamics(args.settle_steps * sim.h)
    scenes.release_balls(sim)
    sim.do_dynamics(20 * sim.h)
    os.environ["GF_TRACE"] = "1"
    sys.stderr.flush()
    prof = bool(os.environ.get("GF_PROFILE_TIMED"))   # ncu --profile-from-start off
    if prof:
        import torch
        torch.cuda.profiler.start()
    sim.do_dynamics(args.steps * sim.h)
    if prof:
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    os.environ.pop("GF_TRACE")
    sim.close()


if __name__ == "__main__":
    main()
