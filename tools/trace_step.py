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
    args = ap.parse_args()
    from paper_2311_04648_b200 import scenes
    sim = scenes.crater_bed(1_000_000, hold_ball=True)
    sim.initialize()
    sim.do_dynamics(args.settle_steps * sim.h)
    scenes.release_balls(sim)
    sim.do_dynamics(20 * sim.h)
    os.environ["GF_TRACE"] = "1"
    sys.stderr.flush()
    sim.do_dynamics(args.steps * sim.h)
    os.environ.pop("GF_TRACE")
    sim.close()


if __name__ == "__main__":
    main()
