"""Profile helper: build one config scene, settle, then run a short window
between cudaProfilerStart/Stop (for ncu --profile-from-start off).

usage: python tools/prof_cfg.py rover|mixer|hopper [n]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    from paper_2311_04648_b200 import scenes
    what = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2_000_000
    if what == "rover":
        sim = scenes.rover_wheel(n, h=1e-5, sinkage=0.0, plunge=0.1)
        sim.initialize()
        sim.do_dynamics(3000 * sim.h)
        sim.set_init_time_step(2e-6)
    elif what == "mixer":
        sim, _ = scenes.mixer(n, h=1e-4)
        sim.set_error_out_velocity(10.0)
        sim.set_fixed_lookahead(2)
        sim.initialize()
        sim.do_dynamics(0.02)
    else:
        import _bulk as BK
        import paper_2311_04648_b200 as gf
        sim, _, _, gate = BK.hopper_sim(gf, scale=float(sys.argv[3]) if len(sys.argv) > 3 else 3.68, fill=1.0,
                                        precision="f32", v_err=10.0, h=float(sys.argv[4]) if len(sys.argv) > 4 else 4e-5)
        sim.initialize()
        BK.settle(sim, 0.3)
        sim.set_family_mask(gate, 0, False)
        sim.do_dynamics(0.02)
    sim.do_dynamics(10 * sim.h)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    sim.do_dynamics(8 * sim.h)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    rr = sim.last_run
    print("n_acs", rr.n_acs, "rebuilds", rr.kt_rebuilds, "ms", rr.dt_ms / 8)
    sim.close()


if __name__ == "__main__":
    main()
