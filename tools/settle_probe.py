"""How fast does the 1M lattice bed settle? touching pairs / max speed per chunk."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2311_04648_b200 import scenes
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 10
per = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
sim = scenes.crater_bed(n, hold_ball=True)
sim.initialize()
t0 = time.time()
for c in range(chunks):
    sim.do_dynamics(per * sim.h)
    rr = sim.last_run
    v = np.linalg.norm(sim.store.lin_vel[: sim.store.n_owners], axis=1)
    z = sim._pos[:, 2]
    print(f"steps {(c + 1) * per}: touching pairs/step {rr.sum_touch_pairs / per:.0f}, acs {rr.n_acs}, "
          f"ms/step {rr.dt_ms / per:.3f}, vmax {v.max():.3f} vmean {v.mean():.4f}, ztop97 {np.percentile(z, 97):.4f}, "
          f"rebuilds {rr.kt_rebuilds}", flush=True)
print("wall", time.time() - t0)
