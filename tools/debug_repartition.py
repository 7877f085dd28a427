"""Step-by-step comparison of a decomposed run (with repartitions) against a
single context: prints the first step whose state differs."""
import sys
import numpy as np
sys.path.insert(0, ".")
from tests.test_gpu_decomp import jostle_box, R
from paper_2311_04648_b200 import decomp

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
travel = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2 * R
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 1   # steps per do_dynamics call
single = jostle_box()
single.initialize()
group = decomp.LoopbackGroup(2, travel=travel)
sims = [jostle_box(decomposition=group.member(r)) for r in range(2)]
for s in sims:
    s.initialize()
h = single.h
last_rep = 0
for k in range(0, steps, chunk):
    single.do_dynamics(chunk * h)
    group.do_dynamics(chunk * h)
    rep = getattr(sims[0].scheduler, "repartitions", 0)
    st = group.gather()
    n = single.store.n_owners
    bad = {}
    for f in ("voxel", "subvoxel", "quat", "lin_vel", "ang_vel"):
        a = np.asarray(getattr(single.store, f)[:n])
        b = np.asarray(st[f])
        d = np.nonzero(np.any((a != b).reshape(n, -1), axis=1))[0]
        if d.size:
            bad[f] = d
    if rep != last_rep:
        print(f"step {k + chunk}: repartition #{rep}", flush=True)
        last_rep = rep
    if bad:
        print(f"step {k + chunk}: mismatch", {f: (v.size, v[:6].tolist()) for f, v in bad.items()})
        o = int(next(iter(bad.values()))[0])
        print("  single v", single.store.lin_vel[o], "group v", st["lin_vel"][o])
        print("  single x", single._pos[o], "group x", st["pos"][o])
        print("  touching single", single._last_touching, "group", sum(s._last_touching for s in sims))
        ca = single._acs
        sel = np.nonzero(np.isin(ca.geom_a, single.store.geoms_of(o)) | np.isin(ca.geom_b, single.store.geoms_of(o)))[0]
        print("  single acs of owner", [(int(ca.kind[i]), int(ca.geom_a[i]), int(ca.geom_b[i]), [float(ca.wildcards[w][i]) for w in ca.wildcards]) for i in sel])
        ga = st["acs"]
        sel = np.nonzero(np.isin(ga.geom_a, single.store.geoms_of(o)) | np.isin(ga.geom_b, single.store.geoms_of(o)))[0]
        print("  group acs of owner", [(int(ga.kind[i]), int(ga.geom_a[i]), int(ga.geom_b[i]), [float(ga.wildcards[w][i]) for w in ga.wildcards]) for i in sel])
        for s in sims:
            st_ = s._dd
            gi = np.nonzero(st_.gids == o)[0]
            print("  rank", st_.rank, "holds", gi, "class", (st_.dd[gi] & 3) if gi.size else None)
        break
else:
    print("no mismatch in", steps, "steps; repartitions", last_rep)
