"""Generate the bulk-observable fixtures (SURVEY.md §8(c) parity leg 3) by
running the REFERENCE `grainforge` itself, in this build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_bulk.py c1
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_bulk.py crater_bed
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_bulk.py crater_drop 2200
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_bulk.py crater_drop 7800
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_bulk.py crater_drop 15000
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_bulk.py hopper

Outputs (tests/golden/):
* bulk_c1.npz           C1 10k settling box (tests/_bulk.py c1_box), pile
                        height and KE every 0.05 s up to 0.5 s.
* bulk_crater_bed.npz   settle_crater_bed's pour and settle (scenarios.py:
                        256-307) restated in tests/_bulk.py crater_settle:
                        settled positions, templates, radii, surface_z,
                        bulk_density, the settle time and the residual KE.
* bulk_crater_<rho>.npz run_crater_drop (scenarios.py:310-346, restated in
                        tests/_bulk.py crater_drop) on that bed, drop height
                        10 cm: penetration depth and the ball's z every
                        0.05 s.  `..._nmax3` repeats a drop with another
                        lookahead: the reference's own spread, which sets the
                        depth tolerance.
The scenario parameters deviate from the reference scenario in v_err and the
lookahead only (tests/_bulk.py explains why: the reference's 24-48 mm margin
costs 2.3 s per step on the host).

The GPU tests (tests/test_gpu_bulk.py) run the same scenes through this
package and compare the observables within stated tolerances.  Nothing under
tests/ reads /root/reference at run time.
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import grainforge as gf  # noqa: E402

import _bulk as BK  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
DROP_HEIGHT = 0.10


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)", flush=True)


def c1():
    t0 = time.time()
    r = BK.run_c1(gf)
    print(f"c1: {time.time() - t0:.0f} s; height {r['height'][-1]:.5f} ke {r['ke'][-1]:.4e}", flush=True)
    save("bulk_c1", t=r["t"], height=r["height"], ke=r["ke"], n=np.int64(10_000),
         n_max=np.int64(4), seconds=np.float64(time.time() - t0))


def crater_bed():
    t0 = time.time()
    bed = BK.crater_settle(gf)
    print(f"crater_bed: {time.time() - t0:.0f} s; {bed['positions'].shape[0]} grains, settled after "
          f"{bed['settle_t']:.1f} s, surface {bed['surface_z']:.5f} bulk {bed['bulk_density']:.1f}", flush=True)
    save("bulk_crater_bed", **{k: np.asarray(v) for k, v in bed.items()},
         seconds=np.float64(time.time() - t0))


def load_bed():
    g = dict(np.load(os.path.join(OUT, "bulk_crater_bed.npz")))
    return {k: (v[()] if v.ndim == 0 else v) for k, v in g.items()}


def crater_drop(rho: float, n_max: int = BK.CRATER_N_MAX):
    bed = load_bed()
    t0 = time.time()
    r = BK.crater_drop(gf, bed, rho, DROP_HEIGHT, n_max=n_max)
    print(f"crater_drop {rho} (n_max {n_max}): {time.time() - t0:.0f} s depth {r['depth_cm']:.3f} cm",
          flush=True)
    fit = BK.crater_fixed_point(float(bed["mu"]), rho * 1e-3, float(bed["bulk_density"]) * 1e-3,
                                BK.CRATER_D * 100.0, DROP_HEIGHT * 100.0)
    tag = "" if n_max == BK.CRATER_N_MAX else f"_nmax{n_max}"
    save(f"bulk_crater_{int(rho)}{tag}", rho_b=np.float64(rho), drop_height=np.float64(DROP_HEIGHT),
         depth_cm=np.float64(r["depth_cm"]), z=r["z"], t_end=np.float64(r["t_end"]),
         n_max=np.int64(n_max), eq7_depth_cm=np.float64(fit), seconds=np.float64(time.time() - t0))


def hopper():
    t0 = time.time()
    r = BK.run_hopper(gf)
    print(f"hopper: {time.time() - t0:.0f} s; {r['n_clumps']} clumps, settled {r['settle_t']:.1f} s, "
          f"discharged {r['frac'][-1]:.3f}", flush=True)
    save("bulk_hopper", t=r["t"], frac=r["frac"], n_clumps=np.int64(r["n_clumps"]),
         settle_t=np.float64(r["settle_t"]), seconds=np.float64(time.time() - t0))


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "c1":
        c1()
    elif what == "crater_bed":
        crater_bed()
    elif what == "hopper":
        hopper()
    elif what == "crater_drop":
        crater_drop(float(sys.argv[2]), *(int(x) for x in sys.argv[3:4]))
    else:
        raise SystemExit(f"unknown fixture {what!r}")
