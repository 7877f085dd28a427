"""Benchmark: M sphere-steps/s of the B200 DEM step (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload at N=1 (the largest single-GPU configuration in BASELINE.json's
configs): configs[4]'s 150M-sphere point -- the settled configs[1] crater
bed (1M polydisperse spheres + projectile, released after 12 000 untimed
settling steps) tiled 15 x 10 side by side in one box (scenes.tiled_bed).
`--tiles 1` times configs[1] itself.

One JSON line on rank 0.  `value` = whole-job sphere-steps/s from CUDA events
on the dT stream (t0 before the first timed step, t1 after the last step with
the kT stream joined), max over ranks.  `e2e` = the same metric through the
C-ABI with host buffers: every step uploads the owner state from pinned host
memory, runs the step, downloads the state.  `--impl reference` times the
reference algorithm on the host cores (the C restatement in oracle/, all
threads) on the same settled bed (prepared on the device, untimed), one
1M-sphere tile per step as the bounded sample.

Multi-GPU (torchrun, one process per GPU): the spatial slab decomposition
(paper_2311_04648_b200/decomp.py) of N beds laid side by side -- each rank
owns one 1M-sphere bed plus its projectile and exchanges ghost state and
ghost forces with its neighbours over NCCL every step (weak scaling).
`--mode replicas` runs N independent beds instead.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

# NCCL's own log lines (NCCL_DEBUG) go to stderr: stdout carries only the JSON line
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "M element-steps/sec at 1/2/4/8 B200; % HBM roofline; CPU-ref x on host cores"
UNIT = "M sphere-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n-spheres", type=int, default=1_000_000, help="spheres per bed (tile)")
    ap.add_argument("--tiles", type=int, default=150,
                    help="N=1: copies of the settled bed in one box (configs[4] size sweep; 150 = 150M "
                         "spheres, the largest single-GPU point); 1 = configs[1] itself")
    ap.add_argument("--n-max", type=int, default=4)
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-f64", action="store_true", help="skip the fp64 parity-build rate")
    ap.add_argument("--amortised-steps", type=int, default=200,
                    help="extra window over several candidate rebuilds (rebuild-amortised rate)")
    ap.add_argument("--prof-steps", type=int, default=20, help="per-kernel event window")
    ap.add_argument("--mode", default="auto", choices=["auto", "single", "replicas", "decomp", "ktdt"],
                    help="auto: single on 1 GPU, decomp (slab decomposition) on N > 1; ktdt: the paper's "
                         "2-GPU split of one scene (rank 0: dT on GPU 0, kT on GPU 1; other ranks idle)")
    ap.add_argument("--settle-steps", type=int, default=12000,
                    help="untimed steps that settle the lattice bed (projectile parked) before the "
                         "projectile is released at the settled surface; 0 = time the raw lattice")
    ap.add_argument("--travel", type=float, default=5e-3,
                    help="decomposition: displacement allowed before a repartition (m)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region (NVML,
    else an nvidia-smi child)."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    # NVML clocks-event reason bits: sw power cap, hw slowdown, sw / hw thermal
    _BITS = (0x8, 0x40, 0x20, 0x4)   # order of summary(): hw, hw thermal, sw thermal, power cap

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self._nvml = None

    def _poll(self):
        """NVML in-process, every 2 ms: a sub-100 ms timed region still gets
        samples (an nvidia-smi child often returns none inside it)."""
        nv, h = self._nvml
        try:
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception:
            mx = 0
        while True:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(self.index), str(sm), str(mx), "", ""] +
                                 ["Active" if rs & b else "Not Active" for b in self._BITS])
            except Exception:
                pass
            if self._stop.wait(0.002):
                break

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nvml = (nv, nv.nvmlDeviceGetHandleByIndex(self.index))
            self._stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self._nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self._nvml is not None:
            self._stop.set()
            self.thread.join(timeout=5)
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def profiled_traffic(kernel, alg_bytes=None):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/ncu_traffic.json).  The capture is of the 16M-sphere point of
    the same sweep (ncu cannot replay the 150M state); with `alg_bytes` the
    captured traffic / algorithmic-byte ratio is applied to this run's
    algorithmic bytes per launch.  Returns (bytes, note)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None, "no capture"
    t = d.get(kernel)
    ref = d.get("_alg_bytes_" + kernel)
    if t is None:
        return None, "no capture"
    if alg_bytes is None or not ref:
        return t, "ncu dram bytes per launch of the captured run"
    ratio = t / ref
    return ratio * alg_bytes, (f"ncu dram bytes (read + write) of the 16M capture = {ratio:.3f} x its algorithmic "
                               "bytes, applied to this launch's algorithmic bytes (profiles/ncu_traffic.json)")


# ---------------------------------------------------------------------------
# CPU legs (oracle restatement of the reference algorithm)
# ---------------------------------------------------------------------------

def cpu_run(scene, steps, warmup, period, lag, nthreads, margin):
    from oracle import oracle as O
    st = O.OracleStepper(scene, margin, period=period, lag=lag, nthreads=nthreads)
    for _ in range(warmup):
        st.step_once()
    t0 = time.perf_counter()
    for _ in range(steps):
        st.step_once()
    return time.perf_counter() - t0


def build_scene(args, device, tiles=1, decomposition=None, hold_ball=False):
    from paper_2311_04648_b200 import scenes
    return scenes.crater_bed(args.n_spheres, n_max=args.n_max, precision=args.precision, device=device,
                             tiles=tiles, decomposition=decomposition, hold_ball=hold_ball,
                             kt_device=getattr(args, "kt_device", None))


def schedule(sim):
    period, lag = sim._schedule()
    return period, lag, sim._current_margin()


DTYPE = ("fp32 contact law (fp64 centre difference and overlap numerator R^2 - d^2), fp32 velocities, "
         "int64 fixed-point owner force/torque sums, fixed-point positions (u64 voxel + 3 x u16)")
DTYPE_F64 = "fp64 contact law and velocities (parity build), fixed-point positions"


def factor(t):
    """tx x ty = t, as square as possible"""
    ty = int(math.isqrt(t))
    while t % ty:
        ty -= 1
    return t // ty, ty


def workload_config(args, world, mode):
    """The `config` object of both arms (identical by construction)."""
    tiles = max(1, args.tiles) if world == 1 else 1
    tx, ty = factor(tiles)
    if world == 1 and tiles > 1:
        wl = (f"configs[4] size-sweep point: the settled configs[1] crater bed ({args.n_spheres} polydisperse "
              f"spheres + projectile) tiled {tx}x{ty} in one box = {tiles * (args.n_spheres + 1)} spheres "
              f"on one B200")
    else:
        wl = (f"configs[1] crater impact bed, {args.n_spheres} polydisperse spheres + projectile"
              + (f" per GPU, {world} beds side by side" if world > 1 else ""))
    return {"workload": wl, "n_spheres_per_bed": args.n_spheres, "tiles": f"{tx}x{ty}",
            "n_max": args.n_max, "h": 1e-5, "v_err": 5.0, "precision": args.precision,
            "settle_steps": args.settle_steps,
            "parallelism": ({"decomp": f"slab decomposition x{world} (NCCL halo + force return)",
                             "replicas": f"replicas x{world}",
                             "ktdt": "2-GPU kT/dT split: dT on GPU 0, kT on GPU 1 (NVLink peer access)"}
                            .get(mode, "single GPU")),
            "inputs_vs_l2": "state + contact arrays larger than L2 (no flush)",
            "bed": ("settled: the untimed settling steps from the HCP lattice with the projectile parked, "
                    "then the projectile released 2 mm above the surface at the 20 cm-drop speed")
            if args.settle_steps > 0 else "raw HCP lattice"}


def settled_source(args, device, tiles=1, decomposition=None):
    """The settled configs[1] bed (device; untimed setup shared by both arms)."""
    from paper_2311_04648_b200 import scenes
    src = build_scene(args, device, tiles=tiles, decomposition=decomposition, hold_ball=args.settle_steps > 0)
    src.initialize()
    t_s = time.perf_counter()
    if args.settle_steps > 0:
        # the reference settles the bed before the drop (scenarios.py:255-307)
        src.do_dynamics(args.settle_steps * src.h)
        scenes.release_balls(src)
    return src, time.perf_counter() - t_s


def reference_arm(args):
    """The reference's algorithm on the host cores (oracle/gf_oracle.c, the C
    restatement of grainforge's numba kernels, OpenMP on every core) on the
    same settled bed the b200 arm times.  The bed is settled on the device
    (untimed input preparation: 12 000 steps are out of reach on the host);
    each timed step advances one 1M-sphere tile -- the bounded sample; the
    per-sphere cost does not depend on how many tiles sit side by side."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from paper_2311_04648_b200 import scenes
    src, _ = settled_source(args, local)
    scene = scenes.oracle_scene(src)
    period, lag, margin = schedule(src)
    src.close()
    n_s = int(np.sum(scene["geom_kind"] == 0))
    threads = os.cpu_count() or 1
    steps = max(1, args.steps)
    warm = max(1, min(args.warmup, 2))
    wall = cpu_run(scene, steps, warm, period, lag, threads, margin)
    value = n_s * steps / wall / 1e6
    mode = "decomp" if world > 1 else "single"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": wall / steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp64 (numba fastmath=False "
        "semantics, -ffp-contract=off)", "data": "synthetic",
        "config": workload_config(args, world, mode),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"each step: one step of one {n_s}-sphere tile of the settled bed "
                                   f"(oracle/gf_oracle.c, OpenMP contact/reduce/integrate loops, serial "
                                   f"detection; period {period}, lag {lag}, margin {margin:.3g} m)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def b200_arm(args):
    rank, world, local = dist_env()
    import torch
    if args.mode == "ktdt":
        # one scene on two GPUs: rank 0 drives both devices
        if rank != 0:
            return
        world, args.kt_device = 1, (1 if torch.cuda.device_count() > 1 else 0)
    mode = args.mode if args.mode != "auto" else ("decomp" if world > 1 else "single")
    if mode == "single" and world > 1:
        mode = "replicas"
    kt_dev = getattr(args, "kt_device", None)
    dist = None
    if world > 1 or mode == "decomp":
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", rank=rank, world_size=world)
    device = local
    from paper_2311_04648_b200 import _lib, decomp, scenes
    dec = decomp.SlabDecomposition(travel=args.travel) if mode == "decomp" else None
    t_setup = time.perf_counter()
    sim, settle_s = settled_source(args, device, tiles=world if mode == "decomp" else 1, decomposition=dec)
    # the CPU baseline's sample: one settled tile
    scene0 = scenes.oracle_scene(sim) if (rank == 0 and world == 1 and not args.no_cpu) else None
    tiles = max(1, args.tiles) if (world == 1 and mode in ("single", "ktdt")) else 1
    if tiles > 1:
        tx, ty = factor(tiles)
        src = sim
        sim = scenes.tiled_bed(src, tx, ty, precision=args.precision, device=device, n_max=args.n_max,
                               kt_device=kt_dev)
        src.close()
        del src
        sim.initialize()
    setup_s = time.perf_counter() - t_setup
    if mode == "decomp":
        cls = sim._dd.dd & 3
        n_s = int(np.sum(cls[sim._sph_owner] == decomp.DD_LOCAL))   # spheres this rank integrates
        n_ghost_owners = int(np.sum(cls == decomp.DD_GHOST))
        n_sph_total = n_s
        if dist is not None:
            t = torch.tensor([n_s], device=f"cuda:{device}", dtype=torch.int64)
            dist.all_reduce(t)
            n_sph_total = int(t.item())
    else:
        n_s = int(sim._sph_geom.size)
        n_ghost_owners = 0
        n_sph_total = n_s * world
    n_o = int(sim.store.n_owners)
    # non-fixed owners, from the host arrays (no device sync)
    n_free0 = int(np.sum(~sim._fixed_flag[sim.store.__dict__["_owner_family"][:n_o]]))
    h = sim.h
    # warm-up (untimed)
    sim.do_dynamics(args.warmup * h)
    ctx = sim._ctx
    if os.environ.get("GF_BENCH_PROF_IN_TIMED"):   # diagnostics: per-kernel events inside the timed steps
        ctx.call("gf_set_profiling", C.c_int(1))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(device)

    barrier()
    rebuilds0 = int(sim.last_run.kt_rebuilds) if sim.last_run is not None else 0
    reps0 = getattr(sim.scheduler, "repartitions", 0)
    dev0 = sim.scheduler.timing["dyn_force"]
    prof_range = bool(os.environ.get("GF_PROFILE_TIMED"))   # ncu --profile-from-start off
    if os.environ.get("GF_BENCH_KT_FREEZE"):   # diagnostics: the dT chain alone (no detections in the timed steps)
        os.environ["GF_KT_FREEZE"] = "1"
    with ClockSampler(device) as clocks:
        if prof_range:
            torch.cuda.profiler.start()
        sim.do_dynamics(args.steps * h)
        barrier()
        if prof_range:
            torch.cuda.profiler.stop()
    os.environ.pop("GF_KT_FREEZE", None)
    rr = sim.last_run
    # device time of the timed steps: CUDA events on the dT stream around
    # every gf_run segment (one segment unless a repartition split the call)
    dt_ms = (sim.scheduler.timing["dyn_force"] - dev0) * 1e3
    repartitions = getattr(sim.scheduler, "repartitions", 0) - reps0
    # rebuild-amortised rate: a longer window (CUDA events on the dT stream,
    # kT joined) spanning several Verlet candidate rebuilds -- a short timed
    # window may contain none (one rebuild every ~40 steps on this bed)
    amort = None
    if args.amortised_steps > 0 and mode in ("single", "ktdt"):
        rb0 = int(sim.last_run.kt_rebuilds)
        d0 = sim.scheduler.timing["dyn_force"]
        barrier()
        sim.do_dynamics(args.amortised_steps * h)
        barrier()
        a_ms = (sim.scheduler.timing["dyn_force"] - d0) * 1e3
        amort = {"value": n_sph_total * args.amortised_steps / (a_ms * 1e-3) / 1e6, "unit": UNIT,
                 "steps": args.amortised_steps, "ms_per_step": a_ms / args.amortised_steps,
                 "kt_candidate_rebuilds": int(sim.last_run.kt_rebuilds) - rb0}
    # per-kernel CUDA events would sit between the kernels of the chain (and
    # break its programmatic dependent launches): the kernel times come from a
    # separate profiled window right after the timed one
    ctx = sim._ctx   # a repartition rebuilds the context
    ctx.call("gf_set_profiling", C.c_int(1))
    prof_steps = max(2 * 2, min(args.steps, args.prof_steps))
    sim.do_dynamics(prof_steps * h)
    barrier()
    ctx = sim._ctx
    times = np.zeros(6)
    ctx.call("gf_kernel_times", _lib.ptr(times))
    ctx.call("gf_set_profiling", C.c_int(0))
    if dist is not None:
        t = torch.tensor([dt_ms], device=f"cuda:{device}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt_ms = float(t.item())
    ms_per_step = dt_ms / args.steps
    value = n_sph_total * args.steps / (dt_ms * 1e-3) / 1e6
    n_acs_avg = float(rr.sum_acs) / max(1, args.steps)
    n_touch_avg = float(rr.sum_touch_pairs) / max(1, args.steps)
    n_free = n_free0

    # --- roofline: dominant kernel (k_contacts_ss) and the whole dT chain ---
    hbm, hbm_kind = peaks()
    steps_prof = max(1.0, times[4])
    t_contacts = times[0] / steps_prof * 1e-3      # contact phase: k_contacts_ss + wall kinds
    t_ss = times[5] / steps_prof * 1e-3            # the fused sphere-sphere kernel alone
    t_chain = (times[0] + times[1] + times[2]) / steps_prof * 1e-3
    vel_b = 12 if args.precision == "f32" else 24
    per_owner = 58 + 54 + 48 + 2 * (vel_b - 12) * 2  # 160 B (fp32), 208 B (fp64)
    # 24 B per ACS entry (ids + history read), 16 B per touching
    # entry (history write); all kinds counted (the wall kinds are ~1% here)
    bytes_contacts = 24.0 * n_acs_avg + 16.0 * n_touch_avg
    bytes_chain = per_owner * n_free + 4.0 * n_s + bytes_contacts
    ach_c = bytes_contacts / t_ss / 1e9 if t_ss > 0 else 0.0
    traffic_c, traffic_note = profiled_traffic("k_contacts_ss", bytes_contacts)
    ach_chain = bytes_chain / t_chain / 1e9 if t_chain > 0 else 0.0

    # --- e2e: host-buffer round trip per step through the C-ABI ---
    e2e = None
    if args.e2e_steps > 0:
        e2e = measure_e2e_decomp(sim, args.e2e_steps, dist) if mode == "decomp" else \
            measure_e2e(sim, args.e2e_steps)
        if e2e is not None and dist is not None:
            t = torch.tensor([e2e.pop("wall")], device=f"cuda:{device}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["value"] = (n_sph_total if mode == "decomp" else n_s * world) * e2e["steps"] / float(t.item()) / 1e6
        elif e2e is not None:
            e2e.pop("wall")

    line = None
    if rank == 0:
        cpu = None
        if scene0 is not None:
            period, lag, margin = schedule(sim)
            csteps = max(1, args.cpu_steps)
            wall = cpu_run(scene0, csteps, 1, period, lag, 1, margin)
            n_s0 = int(np.sum(scene0["geom_kind"] == 0))
            cpu = {"value": n_s0 * csteps / wall / 1e6, "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"{csteps} steps (+1 warm-up) of one {n_s0}-sphere tile of the same settled bed "
                             f"(1/{tiles} of the workload), serial C restatement (oracle/gf_oracle.c)"}
        launches_per_step = 3 + (1 if sim._tri_geom.size or sim._ana_geom.size else 0)
        if mode == "decomp":   # halo: pack/add forces, pack/unpack(+centres) state per peer; guard word x2
            launches_per_step += 2 + 5 * len(sim._dd.peers)
        period, lag, _ = schedule(sim)
        # per detection: snapshot, min/max init, grid, family geometry, filter, 2 scans + inits,
        # compaction, gap fill, wall pairs, place, segment sort, flag reset, history gather (16);
        # per candidate rebuild ~45 (cell sort, candidate count/fill, pair sort passes, segment
        # sorts, sphere-analytic candidates) -- the ncu launch list of the timed steps
        # (profiles/r2/launches_150m_with_rebuilds.csv: 1290 launches in 100 steps, 2 rebuilds)
        kt_launches = 16
        rb_launches = 45 * (int(rr.kt_rebuilds) - rebuilds0)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": (args.gpus if mode == "ktdt" else world),
            "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": DTYPE if args.precision == "f32" else DTYPE_F64,
            "data": "synthetic",
            "config": workload_config(args, world, mode),
            "workload_stats": {"n_spheres": n_s, "n_owners": n_o, "n_spheres_total": n_sph_total,
                               "period": period, "lag": lag, "avg_acs": n_acs_avg,
                               "avg_touching_pairs": n_touch_avg,
                               "kt_candidate_rebuilds_in_timed_steps": int(rr.kt_rebuilds) - rebuilds0,
                               "setup_s": setup_s, "settle_s": settle_s,
                               **({"ghost_owners_rank0": n_ghost_owners, "travel_m": args.travel,
                                   "repartitions_in_timed_steps": repartitions} if mode == "decomp" else {})},
            "rebuild_amortised": amort,
            "roofline": {"bound": "hbm", "kernel": "k_contacts_ss", "achieved": ach_c, "peak": hbm,
                         "unit": "GB/s", "frac": ach_c / hbm, "peak_kind": hbm_kind,
                         "traffic": traffic_c,
                         "traffic_note": traffic_note,
                         "algorithmic_bytes_per_launch": bytes_contacts,
                         "launch_ms": t_ss * 1e3},
            "roofline_dt_chain": {"bound": "hbm", "achieved": ach_chain, "peak": hbm, "unit": "GB/s",
                                  "frac": ach_chain / hbm, "bytes_per_step": bytes_chain,
                                  "ms": t_chain * 1e3,
                                  "share_of_step": t_chain / (ms_per_step * 1e-3)},
            "kernel_ms_per_step": {"window": f"{int(steps_prof)} profiled steps after the timed ones",
                                   "contact_phase": times[0] / steps_prof, "k_contacts_ss": times[5] / steps_prof,
                                   "k_heavy": times[1] / steps_prof,
                                   "k_integrate": times[2] / steps_prof,
                                   "kT_per_cycle": times[3] / max(1, int(steps_prof) // max(1, period))},
            "clocks": clocks.summary(),
            "e2e": e2e,
            "gpu_launches": int(args.steps * launches_per_step + (args.steps // max(1, period)) * kt_launches
                                + rb_launches),
            "cpu_baseline": cpu,
        }
    sim.close()
    if line is not None and mode in ("single", "ktdt") and not args.no_f64 and args.precision == "f32":
        # the reference's own arithmetic (fp64 state and contact law, the
        # bit-exact parity build) on configs[1]'s bed, for comparison
        line["f64_build"] = f64_build_rate(args, device)
    if line is not None:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def f64_build_rate(args, device, steps=100):
    """M sphere-steps/s of the fp64 parity build on the settled configs[1]
    bed (1M spheres + projectile), CUDA events on the dT stream."""
    import torch
    a = argparse.Namespace(**vars(args))
    a.precision = "f64"
    sim, _ = settled_source(a, device)
    try:
        sim.do_dynamics(5 * sim.h)
        torch.cuda.synchronize(device)
        d0 = sim.scheduler.timing["dyn_force"]
        sim.do_dynamics(steps * sim.h)
        torch.cuda.synchronize(device)
        ms = (sim.scheduler.timing["dyn_force"] - d0) * 1e3
        n_s = int(sim._sph_geom.size)
        return {"value": n_s * steps / (ms * 1e-3) / 1e6, "unit": UNIT, "ms_per_step": ms / steps,
                "steps": steps, "dtype": DTYPE_F64,
                "workload": f"configs[1] settled crater bed, {n_s} spheres (one tile), fp64 parity build "
                            "(bit-exact per step against the reference's arithmetic)"}
    finally:
        sim.close()


def measure_e2e(sim, steps):
    """Per step: pinned host state -> device (gf_upload_owners), one step
    (gf_run), device -> pinned host state (gf_download_owners)."""
    import torch
    from paper_2311_04648_b200 import _lib
    ctx = sim._ctx
    n = sim.store.n_owners
    P = _lib.ptr

    def pinned(shape, dtype):
        t = torch.empty(int(np.prod(shape)) * np.dtype(dtype).itemsize, dtype=torch.uint8).pin_memory()
        return t.numpy().view(dtype).reshape(shape)

    vox, sub = pinned((n,), np.uint64), pinned((n, 3), np.uint16)
    quat, lv, av = pinned((n, 4), np.float32), pinned((n, 3), np.float64), pinned((n, 3), np.float64)
    fam = pinned((n,), np.uint8)
    ctx.call("gf_download_owners", P(vox), P(sub), P(quat), P(lv), P(av), P(fam))
    tpl = _lib.carr(sim._tpl_id[sim._own_d2u], np.uint32)
    rows = sim._tpl_rows
    mass, moi = rows[:, 0].copy(), _lib.carr(rows[:, 1:], np.float64)
    rp = _lib.RunParams()
    rp.n_steps = 1
    rp.h = sim.h
    for a in range(3):
        rp.g[a] = float(sim.gravity[a])
    rp.v_err = sim.v_err
    period, lag = sim._schedule()
    rp.margin = sim._current_margin()
    rp.period, rp.lag, rp.n_dyn, rp.write_acc = period, lag, 0, 0
    rr = _lib.RunResult()
    step0 = sim.scheduler.step_counter
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ph = [0.0, 0.0, 0.0]   # host wall per call (each call returns synchronised)
    for i in range(steps):
        ta = time.perf_counter()
        ctx.call("gf_upload_owners", C.c_int64(n), P(vox), P(sub), P(quat), P(lv), P(av), P(fam),
                 P(tpl), C.c_int64(rows.shape[0]), P(mass), P(moi))
        tb = time.perf_counter()
        rp.step0 = step0 + i
        ctx.call("gf_run", C.byref(rp), C.byref(rr))
        tc = time.perf_counter()
        ctx.call("gf_download_owners", P(vox), P(sub), P(quat), P(lv), P(av), P(fam))
        td = time.perf_counter()
        ph[0] += tb - ta; ph[1] += tc - tb; ph[2] += td - tc
    wall = time.perf_counter() - t0
    sim.scheduler.step_counter = step0 + steps
    n_s = int(sim._sph_geom.size)
    per = n * (8 + 6 + 16 + 24 + 24 + 1)
    return {"value": n_s * steps / wall / 1e6, "unit": UNIT, "h2d_bytes_per_step": per,
            "d2h_bytes_per_step": per + 64, "steps": steps, "wall": wall,
            "ms_per_call": {"upload": 1e3 * ph[0] / steps, "run_1_step": 1e3 * ph[1] / steps,
                            "download": 1e3 * ph[2] / steps},
            "path": "gf_upload_owners -> gf_run(1 step) -> gf_download_owners, pinned host buffers"}


def measure_e2e_decomp(sim, steps, dist):
    """The decomposed step end to end: per step the rank's owner state from
    pinned host memory (gf_upload_owners), one step through the public API
    (Simulator.do_dynamics: forces, NCCL ghost-force return, integration,
    NCCL ghost state), the state back to pinned host memory."""
    import torch
    from paper_2311_04648_b200 import _lib
    ctx = sim._ctx
    n = sim.store.n_owners
    P = _lib.ptr

    def pinned(shape, dtype):
        t = torch.empty(int(np.prod(shape)) * np.dtype(dtype).itemsize, dtype=torch.uint8).pin_memory()
        return t.numpy().view(dtype).reshape(shape)

    vox, sub = pinned((n,), np.uint64), pinned((n, 3), np.uint16)
    quat, lv, av = pinned((n, 4), np.float32), pinned((n, 3), np.float64), pinned((n, 3), np.float64)
    fam = pinned((n,), np.uint8)
    ctx.call("gf_download_owners", P(vox), P(sub), P(quat), P(lv), P(av), P(fam))
    tpl = _lib.carr(sim._tpl_id[sim._own_d2u], np.uint32)
    rows = sim._tpl_rows
    mass, moi = rows[:, 0].copy(), _lib.carr(rows[:, 1:], np.float64)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        ctx = sim._ctx
        ctx.call("gf_upload_owners", C.c_int64(n), P(vox), P(sub), P(quat), P(lv), P(av), P(fam),
                 P(tpl), C.c_int64(rows.shape[0]), P(mass), P(moi))
        sim._host_stale = False
        sim.do_dynamics(sim.h)
        sim._ctx.call("gf_download_owners", P(vox), P(sub), P(quat), P(lv), P(av), P(fam))
    wall = time.perf_counter() - t0
    per = n * (8 + 6 + 16 + 24 + 24 + 1)
    return {"value": 0.0, "unit": UNIT, "h2d_bytes_per_step": per, "d2h_bytes_per_step": per + 64,
            "steps": steps, "wall": wall,
            "path": "gf_upload_owners -> Simulator.do_dynamics(1 step; NCCL halo) -> gf_download_owners, "
                    "pinned host buffers, per rank"}


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
