"""Spatial slab decomposition of one DEM scene over several B200 contexts
("slabs + halo + force return").

The reference has no multi-device path (its kT/dT pair shares one address
space, engine.py:90-115); this is the B200 scale-out of the same step.

Layout.  The clump owners are cut into slabs along one axis (the longest
extent of the scene), balanced by owner count.  Rank r's context holds
  * its local owners (centre of mass in slab r) -- integrated here;
  * ghosts: copies of other ranks' owners within ``width`` of slab r;
  * every boundary owner (mesh / analytic), replicated (must be fixed or
    fully prescribed, so every replica moves identically).
Every physical contact is computed on exactly one rank (gf_common.cuh,
dd_keep).  Because the throughput build reduces contact forces as int64
fixed-point sums, the ghost contributions returned to the home rank add up to
the very integers a single context sums: a decomposed run reproduces the
single-context trajectory bit for bit (tests/test_gpu_decomp.py).

Per step (all on each context's dT stream, no host synchronisation):
  gf_step_forces -> ghost forces home (pack_forces / send / add_forces) ->
  gf_step_integrate -> ghost state out (pack_state / send / unpack_state) and
  the guard word min-reduced (a trip stops every rank before the next force
  phase, so no contact history moves past the trip step).

Width.  w = 2 max_reach + margin + 2 travel.  A pair of owners on different
ranks that can touch while both stay within ``travel`` of their partition
coordinate is then a ghost pair on both ranks.  The device guard trips on the
first step an owner moves further (gf_run_result.dd_trip_step); every rank
stops after that same step and the scene is re-partitioned from the gathered
state and contact history (migration), then the run continues.

Transports.  ``torch.distributed`` (NCCL over NVLink / NVSwitch) with one
process per GPU, or ``LoopbackGroup``: several contexts in one process (one
GPU; used by the parity test and for debugging).
"""

from __future__ import annotations

import ctypes as C
import math
import time as _time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from . import broadphase as B
from .core import (GEOM_SPHERE, GEOM_TRIANGLE, OWNER_CLUMP, ConfigurationError)

DD_LOCAL, DD_GHOST, DD_SHARED, DD_PRIMARY = 0, 1, 2, 3
INT64_MAX = (1 << 63) - 1
FORCE_RECORD = 48


class DecompositionError(RuntimeError):
    pass


# ----------------------------------------------------------------------------
# partition (pure numpy: tested on CPU)
# ----------------------------------------------------------------------------
def owner_reach(store) -> np.ndarray:
    """Largest distance from each owner's centre to a point of its geometry
    (sphere |offset| + r, triangle vertex |v|); inf for analytic owners."""
    n, ng = store.n_owners, store.n_geoms
    d = store.__dict__
    go = d["_geom_owner"][:ng]
    kind = d["_geom_kind"][:ng]
    gp = d["_geom_params"][:ng].astype(np.float64)
    reach = np.zeros(n)
    sph = kind == GEOM_SPHERE
    if sph.any():
        np.maximum.at(reach, go[sph], np.linalg.norm(gp[sph, :3], axis=1) + gp[sph, 3])
    tri = kind == GEOM_TRIANGLE
    if tri.any():
        v = gp[tri, :9].reshape(-1, 3, 3)
        np.maximum.at(reach, go[tri], np.linalg.norm(v, axis=2).max(axis=1))
    ana = ~(sph | tri)
    reach[go[ana]] = np.inf
    return reach


def lever_max(store) -> float:
    """The fixed-point torque lever of a context holding the whole store,
    evaluated exactly as gf_upload_geometry does (float32 parameters widened
    to double, same operation order)."""
    ng = store.n_geoms
    d = store.__dict__
    kind = d["_geom_kind"][:ng]
    gp = d["_geom_params"][:ng].astype(np.float32).astype(np.float64)
    lev = 0.0
    s = gp[kind == GEOM_SPHERE]
    if s.shape[0]:
        lev = max(lev, float(np.max(np.sqrt(s[:, 0] * s[:, 0] + s[:, 1] * s[:, 1] + s[:, 2] * s[:, 2]) + s[:, 3])))
    t = gp[kind == GEOM_TRIANGLE]
    if t.shape[0]:
        v = t[:, :9].reshape(-1, 3)
        lev = max(lev, float(np.max(np.sqrt(v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1] + v[:, 2] * v[:, 2]))))
    return lev


def morton_order(pos: np.ndarray) -> np.ndarray:
    """Device order of owners: 63-bit Morton code (21 bits per axis) of the
    positions, stable.  Simulator._build_permutation uses this same function,
    so a decomposed run orders every rank's owners like a single context."""
    n = pos.shape[0]
    if n <= 1:
        return np.arange(n, dtype=np.int64)
    lo = pos.min(axis=0)
    span = max(float((pos.max(axis=0) - lo).max()), 1e-300)
    q = np.minimum((pos - lo) / span * 2097151.0, 2097151.0).astype(np.uint64)

    def spread(x):   # bit i of x -> bit 3 i
        x = x & np.uint64(0x1FFFFF)
        for sh, m in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                      (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
            x = (x | (x << np.uint64(sh))) & np.uint64(m)
        return x

    code = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))
    return np.argsort(code, kind="stable").astype(np.int64)


@dataclass
class SlabPlan:
    n_ranks: int
    axis: int
    cuts: np.ndarray      # (n_ranks - 1,) slab boundaries along axis
    pad: float            # margin + 2 travel + the largest reach of a non-big owner
    travel: float         # guard: allowed displacement before a repartition
    home: np.ndarray      # (n_owners,) home rank, -1 = shared boundary owner
    x: np.ndarray         # (n_owners,) partition-time coordinate along axis
    reach: np.ndarray     # (n_owners,) owner reach (owner_reach)
    big: np.ndarray       # indices of big owners (reach > 2 x median): own halo
    margin: float = 0.0

    @property
    def width(self) -> float:
        """Ghost layer width for the largest non-big owner."""
        r = self.reach[self.home >= 0]
        small = r[~np.isin(np.nonzero(self.home >= 0)[0], self.big)] if r.size else r
        return self.pad + (float(small.max()) if small.size else 0.0)

    def bounds(self, r: int):
        lo = -math.inf if r == 0 else float(self.cuts[r - 1])
        hi = math.inf if r == self.n_ranks - 1 else float(self.cuts[r])
        return lo, hi

    def ghost_on(self, r: int) -> np.ndarray:
        """Owners homed elsewhere that can touch one of rank r's owners while
        every owner stays within `travel` of its partition coordinate:
        within reach_b + pad of slab r, or within reach_a + reach_b + margin
        + 2 travel of a big owner a of rank r."""
        lo, hi = self.bounds(r)
        other = (self.home >= 0) & (self.home != r)
        dist = np.maximum(np.maximum(lo - self.x, self.x - hi), 0.0)
        g = other & (dist <= self.reach + self.pad)
        for a in self.big:
            if self.home[a] == r:
                g |= other & (np.abs(self.x - self.x[a]) <=
                              self.reach + self.reach[a] + self.margin + 2.0 * self.travel)
        return g

    def classes(self, r: int) -> np.ndarray:
        """Per owner: DD class on rank r, or -1 when the owner is absent there."""
        c = np.full(self.home.shape[0], -1, np.int64)
        c[self.home == r] = DD_LOCAL
        c[self.ghost_on(r)] = DD_GHOST
        c[self.home < 0] = DD_PRIMARY if r == 0 else DD_SHARED
        return c

    def halo(self, r: int):
        """{peer: (send, recv)} global owner ids, ascending: `send` = rank r's
        owners that are ghosts on peer, `recv` = peer's owners that are ghosts
        on r.  Both sides derive the same lists, so no handshake is needed."""
        mine = self.home == r
        on_me = self.ghost_on(r)
        out = {}
        for q in range(self.n_ranks):
            if q == r:
                continue
            send = np.nonzero(mine & self.ghost_on(q))[0]
            recv = np.nonzero(on_me & (self.home == q))[0]
            if send.size or recv.size:
                out[q] = (send.astype(np.int64), recv.astype(np.int64))
        return out


def plan_slabs(pos: np.ndarray, eligible: np.ndarray, reach: np.ndarray, n_ranks: int,
               margin: float, travel: float, axis: Optional[int] = None) -> SlabPlan:
    """Balanced slabs of the eligible (clump) owners along `axis` (default:
    the longest extent)."""
    pos = np.asarray(pos, dtype=np.float64)
    eligible = np.asarray(eligible, dtype=bool)
    reach = np.asarray(reach, dtype=np.float64)
    n = pos.shape[0]
    if n_ranks < 1:
        raise ConfigurationError("n_ranks must be >= 1")
    if (1 << 30) <= n:
        raise ConfigurationError("decomposition supports < 2^30 owners")
    pts = pos[eligible]
    if axis is None:
        axis = int(np.argmax(pts.max(axis=0) - pts.min(axis=0))) if pts.shape[0] else 0
    xs = np.sort(pts[:, axis]) if pts.shape[0] else np.zeros(0)
    cuts = np.zeros(max(0, n_ranks - 1))
    for k in range(1, n_ranks):
        if xs.size == 0:
            cuts[k - 1] = 0.0
            continue
        i = min(max(1, (k * xs.size) // n_ranks), xs.size - 1)
        cuts[k - 1] = 0.5 * (xs[i - 1] + xs[i])
    x = pos[:, axis].copy()
    home = np.full(n, -1, np.int64)
    home[eligible] = np.searchsorted(cuts, x[eligible], side="right")
    er = reach[eligible]
    if er.size:
        big_cut = 2.0 * float(np.median(er))
        big = np.nonzero(eligible & (reach > big_cut))[0].astype(np.int64)
        small_max = float(er[er <= big_cut].max())
    else:
        big, small_max = np.zeros(0, np.int64), 0.0
    pad = small_max + margin + 2.0 * travel
    return SlabPlan(n_ranks, int(axis), cuts, pad, float(travel), home, x, reach, big, float(margin))


# ----------------------------------------------------------------------------
# user-facing configuration
# ----------------------------------------------------------------------------
@dataclass
class SlabDecomposition:
    """Pass as ``Simulator(..., precision="f32", decomposition=...)``.  Every
    rank builds the SAME global scene; initialize() keeps this rank's piece.

    n_ranks / rank default to torch.distributed's world size / rank (one
    process per GPU, NCCL); with ``group`` (a LoopbackGroup) the ranks are
    contexts of this process.  ``travel`` (default: the diameter of the
    largest ordinary owner; big owners such as projectiles get their own
    halo) trades ghost-layer width against repartition frequency."""
    n_ranks: Optional[int] = None
    rank: Optional[int] = None
    axis: Optional[int] = None
    travel: Optional[float] = None
    group: Optional["LoopbackGroup"] = None

    def resolve(self):
        if self.group is not None:
            return self.group.n_ranks, int(self.rank)
        import torch.distributed as dist
        n = self.n_ranks if self.n_ranks is not None else dist.get_world_size()
        r = self.rank if self.rank is not None else dist.get_rank()
        return int(n), int(r)


class LoopbackGroup:
    """Several decomposed contexts in ONE process (all on one device): the
    halo moves by device-to-device copies.  Build one Simulator per rank with
    ``decomposition=group.member(r)``, initialize each, then drive them
    together with ``group.do_dynamics``."""

    def __init__(self, n_ranks: int, axis: Optional[int] = None, travel: Optional[float] = None):
        self.n_ranks = int(n_ranks)
        self.axis = axis
        self.travel = travel
        self.sims: list = [None] * self.n_ranks

    def member(self, rank: int) -> SlabDecomposition:
        return SlabDecomposition(self.n_ranks, rank, self.axis, self.travel, group=self)

    def do_dynamics(self, duration: float) -> None:
        sims = self.sims
        if any(s is None or not s._initialized for s in sims):
            raise ConfigurationError("initialize() every member before do_dynamics")
        steps = int(math.ceil(duration / sims[0].h - 1e-9))
        if steps > 0:
            run_ranks(sims, steps, _LoopbackTransport(sims))

    def gather(self) -> dict:
        return gather_state(self.sims, _LoopbackTransport(self.sims))


# ----------------------------------------------------------------------------
# per-rank state attached to a Simulator
# ----------------------------------------------------------------------------
class _Peer:
    def __init__(self, q, send_slots, recv_slots, rec_bytes, device):
        import torch
        dev = torch.device("cuda", device)
        self.q = q
        self.n_send, self.n_recv = int(send_slots.size), int(recv_slots.size)
        # uint32 owner slots of this context (int32 storage, same bits)
        self.send_idx = torch.as_tensor(send_slots.astype(np.int32), device=dev)
        self.recv_idx = torch.as_tensor(recv_slots.astype(np.int32), device=dev)
        self.state_out = torch.empty(max(1, self.n_send) * rec_bytes, dtype=torch.uint8, device=dev)
        self.state_in = torch.empty(max(1, self.n_recv) * rec_bytes, dtype=torch.uint8, device=dev)
        # ghost forces travel the other way: my ghosts from q -> q's locals
        self.force_out = torch.empty(max(1, self.n_recv) * FORCE_RECORD, dtype=torch.uint8, device=dev)
        self.force_in = torch.empty(max(1, self.n_send) * FORCE_RECORD, dtype=torch.uint8, device=dev)
        self.rec_bytes = rec_bytes


class _RankState:
    def __init__(self, plan, rank, gids, geoms, dd, lever, global_store):
        self.plan = plan
        self.rank = rank
        self.gids = gids          # local owner row -> global owner id
        self.geoms = geoms        # local geometry id -> global geometry id
        self.dd = dd              # uint32 class | gid << 2
        self.lever = lever
        self.global_store = global_store
        self.peers: dict = {}
        self.word = None
        self.order = None         # global device order (Morton order of the first partition)


def prepare(sim) -> None:
    """Called at the top of Simulator.initialize(): replace sim.store (the
    global scene) by this rank's piece."""
    dec = sim.decomposition
    n_ranks, rank = dec.resolve()
    prev = getattr(sim, "_dd", None)
    g = prev.global_store if prev is not None else sim.store
    if dec.group is not None:
        dec.group.sims[rank] = sim
    n = g.n_owners
    d = g.__dict__
    from .core import decode_position
    pos = decode_position(d["_voxel"][:n], d["_subvoxel"][:n], g.domain)
    eligible = d["_owner_kind"][:n] == OWNER_CLUMP
    fam = d["_owner_family"][:n]
    for o in np.nonzero(~eligible)[0]:
        f = int(fam[o])
        if not (sim._fixed_flag[f] or (sim._lv_mask[f].all() and sim._av_mask[f].all())):
            raise ConfigurationError(
                f"decomposition: boundary owner {int(o)} (family {f}) must be fixed or fully prescribed "
                "(it is replicated on every rank)")
    reach = owner_reach(g)
    margin = sim._current_margin()
    if dec.travel is not None:
        travel = float(dec.travel)
    else:
        # one diameter of the largest ordinary (non-big) owner
        er = reach[eligible]
        travel = 2.0 * float(er[er <= 2.0 * np.median(er)].max()) if er.size else 0.0
    axis = dec.axis if dec.axis is not None else (prev.plan.axis if prev is not None else None)
    carried = getattr(prev, "next_plan", None) if prev is not None else None
    if carried is not None:
        # incremental migration: the slab cuts stay, owners are re-homed by
        # their current coordinate (repartition computed it from the
        # neighbours' fresh state)
        plan = carried
    else:
        plan = plan_slabs(pos, eligible, reach, n_ranks, margin, travel, axis)
    cls = plan.classes(rank)
    # device order: the Morton order of the scene at the FIRST partition,
    # kept for the scene's life (as a single context keeps its order), so
    # every contact keeps its A/B orientation across repartitions
    order = prev.order if prev is not None else morton_order(pos)
    ids = order[cls[order] >= 0]
    sub, geoms = g.subset(ids)
    dd = (cls[ids].astype(np.uint64) | (ids.astype(np.uint64) << np.uint64(2))).astype(np.uint32)
    st = _RankState(plan, rank, ids, geoms, dd, lever_max(g), g)
    st.order = order
    # contact history handed over by a repartition: keep the pairs this piece holds
    acs = sim._acs0
    if acs.size:
        inv = np.full(g.n_geoms, -1, np.int64)
        inv[geoms] = np.arange(geoms.size)
        ga, gb = inv[acs.geom_a], inv[acs.geom_b]
        keep = (ga >= 0) & (gb >= 0)
        sel = acs.select(keep)
        sel.geom_a, sel.geom_b = ga[keep], gb[keep]
        sim._acs0 = sel
    sim.store = sub
    sim.reorder = False
    sim._dd = st
    # the margin cap follows the global smallest sphere
    sph = d["_geom_kind"][: g.n_geoms] == GEOM_SPHERE
    if sph.any():
        r_min = float(d["_geom_params"][: g.n_geoms][sph, 3].min())
        sim._dd_margin_cap = max(4, int(r_min / (4.0 * sim.v_err * sim.h)))
    else:
        sim._dd_margin_cap = None


def attach(sim) -> None:
    """Called at the end of Simulator.initialize(): decomposition tables and
    halo buffers of the new context."""
    import torch
    st = sim._dd
    sim._margin_cap_steps = sim._dd_margin_cap
    P = _lib.ptr
    ctx = sim._ctx
    ctx.call("gf_set_decomposition", P(st.dd), C.c_double(st.lever), C.c_int(st.plan.axis),
             C.c_double(st.plan.travel))
    rec = int(ctx.L.gf_halo_record_bytes(C.c_void_p(ctx.h)))
    inv = np.full(st.global_store.n_owners, -1, np.int64)
    inv[st.gids] = np.arange(st.gids.size)
    st.peers = {}
    for q, (send, recv) in st.plan.halo(st.rank).items():
        st.peers[q] = _Peer(q, inv[send], inv[recv], rec, sim.device)
    st.word = torch.full((1,), INT64_MAX, dtype=torch.int64, device=torch.device("cuda", sim.device))
    # torch fills on its own stream; the context's streams are non-blocking
    torch.cuda.synchronize(sim.device)


# ----------------------------------------------------------------------------
# halo calls on one context
# ----------------------------------------------------------------------------
def _call(sim, name, *args):
    L = sim._ctx.L
    rc = getattr(L, name)(C.c_void_p(sim._ctx.h), *args)
    if rc != 0:
        raise RuntimeError(f"{name} failed: {sim._ctx.error()}")


def _pack_forces(sim, p):
    if p.n_recv:
        _call(sim, "gf_pack_forces", C.c_void_p(p.recv_idx.data_ptr()), C.c_int64(p.n_recv),
              C.c_void_p(p.force_out.data_ptr()))


def _add_forces(sim, p, buf):
    if p.n_send:
        _call(sim, "gf_add_forces", C.c_void_p(p.send_idx.data_ptr()), C.c_int64(p.n_send),
              C.c_void_p(buf.data_ptr()))


def _pack_state(sim, p):
    if p.n_send:
        _call(sim, "gf_pack_state", C.c_void_p(p.send_idx.data_ptr()), C.c_int64(p.n_send),
              C.c_void_p(p.state_out.data_ptr()))


def _unpack_state(sim, p, buf):
    if p.n_recv:
        _call(sim, "gf_unpack_state", C.c_void_p(p.recv_idx.data_ptr()), C.c_int64(p.n_recv),
              C.c_void_p(buf.data_ptr()))


def _word(sim, mode):
    _call(sim, "gf_trip_word", C.c_void_p(sim._dd.word.data_ptr()), C.c_int(mode))


class _LoopbackTransport:
    """All ranks' contexts in this process (one device): a peer's outgoing
    buffer is read directly; host syncs order the contexts' streams."""

    def __init__(self, sims):
        self.sims = sims

    def _sync(self):
        for s in self.sims:
            _call(s, "gf_sync")

    def forces(self):
        for s in self.sims:
            for p in s._dd.peers.values():
                _pack_forces(s, p)
        self._sync()
        for s in self.sims:
            for q, p in s._dd.peers.items():
                _add_forces(s, p, self.sims[q]._dd.peers[s._dd.rank].force_out)
        self._sync()

    def state(self):
        import torch
        for s in self.sims:
            for p in s._dd.peers.values():
                _pack_state(s, p)
            _word(s, 0)
        self._sync()
        lo = torch.stack([s._dd.word for s in self.sims]).min()
        for s in self.sims:
            for q, p in s._dd.peers.items():
                _unpack_state(s, p, self.sims[q]._dd.peers[s._dd.rank].state_out)
            s._dd.word.fill_(lo)
        torch.cuda.synchronize()
        for s in self.sims:
            _word(s, 1)
        self._sync()

    def allreduce(self, values, op):
        vals = np.asarray(values, dtype=np.float64)
        return vals.max(axis=0) if op == "max" else vals.min(axis=0)

    def allgather(self, payloads):
        return payloads

    def neighbours(self, payloads):
        """Per member: {rank: payload} of its slab neighbours and itself."""
        n = len(payloads)
        return [{q: payloads[q] for q in (r - 1, r, r + 1) if 0 <= q < n} for r in range(n)]


def p2p_exchange(pairs) -> None:
    """One batched point-to-point round: pairs = [(peer, out, n_out, in, n_in)];
    tensors are sent / received whole when the count is non-zero.  Both sides
    derive the counts from the same SlabPlan, so every send has its receive."""
    import torch.distributed as dist
    ops = []
    for q, out, n_out, inp, n_in in pairs:
        if n_out:
            ops.append(dist.P2POp(dist.isend, out, q))
        if n_in:
            ops.append(dist.P2POp(dist.irecv, inp, q))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


class _NcclTransport:
    """One context per process; peers over NCCL (torch.distributed), ordered
    on the context's dT stream: no host synchronisation per step.

    Under a gloo process group (several processes sharing one GPU -- NCCL
    refuses two ranks per device -- used by the multi-process test) the same
    protocol runs with the buffers staged through host memory."""

    def __init__(self, sim):
        import torch.distributed as dist
        self.sim = sim
        self._stream, self._stream_ctx = None, None
        self.staged = dist.get_backend() != "nccl"

    @property
    def stream(self):
        """The context's dT stream as a torch stream (re-wrapped when a
        repartition rebuilt the context)."""
        import torch
        ctx = self.sim._ctx
        ptr = int(ctx.L.gf_stream(C.c_void_p(ctx.h)) or 0)
        if self._stream_ctx != ptr:
            self._stream = torch.cuda.ExternalStream(ptr, device=torch.device("cuda", self.sim.device))
            self._stream_ctx = ptr
        return self._stream

    def _p2p(self, pairs):
        if not self.staged:
            p2p_exchange(pairs)
            return
        self.stream.synchronize()
        host = [(q, out.cpu(), n_out, inp.cpu(), n_in, inp) for q, out, n_out, inp, n_in in pairs]
        p2p_exchange([(q, o, no, i, ni) for q, o, no, i, ni, _ in host])
        for _, _, _, i, ni, dev in host:
            if ni:
                dev.copy_(i)
        import torch
        torch.cuda.synchronize(self.sim.device)

    def _min_word(self, word):
        import torch
        import torch.distributed as dist
        if not self.staged:
            dist.all_reduce(word, op=dist.ReduceOp.MIN)
            return
        self.stream.synchronize()
        h = word.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MIN)
        word.copy_(h)
        torch.cuda.synchronize(self.sim.device)

    def forces(self):
        import torch
        s = self.sim
        with torch.cuda.stream(self.stream):
            for p in s._dd.peers.values():
                _pack_forces(s, p)
            self._p2p([(q, p.force_out, p.n_recv, p.force_in, p.n_send) for q, p in s._dd.peers.items()])
            for p in s._dd.peers.values():
                _add_forces(s, p, p.force_in)

    def state(self):
        import torch
        import torch.distributed as dist
        s = self.sim
        with torch.cuda.stream(self.stream):
            for p in s._dd.peers.values():
                _pack_state(s, p)
            self._p2p([(q, p.state_out, p.n_send, p.state_in, p.n_recv) for q, p in s._dd.peers.items()])
            for p in s._dd.peers.values():
                _unpack_state(s, p, p.state_in)
            # the guard: a trip in this step's integration stops every rank
            # before the next step's force phase (contact history included)
            _word(s, 0)
            self._min_word(s._dd.word)
            _word(s, 1)

    def allreduce(self, values, op):
        import torch
        import torch.distributed as dist
        rows = np.asarray(values, dtype=np.float64)
        local = rows.max(axis=0) if op == "max" else rows.min(axis=0)
        t = torch.as_tensor(local, device="cpu" if self.staged else torch.device("cuda", self.sim.device))
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.MIN)
        return t.cpu().numpy()

    def allgather(self, payloads):
        import torch.distributed as dist
        out = [None] * dist.get_world_size()
        dist.all_gather_object(out, payloads[0])
        return out

    def neighbours(self, payloads):
        """{rank: payload} of this rank's slab neighbours and itself: two
        passes of point-to-point object transfers (right, then left); even
        ranks send first, odd ranks receive first, so a chain never blocks."""
        import torch.distributed as dist
        r, n = dist.get_rank(), dist.get_world_size()
        got = {r: payloads[0]}
        for step in (1, -1):
            dst, src = r + step, r - step
            box = [None]
            send = (lambda: dist.send_object_list([payloads[0]], dst)) if 0 <= dst < n else (lambda: None)

            def recv():
                if 0 <= src < n:
                    dist.recv_object_list(box, src)
                    got[src] = box[0]
            if r % 2 == 0:
                send()
                recv()
            else:
                recv()
                send()
        return [got]


# ----------------------------------------------------------------------------
# driving
# ----------------------------------------------------------------------------
def run_member(sim, steps: int) -> None:
    """Simulator._run of a decomposed simulator (one rank per process)."""
    if sim.decomposition.group is not None:
        raise ConfigurationError("a LoopbackGroup member is driven by group.do_dynamics()")
    run_ranks([sim], steps, _NcclTransport(sim))


def gather(sim) -> dict:
    """gather_state for one rank per process (every rank calls it)."""
    return gather_state([sim], _NcclTransport(sim))


def run_ranks(sims, steps: int, xport) -> None:
    """Advance every rank held by this process by `steps` steps, lockstep,
    repartitioning whenever the travel guard trips."""
    remaining = steps
    while remaining > 0:
        rrs = _lockstep(sims, remaining, xport)
        done = int(rrs[0].steps_done)
        trip = min((int(r.dd_trip_step) for r in rrs if r.dd_trip_step >= 0), default=-1)
        err = max(1 if (r.oob_owner >= 0 or r.bad_owner >= 0) else 0 for r in rrs)
        agreed = xport.allreduce([[err, 0 if trip < 0 else 1, max(s.scheduler.n_max for s in sims)]]
                                 * len(sims), "max")
        for s, rr in zip(sims, rrs):
            s._finish_run(rr, rr.wall_ms * 1e-3, adapt=False)   # raises on this rank's watchdog
        if agreed[0] > 0:
            raise DecompositionError("a watchdog tripped on another rank; the run is stopped")
        for s in sims:
            s._adapt_n_max(waited_event=False)
        n_max = int(xport.allreduce([[max(s.scheduler.n_max for s in sims)]] * len(sims), "max")[0])
        for s in sims:
            s.scheduler.n_max = n_max
            s.margin_policy.n_max = n_max
        remaining -= done
        if agreed[1] > 0:
            repartition(sims, xport)


def _lockstep(sims, steps, xport):
    keep = []
    for s in sims:
        s._push_host()
        rp, arrs = s._run_params(steps)
        keep.append((rp, arrs))
    sched = [(rp.period, rp.lag, rp.margin) for rp, _ in keep]
    if len(set(sched)) != 1:
        raise DecompositionError(f"ranks disagree on the kT/dT schedule: {sched}")
    for s, (rp, _) in zip(sims, keep):
        s._ctx.call("gf_run_begin", C.byref(rp))
    rrs = [_lib.RunResult() for _ in sims]
    try:
        for i in range(steps):
            for s in sims:
                _call(s, "gf_step_forces", C.c_int64(i))
            xport.forces()
            for s in sims:
                _call(s, "gf_step_integrate", C.c_int64(i))
            xport.state()
    finally:
        errs = []
        for s, rr in zip(sims, rrs):
            try:
                s._ctx.call("gf_run_end", C.byref(rr))
            except RuntimeError as e:   # keep the first failure
                errs.append(e)
        if errs:
            raise errs[0]
    return rrs


def _local_payload(sim) -> dict:
    st = sim._dd
    sim._sync_all()
    s = sim.store
    n = s.n_owners
    d = s.__dict__
    cls = st.dd & 3
    mine = (cls == DD_LOCAL) | (cls == DD_PRIMARY)
    rows = np.nonzero(mine)[0]
    out = {"gid": st.gids[rows]}
    for name in ("voxel", "subvoxel", "quat", "lin_vel", "ang_vel", "owner_family", "acc_force",
                 "acc_torque", "ext_force", "ext_torque"):
        out[name] = d["_" + name][:n][rows].copy()
    ca = sim._acs
    out["acs_kind"] = ca.kind.copy()
    out["acs_a"] = st.geoms[ca.geom_a] if ca.size else np.zeros(0, np.int64)
    out["acs_b"] = st.geoms[ca.geom_b] if ca.size else np.zeros(0, np.int64)
    out["acs_wild"] = {k: v.copy() for k, v in ca.wildcards.items()}
    return out


def gather_state(sims, xport) -> dict:
    """Global owner state (by global owner id) and the global contact set
    (global geometry ids, canonical order) assembled from every rank."""
    parts = xport.allgather([_local_payload(s) for s in sims])
    g = sims[0]._dd.global_store
    n = g.n_owners
    d = g.__dict__
    state = {}
    for name in ("voxel", "subvoxel", "quat", "lin_vel", "ang_vel", "owner_family", "acc_force",
                 "acc_torque", "ext_force", "ext_torque"):
        arr = d["_" + name][:n].copy()
        for p in parts:
            arr[p["gid"]] = p[name]
        state[name] = arr
    kind = np.concatenate([p["acs_kind"] for p in parts]) if parts else np.zeros(0, np.uint8)
    ga = np.concatenate([p["acs_a"] for p in parts]).astype(np.int64)
    gb = np.concatenate([p["acs_b"] for p in parts]).astype(np.int64)
    names = list(parts[0]["acs_wild"].keys()) if parts else []
    wild = {k: np.concatenate([p["acs_wild"][k] for p in parts]) for k in names}
    ca = B.ContactArray(kind, ga, gb, wild).canonicalize()
    if ca.size:
        keys = ca.sort_keys()
        first = np.concatenate([[True], keys[1:] != keys[:-1]])
        ca = ca.select(first)
    from .core import decode_position
    state["pos"] = decode_position(state["voxel"], state["subvoxel"], g.domain)
    state["acs"] = ca
    return state


def update_global(sim_or_group, edit) -> None:
    """Host edit of a decomposed scene: gather the global state, apply
    ``edit(global_store)`` on every member's copy of the scene, repartition.
    Every rank calls it with the same edit (one process per GPU), or a
    LoopbackGroup is passed."""
    if isinstance(sim_or_group, LoopbackGroup):
        sims, xport = sim_or_group.sims, _LoopbackTransport(sim_or_group.sims)
    else:
        sims, xport = [sim_or_group], _NcclTransport(sim_or_group)
    repartition(sims, xport, edit)


def _rehome(plan: SlabPlan, pos: np.ndarray) -> SlabPlan:
    """The same cuts (and pad, travel, big owners), owners re-homed by their
    current coordinate."""
    x = pos[:, plan.axis].copy()
    home = plan.home.copy()
    el = home >= 0
    home[el] = np.searchsorted(plan.cuts, x[el], side="right")
    return SlabPlan(plan.n_ranks, plan.axis, plan.cuts.copy(), plan.pad, plan.travel, home, x, plan.reach,
                    plan.big, plan.margin)


def repartition(sims, xport, edit=None) -> None:
    """Migration after a travel-guard trip.  Incremental by default: every
    rank exchanges its owners and contact history with its two slab
    neighbours only (no global gather -- an owner moved at most `travel`, so
    a rank's new piece and every contact it now computes came from itself or
    a neighbour), re-homes owners under the same slab cuts and rebuilds its
    context.  A host edit, or slabs drifted out of balance (the largest
    rank above 1.5x the smallest), take the global path: gather everything
    and cut new balanced slabs."""
    if edit is None:
        counts = [int(np.sum((s._dd.dd & 3) == DD_LOCAL)) for s in sims]
        hi = xport.allreduce([[max(counts)]], "max")[0]
        lo = xport.allreduce([[min(counts)]], "min")[0]
        if lo > 0 and hi <= 1.5 * lo:
            _migrate_neighbours(sims, xport)
            return
    _repartition_global(sims, xport, edit)


_STATE_FIELDS = ("voxel", "subvoxel", "quat", "lin_vel", "ang_vel", "owner_family", "acc_force", "acc_torque",
                 "ext_force", "ext_torque")


def _migrate_neighbours(sims, xport) -> None:
    nb = xport.neighbours([_local_payload(s) for s in sims])
    from .core import decode_position
    for s, parts in zip(sims, nb):
        g = s._dd.global_store
        n = g.n_owners
        d = g.__dict__
        for p in parts.values():
            for name in _STATE_FIELDS:
                d["_" + name][:n][p["gid"]] = p[name]
        kind = np.concatenate([p["acs_kind"] for p in parts.values()])
        ga = np.concatenate([p["acs_a"] for p in parts.values()]).astype(np.int64)
        gb = np.concatenate([p["acs_b"] for p in parts.values()]).astype(np.int64)
        names = list(next(iter(parts.values()))["acs_wild"].keys())
        wild = {k: np.concatenate([p["acs_wild"][k] for p in parts.values()]) for k in names}
        ca = B.ContactArray(kind, ga, gb, wild).canonicalize()
        if ca.size:
            keys = ca.sort_keys()
            ca = ca.select(np.concatenate([[True], keys[1:] != keys[:-1]]))
        pos = decode_position(d["_voxel"][:n], d["_subvoxel"][:n], g.domain)
        s._dd.next_plan = _rehome(s._dd.plan, pos)
        s._acs0_next = ca
    for s in sims:
        s._ctx.close()
        s._ctx = None
        s.store._sync_hook = None
        s.store = s._dd.global_store
        s._acs0 = s._acs0_next
        del s._acs0_next
        s._initialized = False
        s._host_stale = False
        s._host_dirty = False
        s.initialize()
        s.scheduler.repartitions = getattr(s.scheduler, "repartitions", 0) + 1
        s.scheduler.migrations_incremental = getattr(s.scheduler, "migrations_incremental", 0) + 1


def _repartition_global(sims, xport, edit=None) -> None:
    """Gather every rank's owners and contact history, cut new slabs from the
    current positions and rebuild each rank's context (the history is
    carried over, so contacts keep their tangential state)."""
    for s in sims:
        s._dd.next_plan = None
    state = gather_state(sims, xport)
    # every member holds its own copy of the global scene (one per process
    # under NCCL; one per Simulator in a LoopbackGroup): update each
    for s in sims:
        g = s._dd.global_store
        n = g.n_owners
        d = g.__dict__
        for name in ("voxel", "subvoxel", "quat", "lin_vel", "ang_vel", "owner_family", "acc_force",
                     "acc_torque", "ext_force", "ext_torque"):
            d["_" + name][:n] = state[name]
        if edit is not None:
            edit(g)
    for s in sims:
        s._ctx.close()
        s._ctx = None
        s.store._sync_hook = None
        s.store = s._dd.global_store
        s._acs0 = state["acs"]
        s._initialized = False
        s._host_stale = False
        s._host_dirty = False
        s.initialize()
    if edit is None:
        for s in sims:
            s.scheduler.repartitions = getattr(s.scheduler, "repartitions", 0) + 1
