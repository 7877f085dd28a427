"""Host side of the spatial slab decomposition (decomp.py), on CPU: the
partition, the ghost layer's coverage of every possible cross-slab contact,
the one-rank-per-contact rule the device applies (gf_common.cuh dd_keep),
and the halo protocol over torch.distributed (gloo, world size 2 and 3 --
the same p2p_exchange the NCCL transport uses)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_04648_b200 import decomp


def dd_keep(dd, a, b):
    """Python statement of gf_common.cuh dd_keep (the device rule)."""
    ca, cb = dd[a] & 3, dd[b] & 3
    if ca == decomp.DD_GHOST or cb == decomp.DD_GHOST:
        if ca == decomp.DD_LOCAL:
            return (dd[a] >> 2) < (dd[b] >> 2)
        if cb == decomp.DD_LOCAL:
            return (dd[b] >> 2) < (dd[a] >> 2)
        return False
    if ca == decomp.DD_LOCAL or cb == decomp.DD_LOCAL:
        return True
    return ca == decomp.DD_PRIMARY and cb == decomp.DD_PRIMARY


def scene(n=3000, seed=1):
    rng = np.random.default_rng(seed)
    pos = rng.uniform((-0.3, -0.05, 0.0), (0.3, 0.05, 0.1), (n, 3))
    eligible = np.ones(n, bool)
    eligible[-2:] = False                      # two boundary owners (walls)
    reach = np.where(eligible, rng.uniform(0.002, 0.004, n), np.inf)
    reach[:3] = (0.02, 0.013, 0.03)            # big owners (projectiles) with their own halo
    pos[0, 0], pos[1, 0] = 0.0, -0.1          # ... near the slab cuts
    return pos, eligible, reach


@pytest.mark.parametrize("n_ranks", [1, 2, 3, 5])
def test_partition_is_balanced_and_complete(n_ranks):
    pos, el, reach = scene()
    plan = decomp.plan_slabs(pos, el, reach, n_ranks, margin=1e-3, travel=2e-3)
    assert plan.axis == 0                      # longest extent
    homes = plan.home[el]
    counts = np.bincount(homes, minlength=n_ranks)
    assert counts.sum() == el.sum()
    assert counts.max() - counts.min() <= 1
    assert np.all(plan.home[~el] == -1)
    for r in range(n_ranks):
        c = plan.classes(r)
        assert np.all(c[~el] == (decomp.DD_PRIMARY if r == 0 else decomp.DD_SHARED))
        assert np.all((c == decomp.DD_LOCAL) == (plan.home == r))


@pytest.mark.parametrize("n_ranks", [2, 3, 4])
def test_every_contact_is_computed_exactly_once(n_ranks):
    """For every pair of owners that can touch while both stay within
    `travel` of their partition coordinate, exactly one rank holds both and
    computes the pair under dd_keep."""
    pos, el, reach = scene(1500)
    travel = 2e-3
    plan = decomp.plan_slabs(pos, el, reach, n_ranks, margin=1e-3, travel=travel)
    n = pos.shape[0]
    dds = []
    for r in range(n_ranks):
        c = plan.classes(r)
        dd = np.where(c >= 0, c, 0).astype(np.int64) | (np.arange(n, dtype=np.int64) << 2)
        dds.append((c, dd))
    assert plan.big.tolist() == [0, 1, 2]
    idx = np.nonzero(el)[0]
    for i in idx[:400]:
        # worst case: both move `travel` towards each other along the axis
        near = idx[np.abs(pos[idx, plan.axis] - pos[i, plan.axis]) < reach[i] + reach[idx] + 1e-3 + 2 * travel]
        for j in near:
            if j == i:
                continue
            holders = [r for r, (c, dd) in enumerate(dds) if c[i] >= 0 and c[j] >= 0 and dd_keep(dd, i, j)]
            assert len(holders) == 1, (i, j, holders)
            assert plan.home[i] in holders or plan.home[j] in holders
        # every clump-wall pair is computed on the clump's home rank only
        for w in np.nonzero(~el)[0]:
            holders = [r for r, (c, dd) in enumerate(dds) if c[i] >= 0 and dd_keep(dd, i, w)]
            assert holders == [plan.home[i]]


def test_halo_lists_are_symmetric():
    pos, el, reach = scene()
    plan = decomp.plan_slabs(pos, el, reach, 4, margin=1e-3, travel=2e-3)
    halos = [plan.halo(r) for r in range(4)]
    for r in range(4):
        for q, (send, recv) in halos[r].items():
            s2, r2 = halos[q][r]
            np.testing.assert_array_equal(send, r2)
            np.testing.assert_array_equal(recv, s2)
            assert np.all(plan.home[send] == r) and np.all(plan.home[recv] == q)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _halo_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pos, el, reach = scene()
        plan = decomp.plan_slabs(pos, el, reach, world, margin=1e-3, travel=2e-3)
        state = np.arange(pos.shape[0], dtype=np.int64) * 7 + 3    # an owner's "state" = f(gid)
        forces = np.zeros(pos.shape[0], np.int64)
        pairs, peers = [], plan.halo(rank)
        bufs = {}
        for q, (send, recv) in peers.items():
            bufs[q] = (torch.as_tensor(state[send]), torch.zeros(recv.size, dtype=torch.int64))
            pairs.append((q, bufs[q][0], send.size, bufs[q][1], recv.size))
        decomp.p2p_exchange(pairs)
        ok = all(np.array_equal(bufs[q][1].numpy(), state[peers[q][1]]) for q in peers)
        # force return: every ghost sends back (gid + 1); the home adds them up
        pairs, back = [], {}
        for q, (send, recv) in peers.items():
            back[q] = (torch.as_tensor(peers[q][1] + 1), torch.zeros(send.size, dtype=torch.int64))
            pairs.append((q, back[q][0], recv.size, back[q][1], send.size))
        decomp.p2p_exchange(pairs)
        for q, (send, recv) in peers.items():
            np.add.at(forces, send, back[q][1].numpy())
        expect = np.zeros_like(forces)
        for q in range(world):
            if q != rank:
                g = plan.ghost_on(q) & (plan.home == rank)
                expect[g] += np.nonzero(g)[0] + 1
        ok = ok and np.array_equal(forces, expect)
        w = torch.tensor([rank * 10 + 5], dtype=torch.int64)
        dist.all_reduce(w, op=dist.ReduceOp.MIN)   # the guard word
        ok = ok and int(w) == 5
        out[rank] = 1 if ok else 0
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert list(out) == [1] * world


def _neighbour_worker(rank, world, port, out):
    """The incremental migration's exchange: every rank gets exactly its slab
    neighbours' payloads (and its own), and re-homing under the same cuts
    moves an owner only to an adjacent slab."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = decomp._NcclTransport.__new__(decomp._NcclTransport)
        got = x.neighbours([{"rank": rank, "data": np.arange(rank + 3)}])[0]
        want = {q for q in (rank - 1, rank, rank + 1) if 0 <= q < world}
        ok = set(got) == want and all(got[q]["rank"] == q and got[q]["data"].size == q + 3 for q in got)
        pos, el, reach = scene()
        plan = decomp.plan_slabs(pos, el, reach, world, margin=1e-3, travel=2e-3)
        moved = pos.copy()
        moved[:, plan.axis] += np.where(np.arange(pos.shape[0]) % 2 == 0, 1.5e-3, -1.5e-3)
        new = decomp._rehome(plan, moved)
        ok = ok and np.array_equal(new.cuts, plan.cuts) and new.pad == plan.pad
        eligible = plan.home >= 0
        ok = ok and np.all(np.abs(new.home[eligible] - plan.home[eligible]) <= 1)
        out[rank] = 1 if ok else 0
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_neighbour_migration_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_neighbour_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert list(out) == [1] * world
