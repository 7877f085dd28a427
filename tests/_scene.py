"""Test helper: upload an oracle-layout scene dict (tests/golden, oracle.OracleStepper)
straight into a device context through the C-ABI."""

import ctypes as C

import numpy as np

from paper_2311_04648_b200 import _lib
from paper_2311_04648_b200.forces import beta_table

GEOM_SPHERE, GEOM_TRIANGLE, GEOM_PLANE, GEOM_CYLINDER = 0, 1, 2, 3
P = _lib.ptr
A = _lib.carr


def slots(scene):
    kinds = scene["geom_kind"]
    sph = np.nonzero(kinds == GEOM_SPHERE)[0]
    tri = np.nonzero(kinds == GEOM_TRIANGLE)[0]
    ana = np.nonzero((kinds == GEOM_PLANE) | (kinds == GEOM_CYLINDER))[0]
    slot = np.zeros(kinds.shape[0], np.int64)
    for arr in (sph, tri, ana):
        slot[arr] = np.arange(arr.shape[0])
    return sph, tri, ana, slot


def upload_scene(scene, f32_state=False, device=0):
    ctx = _lib.Context(device, f32_state=f32_state)
    s = scene
    ctx.call("gf_set_domain", P(A(s["lo"], np.float64)), P(A(s["hi"], np.float64)),
             C.c_double(float(s["edge"])))
    flags = (A(s["fixed_flag"], np.uint8) | (A(s["prescribed_flag"], np.uint8) << 1)).astype(np.uint8)
    bits = np.array([1, 2, 4], np.uint8)
    lvm = (A(s["lv_mask"], np.uint8) * bits).sum(axis=1).astype(np.uint8)
    avm = (A(s["av_mask"], np.uint8) * bits).sum(axis=1).astype(np.uint8)
    keep = [A(s["mask"], np.uint8).reshape(-1), flags, lvm, avm, A(s["lv_val"], np.float64),
            A(s["av_val"], np.float64)]
    ctx.call("gf_upload_families", *[P(a) for a in keep])
    ps = A(s["pair_stack"], np.float64)
    beta = A(beta_table(ps), np.float64)
    ctx.call("gf_upload_materials", C.c_int(ps.shape[1]), C.c_int(ps.shape[0]), P(ps), P(beta))
    n = s["voxel"].shape[0]
    mm = np.concatenate([s["mass"][:, None], s["moi"]], axis=1)
    rows, tid = np.unique(mm, axis=0, return_inverse=True)
    tid = A(np.asarray(tid).reshape(-1), np.uint32)
    keep = [A(s["voxel"], np.uint64), A(s["subvoxel"], np.uint16), A(s["quat"], np.float32),
            A(s["lin_vel"], np.float64), A(s["ang_vel"], np.float64), A(s["owner_family"], np.uint8),
            tid, A(rows[:, 0], np.float64), A(rows[:, 1:], np.float64)]
    ctx.call("gf_upload_owners", C.c_int64(n), P(keep[0]), P(keep[1]), P(keep[2]), P(keep[3]),
             P(keep[4]), P(keep[5]), P(keep[6]), C.c_int64(rows.shape[0]), P(keep[7]), P(keep[8]))
    ef, et = A(s["ext_force"], np.float64), A(s["ext_torque"], np.float64)
    if np.any(ef != 0) or np.any(et != 0):
        ctx.call("gf_set_external_loads", P(ef), P(et))
    sph, tri, ana, _ = slots(s)
    gp, go, gm = s["geom_params"], s["geom_owner"], s["geom_material"]
    keep = [A(go[sph], np.int64), A(gp[sph, :4], np.float32), A(gm[sph], np.uint8),
            A(go[tri], np.int64), A(gp[tri, :9], np.float32), A(gm[tri], np.uint8),
            A(go[ana], np.int64), A(s["geom_kind"][ana], np.uint8), A(gp[ana, :8], np.float32),
            A(gm[ana], np.uint8)]
    ctx.call("gf_upload_geometry", C.c_int64(sph.size), P(keep[0]), P(keep[1]), P(keep[2]),
             C.c_int64(tri.size), P(keep[3]), P(keep[4]), P(keep[5]), C.c_int64(ana.size),
             P(keep[6]), P(keep[7]), P(keep[8]), P(keep[9]))
    return ctx


def set_acs(ctx, kind, slot_a, slot_b, wild):
    kind, sa, sb = A(kind, np.uint8), A(slot_a, np.int64), A(slot_b, np.int64)
    wild = A(wild, np.float32)
    ctx.call("gf_set_acs", C.c_int64(kind.shape[0]), P(kind), P(sa), P(sb), P(wild), C.c_int(4))


def get_acs(ctx, which=0):
    n = int(ctx.L.gf_acs_size(C.c_void_p(ctx.h), which))
    kind = np.zeros(n, np.uint8)
    sa = np.zeros(n, np.int64)
    sb = np.zeros(n, np.int64)
    wild = np.zeros((n, 4), np.float32)
    if n:
        ctx.call("gf_get_acs", C.c_int(which), P(kind), P(sa), P(sb), P(wild) if which == 0 else None)
    return kind, sa, sb, wild


def download_state(ctx, n):
    vox = np.zeros(n, np.uint64)
    sub = np.zeros((n, 3), np.uint16)
    quat = np.zeros((n, 4), np.float32)
    lv = np.zeros((n, 3))
    av = np.zeros((n, 3))
    ctx.call("gf_download_owners", P(vox), P(sub), P(quat), P(lv), P(av), None)
    af = np.zeros((n, 3))
    at = np.zeros((n, 3))
    ctx.call("gf_download_accumulators", P(af), P(at))
    return dict(voxel=vox, subvoxel=sub, quat=quat, lin_vel=lv, ang_vel=av, acc_f=af, acc_t=at)


def dt_step(ctx, scene, sim_time, step=0, write_acc=1):
    sp = _lib.StepParams()
    sp.h = float(scene["h"])
    for a in range(3):
        sp.g[a] = float(scene["gravity"][a])
    sp.v_err = float(scene["v_err"])
    sp.sim_time = float(sim_time)
    sp.step = step
    sp.write_acc = write_acc
    touching, bad, oob = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    ctx.call("gf_dt_step", C.byref(sp), C.byref(touching), C.byref(bad), C.byref(oob))
    return touching.value, bad.value, oob.value


def run(ctx, scene, n_steps, margin, period=1, lag=0, step0=0):
    rp = _lib.RunParams()
    rp.n_steps = n_steps
    rp.step0 = step0
    rp.h = float(scene["h"])
    for a in range(3):
        rp.g[a] = float(scene["gravity"][a])
    rp.v_err = float(scene["v_err"])
    rp.margin = float(margin)
    rp.period = period
    rp.lag = lag
    rp.n_dyn = 0
    rp.write_acc = 1
    rr = _lib.RunResult()
    ctx.call("gf_run", C.byref(rp), C.byref(rr))
    return rr
