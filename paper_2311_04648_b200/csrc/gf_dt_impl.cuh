// gf_dt_impl.cuh -- dynamics worker (dT) kernels, templated on the storage
// type of owner velocities (VelT = double: the reference's STATE_REAL,
// types.py:20, bitwise parity build; VelT = float: the paper's compact fp32
// velocity layout, throughput build).  Per-contact arithmetic is fp64 scratch
// in both builds (types.py:22), so force evaluation order matches the
// reference statement by statement.
//
// Per step:
//   k_contacts   one thread per ACS entry: contact geometry
//                (_kernels.py:442-491), pair kinematics (forces.py:55-79) and
//                the Hertz-Mindlin core (forces.py:82-182); writes F,
//                F + torque_only_force and the contact point of touching
//                entries plus a touch flag, updates the history in place.
//   k_heavy      one CTA per owner with > kHeavyThreshold incidences (walls,
//                meshes): fixed-order tree reduction of its contributions.
//   k_integrate  one thread per owner: the owner's contributions summed in
//                canonical ACS order (bit-identical to reduce_to_owners,
//                _kernels.py:515-545), then the semi-implicit Euler update,
//                prescriptions, quaternion renormalisation, re-encode /
//                decode and the watchdog (_kernels.py:548-670) -- fused.
#pragma once
#include "gf_context.h"

namespace gf {



template <typename VelT> struct Vel;
template <> struct Vel<double> {
  static __device__ __forceinline__ void load(const void *p, int64_t i, double v[3]) {
    const double2 *q = reinterpret_cast<const double2 *>(p) + 2 * i;
    double2 a = q[0], b = q[1];
    v[0] = a.x; v[1] = a.y; v[2] = b.x;
  }
  static __device__ __forceinline__ void store(void *p, int64_t i, const double v[3]) {
    double2 *q = reinterpret_cast<double2 *>(p) + 2 * i;
    q[0] = make_double2(v[0], v[1]);
    q[1] = make_double2(v[2], 0.0);
  }
};
template <> struct Vel<float> {
  static __device__ __forceinline__ void load(const void *p, int64_t i, double v[3]) {
    float4 a = reinterpret_cast<const float4 *>(p)[i];
    v[0] = a.x; v[1] = a.y; v[2] = a.z;
  }
  static __device__ __forceinline__ void store(void *p, int64_t i, const double v[3]) {
    reinterpret_cast<float4 *>(p)[i] = make_float4(float(v[0]), float(v[1]), float(v[2]), 0.f);
  }
};

struct DtView {
  Domain dom;
  Owners own;
  Spheres sph;
  Tris tri;
  Anas ana;
  Materials mat;
  Families fam;
  int64_t n_acs;
  const uint2 *ids;
  float *wild;
  int W;
  double *out_c;        // [n_acs*9]
  uint8_t *touch;       // [n_acs]
  const uint32_t *inc;  // B-side incidences: contact indices sorted by (B owner, k)
  const uint32_t *inc_start;  // per owner start in inc
  const unsigned long long *seg;  // (kind, sphere A) segment starts of the active array
  int64_t n_sph;
  const uint32_t *heavy;
  const unsigned long long *n_heavy;
  double *heavy_acc;    // [n_owner*6] (only heavy owners written)
  Status *st;
};

// Hertz-Mindlin core (forces.py:82-182); returns false for a false positive.
__device__ __forceinline__ void hertz_mindlin(double overlap, double ts, double b2ax, double b2ay,
                                              double b2az, double vx, double vy, double vz,
                                              double wrx, double wry, double wrz, double mass_eff,
                                              double ra, double rb, int ma, int mb,
                                              const Materials &M, float *wild, double out[6]) {
  const int mm = M.n_mat * M.n_mat, ab = ma * M.n_mat + mb;
  const double e_cnt = M.pair[ab], g_cnt = M.pair[mm + ab];
  const double mu = M.pair[3 * mm + ab], crr = M.pair[4 * mm + ab];
  const double beta = M.beta[ab];
  for (int q = 0; q < 6; ++q) out[q] = 0.0;

  double projection = vx * b2ax + vy * b2ay + vz * b2az;
  double vtx = vx - projection * b2ax;
  double vty = vy - projection * b2ay;
  double vtz = vz - projection * b2az;
  float4 w0 = *reinterpret_cast<const float4 *>(wild);
  double dtx = double(w0.x) + ts * vtx;
  double dty = double(w0.y) + ts * vty;
  double dtz = double(w0.z) + ts * vtz;
  double disp_proj = dtx * b2ax + dty * b2ay + dtz * b2az;
  dtx -= disp_proj * b2ax;
  dty -= disp_proj * b2ay;
  dtz -= disp_proj * b2az;
  double delta_time = double(w0.w) + ts;

  double sqrt_rd = sqrt(overlap * (ra * rb) / (ra + rb));
  double sn = 2.0 * e_cnt * sqrt_rd;
  double k_n = 2.0 / 3.0 * sn;
  double gamma_n = 2.0 * sqrt(5.0 / 6.0) * beta * sqrt(sn * mass_eff);
  double fn = k_n * overlap + gamma_n * projection;
  out[0] = fn * b2ax;
  out[1] = fn * b2ay;
  out[2] = fn * b2az;

  if (crr > 0.0) {
    bool add_rolling = true;
    double r_eff = sqrt((ra * rb) / (ra + rb));
    double kn_simple = 4.0 / 3.0 * e_cnt * sqrt(r_eff);
    double gn_simple = -2.0 * sqrt(5.0 / 3.0 * mass_eff * e_cnt) * beta * pow(r_eff, 0.25);
    double d_coeff = gn_simple / (2.0 * sqrt(kn_simple * mass_eff));
    if (d_coeff < 1.0) {
      double t_collision = kPi * sqrt(mass_eff / (kn_simple * (1.0 - d_coeff * d_coeff)));
      if (delta_time <= t_collision) add_rolling = false;
    }
    if (add_rolling) {
      double v_rot_mag = sqrt(wrx * wrx + wry * wry + wrz * wrz);
      if (v_rot_mag > 1e-12) {
        double fmag = sqrt(out[0] * out[0] + out[1] * out[1] + out[2] * out[2]);
        double scale = crr * fmag / v_rot_mag;
        out[3] = wrx * scale;
        out[4] = wry * scale;
        out[5] = wrz * scale;
      }
    }
  }
  if (mu > 0.0) {
    double kt = 8.0 * g_cnt * sqrt_rd;
    double gt = -2.0 * sqrt(5.0 / 6.0) * beta * sqrt(mass_eff * kt);
    double tfx = -kt * dtx - gt * vtx;
    double tfy = -kt * dty - gt * vty;
    double tfz = -kt * dtz - gt * vtz;
    double ft = sqrt(tfx * tfx + tfy * tfy + tfz * tfz);
    if (ft > 1e-12) {
      double fmag = sqrt(out[0] * out[0] + out[1] * out[1] + out[2] * out[2]);
      double ft_max = fmag * mu;
      if (ft > ft_max) {
        double scale = ft_max / ft;
        tfx *= scale; tfy *= scale; tfz *= scale;
        dtx = (tfx + gt * vtx) / (-kt);
        dty = (tfy + gt * vty) / (-kt);
        dtz = (tfz + gt * vtz) / (-kt);
      }
    } else {
      tfx = 0.0; tfy = 0.0; tfz = 0.0;
    }
    out[0] += tfx;
    out[1] += tfy;
    out[2] += tfz;
  }
  *reinterpret_cast<float4 *>(wild) =
      make_float4(float(dtx), float(dty), float(dtz), float(delta_time));
}

template <typename VelT>
__device__ __forceinline__ void owner_kin(const DtView &v, uint32_t o, double pos[3], double vel[3],
                                          double wg[3], double &mass) {
  decode_pos(v.dom, v.own.voxel[o], v.own.sub[o], pos[0], pos[1], pos[2]);
  Vel<VelT>::load(v.own.lin_vel, o, vel);
  double wl[3];
  Vel<VelT>::load(v.own.ang_vel, o, wl);
  float4 q = v.own.quat[o];
  qrot(double(q.x), double(q.y), double(q.z), double(q.w), wl[0], wl[1], wl[2], wg[0], wg[1], wg[2]);
  mass = v.own.tpl[meta_tpl(v.own.meta[o])].x;
}

// contact geometry of ACS entry `id` (_kernels.py:442-491): depth, B-to-A
// unit vector, B-side curvature radius; A's centre and radius returned too
__device__ __forceinline__ void contact_geometry(const DtView &v, uint2 id, double ca[3], double &ra,
                                                 double &depth, double &bx, double &by, double &bz,
                                                 double &rb) {
  const uint32_t kind = id.y >> kKindShift, sb = id.y & kSlotMask;
  const double4 cA = v.sph.center[id.x];
  ca[0] = cA.x; ca[1] = cA.y; ca[2] = cA.z;
  ra = cA.w;
  if (kind == 0) {
    const double4 cB = v.sph.center[sb];
    double dx = ca[0] - cB.x, dy = ca[1] - cB.y, dz = ca[2] - cB.z;
    double d = sqrt(dx * dx + dy * dy + dz * dz);
    rb = cB.w;
    if (d < 1e-300) {
      depth = ra + rb; bx = 0.0; by = 0.0; bz = 1.0;
    } else {
      double inv = 1.0 / d;
      bx = dx * inv; by = dy * inv; bz = dz * inv;
      depth = ra + rb - d;
    }
  } else if (kind == 1) {
    const double *T = v.tri.world + 9 * size_t(sb);
    double qx, qy, qz;
    closest_on_tri(ca[0], ca[1], ca[2], T, qx, qy, qz);
    double dx = ca[0] - qx, dy = ca[1] - qy, dz = ca[2] - qz;
    double d = sqrt(dx * dx + dy * dy + dz * dz);
    if (d < 1e-300) {
      double e1x = T[3] - T[0], e1y = T[4] - T[1], e1z = T[5] - T[2];
      double e2x = T[6] - T[0], e2y = T[7] - T[1], e2z = T[8] - T[2];
      double nx = e1y * e2z - e1z * e2y, ny = e1z * e2x - e1x * e2z, nz = e1x * e2y - e1y * e2x;
      double nn = sqrt(nx * nx + ny * ny + nz * nz);
      bx = nx / nn; by = ny / nn; bz = nz / nn;
    } else {
      double inv = 1.0 / d;
      bx = dx * inv; by = dy * inv; bz = dz * inv;
    }
    depth = ra - d;
    rb = kFlatRadius;
  } else {
    double gap;
    analytic_gap(v.ana.kind[sb], v.ana.world + 8 * size_t(sb), ca[0], ca[1], ca[2], gap, bx, by, bz, rb);
    depth = ra - gap;
  }
}

namespace {
// narrow phase of the step: one thread per ACS entry, geometry only.
// Touching entries are compacted into tlist (warp-aggregated append); the
// fp64 parity build also records a touch flag per entry for its reduction.
// A false positive leaves its history untouched (forces.py:95-97).
__global__ void __launch_bounds__(256, 4) k_touch(DtView v, uint32_t *tlist, unsigned long long *tlist_n) {
  int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  bool t = false;
  unsigned kind = 0;
  if (k < v.n_acs && !v.st->err) {
    const uint2 id = v.ids[k];
    kind = id.y >> kKindShift;
    double ca[3], ra, depth, bx, by, bz, rb;
    contact_geometry(v, id, ca, ra, depth, bx, by, bz, rb);
    t = depth > 0.0;
    if (!v.own.facc) v.touch[k] = t ? 1 : 0;
  }
  const unsigned m = __ballot_sync(0xffffffffu, t);
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (m && lane == 0) base = atomicAdd(tlist_n, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (t) tlist[base + __popc(m & ((1u << lane) - 1u))] = uint32_t(k);
  // touching counts (integers: order-independent)
  unsigned touching = t ? (kind == 0 ? 2u : 1u) : 0u;
  for (int off = 16; off > 0; off >>= 1) touching += __shfl_down_sync(0xffffffffu, touching, off);
  if (lane == 0 && m) {
    atomicAdd(&v.st->touching, (unsigned long long)touching);
    atomicAdd(&v.st->touch_pairs, (unsigned long long)__popc(m));
  }
}

}  // namespace

// force phase: touching entries only.  Pair kinematics (forces.py:55-79), the
// Hertz-Mindlin core, history update, then either the per-contact output of
// the parity build (F, F + torque-only force, contact point) or the
// fixed-point owner accumulation of the throughput build.
template <typename VelT>
__global__ void __launch_bounds__(128) k_forces(DtView v, double ts, const uint32_t *tlist,
                                                const unsigned long long *tlist_n) {
  const unsigned long long nt = *tlist_n;
  if (v.st->err) return;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < nt;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t k = tlist[i];
    const uint2 id = v.ids[k];
    const uint32_t kind = id.y >> kKindShift, sb = id.y & kSlotMask;
    double ca[3], ra, depth, bx, by, bz, rb;
    contact_geometry(v, id, ca, ra, depth, bx, by, bz, rb);
    const uint32_t oa = v.sph.owner[id.x];
    uint32_t ob;
    int mb;
    if (kind == 0) { ob = v.sph.owner[sb]; mb = v.sph.mat[sb]; }
    else if (kind == 1) { ob = v.tri.owner[sb]; mb = v.tri.mat[sb]; }
    else { ob = v.ana.owner[sb]; mb = v.ana.mat[sb]; }
    double half = ra - 0.5 * depth;
    double px = ca[0] - bx * half, py = ca[1] - by * half, pz = ca[2] - bz * half;
    double pa[3], va[3], wa[3], ma, pb[3], vb[3], wb[3], mbass;
    owner_kin<VelT>(v, oa, pa, va, wa, ma);
    owner_kin<VelT>(v, ob, pb, vb, wb, mbass);
    double rax = px - pa[0], ray = py - pa[1], raz = pz - pa[2];
    double rbx = px - pb[0], rby = py - pb[1], rbz = pz - pb[2];
    double rotax = wa[1] * raz - wa[2] * ray;
    double rotay = wa[2] * rax - wa[0] * raz;
    double rotaz = wa[0] * ray - wa[1] * rax;
    double rotbx = wb[1] * rbz - wb[2] * rby;
    double rotby = wb[2] * rbx - wb[0] * rbz;
    double rotbz = wb[0] * rby - wb[1] * rbx;
    double vx = (va[0] + rotax) - (vb[0] + rotbx);
    double vy = (va[1] + rotay) - (vb[1] + rotby);
    double vz = (va[2] + rotaz) - (vb[2] + rotbz);
    double mass_eff = (ma * mbass) / (ma + mbass);
    double out[6];
    hertz_mindlin(depth, ts, bx, by, bz, vx, vy, vz, rotbx - rotax, rotby - rotay, rotbz - rotaz,
                  mass_eff, ra, rb, v.sph.mat[id.x], mb, v.mat, v.wild + size_t(v.W) * k, out);
    const double tx = out[0] + out[3], ty = out[1] + out[4], tz = out[2] + out[5];
    if (v.own.facc) {
      // throughput build: +F / r_a x T on A, -F / -(r_b x T) on B, as int64
      // fixed point (order-independent sums: bitwise reproducible runs)
      const double2 sa = v.own.tpl_scale[meta_tpl(v.own.meta[oa])];
      const double2 sbs = v.own.tpl_scale[meta_tpl(v.own.meta[ob])];
      unsigned long long *fa = reinterpret_cast<unsigned long long *>(v.own.facc + 6 * size_t(oa));
      unsigned long long *fb = reinterpret_cast<unsigned long long *>(v.own.facc + 6 * size_t(ob));
      const double ta[3] = {ray * tz - raz * ty, raz * tx - rax * tz, rax * ty - ray * tx};
      const double tb[3] = {rby * tz - rbz * ty, rbz * tx - rbx * tz, rbx * ty - rby * tx};
      for (int q = 0; q < 3; ++q) {
        if (sa.x > 0.0) {
          atomicAdd(fa + q, (unsigned long long)__double2ll_rn(out[q] * sa.x));
          atomicAdd(fa + 3 + q, (unsigned long long)__double2ll_rn(ta[q] * sa.y));
        } else {
          atomicAdd(reinterpret_cast<double *>(fa + q), out[q]);
          atomicAdd(reinterpret_cast<double *>(fa + 3 + q), ta[q]);
        }
        if (sbs.x > 0.0) {
          atomicAdd(fb + q, (unsigned long long)__double2ll_rn(-out[q] * sbs.x));
          atomicAdd(fb + 3 + q, (unsigned long long)__double2ll_rn(-tb[q] * sbs.y));
        } else {
          atomicAdd(reinterpret_cast<double *>(fb + q), -out[q]);
          atomicAdd(reinterpret_cast<double *>(fb + 3 + q), -tb[q]);
        }
      }
    } else {
      double *oc = v.out_c + 9 * size_t(k);
      oc[0] = out[0]; oc[1] = out[1]; oc[2] = out[2];
      oc[3] = tx; oc[4] = ty; oc[5] = tz;
      oc[6] = px; oc[7] = py; oc[8] = pz;
    }
  }
}

// one contact's contribution to owner position p (A side +, B side -)
__device__ __forceinline__ void contribute(const DtView &v, uint32_t k, bool side_b, const double p[3],
                                           double af[3], double at[3]) {
  if (!v.touch[k]) return;  // exact: a false positive contributes +-0.0
  const double *oc = v.out_c + 9 * size_t(k);
  double fx = oc[0], fy = oc[1], fz = oc[2];
  double tx = oc[3], ty = oc[4], tz = oc[5];
  double rx = oc[6] - p[0], ry = oc[7] - p[1], rz = oc[8] - p[2];
  if (!side_b) {
    af[0] += fx; af[1] += fy; af[2] += fz;
    at[0] += ry * tz - rz * ty;
    at[1] += rz * tx - rx * tz;
    at[2] += rx * ty - ry * tx;
  } else {
    af[0] -= fx; af[1] -= fy; af[2] -= fz;
    at[0] -= ry * tz - rz * ty;
    at[1] -= rz * tx - rx * tz;
    at[2] -= rx * ty - ry * tx;
  }
}

// A-side contact ranges of owner o: its spheres' segments for kinds 0..2
// (increasing contact index across kinds)
__device__ __forceinline__ void a_ranges(const DtView &v, uint32_t o, unsigned long long lo[3],
                                         unsigned long long hi[3]) {
  const uint32_t f0 = v.sph.first[o], f1 = v.sph.first[o + 1];
  for (int kind = 0; kind < 3; ++kind) {
    lo[kind] = f1 > f0 ? v.seg[kind * v.n_sph + f0] : 0;
    hi[kind] = f1 > f0 ? v.seg[kind * v.n_sph + f1] : 0;
  }
}

// all contributions of owner o in canonical ACS order (the reference's
// reduce_to_owners order, _kernels.py:522-545): merge of the A ranges and the
// sorted B list by contact index
__device__ __forceinline__ void accumulate(const DtView &v, uint32_t o, const double p[3], double af[3],
                                           double at[3]) {
  unsigned long long alo[3], ahi[3];
  a_ranges(v, o, alo, ahi);
  uint32_t b = v.inc_start[o];
  const uint32_t be = v.inc_start[o + 1];
  int kind = 0;
  unsigned long long a = alo[0];
  for (;;) {
    while (kind < 3 && a >= ahi[kind]) {
      ++kind;
      if (kind < 3) a = alo[kind];
    }
    const bool have_a = kind < 3;
    const bool have_b = b < be;
    if (!have_a && !have_b) break;
    uint32_t kb = have_b ? v.inc[b] : 0xFFFFFFFFu;
    if (have_a && (!have_b || a < kb)) {
      contribute(v, uint32_t(a), false, p, af, at);
      ++a;
    } else {
      contribute(v, kb, true, p, af, at);
      ++b;
    }
  }
}

namespace {
// heavy owners: fixed-order block reduction (deterministic run to run)
__global__ void __launch_bounds__(256) k_heavy(DtView v) {
  __shared__ double sh[6][256];
  if (v.st->err) return;
  const unsigned long long nh = *v.n_heavy;
  for (unsigned long long hidx = blockIdx.x; hidx < nh; hidx += gridDim.x) {
    uint32_t o = v.heavy[hidx];
    double p[3];
    decode_pos(v.dom, v.own.voxel[o], v.own.sub[o], p[0], p[1], p[2]);
    unsigned long long alo[3], ahi[3];
    a_ranges(v, o, alo, ahi);
    const unsigned long long na0 = ahi[0] - alo[0], na1 = ahi[1] - alo[1], na2 = ahi[2] - alo[2];
    const uint32_t b0 = v.inc_start[o], b1 = v.inc_start[o + 1];
    const unsigned long long ntot = na0 + na1 + na2 + (b1 - b0);
    double af[3] = {0, 0, 0}, at[3] = {0, 0, 0};
    const unsigned long long chunk = (ntot + blockDim.x - 1) / blockDim.x;
    const unsigned long long e0 = min(ntot, chunk * threadIdx.x), e1 = min(ntot, chunk * (threadIdx.x + 1));
    for (unsigned long long e = e0; e < e1; ++e) {
      if (e < na0) contribute(v, uint32_t(alo[0] + e), false, p, af, at);
      else if (e < na0 + na1) contribute(v, uint32_t(alo[1] + e - na0), false, p, af, at);
      else if (e < na0 + na1 + na2) contribute(v, uint32_t(alo[2] + e - na0 - na1), false, p, af, at);
      else contribute(v, v.inc[b0 + (e - na0 - na1 - na2)], true, p, af, at);
    }
    for (int q = 0; q < 3; ++q) { sh[q][threadIdx.x] = af[q]; sh[3 + q][threadIdx.x] = at[q]; }
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
      if (threadIdx.x < st)
        for (int q = 0; q < 6; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + st];
      __syncthreads();
    }
    if (threadIdx.x < 6) v.heavy_acc[6 * size_t(o) + threadIdx.x] = sh[threadIdx.x][0];
    __syncthreads();
  }
}
}  // namespace

template <typename VelT>
__global__ void __launch_bounds__(128) k_integrate(DtView v, double h, double gx, double gy, double gz,
                                                   double v_err, unsigned long long step, int write_acc) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= v.own.n || v.st->err) return;
  const uint32_t o = uint32_t(i);
  double p[3];
  decode_pos(v.dom, v.own.voxel[o], v.own.sub[o], p[0], p[1], p[2]);
  // --- reduction (reduce_to_owners order) ---
  double af[3] = {0, 0, 0}, at[3] = {0, 0, 0};
  if (v.own.facc) {
    longlong2 *fp = reinterpret_cast<longlong2 *>(v.own.facc + 6 * size_t(o));
    const longlong2 a0 = fp[0], a1 = fp[1], a2 = fp[2];
    const double2 sc = v.own.tpl_scale[meta_tpl(v.own.meta[o])];
    if (sc.x > 0.0) {
      af[0] = double(a0.x) / sc.x; af[1] = double(a0.y) / sc.x; af[2] = double(a1.x) / sc.x;
      at[0] = double(a1.y) / sc.y; at[1] = double(a2.x) / sc.y; at[2] = double(a2.y) / sc.y;
    } else {
      af[0] = __longlong_as_double(a0.x); af[1] = __longlong_as_double(a0.y);
      af[2] = __longlong_as_double(a1.x); at[0] = __longlong_as_double(a1.y);
      at[1] = __longlong_as_double(a2.x); at[2] = __longlong_as_double(a2.y);
    }
    const longlong2 z = make_longlong2(0, 0);
    fp[0] = z; fp[1] = z; fp[2] = z;
  } else {
    unsigned long long alo[3], ahi[3];
    a_ranges(v, o, alo, ahi);
    const unsigned long long ninc = (ahi[0] - alo[0]) + (ahi[1] - alo[1]) + (ahi[2] - alo[2]) +
                                    (v.inc_start[o + 1] - v.inc_start[o]);
    if (ninc > kHeavyThreshold) {
      const double *ha = v.heavy_acc + 6 * size_t(o);
      af[0] = ha[0]; af[1] = ha[1]; af[2] = ha[2];
      at[0] = ha[3]; at[1] = ha[4]; at[2] = ha[5];
    } else if (ninc) {
      accumulate(v, o, p, af, at);
    }
  }
  if (write_acc && v.own.acc) {
    double *a = v.own.acc + 6 * size_t(o);
    a[0] = af[0]; a[1] = af[1]; a[2] = af[2]; a[3] = at[0]; a[4] = at[1]; a[5] = at[2];
  }
  // --- integrate_step (_kernels.py:564-636) ---
  const uint32_t meta = v.own.meta[o];
  const uint32_t fam = meta_family(meta);
  const uint8_t fl = v.fam.flags[fam];
  float4 q = v.own.quat[o];
  double vel[3], w[3];
  bool moved = false;
  if (fl & kFamFixed) {
    double z[3] = {0.0, 0.0, 0.0};
    Vel<VelT>::store(v.own.lin_vel, o, z);
    Vel<VelT>::store(v.own.ang_vel, o, z);
  } else {
    moved = true;
    double qw = double(q.x), qx = double(q.y), qy = double(q.z), qz = double(q.w);
    Vel<VelT>::load(v.own.lin_vel, o, vel);
    Vel<VelT>::load(v.own.ang_vel, o, w);
    if (fl & kFamPrescribed) {
      const uint8_t lm = v.fam.lv_mask[fam], am = v.fam.av_mask[fam];
      const double *lv = v.fam.lv_val + 3 * fam, *av = v.fam.av_val + 3 * fam;
      if (lm & 1) vel[0] = lv[0];
      if (lm & 2) vel[1] = lv[1];
      if (lm & 4) vel[2] = lv[2];
      if (am) {
        double pw[3];
        qrot(qw, qx, qy, qz, w[0], w[1], w[2], pw[0], pw[1], pw[2]);
        if (am & 1) pw[0] = av[0];
        if (am & 2) pw[1] = av[1];
        if (am & 4) pw[2] = av[2];
        qrot(qw, -qx, -qy, -qz, pw[0], pw[1], pw[2], w[0], w[1], w[2]);
      }
    } else {
      const double4 tp = v.own.tpl[meta_tpl(meta)];
      const double m = tp.x;
      double ef[6] = {0, 0, 0, 0, 0, 0};
      if (v.own.ext) {
        const double *e = v.own.ext + 6 * size_t(o);
        for (int c = 0; c < 6; ++c) ef[c] = e[c];
      }
      vel[0] = vel[0] + h * ((af[0] + ef[0]) / m + gx);
      vel[1] = vel[1] + h * ((af[1] + ef[1]) / m + gy);
      vel[2] = vel[2] + h * ((af[2] + ef[2]) / m + gz);
      double tgx = at[0] + ef[3], tgy = at[1] + ef[4], tgz = at[2] + ef[5];
      double tl[3];
      qrot(qw, -qx, -qy, -qz, tgx, tgy, tgz, tl[0], tl[1], tl[2]);
      const double ix = tp.y, iy = tp.z, iz = tp.w;
      double gyx = w[1] * (iz * w[2]) - w[2] * (iy * w[1]);
      double gyy = w[2] * (ix * w[0]) - w[0] * (iz * w[2]);
      double gyz = w[0] * (iy * w[1]) - w[1] * (ix * w[0]);
      w[0] += h * (tl[0] - gyx) / ix;
      w[1] += h * (tl[1] - gyy) / iy;
      w[2] += h * (tl[2] - gyz) / iz;
    }
    p[0] += h * vel[0];
    p[1] += h * vel[1];
    p[2] += h * vel[2];
    double hw = 0.5 * h;
    double dqw = hw * (-qx * w[0] - qy * w[1] - qz * w[2]);
    double dqx = hw * (qw * w[0] + qy * w[2] - qz * w[1]);
    double dqy = hw * (qw * w[1] + qz * w[0] - qx * w[2]);
    double dqz = hw * (qw * w[2] + qx * w[1] - qy * w[0]);
    qw += dqw; qx += dqx; qy += dqy; qz += dqz;
    double inv = 1.0 / sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    q = make_float4(float(qw * inv), float(qx * inv), float(qy * inv), float(qz * inv));
    v.own.quat[o] = q;
    Vel<VelT>::store(v.own.lin_vel, o, vel);
    Vel<VelT>::store(v.own.ang_vel, o, w);
    if (vel[0] * vel[0] + vel[1] * vel[1] + vel[2] * vel[2] > v_err * v_err) {
      atomicMin(&v.st->bad, (step << 40) | o);
      v.st->err = 1;
    }
  }
  (void)moved;
  // --- re-encode every owner (fixed ones too: _kernels.py:654) ---
  uint64_t vox;
  ushort4 s;
  if (!encode_pos(v.dom, p, vox, s)) {
    atomicMin(&v.st->oob, (step << 40) | o);
    v.st->err = 1;
    return;
  }
  v.own.voxel[o] = vox;
  v.own.sub[o] = s;
  // refreshed sphere centres from the decoded position (_kernels.py:657-669)
  const uint32_t s0 = v.sph.first[o], s1 = v.sph.first[o + 1];
  if (s1 > s0) {
    double pd[3];
    decode_pos(v.dom, vox, s, pd[0], pd[1], pd[2]);
    for (uint32_t k = s0; k < s1; ++k) {
      const float4 orr = v.sph.offr[k];
      double r[3];
      qrot(double(q.x), double(q.y), double(q.z), double(q.w), double(orr.x), double(orr.y), double(orr.z),
           r[0], r[1], r[2]);
      v.sph.center[k] = make_double4(add(pd[0], r[0]), add(pd[1], r[1]), add(pd[2], r[2]), double(orr.w));
    }
  }
}

namespace {
// prescribed-motion expressions evaluated on the host, one row per step
__global__ void k_apply_dyn(int n_dyn, const int *spec, const double *vals, double *lv_val, double *av_val) {
  int t = threadIdx.x + blockIdx.x * blockDim.x;
  if (t >= n_dyn) return;
  int fam = spec[3 * t], table = spec[3 * t + 1], ax = spec[3 * t + 2];
  (table == 0 ? lv_val : av_val)[3 * fam + ax] = vals[t];
}

// sphere world centres from the owner pose (_kernels.py:91-106)
__global__ void k_centers(Domain dom, Owners own, Spheres sph) {
  int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= sph.n) return;
  double c[3];
  float r;
  uint32_t o;
  sphere_center(dom, own, sph, uint32_t(k), c, r, o);
  sph.center[k] = make_double4(c[0], c[1], c[2], double(r));
}

// triangle / analytic world transforms (_kernels.py:109-152)
__global__ void k_world(Domain dom, Owners own, Tris tri, Anas ana) {
  int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k < tri.n) {
    uint32_t o = tri.owner[k];
    float4 q = own.quat[o];
    double p[3];
    decode_pos(dom, own.voxel[o], own.sub[o], p[0], p[1], p[2]);
    for (int vtx = 0; vtx < 3; ++vtx) {
      const float *l = tri.local + 9 * size_t(k) + 3 * vtx;
      double r[3];
      qrot(double(q.x), double(q.y), double(q.z), double(q.w), double(l[0]), double(l[1]),
           double(l[2]), r[0], r[1], r[2]);
      for (int ax = 0; ax < 3; ++ax) tri.world[9 * size_t(k) + 3 * vtx + ax] = add(p[ax], r[ax]);
    }
  } else if (k < tri.n + ana.n) {
    int64_t a = k - tri.n;
    uint32_t o = ana.owner[a];
    float4 q = own.quat[o];
    double p[3];
    decode_pos(dom, own.voxel[o], own.sub[o], p[0], p[1], p[2]);
    const float *l = ana.local + 8 * size_t(a);
    double r[3], d[3];
    qrot(double(q.x), double(q.y), double(q.z), double(q.w), double(l[0]), double(l[1]), double(l[2]),
         r[0], r[1], r[2]);
    qrot(double(q.x), double(q.y), double(q.z), double(q.w), double(l[3]), double(l[4]), double(l[5]),
         d[0], d[1], d[2]);
    double *w = ana.world + 8 * size_t(a);
    for (int ax = 0; ax < 3; ++ax) { w[ax] = add(p[ax], r[ax]); w[3 + ax] = d[ax]; }
    w[6] = double(l[6]);
    w[7] = double(l[7]);
  }
}

}  // namespace

template <typename VelT>
int dt_step_impl(Ctx *c, const StepArgs &a, cudaStream_t s) {
  DtView v;
  v.dom = c->dom;
  v.own = owners_view(c);
  v.sph = spheres_view(c);
  v.tri = tris_view(c);
  v.ana = anas_view(c);
  v.mat = materials_view(c);
  v.fam = families_view(c);
  v.n_acs = c->acs.n;
  v.ids = c->acs.ids.as<uint2>();
  v.wild = c->acs.wild.as<float>();
  v.W = c->wild_w;
  v.out_c = c->out_c.as<double>();
  v.touch = c->touch.as<uint8_t>();
  v.inc = c->inc.as<uint32_t>();
  v.inc_start = c->inc_start.as<uint32_t>();
  v.seg = c->acs.seg.as<unsigned long long>();
  v.n_sph = c->n_sph;
  v.heavy = c->heavy.as<uint32_t>();
  v.n_heavy = c->heavy_count.as<unsigned long long>();
  v.heavy_acc = c->heavy_acc.as<double>();
  v.st = c->status.as<Status>();
  GF_CHECK(c, cudaMemsetAsync(&v.st->touching, 0, sizeof(unsigned long long), s));
  cudaEvent_t *ev = prof_events(c);
  if (ev) cudaEventRecord(ev[0], s);
  if (v.n_acs) {
    unsigned long long *tn = c->tlist_n.as<unsigned long long>();
    GF_CHECK(c, cudaMemsetAsync(tn, 0, sizeof(unsigned long long), s));
    k_touch<<<unsigned((v.n_acs + 255) / 256), 256, 0, s>>>(v, c->tlist.as<uint32_t>(), tn);
    k_forces<VelT><<<148 * 8, 128, 0, s>>>(v, a.h, c->tlist.as<uint32_t>(), tn);
  }
  if (ev) cudaEventRecord(ev[1], s);
  if (v.n_acs && !c->fixed_reduce) k_heavy<<<64, 256, 0, s>>>(v);
  if (ev) cudaEventRecord(ev[2], s);
  if (c->n_dyn) {
    k_apply_dyn<<<(c->n_dyn + 127) / 128, 128, 0, s>>>(
        c->n_dyn, c->dyn_spec.as<int>(), c->dyn_vals.as<double>() + size_t(c->n_dyn) * a.dyn_row,
        c->lv_val.as<double>(), c->av_val.as<double>());
  }
  if (c->n_owner) {
    unsigned g = unsigned((c->n_owner + 127) / 128);
    k_integrate<VelT><<<g, 128, 0, s>>>(v, a.h, a.g[0], a.g[1], a.g[2], a.v_err,
                                       (unsigned long long)a.step, a.write_acc);
  }
  if (ev) cudaEventRecord(ev[3], s);
  if ((c->n_tri || c->n_ana) && c->world_moving) {
    int64_t n = c->n_tri + c->n_ana;
    k_world<<<unsigned((n + 127) / 128), 128, 0, s>>>(c->dom, v.own, v.tri, v.ana);
  }
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

}  // namespace gf
