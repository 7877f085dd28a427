// gf_device.cuh -- device-only dT step code: owner/contact views, contact
// geometry, pair kinematics and the force loop, templated on the contact
// model ("core").  Compiled both ahead of time into libgf_b200.so and at run
// time by NVRTC for user force models (the paper's JIT-compiled models,
// PAPER.md:149-158; the reference's ForceModel plugin, forces.py:360-440), so
// it must not include host headers.
#pragma once
#include "gf_common.cuh"

namespace gf {

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in the
// stream drains.  pdl_wait() blocks until the predecessor grid has completed
// and its writes are visible; pdl_launch() (called only after pdl_wait(), so
// every earlier grid is complete too) lets the successor start its prologue.
// Both are no-ops for a normal launch.
#ifndef GF_NO_PDL_ASM
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#else
__device__ __forceinline__ void pdl_wait() {}
__device__ __forceinline__ void pdl_launch() {}
#endif

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
  int acc_all;          // throughput build: also accumulate onto passive owners (write_acc step)
  int pf;               // fused sphere-sphere kernel: list read-ahead + L2 prefetch of the force records
  int blocked;          // fused sphere-sphere kernel: one contiguous entry range per CTA
};

// An owner whose accumulated force never feeds its motion: fixed, or every
// velocity component prescribed (walls).  The throughput build accumulates
// onto it only on the step whose accumulators are reported (write_acc);
// thousands of wall contacts would otherwise serialise on its six words.
__device__ __forceinline__ bool passive_owner(const DtView &v, uint32_t o) {
  const uint32_t f = meta_family(v.own.meta[o]);
  return (v.fam.flags[f] & kFamFixed) || (v.fam.lv_mask[f] == 7 && v.fam.av_mask[f] == 7);
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

// Hertz-Mindlin core (forces.py:82-182) for a touching contact; material
// pair values passed in (beta = restitution damping, forces.py:41-44)
__device__ __forceinline__ void hertz_mindlin_core(double overlap, double ts, double b2ax, double b2ay,
                                                   double b2az, double vx, double vy, double vz,
                                                   double wrx, double wry, double wrz, double mass_eff,
                                                   double ra, double rb, double e_cnt, double g_cnt,
                                                   double mu, double crr, double beta, float *wild,
                                                   double out[6]) {
  for (int q = 0; q < 6; ++q) out[q] = 0.0;
  double projection = vx * b2ax + vy * b2ay + vz * b2az;
  double vtx = vx - projection * b2ax;
  double vty = vy - projection * b2ay;
  double vtz = vz - projection * b2az;
  double dtx = double(wild[0]) + ts * vtx;
  double dty = double(wild[1]) + ts * vty;
  double dtz = double(wild[2]) + ts * vtz;
  double disp_proj = dtx * b2ax + dty * b2ay + dtz * b2az;
  dtx -= disp_proj * b2ax;
  dty -= disp_proj * b2ay;
  dtz -= disp_proj * b2az;
  double delta_time = double(wild[3]) + ts;

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
  wild[0] = float(dtx);
  wild[1] = float(dty);
  wild[2] = float(dtz);
  wild[3] = float(delta_time);
}

// The same law in fp32 for the throughput build's sphere-sphere fast path
// (k_forces_f32): DEM-Engine evaluates its contact models in float once the
// overlap is known.  Same expression order as above.
__device__ __forceinline__ void hertz_mindlin_core_f32(float overlap, float ts, float b2ax, float b2ay,
                                                       float b2az, float vx, float vy, float vz, float wrx,
                                                       float wry, float wrz, float mass_eff, float ra, float rb,
                                                       float e_cnt, float g_cnt, float mu, float crr, float beta,
                                                       const float4 w4, float4 &w_new, float out[6]) {
  for (int q = 0; q < 6; ++q) out[q] = 0.f;
  float projection = vx * b2ax + vy * b2ay + vz * b2az;
  float vtx = vx - projection * b2ax;
  float vty = vy - projection * b2ay;
  float vtz = vz - projection * b2az;
  float dtx = w4.x + ts * vtx;
  float dty = w4.y + ts * vty;
  float dtz = w4.z + ts * vtz;
  float disp_proj = dtx * b2ax + dty * b2ay + dtz * b2az;
  dtx -= disp_proj * b2ax;
  dty -= disp_proj * b2ay;
  dtz -= disp_proj * b2az;
  float delta_time = w4.w + ts;

  const float rr = (ra * rb) / (ra + rb);
  float sqrt_rd = sqrtf(overlap * rr);
  float sn = 2.f * e_cnt * sqrt_rd;
  float k_n = (2.f / 3.f) * sn;
  float gamma_n = 2.f * 0.91287092917527685f * beta * sqrtf(sn * mass_eff);
  float fn = k_n * overlap + gamma_n * projection;
  out[0] = fn * b2ax;
  out[1] = fn * b2ay;
  out[2] = fn * b2az;
  const float fmag = fabsf(fn);
  if (crr > 0.f) {
    bool add_rolling = true;
    float r_eff = sqrtf(rr);
    float kn_simple = (4.f / 3.f) * e_cnt * sqrtf(r_eff);
    float gn_simple = -2.f * sqrtf((5.f / 3.f) * mass_eff * e_cnt) * beta * sqrtf(sqrtf(r_eff));
    float d_coeff = gn_simple / (2.f * sqrtf(kn_simple * mass_eff));
    if (d_coeff < 1.f) {
      float t_collision = float(kPi) * sqrtf(mass_eff / (kn_simple * (1.f - d_coeff * d_coeff)));
      if (delta_time <= t_collision) add_rolling = false;
    }
    if (add_rolling) {
      float v_rot_mag = sqrtf(wrx * wrx + wry * wry + wrz * wrz);
      if (v_rot_mag > 1e-12f) {
        float scale = crr * fmag / v_rot_mag;
        out[3] = wrx * scale;
        out[4] = wry * scale;
        out[5] = wrz * scale;
      }
    }
  }
  if (mu > 0.f) {
    float kt = 8.f * g_cnt * sqrt_rd;
    float gt = -2.f * 0.91287092917527685f * beta * sqrtf(mass_eff * kt);
    float tfx = -kt * dtx - gt * vtx;
    float tfy = -kt * dty - gt * vty;
    float tfz = -kt * dtz - gt * vtz;
    float ft = sqrtf(tfx * tfx + tfy * tfy + tfz * tfz);
    if (ft > 1e-12f) {
      float ft_max = fmag * mu;
      if (ft > ft_max) {
        float scale = ft_max / ft;
        tfx *= scale; tfy *= scale; tfz *= scale;
        const float ik = -1.f / kt;
        dtx = (tfx + gt * vtx) * ik;
        dty = (tfy + gt * vty) * ik;
        dtz = (tfz + gt * vtz) * ik;
      }
    } else {
      tfx = 0.f; tfy = 0.f; tfz = 0.f;
    }
    out[0] += tfx;
    out[1] += tfy;
    out[2] += tfz;
  }
  w_new = make_float4(dtx, dty, dtz, delta_time);
}

// built-in model: pair values and beta from the uploaded tables
__device__ __forceinline__ void hertz_mindlin(double overlap, double ts, double b2ax, double b2ay,
                                              double b2az, double vx, double vy, double vz,
                                              double wrx, double wry, double wrz, double mass_eff,
                                              double ra, double rb, int ma, int mb,
                                              const Materials &M, float *wild, double out[6]) {
  const int mm = M.n_mat * M.n_mat, ab = ma * M.n_mat + mb;
  hertz_mindlin_core(overlap, ts, b2ax, b2ay, b2az, vx, vy, vz, wrx, wry, wrz, mass_eff, ra, rb,
                     M.pair[ab], M.pair[mm + ab], M.pair[3 * mm + ab], M.pair[4 * mm + ab], M.beta[ab],
                     wild, out);
}

// For user models (NVRTC): the default Hertz-Mindlin law with the reference
// core's argument list, beta computed on the device from the CoR row.  Acts
// only for overlap > 0 and leaves history untouched otherwise (forces.py:95-97).
__device__ __forceinline__ void hm_default_core(double overlap, double ts, double sim_time, double b2ax,
                                                double b2ay, double b2az, double vx, double vy, double vz,
                                                double wrx, double wry, double wrz, double mass_eff,
                                                double ra, double rb, int mat_a, int mat_b,
                                                const double *pair, int n_mat, float *wild, double *out) {
  (void)sim_time;
  if (overlap <= 0.0) return;
  const int mm = n_mat * n_mat, ab = mat_a * n_mat + mat_b;
  const double cor = pair[2 * mm + ab];
  const double loge = cor < 1e-12 ? log(1e-12) : log(cor);
  const double beta = loge / sqrt(loge * loge + kPi * kPi);
  hertz_mindlin_core(overlap, ts, b2ax, b2ay, b2az, vx, vy, vz, wrx, wry, wrz, mass_eff, ra, rb, pair[ab],
                     pair[mm + ab], pair[3 * mm + ab], pair[4 * mm + ab], beta, wild, out);
}


// The core contract of the reference (forces.py:82-87): per contact,
// overlap (may be <= 0 for a margin false positive), step size, time, B-to-A
// normal, relative velocity at the contact point, rolling direction,
// effective mass, radii (B = 1e18 for flat, negative for concave), material
// ids, the material pair stack (rows E_cnt, G_cnt, then the model's pair
// properties; pair(row, a, b) = pair[(row * n_mat + a) * n_mat + b]), the
// contact's wildcard (history) row and out[6] = force on A, torque-only
// force.  out arrives zeroed.
struct CoreArgs {
  double overlap, ts, sim_time;
  double b2ax, b2ay, b2az, vx, vy, vz, wrx, wry, wrz;
  double mass_eff, ra, rb;
  int mat_a, mat_b;
  const double *pair;
  int n_mat;
  float *wild;
  const Materials *M;
};

// built-in model: history-based Hertz-Mindlin (skips false positives)
struct HmCore {
  static constexpr bool kAllEntries = false;
  __device__ static __forceinline__ void eval(const CoreArgs &a, double out[6]) {
    if (a.overlap <= 0.0) return;
    hertz_mindlin(a.overlap, a.ts, a.b2ax, a.b2ay, a.b2az, a.vx, a.vy, a.vz, a.wrx, a.wry, a.wrz, a.mass_eff,
                  a.ra, a.rb, a.mat_a, a.mat_b, *a.M, a.wild, out);
  }
};

// Block-level accumulator for the B side of wall / mesh contacts (kinds 1, 2).
// A few owners (the floor, a wheel) take every wall contact of the scene; one
// global atomic per contact and word serialises on those six addresses (13.9
// ms for the 150M bed's floor on a write_acc step, against 0.2 ms when the
// passive side is skipped).  Rows are summed in shared memory -- int64 fixed
// point (exact, order-free) or fp64 for scale-0 owners -- and flushed once per
// block.  A full table falls back to the global atomics.
constexpr int kBcSlots = 8;
constexpr uint32_t kBcEmpty = 0xFFFFFFFFu;
struct BCache {
  unsigned long long w[kBcSlots][6];
  uint32_t own[kBcSlots];
};

__device__ __forceinline__ void bcache_init(BCache &bc) {
  for (int t = threadIdx.x; t < kBcSlots * 6; t += blockDim.x) bc.w[t / 6][t % 6] = 0ull;
  for (int t = threadIdx.x; t < kBcSlots; t += blockDim.x) bc.own[t] = kBcEmpty;
}

// slot of owner o (claimed if new), -1 when the table is full
__device__ __forceinline__ int bcache_slot(BCache &bc, uint32_t o) {
  for (int s = 0; s < kBcSlots; ++s) {
    uint32_t cur = *reinterpret_cast<volatile uint32_t *>(&bc.own[s]);
    if (cur == kBcEmpty) cur = atomicCAS(&bc.own[s], kBcEmpty, o);
    if (cur == kBcEmpty || cur == o) return s;
  }
  return -1;
}

// after a __syncthreads(): add the block's rows to the owner accumulators
__device__ __forceinline__ void bcache_flush(const DtView &v, BCache &bc) {
  for (int t = threadIdx.x; t < kBcSlots * 6; t += blockDim.x) {
    const int s = t / 6, q = t % 6;
    const uint32_t o = bc.own[s];
    if (o == kBcEmpty) continue;
    unsigned long long *f = reinterpret_cast<unsigned long long *>(v.own.facc + 6 * size_t(o)) + q;
    if (v.own.tpl_scale[meta_tpl(v.own.meta[o])].x > 0.0) atomicAdd(f, bc.w[s][q]);
    else atomicAdd(reinterpret_cast<double *>(f), __longlong_as_double((long long)bc.w[s][q]));
  }
}

// Force of one ACS entry with core `Core`; returns false when it produced no
// force (nothing to reduce).  Parity build: writes the per-contact output and
// touch flag; throughput build: fixed-point owner accumulation (wall / mesh B
// sides through the block's BCache when `bc` is given).
template <typename VelT, typename Core>
__device__ __forceinline__ void force_entry(const DtView &v, uint32_t k, double ts, double sim_time,
                                            BCache *bc = nullptr) {
  const uint2 id = v.ids[k];
  const uint32_t kind = id.y >> kKindShift, sb = id.y & kSlotMask;
  double ca[3], ra, depth, bx, by, bz, rb;
  contact_geometry(v, id, ca, ra, depth, bx, by, bz, rb);
  if (!Core::kAllEntries && depth <= 0.0) return;
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
  CoreArgs arg;
  arg.overlap = depth; arg.ts = ts; arg.sim_time = sim_time;
  arg.b2ax = bx; arg.b2ay = by; arg.b2az = bz;
  arg.vx = (va[0] + rotax) - (vb[0] + rotbx);
  arg.vy = (va[1] + rotay) - (vb[1] + rotby);
  arg.vz = (va[2] + rotaz) - (vb[2] + rotbz);
  arg.wrx = rotbx - rotax; arg.wry = rotby - rotay; arg.wrz = rotbz - rotaz;
  arg.mass_eff = (ma * mbass) / (ma + mbass);
  arg.ra = ra; arg.rb = rb;
  arg.mat_a = v.sph.mat[id.x]; arg.mat_b = mb;
  arg.pair = v.mat.pair; arg.n_mat = v.mat.n_mat;
  arg.wild = v.wild + size_t(v.W) * k;
  arg.M = &v.mat;
  double out[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  Core::eval(arg, out);
  if (Core::kAllEntries && out[0] == 0.0 && out[1] == 0.0 && out[2] == 0.0 && out[3] == 0.0 &&
      out[4] == 0.0 && out[5] == 0.0) {
    if (!v.own.facc) v.touch[k] = 0;
    return;
  }
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
    const bool skip_a = !v.acc_all && passive_owner(v, oa);
    bool skip_b = !v.acc_all && passive_owner(v, ob);
    if (bc != nullptr && kind != 0 && !skip_b) {
      const int s = bcache_slot(*bc, ob);
      if (s >= 0) {
        skip_b = true;
        for (int q = 0; q < 3; ++q) {
          if (sbs.x > 0.0) {
            atomicAdd(&bc->w[s][q], (unsigned long long)__double2ll_rn(-out[q] * sbs.x));
            atomicAdd(&bc->w[s][3 + q], (unsigned long long)__double2ll_rn(-tb[q] * sbs.y));
          } else {
            atomicAdd(reinterpret_cast<double *>(&bc->w[s][q]), -out[q]);
            atomicAdd(reinterpret_cast<double *>(&bc->w[s][3 + q]), -tb[q]);
          }
        }
      }
    }
    for (int q = 0; q < 3; ++q) {
      if (skip_a) {
      } else if (sa.x > 0.0) {
        atomicAdd(fa + q, (unsigned long long)__double2ll_rn(out[q] * sa.x));
        atomicAdd(fa + 3 + q, (unsigned long long)__double2ll_rn(ta[q] * sa.y));
      } else {
        atomicAdd(reinterpret_cast<double *>(fa + q), out[q]);
        atomicAdd(reinterpret_cast<double *>(fa + 3 + q), ta[q]);
      }
      if (skip_b) {
      } else if (sbs.x > 0.0) {
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
    v.touch[k] = 1;
  }
}

// Issue the staged fixed-point rows red[6 * i + q] of owners own[i], i < n / 6:
// consecutive lanes take consecutive words, so each RED instruction touches
// the rows of ~5 owners (contiguous 48 B each).  Warp-collective; leaves the
// buffers free for reuse.
__device__ __forceinline__ void red_rows(const DtView &v, const long long *red, const uint32_t *own, int n,
                                         int lane) {
  for (int j = lane; j < n; j += 32) {
    const int i = j / 6, q = j - 6 * i;
    atomicAdd(reinterpret_cast<unsigned long long *>(v.own.facc) + 6 * size_t(own[i]) + q,
              (unsigned long long)red[j]);
  }
  __syncwarp();
}

// A-side contributions of a warp's contacts (entries in A-sorted contact
// order, so equal A owners sit in consecutive lanes): each run's int64
// fixed-point words are summed in registers (exact) and added by the run's
// head lane; boundary owners (scale 0) take fp64 atomics.  Every lane of the
// warp must call it; `out` = force (3), `ta` = torque on A (3).
__device__ __forceinline__ void a_side_sums(const DtView &v, bool use_a, uint32_t oa, double sa_f, double sa_t,
                                            const float *out, const float *ta, int lane,
                                            long long *red = nullptr, uint32_t *own = nullptr) {
  const bool fixed_a = use_a && sa_f > 0.0;
  if (use_a && !fixed_a) {   // boundary owner: fp64 atomics, not aggregated
    unsigned long long *fa = reinterpret_cast<unsigned long long *>(v.own.facc + 6 * size_t(oa));
    for (int q = 0; q < 3; ++q) {
      atomicAdd(reinterpret_cast<double *>(fa + q), double(out[q]));
      atomicAdd(reinterpret_cast<double *>(fa + 3 + q), double(ta[q]));
    }
  }
  const uint32_t key = fixed_a ? oa : 0xFFFFFFFFu;
  const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
  const bool head = lane == 0 || prev != key;
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  const unsigned later = heads & ~((2u << lane) - 1u);   // heads after this lane
  const int run_end = later ? __ffs(later) - 2 : 31;
  // segmented sums over the runs: only as many doubling steps as the longest
  // run needs (runs are short -- an owner's touching partners of higher slot)
  const unsigned runlen = (head && fixed_a) ? unsigned(run_end - lane + 1) : 0u;
  const unsigned maxrun = __reduce_max_sync(0xffffffffu, runlen);
  long long acc[6];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    acc[q] = fixed_a ? __double2ll_rn(double(out[q]) * sa_f) : 0ll;
    acc[3 + q] = fixed_a ? __double2ll_rn(double(ta[q]) * sa_t) : 0ll;
  }
  for (unsigned off = 1; off < maxrun; off <<= 1) {
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const long long o = __shfl_down_sync(0xffffffffu, acc[q], off);
      if (lane + int(off) <= run_end) acc[q] += o;
    }
  }
  if (red == nullptr) {
    if (head && fixed_a) {
      unsigned long long *fa = reinterpret_cast<unsigned long long *>(v.own.facc + 6 * size_t(oa));
#pragma unroll
      for (int q = 0; q < 6; ++q) atomicAdd(fa + q, (unsigned long long)acc[q]);
    }
    return;
  }
  // staged: the run heads' six words go through the warp's shared buffer so
  // that one RED instruction covers ~5 owners' contiguous 48-byte rows (two
  // sectors each) instead of one word of 32 scattered owners
  const unsigned hf = __ballot_sync(0xffffffffu, head && fixed_a);
  if (head && fixed_a) {
    const int h = __popc(hf & ((1u << lane) - 1u));
    own[h] = oa;
#pragma unroll
    for (int q = 0; q < 6; ++q) red[6 * h + q] = acc[q];
  }
  __syncwarp();
  red_rows(v, red, own, 6 * __popc(hf), lane);
}


// Fused sphere-sphere loop of the throughput build for a user model `Core`
// (NVRTC-compiled, gf_nvrtc.cu): every entry of the sphere-sphere block --
// a user core may act at any overlap -- in warps of 32 consecutive entries.
// Geometry in fp64 from the centre records (depth = ra + rb - d, exactly as
// contact_geometry), kinematics from the fp32 records (one load round), the
// core in fp64 with the reference's argument list, history in place, B side
// one atomic per word, A side summed over runs of equal owners.
template <typename Core>
__device__ __forceinline__ void user_ss_loop(const DtView &v, double ts, double sim_time) {
  if (v.st->err) return;
  const unsigned long long n_ss = v.seg[v.n_sph];
  const int lane = threadIdx.x & 31;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long touched = 0;
  for (unsigned long long base = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) & ~31ull; base < n_ss;
       base += stride) {
    const unsigned long long k = base + lane;
    float out[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float ta[3] = {0.f, 0.f, 0.f};
    uint32_t oa = 0xFFFFFFFFu;
    double sa_f = 0.0, sa_t = 0.0;
    bool use_a = false;
    if (k < n_ss) {
      const uint2 id = v.ids[k];
      const uint32_t a = id.x, b = id.y & kSlotMask;
      const double4 cA = v.sph.center[a], cB = v.sph.center[b];
      const SphKin ka = v.sph.kin[a], kb = v.sph.kin[b];
      const double dx = cA.x - cB.x, dy = cA.y - cB.y, dz = cA.z - cB.z;
      const double d = sqrt(dx * dx + dy * dy + dz * dz);
      double depth, bx, by, bz;
      if (d < 1e-300) {
        depth = cA.w + cB.w; bx = 0.0; by = 0.0; bz = 1.0;
      } else {
        const double inv = 1.0 / d;
        bx = dx * inv; by = dy * inv; bz = dz * inv;
        depth = cA.w + cB.w - d;
      }
      if (depth > 0.0) ++touched;
      // contact point p = cA - b (ra - depth / 2); lever arms p - pos_a, p - pos_b
      const double half = cA.w - 0.5 * depth;
      const double rax = ka.r.x - bx * half, ray = ka.r.y - by * half, raz = ka.r.z - bz * half;
      const double rbx = kb.r.x + dx - bx * half, rby = kb.r.y + dy - by * half, rbz = kb.r.z + dz - bz * half;
      const double rotax = ka.w.y * raz - ka.w.z * ray, rotay = ka.w.z * rax - ka.w.x * raz,
                   rotaz = ka.w.x * ray - ka.w.y * rax;
      const double rotbx = kb.w.y * rbz - kb.w.z * rby, rotby = kb.w.z * rbx - kb.w.x * rbz,
                   rotbz = kb.w.x * rby - kb.w.y * rbx;
      CoreArgs arg;
      arg.overlap = depth; arg.ts = ts; arg.sim_time = sim_time;
      arg.b2ax = bx; arg.b2ay = by; arg.b2az = bz;
      arg.vx = (ka.v.x + rotax) - (kb.v.x + rotbx);
      arg.vy = (ka.v.y + rotay) - (kb.v.y + rotby);
      arg.vz = (ka.v.z + rotaz) - (kb.v.z + rotbz);
      arg.wrx = rotbx - rotax; arg.wry = rotby - rotay; arg.wrz = rotbz - rotaz;
      const double ma = ka.v.w, mb = kb.v.w;
      arg.mass_eff = (ma * mb) / (ma + mb);
      arg.ra = cA.w; arg.rb = cB.w;
      arg.mat_a = int(kin_mat(ka)); arg.mat_b = int(kin_mat(kb));
      arg.pair = v.mat.pair; arg.n_mat = v.mat.n_mat;
      arg.wild = v.wild + size_t(v.W) * k;
      arg.M = &v.mat;
      double o6[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      Core::eval(arg, o6);
      if (o6[0] != 0.0 || o6[1] != 0.0 || o6[2] != 0.0 || o6[3] != 0.0 || o6[4] != 0.0 || o6[5] != 0.0) {
        for (int q = 0; q < 6; ++q) out[q] = float(o6[q]);
        const double tx = o6[0] + o6[3], ty = o6[1] + o6[4], tz = o6[2] + o6[5];
        ta[0] = float(ray * tz - raz * ty); ta[1] = float(raz * tx - rax * tz); ta[2] = float(rax * ty - ray * tx);
        const double tb[3] = {rby * tz - rbz * ty, rbz * tx - rbx * tz, rbx * ty - rby * tx};
        if (v.acc_all || !(kin_flags(kb) & kKinPassive)) {
          const double sbf = kin_fscale(kb), sbt = kin_tscale(kb);
          unsigned long long *fb = reinterpret_cast<unsigned long long *>(v.own.facc + 6 * size_t(kin_owner(kb)));
          for (int q = 0; q < 3; ++q) {
            if (sbf > 0.0) {
              atomicAdd(fb + q, (unsigned long long)__double2ll_rn(-o6[q] * sbf));
              atomicAdd(fb + 3 + q, (unsigned long long)__double2ll_rn(-tb[q] * sbt));
            } else {
              atomicAdd(reinterpret_cast<double *>(fb + q), -o6[q]);
              atomicAdd(reinterpret_cast<double *>(fb + 3 + q), -tb[q]);
            }
          }
        }
        oa = kin_owner(ka);
        use_a = v.acc_all || !(kin_flags(ka) & kKinPassive);
        sa_f = kin_fscale(ka);
        sa_t = kin_tscale(ka);
      }
    }
    a_side_sums(v, use_a, oa, sa_f, sa_t, out, ta, lane);
  }
  for (int off = 16; off > 0; off >>= 1) touched += __shfl_down_sync(0xffffffffu, touched, off);
  if (lane == 0 && touched) {
    atomicAdd(&v.st->touching, 2ull * touched);
    atomicAdd(&v.st->touch_pairs, touched);
  }
}

// a user model's wall kinds: every entry from the start of the (kind 1,
// sphere 0) segment, generic path
template <typename VelT, typename Core>
__device__ __forceinline__ void user_walls_loop(const DtView &v, double ts, double sim_time) {
  __shared__ BCache bc;
  __shared__ int s_err;
  bcache_init(bc);
  if (threadIdx.x == 0) s_err = v.st->err;
  __syncthreads();
  if (s_err) return;
  BCache *bcp = v.own.facc ? &bc : nullptr;
  const unsigned long long n = (unsigned long long)v.n_acs, k0 = v.seg[v.n_sph];
  for (unsigned long long i = k0 + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    force_entry<VelT, Core>(v, uint32_t(i), ts, sim_time, bcp);
  if (bcp == nullptr) return;
  __syncthreads();
  bcache_flush(v, bc);
}

// The force loop: entries listed in `list` (touching entries of the built-in
// model) or, for cores that act on every entry (user models may act at
// negative overlap), all entries.
template <typename VelT, typename Core>
__device__ __forceinline__ void forces_loop(const DtView &v, double ts, double sim_time, const uint32_t *list,
                                            const unsigned long long *list_n) {
  __shared__ BCache bc;
  __shared__ int s_err;
  bcache_init(bc);
  if (threadIdx.x == 0) s_err = v.st->err;
  __syncthreads();
  if (s_err) return;
  BCache *bcp = v.own.facc ? &bc : nullptr;
  const unsigned long long n = Core::kAllEntries ? (unsigned long long)v.n_acs : *list_n;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    force_entry<VelT, Core>(v, Core::kAllEntries ? uint32_t(i) : list[i], ts, sim_time, bcp);
  if (bcp == nullptr) return;
  __syncthreads();
  bcache_flush(v, bc);
}

// ---------------------------------------------------------------------------
// Reference-shaped entry points (include/gf_b200.h gf_contact_forces /
// gf_eval_core): the reference's own array layouts, one thread per contact,
// the model core `Core` (built-in Hertz-Mindlin or an NVRTC user model).
// ---------------------------------------------------------------------------
struct RefContacts {
  int64_t n;
  const uint8_t *kind;
  const int64_t *slot_a, *slot_b, *owner_a, *owner_b;
  const uint8_t *mat_a, *mat_b;
  const double *sph_centers;   // (m, 3)
  const float *sph_radii;      // (m,)
  const double *tri_world;     // (n_t, 9)
  const double *ana_world;     // (n_a, 8)
  const uint8_t *ana_kind;
  const double *owner_pos, *lin_vel, *ang_vel_global, *mass;   // (n_o, 3) / (n_o,)
  Materials mat;
  float *wild;                 // (n, W)
  int W;
  double ts, sim_time;
  double *out_ft, *depth, *cp; // (n, 6), (n,), (n, 3)
  unsigned long long *touching;
};

// contact_geom_one (_kernels.py:441-486) on the reference arrays
__device__ __forceinline__ void ref_geom_one(const RefContacts &r, int kd, int64_t i, int64_t j, double &depth,
                                             double &bx, double &by, double &bz, double &px, double &py,
                                             double &pz, double &rb) {
  const double cx = r.sph_centers[3 * i], cy = r.sph_centers[3 * i + 1], cz = r.sph_centers[3 * i + 2];
  const double ra = double(r.sph_radii[i]);
  if (kd == 0) {
    const double dx = cx - r.sph_centers[3 * j], dy = cy - r.sph_centers[3 * j + 1],
                 dz = cz - r.sph_centers[3 * j + 2];
    const double d = sqrt(dx * dx + dy * dy + dz * dz);
    rb = double(r.sph_radii[j]);
    if (d < 1e-300) {
      depth = ra + rb; bx = 0.0; by = 0.0; bz = 1.0;
      px = cx; py = cy; pz = cz;
      return;
    }
    const double inv = 1.0 / d;
    bx = dx * inv; by = dy * inv; bz = dz * inv;
    depth = ra + rb - d;
  } else if (kd == 1) {
    const double *T = r.tri_world + 9 * j;
    double qx, qy, qz;
    closest_on_tri(cx, cy, cz, T, qx, qy, qz);
    const double dx = cx - qx, dy = cy - qy, dz = cz - qz;
    const double d = sqrt(dx * dx + dy * dy + dz * dz);
    if (d < 1e-300) {
      const double e1x = T[3] - T[0], e1y = T[4] - T[1], e1z = T[5] - T[2];
      const double e2x = T[6] - T[0], e2y = T[7] - T[1], e2z = T[8] - T[2];
      bx = e1y * e2z - e1z * e2y; by = e1z * e2x - e1x * e2z; bz = e1x * e2y - e1y * e2x;
      const double nn = sqrt(bx * bx + by * by + bz * bz);
      bx /= nn; by /= nn; bz /= nn;
    } else {
      const double inv = 1.0 / d;
      bx = dx * inv; by = dy * inv; bz = dz * inv;
    }
    depth = ra - d;
    rb = kFlatRadius;
  } else {
    double gap;
    analytic_gap(r.ana_kind[j], r.ana_world + 8 * j, cx, cy, cz, gap, bx, by, bz, rb);
    depth = ra - gap;
  }
  const double half = ra - 0.5 * depth;
  px = cx - bx * half; py = cy - by * half; pz = cz - bz * half;
}

// one entry of make_contact_kernel's sweep (forces.py:553-591)
template <typename Core>
__device__ __forceinline__ void ref_contact_entry(const RefContacts &r, int64_t k) {
  const int kd = r.kind[k];
  const int64_t sa = r.slot_a[k];
  double dep, bx, by, bz, px, py, pz, rb;
  ref_geom_one(r, kd, sa, r.slot_b[k], dep, bx, by, bz, px, py, pz, rb);
  r.depth[k] = dep;
  r.cp[3 * k] = px; r.cp[3 * k + 1] = py; r.cp[3 * k + 2] = pz;
  const int64_t oa = r.owner_a[k], ob = r.owner_b[k];
  const double *pa = r.owner_pos + 3 * oa, *pb = r.owner_pos + 3 * ob;
  const double *va = r.lin_vel + 3 * oa, *vb = r.lin_vel + 3 * ob;
  const double *wa = r.ang_vel_global + 3 * oa, *wb = r.ang_vel_global + 3 * ob;
  const double rax = px - pa[0], ray = py - pa[1], raz = pz - pa[2];
  const double rbx = px - pb[0], rby = py - pb[1], rbz = pz - pb[2];
  const double rotax = wa[1] * raz - wa[2] * ray, rotay = wa[2] * rax - wa[0] * raz,
               rotaz = wa[0] * ray - wa[1] * rax;
  const double rotbx = wb[1] * rbz - wb[2] * rby, rotby = wb[2] * rbx - wb[0] * rbz,
               rotbz = wb[0] * rby - wb[1] * rbx;
  CoreArgs arg;
  arg.overlap = dep; arg.ts = r.ts; arg.sim_time = r.sim_time;
  arg.b2ax = bx; arg.b2ay = by; arg.b2az = bz;
  arg.vx = (va[0] + rotax) - (vb[0] + rotbx);
  arg.vy = (va[1] + rotay) - (vb[1] + rotby);
  arg.vz = (va[2] + rotaz) - (vb[2] + rotbz);
  arg.wrx = rotbx - rotax; arg.wry = rotby - rotay; arg.wrz = rotbz - rotaz;
  const double ma = r.mass[oa], mb = r.mass[ob];
  arg.mass_eff = (ma * mb) / (ma + mb);
  arg.ra = double(r.sph_radii[sa]); arg.rb = rb;
  arg.mat_a = r.mat_a[k]; arg.mat_b = r.mat_b[k];
  arg.pair = r.mat.pair; arg.n_mat = r.mat.n_mat;
  arg.wild = r.wild + size_t(r.W) * k;
  arg.M = &r.mat;
  double out[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  Core::eval(arg, out);
  for (int q = 0; q < 6; ++q) r.out_ft[6 * k + q] = out[q];
  if (dep > 0.0) atomicAdd(r.touching, kd == 0 ? 2ull : 1ull);
}

template <typename Core>
__device__ __forceinline__ void ref_contacts_loop(const RefContacts &r) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < r.n; k += int64_t(gridDim.x) * blockDim.x)
    ref_contact_entry<Core>(r, k);
}

// Batched model core (the reference core's scalar signature, forces.py:82-87):
// args row = overlap, ts, sim_time, b2a xyz, v xyz, wr xyz, mass_eff, ra, rb
struct CoreBatch {
  int64_t n;
  const double *args;    // (n, 15)
  const int *mats;       // (n, 2) int32
  Materials mat;
  float *wild;           // (n, W)
  int W;
  double *out;           // (n, 6)
};

template <typename Core>
__device__ __forceinline__ void core_batch_loop(const CoreBatch &b) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < b.n; k += int64_t(gridDim.x) * blockDim.x) {
    const double *x = b.args + 15 * k;
    CoreArgs arg;
    arg.overlap = x[0]; arg.ts = x[1]; arg.sim_time = x[2];
    arg.b2ax = x[3]; arg.b2ay = x[4]; arg.b2az = x[5];
    arg.vx = x[6]; arg.vy = x[7]; arg.vz = x[8];
    arg.wrx = x[9]; arg.wry = x[10]; arg.wrz = x[11];
    arg.mass_eff = x[12]; arg.ra = x[13]; arg.rb = x[14];
    arg.mat_a = b.mats[2 * k]; arg.mat_b = b.mats[2 * k + 1];
    arg.pair = b.mat.pair; arg.n_mat = b.mat.n_mat;
    arg.wild = b.wild + size_t(b.W) * k;
    arg.M = &b.mat;
    double out[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    Core::eval(arg, out);
    for (int q = 0; q < 6; ++q) b.out[6 * k + q] = out[q];
  }
}

}  // namespace gf
