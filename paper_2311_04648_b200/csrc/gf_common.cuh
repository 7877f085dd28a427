// gf_common.cuh -- device-side data model and exact-arithmetic helpers shared
// by the kT (contact detection) and dT (force / reduce / integrate) kernels.
//
// Exactness: the kT translation unit and the fp64 "parity" dT unit are built
// with -fmad=false, so every helper below rounds each fp64 operation
// separately in the reference's statement order (numba fastmath=False,
// /root/reference/pkg/src/grainforge/_kernels.py:17).  Only log() is avoided
// on the device: restitution damping beta comes from a host table computed
// with the same libm the reference uses (forces.py:41-44).
#pragma once
#ifdef __CUDACC_RTC__
// NVRTC (user force models): no host headers; fixed-width types by hand
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned int uint32_t;
typedef unsigned short uint16_t;
typedef unsigned char uint8_t;
#else
#include <cstdint>
#include <cuda_runtime.h>
#endif

namespace gf {

constexpr int kVoxBits = 21;                       // types.py:28
constexpr int64_t kVoxPerAxis = int64_t(1) << kVoxBits;
constexpr int kSubPerEdge = 65536;                 // types.py:31
constexpr double kFlatRadius = 1.0e18;             // _kernels.py:25
constexpr double kPi = 3.141592653589793;
constexpr int kGeomPlane = 2;                      // core.py:46
constexpr int kGeomCylinder = 3;
constexpr uint32_t kKindShift = 30;                // ACS id word: kind in bits 30-31
constexpr uint32_t kSlotMask = (1u << kKindShift) - 1u;
constexpr int kMaxBins = 1 << 22;                  // broadphase.py:20
constexpr int kFamilies = 256;

// family flag bits (engine.py:264-271)
constexpr uint8_t kFamFixed = 1;
constexpr uint8_t kFamPrescribed = 2;

// ---------------------------------------------------------------------------
// device scene: plain pointers, passed by value to every kernel
// ---------------------------------------------------------------------------
struct Domain {
  double lo[3], hi[3], edge;
};

struct Owners {
  int64_t n;
  uint64_t *voxel;     // packed 3 x 21-bit cells, x lowest (types.py:27-32)
  ushort4 *sub;        // sub-voxel x, y, z (w unused)
  float4 *quat;        // (w, x, y, z) float32 (types.py:15)
  void *lin_vel;       // VelT[4] per owner (x, y, z, pad)
  void *ang_vel;       // VelT[4] per owner, owner-local frame
  uint32_t *meta;      // family (bits 24-31) | template id (bits 0-23)
  double4 *tpl;        // per template: mass, moi x, y, z
  double *acc;         // [n*6] force xyz, torque xyz (global frame), optional
  double *ext;         // [n*6] external force/torque or nullptr
  long long *facc;     // [n*6] fixed-point accumulators (throughput build), zeroed by the integrator
  double2 *tpl_scale;  // per template: fixed-point scale of force, torque
  const uint32_t *dd;  // spatial decomposition: class (bits 0-1) | global owner id << 2, or nullptr
  const double *dd_x0; // partition-time coordinate of each owner along the slab axis
  double dd_travel;    // allowed displacement along the axis before a repartition
  int dd_axis;
  const uint8_t *passive;  // [256] per family: fixed or fully prescribed (its accumulators never feed it)
};

// Spatial decomposition (slab partition across ranks).  Every owner of a
// rank-local context is one of
//   kDdLocal   integrated here; its state is the truth
//   kDdGhost   a copy of an owner integrated on another rank (halo)
//   kDdShared  a boundary owner (mesh / analytic) replicated on every rank
//   kDdPrimary the same, on the one rank that also computes shared-shared pairs
// Each physical contact is computed on exactly one rank: ghost-ghost and
// ghost-shared pairs never (the ghost's home rank has them), local-ghost
// pairs only on the rank owning the lower global owner id.  Integer
// (fixed-point) force contributions of ghosts are returned to their home rank,
// so a decomposed run sums exactly the terms a single context sums.
enum : uint32_t { kDdLocal = 0, kDdGhost = 1, kDdShared = 2, kDdPrimary = 3 };

__host__ __device__ inline bool dd_keep(const uint32_t *dd, uint32_t oa, uint32_t ob) {
  if (!dd) return true;
  const uint32_t a = dd[oa], b = dd[ob], ca = a & 3u, cb = b & 3u;
  if (ca == kDdGhost || cb == kDdGhost) {
    if (ca == kDdLocal) return (a >> 2) < (b >> 2);
    if (cb == kDdLocal) return (b >> 2) < (a >> 2);
    return false;
  }
  if (ca == kDdLocal || cb == kDdLocal) return true;
  return ca == kDdPrimary && cb == kDdPrimary;
}

// Per-sphere kinematics record of the throughput build, written wherever the
// sphere centres are (integrator, refresh, halo unpack) so the contact kernel
// reaches everything it needs one load after the contact list, with no
// further dependent loads -- 48 B, three 16-byte loads:
//   v = owner linear velocity,                  v.w = owner mass (float)
//   w = owner angular velocity (global frame),  w.w = owner id (bits)
//   r = centre minus owner position,            r.w = packed (bits): force-scale
//       exponent (bits 24-31), torque-scale exponent (16-23), material (8-15),
//       flags (0-7; bit 0 = passive owner)
// The fixed-point scales are the owner template's tpl_scale, powers of two by
// construction (gf_context.cu update_fixed_scales), stored as exponents;
// kKinNoScale = boundary owner (scale 0), summed with fp64 atomics.
constexpr uint32_t kKinPassive = 1u;
constexpr int kKinNoScale = -128;
struct SphKin {
  float4 v, w, r;
};
__device__ __forceinline__ uint32_t kin_owner(const SphKin &k) { return __float_as_uint(k.w.w); }
__device__ __forceinline__ uint32_t kin_mat(const SphKin &k) { return (__float_as_uint(k.r.w) >> 8) & 0xFFu; }
__device__ __forceinline__ uint32_t kin_flags(const SphKin &k) { return __float_as_uint(k.r.w) & 0xFFu; }
__device__ __forceinline__ double kin_exp2(int e) {   // 2^e exactly, 0 for kKinNoScale
  return e == kKinNoScale ? 0.0 : __longlong_as_double((long long)(1023 + e) << 52);
}
__device__ __forceinline__ double kin_fscale(const SphKin &k) {
  return kin_exp2(int((signed char)(__float_as_uint(k.r.w) >> 24)));
}
__device__ __forceinline__ double kin_tscale(const SphKin &k) {
  return kin_exp2(int((signed char)((__float_as_uint(k.r.w) >> 16) & 0xFFu)));
}

// one 256-bit read-only load of a 32-byte record (LDG.E.256 on sm_100).  An
// NVRTC older than 12.9 (torch ships 12.8; a process that imported torch has
// it loaded) rejects 256-bit vectors: code compiled there takes two 128-bit
// loads.
#if defined(__CUDACC_RTC__) && (__CUDACC_VER_MAJOR__ * 100 + __CUDACC_VER_MINOR__ < 1209)
#define GF_LD256 0
#else
#define GF_LD256 1
#endif
__device__ __forceinline__ double4 ld256(const double4 *p) {
  double4 r;
#if GF_LD256
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
#else
  const double2 *q = reinterpret_cast<const double2 *>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1);
  r = make_double4(a.x, a.y, b.x, b.y);
#endif
  return r;
}

struct Spheres {
  int64_t n;
  uint32_t *owner;
  float4 *offr;        // local offset xyz + radius (float32 geom params)
  uint8_t *mat;
  double4 *center;     // world centre + radius, refreshed by the integrator
  uint32_t *first;     // [n_owner + 1] CSR: spheres of owner o are [first[o], first[o+1])
  SphKin *kin;         // throughput build only (fp32 velocities), else nullptr
};

struct Tris {
  int64_t n;
  uint32_t *owner;
  float *local;        // [n*9] owner-local vertices
  uint8_t *mat;
  double *world;       // [n*9]
};

struct Anas {
  int64_t n;
  uint32_t *owner;
  uint8_t *kind;
  float *local;        // [n*8]
  uint8_t *mat;
  double *world;       // [n*8]
};

struct Materials {
  int n_mat;
  const double *pair;  // [(2 + n_props) * M * M]: E_cnt, G_cnt, CoR, mu, Crr
  const double *beta;  // [M * M] restitution damping, host-computed
};

struct Families {
  const uint8_t *mask;        // [256*256]
  const uint8_t *flags;       // [256] kFamFixed | kFamPrescribed
  const uint8_t *lv_mask;     // [256] bit ax
  const uint8_t *av_mask;     // [256]
  const double *lv_val;       // [256*3]
  const double *av_val;       // [256*3]
};

// device status block (watchdog records, counters)
struct Status {
  // line 0: watchdog words and stop flags -- read by every dT thread, written
  // only when something trips, so it stays clean in every L1
  unsigned long long bad;    // (step << 40) | owner of first speeding owner, or ~0
  unsigned long long oob;    // same for out-of-domain
  unsigned long long dd_trip;  // first step a local owner exceeded the decomposition travel, or ~0;
                               // later steps are skipped (that step itself completes)
  double oob_pos[3];
  int err;                   // nonzero once a watchdog tripped (kernels stop)
  int rebuild;               // detection phase A: candidate lists must be rebuilt
  unsigned long long pad0[9];
  // line 1: kT counters (atomics on the kT stream)
  unsigned long long acs_total;   // last detection's pair count
  unsigned long long cand_total;   // candidate pairs of the last rebuild
  unsigned long long other_total;  // sphere-triangle / sphere-analytic pairs of the last detection
  unsigned long long cand_overflow;  // candidate fill: pairs beyond the counted capacity (must stay 0)
  unsigned long long pad1[12];
  // line 2: dT counters (one atomic per k_touch block)
  unsigned long long touching;
  unsigned long long touch_pairs;  // touching ACS entries summed over the run's steps
  unsigned long long pad2[14];
};

__host__ __device__ inline uint32_t meta_family(uint32_t m) { return m >> 24; }
__host__ __device__ inline uint32_t meta_tpl(uint32_t m) { return m & 0xFFFFFFu; }

// ---------------------------------------------------------------------------
// exact fp64 helpers (explicit _rn intrinsics: no contraction possible)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }

// compressed position -> fp64 (_kernels.py:55-67)
__device__ __forceinline__ void decode_pos(const Domain &d, uint64_t v, ushort4 s,
                                           double &x, double &y, double &z) {
  const uint64_t m = uint64_t(kVoxPerAxis - 1);
  double cx = double(v & m), cy = double((v >> kVoxBits) & m), cz = double((v >> (2 * kVoxBits)) & m);
  x = add(d.lo[0], mul(add(cx, double(s.x) / double(kSubPerEdge)), d.edge));
  y = add(d.lo[1], mul(add(cy, double(s.y) / double(kSubPerEdge)), d.edge));
  z = add(d.lo[2], mul(add(cz, double(s.z) / double(kSubPerEdge)), d.edge));
}

// fp64 -> compressed position; false when outside the domain box
// (_kernels.py:33-52)
__device__ __forceinline__ bool encode_pos(const Domain &d, const double p[3], uint64_t &v,
                                           ushort4 &s) {
  v = 0;
  unsigned short sv[3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    if (p[ax] < d.lo[ax] || p[ax] > d.hi[ax]) return false;
    double t = sub_(p[ax], d.lo[ax]) / d.edge;
    long long cell = (long long)t;
    if (cell >= kVoxPerAxis) cell = kVoxPerAxis - 1;
    long long q = (long long)mul(sub_(t, double(cell)), double(kSubPerEdge));
    if (q >= kSubPerEdge) q = kSubPerEdge - 1;
    v |= uint64_t(cell) << (kVoxBits * ax);
    sv[ax] = (unsigned short)q;
  }
  s = make_ushort4(sv[0], sv[1], sv[2], 0);
  return true;
}

// r = v + 2 u x (u x v + w v), term order of _kernels.py:75-83
__device__ __forceinline__ void qrot(double qw, double qx, double qy, double qz, double vx,
                                     double vy, double vz, double &rx, double &ry, double &rz) {
  double tx = add(sub_(mul(qy, vz), mul(qz, vy)), mul(qw, vx));
  double ty = add(sub_(mul(qz, vx), mul(qx, vz)), mul(qw, vy));
  double tz = add(sub_(mul(qx, vy), mul(qy, vx)), mul(qw, vz));
  rx = add(vx, mul(2.0, sub_(mul(qy, tz), mul(qz, ty))));
  ry = add(vy, mul(2.0, sub_(mul(qz, tx), mul(qx, tz))));
  rz = add(vz, mul(2.0, sub_(mul(qx, ty), mul(qy, tx))));
}

// kinematics record from the STORED owner state (quaternion, float32
// velocities), identical wherever it is computed
__device__ __forceinline__ void write_kin(const Spheres &sph, uint32_t k, uint32_t o, const float4 q,
                                          const float4 lv, const float4 av, float mass, double2 scale,
                                          uint32_t flags) {
  const float4 orr = sph.offr[k];
  double r[3], w[3];
  qrot(double(q.x), double(q.y), double(q.z), double(q.w), double(orr.x), double(orr.y), double(orr.z), r[0], r[1],
       r[2]);
  qrot(double(q.x), double(q.y), double(q.z), double(q.w), double(av.x), double(av.y), double(av.z), w[0], w[1],
       w[2]);
  // power-of-two scales -> their exponents (ilogb is exact on powers of two)
  const int ef = scale.x > 0.0 ? ilogb(scale.x) : kKinNoScale, et = scale.y > 0.0 ? ilogb(scale.y) : kKinNoScale;
  const uint32_t packed = ((uint32_t(ef) & 0xFFu) << 24) | ((uint32_t(et) & 0xFFu) << 16) |
                          (uint32_t(sph.mat[k]) << 8) | (flags & 0xFFu);
  SphKin kr;
  kr.v = make_float4(lv.x, lv.y, lv.z, mass);
  kr.w = make_float4(float(w[0]), float(w[1]), float(w[2]), __uint_as_float(o));
  kr.r = make_float4(float(r[0]), float(r[1]), float(r[2]), __uint_as_float(packed));
  sph.kin[k] = kr;
}

__device__ __forceinline__ void write_kin_from_state(const Owners &own, const Spheres &sph, uint32_t k, uint32_t o) {
  const uint32_t meta = own.meta[o], t = meta_tpl(meta);
  const uint32_t flags = (own.passive && own.passive[meta_family(meta)]) ? kKinPassive : 0u;
  write_kin(sph, k, o, own.quat[o], reinterpret_cast<const float4 *>(own.lin_vel)[o],
            reinterpret_cast<const float4 *>(own.ang_vel)[o], float(own.tpl[t].x), own.tpl_scale[t], flags);
}

// sphere world centre: owner pos + q * offset (_kernels.py:91-106)
__device__ __forceinline__ void sphere_center(const Domain &d, const Owners &o, const Spheres &s,
                                              uint32_t k, double c[3], float &radius,
                                              uint32_t &owner) {
  owner = s.owner[k];
  float4 orr = s.offr[k];
  float4 q = o.quat[owner];
  double px, py, pz;
  decode_pos(d, o.voxel[owner], o.sub[owner], px, py, pz);
  double rx, ry, rz;
  qrot(double(q.x), double(q.y), double(q.z), double(q.w), double(orr.x), double(orr.y),
       double(orr.z), rx, ry, rz);
  c[0] = add(px, rx);
  c[1] = add(py, ry);
  c[2] = add(pz, rz);
  radius = orr.w;
}

// Ericson RTCD 5.1.5, branch order of _kernels.py:159-194
__device__ inline void closest_on_tri(double px, double py, double pz, const double *t,
                                      double &qx, double &qy, double &qz) {
  double ax = t[0], ay = t[1], az = t[2], bx = t[3], by = t[4], bz = t[5];
  double cx = t[6], cy = t[7], cz = t[8];
  double abx = sub_(bx, ax), aby = sub_(by, ay), abz = sub_(bz, az);
  double acx = sub_(cx, ax), acy = sub_(cy, ay), acz = sub_(cz, az);
  double apx = sub_(px, ax), apy = sub_(py, ay), apz = sub_(pz, az);
  double d1 = add(add(mul(abx, apx), mul(aby, apy)), mul(abz, apz));
  double d2 = add(add(mul(acx, apx), mul(acy, apy)), mul(acz, apz));
  if (d1 <= 0.0 && d2 <= 0.0) { qx = ax; qy = ay; qz = az; return; }
  double bpx = sub_(px, bx), bpy = sub_(py, by), bpz = sub_(pz, bz);
  double d3 = add(add(mul(abx, bpx), mul(aby, bpy)), mul(abz, bpz));
  double d4 = add(add(mul(acx, bpx), mul(acy, bpy)), mul(acz, bpz));
  if (d3 >= 0.0 && d4 <= d3) { qx = bx; qy = by; qz = bz; return; }
  double vc = sub_(mul(d1, d4), mul(d3, d2));
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    double s = d1 / sub_(d1, d3);
    qx = add(ax, mul(s, abx)); qy = add(ay, mul(s, aby)); qz = add(az, mul(s, abz));
    return;
  }
  double cpx = sub_(px, cx), cpy = sub_(py, cy), cpz = sub_(pz, cz);
  double d5 = add(add(mul(abx, cpx), mul(aby, cpy)), mul(abz, cpz));
  double d6 = add(add(mul(acx, cpx), mul(acy, cpy)), mul(acz, cpz));
  if (d6 >= 0.0 && d5 <= d6) { qx = cx; qy = cy; qz = cz; return; }
  double vb = sub_(mul(d5, d2), mul(d1, d6));
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double s = d2 / sub_(d2, d6);
    qx = add(ax, mul(s, acx)); qy = add(ay, mul(s, acy)); qz = add(az, mul(s, acz));
    return;
  }
  double va = sub_(mul(d3, d6), mul(d5, d4));
  if (va <= 0.0 && sub_(d4, d3) >= 0.0 && sub_(d5, d6) >= 0.0) {
    double s = sub_(d4, d3) / add(sub_(d4, d3), sub_(d5, d6));
    qx = add(bx, mul(s, sub_(cx, bx)));
    qy = add(by, mul(s, sub_(cy, by)));
    qz = add(bz, mul(s, sub_(cz, bz)));
    return;
  }
  double denom = 1.0 / add(add(va, vb), vc);
  double v = mul(vb, denom), w = mul(vc, denom);
  qx = add(add(ax, mul(abx, v)), mul(acx, w));
  qy = add(add(ay, mul(aby, v)), mul(acy, w));
  qz = add(add(az, mul(abz, v)), mul(acz, w));
}

// plane / cylinder gap, push direction and signed curvature (_kernels.py:209-231)
__device__ inline void analytic_gap(int kind, const double *prm, double cx, double cy, double cz,
                                    double &gap, double &bx, double &by, double &bz, double &rb) {
  if (kind == kGeomPlane) {
    double nx = prm[3], ny = prm[4], nz = prm[5];
    gap = add(add(mul(sub_(cx, prm[0]), nx), mul(sub_(cy, prm[1]), ny)), mul(sub_(cz, prm[2]), nz));
    bx = nx; by = ny; bz = nz; rb = kFlatRadius;
    return;
  }
  double ax = prm[3], ay = prm[4], az = prm[5];
  double wx = sub_(cx, prm[0]), wy = sub_(cy, prm[1]), wz = sub_(cz, prm[2]);
  double axial = add(add(mul(wx, ax), mul(wy, ay)), mul(wz, az));
  double rx = sub_(wx, mul(axial, ax)), ry = sub_(wy, mul(axial, ay)), rz = sub_(wz, mul(axial, az));
  double rho = sqrt(add(add(mul(rx, rx), mul(ry, ry)), mul(rz, rz)));
  double radius = prm[6], facing = prm[7];
  if (rho < 1e-300) { gap = radius; bx = 0.0; by = 0.0; bz = 0.0; rb = radius; return; }
  double inv = 1.0 / rho;
  if (facing > 0.0) {
    gap = sub_(rho, radius); bx = mul(rx, inv); by = mul(ry, inv); bz = mul(rz, inv); rb = radius;
  } else {
    gap = sub_(radius, rho); bx = mul(-rx, inv); by = mul(-ry, inv); bz = mul(-rz, inv); rb = -radius;
  }
}

// ---------------------------------------------------------------------------
// uniform grid (broadphase.py:160-186, _kernels.py:238-266)
// ---------------------------------------------------------------------------
struct Grid {
  // the reference's grid (bin = 2 (r_max + margin), _grid_for): used only
  // to evaluate its exact pair predicate (the min-corner bin test)
  double glo[3];
  double inv_bin;
  long long nb[3];
  int valid;
  // enumeration grid: cell = 2 (r_cut + margin) over the same origin; spheres
  // with radius > r_cut ("big") are not registered and are paired by k_big
  double inv_cell;
  long long nc[3];
  double r_cut;
};

__device__ __forceinline__ long long axis_bin(double x, double glo, double inv_bin, long long nb) {
  long long i = (long long)mul(sub_(x, glo), inv_bin);
  if (i < 0) i = 0;
  if (i >= nb) i = nb - 1;
  return i;
}

// inclusive per-axis bin range of a margin-enlarged sphere (_kernels.py:253-266)
__device__ __forceinline__ void sphere_range(const Grid &g, const double c[3], float radius,
                                             double margin, long long lo[3], long long hi[3]) {
  double r = add(double(radius), margin);
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    long long l = (long long)mul(sub_(sub_(c[ax], r), g.glo[ax]), g.inv_bin);
    long long h = (long long)mul(sub_(add(c[ax], r), g.glo[ax]), g.inv_bin);
    if (l < 0) l = 0;
    if (h < 0) h = 0;
    if (l >= g.nb[ax]) l = g.nb[ax] - 1;
    if (h >= g.nb[ax]) h = g.nb[ax] - 1;
    lo[ax] = l;
    hi[ax] = h;
  }
}

}  // namespace gf
