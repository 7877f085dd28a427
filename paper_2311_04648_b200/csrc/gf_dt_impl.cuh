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
#include <algorithm>
#include <type_traits>
#include "gf_context.h"
#include "gf_device.cuh"

namespace gf {



namespace {
// narrow phase of the step: one thread per ACS entry, geometry only.
// Touching entries are compacted into tlist (warp-aggregated append); the
// fp64 parity build also records a touch flag per entry for its reduction.
// A false positive leaves its history untouched (forces.py:95-97).
// Block-aggregated append of per-thread counts: returns this thread's first
// output slot in each list; one atomic per block per counter.
__device__ __forceinline__ void block_append(unsigned c0, unsigned c1, unsigned tch, unsigned long long *tlist_n,
                                             Status *st, unsigned long long &w0, unsigned long long &w1) {
  __shared__ unsigned s_cnt[2][8], s_tch[8], s_off[2][8];
  __shared__ unsigned long long s_base[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned p0 = c0, p1 = c1;   // inclusive warp scans
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned u0 = __shfl_up_sync(0xffffffffu, p0, off), u1 = __shfl_up_sync(0xffffffffu, p1, off);
    if (lane >= off) { p0 += u0; p1 += u1; }
  }
  for (int off = 16; off > 0; off >>= 1) tch += __shfl_down_sync(0xffffffffu, tch, off);
  if (lane == 31) {
    s_cnt[0][warp] = p0;
    s_cnt[1][warp] = p1;
  }
  if (lane == 0) s_tch[warp] = tch;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned tot[2] = {0, 0}, tt = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) {
      for (int l = 0; l < 2; ++l) {
        s_off[l][w] = tot[l];
        tot[l] += s_cnt[l][w];
      }
      tt += s_tch[w];
    }
    for (int l = 0; l < 2; ++l) s_base[l] = tot[l] ? atomicAdd(tlist_n + l, (unsigned long long)tot[l]) : 0ull;
    if (tot[0] + tot[1]) {
      atomicAdd(&st->touching, (unsigned long long)tt);
      atomicAdd(&st->touch_pairs, (unsigned long long)(tot[0] + tot[1]));
    }
  }
  __syncthreads();
  w0 = s_base[0] + s_off[0][warp] + (p0 - c0);
  w1 = s_base[1] + s_off[1][warp] + (p1 - c1);
}

// Generic narrow phase over entries [*k0p, n_acs) (from 0 if k0p is null):
// all kinds (parity build / user models) or -- in the throughput build, where
// k_touch_ss takes the sphere-sphere block -- only the wall kinds.  Block-
// uniform grid-stride loop (the tail's length is known only on the device).
__global__ void __launch_bounds__(256, 4) k_touch(DtView v, uint32_t *tlist, uint32_t *tlist_other,
                                                  unsigned long long *tlist_n, unsigned long long step,
                                                  const unsigned long long *k0p) {
  __shared__ int s_live;
  pdl_wait();
  pdl_launch();
  if (threadIdx.x == 0) s_live = !v.st->err && v.st->dd_trip >= step;
  __syncthreads();
  if (!s_live) return;
  const int64_t start = k0p ? int64_t(*k0p) : 0;
  for (int64_t base = start + blockIdx.x * int64_t(blockDim.x); base < v.n_acs;
       base += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = base + threadIdx.x;
    bool t = false;
    unsigned kind = 0;
    if (k < v.n_acs) {
      const uint2 id = v.ids[k];
      kind = id.y >> kKindShift;
      double ca[3], ra, depth, bx, by, bz, rb;
      contact_geometry(v, id, ca, ra, depth, bx, by, bz, rb);
      t = depth > 0.0;
      if (!v.own.facc) v.touch[k] = t ? 1 : 0;
    }
    unsigned long long w0, w1;
    block_append((t && kind == 0) ? 1u : 0u, (t && kind != 0) ? 1u : 0u, t ? (kind == 0 ? 2u : 1u) : 0u,
                 tlist_n, v.st, w0, w1);
    if (t && kind == 0) tlist[w0] = uint32_t(k);
    if (t && kind != 0) tlist_other[w1] = uint32_t(k);
    __syncthreads();   // block_append's shared words are reused next round
  }
}

// Throughput build, sphere-sphere block [0, seg[n_sph]) of the contact
// array: d^2 < (ra + rb)^2 (the predicate k_forces_f32 uses), E entries per
// thread so their centre gathers are in flight together; touching entries
// leave as (a, b, k) records, ascending within the block.
constexpr int kTouchPerThread = 2;
__global__ void __launch_bounds__(256, 4) k_touch_ss(DtView v, uint4 *rec, unsigned long long *tlist_n,
                                                     unsigned long long step) {
  constexpr int E = kTouchPerThread;
  __shared__ int s_live;
  if (threadIdx.x == 0) s_live = !v.st->err && v.st->dd_trip >= step;
  __syncthreads();
  const int64_t n_ss = int64_t(v.seg[v.n_sph]);
  const int64_t k0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * E;
  uint2 id[E];
#pragma unroll
  for (int j = 0; j < E; ++j) id[j] = (s_live && k0 + j < n_ss) ? v.ids[k0 + j] : make_uint2(0u, 0u);
  unsigned m = 0;
  {
    double4 ca[E], cb[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      if (s_live && k0 + j < n_ss) {
        ca[j] = v.sph.center[id[j].x];
        cb[j] = v.sph.center[id[j].y & kSlotMask];
      }
    }
#pragma unroll
    for (int j = 0; j < E; ++j) {
      if (s_live && k0 + j < n_ss) {
        const double dx = ca[j].x - cb[j].x, dy = ca[j].y - cb[j].y, dz = ca[j].z - cb[j].z;
        const double R = ca[j].w + cb[j].w;
        if (float(R * R - (dx * dx + dy * dy + dz * dz)) > 0.f) m |= 1u << j;
      }
    }
  }
  unsigned long long w0, w1;
  block_append(__popc(m), 0u, 2u * __popc(m), tlist_n, v.st, w0, w1);
#pragma unroll
  for (int j = 0; j < E; ++j)
    if (m & (1u << j)) rec[w0++] = make_uint4(id[j].x, id[j].y & kSlotMask, uint32_t(k0 + j), 0u);
}

}  // namespace

// force phase of the built-in Hertz-Mindlin model: touching entries only
// (list0 = sphere-sphere entries unless skip0, then list1 = other kinds)
template <typename VelT>
__global__ void __launch_bounds__(128) k_forces(DtView v, double ts, double sim_time, const uint32_t *list0,
                                                const uint32_t *list1, const unsigned long long *counts,
                                                int skip0) {
  __shared__ BCache bc;
  __shared__ int s_err;
  pdl_wait();
  pdl_launch();
  bcache_init(bc);
  if (threadIdx.x == 0) s_err = v.st->err;
  __syncthreads();
  if (s_err) return;
  BCache *bcp = v.own.facc ? &bc : nullptr;
  const unsigned long long n0 = skip0 ? 0ull : counts[0], n = n0 + counts[1];
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    force_entry<VelT, HmCore>(v, i < n0 ? list0[i] : list1[i - n0], ts, sim_time, bcp);
  if (bcp == nullptr) return;
  __syncthreads();
  bcache_flush(v, bc);
}

// fp32 rotation by q = (w, x, y, z) (lever arms and angular velocities of
// the fp32 fast path; same formula as qrot)
__device__ __forceinline__ void qrotf(const float4 q, float x, float y, float z, float &rx, float &ry, float &rz) {
  const float tx = (q.z * z - q.w * y) + q.x * x;
  const float ty = (q.w * x - q.y * z) + q.x * y;
  const float tz = (q.y * y - q.z * x) + q.x * z;
  rx = x + 2.f * (q.z * tz - q.w * ty);
  ry = y + 2.f * (q.w * tx - q.y * tz);
  rz = z + 2.f * (q.y * ty - q.z * tx);
}

// Throughput build, built-in Hertz-Mindlin: sphere-sphere contacts with the
// centre difference and the overlap numerator R^2 - d^2 in fp64, everything
// after in fp32 (normal, lever arms from the fp32-rotated clump offsets,
// velocities, the contact law).  The other kinds (walls) take k_forces.
// Contributions go to the int64 fixed-point owner accumulators as before.
constexpr int kSmemMat = 256;   // material pairs staged in shared memory (n_mat <= 16)

// pair table rows E_cnt, G_cnt, mu, C_rr, beta as float (forces.py:443-460),
// staged in shared memory when n_mat <= 16
__device__ __forceinline__ bool stage_materials(const DtView &v, float (*s_mat)[kSmemMat]) {
  const int nm = v.mat.n_mat, mm = nm * nm;
  if (mm > kSmemMat) return false;
  for (int q = threadIdx.x; q < mm; q += blockDim.x) {
    s_mat[0][q] = float(v.mat.pair[q]);
    s_mat[1][q] = float(v.mat.pair[mm + q]);
    s_mat[2][q] = float(v.mat.pair[3 * mm + q]);
    s_mat[3][q] = float(v.mat.pair[4 * mm + q]);
    s_mat[4][q] = float(v.mat.beta[q]);
  }
  return true;
}

// Geometry of a touching sphere-sphere entry, as the narrow phase leaves it:
// centre difference A - B (fp64, rounded to fp32), its length, the overlap
// numerator R^2 - d^2 (fp64, rounded) and the radii.
struct SsGeom {
  float dx, dy, dz, d, num, ra, rb;
};

__device__ __forceinline__ bool ss_geom(const DtView &v, uint32_t a, uint32_t b, SsGeom &g) {
  const double4 cA = ld256(v.sph.center + a), cB = ld256(v.sph.center + b);
  const double dx = cA.x - cB.x, dy = cA.y - cB.y, dz = cA.z - cB.z;
  const double d2 = dx * dx + dy * dy + dz * dz;
  const double R = cA.w + cB.w;
  g.num = float(R * R - d2);
  g.dx = float(dx); g.dy = float(dy); g.dz = float(dz);
  g.d = sqrtf(float(d2));
  g.ra = float(cA.w); g.rb = float(cB.w);
  return g.num > 0.f;
}

// Warp-collective force phase of the fp32 sphere-sphere path: lanes with
// `live` evaluate contact (a, b, k) -- kinematics records, Hertz-Mindlin,
// history in place -- and add their contributions to the int64 fixed-point
// owner accumulators: B side one atomic per word, A side summed over runs of
// equal A owners in consecutive lanes (entries arrive in A-sorted order).
// Every lane of the warp must call it.
__device__ __forceinline__ void ss_force_warp(const DtView &v, bool live, uint32_t a, uint32_t b, uint32_t k,
                                              const SsGeom &g, float ts, const float (*s_mat)[kSmemMat],
                                              bool smem, int lane, long long *red = nullptr,
                                              uint32_t *own = nullptr) {
  float out[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float ta[3] = {0.f, 0.f, 0.f};
  uint32_t oa = 0xFFFFFFFFu;
  double sa_f = 0.0, sa_t = 0.0;
  bool use_a = false, b_row = false;
  long long rb6[6];
  uint32_t ob_ = 0;
  if (live) {
    // one load round: kinematics records (mass, scales, flags included) and
    // the history row
    const SphKin ka = v.sph.kin[a], kb = v.sph.kin[b];
    float4 *wp = reinterpret_cast<float4 *>(v.wild) + k;
    const float4 w4 = *wp;
    const int nm = v.mat.n_mat, mm = nm * nm;
    const float depth = g.num / ((g.ra + g.rb) + g.d);
    float bx = 0.f, by = 0.f, bz = 1.f;
    if (g.d > 1e-30f) {
      const float inv = 1.f / g.d;
      bx = g.dx * inv; by = g.dy * inv; bz = g.dz * inv;
    }
    oa = kin_owner(ka);
    const uint32_t ob = kin_owner(kb);
    ob_ = ob;
    // contact point p = cA - b (ra - depth / 2); lever arms p - pos_a, p - pos_b
    const float ha = g.ra - 0.5f * depth;
    const float rax = ka.r.x - bx * ha, ray = ka.r.y - by * ha, raz = ka.r.z - bz * ha;
    const float rbx = kb.r.x + g.dx - bx * ha, rby = kb.r.y + g.dy - by * ha, rbz = kb.r.z + g.dz - bz * ha;
    const float rotax = ka.w.y * raz - ka.w.z * ray, rotay = ka.w.z * rax - ka.w.x * raz,
                rotaz = ka.w.x * ray - ka.w.y * rax;
    const float rotbx = kb.w.y * rbz - kb.w.z * rby, rotby = kb.w.z * rbx - kb.w.x * rbz,
                rotbz = kb.w.x * rby - kb.w.y * rbx;
    const float vx = (ka.v.x + rotax) - (kb.v.x + rotbx);
    const float vy = (ka.v.y + rotay) - (kb.v.y + rotby);
    const float vz = (ka.v.z + rotaz) - (kb.v.z + rotbz);
    const double ma = ka.v.w, mb = kb.v.w;
    const float mass_eff = float((ma * mb) / (ma + mb));
    const int ab = int(kin_mat(ka)) * nm + int(kin_mat(kb));
    float e_cnt, g_cnt, mu, crr, beta;
    if (smem) {
      e_cnt = s_mat[0][ab]; g_cnt = s_mat[1][ab]; mu = s_mat[2][ab]; crr = s_mat[3][ab]; beta = s_mat[4][ab];
    } else {
      e_cnt = float(v.mat.pair[ab]); g_cnt = float(v.mat.pair[mm + ab]); mu = float(v.mat.pair[3 * mm + ab]);
      crr = float(v.mat.pair[4 * mm + ab]); beta = float(v.mat.beta[ab]);
    }
    float4 w_new;
    hertz_mindlin_core_f32(depth, ts, bx, by, bz, vx, vy, vz, rotbx - rotax, rotby - rotay, rotbz - rotaz, mass_eff,
                           g.ra, g.rb, e_cnt, g_cnt, mu, crr, beta, w4, w_new, out);
    *wp = w_new;
    const float tx = out[0] + out[3], ty = out[1] + out[4], tz = out[2] + out[5];
    ta[0] = ray * tz - raz * ty; ta[1] = raz * tx - rax * tz; ta[2] = rax * ty - ray * tx;
    const float tb[3] = {rby * tz - rbz * ty, rbz * tx - rbx * tz, rbx * ty - rby * tx};
    // B side: one atomic per word (B owners are scattered); staged (red !=
    // nullptr): fixed-point rows through the warp's shared buffer below
    if (v.acc_all || !(kin_flags(kb) & kKinPassive)) {
      const double sbf = kin_fscale(kb), sbt = kin_tscale(kb);
      if (red != nullptr && sbf > 0.0) {
        b_row = true;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          rb6[q] = __double2ll_rn(-double(out[q]) * sbf);
          rb6[3 + q] = __double2ll_rn(-double(tb[q]) * sbt);
        }
      } else {
      unsigned long long *fb = reinterpret_cast<unsigned long long *>(v.own.facc + 6 * size_t(ob));
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        if (sbf > 0.0) {
          atomicAdd(fb + q, (unsigned long long)__double2ll_rn(-double(out[q]) * sbf));
          atomicAdd(fb + 3 + q, (unsigned long long)__double2ll_rn(-double(tb[q]) * sbt));
        } else {
          atomicAdd(reinterpret_cast<double *>(fb + q), -double(out[q]));
          atomicAdd(reinterpret_cast<double *>(fb + 3 + q), -double(tb[q]));
        }
      }
      }
    }
    use_a = v.acc_all || !(kin_flags(ka) & kKinPassive);
    sa_f = kin_fscale(ka);
    sa_t = kin_tscale(ka);
  }
  if (red != nullptr) {
    // B rows, compacted: one RED instruction covers ~5 owners' rows
    const unsigned bm = __ballot_sync(0xffffffffu, b_row);
    if (b_row) {
      const int h = __popc(bm & ((1u << lane) - 1u));
      own[h] = ob_;
#pragma unroll
      for (int q = 0; q < 6; ++q) red[6 * h + q] = rb6[q];
    }
    __syncwarp();
    red_rows(v, red, own, 6 * __popc(bm), lane);
  }
  a_side_sums(v, use_a, oa, sa_f, sa_t, out, ta, lane, red, own);
}

// Throughput build, built-in Hertz-Mindlin, split form: force phase over the
// (a, b, k) records k_touch_ss compacted.  Centre difference and the overlap
// numerator R^2 - d^2 in fp64, everything after in fp32 (normal, lever arms
// from the fp32-rotated clump offsets, velocities, the contact law).  The
// other kinds (walls) take k_forces.
static __global__ void __launch_bounds__(256, 4) k_forces_f32(DtView v, double ts_d, double sim_time,
                                                               const uint4 *rec, const unsigned long long *tlist_n) {
  (void)sim_time;
  __shared__ float s_mat[5][kSmemMat];
  if (v.st->err) return;
  const unsigned long long n = *tlist_n;
  const bool smem = stage_materials(v, s_mat);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  // whole warps iterate together (the A-side reduction needs every lane)
  for (unsigned long long base = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) & ~31ull; base < n;
       base += stride) {
    const unsigned long long i = base + lane;
    uint4 t = make_uint4(0u, 0u, 0u, 0u);
    SsGeom g;
    bool live = false;
    if (i < n) {
      t = rec[i];   // sphere A, sphere B, contact index
      live = ss_geom(v, t.x, t.y, g);
    }
    ss_force_warp(v, live, t.x, t.y, t.z, g, float(ts_d), s_mat, smem, lane);
  }
}

// Throughput build, fused form: narrow phase and force phase in one pass over
// the sphere-sphere block [0, seg[n_sph]).  Each warp tests kSsPerLane x 32
// consecutive entries, appends the touching ones -- in contact order -- to
// its shared-memory queue, and runs the force phase on full batches of 32
// queued contacts, so force lanes are never idle on false positives and the
// touching list never goes through HBM.
constexpr int kSsWarps = 8;

template <int kSsPerLane, int kMinBlocks, bool kStaged = true>
static __global__ void __launch_bounds__(256, kMinBlocks) k_contacts_ss(DtView v, double ts_d, unsigned long long step) {
  constexpr int kSsQueue = 32 * (kSsPerLane + 1);
  __shared__ float s_mat[5][kSmemMat];
  // staged fixed-point rows of the warp's force batch (B side, then A side)
  __shared__ long long s_red[kStaged ? kSsWarps : 1][kStaged ? 192 : 1];
  __shared__ uint32_t s_own[kSsWarps][32];   // [0][0] doubles as the block's live flag at entry
  __shared__ uint32_t q_a[kSsWarps][kSsQueue], q_b[kSsWarps][kSsQueue], q_k[kSsWarps][kSsQueue];
  __shared__ float q_g[7][kSsWarps][kSsQueue];
  const bool smem = stage_materials(v, s_mat);   // static tables: before the predecessor drains
  pdl_wait();
  pdl_launch();
  if (threadIdx.x == 0) s_own[0][0] = !v.st->err && v.st->dd_trip >= step;
  __syncthreads();
  const bool block_live = s_own[0][0] != 0;
  __syncthreads();
  if (!block_live) return;
  const float ts = float(ts_d);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long n_ss = v.seg[v.n_sph];
  // work split: grid-stride over the whole block of entries (v.blocked = 0),
  // or one contiguous range of entries per CTA (v.blocked = 1), its warps
  // interleaved inside it, so the B records a CTA gathers stay in its SM's L1
  // across iterations (partners sit close in the Morton order)
  constexpr unsigned long long kCta = (unsigned long long)kSsWarps * 32 * kSsPerLane;
  unsigned long long wstride = (unsigned long long)gridDim.x * kCta;
  unsigned long long w0 = (blockIdx.x * (unsigned long long)kSsWarps + warp) * 32 * kSsPerLane;
  unsigned long long hi = n_ss;
  if (v.blocked) {
    const unsigned long long span = ((n_ss + gridDim.x * kCta - 1) / (gridDim.x * kCta)) * kCta;
    const unsigned long long lo = blockIdx.x * span;
    hi = min(n_ss, lo + span);
    wstride = kCta;
    w0 = lo + (unsigned long long)warp * 32 * kSsPerLane;
  }
  uint32_t *qa = q_a[warp], *qb = q_b[warp], *qk = q_k[warp];
  // the queue is a ring of kSsQueue slots: qh = its head, qn = its length
  // (a batch advances the head; nothing is moved)
  int qn = 0, qh = 0;
  auto ring = [](int x) { return x >= kSsQueue ? x - kSsQueue : x; };   // x < 2 kSsQueue
  unsigned long long touched = 0;
  auto run_batch = [&](int take) {
    const bool live = lane < take;
    SsGeom g;
    uint32_t a = 0, b = 0, k = 0;
    if (live) {
      const int q = ring(qh + lane);
      a = qa[q]; b = qb[q]; k = qk[q];
      g.dx = q_g[0][warp][q]; g.dy = q_g[1][warp][q]; g.dz = q_g[2][warp][q];
      g.d = q_g[3][warp][q]; g.num = q_g[4][warp][q]; g.ra = q_g[5][warp][q]; g.rb = q_g[6][warp][q];
    }
    ss_force_warp(v, live, a, b, k, g, ts, s_mat, smem, lane, kStaged ? s_red[warp] : nullptr,
                  kStaged ? s_own[warp] : nullptr);
    __syncwarp();
    qh = ring(qh + take);
    qn -= take;
  };
  // the contact list is streamed one iteration ahead (its load is off the
  // critical path of the centre gathers); v.pf also prefetches each touching
  // contact's kinematics records and history row into L2 when it is queued,
  // so the force batch's loads find them there
  uint2 id_next[kSsPerLane];
#pragma unroll
  for (int j = 0; j < kSsPerLane; ++j) {
    const unsigned long long e = w0 + 32 * j + lane;
    id_next[j] = e < hi ? __ldcs(v.ids + e) : make_uint2(0u, 0u);
  }
  for (unsigned long long base = w0; base < hi; base += wstride) {
    uint2 id[kSsPerLane];
#pragma unroll
    for (int j = 0; j < kSsPerLane; ++j) {
      id[j] = id_next[j];
      const unsigned long long e = base + wstride + 32 * j + lane;
      if (v.pf) id_next[j] = e < hi ? __ldcs(v.ids + e) : make_uint2(0u, 0u);
    }
    if (!v.pf) {   // A/B switch (GF_SS_PF=0): the round-1 order, list loaded in the iteration
#pragma unroll
      for (int j = 0; j < kSsPerLane; ++j) {
        const unsigned long long e = base + 32 * j + lane;
        id[j] = e < hi ? v.ids[e] : make_uint2(0u, 0u);
      }
    }
    SsGeom g[kSsPerLane];
    bool t[kSsPerLane];
#pragma unroll
    for (int j = 0; j < kSsPerLane; ++j) {
      const unsigned long long e = base + 32 * j + lane;
      t[j] = e < hi && ss_geom(v, id[j].x, id[j].y & kSlotMask, g[j]);
    }
    if (v.pf) {
#pragma unroll
      for (int j = 0; j < kSsPerLane; ++j) {
        if (t[j]) {
          const char *ka = reinterpret_cast<const char *>(v.sph.kin + id[j].x);
          const char *kb = reinterpret_cast<const char *>(v.sph.kin + (id[j].y & kSlotMask));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kb));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kb + 47));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(ka + 47));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const float4 *>(v.wild) +
                                                        (base + 32 * j + lane)));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kSsPerLane; ++j) {
      const unsigned m = __ballot_sync(0xffffffffu, t[j]);
      if (t[j]) {
        const int pos = ring(qh + qn + __popc(m & ((1u << lane) - 1u)));
        qa[pos] = id[j].x; qb[pos] = id[j].y & kSlotMask; qk[pos] = uint32_t(base + 32 * j + lane);
        q_g[0][warp][pos] = g[j].dx; q_g[1][warp][pos] = g[j].dy; q_g[2][warp][pos] = g[j].dz;
        q_g[3][warp][pos] = g[j].d; q_g[4][warp][pos] = g[j].num; q_g[5][warp][pos] = g[j].ra;
        q_g[6][warp][pos] = g[j].rb;
      }
      qn += __popc(m);
      touched += __popc(m);
    }
    __syncwarp();
    while (qn >= 32) run_batch(32);
  }
  if (qn > 0) run_batch(qn);
  if (lane == 0 && touched) {
    atomicAdd(&v.st->touching, 2ull * touched);
    atomicAdd(&v.st->touch_pairs, touched);
  }
}

// ---------------------------------------------------------------------------
// The fused kernel with the B-side centre gathers moved off the L1 data pipe:
// each warp's 32 B rows (32-byte double4 records) are fetched by the TMA unit
// with tile::gather4 (four rows per instruction, eight instructions per 32
// entries) into a per-warp shared-memory stage, one iteration ahead, and
// completed on an mbarrier; the lanes then read their partner's centre from
// shared memory.  The A side stays an LDG (entries are A-sorted, so a warp's
// A loads coalesce).  Everything after the geometry is k_contacts_ss's.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "GF_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra GF_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *tm, uint64_t *bar, int r0, int r1, int r2,
                                            int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ bool ss_geom_cb(const DtView &v, uint32_t a, const double4 &cB, SsGeom &g) {
  const double4 cA = ld256(v.sph.center + a);
  const double dx = cA.x - cB.x, dy = cA.y - cB.y, dz = cA.z - cB.z;
  const double d2 = dx * dx + dy * dy + dz * dz;
  const double R = cA.w + cB.w;
  g.num = float(R * R - d2);
  g.dx = float(dx); g.dy = float(dy); g.dz = float(dz);
  g.d = sqrtf(float(d2));
  g.ra = float(cA.w); g.rb = float(cB.w);
  return g.num > 0.f;
}

constexpr int kTmaStageBytes = 2 * kSsWarps * 32 * 32 + 128;   // two stages of 32 rows x 32 B per warp + alignment slack

template <int kMinBlocks>
static __global__ void __launch_bounds__(256, kMinBlocks)
    k_contacts_ss_tma(DtView v, double ts_d, unsigned long long step, const __grid_constant__ CUtensorMap tm_c) {
  constexpr int kSsQueue = 64;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ float s_mat[5][kSmemMat];
  __shared__ long long s_red[kSsWarps][192];
  __shared__ uint32_t s_own[kSsWarps][32];
  __shared__ uint32_t q_a[kSsWarps][kSsQueue], q_b[kSsWarps][kSsQueue], q_k[kSsWarps][kSsQueue];
  __shared__ float q_g[7][kSsWarps][kSsQueue];
  __shared__ __align__(8) uint64_t s_bar[kSsWarps][2];
  const bool smem = stage_materials(v, s_mat);
  pdl_wait();
  pdl_launch();
  if (threadIdx.x == 0) s_own[0][0] = !v.st->err && v.st->dd_trip >= step;
  __syncthreads();
  const bool block_live = s_own[0][0] != 0;
  __syncthreads();
  if (!block_live) return;
  const float ts = float(ts_d);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long n_ss = v.seg[v.n_sph];
  constexpr unsigned long long kCta = (unsigned long long)kSsWarps * 32;
  unsigned long long wstride = (unsigned long long)gridDim.x * kCta;
  unsigned long long w0 = (blockIdx.x * (unsigned long long)kSsWarps + warp) * 32;
  unsigned long long hi = n_ss;
  if (v.blocked) {
    const unsigned long long span = ((n_ss + gridDim.x * kCta - 1) / (gridDim.x * kCta)) * kCta;
    const unsigned long long lo = blockIdx.x * span;
    hi = min(n_ss, lo + span);
    wstride = kCta;
    w0 = lo + (unsigned long long)warp * 32;
  }
  uint32_t *qa = q_a[warp], *qb = q_b[warp], *qk = q_k[warp];
  // TMA destinations 128-byte aligned whatever the dynamic base
  unsigned char *dsm_a = dsm + ((128u - (smem_u32(dsm) & 127u)) & 127u);
  double4 *cb = reinterpret_cast<double4 *>(dsm_a) + warp * 32;   // stage st at + st * kSsWarps * 32
  uint64_t *bar = s_bar[warp];
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  int qn = 0;
  unsigned long long touched = 0;
  auto run_batch = [&](int take) {
    const bool live = lane < take;
    SsGeom g;
    uint32_t a = 0, b = 0, k = 0;
    if (live) {
      a = qa[lane]; b = qb[lane]; k = qk[lane];
      g.dx = q_g[0][warp][lane]; g.dy = q_g[1][warp][lane]; g.dz = q_g[2][warp][lane];
      g.d = q_g[3][warp][lane]; g.num = q_g[4][warp][lane]; g.ra = q_g[5][warp][lane]; g.rb = q_g[6][warp][lane];
    }
    ss_force_warp(v, live, a, b, k, g, ts, s_mat, smem, lane, s_red[warp], s_own[warp]);
    __syncwarp();
    const int rest = qn - take;
    for (int j = lane; j < rest; j += 32) {
      const int src = take + j;
      const uint32_t xa = qa[src], xb = qb[src], xk = qk[src];
      float xg[7];
#pragma unroll
      for (int f = 0; f < 7; ++f) xg[f] = q_g[f][warp][src];
      __syncwarp(__activemask());
      qa[j] = xa; qb[j] = xb; qk[j] = xk;
#pragma unroll
      for (int f = 0; f < 7; ++f) q_g[f][warp][j] = xg[f];
    }
    __syncwarp();
    qn = rest;
  };
  // 32 partner rows of the entries at `base` into stage st (rows past the
  // block's end read row 0: the byte count stays 1 KB)
  auto issue = [&](int st, uint32_t brow) {
    if (lane == 0) mbar_expect_tx(bar + st, 32 * 32);
    __syncwarp();
    int r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = __shfl_sync(0xffffffffu, int(brow), (lane & 7) * 4 + q);
    if (lane < 8) tma_gather4(cb + st * (kSsWarps * 32) + 4 * lane, &tm_c, bar + st, r[0], r[1], r[2], r[3]);
  };
  unsigned long long base = w0;
  uint2 id_cur = base + lane < hi ? __ldcs(v.ids + base + lane) : make_uint2(0u, 0u);
  if (base < hi) issue(0, base + lane < hi ? (id_cur.y & kSlotMask) : 0u);
  uint2 id_n1 = base + wstride + lane < hi ? __ldcs(v.ids + base + wstride + lane) : make_uint2(0u, 0u);
  for (int it = 0; base < hi; base += wstride, ++it) {
    const unsigned long long nb = base + wstride;
    if (nb < hi) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // the stage's last reads precede the refill
      issue((it + 1) & 1, nb + lane < hi ? (id_n1.y & kSlotMask) : 0u);
    }
    const uint2 id_n2 = nb + wstride + lane < hi ? __ldcs(v.ids + nb + wstride + lane) : make_uint2(0u, 0u);
    mbar_wait(bar + (it & 1), uint32_t(it >> 1) & 1u);
    const double4 cB = cb[(it & 1) * (kSsWarps * 32) + lane];
    const unsigned long long e = base + lane;
    SsGeom g;
    const bool t = e < hi && ss_geom_cb(v, id_cur.x, cB, g);
    __syncwarp();
    const unsigned m = __ballot_sync(0xffffffffu, t);
    if (t) {
      const int pos = qn + __popc(m & ((1u << lane) - 1u));
      qa[pos] = id_cur.x; qb[pos] = id_cur.y & kSlotMask; qk[pos] = uint32_t(e);
      q_g[0][warp][pos] = g.dx; q_g[1][warp][pos] = g.dy; q_g[2][warp][pos] = g.dz;
      q_g[3][warp][pos] = g.d; q_g[4][warp][pos] = g.num; q_g[5][warp][pos] = g.ra; q_g[6][warp][pos] = g.rb;
    }
    qn += __popc(m);
    touched += __popc(m);
    __syncwarp();
    while (qn >= 32) run_batch(32);
    id_cur = id_n1;
    id_n1 = id_n2;
  }
  if (qn > 0) run_batch(qn);
  if (lane == 0 && touched) {
    atomicAdd(&v.st->touching, 2ull * touched);
    atomicAdd(&v.st->touch_pairs, touched);
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

template <typename VelT, int kMinBlocks = 1>
__global__ void __launch_bounds__(128, kMinBlocks) k_integrate(DtView v, double h, double gx, double gy, double gz,
                                                   double v_err, unsigned long long step, int write_acc) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= v.own.n || v.st->err || v.st->dd_trip < step) return;
  const uint32_t o = uint32_t(i);
  // a ghost is integrated on its home rank; its state arrives by halo exchange
  if (v.own.dd && (v.own.dd[o] & 3u) == kDdGhost) return;
  // independent loads first (one latency round)
  const uint32_t meta = v.own.meta[o];
  const uint64_t vox0 = v.own.voxel[o];
  const ushort4 sub0 = v.own.sub[o];
  float4 q = v.own.quat[o];
  const uint32_t s0 = v.sph.first[o], s1 = v.sph.first[o + 1];
  const uint32_t fam = meta_family(meta);
  const uint8_t fl = v.fam.flags[fam];
  const double4 tp = v.own.tpl[meta_tpl(meta)];
  double p[3];
  decode_pos(v.dom, vox0, sub0, p[0], p[1], p[2]);
  // --- reduction (reduce_to_owners order) ---
  double af[3] = {0, 0, 0}, at[3] = {0, 0, 0};
  double2 sc = make_double2(0.0, 0.0);
  // the fp32-velocity build always reduces into the fixed-point accumulators
  // (Ctx::fixed_reduce == f32_state); the fp64 build always by incidence lists
  pdl_wait();   // owner state above is the previous step's; the accumulators are this step's
  pdl_launch();
  if (std::is_same<VelT, float>::value) {
    longlong2 *fp = reinterpret_cast<longlong2 *>(v.own.facc + 6 * size_t(o));
    const longlong2 a0 = fp[0], a1 = fp[1], a2 = fp[2];
    sc = v.own.tpl_scale[meta_tpl(meta)];
    if (sc.x > 0.0) {
      // scales are powers of two: multiplying by the reciprocal is exact
      const double isf = 1.0 / sc.x, ist = 1.0 / sc.y;
      af[0] = double(a0.x) * isf; af[1] = double(a0.y) * isf; af[2] = double(a1.x) * isf;
      at[0] = double(a1.y) * ist; at[1] = double(a2.x) * ist; at[2] = double(a2.y) * ist;
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
  double vel[3] = {0.0, 0.0, 0.0}, w[3] = {0.0, 0.0, 0.0};
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
  // decomposition guard: the static ghost layer covers displacements up to
  // dd_travel along the slab axis
  if (v.own.dd && (v.own.dd[o] & 3u) == kDdLocal && fabs((v.own.dd_axis == 0 ? p[0] : (v.own.dd_axis == 1 ? p[1] : p[2])) - v.own.dd_x0[o]) > v.own.dd_travel)
    atomicMin(&v.st->dd_trip, step);
  // refreshed sphere centres from the decoded position (_kernels.py:657-669)
  if (s1 > s0) {
    // the stored (float32) velocities, for the kinematics records
    const float4 lv4 = make_float4(float(vel[0]), float(vel[1]), float(vel[2]), 0.f);
    const float4 av4 = make_float4(float(w[0]), float(w[1]), float(w[2]), 0.f);
    const uint32_t kflags = (v.own.passive && v.own.passive[fam]) ? kKinPassive : 0u;
    double pd[3];
    decode_pos(v.dom, vox, s, pd[0], pd[1], pd[2]);
    for (uint32_t k = s0; k < s1; ++k) {
      const float4 orr = v.sph.offr[k];
      double r[3];
      qrot(double(q.x), double(q.y), double(q.z), double(q.w), double(orr.x), double(orr.y), double(orr.z),
           r[0], r[1], r[2]);
      v.sph.center[k] = make_double4(add(pd[0], r[0]), add(pd[1], r[1]), add(pd[2], r[2]), double(orr.w));
      // the whole 48-byte record: writing only its velocity half leaves
      // partial sectors that L2 must fill from DRAM (measured slower)
      if (v.sph.kin) write_kin(v.sph, k, o, q, lv4, av4, float(tp.x), sc, kflags);
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
  if (sph.kin) write_kin_from_state(own, sph, uint32_t(k), o);
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

namespace {
// per-step counters (a kernel rather than memsets, so the chain of
// programmatically-serialised launches is not broken)
__global__ void k_step_begin(Status *st, unsigned long long *tn) {
  pdl_wait();
  pdl_launch();
  if (threadIdx.x == 0) {
    st->touching = 0;
    if (tn) { tn[0] = 0; tn[1] = 0; }
  }
}

// launch with programmatic stream serialisation (Ctx::pdl) or plainly
template <typename... KArgs, typename... Args>
cudaError_t launch_ks(const Ctx *c, void (*kern)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s,
                      Args... args) {
  if (!c->pdl) {
    kern<<<g, b, smem, s>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_k(const Ctx *c, void (*kern)(KArgs...), dim3 g, dim3 b, cudaStream_t s, Args... args) {
  return launch_ks(c, kern, g, b, 0, s, args...);
}
}  // namespace

template <typename VelT>
static DtView dt_view(Ctx *c) {
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
  v.acc_all = 1;
  v.pf = c->ss_pf;
  // contiguous per-CTA ranges pay while the gathered records fit L2 (+2.6 % at
  // 1M spheres); at 16M the grid-stride sweep keeps every CTA in one window of
  // the Morton order and wins (-1.5 % blocked): auto = blocked up to 4M spheres
  v.blocked = c->ss_blocked == 2 ? (c->n_sph <= (int64_t(1) << 22)) : c->ss_blocked;
  return v;
}

// first half of a step: narrow phase + contact forces (+ the heavy-owner
// pre-reduction of the parity build).  Split from the integration so a
// decomposed run can return ghost force contributions in between.
template <typename VelT>
int dt_forces_impl(Ctx *c, const StepArgs &a, cudaStream_t s) {
  DtView v = dt_view<VelT>(c);
  v.acc_all = a.write_acc;
  if (c->pdl) {
    GF_CHECK(c, launch_k(c, k_step_begin, dim3(1), dim3(32), s, v.st,
                         v.n_acs ? c->tlist_n.as<unsigned long long>() : (unsigned long long *)nullptr));
  } else {
    GF_CHECK(c, cudaMemsetAsync(&v.st->touching, 0, sizeof(unsigned long long), s));
    if (v.n_acs) GF_CHECK(c, cudaMemsetAsync(c->tlist_n.p, 0, 2 * sizeof(unsigned long long), s));
  }
  cudaEvent_t *ev = prof_events(c);
  if (ev) cudaEventRecord(ev[0], s);
  bool ss_timed = false;   // ev[4] recorded after the fused sphere-sphere kernel
  if (v.n_acs) {
    unsigned long long *tn = c->tlist_n.as<unsigned long long>();
    // the touching lists were sized for the fused path: a user model or the
    // split path switched on since needs the full layout
    if (!ss_fused(c) && c->tlist_words != 5) {
      if (ensure(c, c->tlist, 5 * sizeof(uint32_t) * c->tlist_cap, s)) return -1;
      c->tlist_words = 5;
    }
    // list0: sphere-sphere entries (uint4 records in the fused build), list1: the other kinds
    uint32_t *list0 = c->tlist.as<uint32_t>(), *list1 = list0 + (c->tlist_words == 5 ? 4 * c->tlist_cap : 0);
    // throughput build + built-in model: sphere-sphere contacts take the fp32
    // path (k_forces_f32), the wall kinds the generic k_forces
    const bool fused = std::is_same<VelT, float>::value && c->wild_w == 4 && !c->user_model && v.sph.kin;
    if (fused && c->ss_split == 1) {
      const int64_t per_block = 256 * kTouchPerThread;
      k_touch_ss<<<unsigned((v.n_acs + per_block - 1) / per_block), 256, 0, s>>>(
          v, reinterpret_cast<uint4 *>(list0), tn, (unsigned long long)a.step);
      // the wall kinds: from the start of the (kind 1, sphere 0) segment
      k_touch<<<unsigned(c->n_sm) * 4, 256, 0, s>>>(v, list0, list1, tn, (unsigned long long)a.step, v.seg + c->n_sph);
      k_forces_f32<<<unsigned(c->n_sm) * 8, 256, 0, s>>>(v, a.h, a.sim_time, reinterpret_cast<const uint4 *>(list0), tn);
    } else if (fused) {
      // the sphere-sphere block in one fused pass, then the wall kinds'
      // narrow phase (feeds k_forces below)
      const unsigned long long step = (unsigned long long)a.step;
      const unsigned nsm = unsigned(c->n_sm);
      if (c->ss_split == 2)
        GF_CHECK(c, launch_k(c, k_contacts_ss<1, 4, false>, dim3(nsm * 4), dim3(256), s, v, a.h, step));
      else if (c->ss_split == 3)
        GF_CHECK(c, launch_k(c, k_contacts_ss<2, 4, false>, dim3(nsm * 4), dim3(256), s, v, a.h, step));
      else if (c->ss_tma && center_tmap(c) == 0) {
        if (!c->ss_tma_smem) {
          GF_CHECK(c, cudaFuncSetAttribute(k_contacts_ss_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kTmaStageBytes));
          c->ss_tma_smem = true;
        }
        GF_CHECK(c, launch_ks(c, k_contacts_ss_tma<3>, dim3(nsm * 3), dim3(256), size_t(kTmaStageBytes), s, v, a.h,
                              step, c->tm_center));
      } else if (!c->ss_red)   // per-word REDs (the round-1 kernel; A/B switch GF_SS_RED=0)
        GF_CHECK(c, launch_k(c, k_contacts_ss<2, 3, false>, dim3(nsm * 3), dim3(256), s, v, a.h, step));
      else
        GF_CHECK(c, launch_k(c, k_contacts_ss<2, 3, true>, dim3(nsm * 3), dim3(256), s, v, a.h, step));
      if (ev) cudaEventRecord(ev[4], s);
      ss_timed = true;
      GF_CHECK(c, launch_k(c, k_touch, dim3(unsigned(c->n_sm) * 4), dim3(256), s, v, list0, list1, tn, step,
                           (const unsigned long long *)(v.seg + c->n_sph)));
    } else if (c->user_model && std::is_same<VelT, float>::value && v.sph.kin && c->user_fn_ss) {
      // user model, throughput build: the NVRTC sphere-sphere loop counts its
      // own touching entries; the narrow phase here covers the wall kinds
      k_touch<<<unsigned(c->n_sm) * 4, 256, 0, s>>>(v, list0, list1, tn, (unsigned long long)a.step, v.seg + c->n_sph);
    } else {
      k_touch<<<unsigned(std::min<int64_t>((v.n_acs + 255) / 256, int64_t(c->n_sm) * 16)), 256, 0, s>>>(
          v, list0, list1, tn, (unsigned long long)a.step, nullptr);
    }
    if (c->user_model) {
      if (launch_user_forces(c, v, a.h, a.sim_time, s)) return -1;
    } else {
      GF_CHECK(c, launch_k(c, k_forces<VelT>, dim3(unsigned(c->n_sm) * 8), dim3(128), s, v, a.h, a.sim_time,
                           (const uint32_t *)list0, (const uint32_t *)list1, (const unsigned long long *)tn,
                           fused ? 1 : 0));
    }
  }
  if (ev) {
    if (!ss_timed) cudaEventRecord(ev[4], s);   // no fused sphere-sphere kernel this step
    cudaEventRecord(ev[1], s);
  }
  if (v.n_acs && !c->fixed_reduce) k_heavy<<<64, 256, 0, s>>>(v);
  if (ev) cudaEventRecord(ev[2], s);
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

// second half: prescriptions, integration, world transforms
template <typename VelT>
int dt_integrate_impl(Ctx *c, const StepArgs &a, cudaStream_t s) {
  DtView v = dt_view<VelT>(c);
  cudaEvent_t *ev = prof_current(c);  // the set the force phase opened
  if (c->n_dyn) {
    k_apply_dyn<<<(c->n_dyn + 127) / 128, 128, 0, s>>>(
        c->n_dyn, c->dyn_spec.as<int>(), c->dyn_vals.as<double>() + size_t(c->n_dyn) * a.dyn_row,
        c->lv_val.as<double>(), c->av_val.as<double>());
  }
  if (c->n_owner) {
    unsigned g = unsigned((c->n_owner + 127) / 128);
    // 8 CTAs / SM (64 registers, a few spills) beats 6 at 91 registers
    GF_CHECK(c, launch_k(c, k_integrate<VelT, 8>, dim3(g), dim3(128), s, v, a.h, a.g[0], a.g[1], a.g[2],
                         a.v_err, (unsigned long long)a.step, a.write_acc));
  }
  if (ev) cudaEventRecord(ev[3], s);
  if ((c->n_tri || c->n_ana) && c->world_moving) {
    int64_t n = c->n_tri + c->n_ana;
    c->world_version++;
    k_world<<<unsigned((n + 127) / 128), 128, 0, s>>>(c->dom, v.own, v.tri, v.ana);
  }
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

template <typename VelT>
int dt_step_impl(Ctx *c, const StepArgs &a, cudaStream_t s) {
  if (dt_forces_impl<VelT>(c, a, s)) return -1;
  return dt_integrate_impl<VelT>(c, a, s);
}

}  // namespace gf
