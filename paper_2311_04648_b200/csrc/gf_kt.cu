// gf_kt.cu -- kinematics worker (kT): snapshot, uniform grid, binning,
// sphere-sphere / sphere-triangle / sphere-analytic pair generation in
// canonical order, and the kT -> dT handoff (history remap + incidence lists).
//
// Compiled with -fmad=false: pair predicates are evaluated with the exact
// fp64 arithmetic of the reference so the produced pair lists are
// bit-identical to broadphase.detect_contacts (broadphase.py:202-288).
//
// Binning scheme (B200-native, not the reference's): every sphere is
// registered once, in the bin holding its centre (one radix-sort key per
// sphere instead of the reference's up-to-8 registrations, _kernels.py:269);
// candidates come from the 27-bin neighbourhood.  The reference reports a pair
// iff it passes the distance test AND the bin of the min corner of the two
// enlarged boxes' intersection lies in both spheres' registration ranges
// (_kernels.py:317-321); that exact predicate is evaluated per candidate, so
// the pair SET is the reference's.  A thread owns sphere i and emits the pairs
// (i, j > i), sorted by j, at an exclusive-scan offset: the output is already
// in canonical (kind, a, b) order and no global pair sort is needed.
#include <cub/cub.cuh>
#include <cstdlib>

#include "gf_context.h"

// per-slot candidate counts are u32 (memory); their prefix sums can pass
// 2^32 (a 10.6M-sphere GRC-1 bed at a 1.6 mm margin has ~5e9 candidates), so
// every scan over them accumulates in u64
struct U32ToU64 {
  __host__ __device__ __forceinline__ unsigned long long operator()(const uint32_t x) const { return x; }
};
using CountsU64 = cub::TransformInputIterator<unsigned long long, U32ToU64, const uint32_t *>;

namespace gf {

namespace {

constexpr int kBlock = 256;
constexpr uint32_t kNoCell = uint32_t(kMaxCells);  // key of spheres kept out of the grid (24 bits)
constexpr int kKeyBits = 24;

inline unsigned grid_for(int64_t n, int block = kBlock) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  return unsigned(g);
}

// order-preserving double <-> uint64 for exact atomic min/max
__device__ __forceinline__ unsigned long long ord_key(double x) {
  unsigned long long u = __double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
  unsigned long long u = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double(u);
}

struct KtView {
  Domain dom;
  Owners own;
  Spheres sph;
  int64_t n_tri, n_ana;
  const uint32_t *tri_owner;
  const uint32_t *ana_owner;
  const uint8_t *ana_kind;
  const double *centers;   // snapshot (centre, radius) records viewed as doubles, stride 4
  const uint8_t *sfam;
  const double *tri_world;
  const uint8_t *tfam;
  const double *ana_world;
  const uint8_t *afam;
  const uint8_t *mask;
  const uint32_t *bin_key;   // sorted centre-bin keys
  const uint32_t *sph_sorted;
  const uint32_t *cell_start, *cell_end;
  const uint32_t *tri_start, *tri_entries;
  const Grid *grid;
  double margin;
  const double4 *c4;   // snapshot (centre, radius) records
  int mask_trivial;    // the family mask allows every pair
};

// ---------------------------------------------------------------------------
// snapshot
// ---------------------------------------------------------------------------
// frozen copy of the refreshed sphere centres and families (engine.py:577-596)
// detection snapshot: also the exact min / max of the centres and the
// largest radius (the grid's inputs, broadphase.py:160-186) and -- when
// candidate lists exist -- whether a sphere moved more than skin / 2 since
// their rebuild (the k_disp test), in the same pass over the centres
__global__ void __launch_bounds__(256) k_snapshot(Domain dom, Owners own, Spheres sph, double4 *c4,
                                                  uint8_t *sfam, unsigned long long *mm,
                                                  const double *ref, double lim2, double lim2_big, double r_cut,
                                                  int *flag) {
  double lo[3], hi[3], rmax = 0.0;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    lo[ax] = __longlong_as_double(0x7FF0000000000000ll);
    hi[ax] = -lo[ax];
  }
  bool far = false;
  // two spheres per iteration, every load issued before the dependent ones
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k0 < sph.n; k0 += 2 * stride) {
    const int64_t kk[2] = {k0, k0 + stride};
    double4 c[2];
    uint32_t ow[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (kk[j] < sph.n) {
        c[j] = ld256(sph.center + kk[j]);
        ow[j] = sph.owner[kk[j]];
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t k = kk[j];
      if (k >= sph.n) continue;
      c4[k] = c[j];
      sfam[k] = uint8_t(meta_family(own.meta[ow[j]]));
      if (mm) {
        lo[0] = fmin(lo[0], c[j].x); lo[1] = fmin(lo[1], c[j].y); lo[2] = fmin(lo[2], c[j].z);
        hi[0] = fmax(hi[0], c[j].x); hi[1] = fmax(hi[1], c[j].y); hi[2] = fmax(hi[2], c[j].z);
        rmax = fmax(rmax, c[j].w);
      }
      if (ref) {
        const double dx = c[j].x - ref[3 * k], dy = c[j].y - ref[3 * k + 1], dz = c[j].z - ref[3 * k + 2];
        far = far || dx * dx + dy * dy + dz * dz > ((r_cut > 0.0 && c[j].w > r_cut) ? lim2_big : lim2);
      }
    }
  }
  if (ref && __any_sync(0xffffffffu, far) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
  if (!mm) return;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      lo[ax] = fmin(lo[ax], __shfl_down_sync(0xffffffff, lo[ax], off));
      hi[ax] = fmax(hi[ax], __shfl_down_sync(0xffffffff, hi[ax], off));
    }
    rmax = fmax(rmax, __shfl_down_sync(0xffffffff, rmax, off));
  }
  __shared__ double sh[7][8];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    for (int ax = 0; ax < 3; ++ax) { sh[ax][warp] = lo[ax]; sh[3 + ax][warp] = hi[ax]; }
    sh[6][warp] = rmax;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    const int q = threadIdx.x;
    double acc = sh[q][0];
    for (int w = 1; w < nw; ++w) acc = q < 3 ? fmin(acc, sh[q][w]) : fmax(acc, sh[q][w]);
    if (q < 3) atomicMin(&mm[q], ord_key(acc));
    else atomicMax(&mm[q], ord_key(acc));
  }
}

__global__ void k_geom_family(int64_t n, const uint32_t *owner, const uint32_t *meta, uint8_t *fam) {
  int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k < n) fam[k] = uint8_t(meta_family(meta[owner[k]]));
}

// ---------------------------------------------------------------------------
// grid (broadphase.py:160-186)
// ---------------------------------------------------------------------------
// mm[0..2] = min xyz, mm[3..5] = max xyz (ordered keys), mm[6] = max radius
__global__ void k_minmax_init(unsigned long long *mm) {
  if (threadIdx.x < 3) {
    mm[threadIdx.x] = ord_key(__longlong_as_double(0x7FF0000000000000ll));        // +inf
    mm[3 + threadIdx.x] = ord_key(__longlong_as_double(0xFFF0000000000000ull));   // -inf
  }
  if (threadIdx.x == 3) mm[6] = ord_key(0.0);
}

__global__ void k_minmax(int64_t n_pts, const double *pts, int stride, int64_t n_s, const float4 *offr,
                         unsigned long long *mm) {
  double lo[3] = {__longlong_as_double(0x7FF0000000000000ll), 0, 0};
  lo[1] = lo[0]; lo[2] = lo[0];
  double hi[3] = {-lo[0], -lo[0], -lo[0]};
  double rmax = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n_pts;
       i += int64_t(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      double v = pts[stride * i + ax];
      lo[ax] = fmin(lo[ax], v);
      hi[ax] = fmax(hi[ax], v);
    }
  }
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n_s;
       i += int64_t(gridDim.x) * blockDim.x)
    rmax = fmax(rmax, double(offr[i].w));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      lo[ax] = fmin(lo[ax], __shfl_down_sync(0xffffffff, lo[ax], off));
      hi[ax] = fmax(hi[ax], __shfl_down_sync(0xffffffff, hi[ax], off));
    }
    rmax = fmax(rmax, __shfl_down_sync(0xffffffff, rmax, off));
  }
  __shared__ double sh[7][32];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    for (int ax = 0; ax < 3; ++ax) { sh[ax][warp] = lo[ax]; sh[3 + ax][warp] = hi[ax]; }
    sh[6][warp] = rmax;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    const int q = threadIdx.x;
    double acc = sh[q][0];
    for (int w = 1; w < nw; ++w) acc = q < 3 ? fmin(acc, sh[q][w]) : fmax(acc, sh[q][w]);
    if (q < 3) atomicMin(&mm[q], ord_key(acc));
    else atomicMax(&mm[q], ord_key(acc));
  }
}

// single thread: exact restatement of _grid_for's scalar arithmetic, plus the
// enumeration grid (cell = 2 (r_cut + margin), same growth rule, own cap)
__global__ void k_grid(const unsigned long long *mm, int64_t n_pts, double margin, double bin_override,
                       double r_cut, long long max_cells, double enum_margin, Grid *g) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Grid out;
  out.valid = n_pts > 0;
  double r_max = ord_val(mm[6]);
  double bin_size = bin_override > 0.0 ? bin_override : mul(2.0, add(r_max, margin));
  if (bin_size <= 0.0) bin_size = 1.0;
  double ext[3];
  for (int ax = 0; ax < 3; ++ax) {
    double mn = ord_val(mm[ax]), mx = ord_val(mm[3 + ax]);
    out.glo[ax] = sub_(sub_(mn, add(r_max, margin)), 1e-9);
    double ghi = add(add(mx, add(r_max, margin)), 1e-9);
    ext[ax] = sub_(ghi, out.glo[ax]);
  }
  for (;;) {
    for (int ax = 0; ax < 3; ++ax) {
      double cc = ceil(ext[ax] / bin_size);
      out.nb[ax] = cc < 1.0 ? 1 : (long long)cc;
    }
    if (out.nb[0] * out.nb[1] * out.nb[2] <= (long long)kMaxBins) break;
    bin_size = mul(bin_size, 1.5);
  }
  out.inv_bin = 1.0 / bin_size;
  // enumeration grid; r_cut <= 0 means "every sphere is small"
  double rc = r_cut > 0.0 && r_cut < r_max ? r_cut : r_max;
  out.r_cut = rc;
  double cell = bin_override > 0.0 ? bin_size : 2.0 * (rc + enum_margin);
  if (cell <= 0.0) cell = 1.0;
  for (;;) {
    for (int ax = 0; ax < 3; ++ax) {
      double cc = ceil(ext[ax] / cell);
      out.nc[ax] = cc < 1.0 ? 1 : (long long)cc;
    }
    if (out.nc[0] * out.nc[1] * out.nc[2] <= max_cells) break;
    cell *= 1.5;
  }
  out.inv_cell = 1.0 / cell;
  if (!out.valid) {
    out.nb[0] = out.nb[1] = out.nb[2] = 1;
    out.nc[0] = out.nc[1] = out.nc[2] = 1;
  }
  *g = out;
}

// ---------------------------------------------------------------------------
// binning
// ---------------------------------------------------------------------------
// one key per sphere: its centre's enumeration cell; big spheres are kept out
__global__ void k_bin_keys(int64_t n, const double *centers, const float4 *offr, const Grid *gp,
                           uint32_t *key, uint32_t *val) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  Grid g = *gp;
  val[i] = uint32_t(i);
  if (double(offr[i].w) > g.r_cut) { key[i] = kNoCell; return; }
  long long ix = axis_bin(centers[4 * i], g.glo[0], g.inv_cell, g.nc[0]);
  long long iy = axis_bin(centers[4 * i + 1], g.glo[1], g.inv_cell, g.nc[1]);
  long long iz = axis_bin(centers[4 * i + 2], g.glo[2], g.inv_cell, g.nc[2]);
  key[i] = uint32_t((iz * g.nc[1] + iy) * g.nc[0] + ix);
}

__global__ void k_cell_bounds(int64_t n, const uint32_t *key, uint32_t *start, uint32_t *end) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  uint32_t k = key[i];
  if (k == kNoCell) return;
  if (i == 0 || key[i - 1] != k) start[k] = uint32_t(i);
  if (i == n - 1 || key[i + 1] != k) end[k] = uint32_t(i + 1);
}

// ---------------------------------------------------------------------------
// enumeration-grid registration of triangles (fine cells overlapping the
// triangle's margin-enlarged AABB; _kernels.py:333-351 on the fine grid)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tri_cells(const Grid &g, const double *T, double margin, int r[6]) {
  for (int ax = 0; ax < 3; ++ax) {
    double lo = T[ax], hi = T[ax];
    for (int v = 1; v < 3; ++v) {
      double x = T[3 * v + ax];
      if (x < lo) lo = x;
      if (x > hi) hi = x;
    }
    r[2 * ax] = int(axis_bin(sub_(lo, margin), g.glo[ax], g.inv_cell, g.nc[ax]));
    r[2 * ax + 1] = int(axis_bin(add(hi, margin), g.glo[ax], g.inv_cell, g.nc[ax]));
  }
}

// one CTA per triangle, its threads over the cells of the triangle's
// margin-enlarged box (a wheel's side-disk facet spans thousands of cells)
template <bool FILL>
__global__ void __launch_bounds__(128) k_tri_register(int64_t n_t, const double *tri, const Grid *gp, double margin,
                                                      uint32_t *cnt, uint32_t *cursor, uint32_t *entries) {
  const Grid g = *gp;
  for (int64_t t = blockIdx.x; t < n_t; t += gridDim.x) {
    int r[6];
    tri_cells(g, tri + 9 * t, margin, r);
    const long long nx = r[1] - r[0] + 1, ny = r[3] - r[2] + 1, nz = r[5] - r[4] + 1;
    const long long nc = nx * ny * nz;
    for (long long j = threadIdx.x; j < nc; j += blockDim.x) {
      const int ix = r[0] + int(j % nx), iy = r[2] + int((j / nx) % ny), iz = r[4] + int(j / (nx * ny));
      const int64_t b = (int64_t(iz) * g.nc[1] + iy) * g.nc[0] + ix;
      if (FILL) entries[atomicAdd(&cursor[b], 1u)] = uint32_t(t);
      else atomicAdd(&cnt[b], 1u);
    }
  }
}

// ---------------------------------------------------------------------------
// pair predicates (exact reference arithmetic)
// ---------------------------------------------------------------------------

// The reference reports a sphere pair that passed the distance test only if
// the bin of the min corner mx of the two enlarged boxes' intersection lies in
// both spheres' registration ranges (_kernels.py:317-321).  The lower ends
// always hold (mx >= fl(c - r) and the bin map fl(fl(x - glo) * inv) with
// truncation and clamping is monotone).  If the boxes overlap in the same
// fp64 arithmetic, i.e. fl(c_j - r_j) <= fl(c_i + r_i) and
// fl(c_i - r_i) <= fl(c_j + r_j) on every axis, then mx <= both upper box
// ends and, by the same monotonicity, the upper ends hold too.  Only pairs
// whose boxes do not overlap in fp64 (possible only for ties at zero margin)
// need the full range evaluation.
__device__ __forceinline__ bool bstar_in_ranges(const Grid &g, const double ci[3], double ri, float ri_f,
                                                const double cj[3], double rj, float rj_f, double margin) {
  bool overlap = true;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax)
    overlap = overlap && sub_(cj[ax], rj) <= add(ci[ax], ri) && sub_(ci[ax], ri) <= add(cj[ax], rj);
  if (overlap) return true;
  long long lo_i[3], hi_i[3], lo_j[3], hi_j[3];
  sphere_range(g, ci, ri_f, margin, lo_i, hi_i);
  sphere_range(g, cj, rj_f, margin, lo_j, hi_j);
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    double m = fmax(sub_(ci[ax], ri), sub_(cj[ax], rj));
    long long b = axis_bin(m, g.glo[ax], g.inv_bin, g.nb[ax]);
    if (b < lo_i[ax] || b > hi_i[ax] || b < lo_j[ax] || b > hi_j[ax]) return false;
  }
  return true;
}

// collect_sphere_tri_pairs predicate (_kernels.py:375-401): distance test,
// reported once -- in the enumeration cell (fx, fy, fz) holding the min
// corner -- and only if the reference's dedup bin lies in both reference
// registration ranges
__device__ __forceinline__ bool st_pair(const KtView &v, const Grid &g, uint32_t t,
                                        const double ci[3], float ri_f, const long long lo_i[3],
                                        const long long hi_i[3], uint32_t oi, uint8_t fi,
                                        long long fx, long long fy, long long fz) {
  if (oi == v.tri_owner[t] || !dd_keep(v.own.dd, oi, v.tri_owner[t])) return false;
  if (!v.mask[256 * fi + v.tfam[t]]) return false;
  const double *T = v.tri_world + 9 * size_t(t);
  double qx, qy, qz;
  closest_on_tri(ci[0], ci[1], ci[2], T, qx, qy, qz);
  double dx = sub_(ci[0], qx), dy = sub_(ci[1], qy), dz = sub_(ci[2], qz);
  double rr = add(double(ri_f), v.margin);
  if (add(add(mul(dx, dx), mul(dy, dy)), mul(dz, dz)) >= mul(rr, rr)) return false;
  double m[3] = {sub_(ci[0], rr), sub_(ci[1], rr), sub_(ci[2], rr)};
  double tl[3] = {sub_(fmin(fmin(T[0], T[3]), T[6]), v.margin), sub_(fmin(fmin(T[1], T[4]), T[7]), v.margin),
                  sub_(fmin(fmin(T[2], T[5]), T[8]), v.margin)};
  long long f[3] = {fx, fy, fz};
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    if (tl[ax] > m[ax]) m[ax] = tl[ax];
    if (axis_bin(m[ax], g.glo[ax], g.inv_cell, g.nc[ax]) != f[ax]) return false;
  }
  // reference registration range of the triangle on the reference grid
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    double lo = T[ax], hi = T[ax];
    for (int q = 1; q < 3; ++q) {
      double x = T[3 * q + ax];
      if (x < lo) lo = x;
      if (x > hi) hi = x;
    }
    long long tlo = axis_bin(sub_(lo, v.margin), g.glo[ax], g.inv_bin, g.nb[ax]);
    long long thi = axis_bin(add(hi, v.margin), g.glo[ax], g.inv_bin, g.nb[ax]);
    long long b = axis_bin(m[ax], g.glo[ax], g.inv_bin, g.nb[ax]);
    if (b < lo_i[ax] || b > hi_i[ax] || b < tlo || b > thi) return false;
  }
  return true;
}

// collect_sphere_analytic_pairs predicate (_kernels.py:418-428)
__device__ __forceinline__ bool sa_pair(const KtView &v, uint32_t k, const double ci[3],
                                        float ri_f, uint32_t oi, uint8_t fi) {
  if (oi == v.ana_owner[k] || !dd_keep(v.own.dd, oi, v.ana_owner[k])) return false;
  if (!v.mask[256 * fi + v.afam[k]]) return false;
  double gap, bx, by, bz, rb;
  analytic_gap(v.ana_kind[k], v.ana_world + 8 * size_t(k), ci[0], ci[1], ci[2], gap, bx, by, bz, rb);
  return !(gap >= add(double(ri_f), v.margin));
}

__device__ __forceinline__ void sort_segment_y(uint2 *out, unsigned long long w, unsigned long long cnt) {
  for (unsigned long long p = 1; p < cnt; ++p) {
    uint2 e = out[w + p];
    unsigned long long q = p;
    while (q > 0 && out[w + q - 1].y > e.y) { out[w + q] = out[w + q - 1]; --q; }
    out[w + q] = e;
  }
}

// warp-aggregated append of one pair per active lane (all 32 lanes call it)
__device__ __forceinline__ void append_pair(bool hit, uint2 e, uint2 *tmp, unsigned long long *tmp_n,
                                            unsigned long long cap) {
  unsigned m = __ballot_sync(0xffffffffu, hit);
  if (!m) return;
  int lane = threadIdx.x & 31;
  int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(tmp_n, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (hit) {
    unsigned long long pos = base + __popc(m & ((1u << lane) - 1u));
    if (pos < cap) tmp[pos] = e;
  }
}

// cell-sorted copies of the snapshot spheres: (centre, radius), (slot, owner, family)
__global__ void k_gather_sorted(int64_t n, const uint32_t *sorted, const double *centers,
                                const float4 *offr, const uint32_t *owner, const uint8_t *sfam,
                                const Grid *gp, double4 *sc, uint4 *sm, float4 *sf) {
  int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (u >= n) return;
  uint32_t i = sorted[u];
  const double x = centers[4 * size_t(i)], y = centers[4 * size_t(i) + 1], z = centers[4 * size_t(i) + 2];
  sc[u] = make_double4(x, y, z, double(offr[i].w));
  sm[u] = make_uint4(i, owner[i], sfam[i], 0u);
  const Grid g = *gp;
  sf[u] = make_float4(float(x - g.glo[0]), float(y - g.glo[1]), float(z - g.glo[2]), offr[i].w);
}

// the exact predicate without the owner / family checks (done elsewhere)
__device__ __forceinline__ bool ss_pair_sorted_nomask(const KtView &v, const Grid &g, const double4 &cl,
                                                      const uint4 &ml, const double4 &ch, const uint4 &mh) {
  (void)ml; (void)mh;
  double dx = sub_(cl.x, ch.x), dy = sub_(cl.y, ch.y), dz = sub_(cl.z, ch.z);
  double ri = add(cl.w, v.margin);
  double rj = add(ch.w, v.margin);
  double rr = sub_(add(ri, rj), v.margin);
  if (add(add(mul(dx, dx), mul(dy, dy)), mul(dz, dz)) >= mul(rr, rr)) return false;
  double ci[3] = {cl.x, cl.y, cl.z}, cj[3] = {ch.x, ch.y, ch.z};
  return bstar_in_ranges(g, ci, ri, float(cl.w), cj, rj, float(ch.w), v.margin);
}

// Sphere-triangle and sphere-analytic pairs, one thread per sphere slot.
__global__ void __launch_bounds__(128) k_pairs_other(KtView v, unsigned long long *counts, uint2 *tmp,
                                                     unsigned long long *tmp_n, unsigned long long cap,
                                                     int do_ana) {
  int64_t i64 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t n = v.sph.n;
  const Grid g = *v.grid;
  const bool active = i64 < n && g.valid;
  uint32_t i = uint32_t(active ? i64 : 0);
  double ci[3] = {0, 0, 0};
  float ri_f = 0.f;
  uint32_t oi = 0;
  uint8_t fi = 0;
  long long lo_i[3] = {0, 0, 0}, hi_i[3] = {0, 0, 0};
  if (active) {
    ci[0] = v.centers[4 * i64]; ci[1] = v.centers[4 * i64 + 1]; ci[2] = v.centers[4 * i64 + 2];
    ri_f = v.sph.offr[i].w;
    oi = v.sph.owner[i];
    fi = v.sfam[i];
    if (v.n_tri) sphere_range(g, ci, ri_f, v.margin, lo_i, hi_i);   // only the triangle predicate needs it
  }
  unsigned long long cst = 0, csa = 0;
  if (v.n_tri && active) {
    const double rr = add(double(ri_f), v.margin);
    long long flo[3], fhi[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      flo[ax] = axis_bin(sub_(ci[ax], rr), g.glo[ax], g.inv_cell, g.nc[ax]);
      fhi[ax] = axis_bin(add(ci[ax], rr), g.glo[ax], g.inv_cell, g.nc[ax]);
    }
    for (long long z = flo[2]; z <= fhi[2]; ++z)
      for (long long y = flo[1]; y <= fhi[1]; ++y)
        for (long long x = flo[0]; x <= fhi[0]; ++x) {
          int64_t b = (z * g.nc[1] + y) * g.nc[0] + x;
          for (uint32_t u = v.tri_start[b]; u < v.tri_start[b + 1]; ++u) {
            uint32_t t = v.tri_entries[u];
            if (st_pair(v, g, t, ci, ri_f, lo_i, hi_i, oi, fi, x, y, z)) {
              unsigned long long pos = atomicAdd(tmp_n, 1ull);
              if (pos < cap) tmp[pos] = make_uint2(i, t | (1u << kKindShift));
              ++cst;
            }
          }
        }
  }
  // analytic list: warp-uniform loop (unless k_sa_filter takes the candidates)
  for (int64_t k = 0; do_ana && k < v.n_ana; ++k) {
    bool hit = active && sa_pair(v, uint32_t(k), ci, ri_f, oi, fi);
    if (hit) ++csa;
    append_pair(hit, make_uint2(i, uint32_t(k) | (2u << kKindShift)), tmp, tmp_n, cap);
  }
  if (active) {
    counts[n + i64] = cst;
    if (do_ana) counts[2 * n + i64] = csa;
  }
}

// Sphere-analytic candidates, built with the sphere-sphere lists while no
// mesh / analytic owner moves: analytic k is a candidate of sphere i if its
// gap is below r_i + margin + skin at the rebuild.  Gaps to planes and
// cylinders are 1-Lipschitz in the centre, so a sphere that moved at most
// skin / 2 since (k_disp) can only pass the exact test with a candidate.
// Families / masks are not applied (they may change); clump-mates and the
// decomposition rule are.
__device__ __forceinline__ bool sa_candidate(const KtView &v, uint32_t i, uint32_t k, double reach) {
  const uint32_t oi = v.sph.owner[i];
  if (oi == v.ana_owner[k] || !dd_keep(v.own.dd, oi, v.ana_owner[k])) return false;
  double gap, bx, by, bz, rb;
  analytic_gap(v.ana_kind[k], v.ana_world + 8 * size_t(k), v.centers[4 * size_t(i)], v.centers[4 * size_t(i) + 1],
               v.centers[4 * size_t(i) + 2], gap, bx, by, bz, rb);
  return gap < double(v.sph.offr[i].w) + reach;
}

__global__ void k_sa_count(KtView v, double reach_s, double reach_b, double r_cut, uint32_t *cnt) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= v.sph.n) return;
  const double reach = (r_cut > 0.0 && double(v.sph.offr[i].w) > r_cut) ? reach_b : reach_s;   // big: margin + Sb
  uint32_t c = 0;
  for (int64_t k = 0; k < v.n_ana; ++k) c += sa_candidate(v, uint32_t(i), uint32_t(k), reach) ? 1u : 0u;
  cnt[i] = c;
}

__global__ void k_sa_fill(KtView v, double reach_s, double reach_b, double r_cut, const unsigned long long *off,
                          uint2 *cand) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= v.sph.n) return;
  const double reach = (r_cut > 0.0 && double(v.sph.offr[i].w) > r_cut) ? reach_b : reach_s;
  unsigned long long w = off[i];
  for (int64_t k = 0; k < v.n_ana; ++k)
    if (sa_candidate(v, uint32_t(i), uint32_t(k), reach)) cand[w++] = make_uint2(uint32_t(i), uint32_t(k));
}

// exact sphere-analytic predicate (_kernels.py:418-428) on the candidates
__global__ void k_sa_filter(KtView v, const uint2 *cand, int64_t n_cand, unsigned long long *counts, uint2 *tmp,
                            unsigned long long *tmp_n, unsigned long long cap) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  bool hit = false;
  uint2 p = make_uint2(0u, 0u);
  if (e < n_cand && v.grid->valid) {
    p = cand[e];
    const double ci[3] = {v.centers[4 * size_t(p.x)], v.centers[4 * size_t(p.x) + 1], v.centers[4 * size_t(p.x) + 2]};
    hit = sa_pair(v, p.y, ci, v.sph.offr[p.x].w, v.sph.owner[p.x], v.sfam[p.x]);
    if (hit) atomicAdd(&counts[2 * v.sph.n + p.x], 1ull);
  }
  append_pair(hit, make_uint2(p.x, p.y | (2u << kKindShift)), tmp, tmp_n, cap);
}

// scatter the scratch list into per-(kind, sphere) segments
__global__ void k_place(const unsigned long long *m_p, int64_t n, const uint2 *tmp,
                        const unsigned long long *offsets, unsigned *cursor, uint2 *out) {
  const unsigned long long m = *m_p;
  for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < m;
       e += (unsigned long long)gridDim.x * blockDim.x) {
    uint2 p = tmp[e];
    int64_t seg = int64_t(p.y >> kKindShift) * n + p.x;
    out[offsets[seg] + atomicAdd(&cursor[seg], 1u)] = p;
  }
}

// canonical order inside every (kind, sphere) segment: ascending b
__global__ void k_sort_seg(int64_t nseg, const unsigned long long *offsets, uint2 *out) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nseg) return;
  unsigned long long w = offsets[i], cnt = offsets[i + 1] - w;
  if (cnt > 1) sort_segment_y(out, w, cnt);
}

// the same, with segments longer than kShortSeg (big spheres' candidates)
// left to k_sort_long: one CTA each, bitonic sort in shared memory
constexpr unsigned long long kShortSeg = 64;
constexpr int kLongSeg = 8192;   // longer: insertion sort fallback (correct, slow)
__global__ void k_sort_seg_short(int64_t nseg, const unsigned long long *offsets, uint2 *out, uint32_t *longs,
                                 unsigned long long *n_long) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nseg) return;
  unsigned long long w = offsets[i], cnt = offsets[i + 1] - w;
  if (cnt > kShortSeg) longs[atomicAdd(n_long, 1ull)] = uint32_t(i);
  else if (cnt > 1) sort_segment_y(out, w, cnt);
}

__global__ void __launch_bounds__(1024) k_sort_long(const unsigned long long *offsets, uint2 *out,
                                                    const uint32_t *longs, const unsigned long long *n_long) {
  extern __shared__ uint2 sh[];
  const unsigned long long nl = *n_long;
  for (unsigned long long li = blockIdx.x; li < nl; li += gridDim.x) {
    const uint32_t sg = longs[li];
    const unsigned long long w = offsets[sg], cnt = offsets[sg + 1] - w;
    if (cnt > (unsigned long long)kLongSeg) {
      if (threadIdx.x == 0) sort_segment_y(out, w, cnt);
      __syncthreads();
      continue;
    }
    int p2 = 1;
    while (p2 < int(cnt)) p2 <<= 1;
    for (int t = threadIdx.x; t < p2; t += blockDim.x)
      sh[t] = t < int(cnt) ? out[w + t] : make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
    __syncthreads();
    for (int size = 2; size <= p2; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = threadIdx.x; t < p2; t += blockDim.x) {
          const int u = t ^ stride;
          if (u > t) {
            const bool up = (t & size) == 0;
            const uint2 x = sh[t], y = sh[u];
            if ((x.y > y.y) == up) { sh[t] = y; sh[u] = x; }
          }
        }
        __syncthreads();
      }
    for (int t = threadIdx.x; t < int(cnt); t += blockDim.x) out[w + t] = sh[t];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Verlet candidate lists.  A rebuild enumerates every sphere-sphere pair
// within margin + skin (fp32 test with conservative slack, different owners;
// families / masks are NOT applied -- they may change between detections)
// into per-sphere candidate segments sorted by the partner slot.  Each
// detection then evaluates the exact reference predicate on the candidates
// only.  Exactness: a pair within the margin at a detection was within
// margin + skin at the rebuild if neither sphere moved more than skin / 2
// since, which k_disp checks before every detection.
// ---------------------------------------------------------------------------

// any sphere displaced more than skin / 2 since the rebuild -> flag
__global__ void k_disp(int64_t n, const double4 *c4, const double *ref, double lim2, double lim2_big, double r_cut,
                       int *flag) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  bool far = false;
  if (i < n) {
    const double4 c = c4[i];
    double dx = c.x - ref[3 * i], dy = c.y - ref[3 * i + 1], dz = c.z - ref[3 * i + 2];
    far = dx * dx + dy * dy + dz * dz > ((r_cut > 0.0 && c.w > r_cut) ? lim2_big : lim2);
  }
  if (__any_sync(0xffffffffu, far) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// candidate pairs among small spheres: half stencil on the enumeration grid
// (cell = 2 (r_cut + margin + skin)), one thread per cell-sorted sphere.
// Two passes over the same loops, no shared counters: kFill = false counts
// each thread's hits, kFill = true writes them as (a, b) (a = lower slot) at
// the thread's exclusive-scan offset; a sort by a and a per-segment sort by b
// then give the (a, b)-ordered list.
template <bool kFill>
__global__ void __launch_bounds__(128) k_cand_ss(KtView v, const uint4 *sm, const float4 *sf, double reach_m,
                                                 uint32_t *ucnt, const unsigned long long *uoff,
                                                 uint32_t *ka, uint32_t *kb, unsigned long long cap = 0,
                                                 unsigned long long *ovf = nullptr) {
  int64_t u64 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (u64 >= v.sph.n) return;
  const Grid g = *v.grid;
  bool active = g.valid;
  uint32_t key = active ? v.bin_key[u64] : kNoCell;
  active = active && key != kNoCell;
  const float ext = float(double(max(g.nc[0], max(g.nc[1], g.nc[2]))) / g.inv_cell);
  const float slack = 1e-6f * ext + 1e-30f;
  const float marg = float(reach_m);
  uint32_t hits = 0;
  unsigned long long w_out = kFill ? uoff[u64] : 0ull;
  if (active) {
    const float4 f0 = sf[u64];
    const uint4 m0 = sm[u64];
    const long long cx = key % g.nc[0], cy = (key / g.nc[0]) % g.nc[1], cz = key / (g.nc[0] * g.nc[1]);
    for (int span = 0; span < 6; ++span) {
      uint32_t s0 = 0, s1 = 0;
      if (span == 0) {
        s0 = uint32_t(u64) + 1;
        s1 = v.cell_end[key];
      } else {
        long long dz = span >= 3 ? 1 : 0;
        long long dy = span == 2 ? 1 : (span >= 3 ? span - 4 : 0);
        long long x0 = span == 1 ? cx + 1 : cx - 1, x1 = cx + 1;
        long long y = cy + dy, z = cz + dz;
        if (x0 < 0) x0 = 0;
        if (x1 >= g.nc[0]) x1 = g.nc[0] - 1;
        if (y >= 0 && y < g.nc[1] && z < g.nc[2] && x0 <= x1) {
          long long row = (z * g.nc[1] + y) * g.nc[0];
          uint32_t a0 = 0xFFFFFFFFu;
          for (long long x = x0; x <= x1; ++x) {
            uint32_t st = v.cell_start[row + x];
            if (st == 0xFFFFFFFFu) continue;
            if (a0 == 0xFFFFFFFFu) a0 = st;
            s1 = v.cell_end[row + x];
          }
          s0 = a0 == 0xFFFFFFFFu ? 0 : a0;
          if (a0 == 0xFFFFFFFFu) s1 = 0;
        }
      }
      for (uint32_t w = s0; w < s1; ++w) {
        const float4 f1 = sf[w];
        const float dx = f0.x - f1.x, dy = f0.y - f1.y, dz = f0.z - f1.z;
        const float rr = f0.w + f1.w + marg + slack;
        if (dx * dx + dy * dy + dz * dz < rr * rr * 1.0001f) {
          const uint4 m1 = sm[w];
          if (m1.y != m0.y && dd_keep(v.own.dd, m0.y, m1.y)) {
            if (kFill) {
              if (w_out < cap) {
                ka[w_out] = min(m0.x, m1.x);
                kb[w_out] = max(m0.x, m1.x);
              } else {
                atomicAdd(ovf, 1ull);   // the count pass disagreed: reported, never written
              }
              ++w_out;
            }
            ++hits;
          }
        }
      }
    }
  }
  if (!kFill) ucnt[u64] = hits;
}

// candidate pairs involving big spheres (fp64 distance < r_i + r_j + M)
// Big spheres carry their own, larger skin Sb (Ctx::skin_big_factor): a big
// sphere may move Sb - S/2 before it forces a rebuild (a small one S/2), so
// big-small pairs are enumerated within margin + Sb and big-big pairs within
// margin + 2 Sb - S -- the sum of the two displacement limits in each case.
__global__ void __launch_bounds__(128) k_cand_big(KtView v, const uint32_t *bigs, int64_t n_big,
                                                  const double4 *sc, const uint4 *sm, double reach_m,
                                                  double reach_bb, uint32_t *ka, uint32_t *kb,
                                                  unsigned long long *big_n, unsigned long long cap) {
  const Grid g = *v.grid;
  if (!g.valid) return;
  for (int64_t bi = blockIdx.x; bi < n_big; bi += gridDim.x) {
    const uint32_t B = bigs[bi];
    const double bx = v.centers[4 * size_t(B)], by = v.centers[4 * size_t(B) + 1], bz = v.centers[4 * size_t(B) + 2];
    const double rB = double(v.sph.offr[B].w);
    const uint32_t oB = v.sph.owner[B];
    const double reach = rB + g.r_cut + reach_m;
    const double cbv[3] = {bx, by, bz};
    long long flo[3], fhi[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      flo[ax] = axis_bin(cbv[ax] - reach, g.glo[ax], g.inv_cell, g.nc[ax]);
      fhi[ax] = axis_bin(cbv[ax] + reach, g.glo[ax], g.inv_cell, g.nc[ax]);
    }
    const long long sx = fhi[0] - flo[0] + 1, sy = fhi[1] - flo[1] + 1, sz = fhi[2] - flo[2] + 1;
    const long long ncell = sx * sy * sz;
    for (long long q = threadIdx.x; q < ncell; q += blockDim.x) {
      long long x = flo[0] + q % sx, y = flo[1] + (q / sx) % sy, z = flo[2] + q / (sx * sy);
      long long b = (z * g.nc[1] + y) * g.nc[0] + x;
      uint32_t s0 = v.cell_start[b];
      if (s0 == 0xFFFFFFFFu) continue;
      uint32_t s1 = v.cell_end[b];
      for (uint32_t w = s0; w < s1; ++w) {
        const double4 c1 = sc[w];
        const uint4 m1 = sm[w];
        if (m1.y == oB || !dd_keep(v.own.dd, m1.y, oB)) continue;
        const double dx = bx - c1.x, dy = by - c1.y, dz = bz - c1.z;
        const double rr = rB + c1.w + reach_m;
        if (dx * dx + dy * dy + dz * dz >= rr * rr * (1.0 + 1e-9)) continue;
        const uint32_t a = min(m1.x, B), c = max(m1.x, B);
        const unsigned long long pos = atomicAdd(big_n, 1ull);
        if (pos < cap) { ka[pos] = a; kb[pos] = c; }
      }
    }
    for (int64_t q = threadIdx.x; q < n_big; q += blockDim.x) {
      const uint32_t j = bigs[q];
      if (j <= B || v.sph.owner[j] == oB || !dd_keep(v.own.dd, v.sph.owner[j], oB)) continue;
      const double dx = bx - v.centers[4 * size_t(j)], dy = by - v.centers[4 * size_t(j) + 1],
                   dz = bz - v.centers[4 * size_t(j) + 2];
      const double rr = rB + double(v.sph.offr[j].w) + reach_bb;
      if (dx * dx + dy * dy + dz * dz >= rr * rr * (1.0 + 1e-9)) continue;
      const unsigned long long pos = atomicAdd(big_n, 1ull);
      if (pos < cap) { ka[pos] = B; kb[pos] = j; }
    }
  }
}

// The same pairs grouped by their lower slot without a pair sort (the
// default rebuild, Ctx::rb_slot).  kFill = false counts every slot's pairs:
// hits whose lower slot is the thread's own sphere are summed in a register
// (kept per thread in `own`), the others add one to the partner's counter.
// After an exclusive scan over slots (the segment starts), kFill = true
// reserves the thread's own run with one atomic on its slot's cursor and
// places every other hit at its partner's segment start + that slot's
// cursor.  The order inside a segment is the per-segment sort by b's.
// a fill-pass store guarded by the capacity the count pass sized: a pair the
// count did not see is counted in *ovf (the host fails the rebuild loudly)
// instead of being written past the list
__device__ __forceinline__ void cand_put(uint2 *cand, unsigned long long i, uint2 p, unsigned long long cap,
                                         unsigned long long *ovf) {
  if (i < cap) cand[i] = p;
  else atomicAdd(ovf, 1ull);
}

template <bool kFill>
__global__ void __launch_bounds__(128) k_cand_slot(KtView v, const uint4 *sm, const float4 *sf, double reach_m,
                                                   uint32_t *scnt, uint32_t *own, const unsigned long long *seg,
                                                   uint32_t *cursor, uint2 *cand, unsigned long long cap = 0,
                                                   unsigned long long *ovf = nullptr) {
  int64_t u64 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (u64 >= v.sph.n) return;
  const Grid g = *v.grid;
  bool active = g.valid;
  uint32_t key = active ? v.bin_key[u64] : kNoCell;
  active = active && key != kNoCell;
  const float ext = float(double(max(g.nc[0], max(g.nc[1], g.nc[2]))) / g.inv_cell);
  const float slack = 1e-6f * ext + 1e-30f;
  const float marg = float(reach_m);
  uint32_t mine = 0;
  unsigned long long w_own = 0;
  if (active) {
    const float4 f0 = sf[u64];
    const uint4 m0 = sm[u64];
    if (kFill) {
      const uint32_t n_own = own[u64];
      if (n_own) w_own = seg[m0.x] + atomicAdd(cursor + m0.x, n_own);
    }
    const long long cx = key % g.nc[0], cy = (key / g.nc[0]) % g.nc[1], cz = key / (g.nc[0] * g.nc[1]);
    for (int span = 0; span < 6; ++span) {
      uint32_t s0 = 0, s1 = 0;
      if (span == 0) {
        s0 = uint32_t(u64) + 1;
        s1 = v.cell_end[key];
      } else {
        long long dz = span >= 3 ? 1 : 0;
        long long dy = span == 2 ? 1 : (span >= 3 ? span - 4 : 0);
        long long x0 = span == 1 ? cx + 1 : cx - 1, x1 = cx + 1;
        long long y = cy + dy, z = cz + dz;
        if (x0 < 0) x0 = 0;
        if (x1 >= g.nc[0]) x1 = g.nc[0] - 1;
        if (y >= 0 && y < g.nc[1] && z < g.nc[2] && x0 <= x1) {
          long long row = (z * g.nc[1] + y) * g.nc[0];
          uint32_t a0 = 0xFFFFFFFFu;
          for (long long x = x0; x <= x1; ++x) {
            uint32_t st = v.cell_start[row + x];
            if (st == 0xFFFFFFFFu) continue;
            if (a0 == 0xFFFFFFFFu) a0 = st;
            s1 = v.cell_end[row + x];
          }
          s0 = a0 == 0xFFFFFFFFu ? 0 : a0;
          if (a0 == 0xFFFFFFFFu) s1 = 0;
        }
      }
      for (uint32_t w = s0; w < s1; ++w) {
        const float4 f1 = sf[w];
        const float dx = f0.x - f1.x, dy = f0.y - f1.y, dz = f0.z - f1.z;
        const float rr = f0.w + f1.w + marg + slack;
        if (dx * dx + dy * dy + dz * dz < rr * rr * 1.0001f) {
          const uint4 m1 = sm[w];
          if (m1.y != m0.y && dd_keep(v.own.dd, m0.y, m1.y)) {
            if (m0.x < m1.x) {
              if (kFill) cand_put(cand, w_own + mine, make_uint2(m0.x, m1.x), cap, ovf);
              ++mine;
            } else if (kFill) {
              cand_put(cand, seg[m1.x] + atomicAdd(cursor + m1.x, 1u), make_uint2(m1.x, m0.x), cap, ovf);
            } else {
              atomicAdd(scnt + m1.x, 1u);
            }
          }
        }
      }
    }
    if (!kFill && mine) atomicAdd(scnt + m0.x, mine);
  }
  if (!kFill) own[u64] = mine;
}

// big-sphere pairs into the slot-grouped list (k_cand_big's enumeration)
template <bool kFill>
__global__ void __launch_bounds__(128) k_cand_big_slot(KtView v, const uint32_t *bigs, int64_t n_big,
                                                       const double4 *sc, const uint4 *sm, double reach_m,
                                                       double reach_bb, uint32_t *scnt,
                                                       const unsigned long long *seg, uint32_t *cursor,
                                                       uint2 *cand, unsigned long long cap = 0,
                                                       unsigned long long *ovf = nullptr) {
  const Grid g = *v.grid;
  if (!g.valid) return;
  for (int64_t bi = blockIdx.x; bi < n_big; bi += gridDim.x) {
    const uint32_t B = bigs[bi];
    const double bx = v.centers[4 * size_t(B)], by = v.centers[4 * size_t(B) + 1], bz = v.centers[4 * size_t(B) + 2];
    const double rB = double(v.sph.offr[B].w);
    const uint32_t oB = v.sph.owner[B];
    const double reach = rB + g.r_cut + reach_m;
    const double cbv[3] = {bx, by, bz};
    long long flo[3], fhi[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      flo[ax] = axis_bin(cbv[ax] - reach, g.glo[ax], g.inv_cell, g.nc[ax]);
      fhi[ax] = axis_bin(cbv[ax] + reach, g.glo[ax], g.inv_cell, g.nc[ax]);
    }
    const long long sx = fhi[0] - flo[0] + 1, sy = fhi[1] - flo[1] + 1, sz = fhi[2] - flo[2] + 1;
    const long long ncell = sx * sy * sz;
    for (long long q = threadIdx.x; q < ncell; q += blockDim.x) {
      long long x = flo[0] + q % sx, y = flo[1] + (q / sx) % sy, z = flo[2] + q / (sx * sy);
      long long b = (z * g.nc[1] + y) * g.nc[0] + x;
      uint32_t s0 = v.cell_start[b];
      if (s0 == 0xFFFFFFFFu) continue;
      uint32_t s1 = v.cell_end[b];
      for (uint32_t w = s0; w < s1; ++w) {
        const double4 c1 = sc[w];
        const uint4 m1 = sm[w];
        if (m1.y == oB || !dd_keep(v.own.dd, m1.y, oB)) continue;
        const double dx = bx - c1.x, dy = by - c1.y, dz = bz - c1.z;
        const double rr = rB + c1.w + reach_m;
        if (dx * dx + dy * dy + dz * dz >= rr * rr * (1.0 + 1e-9)) continue;
        const uint32_t a = min(m1.x, B), c = max(m1.x, B);
        if (kFill) cand_put(cand, seg[a] + atomicAdd(cursor + a, 1u), make_uint2(a, c), cap, ovf);
        else atomicAdd(scnt + a, 1u);
      }
    }
    for (int64_t q = threadIdx.x; q < n_big; q += blockDim.x) {
      const uint32_t j = bigs[q];
      if (j <= B || v.sph.owner[j] == oB || !dd_keep(v.own.dd, v.sph.owner[j], oB)) continue;
      const double dx = bx - v.centers[4 * size_t(j)], dy = by - v.centers[4 * size_t(j) + 1],
                   dz = bz - v.centers[4 * size_t(j) + 2];
      const double rr = rB + double(v.sph.offr[j].w) + reach_bb;
      if (dx * dx + dy * dy + dz * dz >= rr * rr * (1.0 + 1e-9)) continue;
      if (kFill) cand_put(cand, seg[B] + atomicAdd(cursor + B, 1u), make_uint2(B, j), cap, ovf);
      else atomicAdd(scnt + B, 1u);
    }
  }
}

// candidates sorted by a -> the (a, b) list and each sphere's segment start
// (the spheres in (previous entry's a, this entry's a] start here)
// Segment-start fills over runs of spheres without entries: a thread fills
// short runs itself and hands runs longer than kGapInline to k_fill_gaps (one
// CTA per run), so a sparse list (a settling terrain, a dilute scene) does not
// leave single threads looping over millions of spheres.
constexpr long long kGapInline = 32;
struct GapList {
  ulonglong2 *run;              // (first sphere | last sphere << 32 folded in .x / .y), value in val
  unsigned long long *val;
  unsigned long long *n;
  unsigned long long cap;
};
__device__ __forceinline__ void seg_fill(unsigned long long *seg, long long lo, long long hi, unsigned long long val,
                                         const GapList &gl) {
  if (hi - lo + 1 <= kGapInline || gl.n == nullptr) {
    for (long long sp = lo; sp <= hi; ++sp) seg[sp] = val;
    return;
  }
  const unsigned long long i = atomicAdd(gl.n, 1ull);
  if (i < gl.cap) {
    gl.run[i] = make_ulonglong2((unsigned long long)lo, (unsigned long long)hi);
    gl.val[i] = val;
  } else {   // cannot happen with cap >= n_sph / kGapInline + 2; stay correct anyway
    for (long long sp = lo; sp <= hi; ++sp) seg[sp] = val;
  }
}

__global__ void k_fill_gaps(unsigned long long *seg, GapList gl) {
  const unsigned long long n = min(*gl.n, gl.cap);
  for (unsigned long long g = blockIdx.x; g < n; g += gridDim.x) {
    const ulonglong2 r = gl.run[g];
    const unsigned long long v = gl.val[g];
    for (unsigned long long sp = r.x + threadIdx.x; sp <= r.y; sp += blockDim.x) seg[sp] = v;
  }
}

__global__ void k_cand_unpack(int64_t total, int64_t n_sph, const uint32_t *ka, const uint32_t *kb, uint2 *cand,
                              unsigned long long *seg, GapList gl) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t a = ka[e];
    cand[e] = make_uint2(uint32_t(a), kb[e]);
    const int64_t ap = e > 0 ? int64_t(ka[e - 1]) : -1;
    if (ap + 1 <= a) seg_fill(seg, ap + 1, a, (unsigned long long)e, gl);
    if (e == total - 1 && a + 1 <= n_sph) seg_fill(seg, a + 1, n_sph, (unsigned long long)total, gl);
  }
}


// Sphere-sphere block of a detection in two coalesced passes over the
// candidate list (sorted by (a, b)):
//   k_filter_bits  the exact reference predicate per candidate; hits as a
//                  bitmask (one word per warp) plus a count per 256-candidate
//                  block (then scanned);
//   k_compact      the hits' rows from the scanned counts and the bitmask:
//                  writes the canonical sphere-sphere block, its per-sphere
//                  segment starts (the spheres in (previous candidate's
//                  sphere, this candidate's sphere] start at this row) and --
//                  when the previous filtered array came from the same
//                  candidate list -- each hit's row in that array (old_pos,
//                  from that array's bitmask and counts), which makes the
//                  history remap at adoption a plain gather.
constexpr int kFcBlock = 256;

// kFcPer candidates per thread (item q of lane l in warp w is candidate
// block_base + w * 32 * kFcPer + q * 32 + l: one bitmask word per (warp, q))
// so their record gathers are in flight together
#ifndef GF_FC_PER
#define GF_FC_PER 2
#endif
constexpr int kFcPer = GF_FC_PER;
constexpr int kFcSpan = kFcBlock * kFcPer;   // candidates per filter block

__global__ void __launch_bounds__(kFcBlock) k_filter_bits(KtView v, const uint2 *cand, int64_t n_cand,
                                                          uint32_t *bits, uint32_t *blk_cnt) {
  __shared__ uint32_t s_cnt[kFcBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t e0 = blockIdx.x * int64_t(kFcSpan) + warp * 32 * kFcPer + lane;
  const Grid g = *v.grid;
  uint2 p[kFcPer];
  double4 ci4[kFcPer], cj4[kFcPer];
#pragma unroll
  for (int q = 0; q < kFcPer; ++q) p[q] = e0 + 32 * q < n_cand ? cand[e0 + 32 * q] : make_uint2(0u, 0u);
#pragma unroll
  for (int q = 0; q < kFcPer; ++q) {
    if (e0 + 32 * q < n_cand) {
      ci4[q] = ld256(v.c4 + p[q].x);
      cj4[q] = ld256(v.c4 + p[q].y);
    }
  }
  uint32_t cnt = 0;
#pragma unroll
  for (int q = 0; q < kFcPer; ++q) {
    const int64_t e = e0 + 32 * q;
    bool hit = false;
    if (e < n_cand && g.valid) {
      hit = v.mask_trivial || v.mask[256 * v.sfam[p[q].x] + v.sfam[p[q].y]] != 0;
      if (hit) {
        const uint4 mi = make_uint4(p[q].x, 0u, 0u, 0u), mj = make_uint4(p[q].y, 1u, 0u, 0u);
        const double4 cl = make_double4(ci4[q].x, ci4[q].y, ci4[q].z, double(float(ci4[q].w)));
        const double4 ch = make_double4(cj4[q].x, cj4[q].y, cj4[q].z, double(float(cj4[q].w)));
        hit = ss_pair_sorted_nomask(v, g, cl, mi, ch, mj);
      }
    }
    const uint32_t word = __ballot_sync(0xffffffffu, hit);
    if (lane == 0 && e < n_cand) bits[e >> 5] = word;
    cnt += __popc(word);
  }
  if (lane == 0) s_cnt[warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < kFcBlock / 32; ++w) t += s_cnt[w];
    blk_cnt[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kFcBlock) k_compact(KtView v, const uint2 *cand, int64_t n_cand,
                                                      const uint32_t *bits, const unsigned long long *blk_pre,
                                                      const uint32_t *obits, const unsigned long long *oblk_pre,
                                                      uint2 *out_ids, unsigned long long *seg, uint32_t *old_pos,
                                                      unsigned long long ss_cap, GapList gl) {
  // the filter block's kFcSpan candidates: kFcSpan / 32 bitmask words; every
  // global load is issued up front so its latency overlaps the word scan
  constexpr int kW = kFcSpan / 32;
  __shared__ uint32_t s_w[kW], s_ow[kW];
  const int64_t w_base = blockIdx.x * int64_t(kW);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long pre = blk_pre[blockIdx.x];
  const unsigned long long opre = obits ? oblk_pre[blockIdx.x] : 0ull;
  uint2 it[kFcPer];
  uint32_t word[kFcPer], oword[kFcPer], ap_g[kFcPer];
#pragma unroll
  for (int q = 0; q < kFcPer; ++q) {
    const int wl = warp + q * (kFcBlock / 32);   // word within the block
    const int64_t e = (w_base + wl) * 32 + lane;
    const bool in = e < n_cand;
    it[q] = in ? cand[e] : make_uint2(0u, 0u);
    ap_g[q] = (in && lane == 0 && e > 0) ? cand[e - 1].x : 0u;
    word[q] = in ? bits[w_base + wl] : 0u;
    oword[q] = (in && obits) ? obits[w_base + wl] : 0u;
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < kFcPer; ++q) {
      const int wl = warp + q * (kFcBlock / 32);
      s_w[wl] = __popc(word[q]);
      s_ow[wl] = __popc(oword[q]);
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {   // exclusive scan of the word counts (kW <= 32)
    const int l = threadIdx.x;
    const uint32_t x0 = l < kW ? s_w[l] : 0u, y0 = l < kW ? s_ow[l] : 0u;
    uint32_t x = x0, y = y0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t xo = __shfl_up_sync(0xffffffffu, x, off), yo = __shfl_up_sync(0xffffffffu, y, off);
      if (l >= off) { x += xo; y += yo; }
    }
    __syncwarp();
    if (l < kW) { s_w[l] = x - x0; s_ow[l] = y - y0; }
  }
  __syncthreads();
  const uint32_t below = (1u << lane) - 1u;
#pragma unroll
  for (int q = 0; q < kFcPer; ++q) {
    const int wl = warp + q * (kFcBlock / 32);
    const int64_t e = (w_base + wl) * 32 + lane;
    const uint32_t prev_x = __shfl_up_sync(0xffffffffu, it[q].x, 1);
    if (e >= n_cand) continue;
    const unsigned long long p = pre + s_w[wl] + __popc(word[q] & below);
    const long long a = (long long)it[q].x;
    const long long ap = e == 0 ? -1 : (long long)(lane ? prev_x : ap_g[q]);
    if (ap + 1 <= a) seg_fill(seg, ap + 1, a, p, gl);
    const bool hit = (word[q] >> lane) & 1u;
    if (hit && p < ss_cap) {   // beyond: the fill phase grows the array and recounts
      out_ids[p] = it[q];
      if (obits)
        old_pos[p] = ((oword[q] >> lane) & 1u) ? uint32_t(opre + s_ow[wl] + __popc(oword[q] & below))
                                              : 0xFFFFFFFFu;
    }
    if (e == n_cand - 1)   // the last candidate closes the block
      if (a + 1 <= v.sph.n) seg_fill(seg, a + 1, v.sph.n, p + (hit ? 1 : 0), gl);
  }
}


__global__ void k_copy_ref(int64_t n, const double4 *c4, double *ref) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double4 c = c4[i];
  ref[3 * i] = c.x;
  ref[3 * i + 1] = c.y;
  ref[3 * i + 2] = c.z;
}

__global__ void k_fill_u32(const Grid *gp, uint32_t *a, uint32_t value, int fine_plus_one) {
  Grid g = *gp;
  int64_t n = g.nc[0] * g.nc[1] * g.nc[2] + fine_plus_one;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    a[i] = value;
}

__global__ void k_bin_ranges(int64_t n, const double *centers, const float4 *offr, const Grid *gp,
                             double margin, long long *out) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  Grid g = *gp;
  double c[3] = {centers[4 * i], centers[4 * i + 1], centers[4 * i + 2]};
  long long lo[3], hi[3];
  sphere_range(g, c, offr[i].w, margin, lo, hi);
  for (int ax = 0; ax < 3; ++ax) {
    out[6 * i + 2 * ax] = lo[ax];
    out[6 * i + 2 * ax + 1] = hi[ax];
  }
}

// ---------------------------------------------------------------------------
// handoff: history remap (broadphase.py:110-135) + incidence lists
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long acs_key(uint2 id) {
  return (static_cast<unsigned long long>(id.y >> kKindShift) << 62) |
         (static_cast<unsigned long long>(id.x) << 31) |
         static_cast<unsigned long long>(id.y & kSlotMask);
}

__global__ void k_merge(int64_t n_new, const uint2 *new_ids, float *new_wild, int64_t n_old,
                        const uint2 *old_ids, const float *old_wild, int W) {
  int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= n_new) return;
  unsigned long long key = acs_key(new_ids[k]);
  int64_t lo = 0, hi = n_old;  // lower_bound
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (acs_key(old_ids[mid]) < key) lo = mid + 1; else hi = mid;
  }
  bool hit = lo < n_old && acs_key(old_ids[lo]) == key;
  for (int q = 0; q < W; ++q) new_wild[int64_t(W) * k + q] = hit ? old_wild[int64_t(W) * lo + q] : 0.0f;
}

// history remap using the old array's per-(kind, sphere) segments: the old
// row of a new pair can only sit in the segment of the same (kind, a)
__global__ void k_merge_seg(int64_t n_new, const uint2 *new_ids, float *new_wild, const uint2 *old_ids,
                            const float *old_wild, const unsigned long long *old_seg, int64_t n_sph,
                            int W) {
  int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= n_new) return;
  const uint2 id = new_ids[k];
  const int64_t seg = int64_t(id.y >> kKindShift) * n_sph + id.x;
  const unsigned long long lo = old_seg[seg], hi = old_seg[seg + 1];
  long long hit = -1;
  for (unsigned long long q = lo; q < hi; ++q) {
    uint32_t y = old_ids[q].y;
    if (y == id.y) { hit = (long long)q; break; }
    if (y > id.y) break;
  }
  if (W == 4) {
    reinterpret_cast<float4 *>(new_wild)[k] =
        hit >= 0 ? reinterpret_cast<const float4 *>(old_wild)[hit] : make_float4(0.f, 0.f, 0.f, 0.f);
  } else {
    for (int q = 0; q < W; ++q) new_wild[int64_t(W) * k + q] = hit >= 0 ? old_wild[int64_t(W) * hit + q] : 0.0f;
  }
}

// history remap at adoption when both arrays were filtered from the same
// candidate list: sphere-sphere rows gather their old row directly (old_pos),
// the wall kinds search their old (kind, a) segment like k_merge_seg
__device__ __forceinline__ long long adopt_wall_hit(const uint2 *new_ids, const uint2 *old_ids,
                                                    const unsigned long long *old_seg, int64_t n_sph, int64_t k) {
  const uint2 id = new_ids[k];
  const int64_t sg = int64_t(id.y >> kKindShift) * n_sph + id.x;
  const unsigned long long lo = old_seg[sg], hi = old_seg[sg + 1];
  for (unsigned long long q = lo; q < hi; ++q) {
    const uint32_t y = old_ids[q].y;
    if (y == id.y) return (long long)q;
    if (y > id.y) break;
  }
  return -1;
}

constexpr int kAdoptPer = 2;   // rows per thread: their gathers are in flight together

__global__ void k_adopt_hist(int64_t n_new, const uint2 *new_ids, const uint32_t *old_pos,
                             const unsigned long long *new_seg, float *new_wild, const uint2 *old_ids,
                             const float *old_wild, const unsigned long long *old_seg, int64_t n_sph, int W) {
  const int64_t k0 = blockIdx.x * int64_t(blockDim.x) * kAdoptPer + threadIdx.x;
  const unsigned long long n_ss = new_seg[n_sph];
  uint32_t q[kAdoptPer];
#pragma unroll
  for (int j = 0; j < kAdoptPer; ++j) {
    const int64_t k = k0 + int64_t(j) * blockDim.x;
    q[j] = (k < n_new && (unsigned long long)k < n_ss) ? old_pos[k] : 0xFFFFFFFFu;   // sphere-sphere rows only
  }
  long long hit[kAdoptPer];
#pragma unroll
  for (int j = 0; j < kAdoptPer; ++j) {
    const int64_t k = k0 + int64_t(j) * blockDim.x;
    hit[j] = -1;
    if (k >= n_new) continue;
    if ((unsigned long long)k < n_ss) hit[j] = q[j] != 0xFFFFFFFFu ? (long long)q[j] : -1;
    else hit[j] = adopt_wall_hit(new_ids, old_ids, old_seg, n_sph, k);
  }
  if (W == 4) {
    float4 w[kAdoptPer];
#pragma unroll
    for (int j = 0; j < kAdoptPer; ++j)
      w[j] = hit[j] >= 0 ? reinterpret_cast<const float4 *>(old_wild)[hit[j]] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < kAdoptPer; ++j) {
      const int64_t k = k0 + int64_t(j) * blockDim.x;
      if (k < n_new) reinterpret_cast<float4 *>(new_wild)[k] = w[j];
    }
  } else {
#pragma unroll
    for (int j = 0; j < kAdoptPer; ++j) {
      const int64_t k = k0 + int64_t(j) * blockDim.x;
      if (k >= n_new) continue;
      for (int c = 0; c < W; ++c) new_wild[int64_t(W) * k + c] = hit[j] >= 0 ? old_wild[int64_t(W) * hit[j] + c] : 0.0f;
    }
  }
}

__global__ void k_seg_count(int64_t n, const uint2 *ids, int64_t n_sph, unsigned long long *cnt) {
  int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  uint2 id = ids[k];
  atomicAdd(&cnt[int64_t(id.y >> kKindShift) * n_sph + id.x], 1ull);
}

// B-side incidences only: the A side of every owner is the contiguous run of
// its spheres' (kind, sphere) segments and needs no list
__global__ void k_inc_keys(int64_t n, const uint2 *ids, const uint32_t *sph_owner,
                           const uint32_t *tri_owner, const uint32_t *ana_owner, uint32_t *key,
                           uint32_t *val) {
  int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  uint2 id = ids[k];
  uint32_t kind = id.y >> kKindShift, sb = id.y & kSlotMask;
  key[k] = kind == 0 ? sph_owner[sb] : (kind == 1 ? tri_owner[sb] : ana_owner[sb]);
  val[k] = uint32_t(k);
}

// per-owner start of its B list; heavy owners (A + B incidences above the
// threshold) are collected for the block reduction
__global__ void k_inc_start(int64_t n_owner, int64_t n_inc, const uint32_t *sorted_key,
                            uint32_t *start, const unsigned long long *seg, const uint32_t *first,
                            int64_t n_sph, uint32_t *heavy, unsigned long long *n_heavy,
                            uint32_t heavy_threshold) {
  int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (o > n_owner) return;
  int64_t lo = 0, hi = n_inc;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (sorted_key[mid] < uint32_t(o)) lo = mid + 1; else hi = mid;
  }
  start[o] = uint32_t(lo);
  if (o < n_owner) {
    int64_t lo2 = lo, hi2 = n_inc;
    while (lo2 < hi2) {
      int64_t mid = (lo2 + hi2) >> 1;
      if (sorted_key[mid] <= uint32_t(o)) lo2 = mid + 1; else hi2 = mid;
    }
    unsigned long long na = 0;
    const uint32_t f0 = first[o], f1 = first[o + 1];
    if (f1 > f0)
      for (int kind = 0; kind < 3; ++kind) na += seg[kind * n_sph + f1] - seg[kind * n_sph + f0];
    if ((unsigned long long)(lo2 - lo) + na > heavy_threshold) {
      unsigned long long slot = atomicAdd(n_heavy, 1ull);
      heavy[slot] = uint32_t(o);
    }
  }
}

}  // namespace

// ===========================================================================
// host entry points
// ===========================================================================

__global__ void k_set_int(int *p, int v) { *p = v; }

// memset of possibly-peer memory from a stream of another device
__global__ void k_zero_u64(unsigned long long *p, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = 0ull;
}

int kt_snapshot(Ctx *c, cudaStream_t s, double margin) {
  KtScratch &k = c->kt;
  DevGuard gs(stream_device(s));   // launched on the stream's device (the dT one in a run)
  {
    // the snapshot lives with the rest of the kT scratch (the kT device of a
    // 2-GPU split: the snapshot kernel stores it over NVLink)
    DevGuard ga(c->kt_device);
    if (ensure(c, k.c4, sizeof(double4) * (c->n_sph + 1), s))
      return -1;
    if (ensure(c, k.sfam, c->n_sph + 1, s)) return -1;
    if (ensure(c, k.tri_world, sizeof(double) * 9 * (c->n_tri + 1), s)) return -1;
    if (ensure(c, k.ana_world, sizeof(double) * 8 * (c->n_ana + 1), s)) return -1;
    if (ensure(c, k.tfam, c->n_tri + 1, s)) return -1;
    if (ensure(c, k.afam, c->n_ana + 1, s)) return -1;
    if (ensure(c, k.minmax, sizeof(unsigned long long) * 8, s) || ensure(c, k.flag, 16, s)) return -1;
  }
  // a detection snapshot (margin >= 0) also reduces the grid inputs and runs
  // the candidate displacement check (kt_begin then skips both)
  static const bool fuse_off = std::getenv("GF_NO_SNAP_FUSE") != nullptr;
  const bool det = margin >= 0.0 && !fuse_off;
  unsigned long long *mm = k.minmax.as<unsigned long long>();
  bool check = false;
  if (det) {
    if (k.cand_valid && c->skin_factor * margin != k.cand_skin) k.cand_valid = false;
    check = k.cand_valid && c->n_sph;
    k_minmax_init<<<1, 32, 0, s>>>(mm);
    if (check) k_set_int<<<1, 1, 0, s>>>(k.flag.as<int>(), 0);   // a kernel: the flag may be peer memory
  }
  const double skin = c->skin_factor * margin, skin_b = c->skin_big_factor * margin;
  // one wave of 3 CTAs / SM, grid-stride (2470 vs 2460 M sphere-steps/s at 8 / SM)
  const int64_t snap_blocks = int64_t(c->n_sm) * 3;
  if (c->n_sph)
    k_snapshot<<<unsigned(std::min<int64_t>(grid_for(c->n_sph), snap_blocks)), kBlock, 0, s>>>(
        c->dom, owners_view(c), spheres_view(c), k.c4.as<double4>(), k.sfam.as<uint8_t>(),
        det ? mm : nullptr, check ? k.ref.as<double>() : nullptr, 0.25 * skin * skin,
        (skin_b - 0.5 * skin) * (skin_b - 0.5 * skin), c->n_big ? c->r_cut : 0.0, k.flag.as<int>());
  k.snap_det = det;
  k.snap_checked = check;
  if (c->n_tri) {
    GF_CHECK(c, cudaMemcpyAsync(k.tri_world.p, c->tri_world.p, sizeof(double) * 9 * c->n_tri,
                                cudaMemcpyDeviceToDevice, s));
    k_geom_family<<<grid_for(c->n_tri), kBlock, 0, s>>>(c->n_tri, c->tri_owner.as<uint32_t>(),
                                                       c->meta.as<uint32_t>(), k.tfam.as<uint8_t>());
  }
  if (c->n_ana) {
    GF_CHECK(c, cudaMemcpyAsync(k.ana_world.p, c->ana_world.p, sizeof(double) * 8 * c->n_ana,
                                cudaMemcpyDeviceToDevice, s));
    k_geom_family<<<grid_for(c->n_ana), kBlock, 0, s>>>(c->n_ana, c->ana_owner.as<uint32_t>(),
                                                       c->meta.as<uint32_t>(), k.afam.as<uint8_t>());
  }
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

static KtView kt_view(Ctx *c, double margin) {
  KtScratch &k = c->kt;
  KtView v;
  v.dom = c->dom;
  v.own = owners_view(c);
  v.sph = spheres_view(c);
  v.n_tri = c->n_tri;
  v.n_ana = c->n_ana;
  v.tri_owner = c->tri_owner.as<uint32_t>();
  v.ana_owner = c->ana_owner.as<uint32_t>();
  v.ana_kind = c->ana_kind.as<uint8_t>();
  v.centers = k.c4.as<double>();   // the (centre, radius) snapshot records, stride 4
  v.sfam = k.sfam.as<uint8_t>();
  v.tri_world = k.tri_world.as<double>();
  v.tfam = k.tfam.as<uint8_t>();
  v.ana_world = k.ana_world.as<double>();
  v.afam = k.afam.as<uint8_t>();
  v.mask = c->fam_mask.as<uint8_t>();
  v.bin_key = k.bin_key.as<uint32_t>();
  v.sph_sorted = k.sph_val.as<uint32_t>();
  v.cell_start = k.cell_start.as<uint32_t>();
  v.cell_end = k.cell_end.as<uint32_t>();
  v.tri_start = k.tri_start.as<uint32_t>();
  v.tri_entries = k.tri_entries.as<uint32_t>();
  v.grid = k.grid.as<Grid>();
  v.margin = margin;
  v.c4 = k.c4.as<double4>();
  v.mask_trivial = c->mask_trivial ? 1 : 0;
  return v;
}

// phase A of a detection: grid, triangle registration, and the displacement
// check that decides whether the candidate lists must be rebuilt (flag copied
// to the pinned status mirror; the host reads it before kt_count)
int kt_begin(Ctx *c, double margin, cudaStream_t s) {
  DevGuard g_kt(stream_device(s));   // the kT device of a 2-GPU split
  KtScratch &k = c->kt;
  const int64_t n = c->n_sph, nt = c->n_tri;
  const int64_t n_pts = n + 3 * nt;
  c->kt_margin = margin;
  const double skin = c->skin_factor * margin;
  if (k.cand_valid && skin != k.cand_skin) k.cand_valid = false;
  if (ensure(c, k.grid, sizeof(Grid), s) || ensure(c, k.minmax, sizeof(unsigned long long) * 8, s) ||
      ensure(c, k.flag, 16, s))
    return -1;
  unsigned long long *mm = k.minmax.as<unsigned long long>();
  const bool snap = k.snap_det;   // the snapshot reduced the sphere centres already
  k.snap_det = false;
  if (!snap) {
    k_minmax_init<<<1, 32, 0, s>>>(mm);
    if (n) k_minmax<<<std::min<int64_t>(grid_for(n), 1184), kBlock, 0, s>>>(n, k.c4.as<double>(), 4, n, c->sph_offr.as<float4>(), mm);
  }
  if (nt) k_minmax<<<std::min<int64_t>(grid_for(3 * nt), 1184), kBlock, 0, s>>>(3 * nt, k.tri_world.as<double>(), 3, 0, nullptr, mm);
  k_grid<<<1, 1, 0, s>>>(mm, n_pts, margin, c->kt_bin_size, c->r_cut, (long long)kMaxCells, margin + skin,
                         k.grid.as<Grid>());
  const Grid *gp = k.grid.as<Grid>();
  int *flag = k.flag.as<int>();
  if (k.cand_valid && n) {
    if (!(snap && k.snap_checked)) {
      GF_CHECK(c, cudaMemsetAsync(flag, 0, sizeof(int), s));
      const double skin_b = c->skin_big_factor * margin;
      k_disp<<<grid_for(n), kBlock, 0, s>>>(n, k.c4.as<double4>(), k.ref.as<double>(), 0.25 * skin * skin,
                                            (skin_b - 0.5 * skin) * (skin_b - 0.5 * skin),
                                            c->n_big ? c->r_cut : 0.0, flag);
    }
  } else {
    k_set_int<<<1, 1, 0, s>>>(flag, 1);
  }
  GF_CHECK(c, cudaMemcpyAsync(&reinterpret_cast<Status *>(c->h_status)->rebuild, flag, sizeof(int),
                              cudaMemcpyDeviceToHost, s));
  if (nt) {
    if (ensure(c, k.tri_cnt, sizeof(uint32_t) * (kMaxCells + 1), s) ||
        ensure(c, k.tri_start, sizeof(uint32_t) * (kMaxCells + 1), s) ||
        ensure(c, k.tri_cursor, sizeof(uint32_t) * (kMaxCells + 1), s))
      return -1;
    k_fill_u32<<<592, 256, 0, s>>>(gp, k.tri_cnt.as<uint32_t>(), 0u, 1);
    k_tri_register<false><<<unsigned(std::min<int64_t>(nt, int64_t(c->n_sm) * 16)), 128, 0, s>>>(nt, k.tri_world.as<double>(), gp, margin,
                                                         k.tri_cnt.as<uint32_t>(), nullptr, nullptr);
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, k.tri_cnt.as<uint32_t>(), k.tri_start.as<uint32_t>(),
                                  kMaxCells + 1, s);
    if (ensure(c, k.cub_tmp, tmp + 16, s, false)) return -1;
    GF_CHECK(c, cub::DeviceScan::ExclusiveSum(k.cub_tmp.p, tmp, k.tri_cnt.as<uint32_t>(),
                                              k.tri_start.as<uint32_t>(), kMaxCells + 1, s));
    uint32_t h_total = 0;
    GF_CHECK(c, cudaMemcpyAsync(&h_total, k.tri_start.as<uint32_t>() + kMaxCells, 4,
                                cudaMemcpyDeviceToHost, s));
    GF_CHECK(c, cudaStreamSynchronize(s));
    if (ensure(c, k.tri_entries, sizeof(uint32_t) * (h_total + 1), s)) return -1;
    GF_CHECK(c, cudaMemcpyAsync(k.tri_cursor.p, k.tri_start.p, sizeof(uint32_t) * (kMaxCells + 1),
                                cudaMemcpyDeviceToDevice, s));
    k_tri_register<true><<<unsigned(std::min<int64_t>(nt, int64_t(c->n_sm) * 16)), 128, 0, s>>>(nt, k.tri_world.as<double>(), gp, margin,
                                                        nullptr, k.tri_cursor.as<uint32_t>(),
                                                        k.tri_entries.as<uint32_t>());
  }
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

// the long-run list of seg_fill (KtScratch::gaps), its counter cleared on s
static int gap_list(Ctx *c, GapList &gl, cudaStream_t s) {
  KtScratch &k = c->kt;
  const unsigned long long cap = (unsigned long long)(c->n_sph / kGapInline) + 4;
  if (ensure(c, k.gaps, (sizeof(ulonglong2) + sizeof(unsigned long long)) * cap + 16, s)) return -1;
  gl.run = k.gaps.as<ulonglong2>();
  gl.val = reinterpret_cast<unsigned long long *>(gl.run + cap);
  gl.n = gl.val + cap;
  gl.cap = cap;
  GF_CHECK(c, cudaMemsetAsync(gl.n, 0, sizeof(unsigned long long), s));
  return 0;
}

// rebuild the candidate lists from the current snapshot (enumeration grid
// with reach margin + skin)
// The candidate rebuild in four resumable stages.  Each stage ends where the
// host needs a device count (to size the next stage's buffers): the count is
// copied to the pinned status block and an event recorded, and the stage
// returns.  kt_count_async / kt_advance (gf_context.cu run_count /
// advance_kt) resume the next stage once the event has completed, between
// the host's dT step enqueues -- so the dT stream stays fed while a rebuild
// runs on the kT stream, instead of the host blocking on each count.
//   A  keys, cell sort, cell bounds, cell-sorted copies, small-pair count + scan
//   B  small-pair fill, big-sphere pairs (count -> host)
//   C  sort by a, unpack, segment sorts, reference centres; sphere-analytic
//      candidate count (-> host)
//   D  sphere-analytic fill, scratch release, bookkeeping
// the fill pass met more pairs than the count pass sized (the pinned mirror
// of Status::cand_overflow, copied after the fill; read once the fill's
// event has completed): fail the rebuild loudly
static int cand_overflowed(Ctx *c) {
  const unsigned long long o = reinterpret_cast<Status *>(c->h_status)->cand_overflow;
  if (!o) return 0;
  set_err(c, "candidate rebuild: the fill pass found " + std::to_string(o) +
                 " pairs beyond the counted capacity (count / fill mismatch)");
  return 1;
}

static int rb_stage_a(Ctx *c, cudaStream_t s) {
  KtScratch &k = c->kt;
  const int64_t n = c->n_sph;
  const double skin = c->skin_factor * c->kt_margin;
  const double reach = c->kt_margin + skin;                         // small-small
  if (ensure_scratch(c, k.bin_key, 4 * (n + 1), s) || ensure_scratch(c, k.bin_key_alt, 4 * (n + 1), s) ||
      ensure_scratch(c, k.sph_val, 4 * (n + 1), s) || ensure_scratch(c, k.sph_val_alt, 4 * (n + 1), s) ||
      ensure(c, k.cursor, 4 * (3 * n + 1), s) || ensure_scratch(c, k.sc, 32 * (n + 1), s) ||
      ensure_scratch(c, k.sm, 16 * (n + 1), s) || ensure_scratch(c, k.sf, 16 * (n + 1), s) ||
      ensure(c, k.cand_n, 16, s) || ensure_scratch(c, k.cand_cnt, 8 * (n + 1), s) ||
      ensure(c, k.ref, 24 * (n + 1), s) ||
      ensure(c, k.cell_start, sizeof(uint32_t) * (kMaxCells + 1), s) ||
      ensure(c, k.cell_end, sizeof(uint32_t) * (kMaxCells + 1), s))
    return -1;
  if (k.cand_cap == 0) {
    int64_t cap = std::max<int64_t>(6 * n, 4096);   // grown to the exact need on overflow below
    if (ensure(c, k.cand, sizeof(uint2) * cap, s)) return -1;
    k.cand_cap = cap;
  }
  if (!c->rb_slot && ensure_scratch(c, k.cand_tmp, sizeof(uint2) * k.cand_cap, s))   // released after big rebuilds
    return -1;
  const Grid *gp = k.grid.as<Grid>();
  if (ensure(c, k.counts, sizeof(unsigned long long) * (3 * n + 1), s)) return -1;
  uint32_t *ucnt = k.cand_cnt.as<uint32_t>();          // per cell-sorted sphere: its hits
  unsigned long long *uoff = k.counts.as<unsigned long long>();   // their exclusive scan (scratch here)
  Status *hs = reinterpret_cast<Status *>(c->h_status);
  hs->cand_total = 0;
  if (n) {
    k_bin_keys<<<grid_for(n), kBlock, 0, s>>>(n, k.c4.as<double>(), c->sph_offr.as<float4>(), gp,
                                             k.bin_key.as<uint32_t>(), k.sph_val.as<uint32_t>());
    size_t tmp = 0;
    cub::DoubleBuffer<uint32_t> dk(k.bin_key.as<uint32_t>(), k.bin_key_alt.as<uint32_t>());
    cub::DoubleBuffer<uint32_t> dv(k.sph_val.as<uint32_t>(), k.sph_val_alt.as<uint32_t>());
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, int(n), 0, kKeyBits, s);
    if (ensure(c, k.cub_tmp, tmp + 16, s, false)) return -1;
    GF_CHECK(c, cub::DeviceRadixSort::SortPairs(k.cub_tmp.p, tmp, dk, dv, int(n), 0, kKeyBits, s));
    if (dk.Current() != k.bin_key.as<uint32_t>()) {
      std::swap(k.bin_key, k.bin_key_alt);
      std::swap(k.sph_val, k.sph_val_alt);
    }
    KtView v = kt_view(c, c->kt_margin);
    k_fill_u32<<<592, 256, 0, s>>>(gp, k.cell_start.as<uint32_t>(), 0xFFFFFFFFu, 0);
    k_cell_bounds<<<grid_for(n), kBlock, 0, s>>>(n, k.bin_key.as<uint32_t>(), k.cell_start.as<uint32_t>(),
                                                k.cell_end.as<uint32_t>());
    k_gather_sorted<<<grid_for(n), kBlock, 0, s>>>(n, k.sph_val.as<uint32_t>(), k.c4.as<double>(),
                                                  c->sph_offr.as<float4>(), c->sph_owner.as<uint32_t>(),
                                                  k.sfam.as<uint8_t>(), gp, k.sc.as<double4>(),
                                                  k.sm.as<uint4>(), k.sf.as<float4>());
    if (c->rb_slot) {   // per-slot pair counts -> segment starts (cand_seg)
      const double skin_b = c->skin_big_factor * c->kt_margin;
      if (ensure_scratch(c, k.cand_own, 4 * (n + 1), s) || ensure_scratch(c, k.cand_seg, 8 * (n + 1), s)) return -1;
      GF_CHECK(c, cudaMemsetAsync(ucnt, 0, 4 * (n + 1), s));
      k_cand_slot<false><<<grid_for(n, 128), 128, 0, s>>>(v, k.sm.as<uint4>(), k.sf.as<float4>(), reach, ucnt,
                                                          k.cand_own.as<uint32_t>(), nullptr, nullptr, nullptr);
      if (c->n_big)
        k_cand_big_slot<false><<<unsigned(std::min<int64_t>(c->n_big, 4096)), 128, 0, s>>>(
            v, c->big_slots.as<uint32_t>(), c->n_big, k.sc.as<double4>(), k.sm.as<uint4>(), c->kt_margin + skin_b,
            c->kt_margin + 2.0 * skin_b - skin, ucnt, nullptr, nullptr, nullptr);
      unsigned long long *seg = k.cand_seg.as<unsigned long long>();
      const CountsU64 ucnt64(ucnt, U32ToU64());
      cub::DeviceScan::ExclusiveSum(nullptr, tmp, ucnt64, seg, int(n + 1), s);
      if (ensure(c, k.cub_tmp, tmp + 16, s, false)) return -1;
      GF_CHECK(c, cub::DeviceScan::ExclusiveSum(k.cub_tmp.p, tmp, ucnt64, seg, int(n + 1), s));
      GF_CHECK(c, cudaMemcpyAsync(&hs->cand_total, seg + n, 8, cudaMemcpyDeviceToHost, s));
      return 0;
    }
    // count, scan, fill: every thread writes its own hits at its own offset
    k_cand_ss<false><<<grid_for(n, 128), 128, 0, s>>>(v, k.sm.as<uint4>(), k.sf.as<float4>(), reach, ucnt,
                                                      nullptr, nullptr, nullptr);
    GF_CHECK(c, cudaMemsetAsync(ucnt + n, 0, sizeof(uint32_t), s));
    const CountsU64 ucnt64(ucnt, U32ToU64());
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, ucnt64, uoff, int(n + 1), s);
    if (ensure(c, k.cub_tmp, tmp + 16, s, false)) return -1;
    GF_CHECK(c, cub::DeviceScan::ExclusiveSum(k.cub_tmp.p, tmp, ucnt64, uoff, int(n + 1), s));
    GF_CHECK(c, cudaMemcpyAsync(&hs->cand_total, uoff + n, 8, cudaMemcpyDeviceToHost, s));
  }
  k.rb_big_cap = k.big_cap > 0 ? k.big_cap : (c->n_big ? std::max<int64_t>(4096 * c->n_big, 65536) : 0);
  return 0;
}

static int rb_stage_b(Ctx *c, cudaStream_t s) {
  KtScratch &k = c->kt;
  const int64_t n = c->n_sph;
  const double skin = c->skin_factor * c->kt_margin, skin_b = c->skin_big_factor * c->kt_margin;
  const double reach = c->kt_margin + skin, reach_big = c->kt_margin + skin_b;
  const double reach_bb = c->kt_margin + 2.0 * skin_b - skin;       // big-big
  const int64_t small = int64_t(reinterpret_cast<Status *>(c->h_status)->cand_total);
  k.rb_small = small;
  const int64_t need = small + k.rb_big_cap + 1;
  if (need > k.cand_cap) {
    const int64_t cap = need + need / 10 + 4096;
    if (ensure_scratch(c, k.cand_tmp, sizeof(uint2) * cap, s) || ensure(c, k.cand, sizeof(uint2) * cap, s)) return -1;
    k.cand_cap = cap;
  }
  // (a, b) halves of cand_tmp; cand holds the sort's alternate halves
  uint32_t *ka = k.cand_tmp.as<uint32_t>(), *kb = ka + k.cand_cap;
  KtView v = kt_view(c, c->kt_margin);
  unsigned long long *ovf = &c->status.as<Status>()->cand_overflow;
  GF_CHECK(c, cudaMemsetAsync(ovf, 0, 8, s));
  if (n)
    k_cand_ss<true><<<grid_for(n, 128), 128, 0, s>>>(v, k.sm.as<uint4>(), k.sf.as<float4>(), reach, nullptr,
                                                     k.counts.as<unsigned long long>(), ka, kb,
                                                     (unsigned long long)small, ovf);
  GF_CHECK(c, cudaMemcpyAsync(&reinterpret_cast<Status *>(c->h_status)->cand_overflow, ovf, 8,
                              cudaMemcpyDeviceToHost, s));
  unsigned long long *big_n = k.cand_n.as<unsigned long long>();
  GF_CHECK(c, cudaMemsetAsync(big_n, 0, 8, s));
  if (c->n_big)
    k_cand_big<<<unsigned(std::min<int64_t>(c->n_big, 4096)), 128, 0, s>>>(
        v, c->big_slots.as<uint32_t>(), c->n_big, k.sc.as<double4>(), k.sm.as<uint4>(), reach_big, reach_bb,
        ka + small, kb + small, big_n, (unsigned long long)k.rb_big_cap);
  GF_CHECK(c, cudaMemcpyAsync(&reinterpret_cast<Status *>(c->h_status)->other_total, big_n, 8,
                              cudaMemcpyDeviceToHost, s));
  return 0;
}

static int rb_lists_tail(Ctx *c, cudaStream_t s);

// returns 1 when the big-sphere pass overflowed (stage B must be redone with
// the grown capacity)
static int rb_stage_c(Ctx *c, cudaStream_t s) {
  KtScratch &k = c->kt;
  const int64_t n = c->n_sph;
  if (cand_overflowed(c)) return -1;
  const int64_t nbig = int64_t(reinterpret_cast<Status *>(c->h_status)->other_total);
  if (nbig > k.rb_big_cap) {
    k.rb_big_cap = nbig + nbig / 4 + 4096;
    return 1;
  }
  k.big_cap = k.rb_big_cap;
  k.n_cand = k.rb_small + nbig;
  const int64_t total = k.n_cand;
  if (ensure_scratch(c, k.cand_seg, 8 * (n + 1), s)) return -1;
  if (total > int64_t(INT32_MAX)) {
    set_err(c, "candidate rebuild: " + std::to_string(total) +
                   " candidates exceed the sort-based rebuild's 2^31 items (use the slot-grouped rebuild, GF_RB_SLOT=1)");
    return -1;
  }
  if (total) {
    // sort by a (only as many bits as slots need; b rides along), then each
    // sphere's segment by b
    const int64_t cap = k.cand_cap;
    uint32_t *ka = k.cand_tmp.as<uint32_t>(), *kb = ka + cap;
    uint32_t *ka2 = k.cand.as<uint32_t>(), *kb2 = ka2 + cap;
    cub::DoubleBuffer<uint32_t> dk(ka, ka2), dv(kb, kb2);
    int bits = 1;
    while ((int64_t(1) << bits) < n) ++bits;
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, int(total), 0, bits, s);
    if (ensure(c, k.cub_tmp, tmp + 16, s, false)) return -1;
    GF_CHECK(c, cub::DeviceRadixSort::SortPairs(k.cub_tmp.p, tmp, dk, dv, int(total), 0, bits, s));
    if (dk.Current() == ka2) std::swap(k.cand, k.cand_tmp);   // sorted halves now in cand_tmp
    const uint32_t *sa = k.cand_tmp.as<uint32_t>(), *sb = sa + cap;
    GapList gl;
    if (gap_list(c, gl, s)) return -1;
    k_cand_unpack<<<unsigned(std::min<int64_t>((total + 255) / 256, int64_t(c->n_sm) * 16)), 256, 0, s>>>(
        total, n, sa, sb, k.cand.as<uint2>(), k.cand_seg.as<unsigned long long>(), gl);
    k_fill_gaps<<<unsigned(c->n_sm) * 4, 256, 0, s>>>(k.cand_seg.as<unsigned long long>(), gl);
  }
  return rb_lists_tail(c, s);
}

// both rebuild variants, once the (a, b) list and its per-sphere segment
// starts are in place: each segment sorted by b, the reference centres, the
// sphere-analytic candidate count (-> host)
static int rb_lists_tail(Ctx *c, cudaStream_t s) {
  KtScratch &k = c->kt;
  const int64_t n = c->n_sph;
  const double skin = c->skin_factor * c->kt_margin, skin_b = c->skin_big_factor * c->kt_margin;
  const double reach = c->kt_margin + skin, reach_big = c->kt_margin + skin_b;
  unsigned long long *big_n = k.cand_n.as<unsigned long long>();
  if (k.n_cand && sync_debug()) {   // GF_SYNC_DEBUG: the segment table against the list it indexes
    std::vector<unsigned long long> hseg(n + 1);
    GF_CHECK(c, cudaMemcpy(hseg.data(), k.cand_seg.p, 8 * (n + 1), cudaMemcpyDeviceToHost));
    unsigned long long mx = 0, bad = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (hseg[i + 1] < hseg[i]) ++bad;
      else mx = std::max(mx, hseg[i + 1] - hseg[i]);
    }
    if (bad || hseg[n] != (unsigned long long)k.n_cand || 8 * hseg[n] > k.cand.bytes) {
      set_err(c, "GF_SYNC_DEBUG: candidate segments: " + std::to_string(bad) + " decreasing, seg[n] " +
                     std::to_string(hseg[n]) + " vs n_cand " + std::to_string(k.n_cand) + ", list bytes " +
                     std::to_string(k.cand.bytes) + ", longest " + std::to_string(mx) + ", seg[0] " +
                     std::to_string(hseg[0]));
      return -1;
    }
  }
  if (k.n_cand) {
    if (ensure(c, k.sa_cnt, 4 * (n + 1), s)) return -1;   // the long-segment list (scratch here)
    GF_CHECK(c, cudaMemsetAsync(big_n, 0, 8, s));
    k_sort_seg_short<<<grid_for(n), kBlock, 0, s>>>(n, k.cand_seg.as<unsigned long long>(), k.cand.as<uint2>(),
                                                   k.sa_cnt.as<uint32_t>(), big_n);
    if (dbg_sync(c, "k_sort_seg_short", -1)) return -1;
    // the opt-in is per device: tracked per context (a process may hold
    // contexts on several devices, and kT and dT may sit on different ones)
    if (!k.sort_long_smem) {
      GF_CHECK(c, cudaFuncSetAttribute(k_sort_long, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(sizeof(uint2) * kLongSeg)));
      k.sort_long_smem = true;
    }
    k_sort_long<<<c->n_sm, 1024, sizeof(uint2) * kLongSeg, s>>>(k.cand_seg.as<unsigned long long>(), k.cand.as<uint2>(),
                                                            k.sa_cnt.as<uint32_t>(), big_n);
    if (dbg_sync(c, "k_sort_long", -1)) return -1;
  }
  if (n) k_copy_ref<<<grid_for(n), kBlock, 0, s>>>(n, k.c4.as<double4>(), k.ref.as<double>());
  // sphere-analytic candidates for the same skin, while the world is static
  k.sa_world_version = ~0ull;
  k.rb_sa = n && c->n_ana && !c->world_moving;
  if (k.rb_sa) {
    KtView v = kt_view(c, c->kt_margin);
    if (ensure(c, k.sa_cnt, 4 * (n + 1), s) || ensure(c, k.sa_off, 8 * (n + 1), s)) return -1;
    k_sa_count<<<grid_for(n), kBlock, 0, s>>>(v, reach, reach_big, c->n_big ? c->r_cut : 0.0, k.sa_cnt.as<uint32_t>());
    GF_CHECK(c, cudaMemsetAsync(k.sa_cnt.as<uint32_t>() + n, 0, 4, s));
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, k.sa_cnt.as<uint32_t>(), k.sa_off.as<unsigned long long>(), int(n + 1), s);
    if (ensure(c, k.cub_tmp, tb + 16, s, false)) return -1;
    GF_CHECK(c, cub::DeviceScan::ExclusiveSum(k.cub_tmp.p, tb, k.sa_cnt.as<uint32_t>(),
                                              k.sa_off.as<unsigned long long>(), int(n + 1), s));
    GF_CHECK(c, cudaMemcpyAsync(&reinterpret_cast<Status *>(c->h_status)->other_total,
                                k.sa_off.as<unsigned long long>() + n, 8, cudaMemcpyDeviceToHost, s));
  }
  return 0;
}

// slot-grouped rebuild, stage B: the list sized from the total, every pair
// placed in its lower slot's segment, then the common tail
static int rb_slot_b(Ctx *c, cudaStream_t s) {
  KtScratch &k = c->kt;
  const int64_t n = c->n_sph;
  const double skin = c->skin_factor * c->kt_margin, skin_b = c->skin_big_factor * c->kt_margin;
  const int64_t total = int64_t(reinterpret_cast<Status *>(c->h_status)->cand_total);
  k.n_cand = total;
  if (total + 1 > k.cand_cap) {
    const int64_t cap = total + total / 10 + 4096;
    if (ensure(c, k.cand, sizeof(uint2) * cap, s)) return -1;
    k.cand_cap = cap;
  }
  if (n && total) {
    KtView v = kt_view(c, c->kt_margin);
    uint32_t *cur = k.cursor.as<uint32_t>();
    const unsigned long long *seg = k.cand_seg.as<unsigned long long>();
    GF_CHECK(c, cudaMemsetAsync(cur, 0, 4 * (n + 1), s));
    unsigned long long *ovf = &c->status.as<Status>()->cand_overflow;
    GF_CHECK(c, cudaMemsetAsync(ovf, 0, 8, s));
    const unsigned long long cap = (unsigned long long)total;
    k_cand_slot<true><<<grid_for(n, 128), 128, 0, s>>>(v, k.sm.as<uint4>(), k.sf.as<float4>(), c->kt_margin + skin,
                                                       nullptr, k.cand_own.as<uint32_t>(), seg, cur,
                                                       k.cand.as<uint2>(), cap, ovf);
    if (c->n_big)
      k_cand_big_slot<true><<<unsigned(std::min<int64_t>(c->n_big, 4096)), 128, 0, s>>>(
          v, c->big_slots.as<uint32_t>(), c->n_big, k.sc.as<double4>(), k.sm.as<uint4>(), c->kt_margin + skin_b,
          c->kt_margin + 2.0 * skin_b - skin, nullptr, seg, cur, k.cand.as<uint2>(), cap, ovf);
    if (dbg_sync(c, "rb_slot_b fill", -1)) return -1;
    GF_CHECK(c, cudaMemcpyAsync(&reinterpret_cast<Status *>(c->h_status)->cand_overflow, ovf, 8,
                                cudaMemcpyDeviceToHost, s));
  }
  return rb_lists_tail(c, s);
}

static int rb_stage_d(Ctx *c, cudaStream_t s) {
  KtScratch &k = c->kt;
  if (c->rb_slot && cand_overflowed(c)) return -1;
  const int64_t n = c->n_sph;
  const double skin = c->skin_factor * c->kt_margin, skin_b = c->skin_big_factor * c->kt_margin;
  const double reach = c->kt_margin + skin, reach_big = c->kt_margin + skin_b;
  if (k.rb_sa) {
    k.n_sa_cand = int64_t(reinterpret_cast<Status *>(c->h_status)->other_total);
    if (ensure(c, k.sa_cand, sizeof(uint2) * (k.n_sa_cand + 1), s)) return -1;
    KtView v = kt_view(c, c->kt_margin);
    k_sa_fill<<<grid_for(n), kBlock, 0, s>>>(v, reach, reach_big, c->n_big ? c->r_cut : 0.0,
                                             k.sa_off.as<unsigned long long>(), k.sa_cand.as<uint2>());
    k.sa_world_version = c->world_version;
  }
  // at 2^24 spheres and up device memory is the limit: the rebuild-only
  // scratch (sort keys, cell-sorted copies, candidate counts and staging,
  // ~170 B / sphere) comes from the stream-ordered pool (ensure_scratch) and
  // goes back to it here, ordered on the kT stream -- no device-wide
  // synchronisation, so the dT stream never stalls on a rebuild
  if (big_scratch(c)) {
    for (DBuf *b : {&k.bin_key, &k.bin_key_alt, &k.sph_val, &k.sph_val_alt, &k.sc, &k.sm, &k.sf, &k.cand_cnt,
                    &k.cand_seg, &k.cand_tmp, &k.cand_own})
      if (release_scratch(c, *b, s)) return -1;
  }
  k.cand_valid = true;
  k.cand_skin = c->skin_factor * c->kt_margin;
  k.rebuilds++;
  k.cand_gen++;   // candidate rows of earlier arrays no longer apply
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

// the whole rebuild, blocking on each count (gf_detect, recounts)
static int rebuild_candidates(Ctx *c, cudaStream_t s) {
  DevGuard g_kt(stream_device(s));   // the kT device of a 2-GPU split
  if (rb_stage_a(c, s)) return -1;
  if (c->rb_slot) {
    GF_CHECK(c, cudaStreamSynchronize(s));
    if (rb_slot_b(c, s)) return -1;
    GF_CHECK(c, cudaStreamSynchronize(s));
    return rb_stage_d(c, s);
  }
  for (;;) {
    GF_CHECK(c, cudaStreamSynchronize(s));
    if (rb_stage_b(c, s)) return -1;
    GF_CHECK(c, cudaStreamSynchronize(s));
    const int rc = rb_stage_c(c, s);
    if (rc < 0) return -1;
    if (rc == 0) break;
  }
  GF_CHECK(c, cudaStreamSynchronize(s));
  return rb_stage_d(c, s);
}

// Non-blocking entry of the count phase: a detection that needs a rebuild
// starts stage A and returns 1 (the caller resumes with kt_advance); else
// the filter / compaction is queued and 0 returned.
int kt_count_async(Ctx *c, cudaStream_t s) {
  DevGuard g_kt(stream_device(s));
  KtScratch &k = c->kt;
  Status *hs = reinterpret_cast<Status *>(c->h_status);
  if (c->rb_async && (!k.cand_valid || hs->rebuild)) {
    hs->cand_total = 0;
    hs->rebuild = 0;   // consumed
    if (rb_stage_a(c, s)) return -1;
    k.rb_stage = 1;
    return 1;
  }
  return kt_count(c, s, false);
}

// Resume a staged rebuild once its pending count is on the host (block =
// wait for it): returns 1 while stages remain, 0 when the rebuild finished
// and the detection's filter / compaction is queued.
int kt_advance(Ctx *c, cudaStream_t s, cudaEvent_t ev, bool block) {
  DevGuard g_kt(stream_device(s));
  KtScratch &k = c->kt;
  while (k.rb_stage > 0) {
    if (block) {
      GF_CHECK(c, cudaEventSynchronize(ev));
    } else {
      const cudaError_t q = cudaEventQuery(ev);
      if (q == cudaErrorNotReady) {
        (void)cudaGetLastError();
        return 1;
      }
      GF_CHECK(c, q);
    }
    if (k.rb_stage == 1 && c->rb_slot) {
      if (rb_slot_b(c, s)) return -1;
      k.rb_stage = 3;
    } else if (k.rb_stage == 1) {
      if (rb_stage_b(c, s)) return -1;
      k.rb_stage = 2;
    } else if (k.rb_stage == 2) {
      const int rc = rb_stage_c(c, s);
      if (rc < 0) return -1;
      if (rc == 1) {   // big pass overflowed: redo stage B with the grown capacity
        if (rb_stage_b(c, s)) return -1;
        k.rb_stage = 2;
      } else {
        k.rb_stage = 3;
      }
    } else {
      if (rb_stage_d(c, s)) return -1;
      k.rb_stage = 0;
      return kt_count(c, s, false) ? -1 : 0;
    }
    GF_CHECK(c, cudaEventRecord(ev, s));
  }
  return 0;
}

// phase B (after the host read the phase-A flag): optional rebuild, exact
// filter of the candidates, sphere-triangle / sphere-analytic pairs, counts,
// scan; the pair total goes to the pinned status mirror
int kt_count(Ctx *c, cudaStream_t s, bool force_rebuild) {
  DevGuard g_kt(stream_device(s));   // the kT device of a 2-GPU split
  KtScratch &k = c->kt;
  const int64_t n = c->n_sph;
  Status *hs = reinterpret_cast<Status *>(c->h_status);
  if (force_rebuild || !k.cand_valid || hs->rebuild) {
    hs->cand_total = 0;
    if (rebuild_candidates(c, s)) return -1;
    hs->rebuild = 0;   // consumed (a recount of this detection must not rebuild again)
  }
  if (ensure(c, k.counts, sizeof(unsigned long long) * (3 * n + 1), s) || ensure(c, k.tmp_n, 16, s))
    return -1;
  if (k.tmp_cap == 0) {   // wall pairs: a few per boundary sphere; grown on overflow
    int64_t cap = std::max<int64_t>(n / 16, 4096);
    if (ensure(c, k.tmp, sizeof(uint2) * cap, s)) return -1;
    k.tmp_cap = cap;
  }
  // the sphere-sphere block is compacted straight into the next array: room
  // for the last block's size + 1/8 (or 3/4 of the candidates) plus the
  // wall-pair scratch capacity; k_compact drops rows beyond it and the fill
  // phase grows the array and redoes the count (rare)
  Acs &out = c->acs_next;
  const int64_t ss_guess = k.last_ss > 0 ? k.last_ss + k.last_ss / 8 + 1024 : (3 * k.n_cand) / 4 + 1024;
  const int64_t need = std::min<int64_t>(k.n_cand, std::max<int64_t>(ss_guess, k.ss_need)) + k.tmp_cap + 1;
  if (need > out.cap) {
    // 25% growth room: the two contact arrays alternate, and a reallocation
    // synchronises the device, so a slowly growing pair count must not
    // trigger one per detection
    int64_t cap = need + need / 4 + 1024;
    DevGuard g_dt(c->device);   // contact arrays live on the dT device
    if (ensure(c, out.ids, sizeof(uint2) * cap, s) || ensure(c, out.wild, sizeof(float) * c->wild_w * cap, s) ||
        ensure(c, out.old_pos, sizeof(uint32_t) * cap, s))
      return -1;
    out.cap = cap;
  }
  {
    DevGuard g_dt(c->device);
    if (ensure(c, out.seg, sizeof(unsigned long long) * (3 * n + 1), s)) return -1;
  }
  KtView v = kt_view(c, c->kt_margin);
  unsigned long long *cnt = k.counts.as<unsigned long long>();
  unsigned long long *tn = k.tmp_n.as<unsigned long long>();
  unsigned long long *oseg = out.seg.as<unsigned long long>();
  GF_CHECK(c, cudaMemsetAsync(cnt + 3 * n, 0, sizeof(unsigned long long), s));
  GF_CHECK(c, cudaMemsetAsync(tn, 0, sizeof(unsigned long long), s));
  // exact filter of the sphere-sphere candidates, then their compaction
  const int prev = k.cslot_cur ^ 1;   // bitmask + counts of the last filtered array
  const bool rows_ok = k.cslot_gen[prev] == k.cand_gen && k.cslot_det[prev] != 0;
  const uint64_t det = ++k.det_serial;
  const int cur = k.cslot_cur;
  const int64_t nblk = (k.n_cand + kFcSpan - 1) / kFcSpan;
  if (ensure(c, k.fbits[cur], 4 * ((k.n_cand + 31) / 32 + 1), s) ||
      ensure(c, k.fcnt, 4 * (nblk + 1), s) || ensure(c, k.fpre[cur], 8 * (nblk + 1), s))
    return -1;
  unsigned long long *ss_tot = k.fpre[cur].as<unsigned long long>() + nblk;   // the block's size
  if (k.n_cand) {
    k_filter_bits<<<unsigned(nblk), kFcBlock, 0, s>>>(v, k.cand.as<uint2>(), k.n_cand, k.fbits[cur].as<uint32_t>(),
                                                      k.fcnt.as<uint32_t>());
    GF_CHECK(c, cudaMemsetAsync(k.fcnt.as<uint32_t>() + nblk, 0, 4, s));
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, k.fcnt.as<uint32_t>(), k.fpre[cur].as<unsigned long long>(),
                                  int(nblk + 1), s);
    if (ensure(c, k.cub_tmp, tb + 16, s, false)) return -1;
    GF_CHECK(c, cub::DeviceScan::ExclusiveSum(k.cub_tmp.p, tb, k.fcnt.as<uint32_t>(),
                                              k.fpre[cur].as<unsigned long long>(), int(nblk + 1), s));
    GapList gl;
    if (gap_list(c, gl, s)) return -1;
    k_compact<<<unsigned(nblk), kFcBlock, 0, s>>>(
        v, k.cand.as<uint2>(), k.n_cand, k.fbits[cur].as<uint32_t>(), k.fpre[cur].as<unsigned long long>(),
        rows_ok ? k.fbits[prev].as<uint32_t>() : nullptr, rows_ok ? k.fpre[prev].as<unsigned long long>() : nullptr,
        out.ids.as<uint2>(), oseg, out.old_pos.as<uint32_t>(), (unsigned long long)(out.cap - k.tmp_cap - 1), gl);
    k_fill_gaps<<<unsigned(c->n_sm) * 4, 256, 0, s>>>(oseg, gl);
  } else {
    k_zero_u64<<<grid_for(n + 1), kBlock, 0, s>>>(oseg, n + 1);   // oseg: the dT device's array
    GF_CHECK(c, cudaMemsetAsync(k.fpre[cur].p, 0, sizeof(unsigned long long), s));
  }
  out.det_id = det;
  out.prev_det = rows_ok ? k.cslot_det[prev] : 0;
  out.pos_valid = rows_ok && k.n_cand > 0;
  k.cslot_det[cur] = det;
  k.cslot_gen[cur] = k.cand_gen;
  k.cslot_cur ^= 1;
  // sphere-triangle / sphere-analytic pairs: per-sphere counts of kinds 1, 2
  static const bool sa_off = std::getenv("GF_NO_SA_CAND") != nullptr;
  const bool sa_cands = !sa_off && c->n_ana && !c->world_moving && k.sa_world_version == c->world_version;
  if (n && sa_cands) {
    // sphere-analytic pairs from the candidates; triangles (if any) as usual
    GF_CHECK(c, cudaMemsetAsync(cnt + 2 * n, 0, sizeof(unsigned long long) * n, s));
    if (c->n_tri)
      k_pairs_other<<<grid_for(n, 128), 128, 0, s>>>(v, cnt, k.tmp.as<uint2>(), tn, (unsigned long long)k.tmp_cap, 0);
    else
      GF_CHECK(c, cudaMemsetAsync(cnt + n, 0, sizeof(unsigned long long) * n, s));
    if (k.n_sa_cand)
      k_sa_filter<<<grid_for(k.n_sa_cand), kBlock, 0, s>>>(v, k.sa_cand.as<uint2>(), k.n_sa_cand, cnt,
                                                           k.tmp.as<uint2>(), tn, (unsigned long long)k.tmp_cap);
  } else if (n) {
    k_pairs_other<<<grid_for(n, 128), 128, 0, s>>>(v, cnt, k.tmp.as<uint2>(), tn, (unsigned long long)k.tmp_cap, 1);
  }
  // their segment starts follow the sphere-sphere block: exclusive scan of
  // counts[n, 3n] seeded with the block's size
  size_t tmp = 0;
  auto init = cub::FutureValue<unsigned long long>(ss_tot);
  cub::DeviceScan::ExclusiveScan(nullptr, tmp, cnt + n, oseg + n, cub::Sum(), init, int(2 * n + 1), s);
  if (ensure(c, k.cub_tmp, tmp + 16, s, false)) return -1;
  GF_CHECK(c, cub::DeviceScan::ExclusiveScan(k.cub_tmp.p, tmp, cnt + n, oseg + n, cub::Sum(), init, int(2 * n + 1),
                                             s));
  Status *st = c->status.as<Status>();
  GF_CHECK(c, cudaMemcpyAsync(&st->acs_total, oseg + 3 * n, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
  GF_CHECK(c, cudaMemcpyAsync(&hs->acs_total, &st->acs_total, sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, s));
  GF_CHECK(c, cudaMemcpyAsync(&hs->other_total, tn, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

// canonical (kind, a, b) array; keeps the segment offsets with the array for
// the next history remap.  Host has synced on the count phase.
int kt_detect_fill(Ctx *c, Acs &out, cudaStream_t s) {
  DevGuard g_kt(stream_device(s));   // the kT device of a 2-GPU split
  KtScratch &k = c->kt;
  const int64_t n = c->n_sph;
  Status *hs = reinterpret_cast<Status *>(c->h_status);
  for (int attempt = 0;; ++attempt) {
    const int64_t ss_total = int64_t(hs->acs_total) - int64_t(hs->other_total);
    const bool tmp_over = (int64_t)hs->other_total > k.tmp_cap;
    const bool ss_over = ss_total > out.cap - k.tmp_cap - 1;
    if (!tmp_over && !ss_over) break;
    if (attempt > 4) { c->err = "contact array sizing did not converge"; return -1; }
    // a scratch list or the sphere-sphere block overflowed: grow, redo
    if (tmp_over) {
      int64_t cap = int64_t(hs->other_total) + int64_t(hs->other_total) / 4 + 4096;
      if (ensure(c, k.tmp, sizeof(uint2) * cap, s)) return -1;
      k.tmp_cap = cap;
    }
    if (ss_over) k.ss_need = ss_total + ss_total / 8 + 1024;
    k.cslot_cur ^= 1;   // the redo rewrites the same detection's rows
    --k.det_serial;
    if (kt_count(c, s)) return -1;
    GF_CHECK(c, cudaStreamSynchronize(s));
    out.n = int64_t(hs->acs_total);
  }
  if (out.n > out.cap) { c->err = "contact array overflow"; return -1; }
  k.last_ss = int64_t(hs->acs_total) - int64_t(hs->other_total);
  if (n && out.n) {
    const unsigned long long *off = out.seg.as<unsigned long long>();
    GF_CHECK(c, cudaMemsetAsync(k.cursor.p, 0, sizeof(unsigned) * 3 * n, s));
    k_place<<<1184, 256, 0, s>>>(k.tmp_n.as<unsigned long long>(), n, k.tmp.as<uint2>(), off,
                                 k.cursor.as<unsigned>(), out.ids.as<uint2>());
    k_sort_seg<<<grid_for(2 * n), kBlock, 0, s>>>(2 * n, off + n, out.ids.as<uint2>());
  }
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

int kt_bin_ranges(Ctx *c, double margin, int64_t *h_out) {
  cudaStream_t s = c->s_kt;
  DevGuard g_kt(c->kt_device);
  const int64_t n = c->n_sph;
  DBuf tmp;
  if (ensure(c, tmp, sizeof(long long) * 6 * (n + 1), s)) return -1;
  k_bin_ranges<<<grid_for(n), kBlock, 0, s>>>(n, c->kt.c4.as<double>(), c->sph_offr.as<float4>(),
                                              c->kt.grid.as<Grid>(), margin, tmp.as<long long>());
  GF_CHECK(c, cudaMemcpyAsync(h_out, tmp.p, sizeof(long long) * 6 * n, cudaMemcpyDeviceToHost, s));
  GF_CHECK(c, cudaStreamSynchronize(s));
  cudaFree(tmp.p);
  return 0;
}


// Persistent contacts (bonded models, engine.py:639-662): an old row whose
// wildcard `col` is > 0 (an intact bond) that the new detection no longer
// holds is re-appended.  k_persist_mark flags them, k_persist_keys /
// k_persist_gather rebuild the array in canonical order.
__global__ void k_persist_mark(int64_t n_old, const uint2 *old_ids, const float *old_wild, int W, int col,
                               const uint2 *new_ids, const unsigned long long *new_seg, int64_t n_sph,
                               uint8_t *lost, unsigned long long *n_lost) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n_old) return;
  uint8_t l = 0;
  if (old_wild[int64_t(W) * i + col] > 0.0f) {
    const uint2 id = old_ids[i];
    const int64_t sg = int64_t(id.y >> kKindShift) * n_sph + id.x;
    bool found = false;
    for (unsigned long long q = new_seg[sg]; q < new_seg[sg + 1]; ++q) {
      const uint32_t y = new_ids[q].y;
      if (y == id.y) { found = true; break; }
      if (y > id.y) break;
    }
    l = found ? 0 : 1;
    if (l) atomicAdd(n_lost, 1ull);
  }
  lost[i] = l;
}

__device__ __forceinline__ unsigned long long persist_key(uint2 id) {
  return (static_cast<unsigned long long>(id.y >> kKindShift) << 60) |
         (static_cast<unsigned long long>(id.x) << 30) | static_cast<unsigned long long>(id.y & kSlotMask);
}

// keys of the new rows (source r) and of the lost old rows (source ~i),
// appended at the positions `pos` (exclusive scan of `lost`)
__global__ void k_persist_keys(int64_t n_new, const uint2 *new_ids, int64_t n_old, const uint2 *old_ids,
                               const uint8_t *lost, const unsigned long long *pos, unsigned long long *keys,
                               long long *src) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t < n_new) {
    keys[t] = persist_key(new_ids[t]);
    src[t] = t;
  } else if (t < n_new + n_old) {
    const int64_t i = t - n_new;
    if (lost[i]) {
      keys[n_new + pos[i]] = persist_key(old_ids[i]);
      src[n_new + pos[i]] = ~static_cast<long long>(i);
    }
  }
}

__global__ void k_persist_gather(int64_t n, const long long *src, const uint2 *new_ids, const float *new_wild,
                                 const uint2 *old_ids, const float *old_wild, int W, uint2 *out_ids,
                                 float *out_wild) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const long long s_ = src[k];
  const bool from_old = s_ < 0;
  const int64_t r = from_old ? ~s_ : s_;
  out_ids[k] = from_old ? old_ids[r] : new_ids[r];
  const float *w = (from_old ? old_wild : new_wild) + int64_t(W) * r;
  for (int q = 0; q < W; ++q) out_wild[int64_t(W) * k + q] = w[q];
}


// re-append the intact bonds the new detection dropped (rare; synchronises
// once per adoption while a persistent column is set)
static int persist_lost(Ctx *c, cudaStream_t s) {
  Acs &nw = c->acs_next;
  Acs &old = c->acs;
  const int W = c->wild_w;
  uint8_t *lost = nullptr;
  unsigned long long *cnt = nullptr, *pos = nullptr;
  GF_CHECK(c, cudaMallocAsync(&lost, size_t(old.n) + 1, s));
  GF_CHECK(c, cudaMallocAsync(&cnt, sizeof(unsigned long long), s));
  GF_CHECK(c, cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
  if (!nw.seg.p && build_segments(c, nw, s)) return -1;
  k_persist_mark<<<grid_for(old.n), kBlock, 0, s>>>(old.n, old.ids.as<uint2>(), old.wild.as<float>(), W,
                                                    c->persist_col, nw.ids.as<uint2>(),
                                                    nw.seg.as<unsigned long long>(), c->n_sph, lost, cnt);
  unsigned long long h_lost = 0;
  GF_CHECK(c, cudaMemcpyAsync(&h_lost, cnt, sizeof(h_lost), cudaMemcpyDeviceToHost, s));
  GF_CHECK(c, cudaStreamSynchronize(s));
  if (h_lost) {
    const int64_t n_tot = nw.n + int64_t(h_lost);
    unsigned long long *keys = nullptr, *keys2 = nullptr;
    long long *src = nullptr, *src2 = nullptr;
    uint2 *ids = nullptr;
    float *wild = nullptr;
    GF_CHECK(c, cudaMallocAsync(&pos, sizeof(unsigned long long) * (old.n + 1), s));
    GF_CHECK(c, cudaMallocAsync(&keys, sizeof(unsigned long long) * n_tot, s));
    GF_CHECK(c, cudaMallocAsync(&keys2, sizeof(unsigned long long) * n_tot, s));
    GF_CHECK(c, cudaMallocAsync(&src, sizeof(long long) * n_tot, s));
    GF_CHECK(c, cudaMallocAsync(&src2, sizeof(long long) * n_tot, s));
    GF_CHECK(c, cudaMallocAsync(&ids, sizeof(uint2) * n_tot, s));
    GF_CHECK(c, cudaMallocAsync(&wild, sizeof(float) * W * n_tot, s));
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, lost, pos, int(old.n), s);
    void *tmp = nullptr;
    GF_CHECK(c, cudaMallocAsync(&tmp, tb + 16, s));
    GF_CHECK(c, cub::DeviceScan::ExclusiveSum(tmp, tb, lost, pos, int(old.n), s));
    cudaFreeAsync(tmp, s);
    k_persist_keys<<<grid_for(nw.n + old.n), kBlock, 0, s>>>(nw.n, nw.ids.as<uint2>(), old.n, old.ids.as<uint2>(),
                                                             lost, pos, keys, src);
    tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, src, src2, int(n_tot), 0, 62, s);
    GF_CHECK(c, cudaMallocAsync(&tmp, tb + 16, s));
    GF_CHECK(c, cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, src, src2, int(n_tot), 0, 62, s));
    cudaFreeAsync(tmp, s);
    k_persist_gather<<<grid_for(n_tot), kBlock, 0, s>>>(n_tot, src2, nw.ids.as<uint2>(), nw.wild.as<float>(),
                                                        old.ids.as<uint2>(), old.wild.as<float>(), W, ids, wild);
    if (n_tot > nw.cap) {
      const int64_t cap = n_tot + n_tot / 4 + 1024;
      if (ensure(c, nw.ids, sizeof(uint2) * cap, s) || ensure(c, nw.wild, sizeof(float) * W * cap, s) ||
          ensure(c, nw.old_pos, sizeof(uint32_t) * cap, s))
        return -1;
      nw.cap = cap;
    }
    GF_CHECK(c, cudaMemcpyAsync(nw.ids.p, ids, sizeof(uint2) * n_tot, cudaMemcpyDeviceToDevice, s));
    GF_CHECK(c, cudaMemcpyAsync(nw.wild.p, wild, sizeof(float) * W * n_tot, cudaMemcpyDeviceToDevice, s));
    for (void *p : {static_cast<void *>(pos), static_cast<void *>(keys), static_cast<void *>(keys2),
                    static_cast<void *>(src), static_cast<void *>(src2), static_cast<void *>(ids),
                    static_cast<void *>(wild)})
      cudaFreeAsync(p, s);
    nw.n = n_tot;
    // the rows no longer mirror the candidate filter: the next adoption
    // searches segments instead of gathering by candidate rank
    nw.det_id = 0;
    nw.pos_valid = false;
    if (build_segments(c, nw, s)) return -1;
    c->persisted += int64_t(h_lost);
  }
  cudaFreeAsync(lost, s);
  cudaFreeAsync(cnt, s);
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

// adopt acs_next: remap history from acs, swap, rebuild incidence lists
int adopt_acs(Ctx *c, cudaStream_t s) {
  Acs &nw = c->acs_next;
  Acs &old = c->acs;
  if (nw.n && old.n && old.seg.p && nw.pos_valid && old.det_id != 0 && old.det_id == nw.prev_det)
    k_adopt_hist<<<unsigned((nw.n + kBlock * kAdoptPer - 1) / (kBlock * kAdoptPer)), kBlock, 0, s>>>(nw.n, nw.ids.as<uint2>(), nw.old_pos.as<uint32_t>(),
                                                  nw.seg.as<unsigned long long>(), nw.wild.as<float>(),
                                                  old.ids.as<uint2>(), old.wild.as<float>(),
                                                  old.seg.as<unsigned long long>(), c->n_sph, c->wild_w);
  else if (nw.n && old.n && old.seg.p)
    k_merge_seg<<<grid_for(nw.n), kBlock, 0, s>>>(nw.n, nw.ids.as<uint2>(), nw.wild.as<float>(),
                                                 old.ids.as<uint2>(), old.wild.as<float>(),
                                                 old.seg.as<unsigned long long>(), c->n_sph, c->wild_w);
  else if (nw.n)
    GF_CHECK(c, cudaMemsetAsync(nw.wild.p, 0, sizeof(float) * c->wild_w * nw.n, s));
  if (c->persist_col >= 0 && old.n && old.seg.p && persist_lost(c, s)) return -1;
  std::swap(c->acs, c->acs_next);
  c->ca_updates++;
  GF_CHECK(c, cudaGetLastError());
  return build_incidence(c, s);
}

// standalone history remap between two canonical arrays given as host
// buffers (broadphase.merge_history); ids are (a, b | kind << 30)
int merge_host(Ctx *c, int64_t n_old, const uint32_t *old_ids, const float *old_wild, int64_t n_new,
               const uint32_t *new_ids, int W, float *out_wild) {
  cudaStream_t s = c->s_dt;
  DBuf a, b, wa, wb;
  if (ensure(c, a, 8 * (n_old + 1), s) || ensure(c, b, 8 * (n_new + 1), s) ||
      ensure(c, wa, 4 * W * (n_old + 1), s) || ensure(c, wb, 4 * W * (n_new + 1), s))
    return -1;
  if (n_old) {
    if (h2d(c, a.p, old_ids, 8 * n_old, s)) return -1;
    if (h2d(c, wa.p, old_wild, 4 * W * n_old, s)) return -1;
  }
  if (n_new) {
    if (h2d(c, b.p, new_ids, 8 * n_new, s)) return -1;
    k_merge<<<grid_for(n_new), kBlock, 0, s>>>(n_new, b.as<uint2>(), wb.as<float>(), n_old, a.as<uint2>(),
                                              wa.as<float>(), W);
    GF_CHECK(c, cudaGetLastError());
    GF_CHECK(c, cudaMemcpyAsync(out_wild, wb.p, 4 * W * n_new, cudaMemcpyDeviceToHost, s));
    GF_CHECK(c, cudaStreamSynchronize(s));
  }
  cudaFree(a.p); cudaFree(b.p); cudaFree(wa.p); cudaFree(wb.p);
  return 0;
}

// per-(kind, sphere) segment offsets of an array installed from the host
int build_segments(Ctx *c, Acs &a, cudaStream_t s) {
  const int64_t n = c->n_sph;
  KtScratch &k = c->kt;
  if (ensure(c, a.seg, sizeof(unsigned long long) * (3 * n + 1), s) ||
      ensure(c, k.counts, sizeof(unsigned long long) * (3 * n + 1), s))
    return -1;
  unsigned long long *cnt = k.counts.as<unsigned long long>();
  GF_CHECK(c, cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (3 * n + 1), s));
  if (a.n) k_seg_count<<<grid_for(a.n), kBlock, 0, s>>>(a.n, a.ids.as<uint2>(), n, cnt);
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, a.seg.as<unsigned long long>(), int(3 * n + 1), s);
  if (ensure(c, k.cub_tmp, tmp + 16, s, false)) return -1;
  GF_CHECK(c, cub::DeviceScan::ExclusiveSum(k.cub_tmp.p, tmp, cnt, a.seg.as<unsigned long long>(),
                                            int(3 * n + 1), s));
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

int build_incidence(Ctx *c, cudaStream_t s) {
  const int64_t n = c->acs.n;
  const int64_t cap = std::max<int64_t>(c->acs.cap, 1);
  // compacted lists of touching entries: sphere-sphere (uint4 records of the
  // split path) at [0, 4 cap) words, the other kinds at [4 cap, 5 cap); the
  // fused throughput path needs only the second (tlist_words says which)
  c->tlist_words = ss_fused(c) ? 1 : 5;
  if (ensure(c, c->tlist, c->tlist_words * sizeof(uint32_t) * cap, s) || ensure(c, c->tlist_n, 16, s)) return -1;
  c->tlist_cap = cap;
  if (c->fixed_reduce) return 0;  // throughput build reduces with atomics
  if (ensure(c, c->out_c, sizeof(double) * 9 * cap, s) || ensure(c, c->touch, cap, s) ||
      ensure(c, c->inc, sizeof(uint32_t) * cap, s) || ensure(c, c->inc_alt, sizeof(uint32_t) * cap, s) ||
      ensure(c, c->inc_key, sizeof(uint32_t) * cap, s) ||
      ensure(c, c->inc_key_alt, sizeof(uint32_t) * cap, s) ||
      ensure(c, c->inc_start, sizeof(uint32_t) * (c->n_owner + 2), s) ||
      ensure(c, c->heavy, sizeof(uint32_t) * (c->n_owner + 1), s))
    return -1;
  if (!c->acs.seg.p && build_segments(c, c->acs, s)) return -1;
  if (n) {
    k_inc_keys<<<grid_for(n), kBlock, 0, s>>>(n, c->acs.ids.as<uint2>(), c->sph_owner.as<uint32_t>(),
                                             c->tri_owner.as<uint32_t>(), c->ana_owner.as<uint32_t>(),
                                             c->inc_key.as<uint32_t>(), c->inc.as<uint32_t>());
    int bits = 1;
    while ((int64_t(1) << bits) < c->n_owner + 1) ++bits;
    size_t tmp = 0;
    cub::DoubleBuffer<uint32_t> dk(c->inc_key.as<uint32_t>(), c->inc_key_alt.as<uint32_t>());
    cub::DoubleBuffer<uint32_t> dv(c->inc.as<uint32_t>(), c->inc_alt.as<uint32_t>());
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, int(n), 0, bits, s);
    if (ensure(c, c->cub_tmp_dt, tmp + 16, s)) return -1;
    GF_CHECK(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp_dt.p, tmp, dk, dv, int(n), 0, bits, s));
    if (dk.Current() != c->inc_key.as<uint32_t>()) {
      std::swap(c->inc_key, c->inc_key_alt);
      std::swap(c->inc, c->inc_alt);
    }
  }
  GF_CHECK(c, cudaMemsetAsync(c->heavy_count.p, 0, sizeof(unsigned long long), s));
  k_inc_start<<<grid_for(c->n_owner + 1), kBlock, 0, s>>>(
      c->n_owner, n, c->inc_key.as<uint32_t>(), c->inc_start.as<uint32_t>(),
      c->acs.seg.as<unsigned long long>(), c->sph_first.as<uint32_t>(), c->n_sph,
      c->heavy.as<uint32_t>(), c->heavy_count.as<unsigned long long>(), kHeavyThreshold);
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

}  // namespace gf
