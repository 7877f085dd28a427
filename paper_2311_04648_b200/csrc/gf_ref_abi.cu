// gf_ref_abi.cu -- the reference's per-kernel dT entry points on the device,
// in the reference's own array layouts (include/gf_b200.h, "reference-shaped
// entry points"):
//   gf_contact_forces         make_contact_kernel's sweep (forces.py:547-593)
//   gf_eval_core              a model core over a batch of contexts
//                             (forces.py:82-87; ForceModel.core / evaluate)
//   gf_reduce                 reduce_to_owners (_kernels.py:515-545) + the
//                             wrapper's m g term (forces.py:600-614)
//   gf_integrate_and_refresh  integrate_step + encode / decode + sphere
//                             centres (_kernels.py:548-670)
// They serve per-contact / per-kernel parity (the fused production step is
// gf_run) and the Python plugin surface.  Host buffers in, host buffers out:
// each call stages its arrays through stream-ordered device allocations on
// the context's dT stream and returns when the results are back.
// Compiled with -fmad=false: fp64 statement-by-statement like numba
// (fastmath=False).
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/gf_b200.h"
#include "gf_context.h"
#include "gf_device.cuh"

struct gf_ctx {
  gf::Ctx c;
};

namespace gf {
namespace {

// stream-ordered staging of one call's arrays; freed (stream-ordered) at scope exit
struct Stage {
  Ctx *c;
  cudaStream_t s;
  std::vector<void *> bufs;
  bool failed = false;
  explicit Stage(Ctx *cc) : c(cc), s(cc->s_dt) {}
  ~Stage() {
    for (void *p : bufs) cudaFreeAsync(p, s);
  }
  template <class T> T *alloc(size_t count) {
    if (failed || count == 0) return nullptr;
    void *p = nullptr;
    if (cudaMallocAsync(&p, count * sizeof(T), s) != cudaSuccess) {
      failed = true;
      set_err(c, "device allocation failed in a reference-shaped entry point");
      return nullptr;
    }
    bufs.push_back(p);
    return reinterpret_cast<T *>(p);
  }
  template <class T> T *in(const T *src, size_t count) {
    T *d = alloc<T>(count);
    if (d && src && cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, s) != cudaSuccess) failed = true;
    return d;
  }
  // a NULL source reads as zeros (optional inputs such as external loads)
  template <class T> T *in_or_zero(const T *src, size_t count) {
    if (src) return in(src, count);
    T *d = alloc<T>(count);
    if (d && cudaMemsetAsync(d, 0, count * sizeof(T), s) != cudaSuccess) failed = true;
    return d;
  }
  template <class T> void out(T *dst, const T *src, size_t count) {
    if (!failed && dst && src && count && cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, s) != cudaSuccess)
      failed = true;
  }
  int finish() {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      set_err(c, std::string("reference-shaped entry point: ") + cudaGetErrorString(e));
      return -1;
    }
    return failed ? -1 : 0;
  }
};

unsigned grid_of(int64_t n, int block) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + block - 1) / block, int64_t(148) * 32)));
}

// beta(CoR) per material pair with the host libm the reference's kernel
// calls (forces.py:41-44 / :122)
std::vector<double> beta_of(const double *pair_stack, int n_mat) {
  const int mm = n_mat * n_mat;
  std::vector<double> b(size_t(mm), 0.0);
  for (int q = 0; q < mm; ++q) {
    const double cor = pair_stack[2 * mm + q];
    const double loge = cor < 1e-12 ? std::log(1e-12) : std::log(cor);
    b[size_t(q)] = loge / std::sqrt(loge * loge + kPi * kPi);
  }
  return b;
}

__global__ void __launch_bounds__(128) k_ref_contacts_hm(RefContacts r) { ref_contacts_loop<HmCore>(r); }
__global__ void __launch_bounds__(128) k_core_batch_hm(CoreBatch b) { core_batch_loop<HmCore>(b); }

// reduce_to_owners: incidence keys (owner << 33 | k << 1 | side), sorted, so
// each owner sums its contributions in the reference loop's order
__global__ void k_red_keys(int64_t n, const int64_t *oa, const int64_t *ob, unsigned long long *keys) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
    keys[2 * k] = (static_cast<unsigned long long>(oa[k]) << 33) | (static_cast<unsigned long long>(k) << 1);
    keys[2 * k + 1] = (static_cast<unsigned long long>(ob[k]) << 33) | (static_cast<unsigned long long>(k) << 1) | 1ull;
  }
}

__global__ void k_red_starts(int64_t m, int64_t n_owner, const unsigned long long *keys, int64_t *start) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= m; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t o = i < m ? int64_t(keys[i] >> 33) : n_owner;
    const int64_t p = i > 0 ? int64_t(keys[i - 1] >> 33) : -1;
    for (int64_t q = p + 1; q <= o && q <= n_owner; ++q) start[q] = i;
  }
}

__global__ void k_red_owners(int64_t n_owner, const unsigned long long *keys, const int64_t *start,
                             const double *forces, const double *tofs, const double *cps, const double *owner_pos,
                             const double *mass, double gx, double gy, double gz, double *acc_f, double *acc_t) {
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < n_owner; o += int64_t(gridDim.x) * blockDim.x) {
    double f[3] = {0.0, 0.0, 0.0}, t[3] = {0.0, 0.0, 0.0};
    const double px = owner_pos[3 * o], py = owner_pos[3 * o + 1], pz = owner_pos[3 * o + 2];
    for (int64_t i = start[o]; i < start[o + 1]; ++i) {
      const unsigned long long key = keys[i];
      const int64_t k = int64_t((key >> 1) & 0xFFFFFFFFull);
      const double fx = forces[3 * k], fy = forces[3 * k + 1], fz = forces[3 * k + 2];
      const double tx = fx + tofs[3 * k], ty = fy + tofs[3 * k + 1], tz = fz + tofs[3 * k + 2];
      const double rx = cps[3 * k] - px, ry = cps[3 * k + 1] - py, rz = cps[3 * k + 2] - pz;
      if (key & 1ull) {
        f[0] -= fx; f[1] -= fy; f[2] -= fz;
        t[0] -= ry * tz - rz * ty; t[1] -= rz * tx - rx * tz; t[2] -= rx * ty - ry * tx;
      } else {
        f[0] += fx; f[1] += fy; f[2] += fz;
        t[0] += ry * tz - rz * ty; t[1] += rz * tx - rx * tz; t[2] += rx * ty - ry * tx;
      }
    }
    if (mass) {   // acc_f += mass[:, None] * gravity (forces.py:613)
      const double m = mass[o];
      f[0] += m * gx; f[1] += m * gy; f[2] += m * gz;
    }
    for (int q = 0; q < 3; ++q) { acc_f[3 * o + q] = f[q]; acc_t[3 * o + q] = t[q]; }
  }
}

struct RefIntegrate {
  double h, gx, gy, gz, v_err;
  int64_t n;
  double *pos;
  float *quat;
  double *lin_vel, *ang_vel;
  const double *mass, *moi, *acc_f, *acc_t, *ext_f, *ext_t;
  const uint8_t *family, *fixed_flag, *lv_mask, *av_mask, *prescribed;
  const double *lv_val, *av_val;
  unsigned long long *bad, *oob;   // first offending owner (min index)
  Domain dom;
};

// integrate_step (_kernels.py:548-636), one thread per owner
__global__ void k_ref_integrate(RefIntegrate r) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < r.n; i += int64_t(gridDim.x) * blockDim.x) {
    const int fam = r.family[i];
    double *lv = r.lin_vel + 3 * i, *av = r.ang_vel + 3 * i;
    if (r.fixed_flag[fam]) {
      lv[0] = 0.0; lv[1] = 0.0; lv[2] = 0.0;
      av[0] = 0.0; av[1] = 0.0; av[2] = 0.0;
      continue;
    }
    float *qf = r.quat + 4 * i;
    double qw = double(qf[0]), qx = double(qf[1]), qy = double(qf[2]), qz = double(qf[3]);
    double vx, vy, vz, wx, wy, wz;
    if (r.prescribed[fam]) {
      vx = lv[0]; vy = lv[1]; vz = lv[2];
      if (r.lv_mask[3 * fam]) vx = r.lv_val[3 * fam];
      if (r.lv_mask[3 * fam + 1]) vy = r.lv_val[3 * fam + 1];
      if (r.lv_mask[3 * fam + 2]) vz = r.lv_val[3 * fam + 2];
      wx = av[0]; wy = av[1]; wz = av[2];
      if (r.av_mask[3 * fam] || r.av_mask[3 * fam + 1] || r.av_mask[3 * fam + 2]) {
        double pwx, pwy, pwz;
        qrot(qw, qx, qy, qz, wx, wy, wz, pwx, pwy, pwz);
        if (r.av_mask[3 * fam]) pwx = r.av_val[3 * fam];
        if (r.av_mask[3 * fam + 1]) pwy = r.av_val[3 * fam + 1];
        if (r.av_mask[3 * fam + 2]) pwz = r.av_val[3 * fam + 2];
        qrot(qw, -qx, -qy, -qz, pwx, pwy, pwz, wx, wy, wz);
      }
    } else {
      const double m = r.mass[i];
      const double *af = r.acc_f + 3 * i, *at = r.acc_t + 3 * i, *ef = r.ext_f + 3 * i, *et = r.ext_t + 3 * i;
      vx = lv[0] + r.h * ((af[0] + ef[0]) / m + r.gx);
      vy = lv[1] + r.h * ((af[1] + ef[1]) / m + r.gy);
      vz = lv[2] + r.h * ((af[2] + ef[2]) / m + r.gz);
      const double tgx = at[0] + et[0], tgy = at[1] + et[1], tgz = at[2] + et[2];
      double tlx, tly, tlz;
      qrot(qw, -qx, -qy, -qz, tgx, tgy, tgz, tlx, tly, tlz);
      wx = av[0]; wy = av[1]; wz = av[2];
      const double ix = r.moi[3 * i], iy = r.moi[3 * i + 1], iz = r.moi[3 * i + 2];
      const double gyx = wy * (iz * wz) - wz * (iy * wy);
      const double gyy = wz * (ix * wx) - wx * (iz * wz);
      const double gyz = wx * (iy * wy) - wy * (ix * wx);
      wx += r.h * (tlx - gyx) / ix;
      wy += r.h * (tly - gyy) / iy;
      wz += r.h * (tlz - gyz) / iz;
    }
    double *p = r.pos + 3 * i;
    p[0] += r.h * vx;
    p[1] += r.h * vy;
    p[2] += r.h * vz;
    const double hw = 0.5 * r.h;
    const double dqw = hw * (-qx * wx - qy * wy - qz * wz);
    const double dqx = hw * (qw * wx + qy * wz - qz * wy);
    const double dqy = hw * (qw * wy + qz * wx - qx * wz);
    const double dqz = hw * (qw * wz + qx * wy - qy * wx);
    qw += dqw; qx += dqx; qy += dqy; qz += dqz;
    const double inv = 1.0 / sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    qf[0] = float(qw * inv); qf[1] = float(qx * inv); qf[2] = float(qy * inv); qf[3] = float(qz * inv);
    lv[0] = vx; lv[1] = vy; lv[2] = vz;
    av[0] = wx; av[1] = wy; av[2] = wz;
    if (vx * vx + vy * vy + vz * vz > r.v_err * r.v_err) atomicMin(r.bad, (unsigned long long)i);
  }
}

// first owner outside the domain box (encode_positions' early return)
__global__ void k_ref_oob(RefIntegrate r) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < r.n; i += int64_t(gridDim.x) * blockDim.x) {
    const double *p = r.pos + 3 * i;
    for (int ax = 0; ax < 3; ++ax)
      if (p[ax] < r.dom.lo[ax] || p[ax] > r.dom.hi[ax]) atomicMin(r.oob, (unsigned long long)i);
  }
}

// encode_positions up to the first out-of-domain owner (that owner's
// sub-voxels of the axes before the failing one are written, as the
// reference's loop does), then -- when every owner encoded -- decode back
// into owner_pos (_kernels.py:654-657)
__global__ void k_ref_encode(RefIntegrate r, uint64_t *voxel, uint16_t *sub) {
  const unsigned long long oob = *r.oob;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < r.n; i += int64_t(gridDim.x) * blockDim.x) {
    if ((unsigned long long)i > oob) continue;
    double *p = r.pos + 3 * i;
    uint64_t v = 0;
    bool ok = true;
    for (int ax = 0; ax < 3 && ok; ++ax) {
      if (p[ax] < r.dom.lo[ax] || p[ax] > r.dom.hi[ax]) { ok = false; break; }
      const double t = sub_(p[ax], r.dom.lo[ax]) / r.dom.edge;
      long long cell = (long long)t;
      if (cell >= kVoxPerAxis) cell = kVoxPerAxis - 1;
      long long q = (long long)mul(sub_(t, double(cell)), double(kSubPerEdge));
      if (q >= kSubPerEdge) q = kSubPerEdge - 1;
      v |= uint64_t(cell) << (kVoxBits * ax);
      sub[3 * i + ax] = (uint16_t)q;
    }
    if (!ok) continue;
    voxel[i] = v;
    if (oob == ~0ull) {
      double x, y, z;
      decode_pos(r.dom, v, make_ushort4(sub[3 * i], sub[3 * i + 1], sub[3 * i + 2], 0), x, y, z);
      p[0] = x; p[1] = y; p[2] = z;
    }
  }
}

// sphere world centres from the refreshed owner poses (_kernels.py:658-669)
__global__ void k_ref_centres(int64_t n_s, const int64_t *sph_geom, const float *geom_params, const int64_t *geom_owner,
                              const double *pos, const float *quat, double *centres) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n_s; k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t g = sph_geom[k], o = geom_owner[g];
    const float *prm = geom_params + 9 * g;
    const float *q = quat + 4 * o;
    double rx, ry, rz;
    qrot(double(q[0]), double(q[1]), double(q[2]), double(q[3]), double(prm[0]), double(prm[1]), double(prm[2]),
         rx, ry, rz);
    centres[3 * k] = pos[3 * o] + rx;
    centres[3 * k + 1] = pos[3 * o + 1] + ry;
    centres[3 * k + 2] = pos[3 * o + 2] + rz;
  }
}


// one output frame's per-sphere columns (io.write_sphere_csv, io.py:132-166):
// centre xyz, |v| of the owner (fp64, the reference's summation order),
// family, owner v xyz; device sphere slot order
__global__ void k_sphere_frame(Spheres sph, Owners own, int f32, double *out) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < sph.n; k += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t o = sph.owner[k];
    const double4 c = sph.center[k];
    double v[3];
    for (int a = 0; a < 3; ++a)
      v[a] = f32 ? double(reinterpret_cast<const float *>(own.lin_vel)[4 * size_t(o) + a])
                 : reinterpret_cast<const double *>(own.lin_vel)[4 * size_t(o) + a];
    double *w = out + 8 * k;
    w[0] = c.x; w[1] = c.y; w[2] = c.z;
    w[3] = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
    w[4] = double(meta_family(own.meta[o]));
    w[5] = v[0]; w[6] = v[1]; w[7] = v[2];
  }
}
}  // namespace
}  // namespace gf

using namespace gf;

extern "C" {

int gf_contact_forces(gf_ctx *ctx, int64_t n, const uint8_t *kind, const int64_t *slot_a, const int64_t *slot_b,
                      const int64_t *owner_a, const int64_t *owner_b, const uint8_t *mat_a, const uint8_t *mat_b,
                      int64_t n_sph, const double *sph_centers, const float *sph_radii, int64_t n_tri,
                      const double *tri_world, int64_t n_ana, const double *ana_world, const uint8_t *ana_kind,
                      int64_t n_owner, const double *owner_pos, const double *lin_vel, const double *ang_vel_global,
                      const double *mass, int n_mat, int n_rows, const double *pair_stack, float *wild, int W,
                      double ts, double sim_time, double *out_ft, double *depth, double *cp, int64_t *touching) {
  if (!ctx) return -1;
  Ctx *c = &ctx->c;
  if (cudaSetDevice(c->device) != cudaSuccess) return -1;
  if (n < 0 || n_mat <= 0 || n_rows < 2) {
    set_err(c, "gf_contact_forces: bad sizes");
    return -1;
  }
  if (c->user_model ? !c->user_fn_ref : W != 4) {
    set_err(c, "gf_contact_forces: the wildcard width does not match the context's force model");
    return -1;
  }
  if (touching) *touching = 0;
  if (n == 0) return 0;
  Stage S(c);
  const size_t mm = size_t(n_mat) * n_mat;
  RefContacts r;
  r.n = n;
  r.kind = S.in(kind, n);
  r.slot_a = S.in(slot_a, n);
  r.slot_b = S.in(slot_b, n);
  r.owner_a = S.in(owner_a, n);
  r.owner_b = S.in(owner_b, n);
  r.mat_a = S.in(mat_a, n);
  r.mat_b = S.in(mat_b, n);
  r.sph_centers = S.in(sph_centers, 3 * size_t(n_sph));
  r.sph_radii = S.in(sph_radii, size_t(n_sph));
  r.tri_world = S.in(tri_world, 9 * size_t(n_tri));
  r.ana_world = S.in(ana_world, 8 * size_t(n_ana));
  r.ana_kind = S.in(ana_kind, size_t(n_ana));
  r.owner_pos = S.in(owner_pos, 3 * size_t(n_owner));
  r.lin_vel = S.in(lin_vel, 3 * size_t(n_owner));
  r.ang_vel_global = S.in(ang_vel_global, 3 * size_t(n_owner));
  r.mass = S.in(mass, size_t(n_owner));
  const std::vector<double> beta = beta_of(pair_stack, n_mat);
  r.mat.n_mat = n_mat;
  r.mat.pair = S.in(pair_stack, size_t(n_rows) * mm);
  r.mat.beta = S.in(beta.data(), mm);
  r.wild = S.in(wild, size_t(W) * n);
  r.W = W;
  r.ts = ts;
  r.sim_time = sim_time;
  r.out_ft = S.alloc<double>(6 * size_t(n));
  r.depth = S.alloc<double>(size_t(n));
  r.cp = S.alloc<double>(3 * size_t(n));
  r.touching = S.alloc<unsigned long long>(1);
  if (S.failed) return S.finish();
  cudaMemsetAsync(r.touching, 0, sizeof(unsigned long long), S.s);
  if (c->user_model) {
    void *args[] = {&r};
    if (cudaLaunchKernel(reinterpret_cast<const void *>(c->user_fn_ref), dim3(grid_of(n, 128)), dim3(128), args, 0,
                         S.s) != cudaSuccess)
      S.failed = true;
  } else {
    k_ref_contacts_hm<<<grid_of(n, 128), 128, 0, S.s>>>(r);
  }
  unsigned long long tch = 0;
  S.out(wild, r.wild, size_t(W) * n);
  S.out(out_ft, r.out_ft, 6 * size_t(n));
  S.out(depth, r.depth, size_t(n));
  S.out(cp, r.cp, 3 * size_t(n));
  S.out(&tch, r.touching, 1);
  const int rc = S.finish();
  if (touching) *touching = int64_t(tch);
  return rc;
}

int gf_eval_core(gf_ctx *ctx, int64_t n, const double *args, const int32_t *mats, int n_mat, int n_rows,
                 const double *pair_stack, float *wild, int W, double *out) {
  if (!ctx) return -1;
  Ctx *c = &ctx->c;
  if (cudaSetDevice(c->device) != cudaSuccess) return -1;
  if (n < 0 || n_mat <= 0 || n_rows < 2) {
    set_err(c, "gf_eval_core: bad sizes");
    return -1;
  }
  if (c->user_model ? !c->user_fn_batch : W != 4) {
    set_err(c, "gf_eval_core: the wildcard width does not match the context's force model");
    return -1;
  }
  if (n == 0) return 0;
  Stage S(c);
  const size_t mm = size_t(n_mat) * n_mat;
  CoreBatch b;
  b.n = n;
  b.args = S.in(args, 15 * size_t(n));
  b.mats = S.in(mats, 2 * size_t(n));
  const std::vector<double> beta = beta_of(pair_stack, n_mat);
  b.mat.n_mat = n_mat;
  b.mat.pair = S.in(pair_stack, size_t(n_rows) * mm);
  b.mat.beta = S.in(beta.data(), mm);
  b.wild = S.in(wild, size_t(W) * n);
  b.W = W;
  b.out = S.alloc<double>(6 * size_t(n));
  if (S.failed) return S.finish();
  if (c->user_model) {
    void *kargs[] = {&b};
    if (cudaLaunchKernel(reinterpret_cast<const void *>(c->user_fn_batch), dim3(grid_of(n, 128)), dim3(128), kargs,
                         0, S.s) != cudaSuccess)
      S.failed = true;
  } else {
    k_core_batch_hm<<<grid_of(n, 128), 128, 0, S.s>>>(b);
  }
  S.out(wild, b.wild, size_t(W) * n);
  S.out(out, b.out, 6 * size_t(n));
  return S.finish();
}

int gf_reduce(gf_ctx *ctx, int64_t n, const int64_t *owner_a, const int64_t *owner_b, const double *forces,
              const double *tofs, const double *cps, int64_t n_owner, const double *owner_pos, const double *mass,
              const double *gravity3, double *acc_force, double *acc_torque) {
  if (!ctx) return -1;
  Ctx *c = &ctx->c;
  if (cudaSetDevice(c->device) != cudaSuccess) return -1;
  if (n < 0 || n_owner < 0 || n >= (int64_t(1) << 31) || n_owner >= (int64_t(1) << 30)) {
    set_err(c, "gf_reduce: sizes out of range");
    return -1;
  }
  if (n_owner == 0) return 0;
  Stage S(c);
  const int64_t m = 2 * n;
  const int64_t *oa = S.in(owner_a, size_t(n)), *ob = S.in(owner_b, size_t(n));
  const double *f = S.in(forces, 3 * size_t(n)), *t = S.in(tofs, 3 * size_t(n)), *p = S.in(cps, 3 * size_t(n));
  const double *pos = S.in(owner_pos, 3 * size_t(n_owner));
  const double *ms = mass ? S.in(mass, size_t(n_owner)) : nullptr;
  unsigned long long *keys = S.alloc<unsigned long long>(size_t(std::max<int64_t>(m, 1)));
  unsigned long long *keys2 = S.alloc<unsigned long long>(size_t(std::max<int64_t>(m, 1)));
  int64_t *start = S.alloc<int64_t>(size_t(n_owner) + 1);
  double *af = S.alloc<double>(3 * size_t(n_owner)), *at = S.alloc<double>(3 * size_t(n_owner));
  if (S.failed) return S.finish();
  const unsigned long long *sorted = keys;
  if (m > 0) {
    k_red_keys<<<grid_of(n, 256), 256, 0, S.s>>>(n, oa, ob, keys);
    int bits = 34;
    while ((int64_t(1) << (bits - 33)) <= n_owner) ++bits;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, keys2, int(m), 0, bits, S.s);
    void *tmp = S.alloc<char>(tmp_bytes);
    if (S.failed) return S.finish();
    cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, keys2, int(m), 0, bits, S.s);
    sorted = keys2;
  }
  k_red_starts<<<grid_of(m + 1, 256), 256, 0, S.s>>>(m, n_owner, sorted, start);
  const double g0 = gravity3 ? gravity3[0] : 0.0, g1 = gravity3 ? gravity3[1] : 0.0, g2 = gravity3 ? gravity3[2] : 0.0;
  k_red_owners<<<grid_of(n_owner, 128), 128, 0, S.s>>>(n_owner, sorted, start, f, t, p, pos, ms, g0, g1, g2, af, at);
  S.out(acc_force, af, 3 * size_t(n_owner));
  S.out(acc_torque, at, 3 * size_t(n_owner));
  return S.finish();
}

int gf_integrate_and_refresh(gf_ctx *ctx, double h, const double *g3, int64_t n, double *owner_pos, float *quat,
                             double *lin_vel, double *ang_vel, const double *mass, const double *moi,
                             const double *acc_force, const double *acc_torque, const double *ext_force,
                             const double *ext_torque, const uint8_t *family, const uint8_t *fixed_flag,
                             const uint8_t *lv_mask, const double *lv_val, const uint8_t *av_mask,
                             const double *av_val, const uint8_t *prescribed_flag, double v_err, const double *lo3,
                             const double *hi3, double edge, uint64_t *voxel, uint16_t *sub, int64_t n_s,
                             const int64_t *sph_geom, int64_t n_geom, const float *geom_params,
                             const int64_t *geom_owner, double *sph_centers, int64_t *bad, int64_t *oob) {
  if (!ctx) return -1;
  Ctx *c = &ctx->c;
  if (cudaSetDevice(c->device) != cudaSuccess) return -1;
  if (n < 0 || n_s < 0 || !g3 || !lo3 || !hi3) {
    set_err(c, "gf_integrate_and_refresh: bad arguments");
    return -1;
  }
  if (bad) *bad = -1;
  if (oob) *oob = -1;
  if (n == 0) return 0;
  Stage S(c);
  RefIntegrate r;
  r.h = h; r.gx = g3[0]; r.gy = g3[1]; r.gz = g3[2]; r.v_err = v_err;
  r.n = n;
  r.pos = S.in(owner_pos, 3 * size_t(n));
  r.quat = S.in(quat, 4 * size_t(n));
  r.lin_vel = S.in(lin_vel, 3 * size_t(n));
  r.ang_vel = S.in(ang_vel, 3 * size_t(n));
  r.mass = S.in(mass, size_t(n));
  r.moi = S.in(moi, 3 * size_t(n));
  r.acc_f = S.in_or_zero(acc_force, 3 * size_t(n));
  r.acc_t = S.in_or_zero(acc_torque, 3 * size_t(n));
  r.ext_f = S.in_or_zero(ext_force, 3 * size_t(n));
  r.ext_t = S.in_or_zero(ext_torque, 3 * size_t(n));
  r.family = S.in(family, size_t(n));
  r.fixed_flag = S.in(fixed_flag, 256);
  r.lv_mask = S.in(lv_mask, 256 * 3);
  r.lv_val = S.in(lv_val, 256 * 3);
  r.av_mask = S.in(av_mask, 256 * 3);
  r.av_val = S.in(av_val, 256 * 3);
  r.prescribed = S.in(prescribed_flag, 256);
  unsigned long long *flags = S.alloc<unsigned long long>(2);
  r.bad = flags;
  r.oob = flags ? flags + 1 : nullptr;
  for (int ax = 0; ax < 3; ++ax) { r.dom.lo[ax] = lo3[ax]; r.dom.hi[ax] = hi3[ax]; }
  r.dom.edge = edge;
  uint64_t *vox = S.in(voxel, size_t(n));
  uint16_t *sb = S.in(sub, 3 * size_t(n));
  const int64_t *sg = S.in(sph_geom, size_t(n_s));
  const float *gp = S.in(geom_params, 9 * size_t(n_geom));
  const int64_t *go = S.in(geom_owner, size_t(n_geom));
  double *cen = S.alloc<double>(3 * size_t(n_s));
  if (S.failed) return S.finish();
  cudaMemsetAsync(flags, 0xFF, 2 * sizeof(unsigned long long), S.s);
  k_ref_integrate<<<grid_of(n, 128), 128, 0, S.s>>>(r);
  k_ref_oob<<<grid_of(n, 256), 256, 0, S.s>>>(r);
  k_ref_encode<<<grid_of(n, 256), 256, 0, S.s>>>(r, vox, sb);
  unsigned long long hf[2] = {~0ull, ~0ull};
  S.out(hf, flags, 2);
  if (S.finish()) return -1;
  if (hf[1] == ~0ull && n_s > 0)
    k_ref_centres<<<grid_of(n_s, 256), 256, 0, S.s>>>(n_s, sg, gp, go, r.pos, r.quat, cen);
  S.out(owner_pos, r.pos, 3 * size_t(n));
  S.out(quat, r.quat, 4 * size_t(n));
  S.out(lin_vel, r.lin_vel, 3 * size_t(n));
  S.out(ang_vel, r.ang_vel, 3 * size_t(n));
  S.out(voxel, vox, size_t(n));
  S.out(sub, sb, 3 * size_t(n));
  if (hf[1] == ~0ull) S.out(sph_centers, cen, 3 * size_t(n_s));
  const int rc = S.finish();
  if (bad) *bad = hf[0] == ~0ull ? -1 : int64_t(hf[0]);
  if (oob) *oob = hf[1] == ~0ull ? -1 : int64_t(hf[1]);
  return rc;
}

int gf_sphere_frame(gf_ctx *ctx, double *out) {
  if (!ctx) return -1;
  Ctx *c = &ctx->c;
  if (cudaSetDevice(c->device) != cudaSuccess) return -1;
  if (!c->n_sph) return 0;
  Stage S(c);
  double *d = S.alloc<double>(8 * size_t(c->n_sph));
  if (S.failed) return S.finish();
  k_sphere_frame<<<grid_of(c->n_sph, 256), 256, 0, S.s>>>(spheres_view(c), owners_view(c), c->f32_state ? 1 : 0, d);
  S.out(out, d, 8 * size_t(c->n_sph));
  return S.finish();
}

}  // extern "C"
