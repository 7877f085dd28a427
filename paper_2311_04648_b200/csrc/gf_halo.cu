// gf_halo.cu -- halo exchange kernels of the spatial decomposition.
//
// A decomposed run gives every rank a context holding its local owners, the
// ghost copies of neighbouring ranks' owners within the halo width, and the
// replicated boundary owners (gf_common.cuh, kDd*).  Per step:
//   forces      contacts computed on this rank (dd_keep decides which)
//   ghost forces pack_forces on the ghosts -> their home rank -> add_forces
//   integrate   local and shared owners (ghosts skipped)
//   ghost state pack_state on the home rank -> unpack_state into the ghosts
// The transport between ranks (NCCL over NVLink, or a device copy for two
// contexts on one GPU) is the caller's; these kernels only gather / scatter
// fixed-size records by owner index, on the context's dT stream.
//
// State record (32 + 2 * sizeof(VelT[4]) bytes): voxel u64 | sub ushort4 |
// quat float4 | lin_vel VelT[4] | ang_vel VelT[4] -- the owner's complete
// dynamic state, copied bit for bit (engine.py:_step_once reads nothing else
// of an owner during a step).  Force record (48 bytes): the six fixed-point
// accumulator words, or fp64 bit patterns for boundary owners.
#include "gf_context.h"

namespace gf {

namespace {

// one thread per 16-byte word of the packed records
__global__ void k_pack_state(Owners own, int vw, const uint32_t *idx, int64_t n, uint4 *out) {
  const int words = 2 + 2 * vw;
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= n * words) return;
  const int64_t r = t / words;
  const int w = int(t - r * words);
  const uint32_t o = idx[r];
  uint4 val;
  if (w == 0) {
    const uint64_t vx = own.voxel[o];
    const ushort4 sb = own.sub[o];
    val = make_uint4(uint32_t(vx), uint32_t(vx >> 32), uint32_t(sb.x) | (uint32_t(sb.y) << 16), uint32_t(sb.z));
  } else if (w == 1) {
    const float4 q = own.quat[o];
    val = make_uint4(__float_as_uint(q.x), __float_as_uint(q.y), __float_as_uint(q.z), __float_as_uint(q.w));
  } else if (w < 2 + vw) {
    val = reinterpret_cast<const uint4 *>(own.lin_vel)[size_t(o) * vw + (w - 2)];
  } else {
    val = reinterpret_cast<const uint4 *>(own.ang_vel)[size_t(o) * vw + (w - 2 - vw)];
  }
  out[t] = val;
}

__global__ void k_unpack_state(Owners own, int vw, const uint32_t *idx, int64_t n, const uint4 *in) {
  const int words = 2 + 2 * vw;
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= n * words) return;
  const int64_t r = t / words;
  const int w = int(t - r * words);
  const uint32_t o = idx[r];
  const uint4 val = in[t];
  if (w == 0) {
    own.voxel[o] = uint64_t(val.x) | (uint64_t(val.y) << 32);
    own.sub[o] = make_ushort4(uint16_t(val.z & 0xFFFFu), uint16_t(val.z >> 16), uint16_t(val.w), 0);
  } else if (w == 1) {
    own.quat[o] = make_float4(__uint_as_float(val.x), __uint_as_float(val.y), __uint_as_float(val.z),
                              __uint_as_float(val.w));
  } else if (w < 2 + vw) {
    reinterpret_cast<uint4 *>(own.lin_vel)[size_t(o) * vw + (w - 2)] = val;
  } else {
    reinterpret_cast<uint4 *>(own.ang_vel)[size_t(o) * vw + (w - 2 - vw)] = val;
  }
}

// world centres of the spheres of the listed owners (after an unpack)
__global__ void k_owner_centers(Domain dom, Owners own, Spheres sph, const uint32_t *idx, int64_t n) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  const uint32_t o = idx[r];
  for (uint32_t k = sph.first[o]; k < sph.first[o + 1]; ++k) {
    double c[3];
    float rad;
    uint32_t ow;
    sphere_center(dom, own, sph, k, c, rad, ow);
    sph.center[k] = make_double4(c[0], c[1], c[2], double(rad));
    if (sph.kin) write_kin_from_state(own, sph, k, o);
  }
}

// ghost contributions out (and cleared: the ghost is not integrated here)
__global__ void k_pack_forces(long long *facc, const uint32_t *idx, int64_t n, longlong2 *out) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= 3 * n) return;
  const int64_t r = t / 3;
  const int w = int(t - 3 * r);
  longlong2 *src = reinterpret_cast<longlong2 *>(facc + 6 * size_t(idx[r])) + w;
  out[t] = *src;
  *src = make_longlong2(0, 0);
}

// returned contributions in: integer addition for fixed-point owners (exact,
// so the order ranks report in does not matter), fp64 for boundary owners
__global__ void k_add_forces(long long *facc, const uint32_t *meta, const double2 *tpl_scale,
                             const uint32_t *idx, int64_t n, const long long *in) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= 6 * n) return;
  const int64_t r = t / 6;
  const int w = int(t - 6 * r);
  const uint32_t o = idx[r];
  long long *dst = facc + 6 * size_t(o) + w;
  const long long add_v = in[t];
  if (tpl_scale[meta_tpl(meta[o])].x > 0.0) {
    *dst += add_v;
  } else {
    *dst = __double_as_longlong(__longlong_as_double(*dst) + __longlong_as_double(add_v));
  }
}

__global__ void k_axis_coords(Domain dom, Owners own, int axis, double *out) {
  const int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (o >= own.n) return;
  double p[3];
  decode_pos(dom, own.voxel[o], own.sub[o], p[0], p[1], p[2]);
  out[o] = p[axis];
}

// the decomposition guard's trip step to / from a transport word (int64,
// INT64_MAX = no trip), so every rank stops after the same step
__global__ void k_trip_word(Status *st, long long *w, int mode) {
  if (mode == 0) {
    const unsigned long long t = st->dd_trip;
    *w = t == ~0ull ? 0x7FFFFFFFFFFFFFFFll : (long long)t;
  } else {
    const long long v = *w;
    if (v != 0x7FFFFFFFFFFFFFFFll) atomicMin(&st->dd_trip, (unsigned long long)v);
  }
}

inline unsigned blocks(int64_t n, int b) { return unsigned((n + b - 1) / b); }

}  // namespace

int halo_record_bytes(const Ctx *c) { return 32 + 2 * (c->f32_state ? 16 : 32); }

int halo_axis_coords(Ctx *c, int axis, double *out, cudaStream_t s) {
  if (!c->n_owner) return 0;
  k_axis_coords<<<blocks(c->n_owner, 128), 128, 0, s>>>(c->dom, owners_view(c), axis, out);
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

int halo_trip_word(Ctx *c, void *word, int mode, cudaStream_t s) {
  k_trip_word<<<1, 1, 0, s>>>(c->status.as<Status>(), reinterpret_cast<long long *>(word), mode);
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

int halo_pack_state(Ctx *c, const uint32_t *idx, int64_t n, void *out, cudaStream_t s) {
  if (n <= 0) return 0;
  const int vw = c->f32_state ? 1 : 2;
  k_pack_state<<<blocks(n * (2 + 2 * vw), 256), 256, 0, s>>>(owners_view(c), vw, idx, n,
                                                              reinterpret_cast<uint4 *>(out));
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

int halo_unpack_state(Ctx *c, const uint32_t *idx, int64_t n, const void *in, cudaStream_t s) {
  if (n <= 0) return 0;
  const int vw = c->f32_state ? 1 : 2;
  const Owners own = owners_view(c);
  k_unpack_state<<<blocks(n * (2 + 2 * vw), 256), 256, 0, s>>>(own, vw, idx, n,
                                                                reinterpret_cast<const uint4 *>(in));
  if (c->n_sph) k_owner_centers<<<blocks(n, 128), 128, 0, s>>>(c->dom, own, spheres_view(c), idx, n);
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

int halo_pack_forces(Ctx *c, const uint32_t *idx, int64_t n, void *out, cudaStream_t s) {
  if (n <= 0) return 0;
  k_pack_forces<<<blocks(3 * n, 256), 256, 0, s>>>(c->facc.as<long long>(), idx, n,
                                                   reinterpret_cast<longlong2 *>(out));
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

int halo_add_forces(Ctx *c, const uint32_t *idx, int64_t n, const void *in, cudaStream_t s) {
  if (n <= 0) return 0;
  k_add_forces<<<blocks(6 * n, 256), 256, 0, s>>>(c->facc.as<long long>(), c->meta.as<uint32_t>(),
                                                  c->tpl_scale.as<double2>(), idx, n,
                                                  reinterpret_cast<const long long *>(in));
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------
// active boxes on the device (engine.py:857-879): every
// clump owner of the active or frozen family is re-tagged by whether its
// position lies inside any box (|p - c| <= half per axis, c = the anchor
// owner's position or a static centre); owners frozen now lose their
// velocities; the re-tagged owners' kinematics records pick up the new
// family's passive flag.  No host round trip of the owner state.
// ---------------------------------------------------------------------------
__global__ void k_active_boxes(Domain dom, Owners own, Spheres sph, int nbox, const double *box,
                               const long long *anchor, uint32_t active, uint32_t frozen, int vel_f32,
                               unsigned long long *n_changed) {
  const int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (o >= own.n) return;
  const uint32_t s0 = sph.first[o], s1 = sph.first[o + 1];
  if (s1 == s0) return;   // not a clump (meshes / analytic boundaries own no spheres)
  const uint32_t meta = own.meta[o], fam = meta_family(meta);
  if (fam != active && fam != frozen) return;
  double p[3];
  decode_pos(dom, own.voxel[o], own.sub[o], p[0], p[1], p[2]);
  bool inside = false;
  for (int b = 0; b < nbox && !inside; ++b) {
    double cx = box[6 * b], cy = box[6 * b + 1], cz = box[6 * b + 2];
    if (anchor[b] >= 0) {
      const uint32_t a = uint32_t(anchor[b]);
      decode_pos(dom, own.voxel[a], own.sub[a], cx, cy, cz);
    }
    inside = fabs(p[0] - cx) <= box[6 * b + 3] && fabs(p[1] - cy) <= box[6 * b + 4] &&
             fabs(p[2] - cz) <= box[6 * b + 5];
  }
  const uint32_t nf = inside ? active : frozen;
  if (nf == fam) return;
  own.meta[o] = (nf << 24) | meta_tpl(meta);
  if (nf == frozen) {
    if (vel_f32) {
      reinterpret_cast<float4 *>(own.lin_vel)[o] = make_float4(0.f, 0.f, 0.f, 0.f);
      reinterpret_cast<float4 *>(own.ang_vel)[o] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      double2 *lv = reinterpret_cast<double2 *>(own.lin_vel) + 2 * o, *av = reinterpret_cast<double2 *>(own.ang_vel) + 2 * o;
      lv[0] = make_double2(0.0, 0.0); lv[1] = make_double2(0.0, 0.0);
      av[0] = make_double2(0.0, 0.0); av[1] = make_double2(0.0, 0.0);
    }
  }
  if (sph.kin)
    for (uint32_t k = s0; k < s1; ++k) write_kin_from_state(own, sph, k, uint32_t(o));
  atomicAdd(n_changed, 1ull);
}

int active_boxes(Ctx *c, int n_box, const double *box, const long long *anchor, uint32_t active, uint32_t frozen,
                 unsigned long long *n_changed, cudaStream_t s) {
  if (!c->n_owner) return 0;
  k_active_boxes<<<blocks(c->n_owner, 256), 256, 0, s>>>(c->dom, owners_view(c), spheres_view(c), n_box, box, anchor,
                                                         active, frozen, c->f32_state ? 1 : 0, n_changed);
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

}  // namespace gf
