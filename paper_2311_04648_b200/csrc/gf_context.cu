#include <cstdio>
// gf_context.cu -- C-ABI (include/gf_b200.h): context, scene upload/download,
// per-kernel entry points and the kT/dT worker protocol (gf_run).
//
// Scheduler (replaces the reference's two threads + _Slot handoffs,
// engine.py:90-115, 669-906): kT and dT are two CUDA streams of one device.
// At a snapshot step the dT stream records the snapshot (sphere centres,
// families, world geometry); the kT stream waits on that event and runs
// detection into the second ACS buffer while the dT stream keeps stepping on
// the active ACS.  `lag` steps later the dT stream waits on the kT completion
// event, remaps the contact history onto the new array (merge_history) and
// swaps the double buffer.  Adoption happens at a fixed step, so runs are
// bitwise reproducible; period = 1, lag = 0 is the reference's sync mode.
#include <algorithm>
#include <cmath>
#include <chrono>
#include <deque>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/gf_b200.h"
#include "gf_context.h"

struct gf_ctx {
  gf::Ctx c;
};

namespace gf {

void set_err(Ctx *c, const std::string &msg) { c->err = msg; }

// Grow-only device buffer: exactly `bytes` (callers that grow repeatedly add
// their own slack); without `keep` the old block is freed first so a large
// buffer never needs twice its size.
int ensure(Ctx *c, DBuf &b, size_t bytes, cudaStream_t s, bool keep) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return 0;
  const size_t nb = bytes + 256;
  void *p = nullptr;
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess && !keep && b.p) {
    cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
  }
  if (e == cudaSuccess) e = cudaMalloc(&p, nb);
  if (e == cudaErrorMemoryAllocation) {
    // blocks parked in the stream-ordered pool (big kT scratch) hold device
    // memory: return them and retry once
    (void)cudaGetLastError();
    cudaMemPool_t pool;
    int cur = c->device;
    cudaGetDevice(&cur);
    if (cudaDeviceGetDefaultMemPool(&pool, cur) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess &&
        cudaMemPoolTrimTo(pool, 0) == cudaSuccess)
      e = cudaMalloc(&p, nb);
  }
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    set_err(c, std::string("device allocation of ") + std::to_string(nb) + " bytes failed: " +
                   cudaGetErrorString(e));
    return -1;
  }
  if (keep && b.p && b.bytes) {
    cudaMemcpyAsync(p, b.p, b.bytes, cudaMemcpyDeviceToDevice, s);
    cudaStreamSynchronize(s);
  }
  if (b.p) cudaFree(b.p);
  b.p = p;
  b.bytes = nb;
  return 0;
}

// GF_SYNC_DEBUG=1 (diagnostics only): synchronise the device after every
// phase of the step and name the phase a kernel fault surfaced in
bool sync_debug() {
  static const bool on = std::getenv("GF_SYNC_DEBUG") != nullptr;
  return on;
}
int dbg_sync(Ctx *c, const char *what, int64_t step) {
  if (!sync_debug()) return 0;
  const cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) return 0;
  set_err(c, std::string("GF_SYNC_DEBUG: ") + cudaGetErrorString(e) + " after " + what + " (step " +
                 std::to_string(step) + ")");
  return -1;
}

int ensure_scratch(Ctx *c, DBuf &b, size_t bytes, cudaStream_t s) {
  if (!big_scratch(c)) return ensure(c, b, bytes, s);
  return ensure_pooled(c, b, bytes, s);
}

int ensure_pooled(Ctx *c, DBuf &b, size_t bytes, cudaStream_t s) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return 0;
  if (b.p) GF_CHECK(c, cudaFreeAsync(b.p, s));
  b.p = nullptr;
  b.bytes = 0;
  const size_t nb = bytes + 256;
  cudaError_t e = cudaMallocAsync(&b.p, nb, s);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    b.p = nullptr;
    set_err(c, std::string("stream-ordered allocation of ") + std::to_string(nb) + " bytes failed: " +
                   cudaGetErrorString(e));
    return -1;
  }
  b.bytes = nb;
  return 0;
}

// The centre records (double4 per sphere) as a 2-D tensor [n_sph rows x 4
// doubles] for TMA tile::gather4 (box = one row); re-encoded when the buffer
// moves.  cuTensorMapEncodeTiled comes from the driver through the runtime's
// entry-point query (no link-time libcuda dependency).
int center_tmap(Ctx *c) {
  void *p = c->sph_center.p;
  if (!p || c->n_sph <= 0) return -1;
  if (p == c->tm_center_ptr && c->n_sph == c->tm_center_n) return 0;
  using Encode = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = nullptr;
  if (!encode) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      c->err = "cuTensorMapEncodeTiled unavailable";
      return -1;
    }
    encode = reinterpret_cast<Encode>(fn);
  }
  const cuuint64_t dims[2] = {4, cuuint64_t(c->n_sph)};
  const cuuint64_t strides[1] = {32};
  const cuuint32_t box[2] = {4, 1};
  const cuuint32_t es[2] = {1, 1};
  if (encode(&c->tm_center, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, p, dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    c->err = "cuTensorMapEncodeTiled failed for the centre records";
    return -1;
  }
  c->tm_center_ptr = p;
  c->tm_center_n = c->n_sph;
  return 0;
}

int release_scratch(Ctx *c, DBuf &b, cudaStream_t s) {
  if (b.p) GF_CHECK(c, cudaFreeAsync(b.p, s));
  b.p = nullptr;
  b.bytes = 0;
  return 0;
}

int h2d(Ctx *c, void *dst, const void *src, size_t bytes, cudaStream_t s) {
  if (!bytes) return 0;
  GF_CHECK(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  GF_CHECK(c, cudaStreamSynchronize(s));
  return 0;
}

static void release(DBuf &b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

Owners owners_view(Ctx *c) {
  Owners o;
  o.n = c->n_owner;
  o.voxel = c->voxel.as<uint64_t>();
  o.sub = c->sub.as<ushort4>();
  o.quat = c->quat.as<float4>();
  o.lin_vel = c->lin_vel.p;
  o.ang_vel = c->ang_vel.p;
  o.meta = c->meta.as<uint32_t>();
  o.tpl = c->tpl.as<double4>();
  o.acc = c->acc.as<double>();
  o.ext = c->has_ext ? c->ext.as<double>() : nullptr;
  o.facc = c->fixed_reduce ? c->facc.as<long long>() : nullptr;
  o.tpl_scale = c->tpl_scale.as<double2>();
  o.dd = c->dd_on ? c->dd.as<uint32_t>() : nullptr;
  o.dd_x0 = c->dd_x0.as<double>();
  o.dd_travel = c->dd_travel;
  o.dd_axis = c->dd_axis;
  o.passive = c->fam_passive.p ? c->fam_passive.as<uint8_t>() : nullptr;
  return o;
}
Spheres spheres_view(Ctx *c) {
  return Spheres{c->n_sph, c->sph_owner.as<uint32_t>(), c->sph_offr.as<float4>(), c->sph_mat.as<uint8_t>(),
                 c->sph_center.as<double4>(), c->sph_first.as<uint32_t>(),
                 c->f32_state ? c->sph_kin.as<SphKin>() : nullptr};
}
Tris tris_view(Ctx *c) {
  return Tris{c->n_tri, c->tri_owner.as<uint32_t>(), c->tri_local.as<float>(), c->tri_mat.as<uint8_t>(),
              c->tri_world.as<double>()};
}
Anas anas_view(Ctx *c) {
  return Anas{c->n_ana, c->ana_owner.as<uint32_t>(), c->ana_kind.as<uint8_t>(), c->ana_local.as<float>(),
              c->ana_mat.as<uint8_t>(), c->ana_world.as<double>()};
}
Materials materials_view(Ctx *c) {
  return Materials{c->n_mat, c->pair.as<double>(), c->beta.as<double>()};
}
Families families_view(Ctx *c) {
  return Families{c->fam_mask.as<uint8_t>(), c->fam_flags.as<uint8_t>(), c->lv_mask.as<uint8_t>(),
                  c->av_mask.as<uint8_t>(), c->lv_val.as<double>(), c->av_val.as<double>()};
}

cudaEvent_t *prof_current(Ctx *c) {
  if (!c->prof || c->prof_used < kProfEv) return nullptr;
  return &c->prof_ev[c->prof_used - kProfEv];
}

cudaEvent_t *prof_events(Ctx *c) {
  if (!c->prof) return nullptr;
  if (c->prof_used + kProfEv > c->prof_ev.size()) {
    for (int q = 0; q < kProfEv; ++q) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->prof_ev.push_back(e);
    }
  }
  cudaEvent_t *ev = &c->prof_ev[c->prof_used];
  c->prof_used += kProfEv;
  return ev;
}

static void prof_collect(Ctx *c) {
  for (size_t i = 0; i + kProfEv <= c->prof_used; i += kProfEv) {
    float m;
    for (int q = 0; q < 3; ++q)
      if (cudaEventElapsedTime(&m, c->prof_ev[i + q], c->prof_ev[i + q + 1]) == cudaSuccess)
        c->prof_ms[q] += m;
    if (cudaEventElapsedTime(&m, c->prof_ev[i], c->prof_ev[i + 4]) == cudaSuccess) c->prof_ms[4] += m;
    c->prof_steps++;
  }
  c->prof_used = 0;
}

// Fixed-point scales of the throughput build's owner accumulators.  A contact
// force on owner o is bounded by F_o = 64 m_o max(v_err / h, |g|) (a larger
// force trips the watchdog within a step).  The scale leaves 13 bits of
// headroom for sums: resolution ~ 2^-50 F_o.  Boundary owners (mass >= 1e13,
// BOUNDARY_MASS in types.py:42) are fixed or prescribed, so their sums never
// feed the dynamics; they accumulate with fp64 atomics (scale 0 marks them).
static int update_fixed_scales(Ctx *c, double h, double v_err, const double *g) {
  if (!c->fixed_reduce || (c->fx_h == h && c->fx_verr == v_err)) return 0;
  double rate = v_err / h;
  double gn = std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
  if (gn > rate) rate = gn;
  double m_clump_max = 0.0;
  for (double m : c->h_tpl_mass)
    if (m < 1e13 && m > m_clump_max) m_clump_max = m;
  if (m_clump_max <= 0.0) m_clump_max = 1.0;
  const double lever = c->lever_override > 0.0 ? c->lever_override : (c->lever_max > 0.0 ? c->lever_max : 1.0);
  std::vector<double> sc(2 * (c->h_tpl_mass.size() + 1), 1.0);
  for (size_t t = 0; t < c->h_tpl_mass.size(); ++t) {
    double m = c->h_tpl_mass[t];
    if (m >= 1e13) {  // boundary owner: fp64 atomics (its sums never feed the dynamics)
      sc[2 * t] = 0.0;
      sc[2 * t + 1] = 0.0;
      continue;
    }
    // powers of two: float-exact (the contact kernel reads them from the fp32
    // kinematics record) and exactly invertible (the integrator multiplies by
    // the reciprocal)
    // (exponents within [-127, 127]: the kinematics records store them in 8 bits)
    auto pow2 = [](double x) { return std::ldexp(1.0, std::min(127, std::max(-127, int(std::floor(std::log2(x)))))); };
    const double sf = pow2(std::ldexp(1.0, 50) / (64.0 * m * rate));
    sc[2 * t] = sf;
    sc[2 * t + 1] = pow2(sf / lever);
  }
  if (!c->h_tpl_mass.empty())
    if (h2d(c, c->tpl_scale.p, sc.data(), 16 * c->h_tpl_mass.size(), c->s_dt)) return -1;
  c->fx_h = h;
  c->fx_verr = v_err;
  // the kinematics records carry the scales
  if (c->f32_state && c->n_sph && c->sph_first.p && refresh_centers(c, c->s_dt)) return -1;
  return 0;
}

static int dt_step(Ctx *c, const StepArgs &a) {
  if (update_fixed_scales(c, a.h, a.v_err, a.g)) return -1;
  return c->f32_state ? dt_step_f32(c, a, c->s_dt) : dt_step_f64(c, a, c->s_dt);
}

// state of one gf_run call (gf_run_begin .. gf_run_end)
struct RunState {
  gf_run_params p{};
  int period = 1, lag = 0;
  int64_t sum_acs = 0;
  // per-detection kT timing: (start, end) event pairs of the detections in
  // flight; a pair whose end has completed is folded into kt_ms and recycled,
  // so a long run holds a handful of events, not one pair per detection
  std::deque<std::pair<cudaEvent_t, cudaEvent_t>> kt_ev;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kt_ev_free;
  double kt_ms = 0.0;
  bool kt_freeze = false;   // GF_KT_FREEZE, read once per run
  std::chrono::steady_clock::time_point w0;
  // GF_TRACE (diagnostics): timed events on both streams + host waits,
  // printed to stderr at gf_run_end
  bool trace = false;
  struct Mark { const char *what; int64_t step; cudaEvent_t ev; };
  std::vector<Mark> marks;
  double host_wait_ms[2] = {0.0, 0.0};   // run_count, run_fill synchronisations
};

static void trace_mark(Ctx *c, const char *what, int64_t step, cudaStream_t s) {
  RunState *R = c->run;
  if (!R || !R->trace) return;
  DevGuard g(stream_device(s));
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  R->marks.push_back({what, step, e});
}

static void free_run(Ctx *c) {
  if (!c->run) return;
  for (auto &e : c->run->kt_ev) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (auto &e : c->run->kt_ev_free) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  delete c->run;
  c->run = nullptr;
}

static int fail_run(Ctx *c) {
  free_run(c);
  return -1;
}

static StepArgs step_args(const RunState *R, int64_t i) {
  const gf_run_params *p = &R->p;
  const int64_t s = p->step0 + i;
  return StepArgs{p->h, {p->g[0], p->g[1], p->g[2]}, p->v_err, double(s) * p->h, s, i,
                  (i == p->n_steps - 1) ? p->write_acc : 0};
}

// kT phases: begun (grid + displacement check queued) -> counted (candidate
// filter + counts queued) -> filled (canonical array queued)
static int run_count(Ctx *c) {
  const auto h0 = std::chrono::steady_clock::now();
  GF_CHECK(c, cudaEventSynchronize(c->ev_disp));
  if (c->run) c->run->host_wait_ms[0] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
  const int rc = kt_count_async(c, c->s_kt);
  if (rc < 0) return -1;
  GF_CHECK(c, cudaEventRecord(c->ev_count, c->s_kt));
  if (rc == 1) {   // a staged candidate rebuild: resumed by advance_kt
    c->kt_phase = 3;
    return 0;
  }
  trace_mark(c, "kt_count_end", c->last_snap, c->s_kt);
  c->kt_phase = 2;
  return 0;
}

// resume a staged rebuild (phase 3) as far as its device counts allow;
// block = wait for each (the fill needs the result now)
static int advance_kt(Ctx *c, bool block) {
  const auto h0 = std::chrono::steady_clock::now();
  const int rc = kt_advance(c, c->s_kt, c->ev_count, block);
  if (block && c->run)
    c->run->host_wait_ms[0] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
  if (rc < 0) return -1;
  if (rc == 0) {
    GF_CHECK(c, cudaEventRecord(c->ev_count, c->s_kt));
    trace_mark(c, "kt_count_end", c->last_snap, c->s_kt);
    c->kt_phase = 2;
  }
  return 0;
}

static int run_fill(Ctx *c) {
  if (c->kt_phase == 1 && run_count(c)) return -1;
  if (c->kt_phase == 3 && advance_kt(c, true)) return -1;
  const auto h0 = std::chrono::steady_clock::now();
  GF_CHECK(c, cudaEventSynchronize(c->ev_count));
  if (c->run) c->run->host_wait_ms[1] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
  c->acs_next.n = int64_t(reinterpret_cast<Status *>(c->h_status)->acs_total);
  if (kt_detect_fill(c, c->acs_next, c->s_kt)) return -1;
  if (c->run && !c->run->kt_ev.empty()) GF_CHECK(c, cudaEventRecord(c->run->kt_ev.back().second, c->s_kt));
  GF_CHECK(c, cudaEventRecord(c->ev_ca, c->s_kt));
  trace_mark(c, "kt_fill_end", c->last_snap, c->s_kt);
  c->fill_done = true;
  return 0;
}

static int run_adopt(Ctx *c) {
  if (!c->fill_done && run_fill(c)) return -1;
  GF_CHECK(c, cudaStreamWaitEvent(c->s_dt, c->ev_ca, 0));
  if (adopt_acs(c, c->s_dt)) return -1;
  GF_CHECK(c, cudaEventRecord(c->ev_adopted, c->s_dt));
  c->next_pending = false;
  c->first_adopt = false;
  return 0;
}

static int reset_status(Ctx *c, cudaStream_t s) {
  Status *st = c->status.as<Status>();
  GF_CHECK(c, cudaMemsetAsync(st, 0xFF, 2 * sizeof(unsigned long long), s));
  GF_CHECK(c, cudaMemsetAsync(&st->touching, 0, sizeof(unsigned long long), s));
  GF_CHECK(c, cudaMemsetAsync(&st->touch_pairs, 0, sizeof(unsigned long long), s));
  GF_CHECK(c, cudaMemsetAsync(&st->err, 0, sizeof(int), s));
  GF_CHECK(c, cudaMemsetAsync(&st->dd_trip, 0xFF, sizeof(unsigned long long), s));
  return 0;
}

static int read_status(Ctx *c, cudaStream_t s, Status *out) {
  GF_CHECK(c, cudaMemcpyAsync(c->h_status, c->status.p, sizeof(Status), cudaMemcpyDeviceToHost, s));
  GF_CHECK(c, cudaStreamSynchronize(s));
  std::memcpy(out, c->h_status, sizeof(Status));
  return 0;
}

static void decode_err(unsigned long long w, int64_t &owner, int64_t &step) {
  if (w == ~0ull) { owner = -1; step = -1; return; }
  owner = int64_t(w & ((1ull << 40) - 1));
  step = int64_t(w >> 40);
}

// enumeration split (csrc/gf_kt.cu): r_cut = the largest radius not above
// twice the median; spheres above it are "big" and paired by k_big
static int set_split(Ctx *c, const float *radii, int64_t stride, int64_t n) {
  std::vector<float> r(n);
  for (int64_t i = 0; i < n; ++i) r[i] = radii[i * stride];
  c->n_big = 0;
  c->r_cut = 0.0;
  if (!n) return 0;
  std::vector<float> sorted(r);
  std::nth_element(sorted.begin(), sorted.begin() + n / 2, sorted.end());
  const double med = sorted[n / 2];
  double rc = 0.0;
  for (float x : r)
    if (double(x) <= 2.0 * med && double(x) > rc) rc = double(x);
  // the big-sphere path (k_big / k_cand_big: atomic appends, long segments)
  // is for a few large bodies such as the crater projectile; a size
  // distribution with a heavy tail (GRC-1 terrain: 5 % of spheres above twice
  // the median) instead raises r_cut so that at most 0.1 % stay big
  const int64_t limit = std::max<int64_t>(64, n / 1000);
  int64_t n_above = 0;
  for (float x : r) n_above += double(x) > rc ? 1 : 0;
  if (n_above > limit) {
    std::vector<float> s2(r);
    std::nth_element(s2.begin(), s2.begin() + (n - limit - 1), s2.end());
    rc = std::max(rc, double(s2[n - limit - 1]));
  }
  std::vector<uint32_t> big;
  for (int64_t i = 0; i < n; ++i)
    if (double(r[i]) > rc) big.push_back(uint32_t(i));
  c->r_cut = rc;
  c->n_big = int64_t(big.size());
  if (ensure(c, c->big_slots, 4 * (big.size() + 1), c->s_dt)) return -1;
  if (!big.empty()) if (h2d(c, c->big_slots.p, big.data(), 4 * big.size(), c->s_dt)) return -1;
  return 0;
}

static void world_moving_update(Ctx *c) {
  // _refresh_moving_world (engine.py:552-568): skip while every mesh /
  // analytic owner sits in a fixed family
  c->world_moving = false;
  std::vector<uint32_t> own;
  auto scan = [&](const DBuf &b, int64_t n) {
    if (!n) return;
    std::vector<uint32_t> h(n);
    cudaMemcpy(h.data(), b.p, 4 * n, cudaMemcpyDeviceToHost);
    own.insert(own.end(), h.begin(), h.end());
  };
  scan(c->tri_owner, c->n_tri);
  scan(c->ana_owner, c->n_ana);
  if (own.empty() || !c->n_owner) return;
  std::vector<uint32_t> meta(c->n_owner);
  cudaMemcpy(meta.data(), c->meta.p, 4 * c->n_owner, cudaMemcpyDeviceToHost);
  for (uint32_t o : own) {
    uint32_t fam = meta_family(meta[o]);
    if (!(c->h_fam_flags.size() == 256 && (c->h_fam_flags[fam] & kFamFixed))) {
      c->world_moving = true;
      return;
    }
  }
}

}  // namespace gf

using namespace gf;

#define CTX_CHECK(ctx)                 \
  if (!(ctx)) return -1;               \
  gf::Ctx *c = &(ctx)->c;              \
  if (cudaSetDevice(c->device) != cudaSuccess) { c->err = "cudaSetDevice failed"; return -1; }

extern "C" {

int gf_nvrtc_compile(const char *cuda_src, const char *include_dir, char *log, size_t log_n) {
  std::string lg;
  int rc = nvrtc_compile_check(cuda_src, include_dir, lg);
  if (log && log_n) {
    std::strncpy(log, lg.c_str(), log_n - 1);
    log[log_n - 1] = 0;
  }
  return rc;
}

int gf_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

gf_ctx *gf_create(int device, int kt_device, uint32_t flags) {
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  gf_ctx *ctx = new gf_ctx();
  Ctx *c = &ctx->c;
  c->device = device;
  c->split = kt_device >= 0;
  c->kt_device = c->split ? kt_device : device;
  c->flags = flags;
  c->f32_state = (flags & GF_STATE_F32) != 0;
  c->fixed_reduce = c->f32_state;
  if (c->split && kt_device != device) {
    // kT kernels write the dT device's contact arrays and read its tables;
    // the dT device's snapshot kernel writes the kT device's snapshot
    int ab = 0, ba = 0;
    cudaDeviceCanAccessPeer(&ab, device, kt_device);
    cudaDeviceCanAccessPeer(&ba, kt_device, device);
    if (!ab || !ba) {
      delete ctx;
      return nullptr;
    }
    cudaError_t e = cudaDeviceEnablePeerAccess(kt_device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) { delete ctx; return nullptr; }
    cudaSetDevice(kt_device);
    e = cudaDeviceEnablePeerAccess(device, 0);
    cudaSetDevice(device);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) { delete ctx; return nullptr; }
    (void)cudaGetLastError();
  }
  // stream priorities (GF_STREAM_PRIO): 0 equal, 1 dT first, 2 kT first
  int prio_lo = 0, prio_hi = 0, mode = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (const char *sp = std::getenv("GF_STREAM_PRIO")) mode = std::atoi(sp);
  cudaStreamCreateWithPriority(&c->s_dt, cudaStreamNonBlocking, mode == 1 ? prio_hi : prio_lo);
  cudaEventCreateWithFlags(&c->ev_snap, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_adopted, cudaEventDisableTiming);
  {
    // the kT stream and the events recorded on it belong to the kT device
    DevGuard g(c->kt_device);
    cudaStreamCreateWithPriority(&c->s_kt, cudaStreamNonBlocking, mode == 2 ? prio_hi : prio_lo);
    cudaEventCreateWithFlags(&c->ev_ca, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_count, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_disp, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_kt_join, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_snap_done, cudaEventDisableTiming);
    if (c->kt_device != device) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, c->kt_device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      (void)cudaGetLastError();
    }
  }
  if (const char *sf = std::getenv("GF_SKIN_FACTOR")) c->skin_factor = std::atof(sf);
  if (const char *sb = std::getenv("GF_SKIN_BIG")) c->skin_big_factor = std::atof(sb);
  if (c->skin_big_factor < c->skin_factor) c->skin_big_factor = c->skin_factor;
  if (const char *sp = std::getenv("GF_SS_SPLIT")) c->ss_split = std::atoi(sp);
  if (const char *sr = std::getenv("GF_SS_RED")) c->ss_red = std::atoi(sr);
  if (const char *sp = std::getenv("GF_SS_PF")) c->ss_pf = std::atoi(sp);
  if (const char *sb = std::getenv("GF_SS_BLOCKED")) c->ss_blocked = std::atoi(sb);
  if (const char *sa = std::getenv("GF_SNAP_ASYNC")) c->snap_async = std::atoi(sa) != 0;
  if (const char *ra = std::getenv("GF_RB_ASYNC")) c->rb_async = std::atoi(ra) != 0;
  if (const char *rs = std::getenv("GF_RB_SLOT")) c->rb_slot = std::atoi(rs) != 0;
  if (const char *st = std::getenv("GF_SS_TMA")) c->ss_tma = std::atoi(st) != 0;
  cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, device);
  if (c->n_sm <= 0) c->n_sm = 148;
  if (const char *pd = std::getenv("GF_PDL")) c->pdl = std::atoi(pd);
  cudaEventCreate(&c->t0);
  cudaEventCreate(&c->t1);
  cudaEventRecord(c->ev_adopted, c->s_dt);
  // the rebuild-only kT scratch of big scenes cycles through the device's
  // stream-ordered pool (ensure_scratch): keep freed blocks mapped in the
  // pool so the next rebuild reuses them instead of remapping tens of GB;
  // ensure() trims the pool if a plain allocation ever runs short
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    (void)cudaGetLastError();
  }
  // pinned status mirror, written by both streams' devices
  if (cudaHostAlloc(&c->h_status, sizeof(Status), cudaHostAllocPortable) != cudaSuccess) { delete ctx; return nullptr; }
  if (ensure(c, c->status, sizeof(Status), c->s_dt) || ensure(c, c->heavy_count, 16, c->s_dt)) {
    delete ctx;
    return nullptr;
  }
  cudaMemsetAsync(c->status.p, 0, sizeof(Status), c->s_dt);   // pad words read by read_status (initcheck)
  reset_status(c, c->s_dt);
  cudaStreamSynchronize(c->s_dt);
  return ctx;
}

void gf_destroy(gf_ctx *ctx) {
  if (!ctx) return;
  Ctx *c = &ctx->c;
  if (c->split) {
    cudaSetDevice(c->kt_device);
    cudaDeviceSynchronize();
  }
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  DBuf *bufs[] = {&c->sph_kin, &c->tlist, &c->tlist_n, &c->facc, &c->tpl_scale, &c->sph_center, &c->sph_first, &c->voxel, &c->sub, &c->quat, &c->lin_vel, &c->ang_vel, &c->meta, &c->tpl, &c->acc,
                  &c->ext, &c->sph_owner, &c->sph_offr, &c->sph_mat, &c->tri_owner, &c->tri_local,
                  &c->tri_mat, &c->tri_world, &c->ana_owner, &c->ana_kind, &c->ana_local, &c->ana_mat,
                  &c->ana_world, &c->pair, &c->beta, &c->fam_mask, &c->fam_flags, &c->lv_mask,
                  &c->av_mask, &c->lv_val, &c->av_val, &c->fam_passive, &c->acs.ids, &c->acs.wild, &c->acs_next.ids,
                  &c->acs_next.wild, &c->out_c, &c->touch, &c->inc, &c->inc_alt, &c->inc_key,
                  &c->inc_key_alt, &c->inc_start, &c->heavy, &c->heavy_count, &c->heavy_acc,
                  &c->cub_tmp_dt, &c->status, &c->dyn_spec, &c->dyn_vals, &c->kt.c4, &c->kt.sfam,
                  &c->kt.tri_world, &c->kt.ana_world, &c->kt.tfam, &c->kt.afam, &c->kt.grid,
                  &c->kt.minmax, &c->kt.bin_key, &c->kt.bin_key_alt, &c->kt.sph_val, &c->kt.sph_val_alt,
                  &c->kt.cell_start, &c->kt.cell_end, &c->kt.tri_ranges, &c->kt.tri_cnt,
                  &c->kt.tri_start, &c->kt.tri_entries, &c->kt.counts, &c->kt.offsets, &c->kt.cub_tmp,
                  &c->kt.total, &c->kt.cursor, &c->kt.tri_cursor, &c->big_slots, &c->kt.sc,
                  &c->kt.sm, &c->kt.sf, &c->kt.cells, &c->kt.n_cells, &c->kt.cand, &c->kt.cand_tmp, &c->kt.cand_n,
                  &c->kt.cand_cnt, &c->kt.cand_own, &c->kt.cand_seg, &c->kt.ref, &c->kt.flag, &c->kt.cflags, &c->kt.sel_n, &c->kt.tmp, &c->kt.tmp_n, &c->acs.seg, &c->acs_next.seg, &c->acs.old_pos, &c->acs_next.old_pos, &c->kt.fbits[0], &c->kt.fbits[1], &c->kt.fpre[0], &c->kt.fpre[1], &c->kt.fcnt, &c->dd, &c->dd_x0, &c->halo_scratch, &c->owner_stage, &c->kt.sa_cnt, &c->kt.sa_off, &c->kt.sa_cand, &c->kt.gaps};
  for (DBuf *b : bufs) release(*b);
  free_run(c);
  if (c->h_status) cudaFreeHost(c->h_status);
  cudaEvent_t evs[] = {c->ev_snap, c->ev_ca, c->ev_adopted, c->ev_count, c->ev_disp, c->ev_kt_join, c->ev_snap_done,
                       c->t0, c->t1};
  for (auto e : evs) cudaEventDestroy(e);
  cudaStreamDestroy(c->s_dt);
  cudaStreamDestroy(c->s_kt);
  delete ctx;
}

int gf_last_error(gf_ctx *ctx, char *buf, size_t n) {
  if (!ctx || !buf || !n) return -1;
  std::strncpy(buf, ctx->c.err.c_str(), n - 1);
  buf[n - 1] = 0;
  return 0;
}

int gf_set_domain(gf_ctx *ctx, const double *lo3, const double *hi3, double edge) {
  CTX_CHECK(ctx);
  for (int a = 0; a < 3; ++a) { c->dom.lo[a] = lo3[a]; c->dom.hi[a] = hi3[a]; }
  c->dom.edge = edge;
  return 0;
}

// Owner state in the reference's host layouts (StateStore arrays, core.py:356-390)
// <-> the device layouts.  The host arrays are copied as they are into a
// device staging buffer (stream-ordered; full PCIe rate from pinned memory)
// and converted on the device, so a per-step host round trip costs the
// transfers, not host-side repacking.
namespace {
__global__ void k_owners_in(int64_t n, const uint16_t *sub3, const double *lv3, const double *av3,
                            const uint8_t *family, const uint32_t *tpl, ushort4 *sub, void *lin_vel,
                            void *ang_vel, uint32_t *meta, int f32) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  sub[i] = make_ushort4(sub3[3 * i], sub3[3 * i + 1], sub3[3 * i + 2], 0);
  meta[i] = (uint32_t(family[i]) << 24) | (tpl[i] & 0xFFFFFFu);
  if (f32) {
    reinterpret_cast<float4 *>(lin_vel)[i] = make_float4(float(lv3[3 * i]), float(lv3[3 * i + 1]), float(lv3[3 * i + 2]), 0.f);
    reinterpret_cast<float4 *>(ang_vel)[i] = make_float4(float(av3[3 * i]), float(av3[3 * i + 1]), float(av3[3 * i + 2]), 0.f);
  } else {
    double2 *l = reinterpret_cast<double2 *>(lin_vel) + 2 * i, *w = reinterpret_cast<double2 *>(ang_vel) + 2 * i;
    l[0] = make_double2(lv3[3 * i], lv3[3 * i + 1]);
    l[1] = make_double2(lv3[3 * i + 2], 0.0);
    w[0] = make_double2(av3[3 * i], av3[3 * i + 1]);
    w[1] = make_double2(av3[3 * i + 2], 0.0);
  }
}

__global__ void k_owners_out(int64_t n, const ushort4 *sub, const void *lin_vel, const void *ang_vel,
                             const uint32_t *meta, uint16_t *sub3, double *lv3, double *av3, uint8_t *family,
                             int f32) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const ushort4 s = sub[i];
  sub3[3 * i] = s.x; sub3[3 * i + 1] = s.y; sub3[3 * i + 2] = s.z;
  family[i] = uint8_t(meta_family(meta[i]));
  if (f32) {
    const float4 l = reinterpret_cast<const float4 *>(lin_vel)[i], w = reinterpret_cast<const float4 *>(ang_vel)[i];
    lv3[3 * i] = l.x; lv3[3 * i + 1] = l.y; lv3[3 * i + 2] = l.z;
    av3[3 * i] = w.x; av3[3 * i + 1] = w.y; av3[3 * i + 2] = w.z;
  } else {
    const double2 *l = reinterpret_cast<const double2 *>(lin_vel) + 2 * i,
                  *w = reinterpret_cast<const double2 *>(ang_vel) + 2 * i;
    const double2 l0 = l[0], l1 = l[1], w0 = w[0], w1 = w[1];
    lv3[3 * i] = l0.x; lv3[3 * i + 1] = l0.y; lv3[3 * i + 2] = l1.x;
    av3[3 * i] = w0.x; av3[3 * i + 1] = w0.y; av3[3 * i + 2] = w1.x;
  }
}

// staging layout for n owners: sub3 u16[3n] | lv f64[3n] | av f64[3n] | tpl u32[n] | family u8[n]
struct Stage {
  uint16_t *sub3;
  double *lv, *av;
  uint32_t *tpl;
  uint8_t *fam;
};
Stage stage_of(DBuf &b, int64_t n) {
  char *p = static_cast<char *>(b.p);
  Stage st;
  st.lv = reinterpret_cast<double *>(p);
  st.av = st.lv + 3 * n;
  st.tpl = reinterpret_cast<uint32_t *>(st.av + 3 * n);
  st.sub3 = reinterpret_cast<uint16_t *>(st.tpl + n);
  st.fam = reinterpret_cast<uint8_t *>(st.sub3 + 3 * n);
  return st;
}
constexpr size_t kStageBytesPerOwner = 24 + 24 + 4 + 6 + 1;
}  // namespace

// world_moving from the host family array and the cached mesh / analytic
// owners (no device read-back)
static void world_moving_from_host(Ctx *c, const uint8_t *family) {
  c->world_moving = false;
  for (const auto *v : {&c->h_tri_owner, &c->h_ana_owner})
    for (uint32_t o : *v)
      if (!(c->h_fam_flags.size() == 256 && (c->h_fam_flags[family[o]] & kFamFixed))) {
        c->world_moving = true;
        return;
      }
}

// host-layout staging of the owner round trips: kept below 2^24 owners,
// from the stream-ordered pool above (see gf_upload_owners)
static int ensure_stage(Ctx *c, int64_t n, cudaStream_t s) {
  const size_t bytes = kStageBytesPerOwner * (n + 1);
  return n >= (int64_t(1) << 24) ? ensure_pooled(c, c->owner_stage, bytes, s) : ensure(c, c->owner_stage, bytes, s);
}

int gf_upload_owners(gf_ctx *ctx, int64_t n, const uint64_t *voxel, const uint16_t *sub,
                     const float *quat, const double *lin_vel, const double *ang_vel,
                     const uint8_t *family, const uint32_t *tpl, int64_t n_tpl,
                     const double *tpl_mass, const double *tpl_moi) {
  CTX_CHECK(ctx);
  if (n_tpl >= (1 << 24)) { c->err = "too many mass-property templates (max 2^24)"; return -1; }
  const bool resized = n != c->n_owner;
  c->n_owner = n;
  c->n_tpl = n_tpl;
  cudaStream_t s = c->s_dt;
  const size_t vb = c->f32_state ? sizeof(float) * 4 : sizeof(double) * 4;
  if (ensure(c, c->voxel, 8 * n, s) || ensure(c, c->sub, 8 * n, s) ||
      ensure(c, c->quat, 16 * n, s) || ensure(c, c->lin_vel, vb * n, s) ||
      ensure(c, c->ang_vel, vb * n, s) || ensure(c, c->meta, 4 * n, s) ||
      ensure(c, c->tpl, 32 * (n_tpl + 1), s) || ensure(c, c->acc, 48 * n, s) ||
      ensure(c, c->facc, 48 * n, s) || ensure(c, c->tpl_scale, 16 * (n_tpl + 1), s))
    return -1;
  // fixed-point scales are set at the first run (update_fixed_scales); until
  // then the kinematics records carry zeros, not uninitialised words
  // (compute-sanitizer initcheck)
  if (c->fx_h < 0.0) GF_CHECK(c, cudaMemsetAsync(c->tpl_scale.p, 0, 16 * (n_tpl + 1), s));
  if (ensure_stage(c, n, s)) return -1;
  // the parity build's incidence-list reduction (the throughput build sums
  // into the fixed-point accumulators instead)
  if (!c->f32_state && (ensure(c, c->heavy_acc, 48 * n, s) || ensure(c, c->inc_start, 4 * (n + 2), s) ||
                        ensure(c, c->heavy, 4 * (n + 1), s)))
    return -1;
  const Stage st = stage_of(c->owner_stage, n);
  if (n) {
    GF_CHECK(c, cudaMemcpyAsync(c->voxel.p, voxel, 8 * n, cudaMemcpyHostToDevice, s));
    GF_CHECK(c, cudaMemcpyAsync(c->quat.p, quat, 16 * n, cudaMemcpyHostToDevice, s));
    GF_CHECK(c, cudaMemcpyAsync(st.sub3, sub, 6 * n, cudaMemcpyHostToDevice, s));
    GF_CHECK(c, cudaMemcpyAsync(st.lv, lin_vel, 24 * n, cudaMemcpyHostToDevice, s));
    GF_CHECK(c, cudaMemcpyAsync(st.av, ang_vel, 24 * n, cudaMemcpyHostToDevice, s));
    GF_CHECK(c, cudaMemcpyAsync(st.fam, family, n, cudaMemcpyHostToDevice, s));
    GF_CHECK(c, cudaMemcpyAsync(st.tpl, tpl, 4 * n, cudaMemcpyHostToDevice, s));
    k_owners_in<<<unsigned((n + 255) / 256), 256, 0, s>>>(n, st.sub3, st.lv, st.av, st.fam, st.tpl,
                                                        c->sub.as<ushort4>(), c->lin_vel.p, c->ang_vel.p,
                                                        c->meta.as<uint32_t>(), c->f32_state ? 1 : 0);
  }
  // mass-property templates: the fixed-point scales (and the kinematics
  // records carrying them) are recomputed only when the masses change
  const bool tpl_changed = resized || c->h_tpl_mass.size() != size_t(n_tpl) ||
                           !std::equal(tpl_mass, tpl_mass + n_tpl, c->h_tpl_mass.begin()) ||
                           c->h_tpl_moi.size() != size_t(3 * n_tpl) ||
                           !std::equal(tpl_moi, tpl_moi + 3 * n_tpl, c->h_tpl_moi.begin());
  if (tpl_changed) {
    std::vector<double> tp(4 * n_tpl);
    for (int64_t t = 0; t < n_tpl; ++t) {
      tp[4 * t] = tpl_mass[t];
      tp[4 * t + 1] = tpl_moi[3 * t];
      tp[4 * t + 2] = tpl_moi[3 * t + 1];
      tp[4 * t + 3] = tpl_moi[3 * t + 2];
    }
    if (n_tpl) GF_CHECK(c, cudaMemcpyAsync(c->tpl.p, tp.data(), 32 * n_tpl, cudaMemcpyHostToDevice, s));
    GF_CHECK(c, cudaStreamSynchronize(s));   // tp is a host temporary
    c->h_tpl_mass.assign(tpl_mass, tpl_mass + n_tpl);
    c->h_tpl_moi.assign(tpl_moi, tpl_moi + 3 * n_tpl);
    c->fx_h = -1.0;  // fixed-point scales recomputed at the next run
  }
  GF_CHECK(c, cudaMemsetAsync(c->acc.p, 0, 48 * n, s));
  GF_CHECK(c, cudaMemsetAsync(c->facc.p, 0, 48 * n, s));
  if (c->has_ext) GF_CHECK(c, cudaMemsetAsync(c->ext.p, 0, 48 * n, s));
  if (c->n_sph && c->sph_first.p && c->sph_center.bytes >= size_t(32 * c->n_sph)) {
    if (refresh_centers(c, s) || refresh_world(c, s)) return -1;
  }
  // the staging buffer is kept for repeated host round trips, except at
  // scene sizes where device memory is the limit (2^24 owners and up): there
  // it goes back to the stream-ordered pool
  if (n >= (int64_t(1) << 24) && release_scratch(c, c->owner_stage, s)) return -1;
  GF_CHECK(c, cudaStreamSynchronize(s));
  world_moving_from_host(c, family);
  return 0;
}

// selected owners' state (trackers: no full-state download);
// row r of the 23-double output = voxel (bits), sub xyz, quat wxyz, v, w,
// family, acc force, acc torque
__global__ void k_read_owners(int64_t n, const long long *idx, const uint64_t *voxel, const ushort4 *sub,
                              const float4 *quat, const void *lin_vel, const void *ang_vel, const uint32_t *meta,
                              const double *acc, int f32, double *out) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  const int64_t o = idx[r];
  double *w = out + 23 * r;
  w[0] = __longlong_as_double((long long)voxel[o]);
  const ushort4 sb = sub[o];
  w[1] = sb.x; w[2] = sb.y; w[3] = sb.z;
  const float4 q = quat[o];
  w[4] = q.x; w[5] = q.y; w[6] = q.z; w[7] = q.w;
  for (int a = 0; a < 3; ++a) {
    w[8 + a] = f32 ? double(reinterpret_cast<const float *>(lin_vel)[4 * o + a])
                   : reinterpret_cast<const double *>(lin_vel)[4 * o + a];
    w[11 + a] = f32 ? double(reinterpret_cast<const float *>(ang_vel)[4 * o + a])
                    : reinterpret_cast<const double *>(ang_vel)[4 * o + a];
  }
  w[14] = double(meta_family(meta[o]));
  for (int a = 0; a < 6; ++a) w[15 + a] = acc ? acc[6 * o + a] : 0.0;
  w[21] = 0.0; w[22] = 0.0;
}

// max |v| over the clump owners (owners with spheres) of non-fixed families
// (Inspector "clump_max_absv", engine.py:198-214)
__global__ void k_clump_max_absv(int64_t n, const uint32_t *first, const uint32_t *meta, const uint8_t *fam_flags,
                                 const void *lin_vel, int f32, unsigned long long *out) {
  double best = 0.0;
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < n; o += int64_t(gridDim.x) * blockDim.x) {
    if (first[o + 1] == first[o] || (fam_flags[meta_family(meta[o])] & kFamFixed)) continue;
    double v2 = 0.0;
    for (int a = 0; a < 3; ++a) {
      const double x = f32 ? double(reinterpret_cast<const float *>(lin_vel)[4 * o + a])
                           : reinterpret_cast<const double *>(lin_vel)[4 * o + a];
      v2 += x * x;
    }
    best = fmax(best, sqrt(v2));
  }
  for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_down_sync(0xffffffffu, best, off));
  // non-negative doubles order like their bit patterns
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

int gf_download_owners(gf_ctx *ctx, uint64_t *voxel, uint16_t *sub, float *quat, double *lin_vel,
                       double *ang_vel, uint8_t *family) {
  CTX_CHECK(ctx);
  const int64_t n = c->n_owner;
  cudaStream_t s = c->s_dt;
  GF_CHECK(c, cudaDeviceSynchronize());   // the kT stream may still read the state
  if (!n) return 0;
  if (ensure_stage(c, n, s)) return -1;
  const Stage st = stage_of(c->owner_stage, n);
  k_owners_out<<<unsigned((n + 255) / 256), 256, 0, s>>>(n, c->sub.as<ushort4>(), c->lin_vel.p, c->ang_vel.p,
                                                       c->meta.as<uint32_t>(), st.sub3, st.lv, st.av, st.fam,
                                                       c->f32_state ? 1 : 0);
  if (voxel) GF_CHECK(c, cudaMemcpyAsync(voxel, c->voxel.p, 8 * n, cudaMemcpyDeviceToHost, s));
  if (quat) GF_CHECK(c, cudaMemcpyAsync(quat, c->quat.p, 16 * n, cudaMemcpyDeviceToHost, s));
  if (sub) GF_CHECK(c, cudaMemcpyAsync(sub, st.sub3, 6 * n, cudaMemcpyDeviceToHost, s));
  if (lin_vel) GF_CHECK(c, cudaMemcpyAsync(lin_vel, st.lv, 24 * n, cudaMemcpyDeviceToHost, s));
  if (ang_vel) GF_CHECK(c, cudaMemcpyAsync(ang_vel, st.av, 24 * n, cudaMemcpyDeviceToHost, s));
  if (family) GF_CHECK(c, cudaMemcpyAsync(family, st.fam, n, cudaMemcpyDeviceToHost, s));
  if (n >= (int64_t(1) << 24) && release_scratch(c, c->owner_stage, s)) return -1;
  GF_CHECK(c, cudaStreamSynchronize(s));
  return 0;
}

int gf_read_owners(gf_ctx *ctx, int64_t n, const int64_t *idx, double *out) {
  CTX_CHECK(ctx);
  if (n <= 0) return 0;
  for (int64_t r = 0; r < n; ++r)
    if (idx[r] < 0 || idx[r] >= c->n_owner) { c->err = "gf_read_owners: owner out of range"; return -1; }
  cudaStream_t s = c->s_dt;
  long long *d_idx = nullptr;
  double *d_out = nullptr;
  GF_CHECK(c, cudaMallocAsync(&d_idx, 8 * n, s));
  GF_CHECK(c, cudaMallocAsync(&d_out, 8 * 23 * n, s));
  GF_CHECK(c, cudaMemcpyAsync(d_idx, idx, 8 * n, cudaMemcpyHostToDevice, s));
  k_read_owners<<<unsigned((n + 127) / 128), 128, 0, s>>>(n, d_idx, c->voxel.as<uint64_t>(), c->sub.as<ushort4>(),
                                                          c->quat.as<float4>(), c->lin_vel.p, c->ang_vel.p,
                                                          c->meta.as<uint32_t>(), c->acc.as<double>(),
                                                          c->f32_state ? 1 : 0, d_out);
  GF_CHECK(c, cudaMemcpyAsync(out, d_out, 8 * 23 * n, cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(d_idx, s);
  cudaFreeAsync(d_out, s);
  GF_CHECK(c, cudaStreamSynchronize(s));
  return 0;
}

int gf_clump_max_absv(gf_ctx *ctx, double *out) {
  CTX_CHECK(ctx);
  *out = 0.0;
  if (!c->n_owner || !c->sph_first.p) return 0;
  cudaStream_t s = c->s_dt;
  unsigned long long *d = nullptr, h = 0;
  GF_CHECK(c, cudaMallocAsync(&d, 8, s));
  GF_CHECK(c, cudaMemsetAsync(d, 0, 8, s));
  k_clump_max_absv<<<unsigned(std::min<int64_t>((c->n_owner + 255) / 256, int64_t(c->n_sm) * 8)), 256, 0, s>>>(
      c->n_owner, c->sph_first.as<uint32_t>(), c->meta.as<uint32_t>(), c->fam_flags.as<uint8_t>(), c->lin_vel.p,
      c->f32_state ? 1 : 0, d);
  GF_CHECK(c, cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(d, s);
  GF_CHECK(c, cudaStreamSynchronize(s));
  std::memcpy(out, &h, 8);
  return 0;
}

int gf_set_owner_families(gf_ctx *ctx, const uint8_t *family) {
  CTX_CHECK(ctx);
  const int64_t n = c->n_owner;
  GF_CHECK(c, cudaDeviceSynchronize());
  std::vector<uint32_t> meta(n);
  GF_CHECK(c, cudaMemcpy(meta.data(), c->meta.p, 4 * n, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < n; ++i) meta[i] = (uint32_t(family[i]) << 24) | (meta[i] & 0xFFFFFFu);
  if (h2d(c, c->meta.p, meta.data(), 4 * n, c->s_dt)) return -1;
  world_moving_update(c);
  // the kinematics records carry the family's passive flag (the integrator
  // refreshes only their velocity halves)
  if (c->f32_state && c->n_sph && c->sph_first.p && c->sph_center.bytes >= size_t(32 * c->n_sph)) {
    if (refresh_centers(c, c->s_dt)) return -1;
    GF_CHECK(c, cudaStreamSynchronize(c->s_dt));
  }
  return 0;
}

int gf_apply_active_boxes(gf_ctx *ctx, int n_box, const double *boxes, const int64_t *anchors, int active_family,
                          int frozen_family, int64_t *n_changed) {
  CTX_CHECK(ctx);
  if (n_box < 0 || active_family < 0 || active_family > 255 || frozen_family < 0 || frozen_family > 255) {
    c->err = "gf_apply_active_boxes: bad arguments";
    return -1;
  }
  for (int b = 0; b < n_box; ++b)
    if (anchors[b] >= c->n_owner) { c->err = "gf_apply_active_boxes: anchor owner out of range"; return -1; }
  if (n_changed) *n_changed = 0;
  if (!c->n_owner || !n_box) return 0;
  cudaStream_t s = c->s_dt;
  double *d_box = nullptr;
  long long *d_anchor = nullptr;
  unsigned long long *d_cnt = nullptr;
  GF_CHECK(c, cudaMallocAsync(&d_box, sizeof(double) * 6 * n_box, s));
  GF_CHECK(c, cudaMallocAsync(&d_anchor, sizeof(long long) * n_box, s));
  GF_CHECK(c, cudaMallocAsync(&d_cnt, sizeof(unsigned long long), s));
  GF_CHECK(c, cudaMemcpyAsync(d_box, boxes, sizeof(double) * 6 * n_box, cudaMemcpyHostToDevice, s));
  GF_CHECK(c, cudaMemcpyAsync(d_anchor, anchors, sizeof(long long) * n_box, cudaMemcpyHostToDevice, s));
  GF_CHECK(c, cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s));
  if (active_boxes(c, n_box, d_box, d_anchor, uint32_t(active_family), uint32_t(frozen_family), d_cnt, s))
    return -1;
  unsigned long long h_cnt = 0;
  GF_CHECK(c, cudaMemcpyAsync(&h_cnt, d_cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(d_box, s);
  cudaFreeAsync(d_anchor, s);
  cudaFreeAsync(d_cnt, s);
  GF_CHECK(c, cudaStreamSynchronize(s));
  if (n_changed) *n_changed = int64_t(h_cnt);
  return 0;
}

int gf_set_persistent_wildcard(gf_ctx *ctx, int col) {
  CTX_CHECK(ctx);
  if (col >= c->wild_w) { c->err = "persistent wildcard column out of range"; return -1; }
  c->persist_col = col < 0 ? -1 : col;
  return 0;
}

int gf_set_external_loads(gf_ctx *ctx, const double *force, const double *torque) {
  CTX_CHECK(ctx);
  const int64_t n = c->n_owner;
  GF_CHECK(c, cudaDeviceSynchronize());
  if (!force && !torque) { c->has_ext = false; return 0; }
  if (ensure(c, c->ext, 48 * n, c->s_dt)) return -1;
  std::vector<double> e(6 * n, 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      if (force) e[6 * i + a] = force[3 * i + a];
      if (torque) e[6 * i + 3 + a] = torque[3 * i + a];
    }
  if (h2d(c, c->ext.p, e.data(), 48 * n, c->s_dt)) return -1;
  c->has_ext = true;
  return 0;
}

int gf_download_accumulators(gf_ctx *ctx, double *acc_force, double *acc_torque) {
  CTX_CHECK(ctx);
  const int64_t n = c->n_owner;
  GF_CHECK(c, cudaDeviceSynchronize());
  std::vector<double> a(6 * n);
  GF_CHECK(c, cudaMemcpy(a.data(), c->acc.p, 48 * n, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < n; ++i)
    for (int q = 0; q < 3; ++q) {
      if (acc_force) acc_force[3 * i + q] = a[6 * i + q];
      if (acc_torque) acc_torque[3 * i + q] = a[6 * i + 3 + q];
    }
  return 0;
}

static int upload_u32(Ctx *c, DBuf &b, const int64_t *src, int64_t n) {
  std::vector<uint32_t> v(n);
  for (int64_t i = 0; i < n; ++i) v[i] = uint32_t(src[i]);
  if (ensure(c, b, 4 * (n + 1), c->s_dt)) return -1;
  if (n && h2d(c, b.p, v.data(), 4 * n, c->s_dt)) return -1;
  return 0;
}

static int upload_raw(Ctx *c, DBuf &b, const void *src, size_t bytes) {
  if (ensure(c, b, bytes + 16, c->s_dt)) return -1;
  if (bytes && h2d(c, b.p, src, bytes, c->s_dt)) return -1;
  return 0;
}

int gf_upload_geometry(gf_ctx *ctx, int64_t n_s, const int64_t *sph_owner, const float *sph_params,
                       const uint8_t *sph_mat, int64_t n_t, const int64_t *tri_owner,
                       const float *tri_local, const uint8_t *tri_mat, int64_t n_a,
                       const int64_t *ana_owner, const uint8_t *ana_kind, const float *ana_local,
                       const uint8_t *ana_mat) {
  CTX_CHECK(ctx);
  c->h_tri_owner.assign(tri_owner, tri_owner + n_t);
  c->h_ana_owner.assign(ana_owner, ana_owner + n_a);
  GF_CHECK(c, cudaDeviceSynchronize());
  if (n_s >= (int64_t(1) << 30) || n_t >= (int64_t(1) << 30)) { c->err = "too many geometries"; return -1; }
  c->n_sph = n_s;
  c->n_tri = n_t;
  c->n_ana = n_a;
  if (upload_u32(c, c->sph_owner, sph_owner, n_s) || upload_raw(c, c->sph_offr, sph_params, 16 * n_s) ||
      upload_raw(c, c->sph_mat, sph_mat, n_s) || upload_u32(c, c->tri_owner, tri_owner, n_t) ||
      upload_raw(c, c->tri_local, tri_local, 36 * n_t) || upload_raw(c, c->tri_mat, tri_mat, n_t) ||
      upload_u32(c, c->ana_owner, ana_owner, n_a) || upload_raw(c, c->ana_kind, ana_kind, n_a) ||
      upload_raw(c, c->ana_local, ana_local, 32 * n_a) || upload_raw(c, c->ana_mat, ana_mat, n_a) ||
      ensure(c, c->tri_world, 72 * (n_t + 1), c->s_dt) || ensure(c, c->ana_world, 64 * (n_a + 1), c->s_dt))
    return -1;
  if (set_split(c, sph_params + 3, 4, n_s)) return -1;
  c->kt.cand_valid = false;
  c->lever_max = 0.0;
  for (int64_t k = 0; k < n_s; ++k) {
    const float *q = sph_params + 4 * k;
    double l = std::sqrt(double(q[0]) * q[0] + double(q[1]) * q[1] + double(q[2]) * q[2]) + double(q[3]);
    if (l > c->lever_max) c->lever_max = l;
  }
  for (int64_t k = 0; k < n_t; ++k)
    for (int v = 0; v < 3; ++v) {
      const float *q = tri_local + 9 * k + 3 * v;
      double l = std::sqrt(double(q[0]) * q[0] + double(q[1]) * q[1] + double(q[2]) * q[2]);
      if (l > c->lever_max) c->lever_max = l;
    }
  c->fx_h = -1.0;
  // spheres grouped by owner (ascending): CSR of each owner's sphere slots
  {
    std::vector<uint32_t> first(c->n_owner + 2, 0);
    for (int64_t k = 0; k < n_s; ++k) {
      if (k && sph_owner[k] < sph_owner[k - 1]) {
        c->err = "sphere slots must be grouped by ascending owner";
        return -1;
      }
      if (sph_owner[k] < 0 || sph_owner[k] >= c->n_owner) { c->err = "sphere owner out of range"; return -1; }
      first[sph_owner[k] + 1]++;
    }
    for (int64_t o = 0; o < c->n_owner; ++o) first[o + 1] += first[o];
    if (upload_raw(c, c->sph_first, first.data(), 4 * (c->n_owner + 1)) ||
        ensure(c, c->sph_center, 32 * (n_s + 1), c->s_dt) ||
        (c->f32_state && ensure(c, c->sph_kin, sizeof(SphKin) * (n_s + 1), c->s_dt)))
      return -1;
  }
  if (refresh_centers(c, c->s_dt)) return -1;
  world_moving_update(c);
  // world transforms of meshes / analytics for the current pose
  if (refresh_world(c, c->s_dt)) return -1;
  GF_CHECK(c, cudaStreamSynchronize(c->s_dt));
  return 0;
}

int gf_upload_materials(gf_ctx *ctx, int n_mat, int n_rows, const double *pair_stack, const double *beta) {
  CTX_CHECK(ctx);
  GF_CHECK(c, cudaDeviceSynchronize());
  if (n_rows < 5) { c->err = "pair stack needs rows E_cnt, G_cnt, CoR, mu, Crr"; return -1; }
  c->n_mat = n_mat;
  c->n_pair_rows = n_rows;
  if (upload_raw(c, c->pair, pair_stack, sizeof(double) * n_rows * n_mat * n_mat) ||
      upload_raw(c, c->beta, beta, sizeof(double) * n_mat * n_mat))
    return -1;
  return 0;
}

int gf_upload_families(gf_ctx *ctx, const uint8_t *mask, const uint8_t *flags, const uint8_t *lv_mask,
                       const uint8_t *av_mask, const double *lv_val, const double *av_val) {
  CTX_CHECK(ctx);
  GF_CHECK(c, cudaDeviceSynchronize());
  if (upload_raw(c, c->fam_mask, mask, 65536) || upload_raw(c, c->fam_flags, flags, 256) ||
      upload_raw(c, c->lv_mask, lv_mask, 256) || upload_raw(c, c->av_mask, av_mask, 256) ||
      upload_raw(c, c->lv_val, lv_val, sizeof(double) * 768) ||
      upload_raw(c, c->av_val, av_val, sizeof(double) * 768))
    return -1;
  c->mask_trivial = true;
  for (int q = 0; q < 65536; ++q)
    if (!mask[q]) { c->mask_trivial = false; break; }
  c->h_fam_flags.assign(flags, flags + 256);
  uint8_t passive[256];
  for (int f = 0; f < 256; ++f)
    passive[f] = ((flags[f] & kFamFixed) || (lv_mask[f] == 7 && av_mask[f] == 7)) ? 1 : 0;
  if (upload_raw(c, c->fam_passive, passive, 256)) return -1;
  world_moving_update(c);
  // the kinematics records carry the passive flag
  if (c->f32_state && c->n_sph && c->sph_first.p && c->sph_center.bytes >= size_t(32 * c->n_sph)) {
    if (refresh_centers(c, c->s_dt)) return -1;
    GF_CHECK(c, cudaStreamSynchronize(c->s_dt));
  }
  return 0;
}

int gf_download_world(gf_ctx *ctx, double *sph_centers, double *tri_world, double *ana_world) {
  CTX_CHECK(ctx);
  GF_CHECK(c, cudaDeviceSynchronize());
  if (sph_centers && c->n_sph) {
    if (kt_snapshot(c, c->s_dt)) return -1;
    GF_CHECK(c, cudaStreamSynchronize(c->s_dt));
    std::vector<double> c4(4 * c->n_sph);
    GF_CHECK(c, cudaMemcpy(c4.data(), c->kt.c4.p, 32 * c->n_sph, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < c->n_sph; ++i)
      for (int ax = 0; ax < 3; ++ax) sph_centers[3 * i + ax] = c4[4 * i + ax];
  }
  if (tri_world && c->n_tri) GF_CHECK(c, cudaMemcpy(tri_world, c->tri_world.p, 72 * c->n_tri, cudaMemcpyDeviceToHost));
  if (ana_world && c->n_ana) GF_CHECK(c, cudaMemcpy(ana_world, c->ana_world.p, 64 * c->n_ana, cudaMemcpyDeviceToHost));
  return 0;
}

int gf_set_acs(gf_ctx *ctx, int64_t n, const uint8_t *kind, const int64_t *slot_a, const int64_t *slot_b,
               const float *wild, int W) {
  CTX_CHECK(ctx);
  GF_CHECK(c, cudaDeviceSynchronize());
  if (W != c->wild_w) { c->err = "wildcard count differs from the active force model's"; return -1; }
  int64_t cap = n + n / 2 + 1024;
  // every array of the capacity carries its candidate-row column: the two
  // arrays alternate, and the compaction writes old_pos into whichever is next
  if (ensure(c, c->acs.ids, 8 * cap, c->s_dt) || ensure(c, c->acs.wild, 4 * W * cap, c->s_dt) ||
      ensure(c, c->acs.old_pos, 4 * cap, c->s_dt))
    return -1;
  c->acs.cap = cap;
  c->acs.n = n;
  c->acs.det_id = 0;   // installed: no candidate rows refer to it
  c->acs.pos_valid = false;
  std::vector<uint32_t> ids(2 * n);
  for (int64_t k = 0; k < n; ++k) {
    ids[2 * k] = uint32_t(slot_a[k]);
    ids[2 * k + 1] = uint32_t(slot_b[k]) | (uint32_t(kind[k]) << kKindShift);
  }
  if (n) {
    if (h2d(c, c->acs.ids.p, ids.data(), 8 * n, c->s_dt)) return -1;
    if (wild) {
      if (h2d(c, c->acs.wild.p, wild, 4 * W * n, c->s_dt)) return -1;
    } else {
      GF_CHECK(c, cudaMemsetAsync(c->acs.wild.p, 0, 4 * W * n, c->s_dt));
    }
  }
  if (build_segments(c, c->acs, c->s_dt) || build_incidence(c, c->s_dt)) return -1;
  GF_CHECK(c, cudaStreamSynchronize(c->s_dt));
  c->ca_updates = std::max<int64_t>(c->ca_updates, 1);
  return 0;
}

int64_t gf_acs_size(gf_ctx *ctx, int which) {
  if (!ctx) return -1;
  return which ? ctx->c.acs_next.n : ctx->c.acs.n;
}

int gf_get_acs(gf_ctx *ctx, int which, uint8_t *kind, int64_t *slot_a, int64_t *slot_b, float *wild) {
  CTX_CHECK(ctx);
  GF_CHECK(c, cudaDeviceSynchronize());
  Acs &a = which ? c->acs_next : c->acs;
  const int64_t n = a.n;
  if (!n) return 0;
  std::vector<uint32_t> ids(2 * n);
  GF_CHECK(c, cudaMemcpy(ids.data(), a.ids.p, 8 * n, cudaMemcpyDeviceToHost));
  for (int64_t k = 0; k < n; ++k) {
    if (slot_a) slot_a[k] = ids[2 * k];
    if (slot_b) slot_b[k] = ids[2 * k + 1] & kSlotMask;
    if (kind) kind[k] = uint8_t(ids[2 * k + 1] >> kKindShift);
  }
  if (wild && !which) GF_CHECK(c, cudaMemcpy(wild, a.wild.p, 4 * c->wild_w * n, cudaMemcpyDeviceToHost));
  return 0;
}

static int detect_now(Ctx *c, double margin, int64_t *n_out) {
  c->kt_margin = margin;
  if (kt_begin(c, margin, c->s_kt)) return -1;
  GF_CHECK(c, cudaStreamSynchronize(c->s_kt));
  if (kt_count(c, c->s_kt)) return -1;
  GF_CHECK(c, cudaStreamSynchronize(c->s_kt));
  c->acs_next.n = int64_t(reinterpret_cast<Status *>(c->h_status)->acs_total);
  if (kt_detect_fill(c, c->acs_next, c->s_kt)) return -1;
  GF_CHECK(c, cudaStreamSynchronize(c->s_kt));
  if (n_out) *n_out = c->acs_next.n;
  return 0;
}

int gf_detect(gf_ctx *ctx, double margin, int64_t *n_out) {
  CTX_CHECK(ctx);
  GF_CHECK(c, cudaDeviceSynchronize());
  if (kt_snapshot(c, c->s_kt)) return -1;
  return detect_now(c, margin, n_out);
}

int gf_detect_snapshot(gf_ctx *ctx, int64_t m, const double *centers, const float *radii,
                       const int64_t *sph_owner, const uint8_t *sph_family, int64_t n_t,
                       const double *tri_world, const int64_t *tri_owner, const uint8_t *tri_family,
                       int64_t n_a, const double *ana_world, const uint8_t *ana_kind,
                       const int64_t *ana_owner, const uint8_t *ana_family, const uint8_t *mask,
                       double margin, double bin_size, double *grid_out, int64_t *nb_out,
                       int64_t *n_out) {
  CTX_CHECK(ctx);
  c->kt_bin_size = bin_size;
  GF_CHECK(c, cudaDeviceSynchronize());
  c->n_sph = m;
  c->n_tri = n_t;
  c->n_ana = n_a;
  std::vector<float> offr(4 * m);
  for (int64_t i = 0; i < m; ++i) { offr[4 * i] = offr[4 * i + 1] = offr[4 * i + 2] = 0.f; offr[4 * i + 3] = radii[i]; }
  KtScratch &k = c->kt;
  if (upload_u32(c, c->sph_owner, sph_owner, m) || upload_raw(c, c->sph_offr, offr.data(), 16 * m) ||
      upload_raw(c, k.sfam, sph_family, m) ||
      upload_u32(c, c->tri_owner, tri_owner, n_t) || upload_raw(c, k.tri_world, tri_world, 72 * n_t) ||
      upload_raw(c, k.tfam, tri_family, n_t) || upload_u32(c, c->ana_owner, ana_owner, n_a) ||
      upload_raw(c, c->ana_kind, ana_kind, n_a) || upload_raw(c, k.ana_world, ana_world, 64 * n_a) ||
      upload_raw(c, k.afam, ana_family, n_a) || upload_raw(c, c->fam_mask, mask, 65536))
    return -1;
  {
    std::vector<double> c4(4 * m);
    for (int64_t i = 0; i < m; ++i) {
      c4[4 * i] = centers[3 * i]; c4[4 * i + 1] = centers[3 * i + 1]; c4[4 * i + 2] = centers[3 * i + 2];
      c4[4 * i + 3] = double(radii[i]);
    }
    if (upload_raw(c, k.c4, c4.data(), 32 * m)) return -1;
  }
  c->mask_trivial = true;
  for (int q = 0; q < 65536; ++q)
    if (!mask[q]) { c->mask_trivial = false; break; }
  if (set_split(c, radii, 1, m)) return -1;
  c->kt.cand_valid = false;
  int rc = detect_now(c, margin, n_out);
  c->kt_bin_size = 0.0;
  if (rc) return -1;
  Grid g;
  GF_CHECK(c, cudaMemcpy(&g, k.grid.p, sizeof(Grid), cudaMemcpyDeviceToHost));
  if (grid_out) { grid_out[0] = g.glo[0]; grid_out[1] = g.glo[1]; grid_out[2] = g.glo[2]; grid_out[3] = g.inv_bin; }
  if (nb_out) { nb_out[0] = g.nb[0]; nb_out[1] = g.nb[1]; nb_out[2] = g.nb[2]; }
  return 0;
}

int gf_bin_ranges(gf_ctx *ctx, double margin, int64_t *out) {
  CTX_CHECK(ctx);
  static_assert(sizeof(long long) == sizeof(int64_t), "int64");
  return kt_bin_ranges(c, margin, out);
}

static void pack_ids(int64_t n, const uint8_t *kind, const int64_t *a, const int64_t *b,
                     std::vector<uint32_t> &ids) {
  ids.resize(2 * n + 2);
  for (int64_t k = 0; k < n; ++k) {
    ids[2 * k] = uint32_t(a[k]);
    ids[2 * k + 1] = uint32_t(b[k]) | (uint32_t(kind[k]) << kKindShift);
  }
}

int gf_set_force_model(gf_ctx *ctx, const char *cuda_src, const char *include_dir, int W, char *log,
                       size_t log_n) {
  CTX_CHECK(ctx);
  GF_CHECK(c, cudaDeviceSynchronize());
  if (W < 1 || W > 64) { c->err = "wildcard count must be in [1, 64]"; return -1; }
  std::string lg;
  int rc = set_user_model(c, cuda_src, include_dir ? include_dir : ".", lg);
  if (log && log_n) {
    std::strncpy(log, lg.c_str(), log_n - 1);
    log[log_n - 1] = 0;
  }
  if (rc) return -1;
  c->wild_w = cuda_src ? W : 4;
  return 0;
}

int gf_set_profiling(gf_ctx *ctx, int on) {
  CTX_CHECK(ctx);
  GF_CHECK(c, cudaDeviceSynchronize());
  c->prof = on != 0;
  c->prof_used = 0;
  for (int q = 0; q < 5; ++q) c->prof_ms[q] = 0.0;
  c->prof_steps = 0;
  return 0;
}

int gf_kernel_times(gf_ctx *ctx, double *out6) {
  CTX_CHECK(ctx);
  for (int q = 0; q < 4; ++q) out6[q] = c->prof_ms[q];
  out6[4] = double(c->prof_steps);
  out6[5] = c->prof_ms[4];
  return 0;
}

int gf_merge_history(gf_ctx *ctx, int64_t n_old, const uint8_t *old_kind, const int64_t *old_a,
                     const int64_t *old_b, const float *old_wild, int64_t n_new,
                     const uint8_t *new_kind, const int64_t *new_a, const int64_t *new_b, int W,
                     float *out_wild) {
  CTX_CHECK(ctx);
  GF_CHECK(c, cudaDeviceSynchronize());
  std::vector<uint32_t> oi, ni;
  pack_ids(n_old, old_kind, old_a, old_b, oi);
  pack_ids(n_new, new_kind, new_a, new_b, ni);
  return merge_host(c, n_old, oi.data(), old_wild, n_new, ni.data(), W, out_wild);
}

int gf_adopt(gf_ctx *ctx) {
  CTX_CHECK(ctx);
  GF_CHECK(c, cudaDeviceSynchronize());
  if (adopt_acs(c, c->s_dt)) return -1;
  GF_CHECK(c, cudaStreamSynchronize(c->s_dt));
  return 0;
}

int gf_dt_step(gf_ctx *ctx, const gf_step_params *p, int64_t *touching, int64_t *bad, int64_t *oob) {
  CTX_CHECK(ctx);
  if (reset_status(c, c->s_dt)) return -1;
  c->n_dyn = 0;
  StepArgs a{p->h, {p->g[0], p->g[1], p->g[2]}, p->v_err, p->sim_time, p->step, 0, p->write_acc};
  if (dt_step(c, a)) return -1;
  Status st;
  if (read_status(c, c->s_dt, &st)) return -1;
  int64_t bs, os;
  if (touching) *touching = int64_t(st.touching);
  if (bad) decode_err(st.bad, *bad, bs);
  if (oob) decode_err(st.oob, *oob, os);
  return 0;
}

// One gf_run call: the deterministic kT/dT schedule over n_steps.  Split into
// begin / per-step forces / per-step integrate / end so a decomposed run can
// exchange ghost forces and ghost state between the halves (gf_run is the
// plain loop over them).
int gf_run_begin(gf_ctx *ctx, const gf_run_params *p) {
  CTX_CHECK(ctx);
  if (c->run) { c->err = "a run is already in progress (gf_run_end missing)"; return -1; }
  RunState *R = new RunState();
  R->w0 = std::chrono::steady_clock::now();
  R->p = *p;
  R->period = p->period < 1 ? 1 : p->period;
  R->lag = p->lag < 0 ? 0 : p->lag;
  R->trace = std::getenv("GF_TRACE") != nullptr;
  R->kt_freeze = std::getenv("GF_KT_FREEZE") != nullptr;
  c->run = R;
  const int64_t N = p->n_steps;
  c->kt_margin = p->margin;
  c->n_dyn = p->n_dyn;
  if (p->n_dyn > 0) {
    if (upload_raw(c, c->dyn_spec, p->dyn_spec, sizeof(int32_t) * 3 * p->n_dyn) ||
        upload_raw(c, c->dyn_vals, p->dyn_vals, sizeof(double) * p->n_dyn * (N > 0 ? N : 1)))
      return fail_run(c);
  }
  if (reset_status(c, c->s_dt)) return fail_run(c);
  if (cudaStreamSynchronize(c->s_dt) != cudaSuccess || cudaEventRecord(c->t0, c->s_dt) != cudaSuccess) {
    c->err = cudaGetErrorString(cudaGetLastError());
    return fail_run(c);
  }
  return 0;
}

int gf_step_forces(gf_ctx *ctx, int64_t i) {
  CTX_CHECK(ctx);
  RunState *R = c->run;
  if (!R) { c->err = "gf_step_forces outside gf_run_begin / gf_run_end"; return -1; }
  const gf_run_params *p = &R->p;
  const int64_t s = p->step0 + i;
  trace_mark(c, "dt_step_begin", s, c->s_dt);
  // 1. a detection due at this step boundary is adopted first
  if (c->next_pending && s >= c->adopt_at) {
    if (run_adopt(c) || dbg_sync(c, "run_adopt", s)) return -1;
    trace_mark(c, "dt_adopted", s, c->s_dt);
  }
  // 2. work order: snapshot on the dT stream, detection on the kT stream
  // GF_KT_FREEZE=1 (timing diagnostics only): no work orders after the first
  // detection, so a run measures the dT chain alone on a frozen contact array
  if (!c->next_pending && (c->first_adopt || (!R->kt_freeze && s - c->last_snap >= R->period))) {
    if (c->snap_async) {
      // the snapshot runs on the kT stream, overlapped with this step's force
      // phase (both only read the state the last integration left); this
      // step's integration waits for it before overwriting the centres
      GF_CHECK(c, cudaEventRecord(c->ev_snap, c->s_dt));
      GF_CHECK(c, cudaStreamWaitEvent(c->s_kt, c->ev_snap, 0));
      GF_CHECK(c, cudaStreamWaitEvent(c->s_kt, c->ev_adopted, 0));
      if (kt_snapshot(c, c->s_kt, p->margin)) return -1;
      GF_CHECK(c, cudaEventRecord(c->ev_snap_done, c->s_kt));
      c->snap_wait = true;
    } else {
      if (kt_snapshot(c, c->s_dt, p->margin) || dbg_sync(c, "kt_snapshot", s)) return -1;
      GF_CHECK(c, cudaEventRecord(c->ev_snap, c->s_dt));
      GF_CHECK(c, cudaStreamWaitEvent(c->s_kt, c->ev_snap, 0));
      GF_CHECK(c, cudaStreamWaitEvent(c->s_kt, c->ev_adopted, 0));
    }
    // retire completed detections' timing events (every one but the newest
    // has been adopted, so its end event is recorded), then reuse a pair
    while (R->kt_ev.size() > 1 || (!R->kt_ev.empty() && cudaEventQuery(R->kt_ev.front().second) == cudaSuccess)) {
      auto e = R->kt_ev.front();
      if (cudaEventQuery(e.second) != cudaSuccess) break;
      float m = 0.f;
      if (cudaEventElapsedTime(&m, e.first, e.second) == cudaSuccess) R->kt_ms += m;
      R->kt_ev.pop_front();
      R->kt_ev_free.push_back(e);
    }
    (void)cudaGetLastError();   // a not-ready query is not an error
    std::pair<cudaEvent_t, cudaEvent_t> e;
    if (!R->kt_ev_free.empty()) {
      e = R->kt_ev_free.back();
      R->kt_ev_free.pop_back();
    } else {
      DevGuard g(c->kt_device);
      GF_CHECK(c, cudaEventCreate(&e.first));
      GF_CHECK(c, cudaEventCreate(&e.second));
    }
    R->kt_ev.push_back(e);
    GF_CHECK(c, cudaEventRecord(e.first, c->s_kt));
    trace_mark(c, "dt_snapshot_end", s, c->s_dt);
    if (kt_begin(c, p->margin, c->s_kt) || dbg_sync(c, "kt_begin", s)) return -1;
    GF_CHECK(c, cudaEventRecord(c->ev_disp, c->s_kt));
      trace_mark(c, "kt_phaseA_end", s, c->s_kt);
    c->kt_phase = 1;
    c->next_pending = true;
    c->fill_done = false;
    c->last_snap = s;
    // the very first detection is waited for (engine.py:679-682)
    c->adopt_at = c->first_adopt ? s : s + R->lag;
    if (c->adopt_at <= s && run_adopt(c)) return -1;
  }
  // 3. advance a staged rebuild; launch the fill as soon as the count is
  // known (no dT stall)
  if (c->next_pending && c->kt_phase == 3 && (advance_kt(c, false) || dbg_sync(c, "advance_kt", s))) return -1;
  if (c->next_pending && !c->fill_done && c->kt_phase == 2) {
    cudaError_t q = cudaEventQuery(c->ev_count);
    if (q == cudaErrorNotReady) {
      if (cudaPeekAtLastError() == cudaErrorNotReady) (void)cudaGetLastError();
    } else if (run_fill(c) || dbg_sync(c, "run_fill", s)) {
      return -1;
    }
  }
  R->sum_acs += c->acs.n;
  const StepArgs a = step_args(R, i);
  if (update_fixed_scales(c, a.h, a.v_err, a.g)) return -1;
  trace_mark(c, "dt_forces_begin", s, c->s_dt);
  const int rc = c->f32_state ? dt_forces_f32(c, a, c->s_dt) : dt_forces_f64(c, a, c->s_dt);
  trace_mark(c, "dt_forces_end", s, c->s_dt);
  if (rc == 0 && dbg_sync(c, "dt_forces", s)) return -1;
  return rc;
}

int gf_step_integrate(gf_ctx *ctx, int64_t i) {
  CTX_CHECK(ctx);
  RunState *R = c->run;
  if (!R) { c->err = "gf_step_integrate outside gf_run_begin / gf_run_end"; return -1; }
  const StepArgs a = step_args(R, i);
  if (c->snap_wait) {   // the kT stream's snapshot of this step's start state
    GF_CHECK(c, cudaStreamWaitEvent(c->s_dt, c->ev_snap_done, 0));
    c->snap_wait = false;
  }
  if (c->f32_state ? dt_integrate_f32(c, a, c->s_dt) : dt_integrate_f64(c, a, c->s_dt)) return -1;
  if (dbg_sync(c, "dt_integrate", a.step)) return -1;
  trace_mark(c, "dt_integrate_end", a.step, c->s_dt);
  // the detection's candidate filter is queued once the dT step is in flight
  if (c->next_pending && c->kt_phase == 1 && (run_count(c) || dbg_sync(c, "run_count", a.step))) return -1;
  if (c->next_pending && c->kt_phase == 3 && (advance_kt(c, false) || dbg_sync(c, "advance_kt", a.step))) return -1;
  return 0;
}

int gf_run_end(gf_ctx *ctx, gf_run_result *r) {
  CTX_CHECK(ctx);
  RunState *R = c->run;
  if (!R) { c->err = "gf_run_end without gf_run_begin"; return -1; }
  std::memset(r, 0, sizeof(*r));
  const gf_run_params *p = &R->p;
  const int64_t N = p->n_steps;
  // finish enqueuing an in-flight detection (its fill) inside this call
  if (c->next_pending && !c->fill_done && run_fill(c)) return fail_run(c);
  // join the kT stream so in-flight detection work counts in the timed window
  if (cudaEventRecord(c->ev_kt_join, c->s_kt) != cudaSuccess ||
      cudaStreamWaitEvent(c->s_dt, c->ev_kt_join, 0) != cudaSuccess ||
      cudaEventRecord(c->t1, c->s_dt) != cudaSuccess || cudaStreamSynchronize(c->s_kt) != cudaSuccess) {
    c->err = cudaGetErrorString(cudaGetLastError());
    return fail_run(c);
  }
  Status st;
  if (read_status(c, c->s_dt, &st)) return fail_run(c);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->t0, c->t1);
  r->dt_ms = ms;
  double kt_ms = R->kt_ms;
  for (auto &e : R->kt_ev) {
    float m = 0.f;
    if (cudaEventElapsedTime(&m, e.first, e.second) == cudaSuccess) kt_ms += m;
  }
  (void)cudaGetLastError();  // an unrecorded timing event is not an error
  r->kt_ms = kt_ms;
  if (R->trace) {
    std::fprintf(stderr, "GF_TRACE host_wait_ms count=%.3f fill=%.3f\n", R->host_wait_ms[0], R->host_wait_ms[1]);
    for (auto &m : R->marks) {
      float ms = -1.f;
      cudaEventElapsedTime(&ms, c->t0, m.ev);
      std::fprintf(stderr, "GF_TRACE %s %lld %.4f\n", m.what, (long long)m.step, ms);
      cudaEventDestroy(m.ev);
    }
    (void)cudaGetLastError();
  }
  if (c->prof) {
    prof_collect(c);
    c->prof_ms[3] += kt_ms;
  }
  decode_err(st.bad, r->bad_owner, r->bad_step);
  decode_err(st.oob, r->oob_owner, r->oob_step);
  int64_t err_step = -1;
  if (r->bad_step >= 0) err_step = r->bad_step;
  if (r->oob_step >= 0 && (err_step < 0 || r->oob_step < err_step)) err_step = r->oob_step;
  r->steps_done = err_step >= 0 ? err_step - p->step0 : N;
  r->dd_trip_step = st.dd_trip == ~0ull ? -1 : int64_t(st.dd_trip);
  if (r->dd_trip_step >= 0 && r->dd_trip_step + 1 - p->step0 < r->steps_done)
    r->steps_done = r->dd_trip_step + 1 - p->step0;
  r->touching = int64_t(st.touching);
  r->sum_touch_pairs = int64_t(st.touch_pairs);
  r->sum_acs = R->sum_acs;
  r->n_acs = c->acs.n;
  r->ca_updates = c->ca_updates;
  r->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - R->w0).count();
  r->kt_rebuilds = c->kt.rebuilds;
  free_run(c);
  return 0;
}

int gf_run(gf_ctx *ctx, const gf_run_params *p, gf_run_result *r) {
  if (gf_run_begin(ctx, p)) return -1;
  for (int64_t i = 0; i < p->n_steps; ++i)
    if (gf_step_forces(ctx, i) || gf_step_integrate(ctx, i)) {
      free_run(&ctx->c);
      return -1;
    }
  return gf_run_end(ctx, r);
}

// ---------------------------------------------------------------------------
// spatial decomposition (gf_halo.cu)
// ---------------------------------------------------------------------------
int gf_set_decomposition(gf_ctx *ctx, const uint32_t *dd, double lever_max, int axis, double travel) {
  CTX_CHECK(ctx);
  if (!dd) {
    c->dd_on = false;
    c->lever_override = 0.0;
  } else {
    if (!c->fixed_reduce) {
      c->err = "spatial decomposition needs the fixed-point owner reduction (GF_STATE_F32)";
      return -1;
    }
    if (c->split) {
      c->err = "spatial decomposition and the 2-GPU kT/dT split are separate modes";
      return -1;
    }
    if (ensure(c, c->dd, 4 * (c->n_owner + 1), c->s_dt)) return -1;
    if (axis < 0 || axis > 2) { c->err = "decomposition axis must be 0, 1 or 2"; return -1; }
    if (h2d(c, c->dd.p, dd, 4 * c->n_owner, c->s_dt)) return -1;
    // partition-time axis coordinate of every owner (device-side decode)
    if (ensure(c, c->dd_x0, 8 * (c->n_owner + 1), c->s_dt)) return -1;
    if (halo_axis_coords(c, axis, c->dd_x0.as<double>(), c->s_dt)) return -1;
    GF_CHECK(c, cudaStreamSynchronize(c->s_dt));
    c->dd_axis = axis;
    c->dd_travel = travel;
    c->dd_on = true;
    c->lever_override = lever_max;
  }
  c->fx_h = -1.0;              // fixed-point scales follow the (global) lever arm
  c->kt.cand_valid = false;    // candidate lists were filtered with the old classes
  return 0;
}

int gf_halo_record_bytes(gf_ctx *ctx) {
  if (!ctx) return -1;
  return halo_record_bytes(&ctx->c);
}

void *gf_stream(gf_ctx *ctx) { return ctx ? reinterpret_cast<void *>(ctx->c.s_dt) : nullptr; }

int gf_pack_state(gf_ctx *ctx, const uint32_t *idx, int64_t n, void *out) {
  CTX_CHECK(ctx);
  return halo_pack_state(c, idx, n, out, c->s_dt);
}

int gf_unpack_state(gf_ctx *ctx, const uint32_t *idx, int64_t n, const void *in) {
  CTX_CHECK(ctx);
  return halo_unpack_state(c, idx, n, in, c->s_dt);
}

int gf_pack_forces(gf_ctx *ctx, const uint32_t *idx, int64_t n, void *out) {
  CTX_CHECK(ctx);
  if (!c->fixed_reduce) { c->err = "gf_pack_forces needs the fixed-point owner reduction"; return -1; }
  return halo_pack_forces(c, idx, n, out, c->s_dt);
}

int gf_add_forces(gf_ctx *ctx, const uint32_t *idx, int64_t n, const void *in) {
  CTX_CHECK(ctx);
  if (!c->fixed_reduce) { c->err = "gf_add_forces needs the fixed-point owner reduction"; return -1; }
  return halo_add_forces(c, idx, n, in, c->s_dt);
}

int gf_trip_word(gf_ctx *ctx, void *word, int mode) {
  CTX_CHECK(ctx);
  return halo_trip_word(c, word, mode, c->s_dt);
}

int gf_sync(gf_ctx *ctx) {
  CTX_CHECK(ctx);
  GF_CHECK(c, cudaStreamSynchronize(c->s_dt));
  return 0;
}

}  // extern "C"
