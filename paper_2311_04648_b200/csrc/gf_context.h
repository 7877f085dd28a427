// gf_context.h -- host-side device context behind the C-ABI (include/gf_b200.h).
#pragma once
#include <cuda.h>   // CUtensorMap
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "gf_common.cuh"

namespace gf {

// A growable device buffer (stream-ordered allocator; no device-wide syncs).
struct DBuf {
  void *p = nullptr;
  size_t bytes = 0;
  template <class T> T *as() const { return reinterpret_cast<T *>(p); }
  void release() {   // callers synchronise first
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// Active contact set in device layout.  ids.x = sphere slot of A;
// ids.y = slot of B within its kind | kind << 30.  Canonical order is
// (kind, a, b), identical to the reference's (kind, geom_a, geom_b) order
// because slots are monotone in geometry id within each kind
// (engine.py:446-455).
struct Acs {
  int64_t n = 0, cap = 0;
  DBuf ids;    // uint2[cap]
  DBuf wild;   // float[cap * W]
  DBuf seg;    // uint64[3 n_sph + 1]: start of each (kind, sphere A) segment
  // history remap by candidate slot (gf_kt.cu k_filter_compact): for each
  // sphere-sphere entry, its row in the array of detection prev_det (~0u:
  // not there); valid only while the candidate list is unchanged
  DBuf old_pos;              // uint32[cap]
  uint64_t det_id = 0;       // detection serial that produced this array (0: installed)
  uint64_t prev_det = 0;     // detection whose rows old_pos refers to
  bool pos_valid = false;
};

struct KtScratch {
  // snapshot (kT works on a frozen copy; engine.py:577-596)
  DBuf c4;           // double4[n_s] (centre, radius)
  DBuf sfam;         // uint8[n_s] sphere family
  DBuf tri_world;    // double[n_t*9]
  DBuf ana_world;    // double[n_a*8]
  DBuf tfam, afam;   // uint8 families of tri / ana
  DBuf grid;         // Grid
  DBuf minmax;       // double[6]
  // binning
  DBuf bin_key, bin_key_alt, sph_val, sph_val_alt;  // uint32[n_s]
  DBuf cell_start, cell_end;                         // uint32[nbins]
  DBuf tri_ranges;                                   // int32[n_t*6]
  DBuf tri_cnt, tri_start, tri_entries;              // tri CSR over bins
  DBuf cursor;       // uint32[3 n_s] fill cursor of each (kind, sphere) segment
  DBuf sc, sm, sf;   // cell-sorted copies: double4 (centre, radius), uint4 (slot, owner, family),
                     // float4 (centre - grid origin, radius) for the conservative fp32 prefilter
  DBuf tmp, tmp_n;   // scratch pair list (uint2) and its append counter
  DBuf cells, n_cells;  // non-empty enumeration cells
  // Verlet candidate lists (rebuilt when a sphere moved > skin / 2)
  DBuf cand, cand_tmp, cand_n, cand_cnt, cand_seg, ref, flag, cflags, sel_n;
  DBuf cand_own;     // slot-grouped rebuild: each cell-sorted sphere's own-slot pair count
  int64_t cand_cap = 0, n_cand = 0, rebuilds = 0, big_cap = 0;
  // hit bitmask and scanned per-block hit counts of the last two filtered
  // arrays (double-buffered), with the detection serial / candidate
  // generation they belong to
  DBuf fbits[2], fpre[2], fcnt;
  int cslot_cur = 0;
  uint64_t cslot_det[2] = {0, 0};
  int64_t cslot_gen[2] = {-1, -1};
  int64_t cand_gen = 0;
  uint64_t det_serial = 0;
  int64_t last_ss = 0, ss_need = 0;
  bool snap_det = false, snap_checked = false;   // the last snapshot reduced the grid inputs / ran k_disp
  // sphere-analytic candidates (while no mesh / analytic owner moves):
  // per-sphere segments of analytic ids within margin + skin at the rebuild
  DBuf sa_cnt, sa_off, sa_cand;
  int64_t n_sa_cand = 0;
  uint64_t sa_world_version = ~0ull;   // sphere-sphere block size of the last detection / after an overflow
  bool cand_valid = false;
  double cand_skin = -1.0;
  int64_t tmp_cap = 0;
  DBuf tri_cursor;   // uint32 per cell
  DBuf gaps;         // long runs of segment starts filled by k_fill_gaps
  // a staged candidate rebuild in flight (gf_kt.cu rb_stage_*): next stage
  // 1..3, 0 = none; its small-pair count and big-pair capacity
  int rb_stage = 0;
  int64_t rb_small = 0, rb_big_cap = 0;
  bool rb_sa = false;
  DBuf counts;       // uint64[3*n_s+1] per sphere SS / ST / SA counts
  DBuf offsets;      // uint64? uint32[3*n_s+1] exclusive scan
  DBuf cub_tmp;
  DBuf total;        // device copy of totals
  int64_t nbins_cap = 0;
  bool sort_long_smem = false;   // k_sort_long's 64 KB dynamic shared memory opted in on this context's device
};

// Sets the current device for a scope (the 2-GPU kT/dT split launches kT work
// on the kT device and allocates contact arrays on the dT device).
struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
// the device a stream belongs to
inline int stream_device(cudaStream_t s) {
  int d = -1;
  if (cudaStreamGetDevice(s, &d) != cudaSuccess) {
    (void)cudaGetLastError();
    cudaGetDevice(&d);
  }
  return d;
}

struct Ctx {
  int device = 0;
  // the paper's 2-GPU split: the kT stream, its scratch and
  // events live on kt_device; contact arrays, state and the dT stream on
  // `device`; kT kernels read the dT device's tables and write the contact
  // arrays through NVLink peer access.  split = false: one device.
  int kt_device = 0;
  bool split = false;
  cudaEvent_t ev_kt_join = nullptr;   // recorded on s_kt (kT device) at the end of a run
  cudaEvent_t ev_snap_done = nullptr; // the kT-stream snapshot of a step's start state is complete
  bool ss_tma = false;      // B-side centre gathers by TMA gather4 in the fused kernel (GF_SS_TMA=1)
  bool ss_tma_smem = false; // its dynamic shared-memory opt-in is set (per context: per device)
  alignas(64) CUtensorMap tm_center;   // the sphere-centre records as a 2-D tensor (rows of 4 doubles)
  void *tm_center_ptr = nullptr;
  int64_t tm_center_n = -1;
  bool rb_slot = true;      // candidate rebuild grouped by slot with atomic cursors (GF_RB_SLOT=0: pair radix sort)
  bool rb_async = true;     // staged non-blocking candidate rebuild inside runs (GF_RB_ASYNC=0: blocking)
  bool snap_async = false;  // snapshot on the kT stream (GF_SNAP_ASYNC=1); measured neutral: the force kernels fill every SM
  bool snap_wait = false;   // the next integration waits for ev_snap_done
  uint32_t flags = 0;
  bool f32_state = false;
  std::string err;
  cudaStream_t s_dt = nullptr, s_kt = nullptr;
  cudaEvent_t ev_snap = nullptr, ev_ca = nullptr, ev_adopted = nullptr, ev_count = nullptr, ev_disp = nullptr;
  int kt_phase = 0;  // in-flight detection: 1 begun, 2 counted, 3 staged rebuild in flight
  cudaEvent_t t0 = nullptr, t1 = nullptr;

  Domain dom{};
  // owners
  int64_t n_owner = 0, n_tpl = 0;
  DBuf voxel, sub, quat, lin_vel, ang_vel, meta, tpl, acc, ext, facc, tpl_scale;
  bool fixed_reduce = false;  // throughput build: int64 fixed-point atomic owner reduction
  std::vector<double> h_tpl_mass;
  double lever_max = 0.0, fx_h = -1.0, fx_verr = -1.0;
  bool has_ext = false;
  // geometry
  int64_t n_sph = 0, n_tri = 0, n_ana = 0;
  DBuf sph_owner, sph_offr, sph_mat, sph_center, sph_first;
  DBuf sph_kin;  // SphKin per sphere (fp32-velocity build)
  DBuf tri_owner, tri_local, tri_mat, tri_world;
  DBuf ana_owner, ana_kind, ana_local, ana_mat, ana_world;
  bool world_moving = true;  // any tri/ana owner not fixed
  // enumeration split: spheres with radius > r_cut are paired by k_big
  double r_cut = 0.0;
  int64_t n_big = 0;
  DBuf big_slots;
  // tables
  int n_mat = 0, n_pair_rows = 0;
  DBuf pair, beta;
  DBuf fam_mask, fam_flags, lv_mask, av_mask, lv_val, av_val, fam_passive;
  std::vector<uint8_t> h_fam_flags;
  bool mask_trivial = true;  // every family pair may contact
  // contact arrays
  int wild_w = 4;
  Acs acs, acs_next;
  bool next_pending = false;
  int64_t next_count = 0;
  // per-contact outputs and incidence lists (sized with acs.cap)
  DBuf out_c;      // double[cap*9]: F(3), F+tof(3), contact point(3)
  DBuf touch;      // uint8[cap]
  DBuf tlist, tlist_n;  // compacted touching entries of the current step (two lists, two counters)
  int64_t tlist_cap = 0;
  DBuf inc, inc_alt, inc_key, inc_key_alt;  // uint32[2*cap]
  DBuf inc_start;  // uint32[n_owner+1]
  DBuf heavy;      // uint32 list of heavy owners
  DBuf heavy_count;  // unsigned long long
  DBuf heavy_acc;  // double[n_owner*6]
  DBuf cub_tmp_dt;
  // flags / counters (device) and pinned host mirrors
  DBuf status;     // Status struct
  void *h_status = nullptr;  // pinned mirror
  KtScratch kt;
  // dynamic prescriptions
  DBuf dyn_spec, dyn_vals;
  int n_dyn = 0;
  double kt_margin = 0.0;
  double kt_bin_size = 0.0;  // > 0: explicit bin size (detect_contacts(bin_size=...))
  double skin_factor = 1.0;  // Verlet skin = skin_factor * margin
  double skin_big_factor = 8.0;  // skin of big spheres (radius > r_cut), >= skin_factor (GF_SKIN_BIG)
  uint64_t world_version = 0;   // bumped whenever mesh / analytic world transforms are recomputed
  int tlist_words = 5;       // words per contact of the touching lists (1 on the fused path)
  int persist_col = -1;      // wildcard column whose > 0 rows persist across detections (bonds), or -1
  int64_t persisted = 0;     // rows re-appended by that rule so far
  int n_sm = 148;             // multiprocessors of the device (grid sizing)
  int ss_blocked = 2;        // fused kernel: contiguous entry range per CTA (1), grid-stride (0), auto by size (2)
  int ss_pf = 1;             // fused kernel read-ahead / prefetch (GF_SS_PF=0: off)
  int ss_red = 1;            // fused sphere-sphere kernel: staged fixed-point rows (GF_SS_RED=0: per-word REDs)
  int ss_split = 0;          // throughput build: split narrow/force sphere-sphere kernels (GF_SS_SPLIT=1)
  // programmatic dependent launch on the dT chain (GF_PDL=1): measured slower
  // on the bench bed (the chain's kernels already fill the GPU), off by default
  int pdl = 0;
  // schedule state (kept across gf_run calls)
  bool first_adopt = true;     // the first do_dynamics detects and waits (engine.py:679-682)
  bool fill_done = false;
  int64_t last_snap = 0;
  int64_t adopt_at = 0;
  int64_t step = 0;
  int64_t ca_updates = 0;
  double t_kt_ms = 0.0, t_dt_ms = 0.0;
  int64_t last_touching = 0;
  // NVRTC user force model (gf_nvrtc.cu)
  bool user_model = false;
  void *user_fn_f64 = nullptr, *user_fn_f32 = nullptr, *user_fn_ss = nullptr, *user_fn_walls = nullptr;
  void *user_fn_ref = nullptr, *user_fn_batch = nullptr;   // gf_contact_forces / gf_eval_core of a user model
  // per-kernel device timing (enabled by gf_set_profiling)
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;   // kProfEv per profiled step: start, contacts, heavy, integrate,
                                      // after the fused sphere-sphere kernel
  size_t prof_used = 0;
  double prof_ms[5] = {0, 0, 0, 0, 0};   // contacts, heavy, integrate, kT, sphere-sphere kernel
  int64_t prof_steps = 0;
  // spatial decomposition (gf_set_decomposition): per-owner class | gid << 2
  DBuf dd, dd_x0;
  bool dd_on = false;
  int dd_axis = 0;
  double dd_travel = 0.0;
  double lever_override = 0.0;   // global lever arm so fixed-point scales agree across ranks
  DBuf owner_stage;              // host-layout staging of gf_upload_owners / gf_download_owners
  std::vector<uint32_t> h_tri_owner, h_ana_owner;   // mesh / analytic owners (world_moving)
  std::vector<double> h_tpl_moi;
  DBuf halo_scratch;             // uint32 index staging for host-index halo calls
  // split-step run in progress (gf_run_begin ... gf_run_end)
  struct RunState *run = nullptr;
};

// take 4 timing events for one profiled dT step (nullptr when off)
constexpr int kProfEv = 5;
// throughput build, built-in model: the fused sphere-sphere contact kernel
inline bool ss_fused(const Ctx *c) { return c->f32_state && c->wild_w == 4 && !c->user_model && c->ss_split != 1; }
cudaEvent_t *prof_events(Ctx *c);
// the set the current step's force phase opened (nullptr when off)
cudaEvent_t *prof_current(Ctx *c);

constexpr uint32_t kHeavyThreshold = 192;
constexpr int64_t kMaxCells = (int64_t(1) << 24) - 1;  // enumeration-grid cell cap; key 2^24-1 = unregistered  // incidences above which an owner is block-reduced

// helpers implemented in gf_context.cu
int ensure(Ctx *c, DBuf &b, size_t bytes, cudaStream_t s, bool keep = false);
// rebuild-only kT scratch: from 2^24 spheres up (big_scratch) it is taken
// from and returned to the stream-ordered pool on the kT stream
// (cudaMallocAsync / cudaFreeAsync: no device-wide sync); below, ensure()
inline bool big_scratch(const Ctx *c) { return c->n_sph >= (int64_t(1) << 24); }
int ensure_scratch(Ctx *c, DBuf &b, size_t bytes, cudaStream_t s);
int ensure_pooled(Ctx *c, DBuf &b, size_t bytes, cudaStream_t s);   // always from the pool
int release_scratch(Ctx *c, DBuf &b, cudaStream_t s);
// host -> device copy ordered on stream s and complete on return: the context's
// streams are non-blocking, so a legacy-stream cudaMemcpy is not ordered
// with kernels launched on them afterwards (its DMA may land after they read)
int h2d(Ctx *c, void *dst, const void *src, size_t bytes, cudaStream_t s);
void set_err(Ctx *c, const std::string &msg);
#define GF_CHECK(c, call)                                                      \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) {                                                   \
      gf::set_err((c), std::string(#call) + ": " + cudaGetErrorString(_e));    \
      return -1;                                                               \
    }                                                                          \
  } while (0)

// views
Owners owners_view(Ctx *c);
Spheres spheres_view(Ctx *c);
Tris tris_view(Ctx *c);
Anas anas_view(Ctx *c);
Materials materials_view(Ctx *c);
Families families_view(Ctx *c);

// kT (gf_kt.cu)
int kt_snapshot(Ctx *c, cudaStream_t s, double margin = -1.0);   // centers/families -> kT scratch
                                                          // (margin >= 0: a detection's, with grid inputs)
int kt_begin(Ctx *c, double margin, cudaStream_t s);               // grid + displacement check
int kt_count(Ctx *c, cudaStream_t s, bool force_rebuild = false);   // candidates -> counts
int center_tmap(Ctx *c);   // (re)encode tm_center for the current centre buffer
int kt_count_async(Ctx *c, cudaStream_t s);   // 1 = a staged rebuild started (resume with kt_advance)
int kt_advance(Ctx *c, cudaStream_t s, cudaEvent_t ev, bool block);   // 1 = stages remain
int kt_detect_fill(Ctx *c, Acs &out, cudaStream_t s);
int kt_bin_ranges(Ctx *c, double margin, int64_t *h_out);
int adopt_acs(Ctx *c, cudaStream_t s);                   // merge history + incidence lists
int build_incidence(Ctx *c, cudaStream_t s);
int build_segments(Ctx *c, Acs &a, cudaStream_t s);
int merge_host(Ctx *c, int64_t n_old, const uint32_t *old_ids, const float *old_wild, int64_t n_new,
               const uint32_t *new_ids, int W, float *out_wild);
int refresh_world(Ctx *c, cudaStream_t s);               // tri/ana world from owner pose
int refresh_centers(Ctx *c, cudaStream_t s);             // sphere world centres from owner pose

// NVRTC user force models (gf_nvrtc.cu)
struct DtView;
int set_user_model(Ctx *c, const char *src, const char *include_dir, std::string &log);
int launch_user_forces(Ctx *c, const DtView &v, double ts, double sim_time, cudaStream_t s);
int nvrtc_compile_check(const char *src, const char *include_dir, std::string &log);

// dT (gf_dt_f64.cu / gf_dt_f32.cu)
struct StepArgs {
  double h, g[3], v_err, sim_time;
  int64_t step;          // global step index (for watchdog records)
  int64_t dyn_row;       // row of the dynamic-prescription table for this step
  int write_acc;         // store per-owner accumulators this step
};
int dt_step_f64(Ctx *c, const StepArgs &a, cudaStream_t s);
// halo exchange of the spatial decomposition (gf_halo.cu)
int halo_record_bytes(const Ctx *c);
int halo_axis_coords(Ctx *c, int axis, double *out, cudaStream_t s);
int halo_trip_word(Ctx *c, void *word, int mode, cudaStream_t s);
int halo_pack_state(Ctx *c, const uint32_t *idx, int64_t n, void *out, cudaStream_t s);
int halo_unpack_state(Ctx *c, const uint32_t *idx, int64_t n, const void *in, cudaStream_t s);
int halo_pack_forces(Ctx *c, const uint32_t *idx, int64_t n, void *out, cudaStream_t s);
int halo_add_forces(Ctx *c, const uint32_t *idx, int64_t n, const void *in, cudaStream_t s);
int active_boxes(Ctx *c, int n_box, const double *box, const long long *anchor, uint32_t active, uint32_t frozen,
                 unsigned long long *n_changed, cudaStream_t s);
int dt_forces_f32(Ctx *c, const StepArgs &a, cudaStream_t s);
int dt_integrate_f32(Ctx *c, const StepArgs &a, cudaStream_t s);
int dt_forces_f64(Ctx *c, const StepArgs &a, cudaStream_t s);
int dt_integrate_f64(Ctx *c, const StepArgs &a, cudaStream_t s);
int dt_step_f32(Ctx *c, const StepArgs &a, cudaStream_t s);

// GF_SYNC_DEBUG=1: device sync + fault attribution (gf_context.cu)
int dbg_sync(Ctx *c, const char *what, int64_t step);
bool sync_debug();

}  // namespace gf
