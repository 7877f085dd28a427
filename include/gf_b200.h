/*
 * gf_b200.h -- C-ABI of the B200-native DEM step (libgf_b200.so).
 *
 * Plain pointers and sizes only; the caller owns every host buffer, the
 * context owns every device buffer.  All array layouts are the reference's
 * numpy layouts (row-major; int64 ids; float32 radii / quaternions / geometry
 * parameters / contact history; float64 state), so a host that holds
 * grainforge.StateStore arrays can pass them through unchanged.
 *
 * Return codes: 0 = ok, < 0 = CUDA/usage error (text via gf_last_error).
 *
 * Reference interfaces each entry point replaces (file:line under
 * /root/reference/pkg/src/grainforge/):
 *   gf_upload_owners / gf_download_owners  StateStore SoA (core.py:356-390)
 *   gf_upload_geometry                     geometry slots (engine.py:444-458)
 *   gf_upload_materials                    material_pair_stack (forces.py:443-460)
 *   gf_upload_families                     family tables (engine.py:264-271, core.py:291-305)
 *   gf_detect / gf_detect_snapshot         broadphase.detect_contacts (broadphase.py:202-288)
 *   gf_bin_ranges                          _kernels.bin_ranges (_kernels.py:252-266)
 *   gf_merge_history                       broadphase.merge_history (broadphase.py:110-135)
 *   gf_adopt                               merge_history + _install_acs (broadphase.py:110-135,
 *                                          engine.py:606-665)
 *   gf_dt_step                             _step_once force/reduce/integrate chain
 *                                          (engine.py:796-843; forces.py:553-591;
 *                                          _kernels.py:516-545, 641-670)
 *   gf_set_force_model                     ForceModel registry + numba specialisation
 *                                          (forces.py:360-440, engine.py:222-232)
 *   gf_run                                 the kT/dT worker protocol of do_dynamics
 *                                          (engine.py:512-526, 669-906)
 *   gf_run_begin / gf_step_forces /        the same protocol one step at a time, split
 *   gf_step_integrate / gf_run_end         between force and integration (engine.py:796-843)
 *   gf_set_decomposition, gf_pack_*,       spatial slab decomposition (no reference
 *   gf_unpack_state, gf_add_forces         counterpart: SURVEY.md 8(e))
 */
#ifndef GF_B200_H
#define GF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gf_ctx gf_ctx;

/* flags for gf_create */
#define GF_STATE_F32 1u /* store owner velocities as float32 (throughput build) */

/* device = the dT device (state, contact arrays, force/integrate kernels).
 * kt_device < 0: kT on the same device as a second stream (one GPU);
 * kt_device >= 0: the paper's 2-GPU split
 * -- the kT stream, its scratch and events on kt_device, the detection
 * snapshot written there and the contact arrays written back over NVLink
 * peer access (enabled here; NULL if the devices cannot reach each other).
 * kt_device == device runs the split bookkeeping on one device. */
gf_ctx *gf_create(int device, int kt_device, uint32_t flags);
void gf_destroy(gf_ctx *ctx);
/* copies the last error message into buf (always NUL-terminated) */
int gf_last_error(gf_ctx *ctx, char *buf, size_t n);
/* 1 when the library and a CUDA device are usable */
int gf_device_count(void);

/* ---- scene --------------------------------------------------------------- */
int gf_set_domain(gf_ctx *ctx, const double *lo3, const double *hi3, double voxel_edge);

/* n owners; sub is (n,3) uint16, quat (n,4) float32 (w,x,y,z), velocities
 * (n,3) float64 (ang_vel in the owner frame), family (n) uint8, tpl (n)
 * uint32 index into n_tpl mass-property rows: tpl_mass (n_tpl),
 * tpl_moi (n_tpl,3). */
int gf_upload_owners(gf_ctx *ctx, int64_t n, const uint64_t *voxel, const uint16_t *sub,
                     const float *quat, const double *lin_vel, const double *ang_vel,
                     const uint8_t *family, const uint32_t *tpl, int64_t n_tpl,
                     const double *tpl_mass, const double *tpl_moi);
/* any pointer may be NULL to skip that field */
int gf_download_owners(gf_ctx *ctx, uint64_t *voxel, uint16_t *sub, float *quat,
                       double *lin_vel, double *ang_vel, uint8_t *family);
int gf_set_owner_families(gf_ctx *ctx, const uint8_t *family);
/* active boxes (engine.py:857-879, ActiveBoxPolicy): every clump owner of
 * active_family or frozen_family is re-tagged by whether its position lies
 * in any box -- boxes (n_box, 6) = centre xyz (used when anchors[b] < 0) and
 * half extents xyz; anchors[b] = owner whose position is the box centre --
 * owners frozen now lose their velocities; on the device, no state round
 * trip.  *n_changed = owners re-tagged. */
int gf_apply_active_boxes(gf_ctx *ctx, int n_box, const double *boxes, const int64_t *anchors,
                          int active_family, int frozen_family, int64_t *n_changed);
/* external loads (n,3) float64 each; both NULL clears them */
int gf_set_external_loads(gf_ctx *ctx, const double *force, const double *torque);
/* selected owners' state without a full download (trackers, engine.py:132-189):
 * idx (n) device owner indices; out (n, 23) float64 per owner = voxel (the
 * uint64 bits), sub-voxel xyz, quaternion wxyz, lin vel, ang vel (local),
 * family, contact force, contact torque (of the last reported step), 2 pad */
int gf_read_owners(gf_ctx *ctx, int64_t n, const int64_t *idx, double *out);
/* max |v| over the clump owners of non-fixed families (Inspector
 * "clump_max_absv", engine.py:198-214), a device reduction */
int gf_clump_max_absv(gf_ctx *ctx, double *out);
/* per-owner contact force/torque of the last stepped step (n,3) each */
int gf_download_accumulators(gf_ctx *ctx, double *acc_force, double *acc_torque);

/* spheres: owner (n_s) int64, params (n_s,4) float32 = offset xyz + radius,
 * material (n_s) uint8.  triangles: owner, local (n_t,9) float32, material.
 * analytics: owner, kind (2 plane / 3 cylinder), local (n_a,8) float32,
 * material.  Slots are the order given (ascending geometry id). */
int gf_upload_geometry(gf_ctx *ctx, int64_t n_s, const int64_t *sph_owner,
                       const float *sph_params, const uint8_t *sph_mat, int64_t n_t,
                       const int64_t *tri_owner, const float *tri_local, const uint8_t *tri_mat,
                       int64_t n_a, const int64_t *ana_owner, const uint8_t *ana_kind,
                       const float *ana_local, const uint8_t *ana_mat);

/* pair stack (n_rows, n_mat, n_mat) float64: E_cnt, G_cnt, CoR, mu, Crr; beta
 * (n_mat, n_mat) restitution damping computed on the host (forces.py:41-44). */
int gf_upload_materials(gf_ctx *ctx, int n_mat, int n_rows, const double *pair_stack,
                        const double *beta);

/* mask (256,256) uint8; flags (256) bit0 fixed, bit1 prescribed; lv_mask /
 * av_mask (256) bit ax set when that component is prescribed; values (256,3). */
int gf_upload_families(gf_ctx *ctx, const uint8_t *mask, const uint8_t *flags,
                       const uint8_t *lv_mask, const uint8_t *av_mask, const double *lv_val,
                       const double *av_val);

/* world geometry derived from the current state; NULL skips a field */
int gf_download_world(gf_ctx *ctx, double *sph_centers, double *tri_world, double *ana_world);

/* ---- contact arrays ------------------------------------------------------- */
/* install an ACS (canonical order) with its (n, W) float32 history */
int gf_set_acs(gf_ctx *ctx, int64_t n, const uint8_t *kind, const int64_t *slot_a,
               const int64_t *slot_b, const float *wild, int W);
int64_t gf_acs_size(gf_ctx *ctx, int which /* 0 = active, 1 = last detected */);
int gf_get_acs(gf_ctx *ctx, int which, uint8_t *kind, int64_t *slot_a, int64_t *slot_b,
               float *wild);

/* ---- kT ------------------------------------------------------------------- */
/* detect on the current state into the "next" array; returns its size */
int gf_detect(gf_ctx *ctx, double margin, int64_t *n_out);
/* detect on an explicit snapshot (broadphase.DetectionSnapshot fields);
 * grid_out = glo xyz + inv_bin, nb_out = bins per axis (may be NULL) */
int gf_detect_snapshot(gf_ctx *ctx, int64_t m, const double *centers, const float *radii,
                       const int64_t *sph_owner, const uint8_t *sph_family, int64_t n_t,
                       const double *tri_world, const int64_t *tri_owner,
                       const uint8_t *tri_family, int64_t n_a, const double *ana_world,
                       const uint8_t *ana_kind, const int64_t *ana_owner,
                       const uint8_t *ana_family, const uint8_t *mask, double margin,
                       double bin_size /* <= 0: 2 (r_max + margin) */, double *grid_out,
                       int64_t *nb_out, int64_t *n_out);
/* per-sphere inclusive bin ranges (n_s,6) int64 of the last detection's grid */
int gf_bin_ranges(gf_ctx *ctx, double margin, int64_t *out);
/* history remap between two canonical arrays of (kind, geometry a, b) given as
 * host buffers; out_wild (n_new, W) receives matched rows, zeros otherwise */
int gf_merge_history(gf_ctx *ctx, int64_t n_old, const uint8_t *old_kind, const int64_t *old_a,
                     const int64_t *old_b, const float *old_wild, int64_t n_new,
                     const uint8_t *new_kind, const int64_t *new_a, const int64_t *new_b, int W,
                     float *out_wild);
/* adopt the last detection: history remap + incidence lists */
int gf_adopt(gf_ctx *ctx);

/* ---- dT ------------------------------------------------------------------- */
typedef struct {
  double h;
  double g[3];
  double v_err;
  double sim_time;
  int64_t step;
  int32_t write_acc;
  int32_t pad;
} gf_step_params;

/* one dT step (force -> reduce -> integrate -> refresh) on the active ACS;
 * returns the touching count and the watchdog owners (-1 = ok) */
int gf_dt_step(gf_ctx *ctx, const gf_step_params *p, int64_t *touching, int64_t *bad,
               int64_t *oob);

/* ---- user force models (NVRTC) ------------------------------------------- */
/* Compile a user contact model from CUDA source (forces.py:82-87 contract):
 *   __device__ void user_core(double overlap, double ts, double sim_time,
 *       double b2ax, double b2ay, double b2az, double vx, double vy, double vz,
 *       double wrx, double wry, double wrz, double mass_eff, double ra, double rb,
 *       int mat_a, int mat_b, const double *pair, int n_mat, float *wild, double *out);
 * pair(row, a, b) = pair[(row * n_mat + a) * n_mat + b]; rows E_cnt, G_cnt,
 * then the model's pair properties.  W = wildcards per contact.  NULL source
 * restores the built-in Hertz-Mindlin model.  include_dir = the directory of
 * gf_device.cuh.  The compiler log is copied to log. */
int gf_set_force_model(gf_ctx *ctx, const char *cuda_src, const char *include_dir, int W, char *log,
                       size_t log_n);
/* bonded models (engine.py:639-662): at every adoption, a contact of the
 * active array whose wildcard `col` is > 0 (an intact bond) and that the new
 * detection no longer holds is re-appended with its history; col < 0 turns
 * it off.  Call after gf_set_force_model (col < W). */
int gf_set_persistent_wildcard(gf_ctx *ctx, int col);
/* NVRTC compile of a user model without a device (validation only) */
int gf_nvrtc_compile(const char *cuda_src, const char *include_dir, char *log, size_t log_n);

/* ---- the whole worker protocol -------------------------------------------- */
typedef struct {
  int64_t n_steps;
  int64_t step0;        /* global step index of the first step */
  double h;
  double g[3];
  double v_err;
  double margin;        /* detection margin (engine._current_margin) */
  int32_t period;       /* snapshot every `period` steps */
  int32_t lag;          /* adopt `lag` steps after the snapshot (0 = sync) */
  int32_t n_dyn;        /* dynamic prescription entries */
  int32_t write_acc;    /* store accumulators on the final step */
  const int32_t *dyn_spec;   /* (n_dyn, 3): family, table (0 lin / 1 ang), axis */
  const double *dyn_vals;    /* (n_steps, n_dyn) values at each step's start time */
} gf_run_params;

typedef struct {
  int64_t steps_done;
  int64_t bad_owner, bad_step;
  int64_t oob_owner, oob_step;
  int64_t touching;     /* last step */
  int64_t n_acs;
  int64_t ca_updates;
  int64_t sum_acs;          /* active-contact entries summed over the run's steps */
  int64_t sum_touch_pairs;  /* touching entries summed over the run's steps */
  double dt_ms, kt_ms;  /* device time of the dT and kT streams */
  double wall_ms;
  int64_t kt_rebuilds;  /* candidate-list rebuilds so far (Verlet skin exceeded) */
  int64_t dd_trip_step; /* decomposition: first step a local owner moved more than `travel`
                           along the slab axis (the run stops after it), or -1 */
} gf_run_result;

int gf_run(gf_ctx *ctx, const gf_run_params *p, gf_run_result *r);

/* gf_run one step at a time: gf_run_begin, then for i in [0, n_steps)
 * gf_step_forces(i) (kT schedule + contact forces) and gf_step_integrate(i)
 * (prescriptions + integration), then gf_run_end.  gf_run is exactly this
 * loop; the split lets a decomposed run exchange ghost forces between the
 * halves and ghost state after the second.  Everything is queued on the dT
 * stream (gf_stream) -- no host synchronisation between the calls. */
int gf_run_begin(gf_ctx *ctx, const gf_run_params *p);
int gf_step_forces(gf_ctx *ctx, int64_t i);
int gf_step_integrate(gf_ctx *ctx, int64_t i);
int gf_run_end(gf_ctx *ctx, gf_run_result *r);

/* ---- spatial decomposition (needs GF_STATE_F32) -------------
 * dd[o] = class | global_owner_id << 2 for every owner of this context:
 * class 0 local (integrated here), 1 ghost (copy of another rank's owner,
 * not integrated), 2 shared boundary owner replicated on every rank, 3 the
 * same on the one rank that also computes shared-shared contacts.  A
 * local-ghost contact is computed only by the rank owning the lower global
 * id, so every physical contact is computed exactly once across ranks.
 * lever_max = the global fixed-point torque lever (max sphere offset+radius
 * / triangle vertex distance over ALL ranks' geometry), so every rank's
 * fixed-point units agree.  axis / travel: the static ghost layer is valid
 * while every local owner stays within `travel` of its current coordinate
 * along `axis`; the first step that breaks it is reported in
 * gf_run_result.dd_trip_step and the run stops after that (complete) step, so
 * the host can repartition.  dd = NULL switches the decomposition off. */
int gf_set_decomposition(gf_ctx *ctx, const uint32_t *dd, double lever_max, int axis, double travel);
/* bytes of one packed owner-state record (64 for GF_STATE_F32) */
int gf_halo_record_bytes(gf_ctx *ctx);
/* the dT stream (a cudaStream_t) the halo calls are queued on, for a
 * transport (NCCL) to order itself against */
void *gf_stream(gf_ctx *ctx);
/* DEVICE arrays: idx = uint32 owner indices of this context; out / in =
 * n records.  pack_state gathers owner state (voxel, sub-voxel, quaternion,
 * velocities) bit for bit; unpack_state scatters it into ghosts and refreshes
 * their sphere centres; pack_forces gathers the 48-byte fixed-point force /
 * torque accumulators of ghosts and clears them; add_forces adds returned
 * accumulators into local owners (exact integer addition). */
int gf_pack_state(gf_ctx *ctx, const uint32_t *idx, int64_t n, void *out);
int gf_unpack_state(gf_ctx *ctx, const uint32_t *idx, int64_t n, const void *in);
int gf_pack_forces(gf_ctx *ctx, const uint32_t *idx, int64_t n, void *out);
int gf_add_forces(gf_ctx *ctx, const uint32_t *idx, int64_t n, const void *in);
/* the guard's trip step and a DEVICE int64 word (INT64_MAX = none): mode 0
 * writes this context's trip step into *word, mode 1 lowers it to *word.
 * A transport min-reduces the word across ranks between the two (every rank
 * then skips the same steps). */
int gf_trip_word(gf_ctx *ctx, void *word, int mode);
/* block until the context's dT stream is idle */
int gf_sync(gf_ctx *ctx);

/* ---- reference-shaped entry points (host buffers in the reference's own
 * layouts; one call = upload, one kernel pass on the context's device, download;
 * fp64 arithmetic statement by statement like numba fastmath=False) ---------- */
/* make_contact_kernel's sweep (forces.py:547-593) with the context's force
 * model (built-in Hertz-Mindlin, W = 4, or the NVRTC model of
 * gf_set_force_model): per entry k of (kind, slot_a, slot_b) the contact
 * geometry (_kernels.py:441-486), pair kinematics (forces.py:55-79) and the
 * core; wild (n, W) float32 updated in place; out_ft (n, 6) = force on A +
 * torque-only force, depth (n), cp (n, 3); *touching = 2 per touching
 * sphere-sphere entry, 1 per touching wall entry.  sph_centers (m, 3)
 * float64, sph_radii (m) float32, tri_world (n_t, 9), ana_world (n_a, 8),
 * owner_pos / lin_vel / ang_vel_global (n_o, 3) float64, mass (n_o). */
int gf_contact_forces(gf_ctx *ctx, int64_t n, const uint8_t *kind, const int64_t *slot_a,
                      const int64_t *slot_b, const int64_t *owner_a, const int64_t *owner_b,
                      const uint8_t *mat_a, const uint8_t *mat_b, int64_t n_sph,
                      const double *sph_centers, const float *sph_radii, int64_t n_tri,
                      const double *tri_world, int64_t n_ana, const double *ana_world,
                      const uint8_t *ana_kind, int64_t n_owner, const double *owner_pos,
                      const double *lin_vel, const double *ang_vel_global, const double *mass,
                      int n_mat, int n_rows, const double *pair_stack, float *wild, int W, double ts,
                      double sim_time, double *out_ft, double *depth, double *cp, int64_t *touching);
/* the model core over n contexts (forces.py:82-87 scalar contract; the
 * ForceModel.core / jit_core / evaluate surface, forces.py:360-405):
 * args (n, 15) = overlap, ts, sim_time, b2a xyz, v xyz, wr xyz, mass_eff, ra,
 * rb; mats (n, 2) int32; wild (n, W) in place; out (n, 6). */
int gf_eval_core(gf_ctx *ctx, int64_t n, const double *args, const int32_t *mats, int n_mat, int n_rows,
                 const double *pair_stack, float *wild, int W, double *out);
/* reduce_to_owners (_kernels.py:515-545): per owner, the contributions in the
 * reference loop's order (+F / r_a x (F + tof) on A, the negation at r_b on
 * B); mass != NULL adds mass * gravity3 afterwards (forces.py:600-614).
 * forces / tofs / cps (n, 3); owner_pos (n_o, 3); out (n_o, 3) each. */
int gf_reduce(gf_ctx *ctx, int64_t n, const int64_t *owner_a, const int64_t *owner_b, const double *forces,
              const double *tofs, const double *cps, int64_t n_owner, const double *owner_pos,
              const double *mass, const double *gravity3, double *acc_force, double *acc_torque);
/* integrate_and_refresh (_kernels.py:548-670): semi-implicit Euler step,
 * re-encode (voxel (n) uint64, sub (n, 3) uint16) and decode, sphere centres
 * (n_s, 3) of sph_geom through geom_params (n_geom, 9) float32 /
 * geom_owner; *bad / *oob = first speeding / out-of-domain owner or -1.
 * fixed_flag / prescribed_flag (256), lv_mask / av_mask (256, 3) uint8,
 * lv_val / av_val (256, 3) float64; ext_force / ext_torque may be NULL. */
int gf_integrate_and_refresh(gf_ctx *ctx, double h, const double *g3, int64_t n, double *owner_pos,
                             float *quat, double *lin_vel, double *ang_vel, const double *mass,
                             const double *moi, const double *acc_force, const double *acc_torque,
                             const double *ext_force, const double *ext_torque, const uint8_t *family,
                             const uint8_t *fixed_flag, const uint8_t *lv_mask, const double *lv_val,
                             const uint8_t *av_mask, const double *av_val, const uint8_t *prescribed_flag,
                             double v_err, const double *lo3, const double *hi3, double edge,
                             uint64_t *voxel, uint16_t *sub, int64_t n_s, const int64_t *sph_geom,
                             int64_t n_geom, const float *geom_params, const int64_t *geom_owner,
                             double *sph_centers, int64_t *bad, int64_t *oob);

/* an output frame's per-sphere columns in one pass on the device
 * (io.write_sphere_csv, io.py:132-166): out (n_s, 8) float64 per device
 * sphere slot = centre xyz, |v| of its owner, owner family, owner v xyz */
int gf_sphere_frame(gf_ctx *ctx, double *out);

/* per-kernel device timing of subsequent gf_run calls (CUDA events on the dT
 * stream); out6 = cumulative ms of {contact phase, k_heavy, k_integrate, kT},
 * the number of profiled steps, then the ms of the fused sphere-sphere kernel
 * (k_contacts_ss) inside the contact phase.  Enabling resets the counters. */
int gf_set_profiling(gf_ctx *ctx, int on);
int gf_kernel_times(gf_ctx *ctx, double *out6);

#ifdef __cplusplus
}
#endif
#endif /* GF_B200_H */
