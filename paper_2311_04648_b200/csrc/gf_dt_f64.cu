// fp64-velocity (parity) build of the dT kernels; compiled with -fmad=false so
// every fp64 operation rounds like the reference (numba fastmath=False).
#include "gf_dt_impl.cuh"
namespace gf {
int dt_step_f64(Ctx *c, const StepArgs &a, cudaStream_t s) { return dt_step_impl<double>(c, a, s); }
int dt_forces_f64(Ctx *c, const StepArgs &a, cudaStream_t s) { return dt_forces_impl<double>(c, a, s); }
int dt_integrate_f64(Ctx *c, const StepArgs &a, cudaStream_t s) { return dt_integrate_impl<double>(c, a, s); }
}  // namespace gf

namespace gf {
int refresh_centers(Ctx *c, cudaStream_t s) {
  if (!c->n_sph) return 0;
  k_centers<<<unsigned((c->n_sph + 127) / 128), 128, 0, s>>>(c->dom, owners_view(c), spheres_view(c));
  GF_CHECK(c, cudaGetLastError());
  return 0;
}

int refresh_world(Ctx *c, cudaStream_t s) {
  int64_t n = c->n_tri + c->n_ana;
  if (!n) return 0;
  c->world_version++;
  k_world<<<unsigned((n + 127) / 128), 128, 0, s>>>(c->dom, owners_view(c), tris_view(c), anas_view(c));
  GF_CHECK(c, cudaGetLastError());
  return 0;
}
}  // namespace gf
