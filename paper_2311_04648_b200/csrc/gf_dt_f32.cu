// fp32-velocity (throughput) build of the dT kernels: owner velocities are
// stored as float32 (the paper's compact layout); force
// arithmetic stays fp64 scratch and FMA contraction is allowed.
#include "gf_dt_impl.cuh"
namespace gf {
int dt_step_f32(Ctx *c, const StepArgs &a, cudaStream_t s) { return dt_step_impl<float>(c, a, s); }
int dt_forces_f32(Ctx *c, const StepArgs &a, cudaStream_t s) { return dt_forces_impl<float>(c, a, s); }
int dt_integrate_f32(Ctx *c, const StepArgs &a, cudaStream_t s) { return dt_integrate_impl<float>(c, a, s); }
}  // namespace gf
