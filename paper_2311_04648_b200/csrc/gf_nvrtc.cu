// gf_nvrtc.cu -- user contact force models compiled from CUDA source at run
// time (the paper's Jitify/NVRTC models; the reference's
// ForceModel plugin contract, forces.py:82-87 and :360-440).
//
// The user supplies a device function with the reference core's argument
// list (overlap, ts, sim_time, B-to-A normal, relative velocity, rolling
// direction, effective mass, radii, material ids, pair stack, wildcard row,
// out[6]).  It is compiled for sm_100a together with gf_device.cuh into a
// force kernel that runs over every ACS entry (a user model may act at
// negative overlap, e.g. cohesion); everything else in the step is the
// ahead-of-time code.  Modules are cached per source text.
#include <nvrtc.h>

#include <map>
#include <string>
#include <vector>

#include "gf_context.h"
#include "gf_device.cuh"

namespace gf {

namespace {
// loaded through the runtime's library API (no libcuda link dependency)
struct UserModule {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t f64 = nullptr, f32 = nullptr, ss = nullptr, walls = nullptr, ref = nullptr, batch = nullptr;
};
std::map<std::string, UserModule> g_cache;

const char *kWrapper = R"(
#include "gf_device.cuh"
namespace gf_user {
using namespace gf;
)";
const char *kWrapperTail = R"(
}  // namespace gf_user
struct GfUserCore {
  static constexpr bool kAllEntries = true;
  __device__ static __forceinline__ void eval(const gf::CoreArgs &a, double out[6]) {
    gf_user::user_core(a.overlap, a.ts, a.sim_time, a.b2ax, a.b2ay, a.b2az, a.vx, a.vy, a.vz, a.wrx,
                       a.wry, a.wrz, a.mass_eff, a.ra, a.rb, a.mat_a, a.mat_b, a.pair, a.n_mat, a.wild,
                       out);
  }
};
extern "C" __global__ void __launch_bounds__(128) gf_user_forces_f64(gf::DtView v, double ts, double t) {
  gf::forces_loop<double, GfUserCore>(v, ts, t, nullptr, nullptr);
}
extern "C" __global__ void __launch_bounds__(128) gf_user_forces_f32(gf::DtView v, double ts, double t) {
  gf::forces_loop<float, GfUserCore>(v, ts, t, nullptr, nullptr);
}
// throughput build: the fused sphere-sphere loop + the wall kinds
extern "C" __global__ void __launch_bounds__(256) gf_user_contacts_ss(gf::DtView v, double ts, double t) {
  gf::user_ss_loop<GfUserCore>(v, ts, t);
}
extern "C" __global__ void __launch_bounds__(128) gf_user_walls_f32(gf::DtView v, double ts, double t) {
  gf::user_walls_loop<float, GfUserCore>(v, ts, t);
}
// the reference-shaped entry points (gf_contact_forces, gf_eval_core)
extern "C" __global__ void __launch_bounds__(128) gf_user_ref_contacts(gf::RefContacts r) {
  gf::ref_contacts_loop<GfUserCore>(r);
}
extern "C" __global__ void __launch_bounds__(128) gf_user_core_batch(gf::CoreBatch b) {
  gf::core_batch_loop<GfUserCore>(b);
}
)";
}  // namespace

int set_user_model(Ctx *c, const char *src, const char *include_dir, std::string &log) {
  if (!src) {
    c->user_model = false;
    return 0;
  }
  std::string key = std::string(src) + "|" + include_dir;
  auto it = g_cache.find(key);
  if (it == g_cache.end()) {
    std::string full = std::string(kWrapper) + src + kWrapperTail;
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, full.c_str(), "gf_user_model.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
      set_err(c, "nvrtcCreateProgram failed");
      return -1;
    }
    std::string inc = std::string("--include-path=") + include_dir;
    // --fmad=false: user cores round like the reference's numba cores (fastmath=False)
    const char *opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--device-as-default-execution-space",
                          inc.c_str(), "-lineinfo", "--fmad=false"};
    nvrtcResult rc = nvrtcCompileProgram(prog, 6, opts);
    size_t ln = 0;
    nvrtcGetProgramLogSize(prog, &ln);
    std::string plog(ln, '\0');
    if (ln) nvrtcGetProgramLog(prog, &plog[0]);
    log = plog;
    if (rc != NVRTC_SUCCESS) {
      set_err(c, std::string("NVRTC compile of the user force model failed:\n") + plog);
      nvrtcDestroyProgram(&prog);
      return -1;
    }
    size_t nbin = 0;
    nvrtcGetCUBINSize(prog, &nbin);
    std::vector<char> cubin(nbin);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    UserModule um;
    if (cudaLibraryLoadData(&um.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
        cudaLibraryGetKernel(&um.f64, um.lib, "gf_user_forces_f64") != cudaSuccess ||
        cudaLibraryGetKernel(&um.f32, um.lib, "gf_user_forces_f32") != cudaSuccess ||
        cudaLibraryGetKernel(&um.ss, um.lib, "gf_user_contacts_ss") != cudaSuccess ||
        cudaLibraryGetKernel(&um.walls, um.lib, "gf_user_walls_f32") != cudaSuccess ||
        cudaLibraryGetKernel(&um.ref, um.lib, "gf_user_ref_contacts") != cudaSuccess ||
        cudaLibraryGetKernel(&um.batch, um.lib, "gf_user_core_batch") != cudaSuccess) {
      set_err(c, std::string("loading the NVRTC user force module failed: ") +
                     cudaGetErrorString(cudaGetLastError()));
      return -1;
    }
    it = g_cache.emplace(key, um).first;
  }
  c->user_fn_f64 = reinterpret_cast<void *>(it->second.f64);
  c->user_fn_f32 = reinterpret_cast<void *>(it->second.f32);
  c->user_fn_ss = reinterpret_cast<void *>(it->second.ss);
  c->user_fn_walls = reinterpret_cast<void *>(it->second.walls);
  c->user_fn_ref = reinterpret_cast<void *>(it->second.ref);
  c->user_fn_batch = reinterpret_cast<void *>(it->second.batch);
  c->user_model = true;
  return 0;
}

// compile only (no device needed): validates a user model source
int nvrtc_compile_check(const char *src, const char *include_dir, std::string &log) {
  std::string full = std::string(kWrapper) + src + kWrapperTail;
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, full.c_str(), "gf_user_model.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    log = "nvrtcCreateProgram failed";
    return -1;
  }
  std::string inc = std::string("--include-path=") + include_dir;
  const char *opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--device-as-default-execution-space",
                        inc.c_str()};
  nvrtcResult rc = nvrtcCompileProgram(prog, 4, opts);
  size_t ln = 0;
  nvrtcGetProgramLogSize(prog, &ln);
  log.assign(ln, '\0');
  if (ln) nvrtcGetProgramLog(prog, &log[0]);
  nvrtcDestroyProgram(&prog);
  return rc == NVRTC_SUCCESS ? 0 : -1;
}

int launch_user_forces(Ctx *c, const DtView &v, double ts, double sim_time, cudaStream_t s) {
  DtView vv = v;
  void *args[] = {&vv, &ts, &sim_time};
  if (c->f32_state && v.sph.kin && c->user_fn_ss) {
    // throughput build: the fused sphere-sphere loop, then the wall kinds
    cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void *>(c->user_fn_ss), dim3(unsigned(c->n_sm) * 4), dim3(256), args,
                                     0, s);
    if (e == cudaSuccess)
      e = cudaLaunchKernel(reinterpret_cast<const void *>(c->user_fn_walls), dim3(unsigned(c->n_sm) * 4), dim3(128), args, 0, s);
    if (e != cudaSuccess) {
      set_err(c, std::string("launching the NVRTC user force kernels failed: ") + cudaGetErrorString(e));
      return -1;
    }
    return 0;
  }
  cudaKernel_t fn = reinterpret_cast<cudaKernel_t>(c->f32_state ? c->user_fn_f32 : c->user_fn_f64);
  unsigned grid = unsigned(std::min<int64_t>((v.n_acs + 127) / 128, int64_t(c->n_sm) * 16));
  if (grid == 0) grid = 1;
  cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void *>(fn), dim3(grid), dim3(128), args, 0, s);
  if (e != cudaSuccess) {
    set_err(c, std::string("launching the NVRTC user force kernel failed: ") + cudaGetErrorString(e));
    return -1;
  }
  return 0;
}

}  // namespace gf
