"""User force models shipped as CUDA source (compiled with NVRTC at
Simulator.initialize, the paper's JIT models).

hertz_mindlin_cohesive -- BASELINE.json configs[3] ("custom user-defined force
model, cohesive contact via NVRTC"): the default Hertz-Mindlin law
(forces.py:82-182) plus a cohesive pull proportional to the Hertzian contact
area, F_c = coh * pi * R_eff * overlap, acting along -B2A on touching
contacts.  Pair property ``coh`` (Pa) mixes as min(A, B) like every pair
property (core.py:122-127).
"""

from .forces import ForceModel, get_force_model, register_force_model

COHESIVE_SRC = r"""
__device__ void user_core(double overlap, double ts, double sim_time,
                          double b2ax, double b2ay, double b2az,
                          double vx, double vy, double vz,
                          double wrx, double wry, double wrz,
                          double mass_eff, double ra, double rb,
                          int mat_a, int mat_b, const double *pair, int n_mat,
                          float *wild, double *out) {
  gf::hm_default_core(overlap, ts, sim_time, b2ax, b2ay, b2az, vx, vy, vz, wrx, wry, wrz,
                      mass_eff, ra, rb, mat_a, mat_b, pair, n_mat, wild, out);
  if (overlap > 0.0) {
    const double coh = pair[(5 * n_mat + mat_a) * n_mat + mat_b];
    const double r_eff = ra * rb / (ra + rb);
    const double f = coh * 3.141592653589793 * r_eff * overlap;
    out[0] -= f * b2ax;
    out[1] -= f * b2ay;
    out[2] -= f * b2az;
  }
}
"""


def cohesive_model() -> ForceModel:
    """Register (once) and return the cohesive Hertz-Mindlin user model."""
    try:
        return get_force_model("hertz_mindlin_cohesive")
    except Exception:
        return register_force_model(ForceModel(
            name="hertz_mindlin_cohesive",
            wildcards=("delta_tan_x", "delta_tan_y", "delta_tan_z", "delta_time"),
            pair_props=("CoR", "mu", "Crr", "coh"),
            device_kernel="nvrtc", cuda_src=COHESIVE_SRC, flip_on_swap=(0, 1, 2)))
