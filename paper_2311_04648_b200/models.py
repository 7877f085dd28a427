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


# ---------------------------------------------------------------------------
# breakage -- the reference's bonded-particle model (forces.py:185-291,
# BREAKAGE_MODEL :433-440): a bonded elastoplastic contact with tensile and
# shear failure and capped bending resistance; broken contacts fall back to
# Hertz-Mindlin under compression.  Pair rows: 0 E_eq, 1 G_cnt, 2 CoR, 3 mu,
# 4 Crr, 5 nu, 6 tension, 7 cohesion.  Wildcards: 0..2 delta_tan, 3
# delta_time, 4 unbroken, 5 initialLength.  Statement order of the
# reference's core; beta from the device log (one-ulp caveat as in
# gf::hm_default_core).
# ---------------------------------------------------------------------------

BREAKAGE_SRC = r"""
__device__ void user_core(double overlap, double ts, double sim_time,
                          double b2ax, double b2ay, double b2az,
                          double vx, double vy, double vz,
                          double wrx, double wry, double wrz,
                          double mass_eff, double ra, double rb,
                          int mat_a, int mat_b, const double *pair, int n_mat,
                          float *wild, double *out) {
  double unbroken = double(wild[4]);
  if (unbroken <= 1e-12) {
    gf::hm_default_core(overlap, ts, sim_time, b2ax, b2ay, b2az, vx, vy, vz, wrx, wry, wrz,
                        mass_eff, ra, rb, mat_a, mat_b, pair, n_mat, wild, out);
    return;
  }
  out[0] = 0.0; out[1] = 0.0; out[2] = 0.0; out[3] = 0.0; out[4] = 0.0; out[5] = 0.0;
  const int mm = n_mat * n_mat, ab = mat_a * n_mat + mat_b;
  const double e_eq = pair[ab];
  const double cor = pair[2 * mm + ab];
  const double mu = pair[3 * mm + ab];
  const double nu_cnt = pair[5 * mm + ab];
  const double tension = pair[6 * mm + ab];
  const double cohesion = pair[7 * mm + ab];
  double projection = vx * b2ax + vy * b2ay + vz * b2az;
  double vtx = vx - projection * b2ax;
  double vty = vy - projection * b2ay;
  double vtz = vz - projection * b2az;
  double dtx = double(wild[0]) + ts * vtx;
  double dty = double(wild[1]) + ts * vty;
  double dtz = double(wild[2]) + ts * vtz;
  double disp_proj = dtx * b2ax + dty * b2ay + dtz * b2az;
  dtx -= disp_proj * b2ax;
  dty -= disp_proj * b2ay;
  dtz -= disp_proj * b2az;
  wild[3] = float(double(wild[3]) + ts);
  const double delta_d = overlap - double(wild[5]);
  const double kn = e_eq * (ra * rb) / (ra + rb);
  const double rmax = ra > rb ? ra : rb;
  const double area = rmax * rmax * gf::kPi;
  const double breaking_force = tension * area;
  const double delta_y = breaking_force / kn;
  const double delta_u = 3.0 * delta_y;
  double fmag;
  if (delta_d > delta_y) fmag = kn * delta_d;
  else fmag = ((delta_u - delta_d) - delta_y) * kn * 0.5;
  const double damping = 0.01 * sqrt(mass_eff * kn);
  out[0] = b2ax * fmag - damping * vx;
  out[1] = b2ay * fmag - damping * vy;
  out[2] = b2az * fmag - damping * vz;
  if (delta_d < delta_u) unbroken = -1.0;
  const double kt = nu_cnt * kn;
  const double norm_mag = sqrt(out[0] * out[0] + out[1] * out[1] + out[2] * out[2]);
  double fs_max;
  if (delta_d > delta_y) fs_max = norm_mag * mu + cohesion * area;
  else fs_max = norm_mag * mu;
  const double loge = cor < 1e-12 ? log(1e-12) : log(cor);
  const double beta = loge / sqrt(loge * loge + gf::kPi * gf::kPi);
  const double gt = -2.0 * sqrt(5.0 / 6.0) * beta * sqrt(mass_eff * kt);
  const double tfx = -kt * dtx - gt * vtx;
  const double tfy = -kt * dty - gt * vty;
  const double tfz = -kt * dtz - gt * vtz;
  out[0] += tfx;
  out[1] += tfy;
  out[2] += tfz;
  if (sqrt(tfx * tfx + tfy * tfy + tfz * tfz) > fs_max) unbroken = -1.0;
  const double v_rot_mag = sqrt(wrx * wrx + wry * wry + wrz * wrz);
  if (v_rot_mag > 1e-12) {
    const double kr = ra * rb * kt;
    const double eta = 0.1;
    const double var_1 = ts * kr / ra;
    const double fmag2 = sqrt(out[0] * out[0] + out[1] * out[1] + out[2] * out[2]);
    const double var_2 = eta * fmag2;
    const double torque_mag = var_1 < var_2 ? var_1 : var_2;
    const double scale = torque_mag / v_rot_mag;
    out[3] = wrx * scale;
    out[4] = wry * scale;
    out[5] = wrz * scale;
  }
  wild[0] = float(dtx);
  wild[1] = float(dty);
  wild[2] = float(dtz);
  wild[4] = float(unbroken);
}
"""

BREAKAGE_WILDCARDS = ("delta_tan_x", "delta_tan_y", "delta_tan_z", "delta_time", "unbroken", "initialLength")
BREAKAGE_PROPS = ("CoR", "mu", "Crr", "nu", "tension", "cohesion")


def breakage_model() -> ForceModel:
    """Register (once) and return the bonded breakage model."""
    try:
        return get_force_model("breakage")
    except Exception:
        return register_force_model(ForceModel(
            "breakage", None, None, BREAKAGE_WILDCARDS, BREAKAGE_PROPS, cuda_src=BREAKAGE_SRC,
            flip_on_swap=(0, 1, 2)))
