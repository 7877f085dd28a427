/*
 * gf_oracle.c -- CPU restatement of the grainforge DEM step (TEST INFRASTRUCTURE).
 *
 * This file is the parity oracle for the B200 build.  It restates, in plain
 * C, the arithmetic of the reference's numba kernels so that tests/, the
 * smoke() check and bench.py's cpu_baseline / --impl reference legs can
 * compare the CUDA path against it.  It is NEVER linked into, loaded by, or
 * called from the product path (paper_2311_04648_b200/).
 *
 * Numerics contract: the reference compiles its kernels with numba
 * `fastmath=False` (/root/reference/pkg/src/grainforge/_kernels.py:17,
 * forces.py:26), i.e. strict IEEE-754 binary64 with every operation rounded
 * separately (no FMA contraction; measured in SURVEY.md Appendix B).  This
 * file is compiled with -ffp-contract=off -fno-fast-math and keeps the
 * reference's operation order statement by statement, so its results are
 * bit-identical to the reference (pinned by tests/test_oracle_golden.py
 * against fixtures produced by the reference itself, tests/golden/).
 *
 * Array conventions follow the numpy layouts of the reference: row-major,
 * int64 indices, float32 radii / quaternions / geometry parameters / history,
 * float64 state and scratch.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define VOX_BITS 21
#define VOX_PER_AXIS (1LL << VOX_BITS)
#define SUB_PER_EDGE 65536
#define FLAT_RADIUS 1.0e18
#define GEOM_PLANE 2
#define PI_D 3.141592653589793

/* ------------------------------------------------------------------------ */
/* compressed coordinates: _kernels.py:32-67                                 */
/* ------------------------------------------------------------------------ */

/* Returns the first owner outside [lo, hi] (stops there, like the
 * reference's early return at _kernels.py:40-41) or -1. */
int64_t orc_encode_positions(int64_t n, const double *pos, const double *lo,
                             const double *hi, double edge, uint64_t *voxel,
                             uint16_t *sub) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t packed = 0;
    for (int ax = 0; ax < 3; ++ax) {
      double p = pos[3 * i + ax];
      if (p < lo[ax] || p > hi[ax]) return i;
      double t = (p - lo[ax]) / edge;
      int64_t cell = (int64_t)t;
      if (cell >= VOX_PER_AXIS) cell = VOX_PER_AXIS - 1;
      int64_t s = (int64_t)((t - (double)cell) * (double)SUB_PER_EDGE);
      if (s >= SUB_PER_EDGE) s = SUB_PER_EDGE - 1;
      packed |= ((uint64_t)cell) << (VOX_BITS * ax);
      sub[3 * i + ax] = (uint16_t)s;
    }
    voxel[i] = packed;
  }
  return -1;
}

void orc_decode_positions(int64_t n, const uint64_t *voxel, const uint16_t *sub,
                          const double *lo, double edge, double *out) {
  const uint64_t mask = (uint64_t)(VOX_PER_AXIS - 1);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t v = voxel[i];
    for (int ax = 0; ax < 3; ++ax) {
      double cell = (double)((v >> (VOX_BITS * ax)) & mask);
      double frac = (double)sub[3 * i + ax] / (double)SUB_PER_EDGE;
      out[3 * i + ax] = lo[ax] + (cell + frac) * edge;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* rigid transforms: _kernels.py:74-152                                      */
/* ------------------------------------------------------------------------ */

/* r = v + 2 u x (u x v + w v), same term order as _kernels.py:77-83 */
static inline void qrot(double qw, double qx, double qy, double qz, double vx,
                        double vy, double vz, double *rx, double *ry,
                        double *rz) {
  double tx = qy * vz - qz * vy + qw * vx;
  double ty = qz * vx - qx * vz + qw * vy;
  double tz = qx * vy - qy * vx + qw * vz;
  *rx = vx + 2.0 * (qy * tz - qz * ty);
  *ry = vy + 2.0 * (qz * tx - qx * tz);
  *rz = vz + 2.0 * (qx * ty - qy * tx);
}

void orc_sphere_world(int64_t n_s, const int64_t *sph_geom,
                      const float *geom_params, const int64_t *geom_owner,
                      const double *owner_pos, const float *quat,
                      double *out_center, float *out_radius) {
  for (int64_t k = 0; k < n_s; ++k) {
    int64_t g = sph_geom[k], o = geom_owner[g];
    const float *p = geom_params + 9 * g;
    const float *q = quat + 4 * o;
    double rx, ry, rz;
    qrot((double)q[0], (double)q[1], (double)q[2], (double)q[3], (double)p[0],
         (double)p[1], (double)p[2], &rx, &ry, &rz);
    out_center[3 * k + 0] = owner_pos[3 * o + 0] + rx;
    out_center[3 * k + 1] = owner_pos[3 * o + 1] + ry;
    out_center[3 * k + 2] = owner_pos[3 * o + 2] + rz;
    if (out_radius) out_radius[k] = p[3];
  }
}

void orc_triangle_world(int64_t n_t, const int64_t *tri_geom,
                        const float *geom_params, const int64_t *geom_owner,
                        const double *owner_pos, const float *quat,
                        double *out) {
  for (int64_t k = 0; k < n_t; ++k) {
    int64_t g = tri_geom[k], o = geom_owner[g];
    const float *q = quat + 4 * o;
    for (int v = 0; v < 3; ++v) {
      const float *l = geom_params + 9 * g + 3 * v;
      double rx, ry, rz;
      qrot((double)q[0], (double)q[1], (double)q[2], (double)q[3],
           (double)l[0], (double)l[1], (double)l[2], &rx, &ry, &rz);
      out[9 * k + 3 * v + 0] = owner_pos[3 * o + 0] + rx;
      out[9 * k + 3 * v + 1] = owner_pos[3 * o + 1] + ry;
      out[9 * k + 3 * v + 2] = owner_pos[3 * o + 2] + rz;
    }
  }
}

void orc_analytic_world(int64_t n_a, const int64_t *ana_geom,
                        const float *geom_params, const int64_t *geom_owner,
                        const double *owner_pos, const float *quat,
                        double *out) {
  for (int64_t k = 0; k < n_a; ++k) {
    int64_t g = ana_geom[k], o = geom_owner[g];
    const float *q = quat + 4 * o;
    const float *p = geom_params + 9 * g;
    double px, py, pz, dx, dy, dz;
    qrot((double)q[0], (double)q[1], (double)q[2], (double)q[3], (double)p[0],
         (double)p[1], (double)p[2], &px, &py, &pz);
    out[8 * k + 0] = owner_pos[3 * o + 0] + px;
    out[8 * k + 1] = owner_pos[3 * o + 1] + py;
    out[8 * k + 2] = owner_pos[3 * o + 2] + pz;
    qrot((double)q[0], (double)q[1], (double)q[2], (double)q[3], (double)p[3],
         (double)p[4], (double)p[5], &dx, &dy, &dz);
    out[8 * k + 3] = dx;
    out[8 * k + 4] = dy;
    out[8 * k + 5] = dz;
    out[8 * k + 6] = (double)p[6];
    out[8 * k + 7] = (double)p[7];
  }
}

void orc_angular_velocity_global(int64_t n, const float *quat,
                                 const double *w_local, double *out) {
  for (int64_t i = 0; i < n; ++i) {
    const float *q = quat + 4 * i;
    qrot((double)q[0], (double)q[1], (double)q[2], (double)q[3],
         w_local[3 * i], w_local[3 * i + 1], w_local[3 * i + 2], &out[3 * i],
         &out[3 * i + 1], &out[3 * i + 2]);
  }
}

/* ------------------------------------------------------------------------ */
/* narrow-phase primitives: _kernels.py:159-231                              */
/* ------------------------------------------------------------------------ */

/* Ericson RTCD 5.1.5 region walk; branch order as _kernels.py:160-194. */
static void closest_on_tri(double px, double py, double pz, const double *t,
                           double *qx, double *qy, double *qz) {
  double ax = t[0], ay = t[1], az = t[2], bx = t[3], by = t[4], bz = t[5];
  double cx = t[6], cy = t[7], cz = t[8];
  double abx = bx - ax, aby = by - ay, abz = bz - az;
  double acx = cx - ax, acy = cy - ay, acz = cz - az;
  double apx = px - ax, apy = py - ay, apz = pz - az;
  double d1 = abx * apx + aby * apy + abz * apz;
  double d2 = acx * apx + acy * apy + acz * apz;
  if (d1 <= 0.0 && d2 <= 0.0) { *qx = ax; *qy = ay; *qz = az; return; }
  double bpx = px - bx, bpy = py - by, bpz = pz - bz;
  double d3 = abx * bpx + aby * bpy + abz * bpz;
  double d4 = acx * bpx + acy * bpy + acz * bpz;
  if (d3 >= 0.0 && d4 <= d3) { *qx = bx; *qy = by; *qz = bz; return; }
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    double s = d1 / (d1 - d3);
    *qx = ax + s * abx; *qy = ay + s * aby; *qz = az + s * abz; return;
  }
  double cpx = px - cx, cpy = py - cy, cpz = pz - cz;
  double d5 = abx * cpx + aby * cpy + abz * cpz;
  double d6 = acx * cpx + acy * cpy + acz * cpz;
  if (d6 >= 0.0 && d5 <= d6) { *qx = cx; *qy = cy; *qz = cz; return; }
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double s = d2 / (d2 - d6);
    *qx = ax + s * acx; *qy = ay + s * acy; *qz = az + s * acz; return;
  }
  double va = d3 * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
    double s = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    *qx = bx + s * (cx - bx); *qy = by + s * (cy - by); *qz = bz + s * (cz - bz);
    return;
  }
  double denom = 1.0 / (va + vb + vc);
  double v = vb * denom, w = vc * denom;
  *qx = ax + abx * v + acx * w;
  *qy = ay + aby * v + acy * w;
  *qz = az + abz * v + acz * w;
}

void orc_closest_point_on_triangle(const double *p, const double *tri,
                                   double *out4) {
  double qx, qy, qz;
  closest_on_tri(p[0], p[1], p[2], tri, &qx, &qy, &qz);
  double dx = p[0] - qx, dy = p[1] - qy, dz = p[2] - qz;
  out4[0] = qx; out4[1] = qy; out4[2] = qz;
  out4[3] = sqrt(dx * dx + dy * dy + dz * dz);
}

/* plane: signed distance along n; cylinder: radial gap with facing sign. */
static void analytic_gap(int kind, const double *prm, double cx, double cy,
                         double cz, double *gap, double *bx, double *by,
                         double *bz, double *rb) {
  if (kind == GEOM_PLANE) {
    double nx = prm[3], ny = prm[4], nz = prm[5];
    *gap = (cx - prm[0]) * nx + (cy - prm[1]) * ny + (cz - prm[2]) * nz;
    *bx = nx; *by = ny; *bz = nz; *rb = FLAT_RADIUS;
    return;
  }
  double ax = prm[3], ay = prm[4], az = prm[5];
  double wx = cx - prm[0], wy = cy - prm[1], wz = cz - prm[2];
  double axial = wx * ax + wy * ay + wz * az;
  double rx = wx - axial * ax, ry = wy - axial * ay, rz = wz - axial * az;
  double rho = sqrt(rx * rx + ry * ry + rz * rz);
  double radius = prm[6], facing = prm[7];
  if (rho < 1e-300) { *gap = radius; *bx = 0.0; *by = 0.0; *bz = 0.0; *rb = radius; return; }
  double inv = 1.0 / rho;
  if (facing > 0.0) {
    *gap = rho - radius; *bx = rx * inv; *by = ry * inv; *bz = rz * inv; *rb = radius;
  } else {
    *gap = radius - rho; *bx = -rx * inv; *by = -ry * inv; *bz = -rz * inv; *rb = -radius;
  }
}

/* ------------------------------------------------------------------------ */
/* uniform grid broad phase: _kernels.py:238-435, broadphase.py:160-288      */
/* ------------------------------------------------------------------------ */

static inline int64_t bin_of(double x, double y, double z, const double *glo,
                             double inv_bin, const int64_t *nb) {
  int64_t ix = (int64_t)((x - glo[0]) * inv_bin);
  int64_t iy = (int64_t)((y - glo[1]) * inv_bin);
  int64_t iz = (int64_t)((z - glo[2]) * inv_bin);
  if (ix < 0) ix = 0;
  if (iy < 0) iy = 0;
  if (iz < 0) iz = 0;
  if (ix >= nb[0]) ix = nb[0] - 1;
  if (iy >= nb[1]) iy = nb[1] - 1;
  if (iz >= nb[2]) iz = nb[2] - 1;
  return (iz * nb[1] + iy) * nb[0] + ix;
}

void orc_bin_ranges(int64_t n, const double *centers, const float *radii,
                    double margin, const double *glo, double inv_bin,
                    const int64_t *nb, int64_t *out) {
  for (int64_t i = 0; i < n; ++i) {
    double r = (double)radii[i] + margin;
    for (int ax = 0; ax < 3; ++ax) {
      int64_t lo = (int64_t)((centers[3 * i + ax] - r - glo[ax]) * inv_bin);
      int64_t hi = (int64_t)((centers[3 * i + ax] + r - glo[ax]) * inv_bin);
      if (lo < 0) lo = 0;
      if (hi < 0) hi = 0;
      if (lo >= nb[ax]) lo = nb[ax] - 1;
      if (hi >= nb[ax]) hi = nb[ax] - 1;
      out[6 * i + 2 * ax] = lo;
      out[6 * i + 2 * ax + 1] = hi;
    }
  }
}

void orc_tri_bin_ranges(int64_t m, const double *tri, double margin,
                        const double *glo, double inv_bin, const int64_t *nb,
                        int64_t *out) {
  for (int64_t t = 0; t < m; ++t) {
    for (int ax = 0; ax < 3; ++ax) {
      double lo = tri[9 * t + ax], hi = tri[9 * t + ax];
      for (int v = 1; v < 3; ++v) {
        double val = tri[9 * t + 3 * v + ax];
        if (val < lo) lo = val;
        if (val > hi) hi = val;
      }
      int64_t l = (int64_t)((lo - margin - glo[ax]) * inv_bin);
      int64_t h = (int64_t)((hi + margin - glo[ax]) * inv_bin);
      if (l < 0) l = 0;
      if (h < 0) h = 0;
      if (l >= nb[ax]) l = nb[ax] - 1;
      if (h >= nb[ax]) h = nb[ax] - 1;
      out[6 * t + 2 * ax] = l;
      out[6 * t + 2 * ax + 1] = h;
    }
  }
}

/* _grid_for (broadphase.py:160-186).  pts: centers then triangle vertices.
 * Returns 0 when there is nothing to bin. */
int orc_grid_for(int64_t n_pts, const double *pts, double r_max, double margin,
                 double *glo, double *inv_bin, int64_t *nb) {
  if (n_pts == 0) return 0;
  double bin_size = 2.0 * (r_max + margin);
  if (bin_size <= 0.0) bin_size = 1.0;
  double mn[3], mx[3];
  for (int ax = 0; ax < 3; ++ax) { mn[ax] = pts[ax]; mx[ax] = pts[ax]; }
  for (int64_t i = 1; i < n_pts; ++i)
    for (int ax = 0; ax < 3; ++ax) {
      double v = pts[3 * i + ax];
      if (v < mn[ax]) mn[ax] = v;
      if (v > mx[ax]) mx[ax] = v;
    }
  double ext[3];
  for (int ax = 0; ax < 3; ++ax) {
    glo[ax] = mn[ax] - (r_max + margin) - 1e-9;
    double ghi = mx[ax] + (r_max + margin) + 1e-9;
    ext[ax] = ghi - glo[ax];
  }
  for (;;) {
    for (int ax = 0; ax < 3; ++ax) {
      double c = ceil(ext[ax] / bin_size);
      nb[ax] = c < 1.0 ? 1 : (int64_t)c;
    }
    if (nb[0] * nb[1] * nb[2] <= (1LL << 22)) break;
    bin_size *= 1.5;
  }
  *inv_bin = 1.0 / bin_size;
  return 1;
}

/* two-pass CSR of every (element, bin) registration; element order within a
 * bin is ascending (_kernels.py:269-283 + broadphase.py:189-199). */
static void csr_bins(int64_t n, const int64_t *ranges, const int64_t *nb,
                     int64_t **starts_out, int64_t **entries_out) {
  int64_t nbins = nb[0] * nb[1] * nb[2];
  int64_t *counts = (int64_t *)calloc((size_t)nbins, sizeof(int64_t));
  int64_t *starts = (int64_t *)calloc((size_t)nbins + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t iz = ranges[6 * i + 4]; iz <= ranges[6 * i + 5]; ++iz)
      for (int64_t iy = ranges[6 * i + 2]; iy <= ranges[6 * i + 3]; ++iy)
        for (int64_t ix = ranges[6 * i + 0]; ix <= ranges[6 * i + 1]; ++ix)
          counts[(iz * nb[1] + iy) * nb[0] + ix]++;
  for (int64_t b = 0; b < nbins; ++b) starts[b + 1] = starts[b] + counts[b];
  int64_t *entries = (int64_t *)malloc(sizeof(int64_t) * (size_t)(starts[nbins] + 1));
  memset(counts, 0, sizeof(int64_t) * (size_t)nbins);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t iz = ranges[6 * i + 4]; iz <= ranges[6 * i + 5]; ++iz)
      for (int64_t iy = ranges[6 * i + 2]; iy <= ranges[6 * i + 3]; ++iy)
        for (int64_t ix = ranges[6 * i + 0]; ix <= ranges[6 * i + 1]; ++ix) {
          int64_t b = (iz * nb[1] + iy) * nb[0] + ix;
          entries[starts[b] + counts[b]++] = i;
        }
  free(counts);
  *starts_out = starts;
  *entries_out = entries;
}

typedef struct {
  int64_t n, cap;
  int64_t *a, *b;
} pairbuf;

static void pb_push(pairbuf *p, int64_t a, int64_t b) {
  if (p->n == p->cap) {
    p->cap = p->cap ? 2 * p->cap : 1024;
    p->a = (int64_t *)realloc(p->a, sizeof(int64_t) * (size_t)p->cap);
    p->b = (int64_t *)realloc(p->b, sizeof(int64_t) * (size_t)p->cap);
  }
  p->a[p->n] = a;
  p->b[p->n] = b;
  p->n++;
}

typedef struct {
  pairbuf ss, st, sa;
} orc_pairs;

/* detect_contacts (broadphase.py:202-288) up to, not including, the slot ->
 * global-id map and canonical sort (done by the numpy wrapper exactly as the
 * reference does).  Returns an opaque handle; read it with orc_pairs_*. */
void *orc_detect(int64_t m, const double *centers, const float *radii,
                 const int64_t *sph_owner, const uint8_t *sph_family,
                 int64_t n_t, const double *tri_world, const int64_t *tri_owner,
                 const uint8_t *tri_family, int64_t n_a, const double *ana_world,
                 const uint8_t *ana_kind, const int64_t *ana_owner,
                 const uint8_t *ana_family, const uint8_t *mask /*256x256*/,
                 double margin, double *grid_out /* glo[3], inv_bin */,
                 int64_t *nb_out) {
  orc_pairs *res = (orc_pairs *)calloc(1, sizeof(orc_pairs));
  double r_max = 0.0;
  for (int64_t i = 0; i < m; ++i)
    if (i == 0 || (double)radii[i] > r_max) r_max = (double)radii[i];
  if (m == 0) r_max = 0.0;
  int64_t npts = m + 3 * n_t;
  double *pts = (double *)malloc(sizeof(double) * 3 * (size_t)(npts + 1));
  memcpy(pts, centers, sizeof(double) * 3 * (size_t)m);
  memcpy(pts + 3 * m, tri_world, sizeof(double) * 9 * (size_t)n_t);
  double glo[3] = {0, 0, 0}, inv_bin = 0.0;
  int64_t nb[3] = {0, 0, 0};
  int have_grid = orc_grid_for(npts, pts, r_max, margin, glo, &inv_bin, nb);
  free(pts);
  if (grid_out) {
    grid_out[0] = glo[0]; grid_out[1] = glo[1]; grid_out[2] = glo[2];
    grid_out[3] = inv_bin;
  }
  if (nb_out) { nb_out[0] = nb[0]; nb_out[1] = nb[1]; nb_out[2] = nb[2]; }

  if (m && have_grid) {
    int64_t *ranges = (int64_t *)malloc(sizeof(int64_t) * 6 * (size_t)m);
    orc_bin_ranges(m, centers, radii, margin, glo, inv_bin, nb, ranges);
    int64_t *starts, *entries;
    csr_bins(m, ranges, nb, &starts, &entries);
    int64_t nbins = nb[0] * nb[1] * nb[2];
    /* collect_sphere_pairs, _kernels.py:286-330 */
    for (int64_t b = 0; b < nbins; ++b) {
      int64_t s0 = starts[b], s1 = starts[b + 1];
      for (int64_t u = s0; u < s1; ++u) {
        int64_t i = entries[u];
        for (int64_t v = u + 1; v < s1; ++v) {
          int64_t j = entries[v];
          if (sph_owner[i] == sph_owner[j]) continue;
          if (!mask[256 * sph_family[i] + sph_family[j]]) continue;
          double dx = centers[3 * i] - centers[3 * j];
          double dy = centers[3 * i + 1] - centers[3 * j + 1];
          double dz = centers[3 * i + 2] - centers[3 * j + 2];
          double ri = (double)radii[i] + margin;
          double rj = (double)radii[j] + margin;
          double rr = ri + rj - margin;
          if (dx * dx + dy * dy + dz * dz >= rr * rr) continue;
          double mx = fmax(centers[3 * i] - ri, centers[3 * j] - rj);
          double my = fmax(centers[3 * i + 1] - ri, centers[3 * j + 1] - rj);
          double mz = fmax(centers[3 * i + 2] - ri, centers[3 * j + 2] - rj);
          if (bin_of(mx, my, mz, glo, inv_bin, nb) != b) continue;
          if (i < j) pb_push(&res->ss, i, j);
          else pb_push(&res->ss, j, i);
        }
      }
    }
    if (n_t) {
      /* tri_bin_ranges + collect_sphere_tri_pairs, _kernels.py:333-406 */
      int64_t *tr = (int64_t *)malloc(sizeof(int64_t) * 6 * (size_t)n_t);
      orc_tri_bin_ranges(n_t, tri_world, margin, glo, inv_bin, nb, tr);
      int64_t *ts, *te;
      csr_bins(n_t, tr, nb, &ts, &te);
      for (int64_t b = 0; b < nbins; ++b) {
        int64_t t0 = ts[b], t1 = ts[b + 1];
        if (t0 == t1) continue;
        for (int64_t u = starts[b]; u < starts[b + 1]; ++u) {
          int64_t i = entries[u];
          for (int64_t v = t0; v < t1; ++v) {
            int64_t t = te[v];
            if (sph_owner[i] == tri_owner[t]) continue;
            if (!mask[256 * sph_family[i] + tri_family[t]]) continue;
            const double *T = tri_world + 9 * t;
            double qx, qy, qz;
            closest_on_tri(centers[3 * i], centers[3 * i + 1], centers[3 * i + 2],
                           T, &qx, &qy, &qz);
            double dx = centers[3 * i] - qx;
            double dy = centers[3 * i + 1] - qy;
            double dz = centers[3 * i + 2] - qz;
            double rr = (double)radii[i] + margin;
            if (dx * dx + dy * dy + dz * dz >= rr * rr) continue;
            double mx = centers[3 * i] - rr;
            double my = centers[3 * i + 1] - rr;
            double mz = centers[3 * i + 2] - rr;
            double tlx = fmin(fmin(T[0], T[3]), T[6]) - margin;
            double tly = fmin(fmin(T[1], T[4]), T[7]) - margin;
            double tlz = fmin(fmin(T[2], T[5]), T[8]) - margin;
            if (tlx > mx) mx = tlx;
            if (tly > my) my = tly;
            if (tlz > mz) mz = tlz;
            if (bin_of(mx, my, mz, glo, inv_bin, nb) != b) continue;
            pb_push(&res->st, i, t);
          }
        }
      }
      free(tr); free(ts); free(te);
    }
    free(ranges); free(starts); free(entries);
  }
  if (m && n_a) {
    /* collect_sphere_analytic_pairs, _kernels.py:409-435 */
    for (int64_t i = 0; i < m; ++i)
      for (int64_t k = 0; k < n_a; ++k) {
        if (sph_owner[i] == ana_owner[k]) continue;
        if (!mask[256 * sph_family[i] + ana_family[k]]) continue;
        double gap, bx, by, bz, rb;
        analytic_gap(ana_kind[k], ana_world + 8 * k, centers[3 * i],
                     centers[3 * i + 1], centers[3 * i + 2], &gap, &bx, &by, &bz, &rb);
        if (gap >= (double)radii[i] + margin) continue;
        pb_push(&res->sa, i, k);
      }
  }
  return res;
}

void orc_pairs_counts(void *h, int64_t *out3) {
  orc_pairs *p = (orc_pairs *)h;
  out3[0] = p->ss.n; out3[1] = p->st.n; out3[2] = p->sa.n;
}

void orc_pairs_copy(void *h, int kind, int64_t *a, int64_t *b) {
  orc_pairs *p = (orc_pairs *)h;
  pairbuf *q = kind == 0 ? &p->ss : (kind == 1 ? &p->st : &p->sa);
  if (q->n) {
    memcpy(a, q->a, sizeof(int64_t) * (size_t)q->n);
    memcpy(b, q->b, sizeof(int64_t) * (size_t)q->n);
  }
}

void orc_pairs_free(void *h) {
  orc_pairs *p = (orc_pairs *)h;
  free(p->ss.a); free(p->ss.b); free(p->st.a); free(p->st.b);
  free(p->sa.a); free(p->sa.b); free(p);
}

/* ------------------------------------------------------------------------ */
/* per-contact geometry: _kernels.py:442-491                                 */
/* ------------------------------------------------------------------------ */

static void contact_geom(int kd, int64_t i, int64_t j, const double *c,
                         const float *rad, const double *tri, const double *ana,
                         const uint8_t *ana_kind, double *depth, double *bx,
                         double *by, double *bz, double *px, double *py,
                         double *pz, double *rb_out) {
  double cx = c[3 * i], cy = c[3 * i + 1], cz = c[3 * i + 2];
  double ra = (double)rad[i];
  double d, rb, dep;
  if (kd == 0) {
    double dx = cx - c[3 * j], dy = cy - c[3 * j + 1], dz = cz - c[3 * j + 2];
    d = sqrt(dx * dx + dy * dy + dz * dz);
    rb = (double)rad[j];
    if (d < 1e-300) {
      *depth = ra + rb; *bx = 0.0; *by = 0.0; *bz = 1.0;
      *px = cx; *py = cy; *pz = cz; *rb_out = rb;
      return;
    }
    double inv = 1.0 / d;
    *bx = dx * inv; *by = dy * inv; *bz = dz * inv;
    dep = ra + rb - d;
  } else if (kd == 1) {
    const double *T = tri + 9 * j;
    double qx, qy, qz;
    closest_on_tri(cx, cy, cz, T, &qx, &qy, &qz);
    double dx = cx - qx, dy = cy - qy, dz = cz - qz;
    d = sqrt(dx * dx + dy * dy + dz * dz);
    if (d < 1e-300) {
      double e1x = T[3] - T[0], e1y = T[4] - T[1], e1z = T[5] - T[2];
      double e2x = T[6] - T[0], e2y = T[7] - T[1], e2z = T[8] - T[2];
      double nx = e1y * e2z - e1z * e2y;
      double ny = e1z * e2x - e1x * e2z;
      double nz = e1x * e2y - e1y * e2x;
      double nn = sqrt(nx * nx + ny * ny + nz * nz);
      *bx = nx / nn; *by = ny / nn; *bz = nz / nn;
    } else {
      double inv = 1.0 / d;
      *bx = dx * inv; *by = dy * inv; *bz = dz * inv;
    }
    dep = ra - d;
    rb = FLAT_RADIUS;
  } else {
    double gap;
    analytic_gap(ana_kind[j], ana + 8 * j, cx, cy, cz, &gap, bx, by, bz, &rb);
    dep = ra - gap;
  }
  double half = ra - 0.5 * dep;
  *depth = dep;
  *px = cx - *bx * half; *py = cy - *by * half; *pz = cz - *bz * half;
  *rb_out = rb;
}

/* ------------------------------------------------------------------------ */
/* Hertz-Mindlin core: forces.py:82-182                                      */
/* ------------------------------------------------------------------------ */

void orc_hertz_mindlin_core(double overlap, double ts, double sim_time,
                            double b2ax, double b2ay, double b2az, double vx,
                            double vy, double vz, double wrx, double wry,
                            double wrz, double mass_eff, double ra, double rb,
                            int64_t mat_a, int64_t mat_b, const double *pair,
                            int64_t n_mat, float *wild, double *out) {
  (void)sim_time;
  for (int k = 0; k < 6; ++k) out[k] = 0.0;
  if (overlap <= 0.0) return; /* false positive: history untouched */
  int64_t mm = n_mat * n_mat, ab = mat_a * n_mat + mat_b;
  double e_cnt = pair[0 * mm + ab], g_cnt = pair[1 * mm + ab];
  double cor = pair[2 * mm + ab], mu = pair[3 * mm + ab], crr = pair[4 * mm + ab];

  double projection = vx * b2ax + vy * b2ay + vz * b2az;
  double vtx = vx - projection * b2ax;
  double vty = vy - projection * b2ay;
  double vtz = vz - projection * b2az;

  double dtx = (double)wild[0] + ts * vtx;
  double dty = (double)wild[1] + ts * vty;
  double dtz = (double)wild[2] + ts * vtz;
  double disp_proj = dtx * b2ax + dty * b2ay + dtz * b2az;
  dtx -= disp_proj * b2ax;
  dty -= disp_proj * b2ay;
  dtz -= disp_proj * b2az;
  double delta_time = (double)wild[3] + ts;

  double sqrt_rd = sqrt(overlap * (ra * rb) / (ra + rb));
  double sn = 2.0 * e_cnt * sqrt_rd;
  double loge = cor < 1e-12 ? log(1e-12) : log(cor);
  double beta = loge / sqrt(loge * loge + PI_D * PI_D);
  double k_n = 2.0 / 3.0 * sn;
  double gamma_n = 2.0 * sqrt(5.0 / 6.0) * beta * sqrt(sn * mass_eff);

  double fn = k_n * overlap + gamma_n * projection;
  out[0] = fn * b2ax;
  out[1] = fn * b2ay;
  out[2] = fn * b2az;

  if (crr > 0.0) {
    int add_rolling = 1;
    double r_eff = sqrt((ra * rb) / (ra + rb));
    double kn_simple = 4.0 / 3.0 * e_cnt * sqrt(r_eff);
    double gn_simple = -2.0 * sqrt(5.0 / 3.0 * mass_eff * e_cnt) * beta * pow(r_eff, 0.25);
    double d_coeff = gn_simple / (2.0 * sqrt(kn_simple * mass_eff));
    if (d_coeff < 1.0) {
      double t_collision = PI_D * sqrt(mass_eff / (kn_simple * (1.0 - d_coeff * d_coeff)));
      if (delta_time <= t_collision) add_rolling = 0;
    }
    if (add_rolling) {
      double v_rot_mag = sqrt(wrx * wrx + wry * wry + wrz * wrz);
      if (v_rot_mag > 1e-12) {
        double fmag = sqrt(out[0] * out[0] + out[1] * out[1] + out[2] * out[2]);
        double scale = crr * fmag / v_rot_mag;
        out[3] = wrx * scale;
        out[4] = wry * scale;
        out[5] = wrz * scale;
      }
    }
  }

  if (mu > 0.0) {
    double kt = 8.0 * g_cnt * sqrt_rd;
    double gt = -2.0 * sqrt(5.0 / 6.0) * beta * sqrt(mass_eff * kt);
    double tfx = -kt * dtx - gt * vtx;
    double tfy = -kt * dty - gt * vty;
    double tfz = -kt * dtz - gt * vtz;
    double ft = sqrt(tfx * tfx + tfy * tfy + tfz * tfz);
    if (ft > 1e-12) {
      double fmag = sqrt(out[0] * out[0] + out[1] * out[1] + out[2] * out[2]);
      double ft_max = fmag * mu;
      if (ft > ft_max) {
        double scale = ft_max / ft;
        tfx *= scale; tfy *= scale; tfz *= scale;
        dtx = (tfx + gt * vtx) / (-kt);
        dty = (tfy + gt * vty) / (-kt);
        dtz = (tfz + gt * vtz) / (-kt);
      }
    } else {
      tfx = 0.0; tfy = 0.0; tfz = 0.0;
    }
    out[0] += tfx;
    out[1] += tfy;
    out[2] += tfz;
  }
  wild[0] = (float)dtx;
  wild[1] = (float)dty;
  wild[2] = (float)dtz;
  wild[3] = (float)delta_time;
}

/* ------------------------------------------------------------------------ */
/* fused ACS sweep: forces.py:547-593 (default model)                        */
/* ------------------------------------------------------------------------ */

int64_t orc_contact_forces(int64_t n, const uint8_t *kind, const int64_t *slot_a,
                           const int64_t *slot_b, const int64_t *owner_a,
                           const int64_t *owner_b, const int64_t *mat_a,
                           const int64_t *mat_b, const double *sph_centers,
                           const float *sph_radii, const double *tri_world,
                           const double *ana_world, const uint8_t *ana_kind,
                           const double *owner_pos, const double *lin_vel,
                           const double *ang_vel_global, const double *mass,
                           const double *pair, int64_t n_mat, int64_t wstride,
                           float *wild, double ts, double sim_time,
                           double *out_ft, double *depth, double *cp,
                           int nthreads, int model) {
  int64_t touching = 0;
#ifdef _OPENMP
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) reduction(+ : touching) num_threads(nthreads)
#endif
  for (int64_t k = 0; k < n; ++k) {
    double dep, bx, by, bz, px, py, pz, rb;
    contact_geom(kind[k], slot_a[k], slot_b[k], sph_centers, sph_radii,
                 tri_world, ana_world, ana_kind, &dep, &bx, &by, &bz, &px, &py,
                 &pz, &rb);
    depth[k] = dep;
    cp[3 * k] = px; cp[3 * k + 1] = py; cp[3 * k + 2] = pz;
    int64_t oa = owner_a[k], ob = owner_b[k];
    const double *wa = ang_vel_global + 3 * oa, *wb = ang_vel_global + 3 * ob;
    /* _pair_kinematics, forces.py:55-79 */
    double rax = px - owner_pos[3 * oa], ray = py - owner_pos[3 * oa + 1],
           raz = pz - owner_pos[3 * oa + 2];
    double rbx = px - owner_pos[3 * ob], rby = py - owner_pos[3 * ob + 1],
           rbz = pz - owner_pos[3 * ob + 2];
    double rotax = wa[1] * raz - wa[2] * ray;
    double rotay = wa[2] * rax - wa[0] * raz;
    double rotaz = wa[0] * ray - wa[1] * rax;
    double rotbx = wb[1] * rbz - wb[2] * rby;
    double rotby = wb[2] * rbx - wb[0] * rbz;
    double rotbz = wb[0] * rby - wb[1] * rbx;
    const double *va = lin_vel + 3 * oa, *vb = lin_vel + 3 * ob;
    double vx = (va[0] + rotax) - (vb[0] + rotbx);
    double vy = (va[1] + rotay) - (vb[1] + rotby);
    double vz = (va[2] + rotaz) - (vb[2] + rotbz);
    double ma = mass[oa], mb = mass[ob];
    double mass_eff = (ma * mb) / (ma + mb);
    double *o6 = out_ft + 6 * k;
    double ra_k = (double)sph_radii[slot_a[k]];
    orc_hertz_mindlin_core(dep, ts, sim_time, bx, by, bz, vx, vy, vz,
                           rotbx - rotax, rotby - rotay, rotbz - rotaz, mass_eff,
                           ra_k, rb, mat_a[k], mat_b[k], pair, n_mat, wild + wstride * k, o6);
    if (model == 1 && dep > 0.0) {
      /* models.py hertz_mindlin_cohesive: F_c = coh * pi * R_eff * overlap along -B2A */
      double coh = pair[(5 * n_mat + mat_a[k]) * n_mat + mat_b[k]];
      double r_eff = ra_k * rb / (ra_k + rb);
      double f = coh * 3.141592653589793 * r_eff * dep;
      o6[0] -= f * bx; o6[1] -= f * by; o6[2] -= f * bz;
    }
    if (dep > 0.0) touching += kind[k] == 0 ? 2 : 1;
  }
  return touching;
}

/* ------------------------------------------------------------------------ */
/* owner reduction: _kernels.py:515-545                                      */
/* ------------------------------------------------------------------------ */

void orc_reduce_to_owners(int64_t n_acs, const int64_t *owner_a,
                          const int64_t *owner_b, const double *out_ft,
                          const double *cps, const double *owner_pos,
                          int64_t n_owner, double *acc_f, double *acc_t) {
  memset(acc_f, 0, sizeof(double) * 3 * (size_t)n_owner);
  memset(acc_t, 0, sizeof(double) * 3 * (size_t)n_owner);
  for (int64_t k = 0; k < n_acs; ++k) {
    int64_t oa = owner_a[k], ob = owner_b[k];
    const double *f = out_ft + 6 * k, *g = out_ft + 6 * k + 3, *c = cps + 3 * k;
    double rax = c[0] - owner_pos[3 * oa], ray = c[1] - owner_pos[3 * oa + 1],
           raz = c[2] - owner_pos[3 * oa + 2];
    double rbx = c[0] - owner_pos[3 * ob], rby = c[1] - owner_pos[3 * ob + 1],
           rbz = c[2] - owner_pos[3 * ob + 2];
    acc_f[3 * oa] += f[0]; acc_f[3 * oa + 1] += f[1]; acc_f[3 * oa + 2] += f[2];
    acc_f[3 * ob] -= f[0]; acc_f[3 * ob + 1] -= f[1]; acc_f[3 * ob + 2] -= f[2];
    double tx = f[0] + g[0], ty = f[1] + g[1], tz = f[2] + g[2];
    acc_t[3 * oa] += ray * tz - raz * ty;
    acc_t[3 * oa + 1] += raz * tx - rax * tz;
    acc_t[3 * oa + 2] += rax * ty - ray * tx;
    acc_t[3 * ob] -= rby * tz - rbz * ty;
    acc_t[3 * ob + 1] -= rbz * tx - rbx * tz;
    acc_t[3 * ob + 2] -= rbx * ty - rby * tx;
  }
}

/* ------------------------------------------------------------------------ */
/* integrator + refresh: _kernels.py:548-670                                 */
/* ------------------------------------------------------------------------ */

typedef struct {
  const uint8_t *fixed_flag;      /* [256] */
  const uint8_t *prescribed_flag; /* [256] */
  const uint8_t *lv_mask;         /* [256*3] */
  const double *lv_val;           /* [256*3] */
  const uint8_t *av_mask;         /* [256*3] */
  const double *av_val;           /* [256*3] */
} orc_family_tables;

static int64_t integrate_one(int64_t i, double h, double gx, double gy,
                             double gz, double *owner_pos, float *quat,
                             double *lin_vel, double *ang_vel,
                             const double *mass, const double *moi,
                             const double *acc_f, const double *acc_t,
                             const double *ext_f, const double *ext_t,
                             const uint8_t *family, const orc_family_tables *ft,
                             double v_err) {
  int fam = family[i];
  double *v = lin_vel + 3 * i, *w = ang_vel + 3 * i;
  if (ft->fixed_flag[fam]) {
    v[0] = 0.0; v[1] = 0.0; v[2] = 0.0;
    w[0] = 0.0; w[1] = 0.0; w[2] = 0.0;
    return 0;
  }
  float *q = quat + 4 * i;
  double qw = (double)q[0], qx = (double)q[1], qy = (double)q[2], qz = (double)q[3];
  double vx, vy, vz, wx, wy, wz;
  if (ft->prescribed_flag[fam]) {
    const uint8_t *lm = ft->lv_mask + 3 * fam, *am = ft->av_mask + 3 * fam;
    const double *lv = ft->lv_val + 3 * fam, *av = ft->av_val + 3 * fam;
    vx = lm[0] ? lv[0] : v[0];
    vy = lm[1] ? lv[1] : v[1];
    vz = lm[2] ? lv[2] : v[2];
    wx = w[0]; wy = w[1]; wz = w[2];
    if (am[0] || am[1] || am[2]) {
      double pwx, pwy, pwz;
      qrot(qw, qx, qy, qz, wx, wy, wz, &pwx, &pwy, &pwz);
      if (am[0]) pwx = av[0];
      if (am[1]) pwy = av[1];
      if (am[2]) pwz = av[2];
      qrot(qw, -qx, -qy, -qz, pwx, pwy, pwz, &wx, &wy, &wz);
    }
  } else {
    double m = mass[i];
    vx = v[0] + h * ((acc_f[3 * i] + ext_f[3 * i]) / m + gx);
    vy = v[1] + h * ((acc_f[3 * i + 1] + ext_f[3 * i + 1]) / m + gy);
    vz = v[2] + h * ((acc_f[3 * i + 2] + ext_f[3 * i + 2]) / m + gz);
    double tgx = acc_t[3 * i] + ext_t[3 * i];
    double tgy = acc_t[3 * i + 1] + ext_t[3 * i + 1];
    double tgz = acc_t[3 * i + 2] + ext_t[3 * i + 2];
    double tlx, tly, tlz;
    qrot(qw, -qx, -qy, -qz, tgx, tgy, tgz, &tlx, &tly, &tlz);
    wx = w[0]; wy = w[1]; wz = w[2];
    double ix = moi[3 * i], iy = moi[3 * i + 1], iz = moi[3 * i + 2];
    double gyx = wy * (iz * wz) - wz * (iy * wy);
    double gyy = wz * (ix * wx) - wx * (iz * wz);
    double gyz = wx * (iy * wy) - wy * (ix * wx);
    wx += h * (tlx - gyx) / ix;
    wy += h * (tly - gyy) / iy;
    wz += h * (tlz - gyz) / iz;
  }
  owner_pos[3 * i] += h * vx;
  owner_pos[3 * i + 1] += h * vy;
  owner_pos[3 * i + 2] += h * vz;
  double hw = 0.5 * h;
  double dqw = hw * (-qx * wx - qy * wy - qz * wz);
  double dqx = hw * (qw * wx + qy * wz - qz * wy);
  double dqy = hw * (qw * wy + qz * wx - qx * wz);
  double dqz = hw * (qw * wz + qx * wy - qy * wx);
  qw += dqw; qx += dqx; qy += dqy; qz += dqz;
  double inv = 1.0 / sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  q[0] = (float)(qw * inv);
  q[1] = (float)(qx * inv);
  q[2] = (float)(qy * inv);
  q[3] = (float)(qz * inv);
  v[0] = vx; v[1] = vy; v[2] = vz;
  w[0] = wx; w[1] = wy; w[2] = wz;
  return (vx * vx + vy * vy + vz * vz > v_err * v_err) ? 1 : 0;
}

/* Returns bad/oob through out2 = {first speeding owner or -1, first
 * out-of-domain owner or -1}.  nthreads > 1 parallelises the per-owner loops
 * (results are identical; on the error path every owner is still encoded). */
void orc_integrate_and_refresh(
    int64_t n, double h, double gx, double gy, double gz, double *owner_pos,
    float *quat, double *lin_vel, double *ang_vel, const double *mass,
    const double *moi, const double *acc_f, const double *acc_t,
    const double *ext_f, const double *ext_t, const uint8_t *family,
    const uint8_t *fixed_flag, const uint8_t *lv_mask, const double *lv_val,
    const uint8_t *av_mask, const double *av_val, const uint8_t *prescribed_flag,
    double v_err, const double *lo, const double *hi, double edge,
    uint64_t *voxel, uint16_t *sub, int64_t n_s, const int64_t *sph_geom,
    const float *geom_params, const int64_t *geom_owner, double *sph_centers,
    int nthreads, int64_t *out2) {
  orc_family_tables ft = {fixed_flag, prescribed_flag, lv_mask, lv_val, av_mask, av_val};
  int64_t bad = -1, oob = -1;
  if (nthreads <= 1) {
    for (int64_t i = 0; i < n; ++i)
      if (integrate_one(i, h, gx, gy, gz, owner_pos, quat, lin_vel, ang_vel, mass,
                        moi, acc_f, acc_t, ext_f, ext_t, family, &ft, v_err) &&
          bad < 0)
        bad = i;
    oob = orc_encode_positions(n, owner_pos, lo, hi, edge, voxel, sub);
    out2[0] = bad; out2[1] = oob;
    if (oob >= 0) return;
    orc_decode_positions(n, voxel, sub, lo, edge, owner_pos);
    orc_sphere_world(n_s, sph_geom, geom_params, geom_owner, owner_pos, quat,
                     sph_centers, NULL);
    return;
  }
#ifdef _OPENMP
  int64_t bad_min = n, oob_min = n;
#pragma omp parallel num_threads(nthreads)
  {
    int64_t lb = n, lo_ = n;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      if (integrate_one(i, h, gx, gy, gz, owner_pos, quat, lin_vel, ang_vel, mass,
                        moi, acc_f, acc_t, ext_f, ext_t, family, &ft, v_err) &&
          i < lb)
        lb = i;
      int64_t r = orc_encode_positions(1, owner_pos + 3 * i, lo, hi, edge,
                                       voxel + i, sub + 3 * i);
      if (r >= 0 && i < lo_) lo_ = i;
    }
#pragma omp critical
    {
      if (lb < bad_min) bad_min = lb;
      if (lo_ < oob_min) oob_min = lo_;
    }
  }
  out2[0] = bad_min < n ? bad_min : -1;
  out2[1] = oob_min < n ? oob_min : -1;
  if (out2[1] >= 0) return;
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t i = 0; i < n; ++i)
    orc_decode_positions(1, voxel + i, sub + 3 * i, lo, edge, owner_pos + 3 * i);
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t k = 0; k < n_s; ++k)
    orc_sphere_world(1, sph_geom + k, geom_params, geom_owner, owner_pos, quat,
                     sph_centers + 3 * k, NULL);
#else
  (void)bad; (void)oob;
  out2[0] = -1; out2[1] = -1;
#endif
}
