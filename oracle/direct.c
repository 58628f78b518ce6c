/* oracle/direct.c -- TEST INFRASTRUCTURE ONLY (never linked into the product path).
 *
 * Plain FP64 O(N^2) direct sums of the Laplace kernel with the explicit 1/(4 pi)
 * of PAPER.md Eq. 4-5.  No blocking, no fast math, one OpenMP loop over
 * targets; each target's sum runs over sources in index order.
 *
 *   G(x, y)          = 1 / (4 pi |x - y|)                         (Eq. 5)
 *   dG/dn_x (x, y)   = -n_x . (x - y) / (4 pi |x - y|^3)           (Eq. 4)
 *   dG/dn_y (x, y)   =  n_y . (x - y) / (4 pi |x - y|^3)           (double layer)
 *
 * Pair (i, j) is skipped when tid[i] == owner[j] (both non-NULL): this is the
 * "j != i" of the discrete operators K' and V (SPEC.md
 * S:364).  A non-skipped pair at zero distance is a hard error (return 1),
 * per SURVEY A14 / SPEC S:356 "charge coincident with a panel centroid".
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const double FOUR_PI = 12.566370614359172953850573533118;

int oracle_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* out[i] = sum_j w[j] * dG/dn_x(x_i, y_j)   (normal derivative at the target) */
int oracle_dn_sum(int64_t nt, const double* x, const double* n, const int64_t* tid,
                  int64_t ns, const double* y, const double* w, const int64_t* owner,
                  double* out) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
  for (int64_t i = 0; i < nt; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < ns; ++j) {
      if (tid && owner && tid[i] == owner[j]) continue;
      double dx = x[3 * i] - y[3 * j], dy = x[3 * i + 1] - y[3 * j + 1], dz = x[3 * i + 2] - y[3 * j + 2];
      double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 == 0.0) { bad = 1; continue; }
      double r = sqrt(r2);
      double ndot = n[3 * i] * dx + n[3 * i + 1] * dy + n[3 * i + 2] * dz;
      s += w[j] * (-ndot / (FOUR_PI * r2 * r));
    }
    out[i] = s;
  }
  return bad;
}

/* out[i] = sum_j w[j] * dG/dn_y(x_i, y_j) with the SOURCE normal m_j (double-layer kernel) */
int oracle_dipole_sum(int64_t nt, const double* x, const int64_t* tid, int64_t ns, const double* y,
                      const double* m, const double* w, const int64_t* owner, double* out) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
  for (int64_t i = 0; i < nt; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < ns; ++j) {
      if (tid && owner && tid[i] == owner[j]) continue;
      double dx = x[3 * i] - y[3 * j], dy = x[3 * i + 1] - y[3 * j + 1], dz = x[3 * i + 2] - y[3 * j + 2];
      double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 == 0.0) { bad = 1; continue; }
      double r = sqrt(r2);
      double mdot = m[3 * j] * dx + m[3 * j + 1] * dy + m[3 * j + 2] * dz;
      s += w[j] * (mdot / (FOUR_PI * r2 * r));
    }
    out[i] = s;
  }
  return bad;
}

/* out[i] = sum_j w[j] * G(x_i, y_j)   (potential) */
int oracle_pot_sum(int64_t nt, const double* x, const int64_t* tid, int64_t ns, const double* y,
                   const double* w, const int64_t* owner, double* out) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
  for (int64_t i = 0; i < nt; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < ns; ++j) {
      if (tid && owner && tid[i] == owner[j]) continue;
      double dx = x[3 * i] - y[3 * j], dy = x[3 * i + 1] - y[3 * j + 1], dz = x[3 * i + 2] - y[3 * j + 2];
      double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 == 0.0) { bad = 1; continue; }
      s += w[j] / (FOUR_PI * sqrt(r2));
    }
    out[i] = s;
  }
  return bad;
}

/* ---------------------------------------------------------------------------------------------
 * Near-field integrals over one flat triangle (SURVEY 8(a) a11 / 8(c) O4 option near_mode = 1;
 * PAPER.md P:415-418 "one may also compute some of these integrals analytically").  The oracle
 * does NOT use the analytic formulas: it integrates
 *     pot = int_T G(x, y) dA_y,     dn = int_T dG/dn_x(x, y) dA_y = -n_x . int_T (x - y)/(4 pi r^3) dA_y
 * numerically -- adaptive 4-way subdivision with the 7-point degree-5 rule, refined until the
 * children agree with the parent to 1e-12 (relative) -- and, when x is a point of T (the single-
 * layer self term), splits T at x into three triangles whose 1/r singularity sits at a vertex and
 * integrates each with the Duffy map y = x + u (p - x) + u v (q - p) (the Jacobian 2 A u cancels
 * 1/r), leaving a smooth 1-D integral done with 48-point Gauss-Legendre.
 * ------------------------------------------------------------------------------------------- */
static const double R7B[7][3] = {{1.0 / 3, 1.0 / 3, 1.0 / 3},
                                 {0.059715871789770, 0.470142064105115, 0.470142064105115},
                                 {0.470142064105115, 0.059715871789770, 0.470142064105115},
                                 {0.470142064105115, 0.470142064105115, 0.059715871789770},
                                 {0.797426985353087, 0.101286507323456, 0.101286507323456},
                                 {0.101286507323456, 0.797426985353087, 0.101286507323456},
                                 {0.101286507323456, 0.101286507323456, 0.797426985353087}};
static const double R7W[7] = {0.225, 0.132394152788506, 0.132394152788506, 0.132394152788506,
                              0.125939180544827, 0.125939180544827, 0.125939180544827};

static double tri_area(const double* a, const double* b, const double* c) {
  double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]}, e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
  return 0.5 * sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
}

static void rule7(const double* x, const double* n, const double* a, const double* b, const double* c,
                  double* pot, double* dn) {
  double ar = tri_area(a, b, c), sp = 0.0, sd = 0.0;
  for (int g = 0; g < 7; ++g) {
    double y[3], d[3];
    for (int k = 0; k < 3; ++k) {
      y[k] = R7B[g][0] * a[k] + R7B[g][1] * b[k] + R7B[g][2] * c[k];
      d[k] = x[k] - y[k];
    }
    double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    sp += R7W[g] / (FOUR_PI * r);
    sd += R7W[g] * (-(n[0] * d[0] + n[1] * d[1] + n[2] * d[2]) / (FOUR_PI * r * r * r));
  }
  *pot = ar * sp;
  *dn = ar * sd;
}

static void adapt(const double* x, const double* n, const double* a, const double* b, const double* c, int depth,
                  double* pot, double* dn) {
  double m01[3], m12[3], m20[3];
  for (int k = 0; k < 3; ++k) {
    m01[k] = 0.5 * (a[k] + b[k]);
    m12[k] = 0.5 * (b[k] + c[k]);
    m20[k] = 0.5 * (c[k] + a[k]);
  }
  const double* kids[4][3] = {{a, m01, m20}, {m01, b, m12}, {m20, m12, c}, {m01, m12, m20}};
  double p0, d0, ps = 0.0, ds = 0.0;
  rule7(x, n, a, b, c, &p0, &d0);
  double pk[4], dk[4];
  for (int t = 0; t < 4; ++t) {
    rule7(x, n, kids[t][0], kids[t][1], kids[t][2], &pk[t], &dk[t]);
    ps += pk[t];
    ds += dk[t];
  }
  if (depth >= 14 || (fabs(ps - p0) <= 1e-12 * fabs(ps) && fabs(ds - d0) <= 1e-12 * fabs(ds) + 1e-14 * fabs(ps))) {
    *pot = ps;
    *dn = ds;
    return;
  }
  *pot = 0.0;
  *dn = 0.0;
  for (int t = 0; t < 4; ++t) {
    double p, d;
    adapt(x, n, kids[t][0], kids[t][1], kids[t][2], depth + 1, &p, &d);
    *pot += p;
    *dn += d;
  }
}

/* 48-point Gauss-Legendre on [0, 1] (nodes/weights by Newton on P_48, computed once) */
static double GLX[48], GLW[48];
static int gl_ready = 0;
static void gl_init(void) {
  if (gl_ready) return;
  const int N = 48;
  for (int i = 0; i < N; ++i) {
    double z = cos(3.14159265358979323846 * (i + 0.75) / (N + 0.5)), pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= N; ++j) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = N * (z * p1 - p2) / (z * z - 1.0);
      double z1 = z;
      z = z1 - p1 / pp;
      if (fabs(z - z1) < 1e-16) break;
    }
    GLX[i] = 0.5 * (1.0 - z);
    GLW[i] = 1.0 / ((1.0 - z * z) * pp * pp);
  }
  gl_ready = 1;
}

/* int over triangle (x, p, q) of G(x, y) dA_y, singular vertex x (Duffy) */
static double duffy_pot(const double* x, const double* p, const double* q) {
  double A = tri_area(x, p, q), s = 0.0;
  for (int i = 0; i < 48; ++i) {
    double v = GLX[i], d[3];
    for (int k = 0; k < 3; ++k) d[k] = p[k] - x[k] + v * (q[k] - p[k]);
    s += GLW[i] / sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  }
  return 2.0 * A * s / FOUR_PI;
}

/* For each pair k: tv = 9 doubles (triangle vertices), x / n = target point and normal,
 * self[k] != 0 when x is a point of the triangle (only pot is then defined; dn = 0 because
 * n_x . (x - y) = 0 on the plane of T).  Outputs pot[k], dn[k]. */
void oracle_tri_integrals(int64_t np, const double* x, const double* n, const double* tv, const int32_t* self,
                          double* pot, double* dn) {
  gl_init();
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t k = 0; k < np; ++k) {
    const double* a = tv + 9 * k;
    const double* b = a + 3;
    const double* c = a + 6;
    if (self && self[k]) {
      pot[k] = duffy_pot(x + 3 * k, a, b) + duffy_pot(x + 3 * k, b, c) + duffy_pot(x + 3 * k, c, a);
      dn[k] = 0.0;
    } else {
      adapt(x + 3 * k, n + 3 * k, a, b, c, 0, pot + k, dn + k);
    }
  }
}
