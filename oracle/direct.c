/* oracle/direct.c -- TEST INFRASTRUCTURE ONLY (never linked into the product path).
 *
 * Plain FP64 O(N^2) direct sums of the Laplace kernel with the explicit 1/(4 pi)
 * of PAPER.md Eq. 4-5.  No blocking, no fast math, one OpenMP loop over
 * targets; each target's sum runs over sources in index order.
 *
 *   G(x, y)          = 1 / (4 pi |x - y|)                         (Eq. 5)
 *   dG/dn_x (x, y)   = -n_x . (x - y) / (4 pi |x - y|^3)           (Eq. 4)
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
