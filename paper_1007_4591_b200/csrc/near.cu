// near.cu -- analytic near-field panel integration, option near_mode = 1 (SURVEY 8(a) a11 and
// 8(c) O4; "For planar elements and polynomial basis functions, one may also
// compute some of these integrals analytically [Hess62, Newman86]").
//
// For every target panel i and source panel j != i with |c_i - c_j| < eta sqrt(A_j), the K-point
// quadrature term of the operators is replaced by the exact integral over the flat triangle T_j:
//   C_ij^K' = n_i . int_{T_j} grad_x G(c_i, y) dA_y - A_j sum_g w_g dG/dn_i(c_i, y_jg)
//   C_ij^V  =       int_{T_j} G(c_i, y) dA_y     - A_j sum_g w_g G(c_i, y_jg)
// and V gains the self term int_{T_i} G(c_i, y) dA_y (K'_ii stays 0: n_i.(c_i - y) = 0 on T_i).
// Closed forms for a flat triangle with unit normal N, height h = N.(x - v0), edges e = (p -> q),
// t_e = (q - p)/|q - p|, m_e = t_e x N, d_e = m_e.(p - x), s-+ = (p|q - x).t_e, R-+ = |p|q - x|,
// L_e = ln((R+ + s+)/(R- + s-)) and the signed solid angle Om (Van Oosterom-Strackee):
//   int_T dA/|x-y|          =  sum_e d_e L_e + h Om
//   int_T grad_x 1/|x-y| dA = -sum_e m_e L_e + N Om
// evaluated in FP64 once per geometry; the per-matvec correction is a CSR SpMV in FP32.
#include <cmath>
#include <cstring>

#include "kernels.cuh"

namespace fmm {

namespace {

constexpr double INV4PI = 0.079577471545947667884441881686257;

__device__ inline void sub3(const double* a, const double* b, double* o) {
  o[0] = a[0] - b[0];
  o[1] = a[1] - b[1];
  o[2] = a[2] - b[2];
}
__device__ inline double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
__device__ inline void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

// pot = int_T G(x, y) dA, grad = int_T grad_x G(x, y) dA (both with the 1/(4 pi))
__device__ void tri_exact(const double* x, const double* v0, const double* v1, const double* v2, double& pot,
                          double* grad) {
  const double* V[3] = {v0, v1, v2};
  double e1[3], e2[3], N[3];
  sub3(v1, v0, e1);
  sub3(v2, v0, e2);
  cross3(e1, e2, N);
  const double nn = sqrt(dot3(N, N));
  N[0] /= nn;
  N[1] /= nn;
  N[2] /= nn;
  double xv[3];
  sub3(x, v0, xv);
  const double h = dot3(N, xv);
  double a[3], b[3], c[3], bc[3];
  sub3(v0, x, a);
  sub3(v1, x, b);
  sub3(v2, x, c);
  cross3(b, c, bc);
  const double la = sqrt(dot3(a, a)), lb = sqrt(dot3(b, b)), lc = sqrt(dot3(c, c));
  const double den = la * lb * lc + dot3(a, b) * lc + dot3(a, c) * lb + dot3(b, c) * la;
  const double om = 2.0 * atan2(dot3(a, bc), den);
  double sp = 0.0, g[3] = {0.0, 0.0, 0.0};
  for (int e = 0; e < 3; ++e) {
    const double* p = V[e];
    const double* q = V[(e + 1) % 3];
    double t[3], m[3], px[3], qx[3];
    sub3(q, p, t);
    const double len = sqrt(dot3(t, t));
    t[0] /= len;
    t[1] /= len;
    t[2] /= len;
    cross3(t, N, m);
    sub3(p, x, px);
    sub3(q, x, qx);
    const double sm = dot3(px, t), sq = dot3(qx, t);
    const double rm = sqrt(dot3(px, px)), rq = sqrt(dot3(qx, qx));
    // (R+ + s+)/(R- + s-) == (R- - s-)/(R+ - s+): take the form with the larger denominators
    double le;
    if (fmin(rq + sq, rm + sm) >= fmin(rm - sm, rq - sq)) le = log((rq + sq) / (rm + sm));
    else le = log((rm - sm) / (rq - sq));
    sp += dot3(m, px) * le;
    g[0] -= m[0] * le;
    g[1] -= m[1] * le;
    g[2] -= m[2] * le;
  }
  pot = INV4PI * (sp + h * om);
  grad[0] = INV4PI * (g[0] + N[0] * om);
  grad[1] = INV4PI * (g[1] + N[1] * om);
  grad[2] = INV4PI * (g[2] + N[2] * om);
}

struct NearGeom {
  const int* perm;     // tree order -> caller panel
  const double* cen;   // caller order [np*3]
  const double* nrm;
  const double* area;
  const double* V;     // vertices
  const int* T;        // triangles
  const double* beta;  // [K*3]
  const double* wq;    // [K]
  int K;
  const int* leaf;     // pan.leaf (tree order)
  const int* beg;      // pan.begin
  const int* nbr_off;
  const int* nbr_idx;
  double eta;
};

__device__ inline bool is_near(const NearGeom& g, int p, int q) {
  double d[3];
  sub3(g.cen + 3 * (size_t)p, g.cen + 3 * (size_t)q, d);
  return sqrt(dot3(d, d)) < g.eta * sqrt(g.area[q]);
}

__global__ void k_near_count(int nrows, int row0, NearGeom g, int* cnt) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int i = row0 + r, p = g.perm[i], leaf = g.leaf[i];
  int c = 0;
  for (int e = g.nbr_off[leaf]; e < g.nbr_off[leaf + 1]; ++e) {
    const int L = g.nbr_idx[e];
    for (int j = g.beg[L]; j < g.beg[L + 1]; ++j)
      if (j != i && is_near(g, p, g.perm[j])) ++c;
  }
  cnt[r] = c;
}

__global__ void k_near_fill(int nrows, int row0, NearGeom g, const long long* __restrict__ off, int* col, float* vkp,
                            float* vsl, float* diag) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int i = row0 + r, p = g.perm[i], leaf = g.leaf[i];
  const double* x = g.cen + 3 * (size_t)p;
  const double* n = g.nrm + 3 * (size_t)p;
  long long w = off[r];
  for (int e = g.nbr_off[leaf]; e < g.nbr_off[leaf + 1]; ++e) {
    const int L = g.nbr_idx[e];
    for (int j = g.beg[L]; j < g.beg[L + 1]; ++j) {
      if (j == i) continue;
      const int q = g.perm[j];
      if (!is_near(g, p, q)) continue;
      const double* v0 = g.V + 3 * (size_t)g.T[3 * (size_t)q];
      const double* v1 = g.V + 3 * (size_t)g.T[3 * (size_t)q + 1];
      const double* v2 = g.V + 3 * (size_t)g.T[3 * (size_t)q + 2];
      double pot, grad[3];
      tri_exact(x, v0, v1, v2, pot, grad);
      double qp = 0.0, qd = 0.0;
      for (int k = 0; k < g.K; ++k) {
        double y[3], d[3];
        for (int a = 0; a < 3; ++a)
          y[a] = g.beta[3 * k] * v0[a] + g.beta[3 * k + 1] * v1[a] + g.beta[3 * k + 2] * v2[a];
        sub3(x, y, d);
        const double rr = sqrt(dot3(d, d));
        qp += g.wq[k] * INV4PI / rr;
        qd += g.wq[k] * (-dot3(n, d)) * INV4PI / (rr * rr * rr);
      }
      col[w] = j;
      vkp[w] = (float)(dot3(n, grad) - g.area[q] * qd);
      vsl[w] = (float)(pot - g.area[q] * qp);
      ++w;
    }
  }
  // single-layer self term of the flat panel (x in the plane of T_p: h = 0)
  const double* v0 = g.V + 3 * (size_t)g.T[3 * (size_t)p];
  const double* v1 = g.V + 3 * (size_t)g.T[3 * (size_t)p + 1];
  const double* v2 = g.V + 3 * (size_t)g.T[3 * (size_t)p + 2];
  double pot, grad[3];
  tri_exact(x, v0, v1, v2, pot, grad);
  diag[r] = (float)pot;
}

// y[i] += b * (sum_k val[k] x[col[k]] + diag[i] x[i]) for the rows [row0, row0 + nrows)
__global__ void k_near_apply(int nrows, int row0, const long long* __restrict__ off, const int* __restrict__ col,
                             const float* __restrict__ val, const float* __restrict__ diag, const float* __restrict__ x,
                             float* __restrict__ y, float b) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int i = row0 + r;
  float s = diag ? diag[r] * x[i] : 0.f;
  for (long long k = off[r]; k < off[r + 1]; ++k) s = fmaf(val[k], x[col[k]], s);
  y[i] = fmaf(b, s, y[i]);
}

__global__ void k_widen_near(int n, const int* __restrict__ in, long long* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

__global__ void k_max_sqrt_area(int64_t n, const double* __restrict__ area, unsigned int* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) atomicMax(out, __float_as_uint((float)sqrt(area[i])));
}

}  // namespace

void build_near(fmmbem_ctx* c, const double* V, const int* T, const double* cen, const double* nrm,
                const double* area, const double* beta, const double* wq, cudaStream_t st) {
  const Tree& Tr = c->tree;
  const double eta = c->opt.near_radius;
  // every near pair must lie in the P2P neighbourhood (adjacent leaves)
  DevBuf<unsigned int> mx;
  mx.alloc(1);
  mx.zero(st);
  k_max_sqrt_area<<<ceil_div(c->np, 256), 256, 0, st>>>(c->np, area, mx.get());
  FMM_CHECK_LAUNCH();
  unsigned int hm = 0;
  FMM_CUDA(cudaMemcpyAsync(&hm, mx.get(), sizeof(hm), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  float msa;
  std::memcpy(&msa, &hm, sizeof(msa));
  if (eta * msa * 1.0001 >= Tr.width(Tr.L))
    throw Error(FMMBEM_E_INVALID, "near_radius * sqrt(max area) exceeds the leaf width; raise leaf_points");
  DevBuf<int> perm;
  perm.alloc(c->np);
  {
    std::vector<int> h(c->pan_ids.begin(), c->pan_ids.end());
    FMM_CUDA(cudaMemcpyAsync(perm.get(), h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    FMM_CUDA(cudaStreamSynchronize(st));
  }
  NearGeom g{perm.get(), cen, nrm, area, V, T, beta, wq, c->K, c->pan.leaf.get(), c->pan.begin.get(),
             Tr.nbr_off.get(), Tr.nbr_idx.get(), eta};
  const int nrows = (int)c->n_own(), row0 = (int)c->pan_lo;
  auto& N = c->near;
  N.off.alloc(nrows + 1);
  DevBuf<int> cnt;
  DevBuf<long long> cnt64;
  cnt.alloc(nrows + 1);
  cnt64.alloc(nrows + 1);
  cnt.zero(st);
  if (nrows > 0) k_near_count<<<ceil_div(nrows, 128), 128, 0, st>>>(nrows, row0, g, cnt.get());
  k_widen_near<<<ceil_div(nrows + 1, 256), 256, 0, st>>>(nrows + 1, cnt.get(), cnt64.get());
  FMM_CHECK_LAUNCH();
  scan_i64(cnt64.get(), N.off.get(), nrows + 1, st);
  long long nnz = 0;
  FMM_CUDA(cudaMemcpyAsync(&nnz, N.off.get() + nrows, sizeof(long long), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  N.nnz = nnz;
  N.col.alloc(std::max<long long>(nnz, 1));
  N.vkp.alloc(std::max<long long>(nnz, 1));
  N.vsl.alloc(std::max<long long>(nnz, 1));
  N.diag.alloc(std::max(nrows, 1));
  if (nrows > 0)
    k_near_fill<<<ceil_div(nrows, 128), 128, 0, st>>>(nrows, row0, g, N.off.get(), N.col.get(), N.vkp.get(),
                                                      N.vsl.get(), N.diag.get());
  FMM_CHECK_LAUNCH();
  FMM_CUDA(cudaStreamSynchronize(st));
}

void apply_near(fmmbem_ctx* c, bool single, const float* x_full, float* y_global, float b, cudaStream_t st) {
  const int nrows = (int)c->n_own();
  if (nrows <= 0) return;
  const auto& N = c->near;
  k_near_apply<<<ceil_div(nrows, 256), 256, 0, st>>>(nrows, (int)c->pan_lo, N.off.get(), N.col.get(),
                                                     single ? N.vsl.get() : N.vkp.get(),
                                                     single ? N.diag.get() : nullptr, x_full, y_global, b);
  FMM_CHECK_LAUNCH();
}

}  // namespace fmm
