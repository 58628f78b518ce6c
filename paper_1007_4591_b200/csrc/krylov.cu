// krylov.cu -- restarted GMRES(m) driver and deterministic FP64 reductions
// ("solving the linear system using Krylov-subspace
// iterative methods such as GMRES", Eq. 6).
//
// The Krylov basis lives on the device in FP32 ([(m+1) x n]); the Arnoldi coefficients are
// reduced in FP64 with a fixed block order (classical Gram-Schmidt applied twice, CGS2: the
// same Krylov space as MGS with two reductions per step); the small Hessenberg problem and
// the Givens rotations run on the host in FP64.  One host<->device synchronisation per
// iteration (the new Hessenberg column, m+2 doubles).
#include <cmath>

#include "kernels.cuh"

namespace fmm {

namespace {

constexpr int RB = 256;      // reduction block
constexpr int RCHUNK = 8192; // elements per block

__device__ inline double block_sum(double v, double* sh) {
  for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  return s;
}

// part[b * nvec + k] = sum_{i in chunk b} V[k][i] * w[i]  (optionally * wt[i].w)
__global__ void __launch_bounds__(RB) k_gemv_t(const float* __restrict__ V, int64_t ld, int nvec, int64_t n,
                                               const float* __restrict__ w, const float4* __restrict__ wt,
                                               double* __restrict__ part) {
  __shared__ double sh[RB / 32];
  const int64_t lo = (int64_t)blockIdx.x * RCHUNK, hi = min(n, lo + RCHUNK);
  for (int k = 0; k < nvec; ++k) {
    const float* v = V + (size_t)k * ld;
    double a = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += RB) {
      double t = (double)v[i] * (double)w[i];
      if (wt) t *= (double)wt[i].w;
      a += t;
    }
    double s = block_sum(a, sh);
    if (threadIdx.x == 0) part[(size_t)blockIdx.x * nvec + k] = s;
  }
}

// out[k] (+)= sum_b part[b * nvec + k]   (fixed order)
__global__ void k_reduce_part(int nb, int nvec, const double* __restrict__ part, double* __restrict__ out,
                              int accumulate) {
  __shared__ double sh[RB / 32];
  const int k = blockIdx.x;
  double a = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) a += part[(size_t)b * nvec + k];
  double s = block_sum(a, sh);
  if (threadIdx.x == 0) out[k] = accumulate ? out[k] + s : s;
}

// w[i] += sgn * sum_k V[k][i] h[k]
__global__ void k_gemv_n(float* __restrict__ w, const float* __restrict__ V, int64_t ld, int nvec, int64_t n,
                         const double* __restrict__ h, double sgn) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = 0.0;
  for (int k = 0; k < nvec; ++k) a += (double)V[(size_t)k * ld + i] * h[k];
  w[i] = (float)((double)w[i] + sgn * a);
}

__global__ void k_scale_to(float* __restrict__ dst, const float* __restrict__ src, int64_t n,
                           const double* __restrict__ nrm2) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = nrm2[0] > 0.0 ? 1.0 / sqrt(nrm2[0]) : 0.0;
  dst[i] = (float)((double)src[i] * s);
}

__global__ void k_sub(float* __restrict__ r, const float* __restrict__ b, const float* __restrict__ ax, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) r[i] = b[i] - ax[i];
}

int nblocks(int64_t n) { return (int)((n + RCHUNK - 1) / RCHUNK); }

// h[0..nvec) = V^T w (accumulate if acc)
void gemv_t(fmmbem_ctx* c, const float* V, int64_t ld, int nvec, int64_t n, const float* w, const float4* wt,
            double* h, bool acc, cudaStream_t s) {
  int nb = nblocks(n);
  size_t need = (size_t)nb * nvec;
  if (c->part.n < need) c->part.alloc(need);
  if (nb > 0) {
    k_gemv_t<<<nb, RB, 0, s>>>(V, ld, nvec, n, w, wt, c->part.get());
    k_reduce_part<<<nvec, RB, 0, s>>>(nb, nvec, c->part.get(), h, acc ? 1 : 0);
  } else if (!acc) {
    FMM_CUDA(cudaMemsetAsync(h, 0, nvec * sizeof(double), s));
  }
  FMM_CHECK_LAUNCH();
  // distributed vectors: every rank holds a slice; the FP64 partial dots are summed over ranks
  if (!acc) comm_allreduce_f64(c, h, nvec, s);
  else throw Error(FMMBEM_E_INVALID, "accumulating distributed dot not supported");
}

}  // namespace

double dot_weighted(fmmbem_ctx* c, int64_t n, const float* a, const float* b, const float4* w_area,
                    cudaStream_t s) {
  if (c->red.n < 1) c->red.alloc(64);
  gemv_t(c, a, n, 1, n, b, w_area, c->red.get(), false, s);
  double h = 0;
  FMM_CUDA(cudaMemcpyAsync(&h, c->red.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  return h;
}

void apply_A(fmmbem_ctx* c, const float* x, float* y, cudaStream_t s);  // api.cu

fmmbem_status gmres_solve(fmmbem_ctx* c, const float* b, float* x, double tol, int m, int max_iters,
                          const float* x0, double* hist, int* iters, double* relres, cudaStream_t s) {
  const int64_t n = c->n_own();
  const int TB = 256;
  const int gb = std::max(1, ceil_div(n, TB));
  c->V.alloc(std::max<size_t>((size_t)(m + 1) * n, 1));
  c->w.alloc(std::max<int64_t>(n, 1));
  c->hd.alloc(m + 2);
  if (c->red.n < 2) c->red.alloc(64);
  float* V = c->V.get();
  float* w = c->w.get();
  double* hd = c->hd.get();
  auto norm2 = [&](const float* v, double* out) { gemv_t(c, v, n, 1, n, v, nullptr, out, false, s); };
  // ||b||
  norm2(b, c->red.get());
  double bn2 = 0;
  FMM_CUDA(cudaMemcpyAsync(&bn2, c->red.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  const double bn = std::sqrt(bn2);
  if (x0) FMM_CUDA(cudaMemcpyAsync(x, x0, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
  else FMM_CUDA(cudaMemsetAsync(x, 0, n * sizeof(float), s));
  int it = 0;
  if (hist) hist[0] = 1.0;
  *iters = 0;
  *relres = 1.0;
  if (bn == 0.0) {
    *relres = 0.0;
    return FMMBEM_OK;
  }
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), col(m + 2);
  bool first = !x0;
  double rel = 1.0;
  while (it < max_iters) {
    // r = b - A x  -> V[0]
    if (first) {
      FMM_CUDA(cudaMemcpyAsync(w, b, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
      first = false;
    } else {
      apply_A(c, x, V, s);  // V[0] as scratch for A x
      k_sub<<<gb, TB, 0, s>>>(w, b, V, n);
      FMM_CHECK_LAUNCH();
    }
    norm2(w, c->red.get());
    double beta2 = 0;
    FMM_CUDA(cudaMemcpyAsync(&beta2, c->red.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    double beta = std::sqrt(beta2);
    rel = beta / bn;
    if (rel <= tol) break;
    k_scale_to<<<gb, TB, 0, s>>>(V, w, n, c->red.get());
    FMM_CHECK_LAUNCH();
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    const int mm = std::min(m, max_iters - it);
    int k = 0;
    for (; k < mm; ++k) {
      apply_A(c, V + (size_t)k * n, w, s);
      // CGS2
      gemv_t(c, V, n, k + 1, n, w, nullptr, hd, false, s);
      k_gemv_n<<<gb, TB, 0, s>>>(w, V, n, k + 1, n, hd, -1.0);
      gemv_t(c, V, n, k + 1, n, w, nullptr, c->red.get(), false, s);
      k_gemv_n<<<gb, TB, 0, s>>>(w, V, n, k + 1, n, c->red.get(), -1.0);
      FMM_CHECK_LAUNCH();
      std::vector<double> h2(k + 1);
      FMM_CUDA(cudaMemcpyAsync(col.data(), hd, (k + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
      FMM_CUDA(cudaMemcpyAsync(h2.data(), c->red.get(), (k + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
      norm2(w, hd + k + 1);
      double nw2 = 0;
      FMM_CUDA(cudaMemcpyAsync(&nw2, hd + k + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
      k_scale_to<<<gb, TB, 0, s>>>(V + (size_t)(k + 1) * n, w, n, hd + k + 1);
      FMM_CHECK_LAUNCH();
      FMM_CUDA(cudaStreamSynchronize(s));
      for (int i = 0; i <= k; ++i) col[i] += h2[i];
      col[k + 1] = std::sqrt(nw2);
      // Givens
      for (int i = 0; i < k; ++i) {
        double t = cs[i] * col[i] + sn[i] * col[i + 1];
        col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
        col[i] = t;
      }
      double den = std::hypot(col[k], col[k + 1]);
      cs[k] = den > 0 ? col[k] / den : 1.0;
      sn[k] = den > 0 ? col[k + 1] / den : 0.0;
      col[k] = den;
      col[k + 1] = 0.0;
      for (int i = 0; i <= k; ++i) H[(size_t)i * m + k] = col[i];
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      ++it;
      rel = std::fabs(g[k + 1]) / bn;
      if (hist) hist[it] = rel;
      if (rel <= tol || nw2 == 0.0) {
        ++k;
        break;
      }
    }
    // y = H^-1 g ; x += V y
    std::vector<double> y(k);
    for (int i = k - 1; i >= 0; --i) {
      double t = g[i];
      for (int j = i + 1; j < k; ++j) t -= H[(size_t)i * m + j] * y[j];
      y[i] = t / H[(size_t)i * m + i];
    }
    FMM_CUDA(cudaMemcpyAsync(hd, y.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
    k_gemv_n<<<gb, TB, 0, s>>>(x, V, n, k, n, hd, 1.0);
    FMM_CHECK_LAUNCH();
    FMM_CUDA(cudaStreamSynchronize(s));
    if (rel <= tol) break;
  }
  *iters = it;
  *relres = rel;
  return rel <= tol ? FMMBEM_OK : FMMBEM_NOT_CONVERGED;
}

}  // namespace fmm
