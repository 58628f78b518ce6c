// farfield.cu -- multipole / local expansions (PAPER.md P:546-566:
// "The MEs are built first at the tree leaves (P2M) and then translated to the center of the
// parent cells (M2M) ... the MEs are first transformed into LEs for all the boxes in the
// interaction list (M2L) ... Each LE is then translated to the centers of all child cells
// (L2L) ... the far-field contribution comes from evaluating the LE of the cell at each point
// location (L2P)").
//
// Expansions are truncated after P terms (degrees 0..P-1; reading A9) in complex
// solid harmonics with the 1/(n+m)! normalisation (Condon-Shortley phase, all m):
//   R_n^m(r) = r^n P_n^m(cos t) e^{i m p} / (n+m)!,   I_n^m(r) = (n-m)! P_n^m(cos t) e^{i m p} / r^{n+1}
//   1/|x - y| = sum_{n,m} conj(R_n^m(y - c)) I_n^m(x - c)                       (|y-c| < |x-c|)
//   R_n^m(a + b) = sum_{j,k} R_j^k(a) R_{n-j}^{m-k}(b)
//   I_n^m(D + r) = sum_{j,k} (-1)^j conj(R_j^k(r)) I_{n+j}^{m+k}(D)             (|r| < |D|)
// Coefficients are scaled by the cell width w of their level:
//   M~_n^m = M_n^m / w^n,  L~_j^k = L_j^k w^{j+1}
// which makes every translation operator level independent:
//   P2M  M~_n^m   = sum_i q_i conj(R_n^m(u_i)),              u = (y - c)/w
//   M2M  M~_n^m(P) = sum_{j,k} 2^-j M~_j^k(C) conj(R_{n-j}^{m-k}(d)),   d = (c_C - c_P)/w_P in {+-1/4}^3
//   M2L  L~_j^k   = (-1)^{j+k} sum_{n,m} M~_n^m I_{j+n}^{m-k}(delta),    delta = (c_t - c_s)/w in Z^3
//   L2L  L~_j^k(C) = 2^-(j+1) sum_{n>=j,m} L~_n^m(P) R_{n-j}^{m-k}(d)
//   L2P  phi(x)   = (1/w) sum_{j,k} L~_j^k R_j^k(u),  grad phi = (1/w^2) sum L~_j^k grad R_j^k(u)
//        dz R_j^k = R_{j-1}^k,  dx R_j^k = (R_{j-1}^{k+1} - R_{j-1}^{k-1})/2,
//        dy R_j^k = -i (R_{j-1}^{k+1} + R_{j-1}^{k-1})/2
// Storage: m >= 0 only, index n(n+1)/2 + m, float2 (re, im); negative orders follow from
// X_n^{-m} = (-1)^m conj(X_n^m).  The kernels here are the generic O(P^4) translations, kept as
// the independent cross-check of the rotation-accelerated O(P^3) M2M / M2L / L2L of m2l_rot.cu
// that run by default, and as the fallback for orders without a rotation instantiation.
#include <cmath>
#include <complex>

#include "kernels.cuh"

namespace fmm {

namespace {

__constant__ float2 c_R8[8][MAX_TERMS * (MAX_TERMS + 1) / 2];  // R_n^m(d_octant)

__host__ __device__ inline int cidx(int n, int m) { return n * (n + 1) / 2 + m; }

__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ void cfma(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, fmaf(-a.y, b.y, acc.x));
  acc.y = fmaf(a.x, b.y, fmaf(a.y, b.x, acc.y));
}
// X_n^m for any m from m >= 0 storage
__device__ __forceinline__ float2 getc(const float2* X, int n, int m) {
  if (m >= 0) return X[cidx(n, m)];
  float2 v = X[cidx(n, -m)];
  return (m & 1) ? make_float2(-v.x, v.y) : make_float2(v.x, -v.y);
}

// ---------------------------------------------------------------- P2M
// CTA per leaf; thread (g, m): source group g (8 groups), order m (16 slots).
__global__ void __launch_bounds__(128) k_p2m(const float4* __restrict__ pos, const float* __restrict__ x, int div,
                                             const int* __restrict__ beg, int P, float inv_w, int leaf_off,
                                             int leaf0, float2* __restrict__ M) {
  __shared__ float2 sm[8][16][MAX_TERMS];
  const int leaf = leaf0 + blockIdx.x;
  const int b = beg[leaf], e = beg[leaf + 1];
  if (b == e) return;
  const int g = threadIdx.x >> 4, m = threadIdx.x & 15;
  float2 acc[MAX_TERMS];
#pragma unroll
  for (int k = 0; k < MAX_TERMS; ++k) acc[k] = make_float2(0.f, 0.f);
  if (m < P) {
    for (int j = b + g; j < e; j += 8) {
      float4 p = pos[j];
      float w = p.w;
      if (x) w *= x[div == 1 ? j : j / div];
      float ux = p.x * inv_w, uy = p.y * inv_w, uz = p.z * inv_w;
      float r2 = ux * ux + uy * uy + uz * uz;
      // R_m^m = (-(x+iy)/2)^m / m!
      float2 rmm = make_float2(1.f, 0.f);
      for (int k = 1; k <= m; ++k) {
        float s = -0.5f / k;
        rmm = make_float2(s * (rmm.x * ux - rmm.y * uy), s * (rmm.x * uy + rmm.y * ux));
      }
      float2 rm2 = make_float2(0.f, 0.f), rm1 = rmm;
#pragma unroll
      for (int k = 0; k < MAX_TERMS; ++k) {
        const int n = m + k;
        if (n < P) {
          float2 r;
          if (k == 0) r = rmm;
          else {
            float inv = 1.f / (float)((n - m) * (n + m));
            float a = (2 * n - 1) * uz;
            r = make_float2((a * rm1.x - r2 * rm2.x) * inv, (a * rm1.y - r2 * rm2.y) * inv);
            rm2 = rm1;
            rm1 = r;
          }
          // acc += w * conj(R)
          acc[k].x = fmaf(w, r.x, acc[k].x);
          acc[k].y = fmaf(-w, r.y, acc[k].y);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < MAX_TERMS; ++k) sm[g][m][k] = acc[k];
  __syncthreads();
  const int NC = P * (P + 1) / 2;
  for (int c = threadIdx.x; c < NC; c += blockDim.x) {
    int n = (int)((sqrtf(8.f * c + 1.f) - 1.f) * 0.5f);
    while (n * (n + 1) / 2 > c) --n;
    while ((n + 1) * (n + 2) / 2 <= c) ++n;
    int mm = c - n * (n + 1) / 2;
    float2 s = make_float2(0.f, 0.f);
    for (int gg = 0; gg < 8; ++gg) {
      s.x += sm[gg][mm][n - mm].x;
      s.y += sm[gg][mm][n - mm].y;
    }
    M[(size_t)(leaf_off + leaf) * NC + c] = s;
  }
}

// ---------------------------------------------------------------- M2M
// Mc / Mp: the child / parent level's expansions addressed by global cell index (ctx.h lvl_ptr)
__global__ void __launch_bounds__(64) k_m2m(int lvl_off, int P, const int* __restrict__ cb,
                                            const int* __restrict__ ce, const uint64_t* __restrict__ key,
                                            const int* __restrict__ scnt, const float2* __restrict__ Mc,
                                            float2* __restrict__ M) {
  extern __shared__ float2 smc[];  // [8][NC] children, then [8][NC] R(d_octant)
  __shared__ int oct[8];
  const int cell = lvl_off + blockIdx.x;
  const int NC = P * (P + 1) / 2;
  if (scnt[cell] == 0) return;
  float2* sR = smc + 8 * NC;
  for (int t = threadIdx.x; t < 8 * NC; t += blockDim.x) sR[t] = c_R8[t / NC][t % NC];
  const int c0 = cb[cell], nch = ce[cell] - c0;
  for (int t = threadIdx.x; t < nch * NC; t += blockDim.x) {
    int ch = t / NC, c = t - ch * NC;
    smc[ch * NC + c] = scnt[c0 + ch] ? Mc[(size_t)(c0 + ch) * NC + c] : make_float2(0.f, 0.f);
  }
  if (threadIdx.x < nch) oct[threadIdx.x] = (int)(key[c0 + threadIdx.x] & 7);
  __syncthreads();
  for (int c = threadIdx.x; c < NC; c += blockDim.x) {
    int n = 0;
    while ((n + 1) * (n + 2) / 2 <= c) ++n;
    const int m = c - n * (n + 1) / 2;
    float2 acc = make_float2(0.f, 0.f);
    for (int ch = 0; ch < nch; ++ch) {
      const float2* Mc = smc + ch * NC;
      const float2* R = sR + oct[ch] * NC;
      float sc = 1.f;
      for (int j = 0; j <= n; ++j, sc *= 0.5f) {
        const int nj = n - j;
        float2 part = make_float2(0.f, 0.f);
        const int klo = max(-j, m - nj), khi = min(j, m + nj);
        for (int k = klo; k <= khi; ++k) {
          float2 a = getc(Mc, j, k), r = getc(R, nj, m - k);
          float2 t = cmulc(a, r);
          part.x += t.x;
          part.y += t.y;
        }
        acc.x = fmaf(sc, part.x, acc.x);
        acc.y = fmaf(sc, part.y, acc.y);
      }
    }
    M[(size_t)cell * NC + c] = acc;
  }
}

// ---------------------------------------------------------------- M2L (O(P^4), all levels)
constexpr int M2L_TPB = 64;
constexpr int M2L_SB = 4;  // sources staged per step

// cmap: cell -> expansion slot (nullptr: slot = cell), ctx.h
__global__ void __launch_bounds__(M2L_TPB) k_m2l(int cell_off, int P, const long long* __restrict__ off,
                                                 const int* __restrict__ idx, const uint64_t* __restrict__ key,
                                                 const int* __restrict__ scnt, const int* __restrict__ tcnt,
                                                 const int* __restrict__ cmap, const float2* __restrict__ M,
                                                 const float2* __restrict__ Itab, float2* __restrict__ Lx) {
  extern __shared__ float2 sm[];
  const int NC = P * (P + 1) / 2, NF = P * P, NIF = (2 * P - 1) * (2 * P - 1);
  float2* Mf = sm;                    // [SB][NF]   full M~ (all m)
  float2* If = sm + M2L_SB * NF;      // [SB][NIF]  full I(delta)
  const int cell = cell_off + blockIdx.x;
  if (tcnt[cell] == 0) return;
  const long long lo = off[cell], hi = off[cell + 1];
  if (lo == hi) return;
  int tx, ty, tz;
  demorton(key[cell], tx, ty, tz);
  // outputs owned by this thread (up to 3 for P <= 16)
  float2 acc[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  for (long long e0 = lo; e0 < hi; e0 += M2L_SB) {
    const int ns = (int)min((long long)M2L_SB, hi - e0);
    __syncthreads();
    for (int q = 0; q < ns; ++q) {
      const int s = idx[e0 + q];
      float2* Mq = Mf + q * NF;
      float2* Iq = If + q * NIF;
      if (scnt[s] == 0) {
        for (int t = threadIdx.x; t < NF; t += M2L_TPB) Mq[t] = make_float2(0.f, 0.f);
        for (int t = threadIdx.x; t < NIF; t += M2L_TPB) Iq[t] = make_float2(0.f, 0.f);
        continue;
      }
      const float2* Ms = M + (size_t)(cmap ? cmap[s] : s) * NC;
      for (int t = threadIdx.x; t < NF; t += M2L_TPB) {
        int n = 0;
        while ((n + 1) * (n + 1) <= t) ++n;
        const int m = t - n * n - n;
        Mq[t] = getc(Ms, n, m);
      }
      int sx, sy, sz;
      demorton(key[s], sx, sy, sz);
      const int d = (tx - sx + 3) * 49 + (ty - sy + 3) * 7 + (tz - sz + 3);
      const float2* It = Itab + (size_t)d * NIF;
      for (int t = threadIdx.x; t < NIF; t += M2L_TPB) Iq[t] = It[t];
    }
    __syncthreads();
#pragma unroll
    for (int o = 0; o < 3; ++o) {
      const int c = threadIdx.x + o * M2L_TPB;
      if (c < NC) {
        int j = 0;
        while ((j + 1) * (j + 2) / 2 <= c) ++j;
        const int k = c - j * (j + 1) / 2;
        float2 a = acc[o];
        for (int q = 0; q < ns; ++q) {
          const float2* Mq = Mf + q * NF;
          const float2* Iq = If + q * NIF;
          for (int n = 0; n < P; ++n) {
            const int l = j + n;
            const float2* Irow = Iq + l * l + l - k;  // I_l^{m-k} at Irow[m]
            const float2* Mrow = Mq + n * n + n;      // M_n^m at Mrow[m]
            for (int m = -n; m <= n; ++m) cfma(a, Mrow[m], Irow[m]);
          }
        }
        acc[o] = a;
      }
    }
  }
#pragma unroll
  for (int o = 0; o < 3; ++o) {
    const int c = threadIdx.x + o * M2L_TPB;
    if (c < NC) {
      int j = 0;
      while ((j + 1) * (j + 2) / 2 <= c) ++j;
      const int k = c - j * (j + 1) / 2;
      const float sg = ((j + k) & 1) ? -1.f : 1.f;
      const size_t t = (size_t)(cmap ? cmap[cell] : cell) * NC + c;
      float2 v = Lx[t];
      v.x = fmaf(sg, acc[o].x, v.x);
      v.y = fmaf(sg, acc[o].y, v.y);
      Lx[t] = v;
    }
  }
}

// ---------------------------------------------------------------- L2L
// Lp / Lx: the parent / child level's local expansions addressed by global cell index (ctx.h lvl_ptr)
__global__ void __launch_bounds__(64) k_l2l(int lvl_off, int P, const int* __restrict__ parent,
                                            const uint64_t* __restrict__ key, const int* __restrict__ tcnt,
                                            const float2* __restrict__ Lp, float2* __restrict__ Lx) {
  extern __shared__ float2 sp[];  // parent L~ [NC], then R(d_octant) [NC]
  const int cell = lvl_off + blockIdx.x;
  if (tcnt[cell] == 0) return;
  const int NC = P * (P + 1) / 2;
  const int p = parent[cell];
  const int oc = (int)(key[cell] & 7);
  float2* R = sp + NC;
  for (int t = threadIdx.x; t < NC; t += blockDim.x) {
    sp[t] = Lp[(size_t)p * NC + t];
    R[t] = c_R8[oc][t];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < NC; c += blockDim.x) {
    int j = 0;
    while ((j + 1) * (j + 2) / 2 <= c) ++j;
    const int k = c - j * (j + 1) / 2;
    float2 acc = make_float2(0.f, 0.f);
    for (int n = j; n < P; ++n) {
      const int nj = n - j;
      const int mlo = max(-n, k - nj), mhi = min(n, k + nj);
      for (int m = mlo; m <= mhi; ++m) cfma(acc, getc(sp, n, m), getc(R, nj, m - k));
    }
    const float sc = ldexpf(1.f, -(j + 1));
    float2 v = Lx[(size_t)cell * NC + c];
    v.x = fmaf(sc, acc.x, v.x);
    v.y = fmaf(sc, acc.y, v.y);
    Lx[(size_t)cell * NC + c] = v;
  }
}

// ---------------------------------------------------------------- L2P
// CTA per leaf; 8 targets at a time, 16 lanes (orders m) per target, reduced by shuffles.
__global__ void __launch_bounds__(128) k_l2p(const float4* __restrict__ pos, const float4* __restrict__ nrm,
                                             const int* __restrict__ beg, int P, float inv_w, int leaf_off,
                                             int leaf0, const float2* __restrict__ Lx, OutArg pot, OutArg dn) {
  __shared__ float2 sl[MAX_TERMS * (MAX_TERMS + 1) / 2];
  const int leaf = leaf0 + blockIdx.x;
  const int b = beg[leaf], e = beg[leaf + 1];
  if (b == e) return;
  const int NC = P * (P + 1) / 2;
  for (int t = threadIdx.x; t < NC; t += blockDim.x) sl[t] = Lx[(size_t)(leaf_off + leaf) * NC + t];
  __syncthreads();
  const int m = threadIdx.x & 15;
  const float cm = (m == 0) ? 1.f : 2.f;
  for (int i0 = b; i0 < e; i0 += 8) {
    const int i = i0 + (threadIdx.x >> 4);
    const bool valid = i < e;
    float4 p = pos[valid ? i : b];
    float ux = p.x * inv_w, uy = p.y * inv_w, uz = p.z * inv_w;
    float r2 = ux * ux + uy * uy + uz * uz;
    float ph = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
    if (m < P) {
      float2 rmm = make_float2(1.f, 0.f);
      for (int k = 1; k <= m; ++k) {
        float s = -0.5f / k;
        rmm = make_float2(s * (rmm.x * ux - rmm.y * uy), s * (rmm.x * uy + rmm.y * ux));
      }
      float2 rm2 = make_float2(0.f, 0.f), r = rmm;
      for (int n = m; n < P; ++n) {
        if (n > m) {
          float inv = 1.f / (float)((n - m) * (n + m));
          float a = (2 * n - 1) * uz;
          float2 nr = make_float2((a * r.x - r2 * rm2.x) * inv, (a * r.y - r2 * rm2.y) * inv);
          rm2 = r;
          r = nr;
        }
        // phi += cm Re(L_n^m R_n^m)
        float2 Ln = sl[cidx(n, m)];
        ph += cm * (Ln.x * r.x - Ln.y * r.y);
        if (n + 1 < P) {
          float2 Lz = sl[cidx(n + 1, m)];
          gz += cm * (Lz.x * r.x - Lz.y * r.y);
          float2 Lm = getc(sl, n + 1, m - 1), Lp = sl[cidx(n + 1, m + 1)];
          // dx: Re(R (Lm - Lp)/2) ; dy: Re(-i/2 R (Lm + Lp)) = Im(R (Lm + Lp))/2
          float2 dmn = make_float2(Lm.x - Lp.x, Lm.y - Lp.y), sum = make_float2(Lm.x + Lp.x, Lm.y + Lp.y);
          gx += cm * 0.5f * (r.x * dmn.x - r.y * dmn.y);
          gy += cm * 0.5f * (r.x * sum.y + r.y * sum.x);
        }
      }
    }
#pragma unroll
    for (int d = 8; d > 0; d >>= 1) {
      ph += __shfl_xor_sync(0xffffffffu, ph, d);
      gx += __shfl_xor_sync(0xffffffffu, gx, d);
      gy += __shfl_xor_sync(0xffffffffu, gy, d);
      gz += __shfl_xor_sync(0xffffffffu, gz, d);
    }
    if (valid && m == 0) {
      if (pot.y) pot.y[i] += pot.b * ph * inv_w;
      if (dn.y) {
        float4 nn = nrm[i];
        dn.y[i] += dn.b * (nn.x * gx + nn.y * gy + nn.z * gz) * inv_w * inv_w;
      }
    }
  }
}

// ---------------------------------------------------------------- host tables (FP64)
using cd = std::complex<double>;

void host_R(int P, double x, double y, double z, std::vector<cd>& R) {  // m >= 0, cidx
  R.assign(P * (P + 1) / 2, 0.0);
  double r2 = x * x + y * y + z * z;
  cd rmm = 1.0;
  for (int m = 0; m < P; ++m) {
    if (m > 0) rmm *= cd(-x, -y) / (2.0 * m);
    cd r1 = rmm, r0 = 0.0;
    R[cidx(m, m)] = rmm;
    for (int n = m + 1; n < P; ++n) {
      cd rn = ((2.0 * n - 1) * z * r1 - r2 * r0) / double((n - m) * (n + m));
      R[cidx(n, m)] = rn;
      r0 = r1;
      r1 = rn;
    }
  }
}

void host_I(int Pn, double x, double y, double z, std::vector<cd>& I) {  // degrees < Pn, m >= 0
  I.assign(Pn * (Pn + 1) / 2, 0.0);
  double r2 = x * x + y * y + z * z, ir2 = 1.0 / r2;
  cd imm = 1.0 / std::sqrt(r2);
  for (int m = 0; m < Pn; ++m) {
    if (m > 0) imm *= -(2.0 * m - 1) * cd(x, y) * ir2;
    cd i1 = imm, i0 = 0.0;
    I[cidx(m, m)] = imm;
    for (int n = m + 1; n < Pn; ++n) {
      cd in = ((2.0 * n - 1) * z * i1 - double((n + m - 1) * (n - m - 1)) * i0) * ir2;
      I[cidx(n, m)] = in;
      i0 = i1;
      i1 = in;
    }
  }
}

}  // namespace

void init_tables(fmmbem_ctx* c) {
  const int P = c->P;
  // octant shifts d = (c_child - c_parent)/w_parent
  float2 h8[8][MAX_TERMS * (MAX_TERMS + 1) / 2] = {};
  std::vector<cd> R;
  for (int o = 0; o < 8; ++o) {
    double dx = (o & 1) ? 0.25 : -0.25, dy = (o & 2) ? 0.25 : -0.25, dz = (o & 4) ? 0.25 : -0.25;
    host_R(P, dx, dy, dz, R);
    for (size_t t = 0; t < R.size(); ++t) h8[o][t] = make_float2((float)R[t].real(), (float)R[t].imag());
  }
  FMM_CUDA(cudaMemcpyToSymbol(c_R8, h8, sizeof(h8)));
  // irregular harmonics of every integer offset in [-3, 3]^3, full m range, degrees < 2P-1
  const int Pn = 2 * P - 1, NIF = Pn * Pn;
  std::vector<float2> tab((size_t)343 * NIF, make_float2(0.f, 0.f));
  std::vector<cd> I;
  for (int a = -3; a <= 3; ++a)
    for (int b = -3; b <= 3; ++b)
      for (int g = -3; g <= 3; ++g) {
        if (std::abs(a) <= 1 && std::abs(b) <= 1 && std::abs(g) <= 1) continue;
        host_I(Pn, a, b, g, I);
        float2* row = tab.data() + (size_t)((a + 3) * 49 + (b + 3) * 7 + (g + 3)) * NIF;
        for (int n = 0; n < Pn; ++n)
          for (int m = -n; m <= n; ++m) {
            cd v = I[cidx(n, std::abs(m))];
            if (m < 0) v = ((-m) & 1 ? -1.0 : 1.0) * std::conj(v);
            row[n * n + n + m] = make_float2((float)v.real(), (float)v.imag());
          }
      }
  c->Itab.alloc(tab.size());
  FMM_CUDA(cudaMemcpy(c->Itab.get(), tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
  c->NI = NIF;
}

// leaf-level kernels address the leaves [lo, hi) through the rank's leaf window (ctx.h)
void check_leaf_window(const fmmbem_ctx* c, int lo, int hi) {
  const Tree& T = c->tree;
  const int64_t a = T.lvl_off[T.L] + lo, b = T.lvl_off[T.L] + hi;
  if (hi > lo && (a < c->win_lo[T.L] || b > c->win_hi[T.L]))
    throw Error(FMMBEM_E_INVALID, "leaf range outside this rank's expansion window");
}

void launch_p2m_range(fmmbem_ctx* c, const SrcArg& s, int lo, int hi, cudaStream_t st) {
  const Tree& T = c->tree;
  const int L = T.L, P = c->P;
  if (L < 2 || hi <= lo) return;
  const PointSet& S = *s.set;
  check_leaf_window(c, lo, hi);
  float2* M = c->lvl_ptr(c->Mx.get(), L);
  if (exp_specialised(P)) {
    launch_p2m_t(P, hi - lo, S.pos.get(), s.x, S.div, S.begin.get(), (float)(1.0 / T.width(L)), (int)T.lvl_off[L],
                 lo, M, st);
  } else {
    k_p2m<<<hi - lo, 128, 0, st>>>(S.pos.get(), s.x, S.div, S.begin.get(), P, (float)(1.0 / T.width(L)),
                                   (int)T.lvl_off[L], lo, M);
    FMM_CHECK_LAUNCH();
  }
}

void launch_upward(fmmbem_ctx* c, const SrcArg& s, cudaStream_t st) {
  const Tree& T = c->tree;
  if (T.L < 2) return;
  c->Mx.zero(st);
  launch_p2m_range(c, s, s.leaf_lo, s.leaf_hi < 0 ? (int)T.n_leaves : s.leaf_hi, st);
  launch_m2m_levels(c, s, st);
}

void launch_m2m_levels(fmmbem_ctx* c, const SrcArg& s, cudaStream_t st) {
  const Tree& T = c->tree;
  const int L = T.L, P = c->P, NC = c->NC;
  if (L < 2) return;
  const int* cnt = s.cnt ? s.cnt : s.set->cell_cnt.get();
  const bool rot = c->m2l_mode == 0 && m2m_rot_supported(P);
  if (rot) init_rot_tables();
  for (int l = L - 1; l >= 2; --l) {  // the parents of this rank's window
    if (rot) {  // Lx is free during the upward sweep: scratch for the per-child translations
      launch_m2m_rot(c, l, cnt, c->Lx.get(), st);
      continue;
    }
    const int n = (int)(c->win_hi[l] - c->win_lo[l]);
    if (n <= 0) continue;
    k_m2m<<<n, 64, 16 * NC * sizeof(float2), st>>>((int)c->win_lo[l], P, T.child_begin.get(), T.child_end.get(),
                                                   T.key.get(), cnt, c->lvl_ptr(c->Mx.get(), l + 1),
                                                   c->lvl_ptr(c->Mx.get(), l));
    FMM_CHECK_LAUNCH();
  }
}

void launch_m2l(fmmbem_ctx* c, const int* src_cnt, const int* tgt_cnt, cudaStream_t st) {
  const Tree& T = c->tree;
  const int L = T.L, P = c->P;
  if (L < 2) return;
  c->Lx.zero(st);
  if (c->m2l_mode == 0 && rot_supported(P)) {
    init_rot_tables();
    launch_m2l_rot(c, m2l_work(c, src_cnt, tgt_cnt, st), st);
    return;
  }
  const int n = (int)(T.n_cells - T.lvl_off[2]);
  const size_t smem = (size_t)M2L_SB * (P * P + (2 * P - 1) * (2 * P - 1)) * sizeof(float2);
  static bool attr = false;
  if (!attr) {
    FMM_CUDA(cudaFuncSetAttribute(k_m2l, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    attr = true;
  }
  k_m2l<<<n, M2L_TPB, smem, st>>>((int)T.lvl_off[2], P, T.m2l_off.get(), T.m2l_idx.get(), T.key.get(), src_cnt,
                                   tgt_cnt, c->slot_map(), c->Mx.get(), c->Itab.get(), c->Lx.get());
  FMM_CHECK_LAUNCH();
}

void launch_downward(fmmbem_ctx* c, const int* tgt_cnt, cudaStream_t st) {
  const Tree& T = c->tree;
  const int L = T.L, P = c->P, NC = c->NC;
  if (L < 2) return;
  const bool rot = c->m2l_mode == 0 && m2m_rot_supported(P);
  if (rot) init_rot_tables();
  for (int l = 2; l < L; ++l) {
    if (rot) {
      launch_l2l_rot(c, l, tgt_cnt, st);
      continue;
    }
    const int n = (int)(c->win_hi[l + 1] - c->win_lo[l + 1]);  // the children in this rank's window
    if (n <= 0) continue;
    k_l2l<<<n, 64, 2 * NC * sizeof(float2), st>>>((int)c->win_lo[l + 1], P, T.parent.get(), T.key.get(), tgt_cnt,
                                                  c->lvl_ptr(c->Lx.get(), l), c->lvl_ptr(c->Lx.get(), l + 1));
    FMM_CHECK_LAUNCH();
  }
}

void launch_l2p(fmmbem_ctx* c, const TgtArg& t, const Outputs& o, cudaStream_t st) {
  const Tree& T = c->tree;
  const int L = T.L;
  if (L < 2) return;
  const PointSet& S = *t.set;
  const int lo = t.leaf_lo, hi = t.leaf_hi < 0 ? (int)T.n_leaves : t.leaf_hi;
  if (hi <= lo) return;
  check_leaf_window(c, lo, hi);
  const float2* Lw = c->lvl_ptr(c->Lx.get(), L);
  if (exp_specialised(c->P)) {
    launch_l2p_t(c->P, hi - lo, S.pos.get(), S.nrm.get(), S.begin.get(), (float)(1.0 / T.width(L)),
                 (int)T.lvl_off[L], lo, Lw, o.pot, o.dn, st);
    return;
  }
  k_l2p<<<hi - lo, 128, 0, st>>>(S.pos.get(), S.nrm.get(), S.begin.get(), c->P, (float)(1.0 / T.width(L)),
                                 (int)T.lvl_off[L], lo, Lw, o.pot, o.dn);
  FMM_CHECK_LAUNCH();
}

}  // namespace fmm
