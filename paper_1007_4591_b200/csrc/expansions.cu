// expansions.cu -- P2M and L2P specialised on the expansion order P (
// formulas in farfield.cu's header).  One warp per leaf.
//
// P2M: lane l owns the sources j = b + l, b + l + 32, ...; the regular solid harmonics of a
// source are generated one order column m at a time (R_m^m by the diagonal recurrence, then
// R_n^m = ((2n-1) u_z R_{n-1}^m - r^2 R_{n-2}^m) / ((n-m)(n+m)) with compile-time reciprocals), so
// only one column of accumulators is live.  Per-lane partial sums go to a private shared-memory
// slot and are reduced over lanes (fixed order, no atomics).
// L2P: lane = target; the leaf's local expansion sits in shared memory (every lane reads the
// same coefficient -> broadcast); potential and gradient accumulate column by column.
#include "kernels.cuh"

namespace fmm {

namespace {

__host__ __device__ constexpr int cx(int n, int m) { return n * (n + 1) / 2 + m; }

// one order column m of the P2M sums of this lane's sources into the lane's slot
template <int P, int m>
__device__ __forceinline__ void p2m_column(float* slot, const float4* __restrict__ pos, const float* __restrict__ x,
                                           int div, int b, int e, int lane, float inv_w) {
  float ar[P - m], ai[P - m];
#pragma unroll
  for (int k = 0; k < P - m; ++k) ar[k] = ai[k] = 0.f;
  for (int j = b + lane; j < e; j += 32) {
    const float4 p = __ldg(pos + j);
    float w = p.w;
    if (x) w *= __ldg(x + (div == 1 ? j : j / div));
    const float ux = p.x * inv_w, uy = p.y * inv_w, uz = p.z * inv_w;
    const float r2 = fmaf(ux, ux, fmaf(uy, uy, uz * uz));
    float rr = 1.f, ri = 0.f;  // R_m^m = (-(x + i y)/2)^m / m!
#pragma unroll
    for (int k = 1; k <= m; ++k) {
      const float s = -0.5f / (float)k;
      const float t = (rr * ux - ri * uy) * s;
      ri = (rr * uy + ri * ux) * s;
      rr = t;
    }
    float pr = 0.f, pi = 0.f, cr = rr, ci = ri;
    ar[0] = fmaf(w, cr, ar[0]);
    ai[0] = fmaf(-w, ci, ai[0]);
#pragma unroll
    for (int n = m + 1; n < P; ++n) {
      const float inv = 1.f / (float)((n - m) * (n + m));
      const float a = (float)(2 * n - 1) * inv * uz, bb = r2 * inv;
      const float nr = a * cr - bb * pr, ni = a * ci - bb * pi;
      pr = cr;
      pi = ci;
      cr = nr;
      ci = ni;
      ar[n - m] = fmaf(w, cr, ar[n - m]);
      ai[n - m] = fmaf(-w, ci, ai[n - m]);
    }
  }
#pragma unroll
  for (int n = m; n < P; ++n) {
    slot[(2 * cx(n, m)) * 33] = ar[n - m];
    slot[(2 * cx(n, m) + 1) * 33] = ai[n - m];
  }
  if constexpr (m + 1 < P) p2m_column<P, m + 1>(slot, pos, x, div, b, e, lane, inv_w);
}

template <int P>
__global__ void __launch_bounds__(32) k_p2m_t(const float4* __restrict__ pos, const float* __restrict__ x, int div,
                                              const int* __restrict__ beg, float inv_w, int leaf_off, int leaf0,
                                              float2* __restrict__ M) {
  constexpr int NC = P * (P + 1) / 2;
  __shared__ float sv[2 * NC * 33];
  const int leaf = leaf0 + blockIdx.x;
  const int b = beg[leaf], e = beg[leaf + 1];
  if (b == e) return;
  const int lane = threadIdx.x;
  p2m_column<P, 0>(sv + lane, pos, x, div, b, e, lane, inv_w);
  __syncwarp();
  for (int c = lane; c < NC; c += 32) {
    float sx = 0.f, sy = 0.f;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) {
      sx += sv[(2 * c) * 33 + l];
      sy += sv[(2 * c + 1) * 33 + l];
    }
    M[(size_t)(leaf_off + leaf) * NC + c] = make_float2(sx, sy);
  }
}

template <int P>
__global__ void __launch_bounds__(32) k_l2p_t(const float4* __restrict__ pos, const float4* __restrict__ nrm,
                                              const int* __restrict__ beg, float inv_w, int leaf_off, int leaf0,
                                              const float2* __restrict__ Lx, OutArg pot, OutArg dn) {
  constexpr int NC = P * (P + 1) / 2;
  __shared__ float2 sl[NC + 1];
  const int leaf = leaf0 + blockIdx.x;
  const int b = beg[leaf], e = beg[leaf + 1];
  if (b == e) return;
  const int lane = threadIdx.x;
  for (int c = lane; c < NC; c += 32) sl[c] = Lx[(size_t)(leaf_off + leaf) * NC + c];
  if (lane == 0) sl[NC] = make_float2(0.f, 0.f);
  __syncwarp();
  const bool want_pot = pot.y != nullptr, want_dn = dn.y != nullptr;
  for (int i = b + lane; i < e; i += 32) {
    const float4 p = pos[i];
    const float ux = p.x * inv_w, uy = p.y * inv_w, uz = p.z * inv_w;
    const float r2 = fmaf(ux, ux, fmaf(uy, uy, uz * uz));
    float ph = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
    float dr = 1.f, di = 0.f;
#pragma unroll
    for (int m = 0; m < P; ++m) {
      if (m > 0) {
        const float s = -0.5f / (float)m;
        const float t = (dr * ux - di * uy) * s;
        di = (dr * uy + di * ux) * s;
        dr = t;
      }
      const float cm = (m == 0) ? 1.f : 2.f;
      float pr = 0.f, pi = 0.f, cr = dr, ci = di;
#pragma unroll
      for (int n = m; n < P; ++n) {
        if (n > m) {
          const float inv = 1.f / (float)((n - m) * (n + m));
          const float a = (float)(2 * n - 1) * inv * uz, bb = r2 * inv;
          const float nr = a * cr - bb * pr, ni = a * ci - bb * pi;
          pr = cr;
          pi = ci;
          cr = nr;
          ci = ni;
        }
        const float2 Ln = sl[cx(n, m)];
        ph = fmaf(cm, Ln.x * cr - Ln.y * ci, ph);
        if (n + 1 < P) {
          const float2 Lz = sl[cx(n + 1, m)];
          gz = fmaf(cm, Lz.x * cr - Lz.y * ci, gz);
          float2 Lm;
          if (m == 0) {  // L_{n+1}^{-1} = -conj(L_{n+1}^1)
            const float2 t = sl[cx(n + 1, 1)];
            Lm = make_float2(-t.x, t.y);
          } else {
            Lm = sl[cx(n + 1, m - 1)];
          }
          const float2 Lp = sl[cx(n + 1, m + 1)];
          const float dmr = Lm.x - Lp.x, dmi = Lm.y - Lp.y, smr = Lm.x + Lp.x, smi = Lm.y + Lp.y;
          gx = fmaf(0.5f * cm, cr * dmr - ci * dmi, gx);
          gy = fmaf(0.5f * cm, cr * smi + ci * smr, gy);
        }
      }
    }
    if (want_pot) pot.y[i] += pot.b * ph * inv_w;
    if (want_dn) {
      const float4 nn = nrm[i];
      dn.y[i] += dn.b * (nn.x * gx + nn.y * gy + nn.z * gz) * inv_w * inv_w;
    }
  }
}

}  // namespace

bool exp_specialised(int P) { return P == 8 || P == 10 || P == 12 || P == 14; }

void launch_p2m_t(int P, int grid, const float4* pos, const float* x, int div, const int* beg, float inv_w,
                  int leaf_off, int leaf0, float2* M, cudaStream_t st) {
  if (grid <= 0) return;
  switch (P) {
    case 8: k_p2m_t<8><<<grid, 32, 0, st>>>(pos, x, div, beg, inv_w, leaf_off, leaf0, M); break;
    case 10: k_p2m_t<10><<<grid, 32, 0, st>>>(pos, x, div, beg, inv_w, leaf_off, leaf0, M); break;
    case 12: k_p2m_t<12><<<grid, 32, 0, st>>>(pos, x, div, beg, inv_w, leaf_off, leaf0, M); break;
    case 14: k_p2m_t<14><<<grid, 32, 0, st>>>(pos, x, div, beg, inv_w, leaf_off, leaf0, M); break;
    default: throw Error(FMMBEM_E_INVALID, "P2M not specialised for this P");
  }
  FMM_CHECK_LAUNCH();
}

void launch_l2p_t(int P, int grid, const float4* pos, const float4* nrm, const int* beg, float inv_w, int leaf_off,
                  int leaf0, const float2* Lx, const OutArg& pot, const OutArg& dn, cudaStream_t st) {
  if (grid <= 0) return;
  switch (P) {
    case 8: k_l2p_t<8><<<grid, 32, 0, st>>>(pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn); break;
    case 10: k_l2p_t<10><<<grid, 32, 0, st>>>(pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn); break;
    case 12: k_l2p_t<12><<<grid, 32, 0, st>>>(pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn); break;
    case 14: k_l2p_t<14><<<grid, 32, 0, st>>>(pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn); break;
    default: throw Error(FMMBEM_E_INVALID, "L2P not specialised for this P");
  }
  FMM_CHECK_LAUNCH();
}

}  // namespace fmm
