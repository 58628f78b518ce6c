// expansions.cu -- P2M and L2P specialised on the expansion order P (
// formulas in farfield.cu's header).  One warp per leaf.
//
// P2M: lane l owns the sources j = b + l, b + l + 32, ...; the regular solid harmonics of a
// source are generated two order columns at a time (R_m^m carried from the previous pass by one
// diagonal step, then R_n^m = ((2n-1) u_z R_{n-1}^m - r^2 R_{n-2}^m) / ((n-m)(n+m)) with
// compile-time reciprocals), so only two columns of accumulators are live.  Per-lane partial sums go to a private shared-memory
// slot and are reduced over lanes (fixed order, no atomics).
// L2P: lane = target; the leaf's local expansion sits in shared memory (every lane reads the
// same coefficient -> broadcast); potential and gradient accumulate column by column.
#include "kernels.cuh"

namespace fmm {

namespace {

__host__ __device__ constexpr int cx(int n, int m) { return n * (n + 1) / 2 + m; }

#ifndef P2M_TILE_N
#define P2M_TILE_N 128
#endif
constexpr int P2M_TILE = P2M_TILE_N;  // sources staged per pass (C5, P = 13: 128 -> 6.30 ms, 256 -> 7.18, 64 -> 8.6)

// accumulate column m of w conj(R_n^m(u)), n = m..P-1, into a[] (re, im packed), starting from the
// column's diagonal R_m^m(u) = (cr, ci)
template <int P, int m>
__device__ __forceinline__ void column_acc(float2 (&a)[P - m], float4 u, float r2, float cr, float ci) {
  float pr = 0.f, pi = 0.f;
  const float2 nw = make_float2(u.w, -u.w);
  a[0] = __ffma2_rn(nw, make_float2(cr, ci), a[0]);
#pragma unroll
  for (int n = m + 1; n < P; ++n) {
    const float inv = 1.f / (float)((n - m) * (n + m));
    const float aa = (float)(2 * n - 1) * inv * u.z, bb = r2 * inv;
    const float nr = aa * cr - bb * pr, ni = aa * ci - bb * pi;
    pr = cr;
    pi = ci;
    cr = nr;
    ci = ni;
    a[n - m] = __ffma2_rn(nw, make_float2(cr, ci), a[n - m]);
  }
}

// R_{k+1}^{k+1} = R_k^k (-(x + i y) / 2) / (k + 1)
template <int k>
__device__ __forceinline__ void diag_step(float ux, float uy, float& rr, float& ri) {
  constexpr float s = -0.5f / (float)(k + 1);
  const float t = (rr * ux - ri * uy) * s;
  ri = (rr * uy + ri * ux) * s;
  rr = t;
}

__host__ __device__ constexpr int p2m_half(int P) { return (P + 1) / 2; }

// Pass m: columns m and m2 = m + H (H = ceil(P/2); the last pass of odd P has column m alone).
// Each source's two diagonals R_m^m, R_m2^m2 live in the lane-private shared slot dg[j] and
// advance by one order per pass (one complex multiply each instead of recomputing m steps).  The
// lanes' partial sums are transposed through red[][33] and lane c (< entries) adds the 32 partials
// of entry c to its register accumulator acc[m] (fixed order, no atomics).
template <int P, int m>
__device__ __forceinline__ void p2m_columns(float2 (&acc)[p2m_half(P)], float2* red, const float4* src, float4* dg,
                                            int ns, int lane) {
  constexpr int H = p2m_half(P);
  constexpr int m2 = m + H;
  constexpr bool single = m2 >= P;
  constexpr int NB = single ? 1 : P - m2;
  constexpr bool last = (m + 1 == H);
  float2 a[P - m], b[NB];
#pragma unroll
  for (int k = 0; k < P - m; ++k) a[k] = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < NB; ++k) b[k] = make_float2(0.f, 0.f);
  for (int j = lane; j < ns; j += 32) {
    const float4 u = src[j];
    float4 d = dg[j];
    const float r2 = fmaf(u.x, u.x, fmaf(u.y, u.y, u.z * u.z));
    column_acc<P, m>(a, u, r2, d.x, d.y);
    if constexpr (!single) column_acc<P, (single ? m : m2)>(b, u, r2, d.z, d.w);
    if constexpr (!last) {
      diag_step<m>(u.x, u.y, d.x, d.y);
      if constexpr (!single && m2 + 1 < P) diag_step<(single ? m : m2)>(u.x, u.y, d.z, d.w);
      dg[j] = d;
    }
  }
#pragma unroll
  for (int k = 0; k < P - m; ++k) red[k * 33 + lane] = a[k];
  if constexpr (!single) {
#pragma unroll
    for (int k = 0; k < P - m2; ++k) red[(P - m + k) * 33 + lane] = b[k];
  }
  __syncwarp();
  constexpr int NE = single ? P - m : 2 * P - m - m2;
  if (lane < NE) {
    float2 s0 = make_float2(0.f, 0.f), s1 = s0;
#pragma unroll
    for (int l = 0; l < 32; l += 2) {
      s0 = __fadd2_rn(s0, red[lane * 33 + l]);
      s1 = __fadd2_rn(s1, red[lane * 33 + l + 1]);
    }
    acc[m] = __fadd2_rn(acc[m], __fadd2_rn(s0, s1));
  }
  __syncwarp();
  if constexpr (!last) p2m_columns<P, m + 1>(acc, red, src, dg, ns, lane);
}

// P2M, one warp per leaf: the leaf's sources are scaled into the cell frame and staged in shared
// memory once (u = (y - c)/w, weight) with their starting diagonals (R_0^0 = 1, R_H^H), then every
// lane accumulates its sources' columns in registers (two columns at a time for ILP) and the column
// pair is reduced over the lanes at once, so shared memory stays small (occupancy) whatever P.
// 28 resident blocks: 72 registers (32 B of spills), P2M 6.31 -> 6.10 ms at C5 (1: 104 registers,
// 7.5 ms; plain bounds: 80 registers, 6.3 ms; 32: 64 registers + 116 B spills, 6.3 ms)
#ifndef P2M_MINB
#define P2M_MINB 28
#endif
#define P2M_BOUNDS __launch_bounds__(32, P2M_MINB)
template <int P>
__global__ void P2M_BOUNDS k_p2m_t(const float4* __restrict__ pos, const float* __restrict__ x, int div,
                                              const int* __restrict__ beg, float inv_w, int leaf_off, int leaf0,
                                              float2* __restrict__ M) {
  constexpr int NC = P * (P + 1) / 2;
  constexpr int H = p2m_half(P);  // passes: columns (m, m + H)
  constexpr int NEMAX = 2 * P - H;
  __shared__ float2 red[NEMAX * 33];
  __shared__ float4 src[P2M_TILE];
  __shared__ float4 dg[P2M_TILE];
  const int leaf = leaf0 + blockIdx.x;
  const int b = beg[leaf], e = beg[leaf + 1];
  if (b == e) return;
  const int lane = threadIdx.x;
  float2 acc[H];
#pragma unroll
  for (int k = 0; k < H; ++k) acc[k] = make_float2(0.f, 0.f);
  for (int t0 = b; t0 < e; t0 += P2M_TILE) {
    const int ns = min(P2M_TILE, e - t0);
    __syncwarp();
    for (int k = lane; k < ns; k += 32) {  // lane k % 32 stages exactly the sources it accumulates
      const int j = t0 + k;
      const float4 p = __ldg(pos + j);
      float w = p.w;
      if (x) w *= __ldg(x + (div == 1 ? j : j / div));
      const float ux = p.x * inv_w, uy = p.y * inv_w;
      src[k] = make_float4(ux, uy, p.z * inv_w, w);
      float hr = 1.f, hi = 0.f;  // R_H^H
#pragma unroll
      for (int q = 1; q <= H; ++q) {
        const float sc = -0.5f / (float)q;
        const float t = (hr * ux - hi * uy) * sc;
        hi = (hr * uy + hi * ux) * sc;
        hr = t;
      }
      dg[k] = make_float4(1.f, 0.f, hr, hi);
    }
    __syncwarp();
    p2m_columns<P, 0>(acc, red, src, dg, ns, lane);
  }
  if (lane < NEMAX) {
    float2* Mo = M + (size_t)(leaf_off + leaf) * NC;
#pragma unroll
    for (int m = 0; m < H; ++m) {
      const int m2 = m + H;
      const int ne = m2 < P ? 2 * P - m - m2 : P - m;
      if (lane >= ne) continue;
      // entry lane: (n = m + lane, m) for lane < P - m, else (n = m2 + lane - (P - m), m2)
      const int n = lane < P - m ? m + lane : m2 + lane - (P - m);
      const int mm = lane < P - m ? m : m2;
      Mo[cx(n, mm)] = acc[m];
    }
  }
}

// L2P, one warp per leaf, lane = target.  Everything that does not depend on the target is done
// once per leaf: the warp turns the leaf's local expansion into coefficient pairs for the
// potential and the three gradient components (grad of sum L_n^m R_n^m lowers the degree:
// d/dz -> L_{n+1}^m, d/dx -/+ i d/dy -> L_{n+1}^{m-1}, L_{n+1}^{m+1}), stored as
//   gxy[c] = (X.re, Y.re, X.im, Y.im),  zph[c] = (Z.re, Phi.re, Z.im, Phi.im)
// so that per target and coefficient (cr + i ci) = R_n^m(u) the update is
//   (gx, gy) += (X.re, Y.re) cr + (X.im, Y.im) ci,  (gz, ph) += (Z.re, Phi.re) cr + (Z.im, Phi.im) ci
// -- four packed FP32x2 FMAs; the recurrence for R_n^m is packed over (re, im) as well.
#ifndef L2P_NT
#define L2P_NT 1
#endif
template <int P, bool POT, bool DN>
__global__ void __launch_bounds__(32) k_l2p_t(const float4* __restrict__ pos, const float4* __restrict__ nrm,
                                              const int* __restrict__ beg, float inv_w, int leaf_off, int leaf0,
                                              const float2* __restrict__ Lx, OutArg pot, OutArg dn) {
  constexpr int NC = P * (P + 1) / 2;
  __shared__ float2 sl[NC];
  __shared__ float4 gxy[NC], zph[NC];
  const int leaf = leaf0 + blockIdx.x;
  const int b = beg[leaf], e = beg[leaf + 1];
  if (b == e) return;
  const int lane = threadIdx.x;
  for (int c = lane; c < NC; c += 32) sl[c] = Lx[(size_t)(leaf_off + leaf) * NC + c];
  __syncwarp();
  for (int c = lane; c < NC; c += 32) {
    int n = 0;
    while (cx(n + 1, 0) <= c) ++n;
    const int m = c - cx(n, 0);
    const float cm = (m == 0) ? 1.f : 2.f;
    const float2 Ln = sl[c];
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f), z = make_float4(0.f, cm * Ln.x, 0.f, -cm * Ln.y);
    if (n + 1 < P) {
      const float2 Lz = sl[cx(n + 1, m)];
      float2 Lm;
      if (m == 0) {  // L_{n+1}^{-1} = -conj(L_{n+1}^1)
        const float2 t = sl[cx(n + 1, 1)];
        Lm = make_float2(-t.x, t.y);
      } else {
        Lm = sl[cx(n + 1, m - 1)];
      }
      const float2 Lp = sl[cx(n + 1, m + 1)];
      // gx += 0.5 cm Re((dmr + i dmi)(cr + i ci)), gy += 0.5 cm (cr smi + ci smr)
      g = make_float4(0.5f * cm * (Lm.x - Lp.x), 0.5f * cm * (Lm.y + Lp.y), -0.5f * cm * (Lm.y - Lp.y),
                      0.5f * cm * (Lm.x + Lp.x));
      z.x = cm * Lz.x;
      z.z = -cm * Lz.y;
    }
    gxy[c] = g;
    zph[c] = z;
  }
  __syncwarp();
  // NT targets per lane (L2P_NT, default 1): the table reads are shared by the lane's targets
  constexpr int NT = L2P_NT;
  for (int i0 = b + lane; i0 < e; i0 += 32 * NT) {
    float ux[NT], uy[NT], uz[NT], r2[NT], dr[NT], di[NT];
    float2 gxy2[NT], gzph[NT];
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const int i = min(i0 + 32 * q, e - 1);
      const float4 p = pos[i];
      ux[q] = p.x * inv_w;
      uy[q] = p.y * inv_w;
      uz[q] = p.z * inv_w;
      r2[q] = fmaf(ux[q], ux[q], fmaf(uy[q], uy[q], uz[q] * uz[q]));
      gxy2[q] = make_float2(0.f, 0.f);
      gzph[q] = make_float2(0.f, 0.f);
      dr[q] = 1.f;
      di[q] = 0.f;
    }
#pragma unroll
    for (int m = 0; m < P; ++m) {
      asm volatile("" ::: "memory");  // re-read the tables per column (without: 168 registers, 1.1 KB spills)
      float2 cur[NT], prev[NT];
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        if (m > 0) {
          const float s = -0.5f / (float)m;
          const float t = (dr[q] * ux[q] - di[q] * uy[q]) * s;
          di[q] = (dr[q] * uy[q] + di[q] * ux[q]) * s;
          dr[q] = t;
        }
        cur[q] = make_float2(dr[q], di[q]);
        prev[q] = make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int n = m; n < P; ++n) {
        if (n > m) {
          const float inv = 1.f / (float)((n - m) * (n + m));
#pragma unroll
          for (int q = 0; q < NT; ++q) {
            const float a = (float)(2 * n - 1) * inv * uz[q], bb = r2[q] * inv;
            const float2 nxt = __ffma2_rn(make_float2(a, a), cur[q], __fmul2_rn(make_float2(-bb, -bb), prev[q]));
            prev[q] = cur[q];
            cur[q] = nxt;
          }
        }
        const int c = cx(n, m);
        if (DN && n + 1 < P) {
          const float4 g = gxy[c];
#pragma unroll
          for (int q = 0; q < NT; ++q) {
            gxy2[q] = __ffma2_rn(make_float2(g.x, g.y), make_float2(cur[q].x, cur[q].x), gxy2[q]);
            gxy2[q] = __ffma2_rn(make_float2(g.z, g.w), make_float2(cur[q].y, cur[q].y), gxy2[q]);
          }
        }
        if (POT || (DN && n + 1 < P)) {
          const float4 z = zph[c];
#pragma unroll
          for (int q = 0; q < NT; ++q) {
            gzph[q] = __ffma2_rn(make_float2(z.x, z.y), make_float2(cur[q].x, cur[q].x), gzph[q]);
            gzph[q] = __ffma2_rn(make_float2(z.z, z.w), make_float2(cur[q].y, cur[q].y), gzph[q]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const int i = i0 + 32 * q;
      if (i >= e) break;
      if (POT) pot.y[i] += pot.b * gzph[q].y * inv_w;
      if (DN) {
        const float4 nn = nrm[i];
        dn.y[i] += dn.b * (nn.x * gxy2[q].x + nn.y * gxy2[q].y + nn.z * gzph[q].x) * inv_w * inv_w;
      }
    }
  }
}

template <int P>
void l2p_dispatch(int grid, const float4* pos, const float4* nrm, const int* beg, float inv_w, int leaf_off, int leaf0,
                  const float2* Lx, const OutArg& pot, const OutArg& dn, cudaStream_t st) {
  const bool wp = pot.y != nullptr, wd = dn.y != nullptr;
  if (wp && wd) k_l2p_t<P, true, true><<<grid, 32, 0, st>>>(pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn);
  else if (wp) k_l2p_t<P, true, false><<<grid, 32, 0, st>>>(pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn);
  else if (wd) k_l2p_t<P, false, true><<<grid, 32, 0, st>>>(pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn);
}

}  // namespace

bool exp_specialised(int P) { return P == 8 || P == 10 || P == 12 || P == 13 || P == 14; }

void launch_p2m_t(int P, int grid, const float4* pos, const float* x, int div, const int* beg, float inv_w,
                  int leaf_off, int leaf0, float2* M, cudaStream_t st) {
  if (grid <= 0) return;
  switch (P) {
    case 8: k_p2m_t<8><<<grid, 32, 0, st>>>(pos, x, div, beg, inv_w, leaf_off, leaf0, M); break;
    case 10: k_p2m_t<10><<<grid, 32, 0, st>>>(pos, x, div, beg, inv_w, leaf_off, leaf0, M); break;
    case 12: k_p2m_t<12><<<grid, 32, 0, st>>>(pos, x, div, beg, inv_w, leaf_off, leaf0, M); break;
    case 13: k_p2m_t<13><<<grid, 32, 0, st>>>(pos, x, div, beg, inv_w, leaf_off, leaf0, M); break;
    case 14: k_p2m_t<14><<<grid, 32, 0, st>>>(pos, x, div, beg, inv_w, leaf_off, leaf0, M); break;
    default: throw Error(FMMBEM_E_INVALID, "P2M not specialised for this P");
  }
  FMM_CHECK_LAUNCH();
}

void launch_l2p_t(int P, int grid, const float4* pos, const float4* nrm, const int* beg, float inv_w, int leaf_off,
                  int leaf0, const float2* Lx, const OutArg& pot, const OutArg& dn, cudaStream_t st) {
  if (grid <= 0) return;
  switch (P) {
    case 8: l2p_dispatch<8>(grid, pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn, st); break;
    case 10: l2p_dispatch<10>(grid, pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn, st); break;
    case 12: l2p_dispatch<12>(grid, pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn, st); break;
    case 13: l2p_dispatch<13>(grid, pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn, st); break;
    case 14: l2p_dispatch<14>(grid, pos, nrm, beg, inv_w, leaf_off, leaf0, Lx, pot, dn, st); break;
    default: throw Error(FMMBEM_E_INVALID, "L2P not specialised for this P");
  }
  FMM_CHECK_LAUNCH();
}

}  // namespace fmm
