// p2p.cu -- near-field direct sums ("the near field
// contribution is obtained from directly computing the interactions between all the points
// in the adjacent cells", "P2P ... the largest fractions").
//
// Work unit = one warp = one chunk of <= 64 targets of one leaf (T = 4 targets per lane in
// registers as two packed FP32x2 pairs; measured at C5: T = 6 / 8 or 128-target chunks are slower).
// The normal-derivative sums (K', A) use the scaled-coordinate form (interact2s, 11 instead of 12
// packed instructions per pair of interactions, -2.8 % at C5).  Surface leaves hold a variable number of targets, so a leaf is cut into chunks
// and a tail chunk with few targets spreads its lanes over S source subsets (split-K, reduced in
// shared memory) -- lanes stay busy whatever the occupancy.  The sources of the (<= 27)
// neighbour leaves stream through a warp-private shared-memory tile, already shifted into the
// target leaf's frame: offsets between leaf centres are exact multiples of the leaf width
// (FP32-exact), so s - x subtracts two numbers of leaf size only.  All lanes of a
// subset read the same source (broadcast LDS.128).  Outputs are owned by one lane (no atomics,
// fixed summation order -> bitwise reproducible).  Only the chunk's own sources are masked (j != i of
// the discrete operator).
//
// Raw outputs, un-normalised potential phi = sum_j w_j / r_ij:
//   pot = phi(x_i),   dn = n_i . grad phi(x_i) = n_i . sum_j w_j (y_j - x_i) / r^3
// Per interaction (dn only): 3 FADD + 3 (r^2) + 1 MUFU.RSQ + 3 (w r^-3) + 3 FFMA = 12 FP32 operations +
// 1 MUFU, counted as 19 flops under the SURVEY 8(d) convention; issued as packed FP32x2 instructions
// over the lane's two targets (6 issue slots + 1 MUFU per interaction).
#include "kernels.cuh"

namespace fmm {

namespace {

#ifndef P2P_TILE
#define P2P_TILE 256
#endif
#ifndef P2P_UNROLL
#define P2P_UNROLL 16
#endif
#define P2P_PRAGMA(x) _Pragma(#x)
#define P2P_UNROLL_LOOP(n) P2P_PRAGMA(unroll n)
constexpr int TILE = P2P_TILE;   // sources per warp tile (256 with unroll 16 measured fastest: 128 / 512 tiles, unroll 4 / 8 / 32 slower)
constexpr int MAXSEG = 32;

struct P2PArgs {
  const int4* items;  // (leaf, first target, target count, 0)
  int n_items;
  int* counter;       // work-item counter of the persistent launch (zeroed before it)
  const float4* tpos;
  const float4* tnrm;
  const int* tbeg;
  const float4* spos;
  const float4* ssc;  // scaled form: per-source (a s, a) prepared by k_scale_src (SC kernels only)
  const unsigned* wmax;  // scaled form: bits of the max |weight| the table was normalised by (k_absmax)
  const float* sx;
  int sdiv;
  const int* sbeg;
  const int* sleaf;
  int ns;
  const int* nbr_off;
  const int* nbr_idx;
  const int4* ijk;
  float h;
  int direct;
  OutArg pot, dn;
  int* flag;
};

__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }

// exponent e of the scaled-form weight normalisation: 2^e > max |w| (k_absmax / k_scale_src)
__device__ __forceinline__ int wmax_exp(unsigned bits) {
  const float m = __uint_as_float(bits);
  return m > 0.f ? ilogbf(m) + 1 : 0;
}

// One source against the lane's two targets with packed FP32x2 arithmetic (FADD2/FMUL2/FFMA2 on
// sm_100a; the scalar source coordinate is a broadcast operand): 12 packed instructions + 2 MUFU.RSQ
// for 2 interactions.  d = s - x (source minus target), so grad phi = sum w d / r^3.
template <bool POT, bool DN, bool MASK, bool CHECK>
__device__ __forceinline__ void interact2(const float4 s, float2 px, float2 py, float2 pz, float2& ap, float2& gx,
                                          float2& gy, float2& gz, bool skipa, bool skipb, int* flag) {
  const float2 dx = __fadd2_rn(bc2(s.x), px), dy = __fadd2_rn(bc2(s.y), py), dz = __fadd2_rn(bc2(s.z), pz);
  float2 r2 = __fmul2_rn(dx, dx);
  r2 = __ffma2_rn(dy, dy, r2);
  r2 = __ffma2_rn(dz, dz, r2);
  float2 w = bc2(s.w);
  if (CHECK) {
    if (r2.x == 0.f || r2.y == 0.f) atomicOr(flag, 1);
  }
  if (MASK) {
    w = make_float2(skipa ? 0.f : s.w, skipb ? 0.f : s.w);
    r2 = make_float2(fmaxf(r2.x, 1e-20f), fmaxf(r2.y, 1e-20f));
  }
  const float2 ri = make_float2(rsqrtf(r2.x), rsqrtf(r2.y));
  if (POT) ap = __ffma2_rn(w, ri, ap);
  if (DN) {
    float2 t = __fmul2_rn(w, ri);
    t = __fmul2_rn(t, __fmul2_rn(ri, ri));
    gx = __ffma2_rn(t, dx, gx);
    gy = __ffma2_rn(t, dy, gy);
    gz = __ffma2_rn(t, dz, gz);
  }
}

// Scaled form for the normal-derivative-only sum (the K' / A matvec): the tile holds (a s, a) with
// a = sign(w) |w|^(-1/2), so d' = a (s - x) = fma(a, -x, a s), r'^2 = a^2 r^2 and
// (r'^-2)^(3/2) d' = sign(w) d / (a^2 r^3) = w d / r^3: 11 packed FP32x2 instructions + 2 MUFU.RSQ
// per 2 interactions (12 in the plain form).  A zero weight becomes a source at 1e18 with a = 1
// (its r'^-3 flushes to zero).  a comes from MUFU.RSQ: relative error ~2^-22 per source weight.
template <bool MASK>
__device__ __forceinline__ void interact2s(const float4 s, float2 px, float2 py, float2 pz, float2& gx, float2& gy,
                                           float2& gz, bool skipa, bool skipb) {
  const float2 dx = __ffma2_rn(bc2(s.w), px, bc2(s.x)), dy = __ffma2_rn(bc2(s.w), py, bc2(s.y)),
               dz = __ffma2_rn(bc2(s.w), pz, bc2(s.z));
  float2 r2 = __fmul2_rn(dx, dx);
  r2 = __ffma2_rn(dy, dy, r2);
  r2 = __ffma2_rn(dz, dz, r2);
  float2 ri = make_float2(rsqrtf(r2.x), rsqrtf(r2.y));
  if (MASK) ri = make_float2(skipa ? 0.f : ri.x, skipb ? 0.f : ri.y);
  const float2 t = __fmul2_rn(__fmul2_rn(ri, ri), ri);
  gx = __ffma2_rn(t, dx, gx);
  gy = __ffma2_rn(t, dy, gy);
  gz = __ffma2_rn(t, dz, gz);
}

template <int T, bool POT, bool DN, bool SELF, bool CHECK, bool SC = false, int MINB = 28>
__global__ void __launch_bounds__(32, MINB) k_p2p(P2PArgs a) {
  constexpr int TL = TILE;
  static_assert(!SC || (DN && !POT && !CHECK), "scaled form: normal derivative only");
  __shared__ float4 tile[TL];
  __shared__ int own[SELF ? TL : 1];
  __shared__ int seg_src[MAXSEG], seg_cum[MAXSEG + 1];
  __shared__ float4 seg_sh[MAXSEG];
  static_assert(4 * T * 32 * sizeof(float) <= sizeof(float4) * TL, "split-K scratch aliases the tile");
  float(*red)[32] = reinterpret_cast<float(*)[32]>(tile);  // used only after the source loop

  // persistent warps: a grid of (SMs x resident warps) one-warp blocks claims the work items in
  // order from a global counter, so no warp slot waits for a block launch; every item is still
  // computed whole by one warp (outputs written once, deterministic)
  const int lane = threadIdx.x;
  int wexp = 0;
  if (SC) wexp = wmax_exp(*a.wmax);
  int item;
  {
    int v = 0;
    if (lane == 0) v = atomicAdd(a.counter, 1);
    item = __shfl_sync(0xffffffffu, v, 0);
  }
  for (; item < a.n_items;) {
  const int4 it = a.items[item];
  const int leaf = it.x, tb = it.y, nt = it.z;
  const int4 tc = a.ijk[leaf];

  // ---- source segments: neighbour leaves (self last) or, in direct mode, everything
  int n_src, self_lo, self_hi, nseg = 0;
  if (!a.direct) {
    const int o = a.nbr_off[leaf], nn = a.nbr_off[leaf + 1] - o;
    int s = -1, cnt = 0, beg = 0;
    const bool valid = lane < nn;
    if (valid) {
      s = a.nbr_idx[o + lane];
      beg = a.sbeg[s];
      cnt = a.sbeg[s + 1] - beg;
    }
    const bool is_self = valid && s == leaf;
    const unsigned vmask = __ballot_sync(0xffffffffu, valid && !is_self);
    const int rank = is_self ? __popc(vmask) : __popc(vmask & ((1u << lane) - 1));
    if (valid) {
      seg_src[rank] = beg;
      int4 sc = a.ijk[s];
      seg_sh[rank] = make_float4((sc.x - tc.x) * a.h, (sc.y - tc.y) * a.h, (sc.z - tc.z) * a.h, 0.f);
      seg_cum[rank + 1] = cnt;
    }
    __syncwarp();
    int incl = (lane < nn) ? seg_cum[lane + 1] : 0;
    __syncwarp();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    if (lane < nn) seg_cum[lane + 1] = incl;
    if (lane == 0) seg_cum[0] = 0;
    __syncwarp();
    nseg = nn;
    n_src = seg_cum[nn];
    if (SELF) {  // only the chunk's own sources j / sdiv in [tb, tb + nt) need the j != i mask
      self_lo = seg_cum[nn - 1] + (tb * a.sdiv - seg_src[nn - 1]);
      self_hi = self_lo + nt * a.sdiv;
    } else {
      self_lo = self_hi = n_src;
    }
  } else {
    n_src = a.ns;
    self_lo = tb * a.sdiv;
    self_hi = (tb + nt) * a.sdiv;
  }

  // ---- lane mapping: tl-th target slot, source subset sub of S
  const int nl_t = (nt + T - 1) / T;          // lanes needed per subset (<= 32)
  const int S = 32 / nl_t;                    // source subsets
  const int tl = lane % nl_t, sub = lane / nl_t;
  const bool lvalid = sub < S;
  static_assert(T % 2 == 0, "packed FP32x2 path: pairs of targets per lane");
  constexpr int NP = T / 2;
  int ti[T];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const int il = tl + k * nl_t;
    ti[k] = tb + (il < nt ? il : 0);
  }
  // negated target coordinates of each packed pair: s + (-x) with a broadcast source operand
  float2 px[NP], py[NP], pz[NP], ap2[NP], gx2[NP], gy2[NP], gz2[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const float4 ta = a.tpos[ti[2 * q]], tb4 = a.tpos[ti[2 * q + 1]];
    px[q] = make_float2(-ta.x, -tb4.x);
    py[q] = make_float2(-ta.y, -tb4.y);
    pz[q] = make_float2(-ta.z, -tb4.z);
    ap2[q] = gx2[q] = gy2[q] = gz2[q] = make_float2(0.f, 0.f);
  }
  const int step = lvalid ? S : 0;
  // per-lane segment cursor of the tile fill: lane l fills v = base + l + 32 q, increasing over the
  // whole kernel, so the segment holding v only ever advances (no per-source search)
  int cur = 0, nxt = 0, jb = 0;
  float4 shv = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!a.direct) {
    nxt = seg_cum[1];
    jb = seg_src[0];
    shv = seg_sh[0];
  }

  for (int base = 0; base < n_src; base += TL) {
    const int tcnt = min(TL, n_src - base);
    __syncwarp();
#pragma unroll
    for (int q = 0; q < TL / 32; ++q) {
      const int k = lane + 32 * q;
      if (k < tcnt) {
        const int v = base + k;
        int j;
        float sx, sy, sz;
        if (!a.direct) {
          if (v >= nxt) {  // v < n_src = seg_cum[nseg]: stops at a segment of the list
            do {
              ++cur;
              nxt = seg_cum[cur + 1];
            } while (v >= nxt);
            jb = seg_src[cur] - seg_cum[cur];
            shv = seg_sh[cur];
          }
          j = jb + v;
          sx = shv.x; sy = shv.y; sz = shv.z;
        } else {
          j = v;
          const int4 sc = a.ijk[a.sleaf[j]];
          sx = (sc.x - tc.x) * a.h; sy = (sc.y - tc.y) * a.h; sz = (sc.z - tc.z) * a.h;
        }
        if (SC) {  // (a s, a) from k_scale_src: shift into the target leaf's frame, a (s + sh)
          const float4 p = __ldg(a.ssc + j);
          tile[k] = make_float4(fmaf(p.w, sx, p.x), fmaf(p.w, sy, p.y), fmaf(p.w, sz, p.z), p.w);
        } else {
          const float4 p = __ldg(a.spos + j);
          float w = p.w;
          if (a.sx) w *= __ldg(a.sx + (a.sdiv == 1 ? j : j / a.sdiv));
          tile[k] = make_float4(p.x + sx, p.y + sy, p.z + sz, w);
        }
        if (SELF) own[k] = (a.sdiv == 1) ? j : j / a.sdiv;
      }
    }
    __syncwarp();
    if (!lvalid) continue;
    const int mlo = SELF ? min(max(self_lo - base, 0), tcnt) : tcnt;
    const int mhi = SELF ? min(max(self_hi - base, 0), tcnt) : tcnt;
    // unmasked: [0, mlo) and [mhi, tcnt)
P2P_UNROLL_LOOP(P2P_UNROLL)
    for (int k = sub; k < mlo; k += step) {
      const float4 sv = tile[k];
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        if (SC) interact2s<false>(sv, px[q], py[q], pz[q], gx2[q], gy2[q], gz2[q], false, false);
        else interact2<POT, DN, false, CHECK>(sv, px[q], py[q], pz[q], ap2[q], gx2[q], gy2[q], gz2[q], false, false,
                                              a.flag);
      }
    }
    if (SELF) {
      int k0 = mhi + ((sub - mhi) % S + S) % S;
P2P_UNROLL_LOOP(P2P_UNROLL)
      for (int k = k0; k < tcnt; k += step) {
        const float4 sv = tile[k];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          if (SC) interact2s<false>(sv, px[q], py[q], pz[q], gx2[q], gy2[q], gz2[q], false, false);
          else interact2<POT, DN, false, CHECK>(sv, px[q], py[q], pz[q], ap2[q], gx2[q], gy2[q], gz2[q], false,
                                                false, a.flag);
        }
      }
      int k1 = mlo + ((sub - mlo) % S + S) % S;
#pragma unroll 4
      for (int k = k1; k < mhi; k += step) {
        const int o = own[k];
        const float4 sv = tile[k];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          if (SC) interact2s<true>(sv, px[q], py[q], pz[q], gx2[q], gy2[q], gz2[q], o == ti[2 * q], o == ti[2 * q + 1]);
          else interact2<POT, DN, true, CHECK>(sv, px[q], py[q], pz[q], ap2[q], gx2[q], gy2[q], gz2[q],
                                               o == ti[2 * q], o == ti[2 * q + 1], a.flag);
        }
      }
    }
  }
  float ap[T], gx[T], gy[T], gz[T];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    ap[2 * q] = ap2[q].x; ap[2 * q + 1] = ap2[q].y;
    gx[2 * q] = gx2[q].x; gx[2 * q + 1] = gx2[q].y;
    gy[2 * q] = gy2[q].x; gy[2 * q + 1] = gy2[q].y;
    gz[2 * q] = gz2[q].x; gz[2 * q + 1] = gz2[q].y;
  }
  // ---- split-K reduction over the S subsets
  if (S > 1) {
    __syncwarp();  // every lane is done reading the tile
#pragma unroll
    for (int q = 0; q < T; ++q) {
      red[4 * q + 0][lane] = ap[q];
      red[4 * q + 1][lane] = gx[q];
      red[4 * q + 2][lane] = gy[q];
      red[4 * q + 3][lane] = gz[q];
    }
    __syncwarp();
    if (sub == 0) {
      for (int g = 1; g < S; ++g) {
#pragma unroll
        for (int q = 0; q < T; ++q) {
          ap[q] += red[4 * q + 0][g * nl_t + tl];
          gx[q] += red[4 * q + 1][g * nl_t + tl];
          gy[q] += red[4 * q + 2][g * nl_t + tl];
          gz[q] += red[4 * q + 3][g * nl_t + tl];
        }
      }
    }
  }
  if (sub == 0) {
#pragma unroll
    for (int q = 0; q < T; ++q) {
      if (tl + q * nl_t >= nt) continue;
      const int i = ti[q];
      if (POT) {
        float v = a.pot.b * ap[q];
        if (a.pot.x) v = fmaf(a.pot.ax, a.pot.x[i], v);
        if (a.pot.acc) v = __fadd_rn(v, a.pot.y[i]);
        a.pot.y[i] = v;
      }
      if (DN) {
        const float4 n = a.tnrm[i];
        float g = fmaf(n.x, gx[q], fmaf(n.y, gy[q], n.z * gz[q]));
        if (SC) g = ldexpf(g, wexp);  // undo the power-of-two normalisation of the weights
        float v = a.dn.b * g;
        if (a.dn.x) v = fmaf(a.dn.d ? fmaf(a.dn.b, a.dn.d[i], a.dn.ax) : a.dn.ax, a.dn.x[i], v);
        if (a.dn.acc) v = __fadd_rn(v, a.dn.y[i]);
        a.dn.y[i] = v;
      }
    }
  }
  __syncwarp();  // shared memory of this item is free
  int v = 0;
  if (lane == 0) v = atomicAdd(a.counter, 1);
  item = __shfl_sync(0xffffffffu, v, 0);
  }
}

// T = 4 targets per lane: two packed FP32x2 pairs per shared-memory source load (a 64-register cap
// for full block residency measured 0.5% faster -- not worth a second instantiation)
constexpr int P2P_T = 4;

template <bool SELF, bool CHECK>
void dispatch(const P2PArgs& a, bool pot, bool dn, bool scaled, bool occ, int grid, cudaStream_t st) {
  if (pot && dn) k_p2p<P2P_T, true, true, SELF, CHECK><<<grid, 32, 0, st>>>(a);
  else if (pot) k_p2p<P2P_T, true, false, SELF, CHECK><<<grid, 32, 0, st>>>(a);
  else if (scaled && !CHECK && occ) k_p2p<P2P_T, false, true, SELF, false, true, 32><<<grid, 32, 0, st>>>(a);
  else if (scaled && !CHECK) k_p2p<P2P_T, false, true, SELF, false, true><<<grid, 32, 0, st>>>(a);
  else k_p2p<P2P_T, false, true, SELF, CHECK><<<grid, 32, 0, st>>>(a);
}

// Scaled-form source table for one matvec: a = sign(w') |w'|^(-1/2) with w' = 2^-e (A_j w_g) x_j,
// stored as (a y, a) in leaf-local coordinates (see interact2s).  2^e is the power of two at or
// above max |w| (k_absmax), so |w'| <= 1 whatever the scale of x: r'^2 = r^2 / |w'| and
// r'^-3 = |w'|^(3/2) r^-3 stay inside FP32 (with -ftz a weight below ~1e-25 max|w| contributes 0,
// a relative change far below FP32 rounding of the sum); the P2P epilogue multiplies by 2^e.
// A zero weight becomes a source at 1e18 with a = 1 (its r'^-3 flushes to zero); the shift
// a * (leaf offset) added in the fill keeps it there.
// bits of max_j |pos_j.w x_j / div| (non-negative floats order like their bit patterns)
__global__ void k_absmax(int64_t n, const float4* __restrict__ spos, const float* __restrict__ sx, int sdiv,
                         unsigned* out) {
  float m = 0.f;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    float w = __ldg(&spos[j].w);
    if (sx) w *= __ldg(sx + (sdiv == 1 ? j : j / sdiv));
    m = fmaxf(m, fabsf(w));
  }
  for (int d = 16; d > 0; d >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, d));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}

__global__ void k_scale_src(int64_t n, const float4* __restrict__ spos, const float* __restrict__ sx, int sdiv,
                            const unsigned* __restrict__ wmax, float4* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int e = wmax_exp(*wmax);
  const float4 p = __ldg(spos + j);
  float w = p.w;
  if (sx) w *= __ldg(sx + (sdiv == 1 ? j : j / sdiv));
  w = ldexpf(w, -e);
  float4 r;
  if (w == 0.f) {
    r = make_float4(1e18f, 1e18f, 1e18f, 1.f);
  } else {
    const float sc = copysignf(rsqrtf(fabsf(w)), w);
    r = make_float4(sc * p.x, sc * p.y, sc * p.z, sc);
  }
  out[j] = r;
}

__global__ void k_count(int nl, int lo, const int* __restrict__ tbeg, const int* __restrict__ sbeg,
                        const int* __restrict__ off, const int* __restrict__ idx, int direct, int ns,
                        unsigned long long* out) {
  int k = lo + blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0;
  if (k < lo + nl) {
    long long nt = tbeg[k + 1] - tbeg[k];
    long long s = 0;
    if (direct) s = ns;
    else
      for (int e = off[k]; e < off[k + 1]; ++e) s += sbeg[idx[e] + 1] - sbeg[idx[e]];
    c = (unsigned long long)(nt * s);
  }
  for (int d = 16; d > 0; d >>= 1) c += __shfl_down_sync(0xffffffffu, c, d);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void k_item_count(int nl, const int* __restrict__ tbeg, int chunk, int* cnt) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nl) cnt[k] = (tbeg[k + 1] - tbeg[k] + chunk - 1) / chunk;
}

__global__ void k_item_fill(int nl, const int* __restrict__ tbeg, int leaf0, int chunk,
                            const int* __restrict__ pos, int4* items) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nl) return;
  const int b = tbeg[k], e = tbeg[k + 1];
  int w = pos[k];
  for (int t = b; t < e; t += chunk) items[w++] = make_int4(leaf0 + k, t, min(chunk, e - t), 0);
}

}  // namespace

// (leaf, target chunk) work items of one target set, built once and cached
const P2PItems& p2p_items(fmmbem_ctx* c, const PointSet& t, int leaf_lo, int leaf_hi, int chunk) {
  for (auto& w : c->p2p_cache)
    if (w->tgt == &t && w->leaf_lo == leaf_lo && w->leaf_hi == leaf_hi && w->chunk == chunk) return *w;
  const int nl = leaf_hi - leaf_lo;
  cudaStream_t st = c->stream;
  auto w = std::make_unique<P2PItems>();
  w->tgt = &t;
  w->leaf_lo = leaf_lo;
  w->leaf_hi = leaf_hi;
  w->chunk = chunk;
  DevBuf<int> cnt, pos;
  cnt.alloc(nl + 1);
  pos.alloc(nl + 1);
  cnt.zero(st);
  if (nl > 0) k_item_count<<<ceil_div(nl, 256), 256, 0, st>>>(nl, t.begin.get() + leaf_lo, chunk, cnt.get());
  FMM_CHECK_LAUNCH();
  scan_ints(cnt.get(), pos.get(), nl + 1, st);
  int n = 0;
  FMM_CUDA(cudaMemcpyAsync(&n, pos.get() + nl, sizeof(int), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  w->n = n;
  w->items.alloc(std::max(1, n));
  if (nl > 0)
    k_item_fill<<<ceil_div(nl, 256), 256, 0, st>>>(nl, t.begin.get() + leaf_lo, leaf_lo, chunk, pos.get(),
                                                    w->items.get());
  FMM_CHECK_LAUNCH();
  FMM_CUDA(cudaStreamSynchronize(st));
  c->p2p_cache.push_back(std::move(w));
  return *c->p2p_cache.back();
}

const float4* prepare_p2p_sources(fmmbem_ctx* c, const SrcArg& s, cudaStream_t st) {
  const int64_t n = s.set->n;
  if ((int64_t)c->p2p_src.n < n) c->p2p_src.alloc(n);
  if (c->p2p_wmax.n < 1) c->p2p_wmax.alloc(1);
  FMM_CUDA(cudaMemsetAsync(c->p2p_wmax.get(), 0, sizeof(unsigned), st));
  if (n > 0)
    k_absmax<<<std::min<int64_t>(4 * 148, ceil_div(n, 256)), 256, 0, st>>>(n, s.set->pos.get(), s.x, s.set->div,
                                                                          c->p2p_wmax.get());
  // several ranks: the normalisation exponent of the WHOLE source vector (max over ranks of the
  // non-negative float bits), so the scaled coordinates -- and the product -- do not depend on the
  // partition (a rank-local exponent changes a = sign(w)/sqrt(|w|/2^e) by sqrt 2 and with it the
  // rounding of the scaled form: 4e-6 relative at 4 ranks on C3)
  if (c->nranks > 1 && s.halo_src) comm_allreduce_u32_max(c, c->p2p_wmax.get(), 1, st, /*second=*/true);
  if (n > 0)
    k_scale_src<<<ceil_div(n, 256), 256, 0, st>>>(n, s.set->pos.get(), s.x, s.set->div, c->p2p_wmax.get(),
                                                   c->p2p_src.get());
  FMM_CHECK_LAUNCH();
  return c->p2p_src.get();
}

void launch_p2p(fmmbem_ctx* c, const TgtArg& t, const SrcArg& s, const Outputs& o, bool self, bool check,
                bool direct, cudaStream_t st) {
  const Tree& T = c->tree;
  const bool pot = o.pot.y != nullptr, dn = o.dn.y != nullptr;
  if (!pot && !dn) return;
  const P2PItems& items =
      p2p_items(c, *t.set, t.leaf_lo, t.leaf_hi < 0 ? (int)c->tree.n_leaves : t.leaf_hi,
                s.set == &c->chg ? c->p2p_chunk_chg : c->p2p_chunk);
  if (items.n == 0) return;
  P2PArgs a{};
  a.items = items.items.get();
  a.n_items = (int)items.n;
  if (c->p2p_counter.n < 1) c->p2p_counter.alloc(1);
  FMM_CUDA(cudaMemsetAsync(c->p2p_counter.get(), 0, sizeof(int), st));
  a.counter = c->p2p_counter.get();
  a.tpos = t.set->pos.get();
  a.tnrm = t.set->nrm.get();
  a.tbeg = t.set->begin.get();
  a.spos = s.set->pos.get();
  a.sx = s.x;
  a.sdiv = s.set->div;
  a.sbeg = s.set->begin.get();
  a.sleaf = s.set->leaf.get();
  a.ns = (int)s.set->n;
  a.nbr_off = T.nbr_off.get();
  a.nbr_idx = T.nbr_idx.get();
  a.ijk = T.leaf_ijk.get();
  a.h = (float)T.width(T.L);
  a.direct = direct ? 1 : 0;
  a.pot = o.pot;
  a.dn = o.dn;
  a.flag = c->flag.get();
  if (dn && !a.tnrm) throw Error(FMMBEM_E_INVALID, "normal derivative requested at targets without normals");
  static const int n_sm = [] {
    int d = 0, v = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return v > 0 ? v : 148;
  }();
  const int grid = (int)std::min<int64_t>(items.n, (int64_t)n_sm * 32);  // 32 one-warp blocks per SM
  const bool sc = c->p2p_scaled != 0 && dn && !pot && !check;
  if (sc) {
    a.ssc = s.scaled;
    if (!a.ssc) a.ssc = prepare_p2p_sources(c, s, st);
    a.wmax = c->p2p_wmax.get();
  }
  if (self) {
    if (check) dispatch<true, true>(a, pot, dn, sc, c->p2p_occ != 0, grid, st);
    else dispatch<true, false>(a, pot, dn, sc, c->p2p_occ != 0, grid, st);
  } else {
    if (check) dispatch<false, true>(a, pot, dn, sc, c->p2p_occ != 0, grid, st);
    else dispatch<false, false>(a, pot, dn, sc, c->p2p_occ != 0, grid, st);
  }
  FMM_CHECK_LAUNCH();
}

int64_t count_p2p(fmmbem_ctx* c, const PointSet& t, const PointSet& s, bool self, bool direct, int leaf_lo,
                  int leaf_hi) {
  const Tree& T = c->tree;
  DevBuf<unsigned long long> out;
  out.alloc(1);
  out.zero(c->stream);
  if (leaf_hi < 0) leaf_hi = (int)T.n_leaves;
  const int nl = leaf_hi - leaf_lo;
  if (nl > 0)
    k_count<<<ceil_div(nl, 256), 256, 0, c->stream>>>(nl, leaf_lo, t.begin.get(), s.begin.get(), T.nbr_off.get(),
                                                       T.nbr_idx.get(), direct ? 1 : 0, (int)s.n, out.get());
  FMM_CHECK_LAUNCH();
  unsigned long long h = 0;
  int tb[2] = {0, 0};
  FMM_CUDA(cudaMemcpyAsync(&h, out.get(), sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  FMM_CUDA(cudaMemcpyAsync(&tb[0], t.begin.get() + leaf_lo, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  FMM_CUDA(cudaMemcpyAsync(&tb[1], t.begin.get() + leaf_hi, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  FMM_CUDA(cudaStreamSynchronize(c->stream));
  int64_t r = (int64_t)h;
  if (self) r -= (int64_t)(tb[1] - tb[0]) * s.div;  // own-panel pairs are excluded (j != i)
  return r;
}

}  // namespace fmm
