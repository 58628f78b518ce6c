// m2l_rot.cu -- rotation-accelerated M2L, O(P^3) per translation ("spherical
// harmonic rotations are performed before each translation at O(p^3) cost").
//
// For a source cell s and target cell t at offset delta = (c_t - c_s)/w = rho (sin t cos p,
// sin t sin p, cos t), the scaled translation L~ = T(delta) M~ (farfield.cu header) is factored
//   M' = Phi(-pi/2) D Phi(t) D^-1 Phi(p + pi/2) M          (rotate delta onto +z)
//   L' = Tz(rho) M',   L'_j^k = (-1)^{j+k} sum_{n>=k} M'_n^k (j+n)! / rho^{j+n+1}   (coaxial)
//   L  = Phi(-pi/2 - p) D^-T Phi(-t) D^T Phi(pi/2) L'       (rotate back)
// where Phi(a) = diag(e^{i m a}) and D = W(Ry(pi/2)), D^-1 = W(Ry(-pi/2)) are FIXED real
// matrices per degree (R_n(Q v) = W^n(Q) R_n(v)); in this basis W^n(Ry(b)) = diag(1/f) d^n(b)
// diag(f), f_m = sqrt((n+m)!(n-m)!), d^n = Wigner's small d.  Ry(t) = S Rz(t) S^-1 with
// S = Rz(pi/2) Ry(pi/2) is what lets one pair of fixed matrices serve every direction.  The two
// Phi(+-pi/2) around Tz cancel (Tz is diagonal in the order k).  Vectors of a real field are
// conjugate symmetric, so each real matrix X acts on the stored m >= 0 half as
//   Re b_m' = sum_{m>=0} E_m'm Re a_m,  Im b_m' = sum_{m>0} F_m'm Im a_m,
//   E_m'm = X_m'm + (-1)^m X_m',-m,  F_m'm = X_m'm - (-1)^m X_m',-m   (E_m'0 = X_m'0, F_m'0 = 0)
// and since X_m',-m = (-1)^{n+m'} X_m'm for all four matrices, E = 0 when n+m+m' is odd and
// F = 0 when it is even: (n+1)^2 FMAs per degree.  One thread owns one (target, source) pair; the
// whole pipeline is unrolled at compile time (P is a template parameter) and the matrix entries are
// compile-time constants (FFMA immediates, see make_rot).  Each thread's working vector lives in a
// private shared-memory slot and streams through registers one degree block (rotations) or one
// order column (coaxial translation) at a time, so registers stay low for any P.  The 32 pairs of a
// warp belong to one target cell and are summed through the same slots.  The unrolled body (~86 KB
// of SASS at P = 12) is far larger than the 32 KB L1.5 instruction cache, so the default kernel
// runs 11 warps per CTA (one CTA per SM, all its shared memory) in lockstep rounds: the warps walk
// the body together and share the fetched lines (measured: 42 -> 28 ms at C5).
#include <cmath>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace fmm {

namespace {

// [matrix][degree block][m'][m]: 0 = D^-1, 1 = D, 2 = D^T, 3 = D^-T.  Entry (m', m) holds E_m'm when
// n + m + m' is even and F_m'm when odd (the other one is a structural zero).  The table is
// evaluated at COMPILE time: with b = +-pi/2 every power of cos(b/2), sin(b/2) collapses to
// 2^-n (+-1)^(m'-m), and W^n = diag(1/f) d^n diag(f) only needs f_m^2 = (n+m)!(n-m)!, so
//   W^n_m'm(+-pi/2) = 2^-n (n+m)!(n-m)! (+-1)^(m'-m) sum_k (-1)^(m'-m+k) / ((n+m-k)! k! (m'-m+k)! (n-m'-k)!)
// is rational -- after unrolling every matrix entry is an FFMA immediate (no constant-cache
// loads, no uniform-register traffic).  init_rot_tables() re-derives the table on the host from
// Wigner's formula in double precision and refuses to run if they disagree.
__host__ __device__ constexpr int pad4(int v) { return (v + 3) & ~3; }
__host__ __device__ constexpr int boff(int n) {  // sum_{k<n} pad4((k+1)^2)
  int o = 0;
  for (int k = 0; k < n; ++k) o += pad4((k + 1) * (k + 1));
  return o;
}
constexpr int RMAXC = 14;  // highest instantiated rotation order
constexpr int TSZ = boff(RMAXC);
struct RotTab {
  float v[4][TSZ];
};
__host__ __device__ constexpr double cfact(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= (double)i;
  return f;
}
// W^n_{mp,m}(+pi/2) for |mp|, |m| <= n < RMAXC, from a factorial table (keeps the constant
// evaluation within the compiler's step budget); W(-pi/2) = (-1)^(mp-m) W(+pi/2)
struct WTab {
  double fact[2 * RMAXC + 1];
  double v[RMAXC][2 * RMAXC - 1][2 * RMAXC - 1];
};
__host__ __device__ constexpr WTab make_w() {
  WTab t{};
  t.fact[0] = 1.0;
  for (int i = 1; i <= 2 * RMAXC; ++i) t.fact[i] = t.fact[i - 1] * (double)i;
  for (int n = 0; n < RMAXC; ++n)
    for (int mp = -n; mp <= n; ++mp)
      for (int m = -n; m <= n; ++m) {
        double s = 0.0;
        const int k0 = (m - mp) > 0 ? (m - mp) : 0, k1 = (n + m) < (n - mp) ? (n + m) : (n - mp);
        for (int k = k0; k <= k1; ++k)
          s += (((mp - m + k) & 1) ? -1.0 : 1.0) /
               (t.fact[n + m - k] * t.fact[k] * t.fact[mp - m + k] * t.fact[n - mp - k]);
        double sc = t.fact[n + m] * t.fact[n - m];
        for (int i = 0; i < n; ++i) sc *= 0.5;
        t.v[n][mp + n][m + n] = s * sc;
      }
  return t;
}
__host__ __device__ constexpr double w_half_pi(const WTab& w, int n, int mp, int m, int sgn) {  // W^n_{mp,m}(sgn pi/2)
  const double v = w.v[n][mp + n][m + n];
  return (sgn < 0 && ((mp - m) & 1)) ? -v : v;
}
__host__ __device__ constexpr double x_entry(const WTab& w, int X, int n, int a, int b) {
  return X == 0 ? w_half_pi(w, n, a, b, -1) : X == 1 ? w_half_pi(w, n, a, b, 1) : X == 2 ? w_half_pi(w, n, b, a, 1)
                                                                                     : w_half_pi(w, n, b, a, -1);
}
__host__ __device__ constexpr RotTab make_rot() {
  constexpr WTab w = make_w();
  RotTab t{};
  for (int X = 0; X < 4; ++X)
    for (int n = 0; n < RMAXC; ++n)
      for (int mp = 0; mp <= n; ++mp)
        for (int m = 0; m <= n; ++m) {
          double v = 0.0;
          if (m == 0) {
            if (((n + mp) & 1) == 0) v = x_entry(w, X, n, mp, 0);  // E_m'0 = X_m'0, F_m'0 = 0
          } else {
            const double sg = (m & 1) ? -1.0 : 1.0;
            v = ((n + m + mp) & 1) == 0 ? x_entry(w, X, n, mp, m) + sg * x_entry(w, X, n, mp, -m)
                                        : x_entry(w, X, n, mp, m) - sg * x_entry(w, X, n, mp, -m);
          }
          t.v[X][boff(n) + mp * (n + 1) + m] = (float)v;
        }
  return t;
}
__device__ constexpr RotTab ROT = make_rot();

__host__ __device__ constexpr float factf(int n) {
  float f = 1.f;
  for (int i = 2; i <= n; ++i) f *= (float)i;
  return f;
}

// Per-thread vector slot in shared memory, coefficient-major / lane-minor ([2*NC][33]): all lanes
// touch the same coefficient at once -> conflict-free; the 33 stride keeps the final per-row
// reduction conflict-free too.
struct Slot {
  float2* base;  // &sv[0][lane]: (re, im) of coefficient c at base[c * 33]
  __device__ __forceinline__ float2 get(int c) const { return base[c * 33]; }
  __device__ __forceinline__ void set(int c, float re, float im) const { base[c * 33] = make_float2(re, im); }
  __device__ __forceinline__ void set(int c, float2 v) const { base[c * 33] = v; }
};

// The M2L slot with its last NREG coefficients in registers: the shared-memory part shrinks to
// (NC - NREG) x 33 float2 per warp, which is what bounds the lockstep kernel's resident warps
// (P = 13: 88 instead of 91 rows -> 10 warps per SM instead of 9).  Every index is a compile-time
// constant after unrolling, so the register entries never spill to local memory.
template <int NC, int NREG>
struct SlotR {
  static constexpr int C0 = NC - NREG;  // first register entry
  float2* base;
  float2 r[NREG > 0 ? NREG : 1];
  __device__ __forceinline__ float2 get(int c) const { return (NREG > 0 && c >= C0) ? r[c - C0] : base[c * 33]; }
  __device__ __forceinline__ void set(int c, float2 v) {
    if (NREG > 0 && c >= C0) r[c - C0] = v;
    else base[c * 33] = v;
  }
  __device__ __forceinline__ void set(int c, float re, float im) { set(c, make_float2(re, im)); }
};

__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }

// one degree block: b = X a (E/F form), a and b in registers
template <int n, int X>
__device__ __forceinline__ void mat_block(const float (&ar)[n + 1], const float (&ai)[n + 1], float (&br)[n + 1],
                                          float (&bi)[n + 1]) {
#pragma unroll
  for (int mp = 0; mp <= n; ++mp) {
    float re = 0.f, im = 0.f;
#pragma unroll
    for (int m = 0; m <= n; ++m) {
      // Wigner parity d_{m',-m}(pi/2) = (-1)^{n+m'} d_{m'm}(pi/2): E vanishes for odd n+m+m',
      // F for even n+m+m' -- half of the products are structural zeros and are skipped here
      if (((n + m + mp) & 1) == 0) re = fmaf(ROT.v[X][boff(n) + mp * (n + 1) + m], ar[m], re);
      else if (m > 0) im = fmaf(ROT.v[X][boff(n) + mp * (n + 1) + m], ai[m], im);
    }
    br[mp] = re;
    bi[mp] = im;
  }
}

// (r + i s) *= (zr + i zi)
__device__ __forceinline__ void cmul_ip(float& r, float& s, float zr, float zi) {
  float t = r * zr - s * zi;
  s = r * zi + s * zr;
  r = t;
}

// M' block n = rho^-n D Phi(t) D^-1 Phi(p + pi/2) M_n
template <int P, int n, class S>
__device__ __forceinline__ void pass_a(S& sl, const float2* __restrict__ Ms, const float (&zar)[P],
                                       const float (&zai)[P], const float (&zbr)[P], const float (&zbi)[P],
                                       float scale, float irho) {
  constexpr int c0 = n * (n + 1) / 2;
  asm volatile("" ::: "memory");  // keep the degree blocks' loads in place (register pressure)
  float ar[n + 1], ai[n + 1], br[n + 1], bi[n + 1];
#pragma unroll
  for (int m = 0; m <= n; ++m) {
    float2 q = __ldg(Ms + c0 + m);
    ar[m] = q.x;
    ai[m] = q.y;
    if (m > 0) cmul_ip(ar[m], ai[m], zar[m], zai[m]);  // Phi(p + pi/2)
  }
  mat_block<n, 0>(ar, ai, br, bi);                    // D^-1
#pragma unroll
  for (int m = 1; m <= n; ++m) cmul_ip(br[m], bi[m], zbr[m], zbi[m]);  // Phi(t)
  mat_block<n, 1>(br, bi, ar, ai);                    // D
#pragma unroll
  for (int m = 0; m <= n; ++m) sl.set(c0 + m, __fmul2_rn(make_float2(ar[m], ai[m]), bc2(scale)));
  if constexpr (n + 1 < P) pass_a<P, n + 1, S>(sl, Ms, zar, zai, zbr, zbi, scale * irho, irho);
}

// coaxial translation of order column k (input scaled by rho^-n, output missing rho^-(j+1))
template <int P, int k, class S>
__device__ __forceinline__ void pass_b(S& sl) {
  asm volatile("" ::: "memory");
  float2 t[P - k];
#pragma unroll
  for (int n = k; n < P; ++n) t[n - k] = sl.get(n * (n + 1) / 2 + k);
#pragma unroll
  for (int j = k; j < P; ++j) {
    const float sg = ((j + k) & 1) ? -1.f : 1.f;
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int n = k; n < P; ++n) acc = __ffma2_rn(bc2(sg * factf(j + n)), t[n - k], acc);  // packed re/im
    sl.set(j * (j + 1) / 2 + k, acc);
  }
  if constexpr (k + 1 < P) pass_b<P, k + 1, S>(sl);
}

// L block j = Phi(-p - pi/2) D^-T Phi(-t) D^T rho^-(j+1) L'_j
template <int P, int n, class S>
__device__ __forceinline__ void pass_c(S& sl, const float (&zar)[P], const float (&zai)[P],
                                       const float (&zbr)[P], const float (&zbi)[P], float scale, float irho) {
  constexpr int c0 = n * (n + 1) / 2;
  asm volatile("" ::: "memory");
  float ar[n + 1], ai[n + 1], br[n + 1], bi[n + 1];
#pragma unroll
  for (int m = 0; m <= n; ++m) {
    const float2 v = __fmul2_rn(sl.get(c0 + m), bc2(scale));
    ar[m] = v.x;
    ai[m] = v.y;
  }
  mat_block<n, 2>(ar, ai, br, bi);                    // D^T
#pragma unroll
  for (int m = 1; m <= n; ++m) cmul_ip(br[m], bi[m], zbr[m], -zbi[m]);  // Phi(-t)
  mat_block<n, 3>(br, bi, ar, ai);                    // D^-T
#pragma unroll
  for (int m = 0; m <= n; ++m) {
    if (m > 0) cmul_ip(ar[m], ai[m], zar[m], -zai[m]);  // Phi(-p - pi/2)
    sl.set(c0 + m, ar[m], ai[m]);
  }
  if constexpr (n + 1 < P) pass_c<P, n + 1, S>(sl, zar, zai, zbr, zbi, scale * irho, irho);
}

// the translated local expansion of source cell s at target (tx, ty, tz) into the thread's slot
template <int P, class S>
__device__ __forceinline__ void translate_pair(S& sl, int tx, int ty, int tz, int s,
                                               const uint64_t* __restrict__ key, const float2* __restrict__ M) {
  constexpr int NC = P * (P + 1) / 2;
  int sx, sy, sz;
  demorton(key[s], sx, sy, sz);
  const float dx = (float)(tx - sx), dy = (float)(ty - sy), dz = (float)(tz - sz);
  const float rxy2 = dx * dx + dy * dy;
  const float rxy = sqrtf(rxy2);
  const float irho = rsqrtf(rxy2 + dz * dz);
  float cp = 1.f, sp = 0.f;
  if (rxy > 0.f) {
    cp = dx / rxy;
    sp = dy / rxy;
  }
  // powers of za = e^{i(p + pi/2)} = i e^{ip} and zb = e^{it}
  float zar[P], zai[P], zbr[P], zbi[P];
  zar[0] = 1.f;
  zai[0] = 0.f;
  zbr[0] = 1.f;
  zbi[0] = 0.f;
  const float ar1 = -sp, ai1 = cp, br1 = dz * irho, bi1 = rxy * irho;
#pragma unroll
  for (int m = 1; m < P; ++m) {
    zar[m] = zar[m - 1] * ar1 - zai[m - 1] * ai1;
    zai[m] = zar[m - 1] * ai1 + zai[m - 1] * ar1;
    zbr[m] = zbr[m - 1] * br1 - zbi[m - 1] * bi1;
    zbi[m] = zbr[m - 1] * bi1 + zbi[m - 1] * br1;
  }
  pass_a<P, 0, S>(sl, M + (size_t)s * NC, zar, zai, zbr, zbi, 1.f, irho);
  pass_b<P, 0, S>(sl);
  pass_c<P, 0, S>(sl, zar, zai, zbr, zbi, irho, irho);
}

// Lockstep variant: the W warps of a CTA (one target row each) start every 32-pair round together
// (__syncthreads per round), so the SM's warps walk the long unrolled body in step and share the
// instruction-cache lines (the body is ~3x the L1.5 I$); dynamic shared memory, W slots.
template <int P, int W, int RPW, int NREG>
__global__ void __launch_bounds__(32 * W) k_m2l_rot_sync(int rows, const int* __restrict__ tcells,
                                                         const int* __restrict__ off, const int* __restrict__ idx,
                                                         const uint64_t* __restrict__ key,
                                                         const float2* __restrict__ M, float2* __restrict__ Lx) {
  // A CTA owns RPW x W consecutive rows (Morton-local); a warp that finishes its row takes the next
  // unclaimed one of the window at the next round, so rows of different lengths do not leave warps
  // idle at the round barriers.  Each row is computed whole by the warp that claims it (fixed chunk
  // order), so the result does not depend on which warp that is.
  constexpr int NC = P * (P + 1) / 2;
  constexpr int NR = (NC + 31) / 32;
  constexpr int NS = NC - NREG;  // shared-memory rows of the slot
  extern __shared__ float2 svdyn[];
  __shared__ int next_row;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r_beg = blockIdx.x * W * RPW, r_end = min(rows, r_beg + W * RPW);
  if (threadIdx.x == 0) next_row = r_beg + W;
  float2* sv = svdyn + (size_t)w * NS * 33;
  SlotR<NC, NREG> sl;
  sl.base = sv + lane;
  int row = r_beg + w;
  int cell = 0, lo = 0, hi = 0, e0 = 0, tx = 0, ty = 0, tz = 0;
  auto start = [&]() {
    if (row < r_end) {
      cell = tcells[row];
      lo = off[row];
      hi = off[row + 1];
      e0 = lo;
      demorton(key[cell], tx, ty, tz);
    }
  };
  start();
  float2 acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = make_float2(0.f, 0.f);
  __syncthreads();
  while (true) {
    const bool active = row < r_end;
    if (!__syncthreads_or(active)) break;  // the round barrier; ends when every warp is out of rows
    if (active) {
      const int e = e0 + lane;
      if (e < hi) {
        translate_pair<P>(sl, tx, ty, tz, idx[e], key, M);
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c) sl.set(c, 0.f, 0.f);
      }
      // the register rows: butterfly sums over the 32 pairs (fixed order)
      float2 rs[NREG > 0 ? NREG : 1];
#pragma unroll
      for (int q = 0; q < NREG; ++q) {
        rs[q] = sl.r[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          rs[q].x += __shfl_xor_sync(0xffffffffu, rs[q].x, o);
          rs[q].y += __shfl_xor_sync(0xffffffffu, rs[q].y, o);
        }
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int c = lane + 32 * r;
        if (c < NS) {
          float2 sum = make_float2(0.f, 0.f);
#pragma unroll 8
          for (int l = 0; l < 32; ++l) sum = __fadd2_rn(sum, sv[c * 33 + l]);
          acc[r] = __fadd2_rn(acc[r], sum);
        } else if (c < NC) {
#pragma unroll
          for (int q = 0; q < NREG; ++q)
            if (c == NS + q) acc[r] = __fadd2_rn(acc[r], rs[q]);
        }
      }
      __syncwarp();
      e0 += 32;
      if (e0 >= hi) {  // row done: flush, claim the next row of the window
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const int c = lane + 32 * r;
          if (c < NC) {
            float2 o = Lx[(size_t)cell * NC + c];
            o.x += acc[r].x;
            o.y += acc[r].y;
            Lx[(size_t)cell * NC + c] = o;
          }
          acc[r] = make_float2(0.f, 0.f);
        }
        int nr = 0;
        if (lane == 0) nr = atomicAdd(&next_row, 1);
        row = __shfl_sync(0xffffffffu, nr, 0);
        start();
      }
    }
  }
}

// one warp per target cell; W warps per CTA start in lockstep on the same (long, unrolled) code
template <int P, int W>
__global__ void __launch_bounds__(32 * W) k_m2l_rot(int rows, const int* __restrict__ tcells,
                                                    const int* __restrict__ off, const int* __restrict__ idx,
                                                    const uint64_t* __restrict__ key, const float2* __restrict__ M,
                                                    float2* __restrict__ Lx) {
  constexpr int NC = P * (P + 1) / 2;
  constexpr int NR = (NC + 31) / 32;
  __shared__ float2 svall[W][NC * 33];
  const int row = blockIdx.x * W + (threadIdx.x >> 5);
  if (row >= rows) return;
  float2* sv = svall[threadIdx.x >> 5];
  const int cell = tcells[row];
  const int lo = off[row], hi = off[row + 1];
  const int lane = threadIdx.x & 31;
  const Slot sl{sv + lane};
  int tx, ty, tz;
  demorton(key[cell], tx, ty, tz);
  float2 acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = make_float2(0.f, 0.f);
  for (int e0 = lo; e0 < hi; e0 += 32) {
    const int e = e0 + lane;
    if (e < hi) {
      translate_pair<P>(sl, tx, ty, tz, idx[e], key, M);
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) sl.set(c, 0.f, 0.f);
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int c = lane + 32 * r;
      if (c < NC) {
        float2 sum = make_float2(0.f, 0.f);
#pragma unroll 8
        for (int l = 0; l < 32; ++l) sum = __fadd2_rn(sum, sv[c * 33 + l]);
        acc[r] = __fadd2_rn(acc[r], sum);
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int c = lane + 32 * r;
    if (c < NC) {
      float2 o = Lx[(size_t)cell * NC + c];
      o.x += acc[r].x;
      o.y += acc[r].y;
      Lx[(size_t)cell * NC + c] = o;
    }
  }
}

// ---------------------------------------------------------------- M2M / L2L by rotation
// Child-parent offsets are the 8 diagonals d = (+-1, +-1, +-1)/4 (parent-width units), |d| = sqrt(3)/4,
// so the coaxial shift coefficients are compile-time constants.  Rotations (verified against the
// direct translations):  multipoles  fwd = X1 Phi(t) X0 Phi(p + pi/2),  back = Phi(-p - pi/2) X1 Phi(-t) X0
//                        locals      fwd = X3 Phi(t) X2 Phi(p + pi/2),  back = Phi(-p - pi/2) X3 Phi(-t) X2
// (X0 = D^-1, X1 = D, X2 = D^T, X3 = D^-T; the Phi(-+pi/2) around the coaxial step cancel).
constexpr float RHO8 = 0.43301270189221932f;  // sqrt(3)/4

__host__ __device__ constexpr float powf_c(float b, int e) {
  float r = 1.f;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// per degree block: a <- XB Phi(zb) XA Phi(za) a   (conj: use conjugated phases)
template <int n, int XA, int XB>
__device__ __forceinline__ void rot_block(float (&ar)[n + 1], float (&ai)[n + 1], const float* zar, const float* zai,
                                          const float* zbr, const float* zbi, float csa, float csb) {
  float br[n + 1], bi[n + 1];
#pragma unroll
  for (int m = 1; m <= n; ++m) cmul_ip(ar[m], ai[m], zar[m], csa * zai[m]);
  mat_block<n, XA>(ar, ai, br, bi);
#pragma unroll
  for (int m = 1; m <= n; ++m) cmul_ip(br[m], bi[m], zbr[m], csb * zbi[m]);
  mat_block<n, XB>(br, bi, ar, ai);
}

// pass over degrees, forward (MODE 0: global src -> slot, 3: slot -> slot) or back rotation
// (4: slot -> slot); in-place slot passes are safe because degree block n only reads block n
template <int P, int n, int XA, int XB, int MODE>
__device__ __forceinline__ void rot_pass(const Slot& sl, const float2* __restrict__ src, const float* zar,
                                         const float* zai, const float* zbr, const float* zbi) {
  constexpr int c0 = n * (n + 1) / 2;
  float ar[n + 1], ai[n + 1];
#pragma unroll
  for (int m = 0; m <= n; ++m) {
    if (MODE == 0) {
      const float2 q = __ldg(src + c0 + m);
      ar[m] = q.x;
      ai[m] = q.y;
    } else {
      const float2 v = sl.get(c0 + m);
      ar[m] = v.x;
      ai[m] = v.y;
    }
  }
  if (MODE != 4) {
    rot_block<n, XA, XB>(ar, ai, zar, zai, zbr, zbi, 1.f, 1.f);
#pragma unroll
    for (int m = 0; m <= n; ++m) sl.set(c0 + m, ar[m], ai[m]);
  } else {
    // back rotation: XB Phi(-t) XA, then Phi(-p - pi/2)
    float br[n + 1], bi[n + 1];
    mat_block<n, XA>(ar, ai, br, bi);
#pragma unroll
    for (int m = 1; m <= n; ++m) cmul_ip(br[m], bi[m], zbr[m], -zbi[m]);
    mat_block<n, XB>(br, bi, ar, ai);
#pragma unroll
    for (int m = 0; m <= n; ++m) {
      if (m > 0) cmul_ip(ar[m], ai[m], zar[m], -zai[m]);
      sl.set(c0 + m, ar[m], ai[m]);
    }
  }
  if constexpr (n + 1 < P) rot_pass<P, n + 1, XA, XB, MODE>(sl, src, zar, zai, zbr, zbi);
}

// warp-cooperative coalesced copies between a contiguous block of `cnt` cells' expansions in
// global memory and the warp's per-lane slots (lane i <-> cell i)
template <int NC>
__device__ __forceinline__ void slots_load(float2* sv, const float2* __restrict__ g, int cnt, int lane) {
  for (int k = lane; k < cnt * NC; k += 32) {
    const int i = k / NC, c = k - i * NC;
    sv[c * 33 + i] = g[k];
  }
}
template <int NC, bool ADD>
__device__ __forceinline__ void slots_store(const float2* sv, float2* __restrict__ g, int cnt, const int* __restrict__ on,
                                            int lane) {
  for (int k = lane; k < cnt * NC; k += 32) {
    const int i = k / NC, c = k - i * NC;
    if (on && !on[i]) continue;
    const float2 v = sv[c * 33 + i];
    if (ADD) {
      const float2 o = g[k];
      g[k] = make_float2(o.x + v.x, o.y + v.y);
    } else {
      g[k] = v;
    }
  }
}

// coaxial M2M along +z by RHO8: M_n^k <- sum_{j=k}^{n} 2^-j M_j^k rho^(n-j)/(n-j)!
template <int P, int k>
__device__ __forceinline__ void coax_m2m(const Slot& sl) {
  float2 t[P - k];
#pragma unroll
  for (int j = k; j < P; ++j) t[j - k] = sl.get(j * (j + 1) / 2 + k);
#pragma unroll
  for (int n = k; n < P; ++n) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = k; j <= n; ++j)
      acc = __ffma2_rn(bc2(1.f / powf_c(2.f, j) * powf_c(RHO8, n - j) / factf(n - j)), t[j - k], acc);
    sl.set(n * (n + 1) / 2 + k, acc);
  }
  if constexpr (k + 1 < P) coax_m2m<P, k + 1>(sl);
}

// coaxial L2L along +z by RHO8: L_j^k <- 2^-(j+1) sum_{n=j}^{P-1} L_n^k rho^(n-j)/(n-j)!
template <int P, int k>
__device__ __forceinline__ void coax_l2l(const Slot& sl) {
  float2 t[P - k];
#pragma unroll
  for (int n = k; n < P; ++n) t[n - k] = sl.get(n * (n + 1) / 2 + k);
#pragma unroll
  for (int j = k; j < P; ++j) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int n = j; n < P; ++n)
      acc = __ffma2_rn(bc2(1.f / powf_c(2.f, j + 1) * powf_c(RHO8, n - j) / factf(n - j)), t[n - k], acc);
    sl.set(j * (j + 1) / 2 + k, acc);
  }
  if constexpr (k + 1 < P) coax_l2l<P, k + 1>(sl);
}

// phase powers of za = e^{i(p + pi/2)}, zb = e^{i t} for the octant of a child key
template <int P>
__device__ __forceinline__ void octant_phases(uint64_t key, float* zar, float* zai, float* zbr, float* zbi) {
  const float sx = (key & 1) ? 1.f : -1.f, sy = (key & 2) ? 1.f : -1.f, sz = (key & 4) ? 1.f : -1.f;
  const float r2 = 0.70710678118654752f;  // |(sx, sy)| / sqrt(2) normalisation
  const float cp = sx * r2, sp = sy * r2;
  const float ct = sz * 0.57735026918962576f, st = 0.81649658092772603f;  // cos t = sz/sqrt(3), sin t = sqrt(2/3)
  const float ar1 = -sp, ai1 = cp;
  zar[0] = 1.f;
  zai[0] = 0.f;
  zbr[0] = 1.f;
  zbi[0] = 0.f;
#pragma unroll
  for (int m = 1; m < P; ++m) {
    zar[m] = zar[m - 1] * ar1 - zai[m - 1] * ai1;
    zai[m] = zar[m - 1] * ai1 + zai[m - 1] * ar1;
    zbr[m] = zbr[m - 1] * ct - zbi[m - 1] * st;
    zbi[m] = zbr[m - 1] * st + zbi[m - 1] * ct;
  }
}

// thread per child cell at one level: T[child] = (translated child multipole); summed per parent below.
// The warp's 32 children are contiguous: their multipoles come in and the results go out through
// the slots with coalesced accesses.
template <int P>
__global__ void __launch_bounds__(32) k_m2m_rot(int c0, int n, const uint64_t* __restrict__ key,
                                                const int* __restrict__ scnt, const float2* __restrict__ M,
                                                float2* __restrict__ T) {
  constexpr int NC = P * (P + 1) / 2;
  __shared__ float2 sv[NC * 33];
  __shared__ int on[32];
  const int lane = threadIdx.x;
  const int b0 = blockIdx.x * 32, cnt = min(32, n - b0);
  const int i = b0 + lane;
  const int cell = c0 + i;
  const bool act = i < n && scnt[cell] > 0;
  on[lane] = act;
  slots_load<NC>(sv, M + (size_t)(c0 + b0) * NC, cnt, lane);
  __syncwarp();
  const Slot sl{sv + lane};
  if (act) {
    float zar[P], zai[P], zbr[P], zbi[P];
    octant_phases<P>(key[cell], zar, zai, zbr, zbi);
    rot_pass<P, 0, 0, 1, 3>(sl, nullptr, zar, zai, zbr, zbi);
    coax_m2m<P, 0>(sl);
    rot_pass<P, 0, 0, 1, 4>(sl, nullptr, zar, zai, zbr, zbi);
  }
  __syncwarp();
  slots_store<NC, false>(sv, T + (size_t)(c0 + b0) * NC, cnt, on, lane);
}

// parent multipole = sum of its children's translated multipoles (fixed order)
__global__ void k_m2m_sum(int c0, int n, int NC, const int* __restrict__ cb, const int* __restrict__ ce,
                          const int* __restrict__ scnt, const float2* __restrict__ T, float2* __restrict__ M) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = t / NC, c = t - i * NC;
  if (i >= n) return;
  const int cell = c0 + i;
  if (scnt[cell] == 0) return;
  float2 s = make_float2(0.f, 0.f);
  for (int ch = cb[cell]; ch < ce[cell]; ++ch) {
    if (scnt[ch] == 0) continue;
    const float2 v = T[(size_t)ch * NC + c];
    s.x += v.x;
    s.y += v.y;
  }
  M[(size_t)cell * NC + c] = s;
}

// thread per child cell: L[child] += translated parent local expansion (coalesced accumulate of the
// warp's 32 contiguous children through the slots)
template <int P>
__global__ void __launch_bounds__(32) k_l2l_rot(int c0, int n, const uint64_t* __restrict__ key,
                                                const int* __restrict__ parent, const int* __restrict__ tcnt,
                                                const float2* __restrict__ Lp, float2* __restrict__ Lx) {
  constexpr int NC = P * (P + 1) / 2;
  __shared__ float2 sv[NC * 33];
  __shared__ int on[32];
  const int lane = threadIdx.x;
  const int b0 = blockIdx.x * 32, cnt = min(32, n - b0);
  const int i = b0 + lane;
  const int cell = c0 + i;
  const bool act = i < n && tcnt[cell] > 0;
  on[lane] = act;
  const Slot sl{sv + lane};
  if (act) {
    float zar[P], zai[P], zbr[P], zbi[P];
    octant_phases<P>(key[cell], zar, zai, zbr, zbi);
    rot_pass<P, 0, 2, 3, 0>(sl, Lp + (size_t)parent[cell] * NC, zar, zai, zbr, zbi);
    coax_l2l<P, 0>(sl);
    rot_pass<P, 0, 2, 3, 4>(sl, nullptr, zar, zai, zbr, zbi);
  }
  __syncwarp();
  slots_store<NC, true>(sv, Lx + (size_t)(c0 + b0) * NC, cnt, on, lane);
}

// Wigner small d^n_{m'm}(b) (explicit sum)
double wigner_d(int n, int mp, int m, double b) {
  auto fact = [](int k) {
    double f = 1;
    for (int i = 2; i <= k; ++i) f *= i;
    return f;
  };
  int s0 = std::max(0, m - mp), s1 = std::min(n + m, n - mp);
  double t = 0, c = std::cos(b / 2), s = std::sin(b / 2);
  for (int k = s0; k <= s1; ++k) {
    double sg = ((mp - m + k) & 1) ? -1.0 : 1.0;
    t += sg / (fact(n + m - k) * fact(k) * fact(mp - m + k) * fact(n - mp - k)) * std::pow(c, 2 * n + m - mp - 2 * k) *
         std::pow(s, mp - m + 2 * k);
  }
  return t * std::sqrt(fact(n + mp) * fact(n - mp) * fact(n + m) * fact(n - m));
}

// compacted interaction lists (sources with points of `src`, targets with points of `tgt`)
__global__ void k_compact_count(int n, int cell_off, const long long* __restrict__ off, const int* __restrict__ idx,
                                const int* __restrict__ scnt, const int* __restrict__ tcnt, int* cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = cell_off + i;
  int m = 0;
  if (tcnt[c] > 0)
    for (long long e = off[c]; e < off[c + 1]; ++e) m += scnt[idx[e]] > 0;
  cnt[i] = m;
}

// the compacted lists hold expansion SLOTS (cmap: cell -> slot, nullptr = identity; ctx.h); a
// needed cell without a slot (a LET plan that missed it) raises flag
__global__ void k_compact_fill(int n, int cell_off, const long long* __restrict__ off, const int* __restrict__ idx,
                               const int* __restrict__ scnt, const int* __restrict__ pos, const int* __restrict__ cmap,
                               int* out_idx, int* out_cell, int* out_off, int* flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = cell_off + i;
  const int start = pos[i], end = pos[i + 1];
  if (start == end) return;
  int w = start;
  for (long long e = off[c]; e < off[c + 1]; ++e)
    if (scnt[idx[e]] > 0) {
      const int sl = cmap ? cmap[idx[e]] : idx[e];
      if (sl < 0) atomicOr(flag, 1);
      out_idx[w++] = sl < 0 ? 0 : sl;
    }
  // row r of the compacted list = number of non-empty rows before i
  const int tc = cmap ? cmap[c] : c;
  if (tc < 0) atomicOr(flag, 1);
  out_cell[pos[n + 1 + i]] = tc < 0 ? 0 : tc;
  out_off[pos[n + 1 + i]] = start;
}

__global__ void k_row_flags(int n, const int* __restrict__ cnt, int* flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = cnt[i] > 0;
}

}  // namespace

// instantiated orders (others use the O(P^4) kernel in farfield.cu)
bool rot_supported(int P) { return P == 8 || P == 10 || P == 12 || P == 13 || P == 14; }

void init_rot_tables() {
  static bool done = false;
  if (done) return;
  static constexpr RotTab host = make_rot();  // the same compile-time table the kernels fold in
  for (int n = 0; n < RMAXC; ++n) {
    std::vector<double> f(2 * n + 1);
    for (int m = -n; m <= n; ++m) f[m + n] = std::sqrt(cfact(n + m) * cfact(n - m));
    // W(+pi/2) = D, W(-pi/2) = D^-1 in the R_n^m basis, from Wigner's formula with cos/sin
    auto W = [&](int mp, int m, double beta) { return wigner_d(n, mp, m, beta) * f[m + n] / f[mp + n]; };
    for (int X = 0; X < 4; ++X)
      for (int mp = 0; mp <= n; ++mp)
        for (int m = 0; m <= n; ++m) {
          auto Xv = [&](int a, int b) {
            switch (X) {
              case 0: return W(a, b, -M_PI / 2);
              case 1: return W(a, b, M_PI / 2);
              case 2: return W(b, a, M_PI / 2);
              default: return W(b, a, -M_PI / 2);
            }
          };
          double v = 0.0;
          const double sg = (m & 1) ? -1.0 : 1.0;
          if (((n + m + mp) & 1) == 0) v = (m == 0) ? Xv(mp, 0) : Xv(mp, m) + sg * Xv(mp, -m);
          else if (m > 0) v = Xv(mp, m) - sg * Xv(mp, -m);
          const double got = host.v[X][boff(n) + mp * (n + 1) + m];
          if (std::fabs(got - v) > 1e-6 * std::max(1.0, std::fabs(v)))
            throw Error(FMMBEM_E_CUDA, "rotation table self-check failed");
        }
  }
  done = true;
}

// Build (or fetch) the compacted M2L work list for (src, tgt): rows = target cells at levels >= 2
// with target points and at least one source cell holding source points.
const M2LWork& m2l_work(fmmbem_ctx* c, const int* src_cnt, const int* tgt_cnt, cudaStream_t st) {
  for (auto& w : c->m2l_cache)
    if (w->src == src_cnt && w->tgt == tgt_cnt) return *w;
  const Tree& T = c->tree;
  auto w = std::make_unique<M2LWork>();
  w->src = src_cnt;
  w->tgt = tgt_cnt;
  const int off0 = (int)T.lvl_off[2];
  const int n = (int)(T.n_cells - off0);
  DevBuf<int> cnt, pos;
  cnt.alloc(2 * (n + 1));
  pos.alloc(2 * (n + 1));
  cnt.zero(st);
  k_compact_count<<<ceil_div(n, 256), 256, 0, st>>>(n, off0, T.m2l_off.get(), T.m2l_idx.get(), src_cnt, tgt_cnt,
                                                     cnt.get());
  k_row_flags<<<ceil_div(n, 256), 256, 0, st>>>(n, cnt.get(), cnt.get() + n + 1);
  FMM_CHECK_LAUNCH();
  scan_ints(cnt.get(), pos.get(), n + 1, st);                    // pair offsets
  scan_ints(cnt.get() + n + 1, pos.get() + n + 1, n + 1, st);    // row ids
  int h[2] = {0, 0};
  FMM_CUDA(cudaMemcpyAsync(&h[0], pos.get() + n, sizeof(int), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaMemcpyAsync(&h[1], pos.get() + 2 * n + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  w->pairs = h[0];
  w->rows = h[1];
  w->idx.alloc(std::max(1, h[0]));
  w->cell.alloc(std::max(1, h[1]));
  w->off.alloc(h[1] + 1);
  DevBuf<int> flag;
  flag.alloc(1);
  flag.zero(st);
  k_compact_fill<<<ceil_div(n, 256), 256, 0, st>>>(n, off0, T.m2l_off.get(), T.m2l_idx.get(), src_cnt, pos.get(),
                                                    c->slot_map(), w->idx.get(), w->cell.get(), w->off.get(),
                                                    flag.get());
  FMM_CHECK_LAUNCH();
  FMM_CUDA(cudaMemcpyAsync(w->off.get() + h[1], &h[0], sizeof(int), cudaMemcpyHostToDevice, st));
  int bad = 0;
  FMM_CUDA(cudaMemcpyAsync(&bad, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
  FMM_CUDA(cudaStreamSynchronize(st));
  if (bad) throw Error(FMMBEM_E_CUDA, "M2L source or target cell without an expansion slot (LET plan)");
  c->m2l_cache.push_back(std::move(w));
  return *c->m2l_cache.back();
}

bool m2m_rot_supported(int P) { return rot_supported(P); }

// M2M of level l (children at l + 1); scratch T must hold n_cells * NC float2
// (the cells of this rank's windows only: children of level l + 1, parents of level l; pointers by
// global cell index through lvl_ptr, ctx.h)
void launch_m2m_rot(fmmbem_ctx* c, int l, const int* scnt, float2* T, cudaStream_t st) {
  const Tree& Tr = c->tree;
  const int ch0 = (int)c->win_lo[l + 1], nch = (int)(c->win_hi[l + 1] - c->win_lo[l + 1]);
  const int p0 = (int)c->win_lo[l], np = (int)(c->win_hi[l] - c->win_lo[l]);
  if (nch <= 0 || np <= 0) return;
  const float2* Mc = c->lvl_ptr(c->Mx.get(), l + 1);
  float2* Tc = c->lvl_ptr(T, l + 1);
  switch (c->P) {
    case 8: k_m2m_rot<8><<<ceil_div(nch, 32), 32, 0, st>>>(ch0, nch, Tr.key.get(), scnt, Mc, Tc); break;
    case 10: k_m2m_rot<10><<<ceil_div(nch, 32), 32, 0, st>>>(ch0, nch, Tr.key.get(), scnt, Mc, Tc); break;
    case 12: k_m2m_rot<12><<<ceil_div(nch, 32), 32, 0, st>>>(ch0, nch, Tr.key.get(), scnt, Mc, Tc); break;
    case 13: k_m2m_rot<13><<<ceil_div(nch, 32), 32, 0, st>>>(ch0, nch, Tr.key.get(), scnt, Mc, Tc); break;
    case 14: k_m2m_rot<14><<<ceil_div(nch, 32), 32, 0, st>>>(ch0, nch, Tr.key.get(), scnt, Mc, Tc); break;
    default: throw Error(FMMBEM_E_INVALID, "M2M rotation not instantiated for this P");
  }
  k_m2m_sum<<<ceil_div((int64_t)np * c->NC, 256), 256, 0, st>>>(p0, np, c->NC, Tr.child_begin.get(),
                                                                 Tr.child_end.get(), scnt, Tc,
                                                                 c->lvl_ptr(c->Mx.get(), l));
  FMM_CHECK_LAUNCH();
}

// L2L from level l to l + 1
void launch_l2l_rot(fmmbem_ctx* c, int l, const int* tcnt, cudaStream_t st) {
  const Tree& Tr = c->tree;
  const int ch0 = (int)c->win_lo[l + 1], nch = (int)(c->win_hi[l + 1] - c->win_lo[l + 1]);
  if (nch <= 0) return;
  const float2* Lp = c->lvl_ptr(c->Lx.get(), l);
  float2* Lc = c->lvl_ptr(c->Lx.get(), l + 1);
#define FMM_L2L_CASE(PP) \
  case PP: k_l2l_rot<PP><<<ceil_div(nch, 32), 32, 0, st>>>(ch0, nch, Tr.key.get(), Tr.parent.get(), tcnt, Lp, Lc); break;
  switch (c->P) {
    FMM_L2L_CASE(8) FMM_L2L_CASE(10) FMM_L2L_CASE(12) FMM_L2L_CASE(13) FMM_L2L_CASE(14)
    default: throw Error(FMMBEM_E_INVALID, "L2L rotation not instantiated for this P");
  }
#undef FMM_L2L_CASE
  FMM_CHECK_LAUNCH();
}

#ifndef M2L_RPW
#define M2L_RPW 16  // rows per warp in a CTA's Morton window
#endif
template <int P, int W, int NREG>
void m2l_sync_launch(const M2LWork& w, const Tree& T, fmmbem_ctx* c, size_t smem, cudaStream_t st) {
  static unsigned long long attr_devices = 0;  // the attribute is per device: set it once on each
  int dev = 0;
  FMM_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !(attr_devices >> dev & 1ULL)) {
    FMM_CUDA(cudaFuncSetAttribute(k_m2l_rot_sync<P, W, M2L_RPW, NREG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr_devices |= 1ULL << dev;
  }
  k_m2l_rot_sync<P, W, M2L_RPW, NREG><<<ceil_div(w.rows, M2L_RPW * W), 32 * W, smem, st>>>((int)w.rows, w.cell.get(), w.off.get(),
                                                                   w.idx.get(), c->slot_keys(), c->Mx.get(),
                                                                   c->Lx.get());
}

// lockstep warps per CTA: as many per-warp slots ((NC - NREG) x 33 float2) as fit the SM's 227 KB of
// shared memory -- one CTA per SM.  NREG = the slot rows kept in registers.  P = 13 (the bench
// order): 11 rows -> 11 warps instead of 9, 168 registers, no spills (C5: M2L 36.6 -> 33.2 ms; 3 rows
// / 10 warps: 35.3 ms); P = 12: 5 rows -> 12 warps.  Other orders: the fewest rows (<= 4) that gain
// one warp while the CTA stays <= 16 warps (>= 128 registers per thread), else none.
#ifndef M2L_NREG13
#define M2L_NREG13 11
#endif
#ifndef M2L_NREG12
#define M2L_NREG12 5  // P = 12 (the charge-FMM order of the bench): 12 warps, M2L 27.2 -> 26.5 ms (13 warps: 28.9)
#endif
constexpr int m2l_nc(int P) { return P * (P + 1) / 2; }
constexpr int m2l_warps_for(int P, int nreg) { return (227 * 1024) / ((m2l_nc(P) - nreg) * 33 * 8); }
constexpr int m2l_nreg(int P) {
  if (P == 13) return M2L_NREG13;
  if (P == 12 && M2L_NREG12) return M2L_NREG12;
  const int w0 = m2l_warps_for(P, 0);
  for (int k = 1; k <= 4; ++k)
    if (m2l_warps_for(P, k) > w0) return m2l_warps_for(P, k) <= 16 ? k : 0;
  return 0;
}
constexpr int m2l_warps(int P) { return m2l_warps_for(P, m2l_nreg(P)); }

void launch_m2l_rot(fmmbem_ctx* c, const M2LWork& w, cudaStream_t st) {
  if (w.rows == 0) return;
  const Tree& T = c->tree;
  // default: the lockstep kernel; FMMBEM_M2L_WARPS = 1 selects the independent-warp kernel (cross-check)
  static const bool indep = [] {
    const char* e = std::getenv("FMMBEM_M2L_WARPS");
    return e && std::atoi(e) == 1;
  }();
#define FMM_ROT_CASE(PP)                                                                                   \
  case PP:                                                                                                 \
    if (!indep) {                                                                                          \
      constexpr int W = m2l_warps(PP), NREG = m2l_nreg(PP);                                               \
      m2l_sync_launch<PP, W, NREG>(w, T, c, (size_t)W * (m2l_nc(PP) - NREG) * 33 * sizeof(float2), st);   \
    } else {                                                                                               \
      k_m2l_rot<PP, 1><<<(int)w.rows, 32, 0, st>>>((int)w.rows, w.cell.get(), w.off.get(), w.idx.get(),   \
                                                   c->slot_keys(), c->Mx.get(), c->Lx.get());              \
    }                                                                                                      \
    break;
  switch (c->P) {
    FMM_ROT_CASE(8) FMM_ROT_CASE(10) FMM_ROT_CASE(12) FMM_ROT_CASE(13) FMM_ROT_CASE(14)
    default: throw Error(FMMBEM_E_INVALID, "rotation M2L not instantiated for this P");
  }
#undef FMM_ROT_CASE
  FMM_CHECK_LAUNCH();
}

}  // namespace fmm
