// p2p.cu -- near-field direct sums ("the near field
// contribution is obtained from directly computing the interactions between all the points
// in the adjacent cells", "P2P ... the largest fractions").
//
// One CTA per target leaf.  The sources of the (<= 27) neighbour leaves are streamed through
// shared memory in tiles, already shifted into the target leaf's frame: offsets between
// leaf centres are exact multiples of the leaf width (FP32-exact), so the
// subtraction s - x involves two numbers of leaf size only.  Every warp reads one source per
// step (broadcast LDS.128); threads own targets (no atomics, fixed summation order).  When a
// leaf has fewer targets than threads, the sources are split between thread groups and the
// partial sums reduced in shared memory (split-K).  The self-leaf block is the only masked
// block (j != i of the discrete operator).
//
// Raw outputs, un-normalised potential phi = sum_j w_j / r_ij:
//   pot = phi(x_i),   dn = n_i . grad phi(x_i) = n_i . sum_j w_j (y_j - x_i) / r^3
// Per interaction (dn only): 3 FADD + 3 (r^2) + 1 MUFU.RSQ + 3 (w r^-3) + 3 FFMA = 12 FP32 + 1 MUFU,
// counted as 19 flops under the SURVEY 8(d) convention.
#include "kernels.cuh"

namespace fmm {

namespace {

constexpr int TPB = 128;
constexpr int TILE = 1024;
constexpr int MAXSEG = 32;

struct P2PArgs {
  const float4* tpos;
  const float4* tnrm;
  const int* tbeg;
  const float4* spos;
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

__device__ __forceinline__ void load_src(const P2PArgs& a, int j, float sx, float sy, float sz, float4* dst) {
  float4 p = __ldg(a.spos + j);
  float w = p.w;
  if (a.sx) w *= __ldg(a.sx + (a.sdiv == 1 ? j : j / a.sdiv));
  *dst = make_float4(p.x + sx, p.y + sy, p.z + sz, w);
}

template <bool POT, bool DN, bool MASK, bool CHECK>
__device__ __forceinline__ void interact(const float4 s, float px, float py, float pz, float& ap, float& gx,
                                         float& gy, float& gz, bool skip, int* flag) {
  float dx = s.x - px, dy = s.y - py, dz = s.z - pz;
  float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  float w = s.w;
  if (CHECK) {
    if (r2 == 0.f) atomicOr(flag, 1);
  }
  if (MASK) {
    w = skip ? 0.f : w;
    r2 = fmaxf(r2, 1e-20f);
  }
  float ri = rsqrtf(r2);
  if (POT) ap = fmaf(w, ri, ap);
  if (DN) {
    float t = w * ri;
    t *= ri * ri;
    gx = fmaf(t, dx, gx);
    gy = fmaf(t, dy, gy);
    gz = fmaf(t, dz, gz);
  }
}

template <bool POT, bool DN, bool SELF, bool CHECK>
__global__ void __launch_bounds__(TPB) k_p2p(P2PArgs a) {
  __shared__ float4 tile[TILE];
  __shared__ int own[SELF ? TILE : 1];
  __shared__ int seg_src[MAXSEG], seg_cum[MAXSEG + 1];
  __shared__ float4 seg_sh[MAXSEG];
  __shared__ float red[4][TPB];
  __shared__ int s_nseg;

  const int leaf = blockIdx.x;
  const int tb = a.tbeg[leaf];
  const int nt = a.tbeg[leaf + 1] - tb;
  if (nt == 0) return;
  const int4 tc = a.ijk[leaf];
  const int tid = threadIdx.x;

  // ---- source segments: neighbour leaves (self last) or, in direct mode, everything
  int n_src, self_lo, self_hi;  // self block = virtual range [self_lo, self_hi)
  if (!a.direct) {
    if (tid < 32) {
      const int o = a.nbr_off[leaf], nn = a.nbr_off[leaf + 1] - o;
      int s = -1, cnt = 0, beg = 0;
      bool valid = tid < nn;
      if (valid) {
        s = a.nbr_idx[o + tid];
        beg = a.sbeg[s];
        cnt = a.sbeg[s + 1] - beg;
      }
      bool is_self = valid && s == leaf;
      unsigned vmask = __ballot_sync(0xffffffffu, valid && !is_self);
      int rank = is_self ? __popc(vmask) : __popc(vmask & ((1u << tid) - 1));
      if (valid) {
        seg_src[rank] = beg;
        int4 sc = a.ijk[s];
        seg_sh[rank] = make_float4((sc.x - tc.x) * a.h, (sc.y - tc.y) * a.h, (sc.z - tc.z) * a.h, 0.f);
      }
      if (valid) seg_cum[rank + 1] = cnt;  // counts in rank order (scanned below)
      __syncwarp();
      int my_cnt = (tid < nn) ? seg_cum[tid + 1] : 0;
      __syncwarp();
      int incl = my_cnt;
      for (int d = 1; d < 32; d <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (tid >= d) incl += v;
      }
      if (tid < nn) seg_cum[tid + 1] = incl;
      if (tid == 0) {
        seg_cum[0] = 0;
        s_nseg = nn;
      }
    }
    __syncthreads();
    const int nn = s_nseg;
    n_src = seg_cum[nn];
    if (SELF) {
      self_lo = seg_cum[nn - 1];
      self_hi = n_src;
    } else {
      self_lo = self_hi = n_src;
    }
  } else {
    n_src = a.ns;
    self_lo = a.sbeg[leaf];
    self_hi = a.sbeg[leaf + 1];
  }

  const int tch = nt <= 32 ? 32 : (nt <= 64 ? 64 : 128);
  const int split = TPB / tch;
  const int lt = tid % tch, grp = tid / tch;

  for (int t0 = 0; t0 < nt; t0 += tch) {
    const int il = t0 + lt;
    const bool tvalid = il < nt;
    const int i = tb + (tvalid ? il : 0);
    float4 tp = a.tpos[i];
    float ap = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;

    for (int base = 0; base < n_src; base += TILE) {
      const int tcnt = min(TILE, n_src - base);
      __syncthreads();
      for (int k = tid; k < tcnt; k += TPB) {
        const int v = base + k;
        int j;
        float sx, sy, sz;
        if (!a.direct) {
          int lo = 0, hi = s_nseg - 1;  // last segment with seg_cum[seg] <= v
          while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (seg_cum[mid] <= v) lo = mid; else hi = mid - 1;
          }
          j = seg_src[lo] + (v - seg_cum[lo]);
          float4 sh = seg_sh[lo];
          sx = sh.x; sy = sh.y; sz = sh.z;
        } else {
          j = v;
          int4 sc = a.ijk[a.sleaf[j]];
          sx = (sc.x - tc.x) * a.h; sy = (sc.y - tc.y) * a.h; sz = (sc.z - tc.z) * a.h;
        }
        load_src(a, j, sx, sy, sz, &tile[k]);
        if (SELF) own[k] = (a.sdiv == 1) ? j : j / a.sdiv;
      }
      __syncthreads();
      // unmasked range of this tile: [0, tcnt) minus the self block
      int mlo = SELF ? min(max(self_lo - base, 0), tcnt) : tcnt;
      int mhi = SELF ? min(max(self_hi - base, 0), tcnt) : tcnt;
      // part 1: [0, mlo) and [mhi, tcnt) unmasked
#pragma unroll 4
      for (int k = grp; k < mlo; k += split)
        interact<POT, DN, false, CHECK>(tile[k], tp.x, tp.y, tp.z, ap, gx, gy, gz, false, a.flag);
      if (SELF) {
        int k0 = mhi + ((grp - mhi) % split + split) % split;
#pragma unroll 4
        for (int k = k0; k < tcnt; k += split)
          interact<POT, DN, false, CHECK>(tile[k], tp.x, tp.y, tp.z, ap, gx, gy, gz, false, a.flag);
        int k1 = mlo + ((grp - mlo) % split + split) % split;
        for (int k = k1; k < mhi; k += split)
          interact<POT, DN, true, CHECK>(tile[k], tp.x, tp.y, tp.z, ap, gx, gy, gz, own[k] == i, a.flag);
      }
    }
    // split-K reduction
    if (split > 1) {
      red[0][tid] = ap;
      red[1][tid] = gx;
      red[2][tid] = gy;
      red[3][tid] = gz;
      __syncthreads();
      if (grp == 0) {
        for (int g = 1; g < split; ++g) {
          ap += red[0][g * tch + lt];
          gx += red[1][g * tch + lt];
          gy += red[2][g * tch + lt];
          gz += red[3][g * tch + lt];
        }
      }
    }
    if (grp == 0 && tvalid) {
      if (POT) {
        float v = a.pot.b * ap;
        if (a.pot.x) v = fmaf(a.pot.ax, a.pot.x[i], v);
        a.pot.y[i] = v;
      }
      if (DN) {
        float4 n = a.tnrm[i];
        float v = a.dn.b * fmaf(n.x, gx, fmaf(n.y, gy, n.z * gz));
        if (a.dn.x) v = fmaf(a.dn.ax, a.dn.x[i], v);
        a.dn.y[i] = v;
      }
    }
  }
}

template <bool SELF, bool CHECK>
void dispatch(const P2PArgs& a, bool pot, bool dn, int grid, cudaStream_t st) {
  if (pot && dn) k_p2p<true, true, SELF, CHECK><<<grid, TPB, 0, st>>>(a);
  else if (pot) k_p2p<true, false, SELF, CHECK><<<grid, TPB, 0, st>>>(a);
  else k_p2p<false, true, SELF, CHECK><<<grid, TPB, 0, st>>>(a);
}

__global__ void k_count(int nl, const int* __restrict__ tbeg, const int* __restrict__ sbeg,
                        const int* __restrict__ off, const int* __restrict__ idx, int direct, int ns, int self,
                        unsigned long long* out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0;
  if (k < nl) {
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

}  // namespace

void launch_p2p(fmmbem_ctx* c, const TgtArg& t, const SrcArg& s, const Outputs& o, bool self, bool check,
                bool direct, cudaStream_t st) {
  const Tree& T = c->tree;
  P2PArgs a{};
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
  const bool pot = o.pot.y != nullptr, dn = o.dn.y != nullptr;
  if (!pot && !dn) return;
  if (dn && !a.tnrm) throw Error(FMMBEM_E_INVALID, "normal derivative requested at targets without normals");
  const int grid = (int)T.n_leaves;
  if (grid == 0) return;
  if (self) {
    if (check) dispatch<true, true>(a, pot, dn, grid, st);
    else dispatch<true, false>(a, pot, dn, grid, st);
  } else {
    if (check) dispatch<false, true>(a, pot, dn, grid, st);
    else dispatch<false, false>(a, pot, dn, grid, st);
  }
  FMM_CHECK_LAUNCH();
}

int64_t count_p2p(fmmbem_ctx* c, const PointSet& t, const PointSet& s, bool self, bool direct) {
  const Tree& T = c->tree;
  DevBuf<unsigned long long> out;
  out.alloc(1);
  out.zero(c->stream);
  int nl = (int)T.n_leaves;
  k_count<<<ceil_div(nl, 256), 256, 0, c->stream>>>(nl, t.begin.get(), s.begin.get(), T.nbr_off.get(),
                                                     T.nbr_idx.get(), direct ? 1 : 0, (int)s.n, self, out.get());
  FMM_CHECK_LAUNCH();
  unsigned long long h = 0;
  FMM_CUDA(cudaMemcpyAsync(&h, out.get(), sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  FMM_CUDA(cudaStreamSynchronize(c->stream));
  int64_t r = (int64_t)h;
  if (self) r -= t.n * s.div;  // own-panel pairs are excluded (j != i)
  return r;
}

}  // namespace fmm
