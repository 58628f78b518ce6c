// dipole.cu -- the double-layer operator K (SURVEY 8(f) NEXT-4 "true double-layer K (dipole
// sources, needed for Green's-representation formulations)"): y_i = sum_{j != i} x_j A_j sum_g w_g
// dG/dn_y(c_i, y_jg) with n_y the SOURCE panel's normal -- the continuum adjoint of the K' of
// Eq. 4.  The far field reuses every expansion kernel: a dipole of moment p = w n at y has
// the potential p . grad_y (1/|x - y|) = sum_{n,m} conj(p . grad R_n^m(y - c)) I_n^m(x - c)
// (farfield.cu's expansion), so only P2M changes:
//   M~_n^m = (1/w_cell) sum_j w_j conj(n_j . grad_u R_n^m(u_j)),
//   n . grad R_n^m = n_z R_{n-1}^m + (n_x - i n_y)/2 R_{n-1}^{m+1} - (n_x + i n_y)/2 R_{n-1}^{m-1}
// (dz R_n^m = R_{n-1}^m, dx R_n^m = (R_{n-1}^{m+1} - R_{n-1}^{m-1})/2, dy R_n^m = -i (R_{n-1}^{m+1} +
// R_{n-1}^{m-1})/2; R_n^{-m} = (-1)^m conj R_n^m).  The near field sums p . (x - s) / |x - s|^3.
// An option of the library (not the paper's hot path): plain kernels, one warp per work item.
#include "kernels.cuh"

namespace fmm {

namespace {

__host__ __device__ inline int dcx(int n, int m) { return n * (n + 1) / 2 + m; }

__device__ __forceinline__ float2 dgetc(const float2* R, int n, int m) {  // R_n^m for any m, 0 if |m| > n
  if (n < 0 || m > n || -m > n) return make_float2(0.f, 0.f);
  if (m >= 0) return R[dcx(n, m)];
  const float2 v = R[dcx(n, -m)];
  return (m & 1) ? make_float2(-v.x, v.y) : make_float2(v.x, -v.y);
}

// P2M of dipole sources: CTA (128 threads) per leaf; per source the regular harmonics of degrees
// < P - 1 are tabulated in shared memory (thread m: column m), then thread c accumulates its
// coefficient (n, m) (fixed source order: deterministic)
__global__ void __launch_bounds__(128) k_p2m_dipole(const float4* __restrict__ pos, const float4* __restrict__ nrm,
                                                    const float* __restrict__ x, int div, const int* __restrict__ beg,
                                                    int P, float inv_w, int leaf_off, int leaf0, float2* __restrict__ M) {
  __shared__ float2 R[MAX_TERMS * (MAX_TERMS + 1) / 2];
  __shared__ float4 su, sn;
  const int leaf = leaf0 + blockIdx.x;
  const int b = beg[leaf], e = beg[leaf + 1];
  if (b == e) return;
  const int NC = P * (P + 1) / 2;
  float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  for (int j = b; j < e; ++j) {
    if (threadIdx.x == 0) {
      const float4 p = pos[j];
      float w = p.w;
      if (x) w *= x[div == 1 ? j : j / div];
      su = make_float4(p.x * inv_w, p.y * inv_w, p.z * inv_w, w * inv_w);
      sn = nrm[j / div];
    }
    __syncthreads();
    const int m = threadIdx.x;
    if (m < P - 1) {  // column m: R_m^m = (-(x + iy)/2)^m / m!, then the degree recurrence
      const float r2 = su.x * su.x + su.y * su.y + su.z * su.z;
      float2 r = make_float2(1.f, 0.f);
      for (int k = 1; k <= m; ++k) {
        const float s = -0.5f / (float)k;
        r = make_float2(s * (r.x * su.x - r.y * su.y), s * (r.x * su.y + r.y * su.x));
      }
      float2 rm2 = make_float2(0.f, 0.f), rm1 = r;
      R[dcx(m, m)] = r;
      for (int n = m + 1; n < P - 1; ++n) {
        const float inv = 1.f / (float)((n - m) * (n + m));
        const float a = (float)(2 * n - 1) * su.z;
        const float2 rn = make_float2((a * rm1.x - r2 * rm2.x) * inv, (a * rm1.y - r2 * rm2.y) * inv);
        R[dcx(n, m)] = rn;
        rm2 = rm1;
        rm1 = rn;
      }
    }
    __syncthreads();
    for (int q = 0; q < 2; ++q) {
      const int c = threadIdx.x + 128 * q;
      if (c >= NC) break;
      int n = 0;
      while (dcx(n + 1, 0) <= c) ++n;
      const int mm = c - dcx(n, 0);
      if (n == 0) continue;  // a dipole has no monopole moment
      const float2 Rz = dgetc(R, n - 1, mm), Ra = dgetc(R, n - 1, mm + 1), Rb = dgetc(R, n - 1, mm - 1);
      // g = n_z Rz + (n_x - i n_y)/2 Ra - (n_x + i n_y)/2 Rb ; acc += w conj(g)
      const float gx = sn.z * Rz.x + 0.5f * (sn.x * Ra.x + sn.y * Ra.y) - 0.5f * (sn.x * Rb.x - sn.y * Rb.y);
      const float gy = sn.z * Rz.y + 0.5f * (sn.x * Ra.y - sn.y * Ra.x) - 0.5f * (sn.x * Rb.y + sn.y * Rb.x);
      acc[q].x = fmaf(su.w, gx, acc[q].x);
      acc[q].y = fmaf(-su.w, gy, acc[q].y);
    }
    __syncthreads();
  }
  for (int q = 0; q < 2; ++q) {
    const int c = threadIdx.x + 128 * q;
    if (c < NC) M[(size_t)(leaf_off + leaf) * NC + c] = acc[q];
  }
}

// Near field: warp per (leaf, target chunk) item, lane per target (chunk <= 64: two per lane);
// sources of the neighbour leaves read through the read-only cache in list order (fixed order).
__global__ void __launch_bounds__(32) k_p2p_dipole(const int4* __restrict__ items, const float4* __restrict__ tpos,
                                                   const float4* __restrict__ spos, const float4* __restrict__ nrm,
                                                   const float* __restrict__ x, int div, const int* __restrict__ sbeg,
                                                   const int* __restrict__ nbr_off, const int* __restrict__ nbr_idx,
                                                   const int4* __restrict__ ijk, const int* __restrict__ sleaf,
                                                   int direct, int ns, float h, float b, float* __restrict__ y) {
  const int4 it = items[blockIdx.x];
  const int leaf = it.x, tb = it.y, nt = it.z;
  const int4 tc = ijk[leaf];
  const int lane = threadIdx.x;
  float tx[2], ty[2], tz[2], acc[2] = {0.f, 0.f};
  int ti[2];
  for (int q = 0; q < 2; ++q) {
    const int il = lane + 32 * q;
    ti[q] = tb + (il < nt ? il : 0);
    const float4 p = tpos[ti[q]];
    tx[q] = p.x;
    ty[q] = p.y;
    tz[q] = p.z;
  }
  const int ne = direct ? 1 : nbr_off[leaf + 1] - nbr_off[leaf];
  for (int e = 0; e < ne; ++e) {  // direct mode (all pairs): one pass over every source
    const int s = direct ? 0 : nbr_idx[nbr_off[leaf] + e];
    const int4 sc = direct ? tc : ijk[s];
    float shx = (sc.x - tc.x) * h, shy = (sc.y - tc.y) * h, shz = (sc.z - tc.z) * h;
    const int j0 = direct ? 0 : sbeg[s], j1 = direct ? ns : sbeg[s + 1];
    for (int j = j0; j < j1; ++j) {
      if (direct) {
        const int4 q = ijk[sleaf[j]];
        shx = (q.x - tc.x) * h;
        shy = (q.y - tc.y) * h;
        shz = (q.z - tc.z) * h;
      }
      const float4 p = __ldg(spos + j);
      const float4 n = __ldg(nrm + j / div);
      float w = p.w;
      if (x) w *= __ldg(x + (div == 1 ? j : j / div));
      const int own = j / div;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (own == ti[q]) continue;  // j != i (flat panel: K_ii = 0)
        const float dx = tx[q] - (p.x + shx), dy = ty[q] - (p.y + shy), dz = tz[q] - (p.z + shz);
        const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        const float ri = rsqrtf(r2);
        acc[q] = fmaf(w * ri * ri * ri, fmaf(n.x, dx, fmaf(n.y, dy, n.z * dz)), acc[q]);
      }
    }
  }
  for (int q = 0; q < 2; ++q)
    if (lane + 32 * q < nt) y[ti[q]] = b * acc[q];
}

}  // namespace

void launch_p2m_dipole(fmmbem_ctx* c, const SrcArg& s, int lo, int hi, cudaStream_t st) {
  const Tree& T = c->tree;
  if (T.L < 2 || hi <= lo) return;
  if (c->P > 16 || c->P * (c->P + 1) / 2 > 256) throw Error(FMMBEM_E_INVALID, "dipole P2M: terms too large");
  check_leaf_window(c, lo, hi);
  k_p2m_dipole<<<hi - lo, 128, 0, st>>>(s.set->pos.get(), c->pan.nrm.get(), s.x, s.set->div, s.set->begin.get(),
                                        c->P, (float)(1.0 / T.width(T.L)), (int)T.lvl_off[T.L], lo,
                                        c->lvl_ptr(c->Mx.get(), T.L));
  FMM_CHECK_LAUNCH();
}

void launch_p2p_dipole(fmmbem_ctx* c, const TgtArg& t, const SrcArg& s, float* y, float b, bool direct,
                       cudaStream_t st) {
  const Tree& T = c->tree;
  const P2PItems& items = p2p_items(c, *t.set, t.leaf_lo, t.leaf_hi < 0 ? (int)T.n_leaves : t.leaf_hi, 64);
  if (items.n == 0) return;
  k_p2p_dipole<<<(int)items.n, 32, 0, st>>>(items.items.get(), t.set->pos.get(), s.set->pos.get(), c->pan.nrm.get(),
                                            s.x, s.set->div, s.set->begin.get(), T.nbr_off.get(), T.nbr_idx.get(),
                                            T.leaf_ijk.get(), s.set->leaf.get(), direct ? 1 : 0, (int)s.set->n,
                                            (float)T.width(T.L), b, y);
  FMM_CHECK_LAUNCH();
}

}  // namespace fmm
