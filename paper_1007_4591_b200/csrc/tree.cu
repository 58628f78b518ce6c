// tree.cu -- GPU octree by Morton sort.
//
// Uniform-depth sparse octree (reading A10): the leaf level L is the smallest level at
// which the mean number of panels per occupied leaf is <= leaf_points; empty cells are
// pruned.  Keys interleave 21 bits per axis, x least significant.  The root
// cube is the bounding cube of centroids and charges, widened by 1e-6 and
// rounded up to an 8-bit mantissa so that every integer multiple of a cell width below
// 2^16 is exact in FP32 (leaf-local coordinates).
// Lists: neighbours = same-level cells with max |d ijk| <= 1 (incl. self);
// interaction list = children of the parent's neighbours that are not neighbours.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "ctx.h"
#include "kernels.cuh"

namespace fmm {

namespace {

__device__ inline int lower_bound_u64(const uint64_t* a, int n, uint64_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ inline int lower_bound_shift(const uint64_t* a, int n, uint64_t v, int shift) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if ((a[mid] >> shift) < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ inline int find_u64(const uint64_t* a, int n, uint64_t v) {
  int i = lower_bound_u64(a, n, v);
  return (i < n && a[i] == v) ? i : -1;
}

__global__ void k_bbox_partial(int64_t n, const double* __restrict__ p, double* out) {
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < 3; ++d) {
      double v = p[3 * i + d];
      mn[d] = fmin(mn[d], v);
      mx[d] = fmax(mx[d], v);
    }
  __shared__ double s[6][256];
  for (int d = 0; d < 3; ++d) { s[d][threadIdx.x] = mn[d]; s[3 + d][threadIdx.x] = mx[d]; }
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int d = 0; d < 3; ++d) {
        s[d][threadIdx.x] = fmin(s[d][threadIdx.x], s[d][threadIdx.x + w]);
        s[3 + d][threadIdx.x] = fmax(s[3 + d][threadIdx.x], s[3 + d][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int d = 0; d < 6; ++d) out[blockIdx.x * 6 + d] = s[d][0];
}

__global__ void k_keys21(int64_t n, const double* __restrict__ p, double x0, double y0, double z0,
                         double inv_h, uint64_t* key, int* idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lim = (double)((1 << MAX_LEVEL) - 1);
  double gx = fmin(fmax(floor((p[3 * i] - x0) * inv_h), 0.0), lim);
  double gy = fmin(fmax(floor((p[3 * i + 1] - y0) * inv_h), 0.0), lim);
  double gz = fmin(fmax(floor((p[3 * i + 2] - z0) * inv_h), 0.0), lim);
  key[i] = morton((uint32_t)gx, (uint32_t)gy, (uint32_t)gz);
  idx[i] = (int)i;
}

// hist[l] += number of i with keys first differing from key[i-1] at level l
__global__ void k_level_hist(int64_t n, const uint64_t* __restrict__ k, unsigned long long* hist) {
  __shared__ unsigned int sh[MAX_LEVEL + 1];
  if (threadIdx.x <= MAX_LEVEL) sh[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = k[i] ^ k[i - 1];
    if (x) {
      int b = 63 - __clzll((long long)x);
      int l0 = MAX_LEVEL - b / 3;
      atomicAdd(&sh[l0], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x <= MAX_LEVEL && sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], (unsigned long long)sh[threadIdx.x]);
}

__global__ void k_shift_keys(int64_t n, const uint64_t* __restrict__ in, int shift, uint64_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] >> shift;
}

__global__ void k_parent_links(int n_child, const uint64_t* __restrict__ ckey, int child_off,
                               int n_par, const uint64_t* __restrict__ pkey, int par_off, int* parent) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_child) return;
  parent[child_off + i] = par_off + lower_bound_u64(pkey, n_par, ckey[i] >> 3);
}

__global__ void k_child_ranges(int n_par, const uint64_t* __restrict__ pkey, int par_off, int n_child,
                               const uint64_t* __restrict__ ckey, int child_off, int* cb, int* ce) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_par) return;
  cb[par_off + i] = child_off + lower_bound_u64(ckey, n_child, pkey[i] << 3);
  ce[par_off + i] = child_off + lower_bound_u64(ckey, n_child, (pkey[i] + 1) << 3);
}

__global__ void k_leaf_ijk(int n, const uint64_t* __restrict__ key, int4* ijk) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x, y, z;
  demorton(key[i], x, y, z);
  ijk[i] = make_int4(x, y, z, 0);
}

// begin[k] = first point (sorted key21) whose leaf key >= leafkey[k]; begin[n_leaves] = n
__global__ void k_set_begin(int nl, const uint64_t* __restrict__ lkey, int np, const uint64_t* __restrict__ pk,
                            int shift, int* begin) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nl) return;
  begin[k] = (k == nl) ? np : lower_bound_shift(pk, np, lkey[k], shift);
}

__global__ void k_point_leaf(int nl, const int* __restrict__ begin, int* leaf) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nl) return;
  for (int i = begin[k]; i < begin[k + 1]; ++i) leaf[i] = k;
}

// panels into tree order with leaf-local FP32 coordinates
__global__ void k_place_panels(int n, const int* __restrict__ perm, const int* __restrict__ leaf,
                               const int4* __restrict__ ijk, const double* __restrict__ cen,
                               const double* __restrict__ nrm, const double* __restrict__ area,
                               double x0, double y0, double z0, double h, float4* pos, float4* nout) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int p = perm[i];
  int4 c = ijk[leaf[i]];
  double cx = x0 + (c.x + 0.5) * h, cy = y0 + (c.y + 0.5) * h, cz = z0 + (c.z + 0.5) * h;
  pos[i] = make_float4((float)(cen[3 * p] - cx), (float)(cen[3 * p + 1] - cy), (float)(cen[3 * p + 2] - cz),
                       (float)area[p]);
  nout[i] = make_float4((float)nrm[3 * p], (float)nrm[3 * p + 1], (float)nrm[3 * p + 2], 0.f);
}

__global__ void k_place_quad(int n, int K, const int* __restrict__ perm, const int* __restrict__ leaf,
                             const int4* __restrict__ ijk, const double* __restrict__ qp,
                             const double* __restrict__ area, const double* __restrict__ wq, double x0,
                             double y0, double z0, double h, float4* pos, int* qleaf) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * K) return;
  int i = t / K, g = t - i * K;
  int p = perm[i];
  int4 c = ijk[leaf[i]];
  double cx = x0 + (c.x + 0.5) * h, cy = y0 + (c.y + 0.5) * h, cz = z0 + (c.z + 0.5) * h;
  const double* y = qp + ((size_t)p * K + g) * 3;
  pos[t] = make_float4((float)(y[0] - cx), (float)(y[1] - cy), (float)(y[2] - cz), (float)(area[p] * wq[g]));
  qleaf[t] = leaf[i];
}

__global__ void k_place_charges(int n, const int* __restrict__ perm, const int* __restrict__ leaf,
                                const int4* __restrict__ ijk, const double* __restrict__ xyz,
                                const double* __restrict__ q, double x0, double y0, double z0, double h,
                                float4* pos) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int p = perm[i];
  int4 c = ijk[leaf[i]];
  double cx = x0 + (c.x + 0.5) * h, cy = y0 + (c.y + 0.5) * h, cz = z0 + (c.z + 0.5) * h;
  pos[i] = make_float4((float)(xyz[3 * p] - cx), (float)(xyz[3 * p + 1] - cy), (float)(xyz[3 * p + 2] - cz),
                       (float)q[p]);
}

// exact duplicate centroids (same key21 run) -> flag
__global__ void k_dup_check(int n, const uint64_t* __restrict__ k, const int* __restrict__ perm,
                            const double* __restrict__ cen, int* flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int p = perm[i];
  for (int j = i - 1, c = 0; j >= 0 && k[j] == k[i] && c < 64; --j, ++c) {
    int q = perm[j];
    if (cen[3 * p] == cen[3 * q] && cen[3 * p + 1] == cen[3 * q + 1] && cen[3 * p + 2] == cen[3 * q + 2])
      atomicMin(flag, min(p, q));
  }
}

__global__ void k_leaf_counts(int nl, const int* __restrict__ begin, int mult, int leaf_off, int* cnt) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nl) cnt[leaf_off + k] = (begin[k + 1] - begin[k]) * mult;
}

__global__ void k_up_counts(int n, int off, const int* __restrict__ cb, const int* __restrict__ ce, int* cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = 0;
  for (int c = cb[off + i]; c < ce[off + i]; ++c) s += cnt[c];
  cnt[off + i] = s;
}

// neighbour lists at the leaf level (pass 0: count, pass 1: fill)
__global__ void k_nbr(int nl, const uint64_t* __restrict__ lkey, const int4* __restrict__ ijk, int L,
                      const int* __restrict__ off, int* cnt_or_idx, int pass) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nl) return;
  int4 c = ijk[k];
  int lim = 1 << L;
  int o = pass ? off[k] : 0, m = 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int x = c.x + dx, y = c.y + dy, z = c.z + dz;
        if (x < 0 || y < 0 || z < 0 || x >= lim || y >= lim || z >= lim) continue;
        int j = find_u64(lkey, nl, morton(x, y, z));
        if (j < 0) continue;
        if (pass) cnt_or_idx[o + m] = j;
        ++m;
      }
  if (!pass) cnt_or_idx[k] = m;
}

// interaction lists for the cells of one level l >= 2 (pass 0: count, pass 1: fill)
__global__ void k_m2l_list(int n, const uint64_t* __restrict__ key, int lvl_off, int par_n,
                           const uint64_t* __restrict__ pkey, int par_off, const int* __restrict__ cb,
                           const int* __restrict__ ce, const uint64_t* __restrict__ allkey, int l,
                           const int* __restrict__ off, int* cnt_or_idx, int pass) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x, y, z;
  demorton(key[i], x, y, z);
  int px = x >> 1, py = y >> 1, pz = z >> 1;
  int lim = 1 << (l - 1);
  int o = pass ? off[lvl_off + i] : 0, m = 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int qx = px + dx, qy = py + dy, qz = pz + dz;
        if (qx < 0 || qy < 0 || qz < 0 || qx >= lim || qy >= lim || qz >= lim) continue;
        int pj = find_u64(pkey, par_n, morton(qx, qy, qz));
        if (pj < 0) continue;
        for (int c = cb[par_off + pj]; c < ce[par_off + pj]; ++c) {
          int cx, cy, cz;
          demorton(allkey[c], cx, cy, cz);
          if (abs(cx - x) <= 1 && abs(cy - y) <= 1 && abs(cz - z) <= 1) continue;
          if (pass) cnt_or_idx[o + m] = c;
          ++m;
        }
      }
  if (!pass) cnt_or_idx[lvl_off + i] = m;
}

template <class T>
void exclusive_scan(const T* in, T* out, int n, cudaStream_t s) {
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s);
  DevBuf<unsigned char> tmp;
  tmp.alloc(tb);
  cub::DeviceScan::ExclusiveSum(tmp.get(), tb, in, out, n, s);
}

void sort_pairs(DevBuf<uint64_t>& kin, DevBuf<int>& vin, DevBuf<uint64_t>& kout, DevBuf<int>& vout, int64_t n,
                cudaStream_t s) {
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.get(), kout.get(), vin.get(), vout.get(), (int)n, 0, 63, s);
  DevBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(tb, 1));
  FMM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, kin.get(), kout.get(), vin.get(), vout.get(), (int)n,
                                           0, 63, s));
}

int64_t unique_sorted(const uint64_t* in, uint64_t* out, int64_t n, cudaStream_t s) {
  DevBuf<int> nsel;
  nsel.alloc(1);
  size_t tb = 0;
  cub::DeviceSelect::Unique(nullptr, tb, in, out, nsel.get(), (int)n, s);
  DevBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(tb, 1));
  FMM_CUDA(cub::DeviceSelect::Unique(tmp.get(), tb, in, out, nsel.get(), (int)n, s));
  int h = 0;
  FMM_CUDA(cudaMemcpyAsync(&h, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  return h;
}

void sort_keys(DevBuf<uint64_t>& kin, DevBuf<uint64_t>& kout, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb, kin.get(), kout.get(), (int)n, 0, 63, s);
  DevBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(tb, 1));
  FMM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), tb, kin.get(), kout.get(), (int)n, 0, 63, s));
}

void bbox(const double* p, int64_t n, double mn[3], double mx[3], cudaStream_t s) {
  if (n == 0) return;
  int blocks = std::min<int64_t>(1024, (n + 255) / 256);
  DevBuf<double> part;
  part.alloc(blocks * 6);
  k_bbox_partial<<<blocks, 256, 0, s>>>(n, p, part.get());
  FMM_CHECK_LAUNCH();
  std::vector<double> h(blocks * 6);
  FMM_CUDA(cudaMemcpyAsync(h.data(), part.get(), blocks * 6 * sizeof(double), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < blocks; ++b)
    for (int d = 0; d < 3; ++d) {
      mn[d] = std::min(mn[d], h[b * 6 + d]);
      mx[d] = std::max(mx[d], h[b * 6 + 3 + d]);
    }
}

}  // namespace

void scan_ints(const int* in, int* out, int n, cudaStream_t s) { exclusive_scan(in, out, n, s); }

// Device-side inputs of the tree build (FP64, caller order).
void build_tree(fmmbem_ctx* c, const double* cen, const double* nrm, const double* area, const double* qpts,
                const double* wq, const double* cxyz, const double* cq, cudaStream_t s) {
  Tree& T = c->tree;
  const int64_t np = c->np, nc = c->nc;
  const int TB = 256;
  // 1. root cube
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  bbox(cen, np, mn, mx, s);
  bbox(cxyz, nc, mn, mx, s);
  double ext = std::max(mx[0] - mn[0], std::max(mx[1] - mn[1], mx[2] - mn[2]));
  if (!(ext > 0)) ext = 1.0;
  double Wr = ext * (1.0 + 1e-6) + 1e-300;
  int e;
  double m = std::frexp(Wr, &e);
  m = std::ceil(m * 256.0) / 256.0;
  T.W = std::ldexp(m, e);
  for (int d = 0; d < 3; ++d) T.x0[d] = 0.5 * (mn[d] + mx[d]) - 0.5 * T.W;
  const double inv_h21 = (double)(1 << MAX_LEVEL) / T.W;

  // 2. Morton keys at depth 21 + stable radix sort
  DevBuf<uint64_t> kp_in, kp;
  DevBuf<int> ip_in, pperm;
  kp_in.alloc(np); kp.alloc(np); ip_in.alloc(np); pperm.alloc(np);
  k_keys21<<<ceil_div(np, TB), TB, 0, s>>>(np, cen, T.x0[0], T.x0[1], T.x0[2], inv_h21, kp_in.get(), ip_in.get());
  FMM_CHECK_LAUNCH();
  sort_pairs(kp_in, ip_in, kp, pperm, np, s);
  kp_in.release(); ip_in.release();
  DevBuf<uint64_t> kc_in, kc;
  DevBuf<int> ic_in, cperm;
  if (nc) {
    kc_in.alloc(nc); kc.alloc(nc); ic_in.alloc(nc); cperm.alloc(nc);
    k_keys21<<<ceil_div(nc, TB), TB, 0, s>>>(nc, cxyz, T.x0[0], T.x0[1], T.x0[2], inv_h21, kc_in.get(), ic_in.get());
    FMM_CHECK_LAUNCH();
    sort_pairs(kc_in, ic_in, kc, cperm, nc, s);
    kc_in.release(); ic_in.release();
  }
  // duplicate centroids
  c->flag.alloc(4);
  int big = 0x7fffffff;
  FMM_CUDA(cudaMemcpyAsync(c->flag.get(), &big, sizeof(int), cudaMemcpyHostToDevice, s));
  k_dup_check<<<ceil_div(np, TB), TB, 0, s>>>((int)np, kp.get(), pperm.get(), cen, c->flag.get());
  FMM_CHECK_LAUNCH();
  int dup = 0;
  FMM_CUDA(cudaMemcpyAsync(&dup, c->flag.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  if (dup != big) throw Error(FMMBEM_E_COINCIDENT, "duplicate panel centroid at triangle " + std::to_string(dup));

  // 3. leaf level
  DevBuf<unsigned long long> hist;
  hist.alloc(MAX_LEVEL + 1);
  hist.zero(s);
  k_level_hist<<<std::min(1024, ceil_div(np, TB)) + 1, TB, 0, s>>>(np, kp.get(), hist.get());
  FMM_CHECK_LAUNCH();
  unsigned long long hh[MAX_LEVEL + 1];
  FMM_CUDA(cudaMemcpyAsync(hh, hist.get(), sizeof(hh), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  int L = MAX_LEVEL;
  unsigned long long cells = 1;
  for (int l = 0; l <= MAX_LEVEL; ++l) {
    cells += hh[l];
    if ((double)np / (double)cells <= (double)c->opt.leaf_points) { L = l; break; }
  }
  T.L = L;
  const int shift = 3 * (MAX_LEVEL - L);

  // 4. leaf keys = unique(keysL(panels) U keysL(charges))
  int64_t nall = np + nc;
  DevBuf<uint64_t> lk_in, lk_sorted;
  lk_in.alloc(nall); lk_sorted.alloc(nall);
  k_shift_keys<<<ceil_div(np, TB), TB, 0, s>>>(np, kp.get(), shift, lk_in.get());
  if (nc) k_shift_keys<<<ceil_div(nc, TB), TB, 0, s>>>(nc, kc.get(), shift, lk_in.get() + np);
  FMM_CHECK_LAUNCH();
  sort_keys(lk_in, lk_sorted, nall, s);
  std::vector<DevBuf<uint64_t>> lvl(L + 1);
  std::vector<int64_t> nlev(L + 1);
  lvl[L].alloc(nall);
  nlev[L] = unique_sorted(lk_sorted.get(), lvl[L].get(), nall, s);
  lk_in.release(); lk_sorted.release();
  for (int l = L - 1; l >= 0; --l) {
    DevBuf<uint64_t> tmp;
    tmp.alloc(nlev[l + 1]);
    k_shift_keys<<<ceil_div(nlev[l + 1], TB), TB, 0, s>>>(nlev[l + 1], lvl[l + 1].get(), 3, tmp.get());
    FMM_CHECK_LAUNCH();
    lvl[l].alloc(nlev[l + 1]);
    nlev[l] = unique_sorted(tmp.get(), lvl[l].get(), nlev[l + 1], s);
  }
  T.lvl_off.assign(L + 2, 0);
  for (int l = 0; l <= L; ++l) T.lvl_off[l + 1] = T.lvl_off[l] + nlev[l];
  T.n_cells = T.lvl_off[L + 1];
  T.n_leaves = nlev[L];
  const int nl = (int)T.n_leaves;
  T.key.alloc(T.n_cells);
  for (int l = 0; l <= L; ++l)
    FMM_CUDA(cudaMemcpyAsync(T.key.get() + T.lvl_off[l], lvl[l].get(), nlev[l] * sizeof(uint64_t),
                             cudaMemcpyDeviceToDevice, s));
  // 5. parent / child links
  T.parent.alloc(T.n_cells);
  T.child_begin.alloc(T.n_cells);
  T.child_end.alloc(T.n_cells);
  int m1 = -1;
  FMM_CUDA(cudaMemcpyAsync(T.parent.get(), &m1, sizeof(int), cudaMemcpyHostToDevice, s));
  for (int l = 1; l <= L; ++l)
    k_parent_links<<<ceil_div(nlev[l], TB), TB, 0, s>>>((int)nlev[l], lvl[l].get(), (int)T.lvl_off[l],
                                                        (int)nlev[l - 1], lvl[l - 1].get(), (int)T.lvl_off[l - 1],
                                                        T.parent.get());
  for (int l = 0; l < L; ++l)
    k_child_ranges<<<ceil_div(nlev[l], TB), TB, 0, s>>>((int)nlev[l], lvl[l].get(), (int)T.lvl_off[l],
                                                        (int)nlev[l + 1], lvl[l + 1].get(), (int)T.lvl_off[l + 1],
                                                        T.child_begin.get(), T.child_end.get());
  {
    // leaves have no children
    std::vector<int> z(nl, 0);
    FMM_CUDA(cudaMemcpyAsync(T.child_begin.get() + T.lvl_off[L], z.data(), nl * sizeof(int), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaMemcpyAsync(T.child_end.get() + T.lvl_off[L], z.data(), nl * sizeof(int), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  FMM_CHECK_LAUNCH();
  T.leaf_ijk.alloc(nl);
  k_leaf_ijk<<<ceil_div(nl, TB), TB, 0, s>>>(nl, lvl[L].get(), T.leaf_ijk.get());
  FMM_CHECK_LAUNCH();

  // 6. point sets
  const double h = T.width(L);
  auto& P = c->pan;
  P.n = np;
  P.begin.alloc(nl + 1);
  P.leaf.alloc(np);
  P.pos.alloc(np);
  P.nrm.alloc(np);
  k_set_begin<<<ceil_div(nl + 1, TB), TB, 0, s>>>(nl, lvl[L].get(), (int)np, kp.get(), shift, P.begin.get());
  k_point_leaf<<<ceil_div(nl, TB), TB, 0, s>>>(nl, P.begin.get(), P.leaf.get());
  k_place_panels<<<ceil_div(np, TB), TB, 0, s>>>((int)np, pperm.get(), P.leaf.get(), T.leaf_ijk.get(), cen, nrm,
                                                 area, T.x0[0], T.x0[1], T.x0[2], h, P.pos.get(), P.nrm.get());
  FMM_CHECK_LAUNCH();
  P.div = 1;
  if (c->K > 1) {
    auto& Q = c->quad;
    const int K = c->K;
    Q.n = np * K;
    Q.div = K;
    Q.pos.alloc(Q.n);
    Q.leaf.alloc(Q.n);
    Q.begin.alloc(nl + 1);
    k_place_quad<<<ceil_div(Q.n, TB), TB, 0, s>>>((int)np, K, pperm.get(), P.leaf.get(), T.leaf_ijk.get(), qpts,
                                                  area, wq, T.x0[0], T.x0[1], T.x0[2], h, Q.pos.get(), Q.leaf.get());
    FMM_CHECK_LAUNCH();
    std::vector<int> b(nl + 1);
    FMM_CUDA(cudaMemcpyAsync(b.data(), P.begin.get(), (nl + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    for (auto& v : b) v *= K;
    FMM_CUDA(cudaMemcpyAsync(Q.begin.get(), b.data(), (nl + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  auto& C = c->chg;
  C.n = nc;
  C.begin.alloc(nl + 1);
  if (nc) {
    C.pos.alloc(nc);
    C.leaf.alloc(nc);
    k_set_begin<<<ceil_div(nl + 1, TB), TB, 0, s>>>(nl, lvl[L].get(), (int)nc, kc.get(), shift, C.begin.get());
    k_point_leaf<<<ceil_div(nl, TB), TB, 0, s>>>(nl, C.begin.get(), C.leaf.get());
    k_place_charges<<<ceil_div(nc, TB), TB, 0, s>>>((int)nc, cperm.get(), C.leaf.get(), T.leaf_ijk.get(), cxyz, cq,
                                                    T.x0[0], T.x0[1], T.x0[2], h, C.pos.get());
    FMM_CHECK_LAUNCH();
    c->chg_ids.alloc(nc);
    FMM_CUDA(cudaMemcpyAsync(c->chg_ids.get(), cperm.get(), nc * sizeof(int), cudaMemcpyDeviceToDevice, s));
  } else {
    C.begin.zero(s);
  }
  // caller ids of the panels
  {
    std::vector<int> pm(np);
    FMM_CUDA(cudaMemcpyAsync(pm.data(), pperm.get(), np * sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    c->pan_ids.assign(pm.begin(), pm.end());
  }
  // subtree counts
  for (PointSet* S : {&c->pan, &c->quad, &c->chg}) {
    if (S == &c->quad && c->K == 1) continue;
    S->cell_cnt.alloc(T.n_cells);
    k_leaf_counts<<<ceil_div(nl, TB), TB, 0, s>>>(nl, (S == &c->quad ? c->pan.begin.get() : S->begin.get()),
                                                  S == &c->quad ? c->K : 1, (int)T.lvl_off[L], S->cell_cnt.get());
    for (int l = L - 1; l >= 0; --l)
      k_up_counts<<<ceil_div(nlev[l], TB), TB, 0, s>>>((int)nlev[l], (int)T.lvl_off[l], T.child_begin.get(),
                                                       T.child_end.get(), S->cell_cnt.get());
    FMM_CHECK_LAUNCH();
  }

  // 7. neighbour lists (leaf level)
  {
    DevBuf<int> cnt;
    cnt.alloc(nl + 1);
    cnt.zero(s);
    k_nbr<<<ceil_div(nl, TB), TB, 0, s>>>(nl, lvl[L].get(), T.leaf_ijk.get(), L, nullptr, cnt.get(), 0);
    FMM_CHECK_LAUNCH();
    T.nbr_off.alloc(nl + 1);
    exclusive_scan(cnt.get(), T.nbr_off.get(), nl + 1, s);
    int tot = 0;
    FMM_CUDA(cudaMemcpyAsync(&tot, T.nbr_off.get() + nl, sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    T.nbr_pairs = tot;
    T.nbr_idx.alloc(std::max(tot, 1));
    k_nbr<<<ceil_div(nl, TB), TB, 0, s>>>(nl, lvl[L].get(), T.leaf_ijk.get(), L, T.nbr_off.get(), T.nbr_idx.get(), 1);
    FMM_CHECK_LAUNCH();
  }
  // 8. interaction lists, levels 2..L
  {
    int nC = (int)T.n_cells;
    DevBuf<int> cnt;
    cnt.alloc(nC + 1);
    cnt.zero(s);
    for (int l = 2; l <= L; ++l)
      k_m2l_list<<<ceil_div(nlev[l], TB), TB, 0, s>>>((int)nlev[l], lvl[l].get(), (int)T.lvl_off[l], (int)nlev[l - 1],
                                                      lvl[l - 1].get(), (int)T.lvl_off[l - 1], T.child_begin.get(),
                                                      T.child_end.get(), T.key.get(), l, nullptr, cnt.get(), 0);
    FMM_CHECK_LAUNCH();
    T.m2l_off.alloc(nC + 1);
    exclusive_scan(cnt.get(), T.m2l_off.get(), nC + 1, s);
    int tot = 0;
    FMM_CUDA(cudaMemcpyAsync(&tot, T.m2l_off.get() + nC, sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    T.m2l_pairs = tot;
    T.m2l_idx.alloc(std::max(tot, 1));
    for (int l = 2; l <= L; ++l)
      k_m2l_list<<<ceil_div(nlev[l], TB), TB, 0, s>>>((int)nlev[l], lvl[l].get(), (int)T.lvl_off[l], (int)nlev[l - 1],
                                                      lvl[l - 1].get(), (int)T.lvl_off[l - 1], T.child_begin.get(),
                                                      T.child_end.get(), T.key.get(), l, T.m2l_off.get(),
                                                      T.m2l_idx.get(), 1);
    FMM_CHECK_LAUNCH();
  }
  FMM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace fmm
