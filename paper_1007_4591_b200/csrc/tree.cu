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
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

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
                           const long long* __restrict__ off, int* cnt_or_idx, int pass) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x, y, z;
  demorton(key[i], x, y, z);
  int px = x >> 1, py = y >> 1, pz = z >> 1;
  int lim = 1 << (l - 1);
  long long o = pass ? off[lvl_off + i] : 0;
  int m = 0;
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


// ---- distributed build: records of panels moving to their owner rank
// record = [key21, global id, centroid xyz, normal xyz, area, K quadrature points xyz] as 64-bit words
__global__ void k_pack_records(int64_t m, const int* __restrict__ perm, const uint64_t* __restrict__ kp,
                               const double* __restrict__ cen, const double* __restrict__ nrm,
                               const double* __restrict__ area, const double* __restrict__ qp, int K, int64_t gid0,
                               int Wd, unsigned long long* rec) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int p = perm[i];
  unsigned long long* r = rec + i * Wd;
  r[0] = kp[i];
  r[1] = (unsigned long long)(gid0 + p);
  for (int d = 0; d < 3; ++d) {
    r[2 + d] = (unsigned long long)__double_as_longlong(cen[3 * (int64_t)p + d]);
    r[5 + d] = (unsigned long long)__double_as_longlong(nrm[3 * (int64_t)p + d]);
  }
  r[8] = (unsigned long long)__double_as_longlong(area[p]);
  if (qp)
    for (int t = 0; t < 3 * K; ++t) r[9 + t] = (unsigned long long)__double_as_longlong(qp[3 * K * (int64_t)p + t]);
}

__global__ void k_rec_keys(int64_t n, const unsigned long long* __restrict__ rec, int Wd, uint64_t* key, int* idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = rec[i * Wd];
  idx[i] = (int)i;
}

__global__ void k_gather_rec(int64_t n, const int* __restrict__ perm, const unsigned long long* __restrict__ in,
                             int Wd, unsigned long long* out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * Wd) return;
  const int64_t i = t / Wd, w = t - i * Wd;
  out[t] = in[(int64_t)perm[i] * Wd + w];
}

// first index of the sorted key21 array whose leaf key (>> shift) is >= b[k], for every boundary k
__global__ void k_split_points(int64_t m, const uint64_t* __restrict__ kp, int shift, const uint64_t* __restrict__ b,
                               int nb, long long* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((kp[mid] >> shift) < b[k]) lo = mid + 1; else hi = mid;
  }
  out[k] = lo;
}

__device__ inline double rec_d(const unsigned long long* r, int w) { return __longlong_as_double((long long)r[w]); }

// owned panels into tree order with leaf-local FP32 coordinates (leaf = global leaf index)
__global__ void k_place_owned(int n, const unsigned long long* __restrict__ rec, int Wd, const int* __restrict__ leaf,
                              const int4* __restrict__ ijk, double x0, double y0, double z0, double h, float4* pos,
                              float4* nout, long long* gid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long* r = rec + (int64_t)i * Wd;
  const int4 c = ijk[leaf[i]];
  const double cx = x0 + (c.x + 0.5) * h, cy = y0 + (c.y + 0.5) * h, cz = z0 + (c.z + 0.5) * h;
  pos[i] = make_float4((float)(rec_d(r, 2) - cx), (float)(rec_d(r, 3) - cy), (float)(rec_d(r, 4) - cz),
                       (float)rec_d(r, 8));
  nout[i] = make_float4((float)rec_d(r, 5), (float)rec_d(r, 6), (float)rec_d(r, 7), 0.f);
  gid[i] = (long long)r[1];
}

__global__ void k_place_owned_quad(int n, int K, const unsigned long long* __restrict__ rec, int Wd,
                                   const int* __restrict__ leaf, const int4* __restrict__ ijk,
                                   const double* __restrict__ wq, double x0, double y0, double z0, double h,
                                   float4* pos) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * K) return;
  const int i = t / K, g = t - i * K;
  const unsigned long long* r = rec + (int64_t)i * Wd;
  const int4 c = ijk[leaf[i]];
  const double cx = x0 + (c.x + 0.5) * h, cy = y0 + (c.y + 0.5) * h, cz = z0 + (c.z + 0.5) * h;
  pos[t] = make_float4((float)(rec_d(r, 9 + 3 * g) - cx), (float)(rec_d(r, 10 + 3 * g) - cy),
                       (float)(rec_d(r, 11 + 3 * g) - cz), (float)(rec_d(r, 8) * wq[g]));
}

// exact duplicate centroids among the owned panels (equal keys are adjacent) -> smallest global id
__global__ void k_dup_check_rec(int n, const unsigned long long* __restrict__ rec, int Wd, long long* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long* a = rec + (int64_t)i * Wd;
  for (int j = i - 1, c = 0; j >= 0 && c < 64; --j, ++c) {
    const unsigned long long* b = rec + (int64_t)j * Wd;
    if (b[0] != a[0]) break;
    if (a[2] == b[2] && a[3] == b[3] && a[4] == b[4])
      atomicMin(flag, (long long)min(a[1], b[1]));
  }
}

__global__ void k_leaf_rank(int nl, const int* __restrict__ bounds, int R, int* lrank) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nl) return;
  int lo = 0, hi = R - 1;  // last r with bounds[r] <= k
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bounds[mid] <= k) lo = mid; else hi = mid - 1;
  }
  lrank[k] = lo;
}

__global__ void k_gather_f4(int64_t n, const int* __restrict__ idx, const float4* __restrict__ src, float4* dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}
__global__ void k_gather_f4_quad(int64_t n, int K, const int* __restrict__ idx, const float4* __restrict__ src,
                                 float4* dst) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * K) return;
  const int64_t i = t / K, g = t - i * K;
  dst[t] = src[(int64_t)idx[i] * K + g];
}
__global__ void k_gather_i64(int64_t n, const int* __restrict__ idx, const long long* __restrict__ src,
                             long long* dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

// local panel counts per leaf: the global count for owned and halo leaves, 0 elsewhere
__global__ void k_local_counts(int nl, const int* __restrict__ gbeg, const int* __restrict__ lrank, int me,
                               const unsigned char* __restrict__ need, int* cnt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nl) return;
  const bool present = (lrank ? lrank[k] == me : true) || (need && need[k]);
  cnt[k] = present ? gbeg[k + 1] - gbeg[k] : 0;
}

__global__ void k_widen(int n, const int* __restrict__ in, long long* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

__global__ void k_point_leaf_off(int nl, const int* __restrict__ begin, int leaf_off, int* leaf) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nl) return;
  for (int i = begin[k]; i < begin[k + 1]; ++i) leaf[i] = leaf_off + k;
}

// subtree-count seed: points of leaf k (global CSR `begin`, times mult) if lo <= k < hi, else 0
__global__ void k_own_leaf_counts(int nl, const int* __restrict__ begin, int mult, int leaf_off, int lo, int hi,
                                  int* cnt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nl) cnt[leaf_off + k] = (k >= lo && k < hi) ? (begin[k + 1] - begin[k]) * mult : 0;
}

}  // namespace

namespace {

// run-length encoding of the sorted level-21 keys kp[0:m) at level l: unique cell keys and counts
int64_t rle_level(const uint64_t* kp, int64_t m, int l, DevBuf<uint64_t>& ukey, DevBuf<int>& ucnt, cudaStream_t s) {
  ukey.alloc(std::max<int64_t>(m, 1));
  ucnt.alloc(std::max<int64_t>(m, 1));
  if (m == 0) return 0;
  DevBuf<uint64_t> sh;
  sh.alloc(m);
  k_shift_keys<<<ceil_div(m, 256), 256, 0, s>>>(m, kp, 3 * (MAX_LEVEL - l), sh.get());
  FMM_CHECK_LAUNCH();
  DevBuf<int> nr;
  nr.alloc(1);
  size_t tb = 0;
  cub::DeviceRunLengthEncode::Encode(nullptr, tb, sh.get(), ukey.get(), ucnt.get(), nr.get(), (int)m, s);
  DevBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(tb, 1));
  FMM_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(), tb, sh.get(), ukey.get(), ucnt.get(), nr.get(), (int)m, s));
  int h = 0;
  FMM_CUDA(cudaMemcpyAsync(&h, nr.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  return h;
}

// sorted unique keys with summed counts of an unsorted (key, count) list of n entries
int64_t reduce_by_key(DevBuf<uint64_t>& k, DevBuf<int>& v, int64_t n, DevBuf<uint64_t>& ok, DevBuf<int>& ov,
                      cudaStream_t s) {
  ok.alloc(std::max<int64_t>(n, 1));
  ov.alloc(std::max<int64_t>(n, 1));
  if (n == 0) return 0;
  DevBuf<uint64_t> ks;
  DevBuf<int> vs;
  ks.alloc(n);
  vs.alloc(n);
  sort_pairs(k, v, ks, vs, n, s);
  DevBuf<int> nr;
  nr.alloc(1);
  size_t tb = 0;
  cub::DeviceReduce::ReduceByKey(nullptr, tb, ks.get(), ok.get(), vs.get(), ov.get(), nr.get(), cub::Sum(), (int)n, s);
  DevBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(tb, 1));
  FMM_CUDA(cub::DeviceReduce::ReduceByKey(tmp.get(), tb, ks.get(), ok.get(), vs.get(), ov.get(), nr.get(), cub::Sum(),
                                          (int)n, s));
  int h = 0;
  FMM_CUDA(cudaMemcpyAsync(&h, nr.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  return h;
}

// every rank's (cell key, panel count) list -> the global sorted cells with summed counts (all ranks)
int64_t merge_cells(fmmbem_ctx* c, DevBuf<uint64_t>& ukey, DevBuf<int>& ucnt, int64_t nu, DevBuf<uint64_t>& gkey,
                    DevBuf<int>& gcnt, cudaStream_t s) {
  const int R = c->nranks;
  if (R == 1) {
    gkey = std::move(ukey);
    gcnt = std::move(ucnt);
    return nu;
  }
  DevBuf<int64_t> mine, all;
  mine.alloc(1);
  all.alloc(R);
  const int64_t h = nu;
  FMM_CUDA(cudaMemcpyAsync(mine.get(), &h, sizeof(h), cudaMemcpyHostToDevice, s));
  comm_allgather_i64(c, mine.get(), all.get(), 1, s);
  std::vector<int64_t> nus(R);
  FMM_CUDA(cudaMemcpyAsync(nus.data(), all.get(), R * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  std::vector<size_t> ok(R + 1, 0), oc(R + 1, 0);
  for (int r = 0; r < R; ++r) {
    ok[r + 1] = ok[r] + nus[r] * sizeof(uint64_t);
    oc[r + 1] = oc[r] + nus[r] * sizeof(int);
  }
  const int64_t tot = (int64_t)(ok[R] / sizeof(uint64_t));
  DevBuf<uint64_t> K;
  DevBuf<int> C;
  K.alloc(std::max<int64_t>(tot, 1));
  C.alloc(std::max<int64_t>(tot, 1));
  comm_allgatherv_bytes(c, ukey.get(), K.get(), ok, s);
  comm_allgatherv_bytes(c, ucnt.get(), C.get(), oc, s);
  return reduce_by_key(K, C, tot, gkey, gcnt, s);
}

}  // namespace

void scan_ints(const int* in, int* out, int n, cudaStream_t s) { exclusive_scan(in, out, n, s); }
void scan_i64(const long long* in, long long* out, int n, cudaStream_t s) { exclusive_scan(in, out, n, s); }

void build_halo(fmmbem_ctx* c, const std::vector<int>& hgb, DevBuf<float4>& opos, DevBuf<float4>& onrm,
                DevBuf<float4>& oquad, DevBuf<long long>& ogid, cudaStream_t s);

// The octree of the whole problem, built by every rank from its own input slice (SURVEY 8(a) a2-a3,
// 8(e)):  (1) root cube from the all-reduced bounding box; (2) level-21 Morton keys of the slice's
// panels, locally sorted; (3) the leaf level L of the depth rule from the global number of occupied
// cells, (4) the replicated leaf skeleton -- every occupied leaf (panels of all ranks, charges) with
// its global panel count -- and from it the cells of every level, their links and lists;
// (5) the cost-weighted contiguous leaf partition; (6) the panels move to the rank owning
// their leaf (grouped send/recv of FP64 records) and are sorted into Morton order; (7) the near-field
// halo: the owned panels each peer's P2P needs and the peers' panels this rank's P2P needs (static
// positions exchanged here, weights per matvec).  Memory per rank: the slice, the owned panels and
// the halo (O(N/R)) plus the O(N/leaf_points) skeleton.  With one rank the same steps reduce to the
// single-GPU build (no exchange).
// nranks > 1, after the plan: the rank keeps the lists of its own leaves / windows only (the full
// lists served the plan on the host) and numbers its expansion slots (plan.h slot_layout): cell ->
// slot map and the slots' keys on the device
void local_lists_and_slots(fmmbem_ctx* c, const HostTree& H, cudaStream_t s) {
  Tree& T = c->tree;
  const ExchangePlan& X = c->xplan;
  const int L = T.L, nl = (int)T.n_leaves;
  const int64_t nc = T.n_cells;
  const int lo = c->leaf_lo, hi = c->leaf_hi;
  {  // neighbour lists of the owned leaves
    std::vector<int> off(nl + 1);
    for (int k = 0; k <= nl; ++k) off[k] = H.nbr_off[std::min(std::max(k, lo), hi)] - H.nbr_off[lo];
    const int n = off[nl];
    T.nbr_off.alloc(nl + 1);
    T.nbr_idx.alloc(std::max(n, 1));
    FMM_CUDA(cudaMemcpyAsync(T.nbr_off.get(), off.data(), (nl + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
    if (n) FMM_CUDA(cudaMemcpyAsync(T.nbr_idx.get(), H.nbr_idx.data() + H.nbr_off[lo], n * sizeof(int),
                                    cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  {  // interaction lists of the window cells (levels >= 2), one contiguous segment per level
    std::vector<long long> off(nc + 1, 0);
    long long n = 0;
    for (int l = 0; l <= L; ++l)
      for (int64_t cc = T.lvl_off[l]; cc < T.lvl_off[l + 1]; ++cc) {
        off[cc] = n;
        if (cc >= X.win_lo[l] && cc < X.win_hi[l]) n += H.m2l_off[cc + 1] - H.m2l_off[cc];
      }
    off[nc] = n;
    T.m2l_off.release();
    T.m2l_idx.release();
    T.m2l_off.alloc(nc + 1);
    T.m2l_idx.alloc(std::max<long long>(n, 1));
    FMM_CUDA(cudaMemcpyAsync(T.m2l_off.get(), off.data(), (nc + 1) * sizeof(long long), cudaMemcpyHostToDevice, s));
    for (int l = 2; l <= L; ++l) {
      const int64_t a = H.m2l_off[X.win_lo[l]], b = H.m2l_off[X.win_hi[l]];
      if (b > a)
        FMM_CUDA(cudaMemcpyAsync(T.m2l_idx.get() + off[X.win_lo[l]], H.m2l_idx.data() + a, (b - a) * sizeof(int),
                                 cudaMemcpyHostToDevice, s));
    }
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  // slots
  c->win_lo = X.win_lo;
  c->win_hi = X.win_hi;
  c->slot_base = X.slot_base;
  c->n_slots = X.n_slots;
  std::vector<int> cmap(nc, -1);
  std::vector<uint64_t> skey(std::max<int64_t>(X.n_slots, 1), 0);
  for (int l = 0; l <= L; ++l)
    for (int64_t cc = X.win_lo[l]; cc < X.win_hi[l]; ++cc) cmap[cc] = (int)(X.slot_base[l] + cc - X.win_lo[l]);
  const int64_t nw = X.n_slots - (int64_t)X.extra.size();
  for (size_t i = 0; i < X.extra.size(); ++i) cmap[X.extra[i]] = (int)(nw + (int64_t)i);
  for (int64_t cc = 0; cc < nc; ++cc)
    if (cmap[cc] >= 0) skey[cmap[cc]] = H.key[cc];
  c->cmap.alloc(nc);
  c->skey.alloc(skey.size());
  FMM_CUDA(cudaMemcpyAsync(c->cmap.get(), cmap.data(), nc * sizeof(int), cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaMemcpyAsync(c->skey.get(), skey.data(), skey.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaStreamSynchronize(s));
}

void build_tree(fmmbem_ctx* c, const PanelInput& in, const double* wq, const double* cxyz, const double* cq,
                cudaStream_t s) {
  Tree& T = c->tree;
  const int R = c->nranks, me = c->rank, K = c->K;
  const int64_t m = in.n, nc = c->nc;
  const int TB = 256;
  // FMMBEM_VERBOSE=1: host-clock time of each setup stage on stderr (synchronising the stream)
  static const bool verbose = std::getenv("FMMBEM_VERBOSE") != nullptr;
  auto t_stage = std::chrono::steady_clock::now();
  auto stage = [&](const char* name) {
    if (!verbose) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[fmmbem rank %d] %-12s %8.1f ms\n", me, name,
                 std::chrono::duration<double, std::milli>(now - t_stage).count());
    t_stage = now;
  };
  // 1. root cube: bounding cube of all ranks' centroids and the (replicated) charges
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  bbox(in.cen, m, mn, mx, s);
  bbox(cxyz, nc, mn, mx, s);
  if (R > 1) {
    double h[6] = {mn[0], mn[1], mn[2], -mx[0], -mx[1], -mx[2]};
    DevBuf<double> d;
    d.alloc(6);
    FMM_CUDA(cudaMemcpyAsync(d.get(), h, sizeof(h), cudaMemcpyHostToDevice, s));
    comm_allreduce_f64_op(c, d.get(), 6, -1, s);
    FMM_CUDA(cudaMemcpyAsync(h, d.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < 3; ++k) {
      mn[k] = h[k];
      mx[k] = -h[3 + k];
    }
  }
  double ext = std::max(mx[0] - mn[0], std::max(mx[1] - mn[1], mx[2] - mn[2]));
  if (!(ext > 0)) ext = 1.0;
  double Wr = ext * (1.0 + 1e-6) + 1e-300;
  int e;
  double mm = std::frexp(Wr, &e);
  mm = std::ceil(mm * 256.0) / 256.0;
  T.W = std::ldexp(mm, e);
  for (int d = 0; d < 3; ++d) T.x0[d] = 0.5 * (mn[d] + mx[d]) - 0.5 * T.W;
  const double inv_h21 = (double)(1 << MAX_LEVEL) / T.W;

  stage("bbox");
  // 2. Morton keys at depth 21 + stable radix sort (ties keep the input order)
  DevBuf<uint64_t> kp;
  DevBuf<int> pperm;
  {
    DevBuf<uint64_t> kp_in;
    DevBuf<int> ip_in;
    kp_in.alloc(std::max<int64_t>(m, 1)); kp.alloc(std::max<int64_t>(m, 1));
    ip_in.alloc(std::max<int64_t>(m, 1)); pperm.alloc(std::max<int64_t>(m, 1));
    if (m) {
      k_keys21<<<ceil_div(m, TB), TB, 0, s>>>(m, in.cen, T.x0[0], T.x0[1], T.x0[2], inv_h21, kp_in.get(), ip_in.get());
      FMM_CHECK_LAUNCH();
      sort_pairs(kp_in, ip_in, kp, pperm, m, s);
    }
  }
  DevBuf<uint64_t> kc;
  DevBuf<int> cperm;
  if (nc) {
    DevBuf<uint64_t> kc_in;
    DevBuf<int> ic_in;
    kc_in.alloc(nc); kc.alloc(nc); ic_in.alloc(nc); cperm.alloc(nc);
    k_keys21<<<ceil_div(nc, TB), TB, 0, s>>>(nc, cxyz, T.x0[0], T.x0[1], T.x0[2], inv_h21, kc_in.get(), ic_in.get());
    FMM_CHECK_LAUNCH();
    sort_pairs(kc_in, ic_in, kc, cperm, nc, s);
  }

  stage("keys+sort");
  // 3. leaf level: the smallest L with (global panels) / (occupied cells at L) <= leaf_points
  int64_t np = m;
  if (R > 1) {
    DevBuf<double> d;
    d.alloc(1);
    double h = (double)m;
    FMM_CUDA(cudaMemcpyAsync(d.get(), &h, sizeof(h), cudaMemcpyHostToDevice, s));
    comm_allreduce_f64_op(c, d.get(), 1, 0, s);
    FMM_CUDA(cudaMemcpyAsync(&h, d.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    np = (int64_t)h;
  }
  c->np = np;
  if (np * (int64_t)K >= (1LL << 31)) throw Error(FMMBEM_E_INVALID, "problem too large for 32-bit point indices");
  int L = MAX_LEVEL;
  DevBuf<uint64_t> gkey;  // global occupied leaf cells (panels) and their panel counts
  DevBuf<int> gcnt;
  int64_t ngl = 0;
  if (R == 1) {  // one rank: occupied cells per level from the key differences of the sorted keys
    DevBuf<unsigned long long> hist;
    hist.alloc(MAX_LEVEL + 1);
    hist.zero(s);
    if (m > 1) k_level_hist<<<std::min(1024, ceil_div(m, TB)) + 1, TB, 0, s>>>(m, kp.get(), hist.get());
    FMM_CHECK_LAUNCH();
    unsigned long long hh[MAX_LEVEL + 1];
    FMM_CUDA(cudaMemcpyAsync(hh, hist.get(), sizeof(hh), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    unsigned long long cells = 1;
    for (int l = 0; l <= MAX_LEVEL; ++l) {
      cells += hh[l];
      if ((double)np / (double)cells <= (double)c->opt.leaf_points) { L = l; break; }
    }
    DevBuf<uint64_t> uk;
    DevBuf<int> uc;
    ngl = rle_level(kp.get(), m, L, uk, uc, s);
    ngl = merge_cells(c, uk, uc, ngl, gkey, gcnt, s);
  } else {  // several ranks: merge the ranks' occupied cells level by level, from the first candidate
    int l0 = 0;
    while (l0 < MAX_LEVEL && std::pow(8.0, l0) * c->opt.leaf_points < (double)np) ++l0;
    for (int l = l0; l <= MAX_LEVEL; ++l) {
      DevBuf<uint64_t> uk;
      DevBuf<int> uc;
      const int64_t nu = rle_level(kp.get(), m, l, uk, uc, s);
      ngl = merge_cells(c, uk, uc, nu, gkey, gcnt, s);
      if ((double)np / (double)std::max<int64_t>(ngl, 1) <= (double)c->opt.leaf_points || l == MAX_LEVEL) {
        L = l;
        break;
      }
    }
  }
  T.L = L;
  const int shift = 3 * (MAX_LEVEL - L);

  stage("leaf level");
  // 4. leaf skeleton = panel cells U charge cells (charges replicated), panel count per leaf
  std::vector<DevBuf<uint64_t>> lvl(L + 1);
  std::vector<int64_t> nlev(L + 1);
  DevBuf<int> lcnt_all;  // panel count per leaf
  {
    const int64_t tot = ngl + nc;
    DevBuf<uint64_t> k;
    DevBuf<int> v;
    k.alloc(std::max<int64_t>(tot, 1));
    v.alloc(std::max<int64_t>(tot, 1));
    if (ngl) {
      FMM_CUDA(cudaMemcpyAsync(k.get(), gkey.get(), ngl * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
      FMM_CUDA(cudaMemcpyAsync(v.get(), gcnt.get(), ngl * sizeof(int), cudaMemcpyDeviceToDevice, s));
    }
    if (nc) {
      k_shift_keys<<<ceil_div(nc, TB), TB, 0, s>>>(nc, kc.get(), shift, k.get() + ngl);
      FMM_CUDA(cudaMemsetAsync(v.get() + ngl, 0, nc * sizeof(int), s));
      FMM_CHECK_LAUNCH();
    }
    nlev[L] = reduce_by_key(k, v, tot, lvl[L], lcnt_all, s);
  }
  gkey.release();
  gcnt.release();
  for (int l = L - 1; l >= 0; --l) {
    DevBuf<uint64_t> tmp;
    tmp.alloc(std::max<int64_t>(nlev[l + 1], 1));
    k_shift_keys<<<ceil_div(nlev[l + 1], TB), TB, 0, s>>>(nlev[l + 1], lvl[l + 1].get(), 3, tmp.get());
    FMM_CHECK_LAUNCH();
    lvl[l].alloc(std::max<int64_t>(nlev[l + 1], 1));
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
  // parent / child links
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
  FMM_CUDA(cudaMemsetAsync(T.child_begin.get() + T.lvl_off[L], 0, nl * sizeof(int), s));  // leaves: no children
  FMM_CUDA(cudaMemsetAsync(T.child_end.get() + T.lvl_off[L], 0, nl * sizeof(int), s));
  FMM_CHECK_LAUNCH();
  T.leaf_ijk.alloc(nl);
  k_leaf_ijk<<<ceil_div(nl, TB), TB, 0, s>>>(nl, lvl[L].get(), T.leaf_ijk.get());
  FMM_CHECK_LAUNCH();
  stage("skeleton");
  // global panel CSR over the leaves
  c->gbeg.alloc(nl + 1);
  {
    DevBuf<int> cnt;
    cnt.alloc(nl + 1);
    FMM_CUDA(cudaMemsetAsync(cnt.get() + nl, 0, sizeof(int), s));
    FMM_CUDA(cudaMemcpyAsync(cnt.get(), lcnt_all.get(), nl * sizeof(int), cudaMemcpyDeviceToDevice, s));
    exclusive_scan(cnt.get(), c->gbeg.get(), nl + 1, s);
  }
  lcnt_all.release();
  // neighbour lists (leaf level) and interaction lists (levels 2..L)
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
  {
    // interaction-list offsets are 64-bit: ~100 entries per cell exceed 2^31 beyond ~2e7 cells (22^3 array)
    int nC = (int)T.n_cells;
    DevBuf<int> cnt;
    cnt.alloc(nC + 1);
    cnt.zero(s);
    for (int l = 2; l <= L; ++l)
      k_m2l_list<<<ceil_div(nlev[l], TB), TB, 0, s>>>((int)nlev[l], lvl[l].get(), (int)T.lvl_off[l], (int)nlev[l - 1],
                                                      lvl[l - 1].get(), (int)T.lvl_off[l - 1], T.child_begin.get(),
                                                      T.child_end.get(), T.key.get(), l, nullptr, cnt.get(), 0);
    FMM_CHECK_LAUNCH();
    DevBuf<long long> cnt64;
    cnt64.alloc(nC + 1);
    k_widen<<<ceil_div(nC + 1, TB), TB, 0, s>>>(nC + 1, cnt.get(), cnt64.get());
    FMM_CHECK_LAUNCH();
    T.m2l_off.alloc(nC + 1);
    exclusive_scan(cnt64.get(), T.m2l_off.get(), nC + 1, s);
    long long tot = 0;
    FMM_CUDA(cudaMemcpyAsync(&tot, T.m2l_off.get() + nC, sizeof(long long), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    T.m2l_pairs = tot;
    T.m2l_idx.alloc(std::max<long long>(tot, 1));
    for (int l = 2; l <= L; ++l)
      k_m2l_list<<<ceil_div(nlev[l], TB), TB, 0, s>>>((int)nlev[l], lvl[l].get(), (int)T.lvl_off[l], (int)nlev[l - 1],
                                                      lvl[l - 1].get(), (int)T.lvl_off[l - 1], T.child_begin.get(),
                                                      T.child_end.get(), T.key.get(), l, T.m2l_off.get(),
                                                      T.m2l_idx.get(), 1);
    FMM_CHECK_LAUNCH();
  }

  stage("lists");
  // charges (replicated): their leaf CSR (the targets of the reaction potential count in the LET)
  auto& C = c->chg;
  C.n = nc;
  C.begin.alloc(nl + 1);
  if (nc) k_set_begin<<<ceil_div(nl + 1, TB), TB, 0, s>>>(nl, lvl[L].get(), (int)nc, kc.get(), shift, C.begin.get());
  else C.begin.zero(s);
  FMM_CHECK_LAUNCH();

  // 5. contiguous cost-weighted leaf partition, halo and LET plan (every rank derives the same one)
  if (R > 1) {
    HostTree H;
    H.L = L;
    H.lvl_off = T.lvl_off;
    H.key.resize(T.n_cells);
    H.nbr_off.resize(nl + 1);
    H.nbr_idx.resize(T.nbr_pairs);
    H.m2l_off.resize(T.n_cells + 1);
    std::vector<int> gb(nl + 1), cb(nl + 1);
    FMM_CUDA(cudaMemcpyAsync(H.key.data(), T.key.get(), T.n_cells * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaMemcpyAsync(H.nbr_off.data(), T.nbr_off.get(), (nl + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaMemcpyAsync(H.nbr_idx.data(), T.nbr_idx.get(), T.nbr_pairs * sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaMemcpyAsync(H.m2l_off.data(), T.m2l_off.get(), (T.n_cells + 1) * sizeof(long long), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaMemcpyAsync(gb.data(), c->gbeg.get(), (nl + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaMemcpyAsync(cb.data(), C.begin.get(), (nl + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    std::vector<int> pan(nl), tgt(nl);
    for (int k = 0; k < nl; ++k) {
      pan[k] = gb[k + 1] - gb[k];
      tgt[k] = pan[k] + cb[k + 1] - cb[k];
    }
    // the partition needs only the list lengths; the rest of the plan reads the lists of this
    // rank's window cells, so only those come to the host (~1/R of 10 GB at 1e9 panels)
    plan_partition(H, pan, K, R, c->xplan);
    plan_windows(H, me, c->xplan);
    {
      const ExchangePlan& X = c->xplan;
      HostVec<int64_t> full = std::move(H.m2l_off);
      H.m2l_off.resize(T.n_cells + 1);
      int64_t pos = 0;
      std::vector<int64_t> seg_dst(L + 1, 0);
      for (int l = 0; l <= L; ++l) {
        const int64_t wlo = X.win_lo[l], whi = X.win_hi[l], base = full[wlo];
        seg_dst[l] = pos;
        for (int64_t cc = T.lvl_off[l]; cc < T.lvl_off[l + 1]; ++cc)
          H.m2l_off[cc] = pos + (cc < wlo ? 0 : (cc < whi ? full[cc] - base : full[whi] - base));
        pos += full[whi] - base;
      }
      H.m2l_off[T.n_cells] = pos;
      H.m2l_idx.resize(std::max<int64_t>(pos, 1));
      for (int l = 0; l <= L; ++l) {
        const int64_t a = full[X.win_lo[l]], b = full[X.win_hi[l]];
        if (b > a)
          FMM_CUDA(cudaMemcpyAsync(H.m2l_idx.data() + seg_dst[l], T.m2l_idx.get() + a, (b - a) * sizeof(int),
                                   cudaMemcpyDeviceToHost, s));
      }
      FMM_CUDA(cudaStreamSynchronize(s));
    }
    plan_lists(H, pan, tgt, R, me, c->xplan);
    c->leaf_bounds = c->xplan.leaf_bounds;
    c->leaf_lo = (int)c->leaf_bounds[me];
    c->leaf_hi = (int)c->leaf_bounds[me + 1];
    long long own = 0, n_own_p = 0;  // exact P2P interactions of the owned targets (j != i excluded)
    for (int k = c->leaf_lo; k < c->leaf_hi; ++k) {
      long long sn = 0;
      for (int e = H.nbr_off[k]; e < H.nbr_off[k + 1]; ++e) sn += pan[H.nbr_idx[e]];
      own += (long long)pan[k] * sn * K;
      n_own_p += pan[k];
    }
    c->p2p_inter_kp = own - n_own_p * K;
    local_lists_and_slots(c, H, s);
  } else {
    c->leaf_bounds = {0, nl};
    c->leaf_lo = 0;
    c->leaf_hi = nl;
    c->win_lo.assign(L + 1, 0);
    c->win_hi.assign(L + 1, 0);
    c->slot_base.assign(L + 1, 0);
    for (int l = 0; l <= L; ++l) {
      c->win_lo[l] = c->slot_base[l] = T.lvl_off[l];
      c->win_hi[l] = T.lvl_off[l + 1];
    }
    c->n_slots = T.n_cells;
  }
  const int leaf_lo = c->leaf_lo, leaf_hi = c->leaf_hi;
  std::vector<int> hgb(nl + 1);
  FMM_CUDA(cudaMemcpyAsync(hgb.data(), c->gbeg.get(), (nl + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  const int64_t n_own = hgb[leaf_hi] - hgb[leaf_lo];

  stage("plan");
  // 6. panels to their owners: FP64 records in the slice's key order, one contiguous segment per rank
  const int Wd = 9 + (K > 1 ? 3 * K : 0);
  DevBuf<unsigned long long> orec;  // owned records, Morton order
  {
    DevBuf<unsigned long long> rec;
    rec.alloc(std::max<int64_t>(m, 1) * Wd);
    if (m)
      k_pack_records<<<ceil_div(m, TB), TB, 0, s>>>(m, pperm.get(), kp.get(), in.cen, in.nrm, in.area,
                                                    K > 1 ? in.qp : nullptr, K, in.gid0, Wd, rec.get());
    FMM_CHECK_LAUNCH();
    std::vector<int64_t> split(R + 1, 0);
    split[R] = m;
    if (R > 1) {
      std::vector<uint64_t> hb(R - 1);
      for (int r = 1; r < R; ++r) {
        const int lb = (int)c->leaf_bounds[r];
        if (lb < nl) FMM_CUDA(cudaMemcpyAsync(&hb[r - 1], lvl[L].get() + lb, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        else hb[r - 1] = ~0ULL >> 1;
      }
      FMM_CUDA(cudaStreamSynchronize(s));
      DevBuf<uint64_t> db;
      DevBuf<long long> dp;
      db.alloc(R - 1);
      dp.alloc(R - 1);
      FMM_CUDA(cudaMemcpyAsync(db.get(), hb.data(), (R - 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
      k_split_points<<<1, 64, 0, s>>>(m, kp.get(), shift, db.get(), R - 1, dp.get());
      FMM_CHECK_LAUNCH();
      std::vector<long long> hp(R - 1);
      FMM_CUDA(cudaMemcpyAsync(hp.data(), dp.get(), (R - 1) * sizeof(long long), cudaMemcpyDeviceToHost, s));
      FMM_CUDA(cudaStreamSynchronize(s));
      for (int r = 1; r < R; ++r) split[r] = std::max<int64_t>(split[r - 1], hp[r - 1]);
    }
    kp.release();
    pperm.release();
    DevBuf<unsigned long long> recv;
    const unsigned long long* got = rec.get();
    if (R > 1) {
      DevBuf<int64_t> mine, all;
      mine.alloc(R);
      all.alloc((size_t)R * R);
      std::vector<int64_t> sc(R), M((size_t)R * R);
      for (int p = 0; p < R; ++p) sc[p] = split[p + 1] - split[p];
      FMM_CUDA(cudaMemcpyAsync(mine.get(), sc.data(), R * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      comm_allgather_i64(c, mine.get(), all.get(), R, s);
      FMM_CUDA(cudaMemcpyAsync(M.data(), all.get(), (size_t)R * R * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      FMM_CUDA(cudaStreamSynchronize(s));
      int64_t rtot = 0;
      std::vector<int64_t> roff(R + 1, 0);
      for (int p = 0; p < R; ++p) roff[p + 1] = roff[p] + M[(size_t)p * R + me];
      rtot = roff[R];
      if (rtot != n_own) throw Error(FMMBEM_E_CUDA, "panel migration: received count differs from the partition");
      recv.alloc(std::max<int64_t>(rtot, 1) * Wd);
      const size_t rb = Wd * sizeof(unsigned long long);
      std::vector<const void*> sp(R);
      std::vector<void*> rp(R);
      std::vector<size_t> sb(R), rbs(R);
      for (int p = 0; p < R; ++p) {
        sp[p] = rec.get() + split[p] * Wd;
        sb[p] = (size_t)sc[p] * rb;
        rp[p] = recv.get() + roff[p] * Wd;
        rbs[p] = (size_t)(roff[p + 1] - roff[p]) * rb;
      }
      comm_alltoallv_bytes(c, sp, sb, rp, rbs, s);
      FMM_CUDA(cudaStreamSynchronize(s));
      rec.release();
      got = recv.get();
    } else if (m != n_own) {
      throw Error(FMMBEM_E_CUDA, "single-rank partition does not cover the panels");
    }
    // merge the sources' sorted segments: stable sort by key (ties: source rank, then slice order)
    orec.alloc(std::max<int64_t>(n_own, 1) * Wd);
    if (n_own) {
      DevBuf<uint64_t> k_in, k_out;
      DevBuf<int> i_in, i_out;
      k_in.alloc(n_own); k_out.alloc(n_own); i_in.alloc(n_own); i_out.alloc(n_own);
      k_rec_keys<<<ceil_div(n_own, TB), TB, 0, s>>>(n_own, got, Wd, k_in.get(), i_in.get());
      FMM_CHECK_LAUNCH();
      sort_pairs(k_in, i_in, k_out, i_out, n_own, s);
      k_gather_rec<<<ceil_div(n_own * Wd, TB), TB, 0, s>>>(n_own, i_out.get(), got, Wd, orec.get());
      FMM_CHECK_LAUNCH();
    }
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  stage("migration");
  // duplicate centroids (always in one leaf, hence on one rank; the verdict is made collective)
  {
    DevBuf<long long> f;
    f.alloc(1);
    const long long big = 0x7fffffffffffffffLL;
    FMM_CUDA(cudaMemcpyAsync(f.get(), &big, sizeof(big), cudaMemcpyHostToDevice, s));
    if (n_own) k_dup_check_rec<<<ceil_div(n_own, TB), TB, 0, s>>>((int)n_own, orec.get(), Wd, f.get());
    FMM_CHECK_LAUNCH();
    long long hf = big;
    FMM_CUDA(cudaMemcpyAsync(&hf, f.get(), sizeof(hf), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    double fd = (hf == big) ? 1e300 : (double)hf;
    if (R > 1) {
      DevBuf<double> d;
      d.alloc(1);
      FMM_CUDA(cudaMemcpyAsync(d.get(), &fd, sizeof(fd), cudaMemcpyHostToDevice, s));
      comm_allreduce_f64_op(c, d.get(), 1, -1, s);
      FMM_CUDA(cudaMemcpyAsync(&fd, d.get(), sizeof(fd), cudaMemcpyDeviceToHost, s));
      FMM_CUDA(cudaStreamSynchronize(s));
    }
    if (fd < 1e300) throw Error(FMMBEM_E_COINCIDENT, "duplicate panel centroid at triangle " + std::to_string((long long)fd));
  }

  stage("dup check");
  // 7. owned point data (leaf-local FP32), then the near-field halo
  const double h = T.width(L);
  DevBuf<float4> opos, onrm, oquad;
  DevBuf<long long> ogid;
  DevBuf<int> oleaf;
  opos.alloc(std::max<int64_t>(n_own, 1));
  onrm.alloc(std::max<int64_t>(n_own, 1));
  ogid.alloc(std::max<int64_t>(n_own, 1));
  oleaf.alloc(std::max<int64_t>(n_own, 1));
  if (K > 1) oquad.alloc(std::max<int64_t>(n_own, 1) * K);
  {
    const int nol = leaf_hi - leaf_lo;
    DevBuf<int> ob;
    ob.alloc(nol + 1);
    std::vector<int> hob(nol + 1);
    for (int k = 0; k <= nol; ++k) hob[k] = hgb[leaf_lo + k] - hgb[leaf_lo];
    FMM_CUDA(cudaMemcpyAsync(ob.get(), hob.data(), (nol + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
    if (nol > 0) k_point_leaf_off<<<ceil_div(nol, TB), TB, 0, s>>>(nol, ob.get(), leaf_lo, oleaf.get());
    if (n_own) {
      k_place_owned<<<ceil_div(n_own, TB), TB, 0, s>>>((int)n_own, orec.get(), Wd, oleaf.get(), T.leaf_ijk.get(),
                                                       T.x0[0], T.x0[1], T.x0[2], h, opos.get(), onrm.get(), ogid.get());
      if (K > 1)
        k_place_owned_quad<<<ceil_div(n_own * K, TB), TB, 0, s>>>((int)n_own, K, orec.get(), Wd, oleaf.get(),
                                                                  T.leaf_ijk.get(), wq, T.x0[0], T.x0[1], T.x0[2], h,
                                                                  oquad.get());
    }
    FMM_CHECK_LAUNCH();
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  orec.release();
  auto& P = c->pan;
  P.div = 1;
  if (R == 1) {
    c->pan_lo = 0;
    c->pan_hi = n_own;
    P.n = n_own;
    P.pos = std::move(opos);
    P.nrm = std::move(onrm);
    P.leaf = std::move(oleaf);
    P.begin.alloc(nl + 1);
    FMM_CUDA(cudaMemcpyAsync(P.begin.get(), c->gbeg.get(), (nl + 1) * sizeof(int), cudaMemcpyDeviceToDevice, s));
    c->pan_ids.resize(n_own);
    if (n_own)
      FMM_CUDA(cudaMemcpyAsync(c->pan_ids.data(), ogid.get(), n_own * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    if (K > 1) {
      c->quad.pos = std::move(oquad);
    }
    FMM_CUDA(cudaStreamSynchronize(s));
  } else {
    build_halo(c, hgb, opos, onrm, oquad, ogid, s);
  }
  if (K > 1) {
    auto& Q = c->quad;
    Q.n = P.n * K;
    Q.div = K;
    Q.leaf.alloc(std::max<int64_t>(Q.n, 1));
    Q.begin.alloc(nl + 1);
    std::vector<int> b(nl + 1);
    FMM_CUDA(cudaMemcpyAsync(b.data(), P.begin.get(), (nl + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    for (auto& v : b) v *= K;
    FMM_CUDA(cudaMemcpyAsync(Q.begin.get(), b.data(), (nl + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
    if (Q.n) k_point_leaf<<<ceil_div(nl, TB), TB, 0, s>>>(nl, Q.begin.get(), Q.leaf.get());
    FMM_CHECK_LAUNCH();
    FMM_CUDA(cudaStreamSynchronize(s));
  }

  stage("points+halo");
  // 8. charges (replicated): tree order, leaf-local coordinates
  if (nc) {
    C.pos.alloc(nc);
    C.leaf.alloc(nc);
    k_point_leaf<<<ceil_div(nl, TB), TB, 0, s>>>(nl, C.begin.get(), C.leaf.get());
    k_place_charges<<<ceil_div(nc, TB), TB, 0, s>>>((int)nc, cperm.get(), C.leaf.get(), T.leaf_ijk.get(), cxyz, cq,
                                                    T.x0[0], T.x0[1], T.x0[2], h, C.pos.get());
    FMM_CHECK_LAUNCH();
    c->chg_ids.alloc(nc);
    FMM_CUDA(cudaMemcpyAsync(c->chg_ids.get(), cperm.get(), nc * sizeof(int), cudaMemcpyDeviceToDevice, s));
  }

  stage("charges");
  // 9. subtree counts: panels of ALL ranks (sources: a cell with any panel has a multipole), charges
  {
    auto up = [&](DevBuf<int>& cnt, const int* beg, int mult, int lo, int hi) {
      cnt.alloc(T.n_cells);
      k_own_leaf_counts<<<ceil_div(nl, TB), TB, 0, s>>>(nl, beg, mult, (int)T.lvl_off[L], lo, hi, cnt.get());
      for (int l = L - 1; l >= 0; --l)
        k_up_counts<<<ceil_div(nlev[l], TB), TB, 0, s>>>((int)nlev[l], (int)T.lvl_off[l], T.child_begin.get(),
                                                         T.child_end.get(), cnt.get());
      FMM_CHECK_LAUNCH();
    };
    up(c->pan.cell_cnt, c->gbeg.get(), 1, 0, nl);
    if (K > 1) up(c->quad.cell_cnt, c->gbeg.get(), K, 0, nl);
    up(c->chg.cell_cnt, c->chg.begin.get(), 1, 0, nl);
    if (R > 1) {  // owned points only (targets of this rank; P2M of the owned leaves)
      up(c->pan_own_cnt, c->gbeg.get(), 1, leaf_lo, leaf_hi);
      if (K > 1) up(c->quad_own_cnt, c->gbeg.get(), K, leaf_lo, leaf_hi);
      up(c->chg_own_cnt, c->chg.begin.get(), 1, leaf_lo, leaf_hi);
    }
  }
  FMM_CUDA(cudaStreamSynchronize(s));
  stage("counts");
}

// Near-field halo (SURVEY 8(e) per-apply step 1): which owned leaves each peer's P2P needs and which
// peer leaves this rank's P2P needs, from the replicated skeleton (no handshake: both sides derive
// the same leaf lists in increasing order), then the static exchange of the halo positions.
void build_halo(fmmbem_ctx* c, const std::vector<int>& hgb, DevBuf<float4>& opos, DevBuf<float4>& onrm,
                DevBuf<float4>& oquad, DevBuf<long long>& ogid, cudaStream_t s) {
  const Tree& T = c->tree;
  const int R = c->nranks, me = c->rank, K = c->K, nl = (int)T.n_leaves, TB = 256;
  const int leaf_lo = c->leaf_lo, leaf_hi = c->leaf_hi;
  const int64_t n_own = hgb[leaf_hi] - hgb[leaf_lo];
  const ExchangePlan& X = c->xplan;
  auto& H = c->halo;
  H.scnt.assign(R, 0);
  H.soff.assign(R + 1, 0);
  H.rcnt.assign(R, 0);
  H.roff.assign(R + 1, 0);
  std::vector<int> sidx;
  std::vector<unsigned char> hn(nl, 0);
  for (int p = 0; p < R; ++p) {
    H.soff[p] = (int64_t)sidx.size();
    for (int k : X.halo_send[p])
      for (int j = hgb[k]; j < hgb[k + 1]; ++j) sidx.push_back(j - hgb[leaf_lo]);
    H.scnt[p] = (int64_t)sidx.size() - H.soff[p];
    for (int k : X.halo_recv[p]) {
      H.rcnt[p] += hgb[k + 1] - hgb[k];
      hn[k] = 1;
    }
  }
  H.soff[R] = (int64_t)sidx.size();
  DevBuf<int> bounds, lrank;
  bounds.alloc(R + 1);
  std::vector<int> hb(c->leaf_bounds.begin(), c->leaf_bounds.end());
  FMM_CUDA(cudaMemcpyAsync(bounds.get(), hb.data(), (R + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
  lrank.alloc(nl);
  k_leaf_rank<<<ceil_div(nl, TB), TB, 0, s>>>(nl, bounds.get(), R, lrank.get());
  DevBuf<unsigned char> need;
  need.alloc(nl);
  FMM_CUDA(cudaMemcpyAsync(need.get(), hn.data(), nl, cudaMemcpyHostToDevice, s));
  FMM_CHECK_LAUNCH();
  // local layout [halo of ranks < me | owned | halo of ranks > me]
  int64_t o = 0;
  for (int p = 0; p < me; ++p) {
    H.roff[p] = o;
    o += H.rcnt[p];
  }
  c->pan_lo = o;
  c->pan_hi = o + n_own;
  o = c->pan_hi;
  for (int p = me + 1; p < R; ++p) {
    H.roff[p] = o;
    o += H.rcnt[p];
  }
  H.roff[me] = c->pan_lo;
  const int64_t nloc = o;
  H.sent = H.soff[R];
  H.recv = nloc - n_own;
  H.sidx.alloc(std::max<int64_t>(H.sent, 1));
  if (H.sent) FMM_CUDA(cudaMemcpyAsync(H.sidx.get(), sidx.data(), H.sent * sizeof(int), cudaMemcpyHostToDevice, s));
  H.sbuf.alloc(std::max<int64_t>(H.sent, 1));
  // local CSR over all leaves (owned + halo leaves)
  auto& P = c->pan;
  P.n = nloc;
  P.begin.alloc(nl + 1);
  {
    DevBuf<int> cnt;
    cnt.alloc(nl + 1);
    FMM_CUDA(cudaMemsetAsync(cnt.get() + nl, 0, sizeof(int), s));
    k_local_counts<<<ceil_div(nl, TB), TB, 0, s>>>(nl, c->gbeg.get(), lrank.get(), me, need.get(), cnt.get());
    FMM_CHECK_LAUNCH();
    exclusive_scan(cnt.get(), P.begin.get(), nl + 1, s);
    int chk[2] = {0, 0};
    FMM_CUDA(cudaMemcpyAsync(&chk[0], P.begin.get() + leaf_lo, sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaMemcpyAsync(&chk[1], P.begin.get() + nl, sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    if (chk[0] != c->pan_lo || chk[1] != nloc) throw Error(FMMBEM_E_CUDA, "halo layout mismatch");
  }
  // static exchange: positions (+ quadrature points) and global ids of the halo panels
  P.pos.alloc(std::max<int64_t>(nloc, 1));
  P.nrm.alloc(std::max<int64_t>(nloc, 1));  // halo normals: the double layer's dipole sources
  if (n_own) {
    FMM_CUDA(cudaMemcpyAsync(P.pos.get() + c->pan_lo, opos.get(), n_own * sizeof(float4), cudaMemcpyDeviceToDevice, s));
    FMM_CUDA(cudaMemcpyAsync(P.nrm.get() + c->pan_lo, onrm.get(), n_own * sizeof(float4), cudaMemcpyDeviceToDevice, s));
  }
  DevBuf<long long> lgid;
  lgid.alloc(std::max<int64_t>(nloc, 1));
  if (n_own)
    FMM_CUDA(cudaMemcpyAsync(lgid.get() + c->pan_lo, ogid.get(), n_own * sizeof(long long), cudaMemcpyDeviceToDevice, s));
  DevBuf<float4> lquad;
  if (K > 1) {
    lquad.alloc(std::max<int64_t>(nloc, 1) * K);
    if (n_own)
      FMM_CUDA(cudaMemcpyAsync(lquad.get() + c->pan_lo * K, oquad.get(), n_own * K * sizeof(float4),
                               cudaMemcpyDeviceToDevice, s));
  }
  {
    const int64_t ns = std::max<int64_t>(H.sent, 1);
    DevBuf<float4> spos, snrm, squad;
    DevBuf<long long> sgid;
    spos.alloc(ns);
    snrm.alloc(ns);
    sgid.alloc(ns);
    if (K > 1) squad.alloc(ns * K);
    if (H.sent) {
      k_gather_f4<<<ceil_div(H.sent, TB), TB, 0, s>>>(H.sent, H.sidx.get(), opos.get(), spos.get());
      k_gather_f4<<<ceil_div(H.sent, TB), TB, 0, s>>>(H.sent, H.sidx.get(), onrm.get(), snrm.get());
      k_gather_i64<<<ceil_div(H.sent, TB), TB, 0, s>>>(H.sent, H.sidx.get(), ogid.get(), sgid.get());
      if (K > 1) k_gather_f4_quad<<<ceil_div(H.sent * K, TB), TB, 0, s>>>(H.sent, K, H.sidx.get(), oquad.get(), squad.get());
      FMM_CHECK_LAUNCH();
    }
    auto xchg = [&](const void* sb, void* rb, size_t w) {
      std::vector<const void*> sp(R);
      std::vector<void*> rp(R);
      std::vector<size_t> sn(R, 0), rn(R, 0);
      for (int p = 0; p < R; ++p) {
        sp[p] = static_cast<const char*>(sb) + H.soff[p] * w;
        rp[p] = static_cast<char*>(rb) + H.roff[p] * w;
        if (p != me) {
          sn[p] = H.scnt[p] * w;
          rn[p] = H.rcnt[p] * w;
        }
      }
      comm_alltoallv_bytes(c, sp, sn, rp, rn, s);
    };
    xchg(spos.get(), P.pos.get(), sizeof(float4));
    xchg(snrm.get(), P.nrm.get(), sizeof(float4));
    xchg(sgid.get(), lgid.get(), sizeof(long long));
    if (K > 1) xchg(squad.get(), lquad.get(), K * sizeof(float4));
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  P.leaf.alloc(std::max<int64_t>(nloc, 1));
  k_point_leaf<<<ceil_div(nl, TB), TB, 0, s>>>(nl, P.begin.get(), P.leaf.get());
  FMM_CHECK_LAUNCH();
  c->pan_ids.resize(nloc);
  if (nloc) FMM_CUDA(cudaMemcpyAsync(c->pan_ids.data(), lgid.get(), nloc * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  if (K > 1) c->quad.pos = std::move(lquad);
  c->xext.alloc(std::max<int64_t>(nloc, 1));
  FMM_CUDA(cudaStreamSynchronize(s));
}

// Per-matvec near-field halo (SURVEY 8(e) per-apply step 1): x_ext = [halo | x_owned | halo], the
// halo weights by grouped ncclSend / ncclRecv on the second communicator (stream-ordered on st).
__global__ void k_gather_x(int64_t n, const int* __restrict__ idx, const float* __restrict__ x, float* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = x[idx[i]];
}

void halo_copy_owned(fmmbem_ctx* c, const float* x_owned, cudaStream_t st) {
  const int64_t n = c->n_own();
  if (n) FMM_CUDA(cudaMemcpyAsync(c->xext.get() + c->pan_lo, x_owned, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
}

void halo_exchange(fmmbem_ctx* c, const float* x_owned, cudaStream_t st) {
  auto& H = c->halo;
  const int R = c->nranks, me = c->rank;
  if (H.sent) k_gather_x<<<ceil_div(H.sent, 256), 256, 0, st>>>(H.sent, H.sidx.get(), x_owned, H.sbuf.get());
  FMM_CHECK_LAUNCH();
  std::vector<const void*> sp(R);
  std::vector<void*> rp(R);
  std::vector<size_t> sn(R, 0), rn(R, 0);
  for (int p = 0; p < R; ++p) {
    sp[p] = H.sbuf.get() + H.soff[p];
    rp[p] = c->xext.get() + H.roff[p];
    if (p != me) {
      sn[p] = H.scnt[p] * sizeof(float);
      rn[p] = H.rcnt[p] * sizeof(float);
    }
  }
  comm_alltoallv_bytes(c, sp, sn, rp, rn, st, /*second=*/true);
}

}  // namespace fmm
