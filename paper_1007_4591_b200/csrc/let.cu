// let.cu -- local essential tree exchange of multipoles ("for the
// far-field, the data that needs to be communicated consists of ME coefficients of the cells in the
// interaction list, at every level of the tree").
//
// After the partition every rank knows every rank's contiguous leaf range, so each cell (levels >= 2)
// is either PURE -- all the leaves below it belong to one rank, which computes its complete
// multipole -- or SHARED -- the leaves below it straddle a rank boundary and several ranks hold
// partial multipoles.  Per matvec:
//   * every pure cell that rank p's targets need (it is in the interaction list of a target cell
//     holding p's panels) and that rank r owns is sent r -> p with grouped ncclSend / ncclRecv;
//   * the few shared cells are summed with one small ncclAllReduce.
// The lists are derived identically on every rank from the replicated tree and partition, in
// increasing cell order, so sender and receiver agree without any handshake.
#include <cub/cub.cuh>

#include "kernels.cuh"

namespace fmm {

namespace {

__device__ inline int lb_u64(const uint64_t* a, int n, uint64_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ inline int rank_of_leaf(const int* bounds, int R, int leaf) {
  int lo = 0, hi = R - 1;  // last r with bounds[r] <= leaf
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (bounds[mid] <= leaf) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// per cell of levels >= 2: first / end leaf of its subtree, owner rank (-1 = shared)
__global__ void k_cell_owner(int n, int c0, const uint64_t* __restrict__ key, const int* __restrict__ lvl_of,
                             int L, const uint64_t* __restrict__ lkey, int nl, const int* __restrict__ bounds, int R,
                             int* first, int* end, int* owner) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = c0 + i, l = lvl_of[c];
  const int sh = 3 * (L - l);
  const int f = lb_u64(lkey, nl, key[c] << sh), e = lb_u64(lkey, nl, (key[c] + 1) << sh);
  first[i] = f;
  end[i] = e;
  owner[i] = (e > f && rank_of_leaf(bounds, R, f) == rank_of_leaf(bounds, R, e - 1)) ? rank_of_leaf(bounds, R, f) : -1;
}

// need[s] = 1 if s (a source cell with sources) is in the interaction list of a target cell that holds
// panels of the leaf range [a, b)  (panel prefix sums over leaves decide "holds")
__global__ void k_mark_need(int n, int c0, const int* __restrict__ first, const int* __restrict__ end,
                            const long long* __restrict__ ppre, int a, int b, const int* __restrict__ off,
                            const int* __restrict__ idx, const int* __restrict__ scnt, unsigned char* need) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int f = max(first[i], a), e = min(end[i], b);
  if (e <= f || ppre[e] - ppre[f] == 0) return;
  const int c = c0 + i;
  for (int k = off[c]; k < off[c + 1]; ++k) {
    const int s = idx[k];
    if (scnt[s] > 0) need[s - c0] = 1;  // benign race: every writer stores 1
  }
}

__global__ void k_flag(int n, const unsigned char* __restrict__ need, const int* __restrict__ owner, int want_owner,
                       int shared_mode, const int* __restrict__ scnt, int c0, int* flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (shared_mode) flag[i] = (owner[i] < 0 && scnt[c0 + i] > 0) ? 1 : 0;
  else flag[i] = (need[i] && owner[i] == want_owner) ? 1 : 0;
}

__global__ void k_pack(int n, int NC, const int* __restrict__ cells, const float2* __restrict__ M, float2* buf) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * NC) return;
  const int i = (int)(t / NC), c = (int)(t - (int64_t)i * NC);
  buf[t] = M[(size_t)cells[i] * NC + c];
}

__global__ void k_unpack(int n, int NC, const int* __restrict__ cells, const float2* __restrict__ buf, float2* M) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * NC) return;
  const int i = (int)(t / NC), c = (int)(t - (int64_t)i * NC);
  M[(size_t)cells[i] * NC + c] = buf[t];
}

__global__ void k_level_of(int n, int off, int l, int* lvl) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) lvl[off + i] = l;
}

// compact indices (c0 + i) with flag[i] into out; returns count
int select_cells(const int* flag, int n, int c0, DevBuf<int>& out, cudaStream_t s) {
  DevBuf<int> pos;
  pos.alloc(n + 1);
  scan_ints(flag, pos.get(), n + 1, s);
  int tot = 0;
  FMM_CUDA(cudaMemcpyAsync(&tot, pos.get() + n, sizeof(int), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  out.alloc(std::max(tot, 1));
  std::vector<int> hf(n), hp(n + 1);
  // small host pass keeps the order explicit (cells in increasing index)
  FMM_CUDA(cudaMemcpyAsync(hf.data(), flag, n * sizeof(int), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  std::vector<int> h;
  h.reserve(tot);
  for (int i = 0; i < n; ++i)
    if (hf[i]) h.push_back(c0 + i);
  if (tot) FMM_CUDA(cudaMemcpyAsync(out.get(), h.data(), tot * sizeof(int), cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  return tot;
}

}  // namespace

void build_let(fmmbem_ctx* c, const std::vector<int64_t>& leaf_bounds, cudaStream_t s) {
  const Tree& T = c->tree;
  const int R = c->nranks, me = c->rank, L = T.L;
  auto& X = c->let;
  X.ready = false;
  if (R <= 1 || L < 2) return;
  const int c0 = (int)T.lvl_off[2], n = (int)(T.n_cells - c0), nl = (int)T.n_leaves;
  const PointSet& S = (c->K == 1) ? c->pan : c->quad;
  DevBuf<int> lvl, first, end, owner, bounds, flag;
  lvl.alloc(T.n_cells);
  for (int l = 0; l <= L; ++l) {
    const int m = (int)(T.lvl_off[l + 1] - T.lvl_off[l]);
    if (m) k_level_of<<<ceil_div(m, 256), 256, 0, s>>>(m, (int)T.lvl_off[l], l, lvl.get());
  }
  bounds.alloc(R + 1);
  std::vector<int> hb(leaf_bounds.begin(), leaf_bounds.end());
  FMM_CUDA(cudaMemcpyAsync(bounds.get(), hb.data(), (R + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
  first.alloc(n);
  end.alloc(n);
  owner.alloc(n);
  k_cell_owner<<<ceil_div(n, 256), 256, 0, s>>>(n, c0, T.key.get(), lvl.get(), L, T.key.get() + T.lvl_off[L], nl,
                                                 bounds.get(), R, first.get(), end.get(), owner.get());
  FMM_CHECK_LAUNCH();
  // panel prefix sums over leaves
  DevBuf<long long> ppre;
  {
    std::vector<int> b(nl + 1);
    FMM_CUDA(cudaMemcpyAsync(b.data(), c->pan.begin.get(), (nl + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    std::vector<long long> pp(nl + 1);
    for (int k = 0; k <= nl; ++k) pp[k] = b[k];
    ppre.alloc(nl + 1);
    FMM_CUDA(cudaMemcpyAsync(ppre.get(), pp.data(), (nl + 1) * sizeof(long long), cudaMemcpyHostToDevice, s));
  }
  DevBuf<unsigned char> need;
  need.alloc(n);
  flag.alloc(n + 1);
  X.send.clear();
  X.recv.clear();
  X.send.resize(R);
  X.recv.resize(R);
  X.nsend.assign(R, 0);
  X.nrecv.assign(R, 0);
  for (int p = 0; p < R; ++p) {
    need.zero(s);
    k_mark_need<<<ceil_div(n, 256), 256, 0, s>>>(n, c0, first.get(), end.get(), ppre.get(), (int)leaf_bounds[p],
                                                 (int)leaf_bounds[p + 1], T.m2l_off.get(), T.m2l_idx.get(),
                                                 S.cell_cnt.get(), need.get());
    FMM_CHECK_LAUNCH();
    if (p != me) {  // pure cells I own that p needs
      FMM_CUDA(cudaMemsetAsync(flag.get() + n, 0, sizeof(int), s));
      k_flag<<<ceil_div(n, 256), 256, 0, s>>>(n, need.get(), owner.get(), me, 0, S.cell_cnt.get(), c0, flag.get());
      X.nsend[p] = select_cells(flag.get(), n, c0, X.send[p], s);
    } else {  // pure cells owned by r that I need
      for (int r = 0; r < R; ++r) {
        if (r == me) continue;
        FMM_CUDA(cudaMemsetAsync(flag.get() + n, 0, sizeof(int), s));
        k_flag<<<ceil_div(n, 256), 256, 0, s>>>(n, need.get(), owner.get(), r, 0, S.cell_cnt.get(), c0, flag.get());
        X.nrecv[r] = select_cells(flag.get(), n, c0, X.recv[r], s);
      }
    }
  }
  FMM_CUDA(cudaMemsetAsync(flag.get() + n, 0, sizeof(int), s));
  k_flag<<<ceil_div(n, 256), 256, 0, s>>>(n, need.get(), owner.get(), 0, 1, S.cell_cnt.get(), c0, flag.get());
  X.nshared = select_cells(flag.get(), n, c0, X.shared, s);
  int64_t ts = 0, tr = 0;
  for (int p = 0; p < R; ++p) {
    ts += X.nsend[p];
    tr += X.nrecv[p];
  }
  X.sbuf.alloc(std::max<int64_t>(ts, 1) * c->NC);
  X.rbuf.alloc(std::max<int64_t>(tr, 1) * c->NC);
  X.shbuf.alloc(std::max<int64_t>(X.nshared, 1) * c->NC);
  X.cells_sent = ts;
  X.cells_recv = tr;
  X.ready = true;
}

// the multipole part of the LET: pure cells point to point, shared cells summed
void exchange_let(fmmbem_ctx* c, cudaStream_t s) {
  auto& X = c->let;
  const int R = c->nranks, NC = c->NC;
  float2* M = c->Mx.get();
  int64_t so = 0;
  for (int p = 0; p < R; ++p) {
    if (X.nsend[p]) {
      const int64_t m = (int64_t)X.nsend[p] * NC;
      k_pack<<<ceil_div(m, 256), 256, 0, s>>>(X.nsend[p], NC, X.send[p].get(), M, X.sbuf.get() + so);
      so += m;
    }
  }
  if (X.nshared)
    k_pack<<<ceil_div((int64_t)X.nshared * NC, 256), 256, 0, s>>>(X.nshared, NC, X.shared.get(), M, X.shbuf.get());
  FMM_CHECK_LAUNCH();
  std::vector<size_t> sc(R), rc(R);
  std::vector<float*> sp(R), rp(R);
  int64_t ro = 0;
  so = 0;
  for (int p = 0; p < R; ++p) {
    sc[p] = (size_t)X.nsend[p] * NC * 2;
    rc[p] = (size_t)X.nrecv[p] * NC * 2;
    sp[p] = reinterpret_cast<float*>(X.sbuf.get() + so);
    rp[p] = reinterpret_cast<float*>(X.rbuf.get() + ro);
    so += (int64_t)X.nsend[p] * NC;
    ro += (int64_t)X.nrecv[p] * NC;
  }
  comm_sendrecv_f32(c, sp, sc, rp, rc, s);
  if (X.nshared)
    comm_allreduce_f32(c, reinterpret_cast<float*>(X.shbuf.get()), (size_t)X.nshared * NC * 2, s);
  ro = 0;
  for (int p = 0; p < R; ++p) {
    if (X.nrecv[p]) {
      const int64_t m = (int64_t)X.nrecv[p] * NC;
      k_unpack<<<ceil_div(m, 256), 256, 0, s>>>(X.nrecv[p], NC, X.recv[p].get(), X.rbuf.get() + ro, M);
      ro += m;
    }
  }
  if (X.nshared)
    k_unpack<<<ceil_div((int64_t)X.nshared * NC, 256), 256, 0, s>>>(X.nshared, NC, X.shared.get(), X.shbuf.get(), M);
  FMM_CHECK_LAUNCH();
}

}  // namespace fmm
