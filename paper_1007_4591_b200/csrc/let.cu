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
// increasing cell order, so sender and receiver agree without any handshake.  Multipoles live in
// the rank's expansion slots (plan.h slot_layout): the lists are stored as slots.  The charge-FMM
// has its own pair of lists (cells with charges that the panels of a peer need).
#include <cub/cub.cuh>

#include "kernels.cuh"

namespace fmm {

namespace {

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


}  // namespace

namespace {

// device copies of one pair of LET cell lists, as expansion SLOTS (plan.h slot_layout)
void build_one(fmmbem_ctx* c, LetPlan& X, const std::vector<std::vector<int>>& snd,
               const std::vector<std::vector<int>>& rcv, const std::vector<int>& shr, cudaStream_t s) {
  const int R = c->nranks, me = c->rank;
  const ExchangePlan& P = c->xplan;
  X.ready = false;
  auto up = [&](const std::vector<int>& v, DevBuf<int>& d) {
    std::vector<int> sl(v.size());
    for (size_t i = 0; i < v.size(); ++i) {
      const int64_t k = P.slot(v[i]);
      if (k < 0) throw Error(FMMBEM_E_CUDA, "LET cell without an expansion slot");
      sl[i] = (int)k;
    }
    d.alloc(std::max<size_t>(sl.size(), 1));
    if (!sl.empty()) FMM_CUDA(cudaMemcpyAsync(d.get(), sl.data(), sl.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    return (int)sl.size();
  };
  X.send.clear();
  X.recv.clear();
  X.send.resize(R);
  X.recv.resize(R);
  X.nsend.assign(R, 0);
  X.nrecv.assign(R, 0);
  int64_t ts = 0, tr = 0;
  for (int p = 0; p < R; ++p) {
    if (p == me) continue;
    X.nsend[p] = up(snd[p], X.send[p]);
    X.nrecv[p] = up(rcv[p], X.recv[p]);
    ts += X.nsend[p];
    tr += X.nrecv[p];
  }
  X.nshared = up(shr, X.shared);
  X.sbuf.alloc(std::max<int64_t>(ts, 1) * c->NC);
  X.rbuf.alloc(std::max<int64_t>(tr, 1) * c->NC);
  X.shbuf.alloc(std::max<int64_t>(X.nshared, 1) * c->NC);
  X.cells_sent = ts;
  X.cells_recv = tr;
  X.ready = true;
}

}  // namespace

// the LET plans of the panel and the charge multipoles (plan.cu; identical derivation on every rank)
void build_let(fmmbem_ctx* c, cudaStream_t s) {
  c->let.ready = c->let_chg.ready = false;
  if (c->nranks <= 1 || c->tree.L < 2) return;
  const ExchangePlan& P = c->xplan;
  build_one(c, c->let, P.let_send, P.let_recv, P.let_shared, s);
  build_one(c, c->let_chg, P.let_send_chg, P.let_recv_chg, P.let_shared_chg, s);
}

// the multipole part of the LET: pure cells point to point, shared cells summed
void exchange_let(fmmbem_ctx* c, const LetPlan& X, cudaStream_t s) {
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
