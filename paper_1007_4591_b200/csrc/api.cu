// api.cu -- the C ABI of libfmmbem (include/fmmbem.h) and the orchestration of one FMM
// evaluation.  Every step of the path runs in this library's kernels;
// the host only validates, launches and runs the small FP64 GMRES least-squares problem.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "kernels.cuh"

static thread_local std::string g_err = "";

namespace fmm {

namespace {

constexpr double FOUR_PI = 12.566370614359172953850573533118;
constexpr double KCAL = 4.0 * 3.14159265358979323846 * 332.0637;  // SPEC S:409 (A13)

// Appendix C quadrature rules (barycentric beta, weight); K = 1 is the paper's centroid rule
// (P:409-411).  Independent copy of the table (the oracle keeps its own).
void quad_rule(int K, std::vector<double>& beta, std::vector<double>& w) {
  beta.clear();
  w.clear();
  auto add3 = [&](double a, double b, double wt) {
    double p[3][3] = {{a, b, b}, {b, a, b}, {b, b, a}};
    for (auto& r : p) {
      beta.insert(beta.end(), r, r + 3);
      w.push_back(wt);
    }
  };
  if (K == 1) {
    beta = {1.0 / 3, 1.0 / 3, 1.0 / 3};
    w = {1.0};
  } else if (K == 3) {
    add3(2.0 / 3, 1.0 / 6, 1.0 / 3);
  } else if (K == 6) {
    add3(0.108103018168070, 0.445948490915965, 0.223381589678011);
    add3(0.816847572980459, 0.091576213509771, 0.109951743655322);
  } else if (K == 7) {
    beta = {1.0 / 3, 1.0 / 3, 1.0 / 3};
    w = {0.225};
    add3(0.059715871789770, 0.470142064105115, 0.132394152788506);
    add3(0.797426985353087, 0.101286507323456, 0.125939180544827);
  }
}

// Panel prep: FP64 centroid, unit normal from
// the winding, area, quadrature points.  Bad triangles are flagged by the smallest offending index
// per kind: bad[0] vertex index out of range, bad[1] non-finite vertex, bad[2] degenerate.
__global__ void k_prep(int64_t np, int64_t nv, const double* __restrict__ V, const int* __restrict__ T, int K,
                       const double* __restrict__ beta, double atol, double* cen, double* nrm, double* area,
                       double* qp, unsigned long long* bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= np) return;
  int a = T[3 * i], b = T[3 * i + 1], c = T[3 * i + 2];
  if (a < 0 || b < 0 || c < 0 || a >= nv || b >= nv || c >= nv) {
    atomicMin(&bad[0], (unsigned long long)i);
    return;
  }
  const double* A = V + 3 * (int64_t)a;
  const double* B = V + 3 * (int64_t)b;
  const double* C = V + 3 * (int64_t)c;
  for (int d = 0; d < 3; ++d)
    if (!isfinite(A[d]) || !isfinite(B[d]) || !isfinite(C[d])) {
      atomicMin(&bad[1], (unsigned long long)i);
      return;
    }
  double e1[3] = {B[0] - A[0], B[1] - A[1], B[2] - A[2]};
  double e2[3] = {C[0] - A[0], C[1] - A[1], C[2] - A[2]};
  double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
  double nn = sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
  if (!(0.5 * nn >= atol)) {
    atomicMin(&bad[2], (unsigned long long)i);
    return;
  }
  for (int d = 0; d < 3; ++d) {
    cen[3 * i + d] = (A[d] + B[d] + C[d]) / 3.0;
    nrm[3 * i + d] = cr[d] / nn;
  }
  area[i] = 0.5 * nn;
  if (qp)
    for (int g = 0; g < K; ++g)
      for (int d = 0; d < 3; ++d)
        qp[(i * K + g) * 3 + d] = beta[3 * g] * A[d] + beta[3 * g + 1] * B[d] + beta[3 * g + 2] * C[d];
}

// bounding box of the finite vertex coordinates: out = (min xyz, -max xyz) per block
__global__ void k_vbox(int64_t n, const double* __restrict__ V, double* out) {
  double v[6] = {1e300, 1e300, 1e300, 1e300, 1e300, 1e300};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < 3; ++d) {
      const double x = V[3 * i + d];
      if (isfinite(x)) {
        v[d] = fmin(v[d], x);
        v[3 + d] = fmin(v[3 + d], -x);
      }
    }
  for (int k = 0; k < 6; ++k)
    for (int o = 16; o > 0; o >>= 1) v[k] = fmin(v[k], __shfl_xor_sync(0xffffffffu, v[k], o));
  __shared__ double sh[8][6];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 6; ++k) sh[w][k] = v[k];
  __syncthreads();
  if (threadIdx.x < 6) {
    double r = 1e300;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = fmin(r, sh[i][threadIdx.x]);
    out[blockIdx.x * 6 + threadIdx.x] = r;
  }
}

__global__ void k_scale(float* y, const float* x, int64_t n, float s) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = s * x[i];
}

// psi_j = sum_g (A_j w_g / A_j) psi_jg
__global__ void k_quad_reduce(int64_t np, int K, const float* __restrict__ psiq, const float4* __restrict__ qpos,
                              const float4* __restrict__ ppos, float* psi) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= np) return;
  float s = 0.f, ia = 1.f / ppos[i].w;
  for (int g = 0; g < K; ++g) s = fmaf(qpos[i * K + g].w * ia, psiq[i * K + g], s);
  psi[i] = s;
}

__global__ void k_unpermute(int64_t n, const int* __restrict__ ids, const float* __restrict__ v, double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[ids[i]] = (double)v[i];
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Stream ordering between entry points (the library's internal state -- expansions, staging
// buffers, the P2P source table -- is shared by every call): each call first makes the stream it
// runs on wait for the end of the previous call, and records c->done when its own work is queued.
void order_after_last(fmmbem_ctx* c, cudaStream_t st) { FMM_CUDA(cudaStreamWaitEvent(st, c->done, 0)); }
void mark_done(fmmbem_ctx* c, cudaStream_t st) { FMM_CUDA(cudaEventRecord(c->done, st)); }

bool multi(const fmmbem_ctx* c) { return c->nranks > 1; }

// Sources of the panel operators (K', V, A): x_local is this rank's slice.  With nranks > 1 the
// source weights live in c->xext = [halo | owned | halo] (local point indices): the owned slice is
// copied in here (before the far-field fork: P2M reads it), the peers' halo weights arrive by the
// grouped send / recv fmm_eval issues on the caller's stream for the near field (P2P).
SrcArg kp_src(fmmbem_ctx* c, const float* x_local, cudaStream_t st, bool* distributed) {
  SrcArg s;
  s.set = (c->K == 1) ? &c->pan : &c->quad;
  s.x = x_local;
  *distributed = false;
  if (multi(c)) {
    halo_copy_owned(c, x_local, st);
    s.x = c->xext.get();
    s.halo_src = x_local;
    s.leaf_lo = c->leaf_lo;
    s.leaf_hi = c->leaf_hi;
    s.cnt = (c->K == 1) ? c->pan_own_cnt.get() : c->quad_own_cnt.get();
    *distributed = true;
  }
  return s;
}

// targets = this rank's panels (all panels on one GPU)
TgtArg own_targets(fmmbem_ctx* c, bool quad) {
  TgtArg t;
  t.set = quad ? &c->quad : &c->pan;
  if (multi(c)) {
    t.leaf_lo = c->leaf_lo;
    t.leaf_hi = c->leaf_hi;
    t.cnt = quad ? c->quad_own_cnt.get() : c->pan_own_cnt.get();
  }
  return t;
}

// FMMBEM_VERBOSE: device bytes held by the ctx after create, by group, on stderr
void report_memory(const fmmbem_ctx* c) {
  auto b = [](const auto& d) { return (double)d.n * sizeof(*d.p); };
  auto pts = [&](const PointSet& p) { return b(p.pos) + b(p.nrm) + b(p.leaf) + b(p.begin) + b(p.cell_cnt); };
  const Tree& T = c->tree;
  double m2lw = 0, items = 0, let = 0;
  for (const auto& w : c->m2l_cache) m2lw += b(w->idx) + b(w->cell) + b(w->off);
  for (const auto& w : c->p2p_cache) items += b(w->items);
  for (const LetPlan* X : {&c->let, &c->let_chg}) {
    for (const auto& d : X->send) let += b(d);
    for (const auto& d : X->recv) let += b(d);
    let += b(X->shared) + b(X->sbuf) + b(X->rbuf) + b(X->shbuf);
  }
  const double skel = b(T.key) + b(T.parent) + b(T.child_begin) + b(T.child_end) + b(T.leaf_ijk) + b(c->gbeg) +
                      b(c->pan_own_cnt) + b(c->quad_own_cnt) + b(c->chg_own_cnt) + b(c->cmap) + b(c->skey);
  const double lists = b(T.nbr_off) + b(T.nbr_idx) + b(T.m2l_off) + b(T.m2l_idx);
  const double other = b(c->xext) + b(c->p2p_src) + b(c->halo.sidx) + b(c->halo.sbuf) + b(c->selfd) +
                       b(c->near.off) + b(c->near.col) + b(c->near.vkp) + b(c->near.vsl) + b(c->near.diag) +
                       b(c->Itab) + b(c->tmp_x) + b(c->tmp_y) + b(c->chg_ids);
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  std::fprintf(stderr,
               "[fmmbem rank %d] device GB: points %.3f (panels %.3f, quad %.3f, charges %.3f), expansions %.3f "
               "(%lld of %lld cells), skeleton %.3f, lists %.3f, M2L work %.3f, P2P items %.3f, LET %.3f, "
               "other %.3f; device used %.3f\n",
               c->rank, (pts(c->pan) + pts(c->quad) + pts(c->chg)) / 1e9, pts(c->pan) / 1e9, pts(c->quad) / 1e9,
               pts(c->chg) / 1e9, (b(c->Mx) + b(c->Lx)) / 1e9, (long long)c->n_slots, (long long)T.n_cells,
               skel / 1e9, lists / 1e9, m2lw / 1e9, items / 1e9, let / 1e9, other / 1e9, (double)(tot - fr) / 1e9);
}

}  // namespace

enum : int {
  E_START = 0, E_UP0, E_UP1, E_AR0, E_AR1, E_M2L0, E_M2L1, E_DN1, E_P2P0, E_P2P1, E_L2P0, E_L2P1, E_AG0, E_AG1,
  E_NEAR1, E_XG0, E_XG1, E_P2M1, E_L2L1, E_BIB0, E_BIB1, E_END
};

// Option self_term = 1: K'_ii = -H_i sqrt(A_i / pi) / 4, the principal-value integral of
// dG/dn_i over panel i modelled as a spherical cap of mean curvature H_i.  H_i from the mesh in
// FP64 on the host: vertex normals = normalised sums of the incident faces' area-weighted normals;
// the normal curvature along the chord centroid -> vertex a is (n_a - n_i).(v_a - c_i)/|v_a - c_i|^2,
// and H_i is the mean over the three vertices.  Stored in local order, times 4 pi (the kernels
// sum raw 1/r^3 terms and apply 1/(4 pi) in the epilogue).
void build_self_term(fmmbem_ctx* c, const fmmbem_mesh* mesh, cudaStream_t s) {
  const int64_t nv = mesh->n_vertices, np = mesh->n_triangles;
  const double* V = mesh->xyz;
  const int* T = mesh->tri;
  std::vector<double> vn(3 * nv, 0.0), fn(3 * np), cen(3 * np), area(np);
  for (int64_t t = 0; t < np; ++t) {
    const double* a = V + 3 * T[3 * t];
    const double* b = V + 3 * T[3 * t + 1];
    const double* q = V + 3 * T[3 * t + 2];
    const double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]}, e2[3] = {q[0] - a[0], q[1] - a[1], q[2] - a[2]};
    const double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
    const double len = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
    area[t] = 0.5 * len;
    for (int d = 0; d < 3; ++d) {
      fn[3 * t + d] = cr[d] / len;
      cen[3 * t + d] = (a[d] + b[d] + q[d]) / 3.0;
      for (int k = 0; k < 3; ++k) vn[3 * T[3 * t + k] + d] += 0.5 * cr[d];  // area-weighted face normal
    }
  }
  for (int64_t v = 0; v < nv; ++v) {
    const double l = std::sqrt(vn[3 * v] * vn[3 * v] + vn[3 * v + 1] * vn[3 * v + 1] + vn[3 * v + 2] * vn[3 * v + 2]);
    if (l > 0)
      for (int d = 0; d < 3; ++d) vn[3 * v + d] /= l;
  }
  const int64_t nloc = c->pan.n;  // local points (owned + halo), pan_ids = their global triangle ids
  std::vector<float> dl(nloc);
  for (int64_t k = 0; k < nloc; ++k) {
    const int64_t t = c->pan_ids[k];
    double H = 0.0;
    for (int j = 0; j < 3; ++j) {
      const int64_t v = T[3 * t + j];
      double num = 0.0, den = 0.0;
      for (int d = 0; d < 3; ++d) {
        const double ch = V[3 * v + d] - cen[3 * t + d];
        num += (vn[3 * v + d] - fn[3 * t + d]) * ch;
        den += ch * ch;
      }
      H += num / den;
    }
    H /= 3.0;
    dl[k] = (float)(-H * std::sqrt(area[t] / M_PI) / 4.0 * 4.0 * M_PI);
  }
  c->selfd.alloc(std::max<int64_t>(nloc, 1));
  if (nloc) FMM_CUDA(cudaMemcpyAsync(c->selfd.get(), dl.data(), nloc * sizeof(float), cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaStreamSynchronize(s));
}

// One FMM (or direct) evaluation.  With c->overlap the near field (P2P, independent of every
// expansion) runs on a side stream concurrently with the upward sweep, the multipole exchange and
// M2L/L2L; L2P then waits for it (y is first written by P2P, L2P accumulates).
void fmm_eval(fmmbem_ctx* c, const TgtArg& t, const SrcArg& s, const Outputs& o, bool self, bool check,
              cudaStream_t st, bool timing, bool distributed) {
  const bool direct = c->opt.direct != 0 || c->tree.L < 2;
  auto rec = [&](int e, cudaStream_t q) {
    if (timing) cudaEventRecord(c->ev[e], q);
  };
  rec(E_START, st);
  // with overlap the far-field chain (upward sweep, multipole exchange, M2L, L2L) runs on a
  // high-priority internal stream and the near field on the caller's stream: the block scheduler
  // gives the chain (and NCCL) SMs first and P2P fills the rest
  const bool ovl = c->overlap && !direct;
  cudaStream_t fs = ovl ? c->side : st;
  if (ovl) {
    FMM_CUDA(cudaEventRecord(c->fork, st));
    FMM_CUDA(cudaStreamWaitEvent(fs, c->fork, 0));
  }
  if (!direct) {
    rec(E_UP0, fs);
    const SrcArg& sf = s;
    c->Mx.zero(fs);  // the upward sweep, split for the phase events: P2M, then M2M level by level
    if (sf.dipole) launch_p2m_dipole(c, sf, sf.leaf_lo, sf.leaf_hi < 0 ? (int)c->tree.n_leaves : sf.leaf_hi, fs);
    else launch_p2m_range(c, sf, sf.leaf_lo, sf.leaf_hi < 0 ? (int)c->tree.n_leaves : sf.leaf_hi, fs);
    rec(E_P2M1, fs);
    launch_m2m_levels(c, sf, fs);
    rec(E_UP1, fs);
    if (distributed) {  // the multipoles this rank's interaction lists need (LET)
      rec(E_AR0, fs);
      const LetPlan& X = (s.set == &c->chg) ? c->let_chg : c->let;
      if (!X.ready) throw Error(FMMBEM_E_CUDA, "distributed evaluation without a LET plan");
      exchange_let(c, X, fs);
      rec(E_AR1, fs);
    }
    const int* tcnt = t.cnt ? t.cnt : t.set->cell_cnt.get();
    rec(E_M2L0, fs);
    launch_m2l(c, s.set->cell_cnt.get(), tcnt, fs);
    rec(E_M2L1, fs);
    launch_downward(c, tcnt, fs);
    rec(E_DN1, fs);
    rec(E_L2L1, fs);
  }
  if (ovl) FMM_CUDA(cudaEventRecord(c->join, fs));
  if (s.halo_src) {  // the peers' halo weights for the near field, overlapped with the far chain
    rec(E_XG0, st);
    halo_exchange(c, s.halo_src, st);
    rec(E_XG1, st);
  }
  rec(E_P2P0, st);
  if (s.dipole) launch_p2p_dipole(c, t, s, o.pot.y, o.pot.b, c->opt.direct != 0 || c->tree.L < 2, st);
  else launch_p2p(c, t, s, o, self, check, c->opt.direct != 0, st);
  rec(E_P2P1, st);
  if (ovl) FMM_CUDA(cudaStreamWaitEvent(st, c->join, 0));
  rec(E_L2P0, st);
  if (!direct) {
    Outputs acc = o;
    acc.pot.x = nullptr;
    acc.dn.x = nullptr;
    launch_l2p(c, t, acc, st);
  }
  rec(E_L2P1, st);
  c->timed_comm = timing && distributed && !direct;
  c->timed_xg = timing && s.halo_src != nullptr;
}

// y = op(x) on this rank's panels; x, y local slices (pointers are shifted so that the kernels'
// global tree indices land in the slice)
Outputs op_outputs(fmmbem_ctx* c, fmmbem_op op, const float* xg, float* yg) {
  Outputs o;
  if (op == FMMBEM_OP_SINGLE || op == FMMBEM_OP_DOUBLE) {
    o.pot.y = yg;
    o.pot.b = (float)(1.0 / FOUR_PI);
  } else {
    o.dn.y = yg;
    if (op == FMMBEM_OP_KPRIME) {
      o.dn.b = (float)(1.0 / FOUR_PI);
    } else {  // A = I - f K'
      o.dn.x = xg;
      o.dn.ax = 1.f;
      o.dn.b = (float)(-c->f / FOUR_PI);
    }
    if (c->selfd.n) {  // K'_ii = d_i (stored times 4 pi, like the raw kernel sums)
      o.dn.x = xg;
      o.dn.d = c->selfd.get();
    }
  }
  return o;
}

void apply_op(fmmbem_ctx* c, fmmbem_op op, const float* x, float* y, cudaStream_t st, bool timing) {
  TgtArg t = own_targets(c, false);
  float* yg = y - c->pan_lo;
  const float* xg = x - c->pan_lo;
  Outputs o = op_outputs(c, op, xg, yg);
  bool dist = false;
  if (timing) cudaEventRecord(c->ev[E_AG0], st);
  SrcArg s = kp_src(c, x, st, &dist);
  s.dipole = (op == FMMBEM_OP_DOUBLE);
  if (timing) cudaEventRecord(c->ev[E_AG1], st);
  fmm_eval(c, t, s, o, /*self=*/true, /*check=*/false, st, timing, dist);
  if (c->opt.near_mode && op != FMMBEM_OP_DOUBLE) {  // analytic near-field correction (a11): y += b C x
    const bool single = (op == FMMBEM_OP_SINGLE);
    const float b = (op == FMMBEM_OP_A) ? (float)(-c->f) : 1.f;
    apply_near(c, single, s.x, yg, b, st);
  }
  if (timing) cudaEventRecord(c->ev[E_NEAR1], st);
  c->timed_near = timing;
  c->timed_fields = false;
}

void apply_A(fmmbem_ctx* c, const float* x, float* y, cudaStream_t s) { apply_op(c, FMMBEM_OP_A, x, y, s, false); }

void ensure_fields(fmmbem_ctx* c, cudaStream_t st) {
  if (c->have_fields) return;
  const int64_t n = c->n_own();
  c->En.alloc(std::max<int64_t>(n, 1));
  c->psi.alloc(std::max<int64_t>(n, 1));
  if (c->nc == 0) {
    c->En.zero(st);
    c->psi.zero(st);
    c->have_fields = true;
    return;
  }
  FMM_CUDA(cudaMemsetAsync(c->flag.get(), 0, sizeof(int), st));
  TgtArg t = own_targets(c, false);
  SrcArg s;  // the charges of this rank's leaves; the other ranks' charge multipoles by the LET
  s.set = &c->chg;
  if (multi(c)) {
    s.leaf_lo = c->leaf_lo;
    s.leaf_hi = c->leaf_hi;
    s.cnt = c->chg_own_cnt.get();
  }
  Outputs o;
  o.dn.y = c->En.get() - c->pan_lo;
  o.dn.b = (float)(1.0 / (FOUR_PI * c->eps_in));  // E_n carries 1/eps_I (Eq. 1, reading A2)
  if (c->K == 1) {
    o.pot.y = c->psi.get() - c->pan_lo;
    o.pot.b = (float)(1.0 / FOUR_PI);
  }
  // the charge-FMM runs at its own order (options.charge_terms): every far-field launcher reads
  // c->P / c->NC, and the expansion / LET buffers are sized for terms >= charge_terms
  struct OrderScope {
    fmmbem_ctx* c;
    int P0, NC0;
    OrderScope(fmmbem_ctx* c_, int P) : c(c_), P0(c_->P), NC0(c_->NC) {
      c->P = P;
      c->NC = P * (P + 1) / 2;
    }
    ~OrderScope() {
      c->P = P0;
      c->NC = NC0;
    }
  } order(c, c->P_chg);
  // phase events of this charge-FMM (fmmbem_last_timing reports them until the next matvec)
  if (c->p2p_inter_chg < 0 && c->tree.L >= 2 && !c->opt.direct)
    c->p2p_inter_chg = count_p2p(c, c->pan, c->chg, false, false, c->leaf_lo, c->leaf_hi);
  cudaEventRecord(c->ev[E_AG0], st);
  // the charge-on-panel-point check (A14) depends on the geometry only: done at the first evaluation
  const bool check = !c->fields_checked;
  fmm_eval(c, t, s, o, false, check, st, true, multi(c));
  cudaEventRecord(c->ev[E_NEAR1], st);
  c->timed_near = true;
  c->timed_xg = false;
  c->timed_fields = true;
  if (c->K > 1) {
    DevBuf<float> psiq;
    psiq.alloc(c->quad.n);
    TgtArg tq = own_targets(c, true);
    Outputs oq;
    oq.pot.y = psiq.get();
    oq.pot.b = (float)(1.0 / FOUR_PI);
    fmm_eval(c, tq, s, oq, false, check, st, false, multi(c));
    if (n > 0)
      k_quad_reduce<<<ceil_div(n, 256), 256, 0, st>>>(n, c->K, psiq.get() + c->pan_lo * c->K,
                                                      c->quad.pos.get() + c->pan_lo * c->K,
                                                      c->pan.pos.get() + c->pan_lo, c->psi.get());
    FMM_CHECK_LAUNCH();
    FMM_CUDA(cudaStreamSynchronize(st));
  }
  int flag = 0;  // only the checked evaluation can raise it: later calls stay asynchronous
  if (check) {
    FMM_CUDA(cudaMemcpyAsync(&flag, c->flag.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
  }
  if (check && multi(c)) {  // the verdict is collective: every rank throws or none does
    double f = flag ? 1.0 : 0.0;
    c->red.alloc(std::max<size_t>(c->red.n, 64));
    FMM_CUDA(cudaMemcpyAsync(c->red.get(), &f, sizeof(f), cudaMemcpyHostToDevice, st));
    comm_allreduce_f64(c, c->red.get(), 1, st);
    FMM_CUDA(cudaMemcpyAsync(&f, c->red.get(), sizeof(f), cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    flag = f > 0.0;
  }
  if (flag) throw Error(FMMBEM_E_COINCIDENT, "a charge coincides with a panel quadrature point");
  c->fields_checked = true;
  c->have_fields = true;
}

void fill_timing(fmmbem_ctx* c, bool direct) {
  fmmbem_timing& T = c->last;
  const double g = T.gmres, tr = T.tree, bb = T.bibee;
  std::memset(&T, 0, sizeof(T));
  T.gmres = g;
  T.tree = tr;
  T.bibee = bb;
  if (!c->timed_near) return;
  cudaEventSynchronize(c->ev[E_NEAR1]);
  auto el = [&](int a, int b) {
    float ms = 0.f;
    return cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]) == cudaSuccess ? (double)ms : 0.0;
  };
  if (!direct) {
    T.upward = el(E_UP0, E_UP1);
    T.p2m = el(E_UP0, E_P2M1);
    T.m2m = el(E_P2M1, E_UP1);
    T.m2l = el(E_M2L0, E_M2L1);
    T.l2l = el(E_M2L1, E_DN1);
    T.leaf_l2p = el(E_L2P0, E_L2P1);
    T.l2p = T.l2l + T.leaf_l2p;
  }
  T.p2p = el(E_P2P0, E_P2P1);
  T.near = el(E_L2P1, E_NEAR1);
  if (c->timed_comm) T.comm = el(E_AR0, E_AR1) + (c->timed_xg ? el(E_XG0, E_XG1) : el(E_AG0, E_AG1));
  T.total = el(E_AG0, E_NEAR1);  // wall time of the whole product (overlapped phases counted once)
  T.p2p_interactions = c->timed_fields ? c->p2p_inter_chg : c->p2p_inter_kp;
  T.m2l_pairs = direct ? 0 : c->m2l_pairs_kp;
}

}  // namespace fmm

using namespace fmm;

#define API_BEGIN try {
#define API_END                                    \
  }                                                \
  catch (const fmm::Error& e) {                    \
    g_err = e.what();                              \
    return e.code;                                 \
  }                                                \
  catch (const std::exception& e) {                \
    g_err = e.what();                              \
    return FMMBEM_E_CUDA;                          \
  }

extern "C" {

const char* fmmbem_last_error(void) { return g_err.c_str(); }

int32_t fmmbem_abi_version(void) { return FMMBEM_ABI_VERSION; }

int64_t fmmbem_struct_size(const char* name) {
  if (!name) return -1;
  const std::string n(name);
  if (n == "options") return sizeof(fmmbem_options);
  if (n == "timing") return sizeof(fmmbem_timing);
  if (n == "energy") return sizeof(fmmbem_energy);
  if (n == "tree_info") return sizeof(fmmbem_tree_info);
  if (n == "solve_options") return sizeof(fmmbem_solve_options);
  return -1;
}

fmmbem_status fmmbem_default_options(fmmbem_options* o) {
  if (!o) return FMMBEM_E_INVALID;
  std::memset(o, 0, sizeof(*o));
  o->struct_size = sizeof(fmmbem_options);
  o->terms = 10;
  o->leaf_points = 64;
  o->quad_points = 1;
  o->near_mode = 0;
  o->near_radius = 3.f;
  o->self_term = 0;
  o->direct = 0;
  o->deterministic = 1;
  o->device = 0;
  o->rank = 0;
  o->nranks = 1;
  o->nccl_id = nullptr;
  o->input_mode = 0;
  o->charge_terms = 0;
  return FMMBEM_OK;
}

fmmbem_status fmmbem_create(const fmmbem_mesh* mesh, const fmmbem_charges* chg, double eps_in, double eps_out,
                            const fmmbem_options* opt_in, fmmbem_ctx** out) {
  if (out) *out = nullptr;
  fmmbem_ctx* c = nullptr;
  API_BEGIN
  if (!out || !mesh) throw Error(FMMBEM_E_INVALID, "null argument");
  fmmbem_options opt;
  fmmbem_default_options(&opt);
  if (opt_in) {
    if (opt_in->struct_size != (int)sizeof(fmmbem_options)) throw Error(FMMBEM_E_INVALID, "options.struct_size mismatch");
    opt = *opt_in;
  }
  if (opt.terms < 2 || opt.terms > MAX_TERMS) throw Error(FMMBEM_E_INVALID, "terms must be in [2, 16]");
  if (opt.leaf_points < 1) throw Error(FMMBEM_E_INVALID, "leaf_points must be >= 1");
  if (!(opt.quad_points == 1 || opt.quad_points == 3 || opt.quad_points == 6 || opt.quad_points == 7))
    throw Error(FMMBEM_E_INVALID, "quad_points must be 1, 3, 6 or 7");
  if (opt.near_mode != 0 && opt.near_mode != 1) throw Error(FMMBEM_E_INVALID, "near_mode must be 0 or 1");
  if (opt.near_mode == 1 && !(opt.near_radius > 0.f)) throw Error(FMMBEM_E_INVALID, "near_radius must be > 0");
  if (opt.self_term != 0 && opt.self_term != 1) throw Error(FMMBEM_E_INVALID, "self_term must be 0 or 1");
  if (opt.nranks < 1 || opt.nranks > 64 || opt.rank < 0 || opt.rank >= opt.nranks)
    throw Error(FMMBEM_E_INVALID, "bad rank / nranks (1..64 ranks)");
  if (opt.nranks > 1 && !opt.nccl_id) throw Error(FMMBEM_E_INVALID, "nranks > 1 needs options.nccl_id");
  if (opt.nranks > 1 && opt.direct) throw Error(FMMBEM_E_INVALID, "direct mode is single-GPU only");
  if (opt.input_mode != 0 && opt.input_mode != 1) throw Error(FMMBEM_E_INVALID, "input_mode must be 0 or 1");
  if (opt.charge_terms != 0 && (!rot_supported(opt.charge_terms) || opt.charge_terms > opt.terms))
    throw Error(FMMBEM_E_INVALID, "charge_terms must be 0 or one of 8, 10, 12, 13, 14 and <= terms");
  const bool parts = opt.nranks > 1 && opt.input_mode == 1;
  if (parts && (opt.near_mode || opt.self_term))
    throw Error(FMMBEM_E_INVALID, "near_mode / self_term need the full mesh on every rank (input_mode 0)");
  if (!(eps_in > 0) || !(eps_out > 0) || eps_in == eps_out || !std::isfinite(eps_in) || !std::isfinite(eps_out))
    throw Error(FMMBEM_E_INVALID, "need eps_in, eps_out > 0 and eps_in != eps_out");
  if (mesh->n_triangles < 0 || mesh->n_vertices < 0 || (mesh->n_triangles > 0 && (!mesh->xyz || !mesh->tri)))
    throw Error(FMMBEM_E_INVALID, "bad mesh arrays");
  if (!parts && (mesh->n_triangles < 1 || mesh->n_vertices < 3)) throw Error(FMMBEM_E_INVALID, "empty mesh");
  const int64_t nc = chg ? chg->n : 0;
  if (nc < 0 || (nc > 0 && (!chg->xyz || !chg->q))) throw Error(FMMBEM_E_INVALID, "bad charges");
  if (mesh->n_triangles * (int64_t)opt.quad_points >= (1LL << 31) || mesh->n_vertices >= (1LL << 31))
    throw Error(FMMBEM_E_INVALID, "problem too large for 32-bit point indices");
  for (int64_t i = 0; i < nc; ++i) {
    if (!std::isfinite(chg->q[i]) || !std::isfinite(chg->xyz[3 * i]) || !std::isfinite(chg->xyz[3 * i + 1]) ||
        !std::isfinite(chg->xyz[3 * i + 2]))
      throw Error(FMMBEM_E_INVALID, "non-finite charge " + std::to_string(i));
  }
  c = new fmmbem_ctx();
  c->opt = opt;
  c->device = opt.device;
  DevGuard dg(c->device);
  FMM_CUDA(cudaSetDevice(c->device));
  FMM_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  {
    int lo = 0, hi = 0;  // hi = greatest priority (numerically lowest)
    FMM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    FMM_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi));
  }
  for (auto& e : c->ev) FMM_CUDA(cudaEventCreate(&e));
  FMM_CUDA(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
  FMM_CUDA(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
  FMM_CUDA(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
  c->P = opt.terms;
  if (const char* e = std::getenv("FMMBEM_M2L")) c->m2l_mode = (std::string(e) == "p4") ? 1 : 0;
  if (const char* e = std::getenv("FMMBEM_P2P_CHUNK")) c->p2p_chunk = std::max(8, std::min(256, std::atoi(e)));
  if (const char* e = std::getenv("FMMBEM_P2P_OCC")) c->p2p_occ = std::atoi(e);
  if (const char* e = std::getenv("FMMBEM_P2P_PLAIN")) c->p2p_scaled = std::atoi(e) ? 0 : 1;
  if (const char* e = std::getenv("FMMBEM_P2P_CHUNK_CHG")) c->p2p_chunk_chg = std::max(8, std::min(256, std::atoi(e)));
  c->p2p_chunk = std::min(c->p2p_chunk, 128);  // <= 32 lanes x 4 targets per subset
  c->p2p_chunk_chg = std::min(c->p2p_chunk_chg, 128);
  // near field concurrent with the far field: default on with several ranks (hides the exchange)
  c->overlap = opt.nranks > 1 ? 1 : 0;
  if (const char* e = std::getenv("FMMBEM_OVERLAP")) c->overlap = std::atoi(e);
  c->NC = c->P * (c->P + 1) / 2;
  c->P_chg = opt.charge_terms ? opt.charge_terms : c->P;
  if (const char* e = std::getenv("FMMBEM_CHARGE_TERMS")) {  // A/B knob (same rules as the option)
    const int v = std::atoi(e);
    if (rot_supported(v) && v <= c->P) c->P_chg = v;
  }
  if (c->m2l_mode != 0) c->P_chg = c->P;  // the O(P^4) tables are built for terms only
  c->K = opt.quad_points;
  c->eps_in = eps_in;
  c->eps_out = eps_out;
  c->f = 2.0 * (eps_out - eps_in) / (eps_in + eps_out);  // reading A1
  c->eps_hat = 1.0 - eps_in / eps_out;
  c->nc = nc;
  c->rank = opt.rank;
  c->nranks = opt.nranks;
  cudaStream_t s = c->stream;
  if (c->nranks > 1) comm_init(c, opt.nccl_id);
  const int R = c->nranks, me = c->rank;
  // this rank's input slice: input_mode 0 = [r n / R, (r + 1) n / R) of the full mesh every rank
  // passes; input_mode 1 = the rank's own panels, global ids after those of the lower ranks
  const int64_t nt = mesh->n_triangles, nv = mesh->n_vertices;
  int64_t t0 = 0, m = nt;
  if (R > 1 && !parts) {
    t0 = nt * me / R;
    m = nt * (me + 1) / R - t0;
  }
  int64_t gid0 = t0;
  if (parts) {
    DevBuf<int64_t> mine, all;
    mine.alloc(1);
    all.alloc(R);
    FMM_CUDA(cudaMemcpyAsync(mine.get(), &m, sizeof(m), cudaMemcpyHostToDevice, s));
    comm_allgather_i64(c, mine.get(), all.get(), 1, s);
    std::vector<int64_t> h(R);
    FMM_CUDA(cudaMemcpyAsync(h.data(), all.get(), R * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    gid0 = 0;
    int64_t tot = 0;
    for (int r = 0; r < R; ++r) {
      if (r < me) gid0 += h[r];
      tot += h[r];
    }
    if (tot < 1) throw Error(FMMBEM_E_INVALID, "empty mesh");
  }
  // upload + panel prep (FP64) of the slice
  DevBuf<double> dV, cen, nrm, area, qp, beta, wq, cx, cq;
  DevBuf<int> dT;
  dV.alloc(std::max<int64_t>(3 * nv, 1));
  dT.alloc(std::max<int64_t>(3 * m, 1));
  if (nv) FMM_CUDA(cudaMemcpyAsync(dV.get(), mesh->xyz, 3 * nv * sizeof(double), cudaMemcpyHostToDevice, s));
  if (m) FMM_CUDA(cudaMemcpyAsync(dT.get(), mesh->tri + 3 * t0, 3 * m * sizeof(int), cudaMemcpyHostToDevice, s));
  std::vector<double> hb, hw;
  quad_rule(c->K, hb, hw);
  beta.alloc(hb.size());
  wq.alloc(hw.size());
  FMM_CUDA(cudaMemcpyAsync(beta.get(), hb.data(), hb.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaMemcpyAsync(wq.get(), hw.data(), hw.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  // degeneracy tolerance 1e-14 bbox_diag^2 from the vertex bounding box of all ranks
  double box[6] = {1e300, 1e300, 1e300, 1e300, 1e300, 1e300};
  {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(1024, (nv + 255) / 256));
    DevBuf<double> part;
    part.alloc(blocks * 6);
    k_vbox<<<blocks, 256, 0, s>>>(nv, dV.get(), part.get());
    FMM_CHECK_LAUNCH();
    std::vector<double> h(blocks * 6);
    FMM_CUDA(cudaMemcpyAsync(h.data(), part.get(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    for (int b = 0; b < blocks; ++b)
      for (int k = 0; k < 6; ++k) box[k] = std::min(box[k], h[b * 6 + k]);
    if (parts) {
      DevBuf<double> d;
      d.alloc(6);
      FMM_CUDA(cudaMemcpyAsync(d.get(), box, sizeof(box), cudaMemcpyHostToDevice, s));
      comm_allreduce_f64_op(c, d.get(), 6, -1, s);
      FMM_CUDA(cudaMemcpyAsync(box, d.get(), sizeof(box), cudaMemcpyDeviceToHost, s));
      FMM_CUDA(cudaStreamSynchronize(s));
    }
  }
  double diag2 = 0;
  for (int d = 0; d < 3; ++d) {
    const double ext = -box[3 + d] - box[d];
    if (ext > 0 && ext < 1e300) diag2 += ext * ext;
  }
  cen.alloc(std::max<int64_t>(3 * m, 1));
  nrm.alloc(std::max<int64_t>(3 * m, 1));
  area.alloc(std::max<int64_t>(m, 1));
  if (c->K > 1) qp.alloc(std::max<int64_t>(3 * m * c->K, 1));
  {
    DevBuf<unsigned long long> bad;
    bad.alloc(3);
    const unsigned long long none[3] = {~0ULL, ~0ULL, ~0ULL};
    FMM_CUDA(cudaMemcpyAsync(bad.get(), none, sizeof(none), cudaMemcpyHostToDevice, s));
    if (m)
      k_prep<<<ceil_div(m, 256), 256, 0, s>>>(m, nv, dV.get(), dT.get(), c->K, beta.get(), 1e-14 * diag2, cen.get(),
                                              nrm.get(), area.get(), c->K > 1 ? qp.get() : nullptr, bad.get());
    FMM_CHECK_LAUNCH();
    unsigned long long hbad[3];
    FMM_CUDA(cudaMemcpyAsync(hbad, bad.get(), sizeof(hbad), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    double g[3];  // global triangle id of the first bad triangle of each kind, agreed by every rank
    for (int k = 0; k < 3; ++k) g[k] = hbad[k] == ~0ULL ? 1e300 : (double)(gid0 + (int64_t)hbad[k]);
    if (R > 1) {
      DevBuf<double> d;
      d.alloc(3);
      FMM_CUDA(cudaMemcpyAsync(d.get(), g, sizeof(g), cudaMemcpyHostToDevice, s));
      comm_allreduce_f64_op(c, d.get(), 3, -1, s);
      FMM_CUDA(cudaMemcpyAsync(g, d.get(), sizeof(g), cudaMemcpyDeviceToHost, s));
      FMM_CUDA(cudaStreamSynchronize(s));
    }
    if (g[0] < 1e300) throw Error(FMMBEM_E_DEGENERATE, "triangle index out of range " + std::to_string((long long)g[0]));
    if (g[1] < 1e300) throw Error(FMMBEM_E_INVALID, "non-finite vertex in triangle " + std::to_string((long long)g[1]));
    if (g[2] < 1e300) throw Error(FMMBEM_E_DEGENERATE, "degenerate triangle " + std::to_string((long long)g[2]));
  }
  if (nc) {
    cx.alloc(3 * nc);
    cq.alloc(nc);
    FMM_CUDA(cudaMemcpyAsync(cx.get(), chg->xyz, 3 * nc * sizeof(double), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaMemcpyAsync(cq.get(), chg->q, nc * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  PanelInput pin;
  pin.n = m;
  pin.gid0 = gid0;
  pin.cen = cen.get();
  pin.nrm = nrm.get();
  pin.area = area.get();
  pin.qp = c->K > 1 ? qp.get() : nullptr;
  const auto t_tree = std::chrono::steady_clock::now();
  build_tree(c, pin, wq.get(), cx.get(), cq.get(), s);  // synchronises s
  c->last.tree = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_tree).count();
  init_tables(c);
  c->Mx.alloc((size_t)std::max<int64_t>(c->n_slots, 1) * c->NC);  // rank-local slots (ctx.h)
  c->Lx.alloc((size_t)std::max<int64_t>(c->n_slots, 1) * c->NC);
  c->red.alloc(64);
  c->flag.alloc(4);
  const PointSet& src = (c->K == 1) ? c->pan : c->quad;
  const bool direct = c->opt.direct != 0 || c->tree.L < 2;
  if (R == 1) c->p2p_inter_kp = count_p2p(c, c->pan, src, true, direct);
  if (R > 1 && !direct) build_let(c, s);
  if (c->opt.near_mode == 1) {
    if (R > 1) {  // the analytic near field needs FP64 geometry of every local (owned + halo) panel
      cen.alloc(3 * nt);
      nrm.alloc(3 * nt);
      area.alloc(nt);
      DevBuf<unsigned long long> bad;
      bad.alloc(3);
      dT.alloc(3 * nt);
      FMM_CUDA(cudaMemcpyAsync(dT.get(), mesh->tri, 3 * nt * sizeof(int), cudaMemcpyHostToDevice, s));
      k_prep<<<ceil_div(nt, 256), 256, 0, s>>>(nt, nv, dV.get(), dT.get(), 1, beta.get(), 0.0, cen.get(), nrm.get(),
                                               area.get(), nullptr, bad.get());
      FMM_CHECK_LAUNCH();
    }
    build_near(c, dV.get(), dT.get(), cen.get(), nrm.get(), area.get(), beta.get(), wq.get(), s);
  }
  if (c->opt.self_term == 1) build_self_term(c, mesh, s);
  dV.release();
  dT.release();
  c->m2l_pairs_kp = 0;
  if (!direct) {
    const int* tc = (R > 1) ? c->pan_own_cnt.get() : c->pan.cell_cnt.get();
    if (rot_supported(c->P) && c->m2l_mode == 0) c->m2l_pairs_kp = m2l_work(c, src.cell_cnt.get(), tc, s).pairs;
    else c->m2l_pairs_kp = c->tree.m2l_pairs;
  }
  // everything a matvec allocates or builds lazily is prepared here: no allocation (an implicit
  // device synchronisation) can then fall between the concurrent NCCL exchanges of a matvec
  p2p_items(c, c->pan, c->leaf_lo, c->leaf_hi, c->p2p_chunk);
  c->p2p_src.alloc(std::max<int64_t>(src.n, 1));
  c->p2p_wmax.alloc(1);
  c->p2p_counter.alloc(1);
  FMM_CUDA(cudaStreamSynchronize(s));
  if (std::getenv("FMMBEM_VERBOSE")) report_memory(c);
  *out = c;
  return FMMBEM_OK;
  }
  catch (const fmm::Error& e) {
    g_err = e.what();
    fmmbem_destroy(c);
    return e.code;
  }
  catch (const std::exception& e) {
    g_err = e.what();
    fmmbem_destroy(c);
    return FMMBEM_E_CUDA;
  }
}

void fmmbem_destroy(fmmbem_ctx* c) {
  if (!c) return;
  {
    DevGuard dg(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    try {
      comm_destroy(c);
    } catch (...) {
    }
    if (c->side) cudaStreamSynchronize(c->side);
    for (auto& e : c->ev)
      if (e) cudaEventDestroy(e);
    if (c->cstream) {
      cudaStreamDestroy(c->cstream);
      for (auto& e : c->pev) cudaEventDestroy(e);
    }
    if (c->fork) cudaEventDestroy(c->fork);
    if (c->join) cudaEventDestroy(c->join);
    if (c->done) cudaEventDestroy(c->done);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
  }
}

int64_t fmmbem_num_local_panels(const fmmbem_ctx* c) { return c ? c->n_own() : 0; }

fmmbem_status fmmbem_local_panel_ids(const fmmbem_ctx* c, int64_t* ids) {
  if (!c || !ids) return FMMBEM_E_INVALID;
  std::memcpy(ids, c->pan_ids.data() + c->pan_lo, c->n_own() * sizeof(int64_t));
  return FMMBEM_OK;
}

fmmbem_status fmmbem_get_unique_id(void* id128) {
  API_BEGIN
  if (!id128) throw Error(FMMBEM_E_INVALID, "null id buffer");
  comm_unique_id(id128);
  return FMMBEM_OK;
  API_END
}

fmmbem_status fmmbem_split_costs(const double* costs, int64_t n, int32_t parts, int64_t* bounds) {
  API_BEGIN
  if (!costs || !bounds || n < 0 || parts < 1) throw Error(FMMBEM_E_INVALID, "split_costs: bad arguments");
  split_costs(costs, n, parts, bounds);
  return FMMBEM_OK;
  API_END
}

fmmbem_status fmmbem_matvec(fmmbem_ctx* c, fmmbem_op op, const float* x, float* y, void* stream) {
  API_BEGIN
  if (!c || !x || !y || x == y) throw Error(FMMBEM_E_INVALID, "matvec: null or aliased vectors");
  if (op < FMMBEM_OP_KPRIME || op > FMMBEM_OP_DOUBLE) throw Error(FMMBEM_E_INVALID, "matvec: bad op");
  if (op == FMMBEM_OP_DOUBLE && c->opt.near_mode)
    throw Error(FMMBEM_E_INVALID, "matvec: the double layer has no analytic near-field option");
  DevGuard dg(c->device);
  cudaStream_t st = (cudaStream_t)stream;
  order_after_last(c, st);
  apply_op(c, op, x, y, st, true);
  mark_done(c, st);
  return FMMBEM_OK;
  API_END
}

// Host-buffer matvec with the transfers pipelined against the kernels (K = 1, no near-field
// option): x arrives in NCH (default 8) Morton-contiguous chunks of the rank's leaves on a copy
// stream and P2M of each chunk's leaves starts as soon as it lands; the far field runs next (with
// several ranks: the LET exchange, then M2L / L2L) and L2P writes y first; the near-field halo is
// exchanged once x is complete; P2P then adds the near field chunk by chunk and each chunk of y
// leaves for the host while the next chunk computes.  Same operations as apply_op (P2P and L2P
// swap order; P2P accumulates).
void matvec_host_pipelined(fmmbem_ctx* c, fmmbem_op op, const float* xh, float* yh) {
  constexpr int NCH_MAX = 16;
  static const int NCH = [] {  // transfer chunks (FMMBEM_E2E_CHUNKS, default 8)
    const char* e = std::getenv("FMMBEM_E2E_CHUNKS");
    const int v = e ? std::atoi(e) : 8;
    return v < 1 ? 1 : (v > 16 ? 16 : v);
  }();
  cudaStream_t st = c->stream;
  const Tree& T = c->tree;
  const bool dist = multi(c);
  const int64_t own0 = c->pan_lo, n = c->n_own();
  const int l0 = c->leaf_lo, l1 = c->leaf_hi;
  if (c->h_pan_begin.empty()) {
    c->h_pan_begin.resize(T.n_leaves + 1);
    FMM_CUDA(cudaMemcpy(c->h_pan_begin.data(), c->pan.begin.get(), (T.n_leaves + 1) * sizeof(int),
                        cudaMemcpyDeviceToHost));
  }
  if (!c->cstream) {
    FMM_CUDA(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
    for (auto& e : c->pev) FMM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const auto& hb = c->h_pan_begin;  // local point index of each leaf's first panel
  int lb[NCH_MAX + 1];
  lb[0] = l0;
  for (int k = 1; k < NCH; ++k) {
    const int64_t goal = own0 + n * k / NCH;
    lb[k] = (int)(std::lower_bound(hb.begin() + l0, hb.begin() + l1, (int)goal) - hb.begin());
    lb[k] = std::max(lb[k - 1], std::min(lb[k], l1));
  }
  lb[NCH] = l1;
  // x in local point indexing (owned block at own0; with several ranks the halo segments of xext
  // around it are filled by the halo exchange); y owned-relative
  float* x = dist ? c->xext.get() : c->tmp_x.get();
  float* y = c->tmp_y.get();
  cudaEvent_t* eh = c->pev;            // x chunk k on the device
  cudaEvent_t* ep = c->pev + NCH_MAX;  // y chunk k final
  cudaEvent_t e0 = c->pev[2 * NCH_MAX];  // previous work on st done with x / y
  FMM_CUDA(cudaEventRecord(e0, st));
  FMM_CUDA(cudaStreamWaitEvent(c->cstream, e0, 0));
  for (int k = 0; k < NCH; ++k) {
    const int64_t p0 = hb[lb[k]], p1 = hb[lb[k + 1]];
    if (p1 > p0)
      FMM_CUDA(cudaMemcpyAsync(x + p0, xh + (p0 - own0), (p1 - p0) * sizeof(float), cudaMemcpyHostToDevice,
                               c->cstream));
    FMM_CUDA(cudaEventRecord(eh[k], c->cstream));
  }
  SrcArg s;
  s.set = &c->pan;
  s.x = x;
  const int* tcnt = c->pan.cell_cnt.get();
  if (dist) {
    s.leaf_lo = l0;
    s.leaf_hi = l1;
    s.cnt = c->pan_own_cnt.get();
    s.halo_src = x + own0;  // distributed sources: the P2P weight exponent is taken over all ranks
    tcnt = c->pan_own_cnt.get();
  }
  c->Mx.zero(st);
  for (int k = 0; k < NCH; ++k) {
    FMM_CUDA(cudaStreamWaitEvent(st, eh[k], 0));
    launch_p2m_range(c, s, lb[k], lb[k + 1], st);
  }
  launch_m2m_levels(c, s, st);
  if (dist) exchange_let(c, c->let, st);
  launch_m2l(c, c->pan.cell_cnt.get(), tcnt, st);
  launch_downward(c, tcnt, st);
  Outputs o = op_outputs(c, op, x, y - own0);
  FMM_CUDA(cudaMemsetAsync(y, 0, std::max<int64_t>(n, 1) * sizeof(float), st));
  TgtArg t = own_targets(c, false);
  Outputs far = o;
  far.pot.x = far.dn.x = nullptr;
  far.pot.d = far.dn.d = nullptr;
  launch_l2p(c, t, far, st);
  if (dist) halo_exchange(c, x + own0, st);  // the peers' weights for the near field
  o.pot.acc = o.dn.acc = 1;
  if (c->p2p_scaled && op != FMMBEM_OP_SINGLE) s.scaled = prepare_p2p_sources(c, s, st);  // once for all chunks
  for (int k = 0; k < NCH; ++k) {
    TgtArg tk = t;
    tk.leaf_lo = lb[k];
    tk.leaf_hi = lb[k + 1];
    launch_p2p(c, tk, s, o, /*self=*/true, /*check=*/false, /*direct=*/false, st);
    FMM_CUDA(cudaEventRecord(ep[k], st));
    FMM_CUDA(cudaStreamWaitEvent(c->cstream, ep[k], 0));
    const int64_t p0 = hb[lb[k]], p1 = hb[lb[k + 1]];
    if (p1 > p0)
      FMM_CUDA(cudaMemcpyAsync(yh + (p0 - own0), y + (p0 - own0), (p1 - p0) * sizeof(float),
                               cudaMemcpyDeviceToHost, c->cstream));
  }
  FMM_CUDA(cudaStreamSynchronize(c->cstream));
  FMM_CUDA(cudaStreamSynchronize(st));
}

fmmbem_status fmmbem_matvec_host(fmmbem_ctx* c, fmmbem_op op, const float* xh, float* yh) {
  API_BEGIN
  if (!c || !xh || !yh) throw Error(FMMBEM_E_INVALID, "matvec_host: null vectors");
  if (op < FMMBEM_OP_KPRIME || op > FMMBEM_OP_DOUBLE) throw Error(FMMBEM_E_INVALID, "matvec: bad op");
  if (op == FMMBEM_OP_DOUBLE && c->opt.near_mode)
    throw Error(FMMBEM_E_INVALID, "matvec: the double layer has no analytic near-field option");
  DevGuard dg(c->device);
  cudaStream_t st = c->stream;
  order_after_last(c, st);
  const int64_t n = c->n_own();
  c->tmp_x.alloc(std::max<int64_t>(n, 1));
  c->tmp_y.alloc(std::max<int64_t>(n, 1));
  const bool pipelined = c->K == 1 && c->opt.near_mode == 0 && c->opt.direct == 0 && c->tree.L >= 2 &&
                         op != FMMBEM_OP_DOUBLE && (c->nranks == 1 || c->let.ready) &&
                         std::getenv("FMMBEM_E2E_PLAIN") == nullptr;
  if (pipelined) {
    matvec_host_pipelined(c, op, xh, yh);
    mark_done(c, st);
    return FMMBEM_OK;
  }
  FMM_CUDA(cudaMemcpyAsync(c->tmp_x.get(), xh, n * sizeof(float), cudaMemcpyHostToDevice, st));
  apply_op(c, op, c->tmp_x.get(), c->tmp_y.get(), st, true);
  FMM_CUDA(cudaMemcpyAsync(yh, c->tmp_y.get(), n * sizeof(float), cudaMemcpyDeviceToHost, st));
  mark_done(c, st);
  FMM_CUDA(cudaStreamSynchronize(st));
  return FMMBEM_OK;
  API_END
}

fmmbem_status fmmbem_charge_fields(fmmbem_ctx* c, float* En, float* psi) {
  API_BEGIN
  if (!c) throw Error(FMMBEM_E_INVALID, "null ctx");
  DevGuard dg(c->device);
  order_after_last(c, c->stream);
  ensure_fields(c, c->stream);
  const size_t nb = c->n_own() * sizeof(float);
  if (En) FMM_CUDA(cudaMemcpyAsync(En, c->En.get(), nb, cudaMemcpyDeviceToDevice, c->stream));
  if (psi) FMM_CUDA(cudaMemcpyAsync(psi, c->psi.get(), nb, cudaMemcpyDeviceToDevice, c->stream));
  mark_done(c, c->stream);
  FMM_CUDA(cudaStreamSynchronize(c->stream));
  return FMMBEM_OK;
  API_END
}

fmmbem_status fmmbem_reset_fields(fmmbem_ctx* c) {
  if (!c) return FMMBEM_E_INVALID;
  c->have_fields = false;
  return FMMBEM_OK;
}

fmmbem_status fmmbem_bibee_energy(fmmbem_ctx* c, fmmbem_bibee v, float* sig, fmmbem_energy* out) {
  API_BEGIN
  if (!c || !out) throw Error(FMMBEM_E_INVALID, "null argument");
  if (v < FMMBEM_BIBEE_CFA || v > FMMBEM_BIBEE_LB) throw Error(FMMBEM_E_INVALID, "bad BIBEE variant");
  DevGuard dg(c->device);
  cudaStream_t st = c->stream;
  order_after_last(c, st);
  FMM_CUDA(cudaEventRecord(c->ev[E_BIB0], st));
  ensure_fields(c, st);
  const double s = (v == FMMBEM_BIBEE_CFA) ? -0.5 : (v == FMMBEM_BIBEE_P ? 0.0 : 0.5);
  const double d = 1.0 - c->f * s;
  if (d == 0.0) throw Error(FMMBEM_E_INVALID, "1 - f s == 0 (SPEC S:383)");
  const int64_t n = c->n_own();
  float* sh = sig;
  if (!sh) {  // ctx scratch, allocated once (an allocation here would stall the timed interval)
    c->tmp_y.alloc(std::max<int64_t>(std::max<int64_t>(n, 1), (int64_t)c->tmp_y.n));
    sh = c->tmp_y.get();
  }
  // sigma_hat = f E / (1 - f s)   (Eq. 7 with K' -> s I, reading A3)
  if (n > 0) k_scale<<<ceil_div(n, 256), 256, 0, st>>>(sh, c->En.get(), n, (float)(c->f / d));
  FMM_CHECK_LAUNCH();
  const double e = 0.5 * dot_weighted(c, n, sh, c->psi.get(), c->pan.pos.get() + c->pan_lo, st);  // A20
  FMM_CUDA(cudaEventRecord(c->ev[E_BIB1], st));
  mark_done(c, st);
  {
    float ms = 0.f;
    FMM_CUDA(cudaEventSynchronize(c->ev[E_BIB1]));
    FMM_CUDA(cudaEventElapsedTime(&ms, c->ev[E_BIB0], c->ev[E_BIB1]));
    c->last.bibee = ms;
  }
  out->dG_internal = e;
  out->dG_kcal_mol = e * KCAL;
  out->iterations = 0;
  out->rel_residual = 0.0;
  return FMMBEM_OK;
  API_END
}

fmmbem_status fmmbem_solve(fmmbem_ctx* c, const fmmbem_solve_options* so, float* sigma, double* hist,
                           fmmbem_energy* out) {
  API_BEGIN
  if (!c || !out) throw Error(FMMBEM_E_INVALID, "null argument");
  fmmbem_solve_options o{1e-6, 30, 200, nullptr};
  if (so) o = *so;
  if (!(o.tol > 0 && o.tol < 1) || o.restart < 1 || o.max_iters < 1)
    throw Error(FMMBEM_E_INVALID, "bad solve options");
  DevGuard dg(c->device);
  cudaStream_t st = c->stream;
  order_after_last(c, st);
  ensure_fields(c, st);
  if (c->red.n < (size_t)o.restart + 2) c->red.alloc(o.restart + 2 + 64);
  DevBuf<float> b, xs;
  const int64_t n = c->n_own();
  b.alloc(std::max<int64_t>(n, 1));
  float* x = sigma;
  if (!x) {
    xs.alloc(std::max<int64_t>(n, 1));
    x = xs.get();
  }
  if (n > 0) k_scale<<<ceil_div(n, 256), 256, 0, st>>>(b.get(), c->En.get(), n, (float)c->f);  // b = f E
  FMM_CHECK_LAUNCH();
  if (hist)
    for (int i = 0; i <= o.max_iters; ++i) hist[i] = -1.0;
  int its = 0;
  double rr = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  fmmbem_status stt = gmres_solve(c, b.get(), x, o.tol, o.restart, o.max_iters, o.x0_dev, hist, &its, &rr, st);
  cudaEventRecord(e1, st);
  const double e = 0.5 * dot_weighted(c, n, x, c->psi.get(), c->pan.pos.get() + c->pan_lo, st);
  mark_done(c, st);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  c->last.gmres = ms;
  out->dG_internal = e;
  out->dG_kcal_mol = e * KCAL;
  out->iterations = its;
  out->rel_residual = rr;
  return stt;
  API_END
}

fmmbem_status fmmbem_reaction_potential(fmmbem_ctx* c, const float* sigma, double* phi) {
  API_BEGIN
  if (!c || !sigma || !phi) throw Error(FMMBEM_E_INVALID, "null argument");
  if (c->nc == 0) return FMMBEM_OK;
  DevGuard dg(c->device);
  cudaStream_t st = c->stream;
  order_after_last(c, st);
  DevBuf<float> y;
  DevBuf<double> yd;
  y.alloc(c->nc);
  yd.alloc(c->nc);
  y.zero(st);
  yd.zero(st);
  // targets: the charges of this rank's leaves (every charge with one rank); sources: the panels
  // (owned + halo weights, the LET multipoles of the other ranks' panels)
  TgtArg t;
  t.set = &c->chg;
  bool dist = false;
  SrcArg s = kp_src(c, sigma, st, &dist);
  int64_t c0 = 0, c1 = c->nc;
  if (multi(c)) {
    t.leaf_lo = c->leaf_lo;
    t.leaf_hi = c->leaf_hi;
    t.cnt = c->chg_own_cnt.get();
    int h[2];
    FMM_CUDA(cudaMemcpyAsync(&h[0], c->chg.begin.get() + c->leaf_lo, sizeof(int), cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaMemcpyAsync(&h[1], c->chg.begin.get() + c->leaf_hi, sizeof(int), cudaMemcpyDeviceToHost, st));
    FMM_CUDA(cudaStreamSynchronize(st));
    c0 = h[0];
    c1 = h[1];
  }
  Outputs o;
  o.pot.y = y.get();
  o.pot.b = (float)(1.0 / FOUR_PI);
  fmm_eval(c, t, s, o, false, false, st, false, dist);
  if (c1 > c0)
    k_unpermute<<<ceil_div(c1 - c0, 256), 256, 0, st>>>(c1 - c0, c->chg_ids.get() + c0, y.get() + c0, yd.get());
  FMM_CHECK_LAUNCH();
  comm_allreduce_f64(c, yd.get(), c->nc, st);  // every charge written by exactly one rank
  FMM_CUDA(cudaMemcpyAsync(phi, yd.get(), c->nc * sizeof(double), cudaMemcpyDeviceToHost, st));
  mark_done(c, st);
  FMM_CUDA(cudaStreamSynchronize(st));
  return FMMBEM_OK;
  API_END
}

fmmbem_status fmmbem_last_timing(const fmmbem_ctx* c, fmmbem_timing* out) {
  API_BEGIN
  if (!c || !out) throw Error(FMMBEM_E_INVALID, "null argument");
  DevGuard dg(c->device);
  fill_timing(const_cast<fmmbem_ctx*>(c), c->opt.direct != 0 || c->tree.L < 2);
  *out = c->last;
  return FMMBEM_OK;
  API_END
}

fmmbem_status fmmbem_tree_info_get(const fmmbem_ctx* c, fmmbem_tree_info* o) {
  if (!c || !o) return FMMBEM_E_INVALID;
  o->levels = c->tree.L;
  o->n_leaves = c->tree.n_leaves;
  o->n_cells = c->tree.n_cells;
  o->n_panels = c->np;
  o->n_charges = c->nc;
  o->nbr_pairs = c->tree.nbr_pairs;
  o->m2l_pairs = c->tree.m2l_pairs;
  o->root_width = c->tree.W;
  for (int d = 0; d < 3; ++d) o->root_origin[d] = c->tree.x0[d];
  o->expansion_slots = c->n_slots;
  o->let_send_peers = o->let_recv_peers = 0;
  for (int p = 0; p < (int)c->let.nsend.size(); ++p) {
    o->let_send_peers += c->let.nsend[p] > 0;
    o->let_recv_peers += c->let.nrecv[p] > 0;
  }
  o->let_cells_sent = c->let.cells_sent;
  o->let_cells_recv = c->let.cells_recv;
  o->let_shared_cells = c->let.nshared;
  o->halo_panels_sent = c->halo.sent;
  o->halo_panels_recv = c->halo.recv;
  return FMMBEM_OK;
}

}  // extern "C"
