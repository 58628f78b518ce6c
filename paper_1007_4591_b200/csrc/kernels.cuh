// kernels.cuh -- launch interfaces shared by the .cu files of libfmmbem.
#pragma once
#include <vector>

#include "ctx.h"

namespace fmm {

// y[i] = ax * x[i] + b * raw[i]   (x may be null)  -- or, for accumulate = true, y[i] += b * raw[i]
struct OutArg {
  float* y = nullptr;
  const float* x = nullptr;
  float ax = 0.f;
  float b = 1.f;
  const float* d = nullptr;  // optional diagonal: y_i += b d_i x_i (curvature self-term, option self_term)
  int acc = 0;               // P2P: add to y instead of overwriting it (far field written first)
};

// A source set for one apply: weight of point j = (x ? x[j / div] : 1) * pos[j].w
// A leaf range [leaf_lo, leaf_hi) (hi < 0: all leaves) restricts the work to this rank's part
// (multi-GPU); cnt = per-cell subtree point counts used to skip empty cells
// (nullptr: the set's full counts).
struct SrcArg {
  const PointSet* set = nullptr;
  const float* x = nullptr;
  const float* halo_src = nullptr;  // nranks > 1: owned weights whose halo exchange fmm_eval runs before P2P
  bool dipole = false;  // double layer: sources are dipoles of moment w n (pan.nrm of the source's panel)
  const float4* scaled = nullptr;  // prepared scaled-form P2P sources (prepare_p2p_sources), else built in launch_p2p
  int leaf_lo = 0, leaf_hi = -1;
  const int* cnt = nullptr;
};

// targets: positions (+ normals for normal-derivative outputs)
struct TgtArg {
  const PointSet* set = nullptr;
  int leaf_lo = 0, leaf_hi = -1;
  const int* cnt = nullptr;
};

struct Outputs {
  OutArg pot;  // potential  phi = sum w / r                (raw, before b)
  OutArg dn;   // normal derivative n . grad phi             (raw, before b)
};

void build_tree(fmmbem_ctx* c, const PanelInput& in, const double* wq, const double* cxyz, const double* cq,
                cudaStream_t s);
// per-matvec near-field halo (nranks > 1): owned x into c->xext, then the peers' halo weights
void halo_copy_owned(fmmbem_ctx* c, const float* x_owned, cudaStream_t st);
void halo_exchange(fmmbem_ctx* c, const float* x_owned, cudaStream_t st);

// near field; writes y = ax x + b raw (overwrites)
// per-matvec scaled-form source table (a y, a) of the K' / A near field into c->p2p_src
const float4* prepare_p2p_sources(fmmbem_ctx* c, const SrcArg& s, cudaStream_t st);
void launch_p2p(fmmbem_ctx* c, const TgtArg& t, const SrcArg& s, const Outputs& o, bool self, bool check,
                bool direct, cudaStream_t st);
const P2PItems& p2p_items(fmmbem_ctx* c, const PointSet& t, int leaf_lo, int leaf_hi, int chunk);

// analytic near field (near.cu)
void build_near(fmmbem_ctx* c, const double* V, const int* T, const double* cen, const double* nrm,
                const double* area, const double* beta, const double* wq, cudaStream_t st);
void apply_near(fmmbem_ctx* c, bool single, const float* x_full, float* y_global, float b, cudaStream_t st);

// multi-GPU (comm.cu); all no-ops when nranks == 1
void comm_unique_id(void* id128);
void comm_init(fmmbem_ctx* c, const void* id128);
void comm_destroy(fmmbem_ctx* c);
void comm_allreduce_f32(fmmbem_ctx* c, float* buf, size_t n, cudaStream_t s);
void comm_allreduce_f64(fmmbem_ctx* c, double* buf, size_t n, cudaStream_t s);
void comm_allgatherv_f32(fmmbem_ctx* c, const float* mine, float* full, const std::vector<int64_t>& offs,
                         cudaStream_t s, bool second = false);
void split_costs(const double* cost, int64_t n, int parts, int64_t* bounds);
void comm_allreduce_f64_op(fmmbem_ctx* c, double* buf, size_t n, int op /* -1 min, 0 sum, +1 max */, cudaStream_t s);
void comm_allreduce_u32_max(fmmbem_ctx* c, unsigned* buf, size_t n, cudaStream_t s, bool second = false);
void comm_allgather_i64(fmmbem_ctx* c, const int64_t* mine, int64_t* all, size_t n, cudaStream_t s);
void comm_allgatherv_bytes(fmmbem_ctx* c, const void* mine, void* full, const std::vector<size_t>& offs,
                           cudaStream_t s);
void comm_alltoallv_bytes(fmmbem_ctx* c, const std::vector<const void*>& sbuf, const std::vector<size_t>& sbytes,
                          const std::vector<void*>& rbuf, const std::vector<size_t>& rbytes, cudaStream_t s,
                          bool second = false);
void comm_sendrecv_f32(fmmbem_ctx* c, const std::vector<float*>& sbuf, const std::vector<size_t>& scnt,
                       const std::vector<float*>& rbuf, const std::vector<size_t>& rcnt, cudaStream_t s);
void build_let(fmmbem_ctx* c, cudaStream_t s);
void exchange_let(fmmbem_ctx* c, const LetPlan& X, cudaStream_t s);
// exact interaction count of launch_p2p(t, s) (list mode) -- setup-time helper
int64_t count_p2p(fmmbem_ctx* c, const PointSet& t, const PointSet& s, bool self, bool direct, int leaf_lo = 0,
                  int leaf_hi = -1);

// far field (expansions in c->Mx / c->Lx); l2p accumulates y += b far
void launch_upward(fmmbem_ctx* c, const SrcArg& s, cudaStream_t st);
// the two halves of launch_upward: P2M over leaves [lo, hi) (Mx must be zeroed first), then M2M
void launch_p2m_range(fmmbem_ctx* c, const SrcArg& s, int lo, int hi, cudaStream_t st);
void check_leaf_window(const fmmbem_ctx* c, int lo, int hi);  // throws unless [lo, hi) has expansion slots
void launch_m2m_levels(fmmbem_ctx* c, const SrcArg& s, cudaStream_t st);
void launch_m2l(fmmbem_ctx* c, const int* src_cnt, const int* tgt_cnt, cudaStream_t st);
void launch_downward(fmmbem_ctx* c, const int* tgt_cnt, cudaStream_t st);
void launch_l2p(fmmbem_ctx* c, const TgtArg& t, const Outputs& o, cudaStream_t st);
void init_tables(fmmbem_ctx* c);

// double-layer operator (dipole.cu): P2M of dipole sources over leaves [lo, hi), near field y = b sum
void launch_p2m_dipole(fmmbem_ctx* c, const SrcArg& s, int lo, int hi, cudaStream_t st);
void launch_p2p_dipole(fmmbem_ctx* c, const TgtArg& t, const SrcArg& s, float* y, float b, bool direct,
                       cudaStream_t st);

// order-specialised P2M / L2P (expansions.cu)
bool exp_specialised(int P);
void launch_p2m_t(int P, int grid, const float4* pos, const float* x, int div, const int* beg, float inv_w,
                  int leaf_off, int leaf0, float2* M, cudaStream_t st);
void launch_l2p_t(int P, int grid, const float4* pos, const float4* nrm, const int* beg, float inv_w, int leaf_off,
                  int leaf0, const float2* Lx, const OutArg& pot, const OutArg& dn, cudaStream_t st);

// rotation-accelerated M2L (m2l_rot.cu)
bool rot_supported(int P);
void init_rot_tables();
const M2LWork& m2l_work(fmmbem_ctx* c, const int* src_cnt, const int* tgt_cnt, cudaStream_t st);
void launch_m2l_rot(fmmbem_ctx* c, const M2LWork& w, cudaStream_t st);
bool m2m_rot_supported(int P);
void launch_m2m_rot(fmmbem_ctx* c, int l, const int* scnt, float2* T, cudaStream_t st);
void launch_l2l_rot(fmmbem_ctx* c, int l, const int* tcnt, cudaStream_t st);
void scan_ints(const int* in, int* out, int n, cudaStream_t s);  // exclusive
void scan_i64(const long long* in, long long* out, int n, cudaStream_t s);  // exclusive

// Krylov / reductions
double dot_weighted(fmmbem_ctx* c, int64_t n, const float* a, const float* b, const float4* w_area,
                    cudaStream_t s);
fmmbem_status gmres_solve(fmmbem_ctx* c, const float* b, float* x, double tol, int restart, int max_iters,
                          const float* x0, double* hist, int* iters, double* relres, cudaStream_t s);

// one full FMM (or direct) evaluation of targets t from sources s
void fmm_eval(fmmbem_ctx* c, const TgtArg& t, const SrcArg& s, const Outputs& o, bool self, bool check,
              cudaStream_t st, bool timing, bool distributed);

}  // namespace fmm
