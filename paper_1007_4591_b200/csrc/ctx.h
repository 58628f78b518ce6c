// ctx.h -- internal state of one fmmbem_ctx (CUDA path).
#pragma once
#include <array>
#include <memory>
#include <cuda_runtime.h>

#include "common.cuh"
#include "plan.h"

namespace fmm {

// Points of one kind in leaf (Morton) order.  pos.xyz = coordinates relative to the
// centre of the point's leaf (FP32), pos.w = per-point weight factor
// (panel area * quadrature weight for sources; charge q for charges).
struct PointSet {
  int64_t n = 0;
  DevBuf<float4> pos;
  DevBuf<float4> nrm;   // unit normals (panel targets only)
  DevBuf<int> leaf;     // leaf index of each point
  DevBuf<int> begin;    // [n_leaves + 1] CSR of points per leaf
  DevBuf<int> cell_cnt; // [n_cells] number of points in each cell's subtree
  int div = 1;          // the x-vector index of point j is j / div (K for quadrature sources)
};

struct Tree {
  int L = 0;                  // leaf level (root = 0)
  double x0[3] = {0, 0, 0};   // root cube min corner
  double W = 1.0;             // root cube width (8-bit mantissa -> exact integer*h in FP32)
  int64_t n_leaves = 0, n_cells = 0;
  std::vector<int64_t> lvl_off;  // [L + 2] first global cell index per level (level-major)
  DevBuf<uint64_t> key;          // [n_cells] Morton key at the cell's level
  DevBuf<int> parent;            // [n_cells] global parent index (-1 at the root)
  DevBuf<int> child_begin, child_end;  // [n_cells] global child range (level + 1)
  DevBuf<int4> leaf_ijk;         // [n_leaves] integer leaf coordinates
  DevBuf<int> nbr_off, nbr_idx;  // leaf-level neighbour CSR (leaf indices, incl. self)
  DevBuf<long long> m2l_off;     // [n_cells+1] interaction-list CSR offsets (64-bit: > 2^31 entries at 1e9 panels)
  DevBuf<int> m2l_idx;           // global source cell index of each interaction-list entry
  int64_t nbr_pairs = 0, m2l_pairs = 0;  // list entries of the whole tree (the device lists of a rank
                                          // of several hold its owned leaves' / windows' entries only)
  double width(int l) const { return W / (double)(1LL << l); }
};

// compacted M2L work for one (source set, target set) pair: rows = target cells
struct M2LWork {
  const int* src = nullptr;  // source / target subtree-count arrays that define the work
  const int* tgt = nullptr;
  int64_t pairs = 0, rows = 0;
  DevBuf<int> idx;   // [pairs] source cells
  DevBuf<int> cell;  // [rows] target cells
  DevBuf<int> off;   // [rows + 1]
};

// P2P work items (leaf, first target, count) of one target set
struct P2PItems {
  const PointSet* tgt = nullptr;
  int leaf_lo = 0, leaf_hi = 0, chunk = 0;
  int64_t n = 0;
  DevBuf<int4> items;
};

// analytic near-field correction (near_mode = 1): CSR over this rank's target rows
struct NearCSR {
  int64_t nnz = 0;
  DevBuf<long long> off;  // 64-bit: ~28 pairs per panel exceed 2^31 entries at C5
  DevBuf<int> col;
  DevBuf<float> vkp, vsl, diag;
};

// local-essential-tree multipole exchange (let.cu)
struct LetPlan {
  bool ready = false;
  std::vector<DevBuf<int>> send, recv;  // per peer: cells (global index), increasing
  std::vector<int> nsend, nrecv;
  DevBuf<int> shared;                   // cells straddling a rank boundary (partial on several ranks)
  int nshared = 0;
  DevBuf<float2> sbuf, rbuf, shbuf;
  int64_t cells_sent = 0, cells_recv = 0;
};

// panels of this rank's input slice (device, FP64, in the caller's order of the slice)
struct PanelInput {
  int64_t n = 0;     // panels in the slice
  int64_t gid0 = 0;  // global id (caller triangle index) of the slice's first panel
  const double* cen = nullptr;
  const double* nrm = nullptr;
  const double* area = nullptr;
  const double* qp = nullptr;  // K > 1: quadrature points [n][K][3]
};

// near-field halo (multi-GPU, SURVEY 8(e) "halo source weights"): the owned panels every peer's
// P2P needs (their leaves neighbour a leaf of the peer) and the peers' panels this rank's P2P needs.
// Local point arrays are [halo of lower ranks | owned | halo of higher ranks], in leaf order.
struct HaloPlan {
  std::vector<int64_t> scnt, soff;  // per peer: panels sent, first entry in sidx
  std::vector<int64_t> rcnt, roff;  // per peer: panels received, first local index of the segment
  DevBuf<int> sidx;                 // owned-relative index of every panel sent (peers concatenated)
  DevBuf<float> sbuf;               // packed x of one matvec
  int64_t sent = 0, recv = 0;
};

}  // namespace fmm

struct fmmbem_ctx {
  fmmbem_options opt{};
  int P = 10, K = 1, NC = 55;  // terms, quadrature points, complex coefficients per expansion
  int P_chg = 10;              // order of the charge-FMM (options.charge_terms; ensure_fields swaps it in)
  double eps_in = 4, eps_out = 80, f = 0, eps_hat = 0;
  int64_t np = 0, nc = 0;  // panels of ALL ranks, charges (replicated)
  int device = 0;
  cudaStream_t stream = nullptr;  // internal stream for setup / host-buffer calls

  fmm::Tree tree;
  fmm::PointSet pan;   // panels: targets (centroid + normal); sources when K == 1
  fmm::PointSet quad;  // quadrature points (K > 1), panel-major within each leaf
  fmm::PointSet chg;   // charges
  std::vector<int64_t> pan_ids;     // local -> caller triangle index
  fmm::DevBuf<int> chg_ids;         // local charge -> caller charge index

  // expansions [n_slots * NC]: slot_base[l] + (cell - win_lo[l]) for the cells of level l in this
  // rank's window, then the LET cells received / shared from outside it (plan.h slot_layout); one
  // GPU: slot = cell.  lvl_ptr(X, l) addresses a level's window by GLOBAL cell index.
  fmm::DevBuf<float2> Mx, Lx;
  std::vector<int64_t> win_lo, win_hi, slot_base;  // [L + 1]
  int64_t n_slots = 0;
  fmm::DevBuf<int> cmap;            // [n_cells] cell -> slot or -1 (nranks > 1; empty on one GPU)
  fmm::DevBuf<uint64_t> skey;       // [n_slots] Morton key of each slot (nranks > 1)
  const int* slot_map() const { return cmap.n ? cmap.get() : nullptr; }
  const uint64_t* slot_keys() const { return skey.n ? skey.get() : tree.key.get(); }
  float2* lvl_ptr(float2* X, int l) const { return X + (slot_base[l] - win_lo[l]) * NC; }
  fmm::DevBuf<float2> Itab;         // M2L irregular-harmonic table [343 * NI]
  int NI = 0;
  fmm::DevBuf<float> tmp_x, tmp_y;  // host-buffer matvec staging / scratch
  std::vector<int> h_pan_begin;      // host copy of pan.begin (pipelined host-buffer matvec)
  cudaStream_t cstream = nullptr;    // copy stream of the pipelined host-buffer matvec
  cudaEvent_t pev[33] = {};          // its chunk events (2 x 16 + 1)
  fmm::DevBuf<float> En, psi;       // charge fields (cached)
  bool have_fields = false;
  bool fields_checked = false;       // the charge / panel-point coincidence check passed once
  fmm::DevBuf<int> flag;            // device error flags
  fmm::DevBuf<double> red;          // reduction scratch

  // GMRES workspace
  fmm::DevBuf<float> V;     // [(m+1) * np]
  fmm::DevBuf<float> w;     // [np]
  fmm::DevBuf<double> hd;   // [m+2]
  fmm::DevBuf<double> part; // partial sums [blocks * (m+2)]

  std::vector<std::unique_ptr<fmm::M2LWork>> m2l_cache;
  std::vector<std::unique_ptr<fmm::P2PItems>> p2p_cache;
  int m2l_mode = 0;  // 0 = rotation O(P^3) when available, 1 = plain O(P^4)
  int p2p_chunk = 64;   // P2P targets per work item (FMMBEM_P2P_CHUNK)
  int p2p_chunk_chg = 128; // ... of the charge-source near field (FMMBEM_P2P_CHUNK_CHG; 128 measured 2.6 vs 3.8 ms at C5)
  fmm::DevBuf<float4> p2p_src;  // scaled-form P2P sources of the current matvec (a y, a)
  fmm::DevBuf<int> p2p_counter;  // work-item counter of the persistent P2P launch
  fmm::DevBuf<unsigned> p2p_wmax;  // bits of max |w| the table was normalised by (power of two, P2P epilogue)
  int p2p_occ = 1;      // scaled K' P2P at 32 resident warps per SM (<= 64 registers; FMMBEM_P2P_OCC=0 -> 72)
  int p2p_scaled = 1;   // scaled-coordinate K' P2P (FMMBEM_P2P_PLAIN=1 -> plain form)
  int64_t p2p_inter_kp = 0;   // exact P2P interaction count of the K' / A matvec
  int64_t p2p_inter_chg = -1; // exact P2P interaction count of the charge-FMM (owned targets; -1 = not counted)
  int64_t m2l_pairs_kp = 0;
  // multi-GPU partition: this rank owns leaves [leaf_lo, leaf_hi); its panels are the
  // local points [pan_lo, pan_hi) of pan (the rest of pan is the near-field halo)
  void* comm = nullptr;   // ncclComm_t (nranks > 1)
  void* comm2 = nullptr;  // second communicator (ncclCommSplit) for the halo exchange, so it can run
                          // on the caller's stream concurrently with the multipole exchange
  int rank = 0, nranks = 1;
  int leaf_lo = 0, leaf_hi = 0;
  int64_t pan_lo = 0, pan_hi = 0;
  fmm::DevBuf<int> pan_own_cnt, quad_own_cnt, chg_own_cnt;  // subtree counts of owned points
  fmm::DevBuf<float> selfd;                    // [np] curvature self-term K'_ii in local order (self_term = 1)
  fmm::NearCSR near;                           // near_mode = 1 corrections
  fmm::LetPlan let;                            // multipole LET exchange plan (nranks > 1), panel sources
  fmm::LetPlan let_chg;                        // ... charge sources (the charge-FMM)
  std::vector<int64_t> leaf_bounds;            // [nranks + 1] leaf partition
  fmm::DevBuf<int> gbeg;                       // [n_leaves + 1] GLOBAL panel CSR over leaves (all ranks)
  fmm::HaloPlan halo;                          // near-field halo exchange (nranks > 1)
  fmm::ExchangePlan xplan;                     // host plan: partition, halo leaves, LET cells (plan.cu)
  fmm::DevBuf<float> xext;                     // [pan.n] source weights incl. the halo (nranks > 1)
  int64_t n_own() const { return pan_hi - pan_lo; }
  fmmbem_timing last{};
  // phase events (E_* in api.cu); recorded on the stream that runs the phase
  cudaEvent_t ev[24] = {};
  cudaEvent_t fork = nullptr, join = nullptr;  // untimed fork/join of the far-field stream
  cudaEvent_t done = nullptr;  // end of the last stream-ordered call (every entry point waits on it first)
  cudaStream_t side = nullptr;                 // far-field chain runs here when overlap is on
  int overlap = 0;                             // 1: P2P concurrent with the upward/M2L/exchange chain
  bool timed_xg = false;
  bool timed_comm = false, timed_near = false;
  bool timed_fields = false;  // the last timed evaluation was the charge-FMM
};
