// plan.cu -- the multi-GPU exchange plan, host code.
//
// Given the replicated leaf skeleton (sorted leaf keys at level L with their panel / charge counts)
// every rank derives the SAME plan, without any handshake:
//   * the cost-weighted contiguous leaf partition ("equally distribute the Morton-indexed
//     boxes", weighted by P2P + M2L work instead of counted);
//   * the near-field halo: rank r sends peer p its leaves that neighbour a leaf of p (P2P of p
//     needs their panels) and receives p's leaves that neighbour one of its own;
//   * the local essential tree ("the data that needs to be communicated consists of ME
//     coefficients of the cells in the interaction list, at every level"): a cell of level >= 2 is
//     PURE (all its leaves on one rank, which computes its whole multipole) or SHARED (straddles a
//     boundary: partial multipoles on several ranks, summed by one all-reduce); rank r sends p the
//     pure cells it owns that are in the interaction list of a cell holding targets of p.
// fmmbem_create copies its device skeleton to the host and calls plan_exchange; fmmbem_plan_create
// (ABI, host only) builds the skeleton lists here first, so tests can check the plan on a CPU.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <thread>
#include <string>
#include <vector>

#include "plan.h"

namespace fmm {

namespace {

int lower_bound_key(const HostVec<uint64_t>& a, int64_t lo, int64_t hi, uint64_t v) {
  return (int)(std::lower_bound(a.begin() + lo, a.begin() + hi, v) - a.begin());
}

}  // namespace

// Host skeleton from sorted unique leaf keys (level L): the same definitions as tree.cu's kernels
// (P:566): neighbours = same-level cells with max |d ijk| <= 1 (incl. self); interaction list =
// children of the parent's neighbours that are not neighbours.
void host_tree(const uint64_t* leaf_keys, int64_t nl, int L, HostTree& T) {
  T.L = L;
  std::vector<std::vector<uint64_t>> lvl(L + 1);
  lvl[L].assign(leaf_keys, leaf_keys + nl);
  for (int l = L - 1; l >= 0; --l) {
    for (uint64_t k : lvl[l + 1])
      if (lvl[l].empty() || lvl[l].back() != (k >> 3)) lvl[l].push_back(k >> 3);
  }
  T.lvl_off.assign(L + 2, 0);
  for (int l = 0; l <= L; ++l) T.lvl_off[l + 1] = T.lvl_off[l] + (int64_t)lvl[l].size();
  T.key.clear();
  for (int l = 0; l <= L; ++l) T.key.insert(T.key.end(), lvl[l].begin(), lvl[l].end());
  const int64_t nc = T.lvl_off[L + 1];
  T.child_b.assign(nc, 0);
  T.child_e.assign(nc, 0);
  for (int l = 0; l < L; ++l)
    for (int64_t i = T.lvl_off[l]; i < T.lvl_off[l + 1]; ++i) {
      T.child_b[i] = lower_bound_key(T.key, T.lvl_off[l + 1], T.lvl_off[l + 2], T.key[i] << 3);
      T.child_e[i] = lower_bound_key(T.key, T.lvl_off[l + 1], T.lvl_off[l + 2], (T.key[i] + 1) << 3);
    }
  auto find = [&](int l, int x, int y, int z) -> int {
    const int lim = 1 << l;
    if (x < 0 || y < 0 || z < 0 || x >= lim || y >= lim || z >= lim) return -1;
    const uint64_t k = morton(x, y, z);
    const int i = lower_bound_key(T.key, T.lvl_off[l], T.lvl_off[l + 1], k);
    return (i < T.lvl_off[l + 1] && T.key[i] == k) ? i : -1;
  };
  // neighbour lists of the leaves (leaf indices)
  T.nbr_off.assign(nl + 1, 0);
  T.nbr_idx.clear();
  for (int64_t k = 0; k < nl; ++k) {
    int x, y, z;
    demorton(T.key[T.lvl_off[L] + k], x, y, z);
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int j = find(L, x + dx, y + dy, z + dz);
          if (j >= 0) T.nbr_idx.push_back(j - (int)T.lvl_off[L]);
        }
    T.nbr_off[k + 1] = (int)T.nbr_idx.size();
  }
  // interaction lists of every cell of levels >= 2 (global cell indices)
  T.m2l_off.assign(nc + 1, 0);
  T.m2l_idx.clear();
  for (int64_t c = 0; c < nc; ++c) {
    int l = 0;
    while (c >= T.lvl_off[l + 1]) ++l;
    if (l >= 2) {
      int x, y, z;
      demorton(T.key[c], x, y, z);
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int p = find(l - 1, (x >> 1) + dx, (y >> 1) + dy, (z >> 1) + dz);
            if (p < 0) continue;
            for (int ch = T.child_b[p]; ch < T.child_e[p]; ++ch) {
              int cx, cy, cz;
              demorton(T.key[ch], cx, cy, cz);
              if (std::abs(cx - x) <= 1 && std::abs(cy - y) <= 1 && std::abs(cz - z) <= 1) continue;
              T.m2l_idx.push_back(ch);
            }
          }
    }
    T.m2l_off[c + 1] = (int64_t)T.m2l_idx.size();
  }
}

// [0, n) split over nth host threads: f(lo, hi, thread)
template <class F>
void parallel_for(int64_t n, int nth, F f) {
  nth = (int)std::max<int64_t>(1, std::min<int64_t>(nth, n / 4096));
  if (nth <= 1) {
    f((int64_t)0, n, 0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nth; ++t) th.emplace_back(f, n * t / nth, n * (t + 1) / nth, t);
  for (auto& t : th) t.join();
}

// Partition + halo + LET (see the file header).  leaf_pan / leaf_tgt: panels / target points
// (panels + charges) per leaf of all ranks; K: quadrature points per panel (P2P sources).
// Every loop is split over the host threads a rank may use (hardware threads / ranks, <= 16);
// the results do not depend on the split.
namespace {
bool plan_verbose() {
  static const bool v = std::getenv("FMMBEM_VERBOSE") != nullptr;
  return v;
}
int plan_threads(int R) {
  return (int)std::min(16u, std::max(1u, std::thread::hardware_concurrency() / (unsigned)std::max(1, R)));
}
}  // namespace

// the cost-weighted contiguous leaf partition (needs only the neighbour lists and the per-leaf
// interaction-list lengths: fmmbem_create calls it before copying any interaction list to the host)
void plan_partition(const HostTree& T, const std::vector<int>& leaf_pan, int K, int R, ExchangePlan& X) {
  const int nth = plan_threads(R);
  const int L = T.L;
  const int64_t nl = T.lvl_off[L + 1] - T.lvl_off[L];
  const int64_t leaf0 = T.lvl_off[L];
  // leaf cost: P2P interactions + M2L translations (~600 interaction-equivalents each) + per point
  std::vector<double> cost(nl);
  parallel_for(nl, nth, [&](int64_t lo_k, int64_t hi_k, int) {
    for (int64_t k = lo_k; k < hi_k; ++k) {
      long long s = 0;
      for (int e = T.nbr_off[k]; e < T.nbr_off[k + 1]; ++e) s += leaf_pan[T.nbr_idx[e]];
      const long long nt = leaf_pan[k];
      const double m2l = (double)(T.m2l_off[leaf0 + k + 1] - T.m2l_off[leaf0 + k]);
      cost[k] = (double)(nt * s * K) + (nt ? 600.0 * m2l : 0.0) + 50.0 * (double)nt;
    }
  });
  X.leaf_bounds.assign(R + 1, 0);
  split_costs(cost.data(), nl, R, X.leaf_bounds.data());
}

void plan_exchange(const HostTree& T, const std::vector<int>& leaf_pan, const std::vector<int>& leaf_tgt, int K,
                   int R, int me, ExchangePlan& X) {
  plan_partition(T, leaf_pan, K, R, X);
  plan_lists(T, leaf_pan, leaf_tgt, R, me, X);
}

// Halo, LET and slots for the partition in X.leaf_bounds.  Reads the interaction lists of this
// rank's window cells only (the cells it owns and the cells holding its targets), so fmmbem_create
// passes a tree whose lists outside the windows are empty.
void plan_lists(const HostTree& T, const std::vector<int>& leaf_pan, const std::vector<int>& leaf_tgt, int R, int me,
                ExchangePlan& X) {
  auto t_last = std::chrono::steady_clock::now();
  auto stage = [&](const char* what) {
    if (!plan_verbose()) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[fmmbem plan %d] %-14s %8.1f ms\n", me, what,
                 std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  const int nth = plan_threads(R);
  const int L = T.L;
  const int64_t nl = T.lvl_off[L + 1] - T.lvl_off[L], nc = T.lvl_off[L + 1];
  const int64_t leaf0 = T.lvl_off[L];
  std::vector<int> lrank(nl);
  for (int r = 0; r < R; ++r)
    for (int64_t k = X.leaf_bounds[r]; k < X.leaf_bounds[r + 1]; ++k) lrank[k] = r;
  // near-field halo: per-thread chunks of leaves, concatenated in leaf order
  X.halo_send.assign(R, {});
  X.halo_recv.assign(R, {});
  {
    std::vector<std::vector<std::vector<int>>> hs(nth, std::vector<std::vector<int>>(R)), hr(hs);
    parallel_for(nl, nth, [&](int64_t lo_k, int64_t hi_k, int t) {
      for (int64_t k = lo_k; k < hi_k; ++k) {
        if (lrank[k] == me) {
          unsigned long long m = 0;
          for (int e = T.nbr_off[k]; e < T.nbr_off[k + 1]; ++e) m |= 1ULL << lrank[T.nbr_idx[e]];
          for (int p = 0; p < R; ++p)
            if (p != me && (m >> p & 1ULL)) hs[t][p].push_back((int)k);
        } else {
          bool need = false;
          for (int e = T.nbr_off[k]; e < T.nbr_off[k + 1] && !need; ++e) need = lrank[T.nbr_idx[e]] == me;
          if (need) hr[t][lrank[k]].push_back((int)k);
        }
      }
    });
    for (int t = 0; t < nth; ++t)
      for (int p = 0; p < R; ++p) {
        X.halo_send[p].insert(X.halo_send[p].end(), hs[t][p].begin(), hs[t][p].end());
        X.halo_recv[p].insert(X.halo_recv[p].end(), hr[t][p].begin(), hr[t][p].end());
      }
  }
  stage("halo");
  // local essential tree: leaf range [first, end) and owner of every cell (levels >= 2), sources
  // per cell.  Panel multipoles serve every target point (K', V, A at panels; the reaction
  // potential at the charges); charge multipoles serve the panels (E_n, psi of the charge-FMM).
  std::vector<long long> tpre(nl + 1, 0), ppre(nl + 1, 0);
  for (int64_t k = 0; k < nl; ++k) {
    tpre[k + 1] = tpre[k] + leaf_tgt[k];
    ppre[k + 1] = ppre[k] + leaf_pan[k];
  }
  const int c0l = std::min(2, L + 1);
  const int64_t c0 = T.lvl_off[c0l];
  std::vector<int> first(nc, 0), end(nc, 0), owner(nc, -1);
  std::vector<char> has_src(nc, 0), has_chg(nc, 0);
  std::vector<unsigned long long> tmask(nc, 0), pmask(nc, 0);  // ranks with targets / panels below
  for (int l = c0l; l <= L; ++l) {  // the cells of a level and the leaves are both key-sorted: one sweep
    const int sh = 3 * (L - l);
    int64_t j = 0;
    for (int64_t c = T.lvl_off[l]; c < T.lvl_off[l + 1]; ++c) {
      while (j < nl && (T.key[leaf0 + j] >> sh) < T.key[c]) ++j;
      first[c] = (int)j;
      while (j < nl && (T.key[leaf0 + j] >> sh) == T.key[c]) ++j;
      end[c] = (int)j;
    }
  }
  parallel_for(nc - c0, nth, [&](int64_t lo_i, int64_t hi_i, int) {
    for (int64_t c = c0 + lo_i; c < c0 + hi_i; ++c) {
      if (end[c] <= first[c]) continue;
      if (lrank[first[c]] == lrank[end[c] - 1]) owner[c] = lrank[first[c]];
      has_src[c] = ppre[end[c]] > ppre[first[c]];
      has_chg[c] = (tpre[end[c]] - tpre[first[c]]) > (ppre[end[c]] - ppre[first[c]]);
      unsigned long long tm = 0, pm = 0;
      for (int p = lrank[first[c]]; p <= lrank[end[c] - 1]; ++p) {
        const int f = std::max(first[c], (int)X.leaf_bounds[p]), e = std::min(end[c], (int)X.leaf_bounds[p + 1]);
        if (e > f && tpre[e] > tpre[f]) tm |= 1ULL << p;
        if (e > f && ppre[e] > ppre[f]) pm |= 1ULL << p;
      }
      tmask[c] = tm;
      pmask[c] = pm;
    }
  });
  stage("cell ranges");
  // Which pure cells move: the interaction lists are symmetric (s in list(c) <=> c in list(s): the
  // parents are neighbours, the cells are not), so the ranks that need a pure cell s (targets below
  // some c whose list holds s) are the OR of tmask over s's OWN list.  Each rank evaluates that for
  // the cells it owns (to send) and for the cells of the lists of the cells holding its targets (to
  // receive) -- about 2/R of one pass over all lists, no atomics.
  X.let_send.assign(R, {});
  X.let_recv.assign(R, {});
  X.let_shared.clear();
  X.let_send_chg.assign(R, {});
  X.let_recv_chg.assign(R, {});
  X.let_shared_chg.clear();
  std::vector<unsigned long long> need(nc, 0), need_c(nc, 0);
  // the cells this rank sends: the OR of tmask / pmask over their own lists
  parallel_for(nc - c0, nth, [&](int64_t lo_i, int64_t hi_i, int) {
    for (int64_t s_ = c0 + lo_i; s_ < c0 + hi_i; ++s_) {
      if (owner[s_] != me || !(has_src[s_] || has_chg[s_])) continue;
      unsigned long long m = 0, mc = 0;
      for (int64_t k = T.m2l_off[s_]; k < T.m2l_off[s_ + 1]; ++k) {
        m |= tmask[T.m2l_idx[k]];
        mc |= pmask[T.m2l_idx[k]];
      }
      need[s_] = has_src[s_] ? m : 0;
      need_c[s_] = has_chg[s_] ? mc : 0;
    }
  });
  // the cells this rank receives: those in the lists of the cells holding its targets / panels
  {
    std::unique_ptr<std::atomic<unsigned char>[]> flag(new std::atomic<unsigned char>[nc]);
    for (int64_t c = 0; c < nc; ++c) flag[c].store(0, std::memory_order_relaxed);
    const unsigned long long bit = 1ULL << me;
    parallel_for(nc - c0, nth, [&](int64_t lo_i, int64_t hi_i, int) {
      for (int64_t c = c0 + lo_i; c < c0 + hi_i; ++c) {
        const bool t = tmask[c] & bit, p = pmask[c] & bit;
        if (!t) continue;
        for (int64_t k = T.m2l_off[c]; k < T.m2l_off[c + 1]; ++k) {
          const int s_ = T.m2l_idx[k];
          if (owner[s_] < 0 || owner[s_] == me) continue;
          const unsigned char f = (has_src[s_] ? 1 : 0) | ((p && has_chg[s_]) ? 2 : 0);
          if (f && (flag[s_].load(std::memory_order_relaxed) & f) != f) flag[s_].fetch_or(f, std::memory_order_relaxed);
        }
      }
    });
    for (int64_t c = c0; c < nc; ++c) {
      const unsigned char f = flag[c].load(std::memory_order_relaxed);
      if (f & 1) need[c] |= bit;
      if (f & 2) need_c[c] |= bit;
    }
  }
  auto lists = [&](const std::vector<char>& has, const std::vector<unsigned long long>& nd,
                   std::vector<std::vector<int>>& snd, std::vector<std::vector<int>>& rcv, std::vector<int>& shr) {
    for (int64_t c = c0; c < nc; ++c) {
      const unsigned long long m = nd[c];
      if (owner[c] < 0) {
        if (has[c]) shr.push_back((int)c);
        continue;
      }
      if (owner[c] == me) {
        for (int p = 0; p < R; ++p)
          if (p != me && (m >> p & 1ULL)) snd[p].push_back((int)c);
      } else if (m >> me & 1ULL) {
        rcv[owner[c]].push_back((int)c);
      }
    }
  };
  stage("need pass");
  lists(has_src, need, X.let_send, X.let_recv, X.let_shared);
  lists(has_chg, need_c, X.let_send_chg, X.let_recv_chg, X.let_shared_chg);
  stage("LET lists");
  slot_layout(T, me, X);
  stage("slots");
}

// Windows of this rank's cells per level and the slot numbering (plan.h).  A cell of level l holds
// a leaf of [lo, hi) iff its key lies between the level-l ancestors of leaves lo and hi - 1.
void plan_windows(const HostTree& T, int me, ExchangePlan& X) {
  const int L = T.L;
  const int64_t leaf0 = T.lvl_off[L];
  const int64_t lo = X.leaf_bounds[me], hi = X.leaf_bounds[me + 1];
  X.lvl_off = T.lvl_off;
  X.win_lo.assign(L + 1, 0);
  X.win_hi.assign(L + 1, 0);
  for (int l = 0; l <= L; ++l) {
    X.win_lo[l] = X.win_hi[l] = T.lvl_off[l];
    if (hi > lo) {
      const int sh = 3 * (L - l);
      X.win_lo[l] = lower_bound_key(T.key, T.lvl_off[l], T.lvl_off[l + 1], T.key[leaf0 + lo] >> sh);
      X.win_hi[l] = lower_bound_key(T.key, T.lvl_off[l], T.lvl_off[l + 1], T.key[leaf0 + hi - 1] >> sh) + 1;
    }
  }
}

void slot_layout(const HostTree& T, int me, ExchangePlan& X) {
  const int L = T.L;
  plan_windows(T, me, X);
  X.slot_base.assign(L + 1, 0);
  int64_t n = 0;
  for (int l = 0; l <= L; ++l) {
    X.slot_base[l] = n;
    n += X.win_hi[l] - X.win_lo[l];
  }
  std::vector<int> ex;
  auto add = [&](const std::vector<int>& v) { ex.insert(ex.end(), v.begin(), v.end()); };
  for (size_t p = 0; p < X.let_recv.size(); ++p) add(X.let_recv[p]);
  for (size_t p = 0; p < X.let_recv_chg.size(); ++p) add(X.let_recv_chg[p]);
  add(X.let_shared);
  add(X.let_shared_chg);
  std::sort(ex.begin(), ex.end());
  ex.erase(std::unique(ex.begin(), ex.end()), ex.end());
  X.extra.clear();
  X.n_slots = n;
  for (int c : ex)
    if (X.slot(c) < 0) X.extra.push_back(c);
  X.n_slots = n + (int64_t)X.extra.size();
}

int64_t ExchangePlan::slot(int64_t c) const {
  if (c < 0 || lvl_off.empty() || c >= lvl_off.back()) return -1;
  const int l = (int)(std::upper_bound(lvl_off.begin(), lvl_off.end(), c) - lvl_off.begin()) - 1;
  if (c >= win_lo[l] && c < win_hi[l]) return slot_base[l] + (c - win_lo[l]);
  const auto it = std::lower_bound(extra.begin(), extra.end(), (int)c);
  if (it == extra.end() || *it != c) return -1;
  const int64_t nw = slot_base.back() + (win_hi.back() - win_lo.back());
  return nw + (it - extra.begin());
}

}  // namespace fmm

using namespace fmm;

struct fmmbem_plan {
  HostTree tree;
  ExchangePlan plan;
};

extern "C" {

fmmbem_status fmmbem_plan_create(const uint64_t* leaf_keys, const int32_t* leaf_panels, const int32_t* leaf_charges,
                                 int64_t n_leaves, int32_t level, int32_t quad_points, int32_t nranks, int32_t rank,
                                 fmmbem_plan** out) {
  if (out) *out = nullptr;
  if (!out || !leaf_keys || !leaf_panels || n_leaves < 1 || level < 0 || level > MAX_LEVEL || nranks < 1 ||
      nranks > 64 || rank < 0 || rank >= nranks || quad_points < 1)
    return FMMBEM_E_INVALID;
  for (int64_t k = 1; k < n_leaves; ++k)
    if (!(leaf_keys[k - 1] < leaf_keys[k])) return FMMBEM_E_INVALID;
  try {
    auto* p = new fmmbem_plan();
    host_tree(leaf_keys, n_leaves, level, p->tree);
    std::vector<int> pan(leaf_panels, leaf_panels + n_leaves), tgt(pan);
    if (leaf_charges)
      for (int64_t k = 0; k < n_leaves; ++k) tgt[k] += leaf_charges[k];
    plan_exchange(p->tree, pan, tgt, quad_points, nranks, rank, p->plan);
    *out = p;
    return FMMBEM_OK;
  } catch (...) {
    return FMMBEM_E_NOMEM;
  }
}

void fmmbem_plan_destroy(fmmbem_plan* p) { delete p; }

int64_t fmmbem_plan_list(const fmmbem_plan* p, int32_t list, int32_t peer, int64_t* out) {
  if (!p) return -1;
  const auto& X = p->plan;
  const auto& T = p->tree;
  const int R = (int)X.leaf_bounds.size() - 1;
  auto emit = [&](const auto& v) -> int64_t {
    if (out)
      for (size_t i = 0; i < v.size(); ++i) out[i] = (int64_t)v[i];
    return (int64_t)v.size();
  };
  const bool per_peer = (list >= FMMBEM_PLAN_HALO_SEND && list <= FMMBEM_PLAN_LET_RECV) ||
                        list == FMMBEM_PLAN_LET_SEND_CHG || list == FMMBEM_PLAN_LET_RECV_CHG;
  if (per_peer && (peer < 0 || peer >= R)) return -1;
  const int64_t nl = T.lvl_off[T.L + 1] - T.lvl_off[T.L], nc = T.lvl_off[T.L + 1];
  if (list == FMMBEM_PLAN_NEIGHBOURS) {
    if (peer < 0 || peer >= nl) return -1;
    std::vector<int> v(T.nbr_idx.begin() + T.nbr_off[peer], T.nbr_idx.begin() + T.nbr_off[peer + 1]);
    return emit(v);
  }
  if (list == FMMBEM_PLAN_INTERACTION) {
    if (peer < 0 || peer >= nc) return -1;
    std::vector<int> v(T.m2l_idx.begin() + T.m2l_off[peer], T.m2l_idx.begin() + T.m2l_off[peer + 1]);
    return emit(v);
  }
  switch (list) {
    case FMMBEM_PLAN_HALO_SEND: return emit(X.halo_send[peer]);
    case FMMBEM_PLAN_HALO_RECV: return emit(X.halo_recv[peer]);
    case FMMBEM_PLAN_LET_SEND: return emit(X.let_send[peer]);
    case FMMBEM_PLAN_LET_RECV: return emit(X.let_recv[peer]);
    case FMMBEM_PLAN_LET_SHARED: return emit(X.let_shared);
    case FMMBEM_PLAN_LEAF_BOUNDS: return emit(X.leaf_bounds);
    case FMMBEM_PLAN_CELL_KEYS: return emit(T.key);
    case FMMBEM_PLAN_LEVEL_OFFSETS: return emit(T.lvl_off);
    case FMMBEM_PLAN_LET_SEND_CHG: return emit(X.let_send_chg[peer]);
    case FMMBEM_PLAN_LET_RECV_CHG: return emit(X.let_recv_chg[peer]);
    case FMMBEM_PLAN_LET_SHARED_CHG: return emit(X.let_shared_chg);
    case FMMBEM_PLAN_EXTRA_CELLS: return emit(X.extra);
    case FMMBEM_PLAN_CELL_WINDOWS: {
      std::vector<int64_t> v;
      for (size_t l = 0; l < X.win_lo.size(); ++l) {
        v.push_back(X.win_lo[l]);
        v.push_back(X.win_hi[l]);
      }
      return emit(v);
    }
    default: return -1;
  }
}

}  // extern "C"
