// plan.h -- host-side multi-GPU exchange plan (plan.cu): partition, near-field halo, LET.
#pragma once
#include <stdint.h>

#include <memory>
#include <utility>
#include <vector>

#include "common.cuh"

namespace fmm {

// std::vector whose resize() leaves new elements uninitialised (the host copies of the device
// lists are overwritten by cudaMemcpy right away: zeroing 10 GB at 1e9 panels costs seconds)
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using HostVec = std::vector<T, NoInitAlloc<T>>;

// The octree skeleton on the host: cells of every level (level-major, sorted keys), child ranges,
// leaf neighbour lists (leaf indices) and interaction lists (global cell indices).
struct HostTree {
  int L = 0;
  std::vector<int64_t> lvl_off;
  HostVec<uint64_t> key;
  std::vector<int> child_b, child_e;
  HostVec<int> nbr_off, nbr_idx;
  HostVec<int64_t> m2l_off;
  HostVec<int> m2l_idx;
};

struct ExchangePlan {
  std::vector<int64_t> leaf_bounds;                  // [R + 1] contiguous leaf ranges
  std::vector<std::vector<int>> halo_send, halo_recv;  // per peer: leaves (increasing)
  std::vector<std::vector<int>> let_send, let_recv;    // per peer: pure cells (increasing), panel sources
  std::vector<int> let_shared;                         // cells straddling ranks (with panel sources)
  std::vector<std::vector<int>> let_send_chg, let_recv_chg;  // the same for charge sources (charge-FMM)
  std::vector<int> let_shared_chg;
  // rank-local expansion storage: the cells of level l holding a leaf of this rank form the window
  // [win_lo[l], win_hi[l]) (contiguous: leaves and cells are in Morton order); they get the slots
  // slot_base[l] + (cell - win_lo[l]), and the LET cells received or shared that lie outside the
  // windows (`extra`, increasing) follow them.
  std::vector<int64_t> lvl_off, win_lo, win_hi, slot_base;  // [L + 2] / [L + 1]
  std::vector<int> extra;
  int64_t n_slots = 0;
  int64_t slot(int64_t cell) const;  // -1: no slot on this rank
};

void host_tree(const uint64_t* leaf_keys, int64_t nl, int L, HostTree& T);
void plan_exchange(const HostTree& T, const std::vector<int>& leaf_pan, const std::vector<int>& leaf_tgt, int K,
                   int R, int me, ExchangePlan& X);  // = plan_partition + plan_lists
void plan_partition(const HostTree& T, const std::vector<int>& leaf_pan, int K, int R, ExchangePlan& X);
void plan_lists(const HostTree& T, const std::vector<int>& leaf_pan, const std::vector<int>& leaf_tgt, int R, int me,
                ExchangePlan& X);
void plan_windows(const HostTree& T, int me, ExchangePlan& X);  // win_lo / win_hi of X.leaf_bounds[me..]
void slot_layout(const HostTree& T, int me, ExchangePlan& X);  // windows + extra cells (plan_exchange calls it)
void split_costs(const double* cost, int64_t n, int parts, int64_t* bounds);

}  // namespace fmm
