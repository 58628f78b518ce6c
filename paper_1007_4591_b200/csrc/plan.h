// plan.h -- host-side multi-GPU exchange plan (plan.cu): partition, near-field halo, LET.
#pragma once
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace fmm {

// The octree skeleton on the host: cells of every level (level-major, sorted keys), child ranges,
// leaf neighbour lists (leaf indices) and interaction lists (global cell indices).
struct HostTree {
  int L = 0;
  std::vector<int64_t> lvl_off;
  std::vector<uint64_t> key;
  std::vector<int> child_b, child_e;
  std::vector<int> nbr_off, nbr_idx;
  std::vector<int64_t> m2l_off;
  std::vector<int> m2l_idx;
};

struct ExchangePlan {
  std::vector<int64_t> leaf_bounds;                  // [R + 1] contiguous leaf ranges
  std::vector<std::vector<int>> halo_send, halo_recv;  // per peer: leaves (increasing)
  std::vector<std::vector<int>> let_send, let_recv;    // per peer: pure cells (increasing)
  std::vector<int> let_shared;                         // cells straddling ranks (with sources)
};

void host_tree(const uint64_t* leaf_keys, int64_t nl, int L, HostTree& T);
void plan_exchange(const HostTree& T, const std::vector<int>& leaf_pan, const std::vector<int>& leaf_tgt, int K,
                   int R, int me, ExchangePlan& X);
void split_costs(const double* cost, int64_t n, int parts, int64_t* bounds);

}  // namespace fmm
