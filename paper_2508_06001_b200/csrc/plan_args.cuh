// Planner kernel arguments (device views of the plan SoA and its scratch)
// shared by the multi-kernel path, the fused planner and the diagnostics
// (tools/micro/greedy_prod.cu).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace sb {

constexpr int kMaxBags = 64;         // bags per replica on the fused planner and the register greedy
constexpr int kMaxBagsLarge = 1024;  // bags per replica on the multi-kernel path (k_greedy_many, k_emit tables)

struct PlanArgs {
  int W, U, M, R;
  double d_model, gamma;
  int64_t max_seqs;
  const int32_t *bag_off, *bag_ranks, *bag_size, *rank_bag, *rank_member;
  const uint64_t* ids;
  const int64_t* lens;
  const int64_t* rank_off;
  const double* w_in;  // non-null: caller-supplied workloads (assign_to_bags)
  double* w;
  int32_t* seq_rank;
  int64_t* seq_off;
  uint64_t* hash;
  uint64_t *sk_hi, *sk_lo, *tk_hi, *tk_lo;
  uint32_t *sk_v, *tk_v;
  double* sorted_w;
  int32_t* sorted_idx;
  int32_t* pick;
  int32_t *seq_bag, *seq_G;
  int32_t* greedy_q;  // hybrid path: the greedy kernel's per-position rank inside the bag
  int64_t* seq_chunk_base;
  double* rep_total;
  int32_t* sentinel;
  int32_t* bag_count;
  int64_t* bag_rows;
  int64_t* rep_chunks;
  int64_t* rep_cbase;  // R+1: first chunk of each replica
  int32_t* bag_seq;    // N: sequences grouped by (replica, bag), q ascending
  int32_t* tile_cnt;   // R * ceil(N / kEmitTile) * M: picks per (replica, tile, bag)
  int64_t* list_sum;   // W * ceil(N / kListTile) * 4: per-tile sums of k_lists' four domains
  int32_t* list_tie;   // W: reverse order of rank r needs the std::sort replay
  int64_t *bag_cbase, *bag_sbase;  // R*M
  unsigned long long* send_count;
  int64_t *n_chunks, *n_seqs;
  uint64_t* c_id;
  int32_t *c_idx, *c_src, *c_dst;
  int64_t *c_start, *c_end, *c_src_row, *c_dst_row, *c_seq_base;
  int32_t* c_seq;
  int64_t *send_off, *recv_off;
  int32_t *send_idx, *recv_idx, *rev_recv_idx;
  int64_t *origin_rows, *target_rows;
  double *per_gpu, *per_bag_occ, *total, *wir;
  int32_t* violations;
  int32_t* status;
  long long* trace;  // optional per-phase timestamps (small path)
};

__device__ __forceinline__ bool seqs_ok(const PlanArgs& a) { return a.rank_off[a.W] <= a.max_seqs; }

__device__ __forceinline__ double occupancy(double asg, double cap) {  // balancer.cpp:32-35
  if (cap > 0.0) return __ddiv_rn(asg, cap);
  return asg > 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0;
}

}  // namespace sb
