// The multi-knapsack greedy (balancer.cpp:44-62) on one warp: used by the
// fused planner (planner_small.cuh), the large path's k_greedy /
// k_greedy_staged (planner.cu) and the diagnostics (tools/micro/greedy_prod.cu).
#pragma once

#include "plan_args.cuh"

namespace sb {

// Correctly rounded a / b for the occupancy update, b > 0 normal, a >= 0
// finite, with r = __drcp_rn(b) precomputed per bag: one Newton refinement
// makes y faithful, then Markstein's fused correction y + r*(a - b*y)
// rounds to RN(a/b).  Five dependent FP64 ops instead of the ~25-op
// general __ddiv_rn sequence on the greedy's critical path; bit-identity
// with __ddiv_rn is asserted by sb_selftest_div over random operands in the
// planner's range (tests/test_gpu_parity.py).
__device__ __forceinline__ double div_rn_markstein(double a, double b, double r) {
  double y = __dmul_rn(a, r);
  double e = __fma_rn(-b, y, a);
  y = __fma_rn(r, e, y);
  e = __fma_rn(-b, y, a);
  return __fma_rn(r, e, y);
}

// ---------------------------------------------------------------- greedy
// balancer.cpp:44-62.  One warp per replica; bag j lives in lane j%32, slot
// j/32.  Per sequence every lane forms key = (infeasible << 63 | bits(occ))
// for its bags; the warp takes the lexicographic minimum of (key, j), which
// is exactly "feasible bag with minimum occupancy, else global minimum, ties
// to the lowest bag id" (occ >= 0, so its IEEE bits order like its value).
//
// Latency design (the loop is one dependent chain per sequence):
//  * the argmin is three REDUX.MIN (high word, low word among high-word
//    ties, lowest bag among exact ties) -- no vote/branch, ~50 cycles each;
//  * both possible keys of the NEXT step are formed during this one: kWin
//    (this bag wins now: new occupancy by a Markstein division, feasibility
//    against w_{t+1}) and kNot (it does not: old occupancy, feasibility
//    against w_{t+1}), so the chain is select -> REDUX x3 -> select;
//  * occupancy is computed branch-free (both arms, select): a divergent
//    branch would put BSSY/BSYNC on the chain.
// Measured on B200 (tools/micro/greedy_micro.cu): 154 cycles per sequence,
// down from 305 for the vote-based argmin with an in-loop division branch.
// `getw(p)` returns the workload of the p-th sequence in greedy order.
__device__ __forceinline__ double occupancy_sel(double asg, double cap, double rcap) {
  const double q = div_rn_markstein(asg, cap, rcap);  // rcap == 0 when cap == 0: finite, discarded
  const double z = asg > 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0;
  return cap > 0.0 ? q : z;
}

__device__ __forceinline__ uint64_t greedy_key(bool feasible, double occ) {
  return (feasible ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ);
}

constexpr int kGreedyChunk = 1024;  // `hook(p0)` runs before every chunk of this many steps

// One bag per replica (g8n1, g4n1, ...): every pick is bag 0 (balancer.cpp:44-62
// with m == 1), so the argmin chain disappears.  What stays serial is the FP64
// prefix in greedy order -- `capacity - assigned >= w` decides the violation
// count (balancer.cpp:159-163) and `assigned` the occupancy and per-GPU load --
// one DADD per sequence on lane 0; the other lanes write the picks.  Used by
// the fused planner (the large path runs k_single_bag_fill + k_single_bag_chain).
template <int CHUNK, class GetW, class Hook>
__device__ __forceinline__ void greedy_single_bag(const PlanArgs& a, int rep, int64_t n, double target, GetW getw,
                                                  Hook hook, int32_t* pick_out, int32_t* bagcnt_out,
                                                  int* viol_out, int32_t* q_out) {
  const int lane = threadIdx.x & 31;
  const int nn = (int)n;
  const int size = a.bag_size[0];
  const double cap = __dmul_rn((double)size, target);  // balancer.cpp:30
  double asg = 0.0;
  int viol = 0;
  auto run = [&](int p0, int p1) {
    for (int p = p0 + lane; p < p1; p += 32) {
      pick_out[p] = 0;
      if (q_out) q_out[p] = p;  // every sequence joins bag 0, in greedy order
    }
    if (lane == 0) {
      // the DADD on `asg` is the only chain: eight violation counters keep the
      // predicated increments off it (one counter was a second ~8-cycle chain)
      int v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int p = p0;
      for (; p + 8 <= p1; p += 8) {
        double w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = getw(p + k);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          v[k] += __dsub_rn(cap, asg) >= w[k] ? 0 : 1;
          asg = __dadd_rn(asg, w[k]);
        }
      }
      for (; p < p1; ++p) {
        const double w = getw(p);
        v[0] += __dsub_rn(cap, asg) >= w ? 0 : 1;
        asg = __dadd_rn(asg, w);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) viol += v[k];
    }
    __syncwarp();
  };
  if constexpr (CHUNK == 0) {
    run(0, nn);
  } else {
    hook(0);
    for (int p0 = 0; p0 < nn; p0 += CHUNK) {
      if (p0 > 0) hook(p0);
      run(p0, nn - p0 < CHUNK ? nn : p0 + CHUNK);
    }
  }
  if (lane != 0) return;
  if (bagcnt_out) bagcnt_out[rep] = nn;
  a.bag_count[rep] = nn;
  a.per_bag_occ[rep] = occupancy(asg, cap);  // balancer.cpp:170-175
  const double per = __ddiv_rn(asg, (double)size);  // balancer.cpp:199-202
  for (int k = 0; k < size; ++k) a.per_gpu[rep * a.U + a.bag_ranks[a.bag_off[0] + k]] = per;
  atomicAdd(viol_out, viol);
}

// CHUNK > 0: `hook(p0)` runs before every CHUNK steps (the large path's
// shared-memory ring); CHUNK == 0: one flat loop (the nested form costs the
// fused planner ~45 cycles per sequence in code generation).
// `q_out` (optional): per greedy position, the sequence's rank inside its
// bag (the stable bag partition of balancer.cpp:178-192), stored by the
// winning lane off the chain.
struct NoDone {
  __device__ void operator()() const {}
};

// `done()` runs once the picks are all stored, before the per-bag epilogue
// (the fused planner hands the picks to another warp there).  SB_TRACE_P3
// (diagnostics build) marks the setup and epilogue in trace slots 7, 11, 12.
template <int BPL, int CHUNK, bool QOUT = false, bool PADDED = false, class GetW, class Hook, class Done = NoDone>
__device__ __forceinline__ void greedy_warp(const PlanArgs& a, int rep, int64_t n, double total_rep, GetW getw,
                                            Hook hook, int32_t* pick_out, int32_t* bagcnt_out, int* viol_out,
                                            int32_t* q_out = nullptr, Done done = Done()) {
  const int lane = threadIdx.x & 31;
#ifdef SB_TRACE_P3
  if (a.trace && rep == 0 && lane == 0) a.trace[11] = clock64();
#endif
  const double target = __ddiv_rn(total_rep, (double)a.U);  // balancer.cpp:26
#ifdef SB_TRACE_P3
  if (a.trace && rep == 0 && lane == 0) a.trace[12] = clock64() + (target == 12345.0 ? 1 : 0);
#endif
  if (a.M == 1) {
    greedy_single_bag<CHUNK>(a, rep, n, target, getw, hook, pick_out, bagcnt_out, viol_out, q_out);
    done();
    return;
  }
  double cap[BPL], rcap[BPL], asg[BPL], occ[BPL], rem[BPL];
  uint64_t key[BPL];
  int cnt[BPL];
  bool act[BPL];  // loop-invariant: a.M is not re-read inside the chain
  const int M = a.M;
  hook(0);
  double w_a = n > 0 ? getw(0) : 0.0, w_b = n > 1 ? getw(1) : 0.0, w_c = n > 2 ? getw(2) : 0.0;
#pragma unroll
  for (int i = 0; i < BPL; ++i) {
    const int j = lane + 32 * i;
    act[i] = j < M;
    const int size = act[i] ? a.bag_size[j] : 0;
    cap[i] = __dmul_rn((double)size, target);  // balancer.cpp:30
    rcap[i] = cap[i] > 0.0 ? __drcp_rn(cap[i]) : 0.0;
    asg[i] = 0.0;
    occ[i] = 0.0;  // occupancy(0, cap): +0 for cap > 0 and for cap == 0 (balancer.cpp:32-35)
    rem[i] = __dsub_rn(cap[i], 0.0);
    key[i] = act[i] ? greedy_key(rem[i] >= w_a, occ[i]) : ~0ull;
    cnt[i] = 0;
  }
  int viol = 0;
  const int nn = (int)n;  // <= max_seqs < 2^31: 32-bit loop arithmetic
  if (a.trace && rep == 0 && lane == 0) a.trace[14] = clock64();  // diagnostics: setup | chain | epilogue
  auto step = [&](int p) {
    const double w = w_a, wn = w_b;  // w_p and w_{p+1} (0 past the end: unused)
    w_a = w_b;
    w_b = w_c;
    // prefetch under this step: clamped, or straight when getw is readable 3
    // past the end (PADDED: the staged kernels pad their buffer)
    w_c = getw(PADDED ? p + 3 : (p + 3 < nn ? p + 3 : nn - 1));
    double nasg[BPL], nocc[BPL], nrem[BPL];
    uint64_t kwin[BPL], knot[BPL];
    uint64_t best = ~0ull;
    uint32_t best_j = 0xffffffffu;
#pragma unroll
    for (int i = 0; i < BPL; ++i) {
      nasg[i] = __dadd_rn(asg[i], w);
      nocc[i] = occupancy_sel(nasg[i], cap[i], rcap[i]);
      nrem[i] = __dsub_rn(cap[i], nasg[i]);
      kwin[i] = act[i] ? greedy_key(nrem[i] >= wn, nocc[i]) : ~0ull;
      knot[i] = act[i] ? greedy_key(rem[i] >= wn, occ[i]) : ~0ull;
      if (BPL == 1 || key[i] < best) {  // strict: slot 0 (lower bag id) keeps ties
        best = key[i];
        best_j = (uint32_t)(lane + 32 * i);
      }
    }
    const uint32_t khi = (uint32_t)(best >> 32), klo = (uint32_t)best;
    const uint32_t m1 = __reduce_min_sync(0xffffffffu, khi);
    const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
    const uint32_t pick = __reduce_min_sync(0xffffffffu, (khi == m1 && klo == m2) ? best_j : 0xffffffffu);
    viol += (int)(m1 >> 31);  // winner infeasible: fallback pick == capacity violation
#pragma unroll
    for (int i = 0; i < BPL; ++i) {
      const bool won = (uint32_t)(lane + 32 * i) == pick;
      if (QOUT && won) q_out[p] = cnt[i];
      key[i] = won ? kwin[i] : knot[i];
      asg[i] = won ? nasg[i] : asg[i];
      occ[i] = won ? nocc[i] : occ[i];
      rem[i] = won ? nrem[i] : rem[i];
      cnt[i] += won ? 1 : 0;
    }
    if (lane == 0) pick_out[p] = (int)pick;
  };
  if constexpr (CHUNK == 0) {
    for (int p = 0; p < nn; ++p) step(p);
  } else {
    for (int p0 = 0; p0 < nn; p0 += CHUNK) {
      if (p0 > 0) hook(p0);
      const int p1 = nn - p0 < CHUNK ? nn : p0 + CHUNK;
      for (int p = p0; p < p1; ++p) step(p);
    }
  }
  if (a.trace && rep == 0 && lane == 0) a.trace[15] = clock64();
  done();
#pragma unroll
  for (int i = 0; i < BPL; ++i) {
    const int j = lane + 32 * i;
    if (j < a.M) {
      if (bagcnt_out) bagcnt_out[rep * a.M + j] = cnt[i];
      a.bag_count[rep * a.M + j] = cnt[i];
      a.per_bag_occ[rep * a.M + j] = occ[i];  // balancer.cpp:170-175 (replay == greedy)
      const int g = a.bag_size[j];
      const double per = __ddiv_rn(asg[i], (double)g);  // balancer.cpp:199-202
      for (int k = 0; k < g; ++k) a.per_gpu[rep * a.U + a.bag_ranks[a.bag_off[j] + k]] = per;
    }
  }
  if (lane == 0) atomicAdd(viol_out, viol);
#ifdef SB_TRACE_P3
  if (a.trace && rep == 0 && lane == 0) a.trace[7] = clock64();
#endif
}

}  // namespace sb
