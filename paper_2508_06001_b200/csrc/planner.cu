// Device planner: the reference's plan_routing (balancer.cpp:105-225),
// identity_plan (:227-240) and the receive order of reverse_plan (:242-287),
// reproduced bit-exactly on the GPU.
//
// Pipeline (no host synchronisation, graph-capturable):
//   k_totals      R+1 CTAs     serial per-replica / global FP64 totals, forked
//                              onto a side stream at the start (workloads
//                              recomputed from lengths), joined before the greedy
//   k_prep_seq    seq grid     workloads (FP64, reference operation order), owner
//                              rank, duplicate-id hash
//   k_prep_rows   W CTAs       per-rank origin row offsets (block scan)
//   k_sort_tiles  tiles        2048-record bitonic tiles in shared memory
//   k_merge_pass  x log2(n/2048)  co-rank merges, one record per thread
//   k_sort_finish              greedy order (workload desc, id asc)
//   k_greedy      R warps      the multi-knapsack greedy: lane = bag, warp
//                              argmin via REDUX, speculative next-step keys
//   k_emit        R CTAs       stable bag partition (match_any + scan)
//   k_emit_chunks chunk grid   chunk emission in the reference's chunk order
//   k_lists       W CTAs       send/recv manifests, receive-side row offsets,
//                              reverse receive order, Ulysses sequence bases
//   k_finalize    1 CTA        WIR, chunk count
// Batches of <= 2048 sequences take the fused single-CTA planner instead
// (planner_small.cuh).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <limits>
#include <new>
#include <utility>

#include "block_sort.cuh"
#include "common.cuh"
#include "greedy.cuh"
#include "internal.hpp"
#include "plan_args.cuh"
#include "serial_sum.cuh"
#include "stdsort.cuh"
#include "tma.cuh"

namespace sb {

__device__ __forceinline__ uint64_t hash_slot(uint64_t id) { return splitmix64(id ^ 0x5eedULL); }

__global__ void k_selftest_div(uint64_t seed, int64_t n, unsigned long long* mismatches) {
  unsigned long long bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h1 = splitmix64(seed ^ (uint64_t)(2 * i)), h2 = splitmix64(seed ^ (uint64_t)(2 * i + 1));
    // capacities and assigned loads spanning the planner's range: sums of
    // 24 l d^2 + g 4 l^2 d terms, 1e6 .. 1e22, plus exact-quotient cases
    const double b = ldexp(1.0 + (double)(h1 >> 12) * 0x1.0p-52, 20 + (int)(h1 & 31) * 2);
    double a;
    if ((h2 & 7) == 0) a = __dmul_rn(b, (double)((h2 >> 3) & 0xffff));  // exact multiples
    else a = __dmul_rn(b, (double)(h2 >> 11) * 0x1.0p-53 * 2.5);         // occupancies in [0, 2.5)
    if (__double_as_longlong(div_rn_markstein(a, b, __drcp_rn(b))) != __double_as_longlong(__ddiv_rn(a, b))) ++bad;
  }
  if (bad) atomicAdd(mismatches, bad);
}

// ------------------------------------------------------------------ prep
// Per sequence (grid over the capacity, one thread per gathered sequence):
// workload (balancer.cpp:144; or the caller's for assign_to_bags), owning
// rank and the length check (workload_model.cpp:66); the duplicate-id check
// (open addressing in global memory) is k_prep_dup on the side stream.
__device__ __forceinline__ double seq_workload(const PlanArgs& a, int64_t i) {
  if (a.w_in) return a.w_in[i];
  const int64_t len = a.lens[i];
  return gamma_weighted_workload(len < 0 ? 0 : len, a.d_model, a.gamma);
}

__global__ void __launch_bounds__(256) k_prep_seq(PlanArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (!seqs_ok(a)) {
    if (i == 0) atomicOr(a.status, ST_CAPACITY);
    return;
  }
  if (i >= a.rank_off[a.W]) return;
  int lo = 0, hi = a.W;  // rank r with rank_off[r] <= i < rank_off[r+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (a.rank_off[mid] <= i) lo = mid;
    else hi = mid;
  }
  const int r = lo;
  if (a.lens[i] < 0) atomicOr(a.status, ST_NEG_LENGTH);
  const double wi = seq_workload(a, i);
  if (a.w_in && !(wi >= 0.0)) atomicOr(a.status, ST_NEG_LENGTH);  // balancer.cpp:18-20
  a.w[i] = wi;
  a.seq_rank[i] = r;
}

// The duplicate-id check inside each replica (divergence), on the
// planner's side stream after the totals: only the status word depends on
// it, so it runs beside the sort and the greedy and is joined at the end.
__global__ void __launch_bounds__(256) k_prep_dup(PlanArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (!seqs_ok(a) || a.w_in || i >= a.rank_off[a.W]) return;
  int lo = 0, hi = a.W;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (a.rank_off[mid] <= i) lo = mid;
    else hi = mid;
  }
  const int rep = lo / a.U;
  const int64_t rlo = a.rank_off[rep * a.U], rhi = a.rank_off[rep * a.U + a.U];
  const int64_t tsize = 2 * (rhi - rlo);
  uint64_t* tab = a.hash + 2 * rlo;
  const uint64_t id = a.ids[i];
  if (id == ~0ull) {
    if (atomicAdd(&a.sentinel[rep], 1) > 0) atomicOr(a.status, ST_DUP_ID);
    return;
  }
  uint64_t slot = hash_slot(id) % (uint64_t)tsize;
  while (true) {
    const unsigned long long old =
        atomicCAS(reinterpret_cast<unsigned long long*>(tab + slot), ~0ull, (unsigned long long)id);
    if (old == ~0ull) break;
    if (old == id) {
      atomicOr(a.status, ST_DUP_ID);
      break;
    }
    slot = (slot + 1 == (uint64_t)tsize) ? 0 : slot + 1;
  }
}

// Per rank: origin packing offsets (block scan of the lengths in buffer
// order), one pass: each thread owns a contiguous slice, one block scan of the
// slice sums.  Runs on the side stream beside the totals (nothing before the
// greedy reads it).
constexpr int kPrepRowsThreads = 1024;

__global__ void __launch_bounds__(kPrepRowsThreads) k_prep_rows(PlanArgs a) {
  __shared__ int64_t sh[33];
  const int r = blockIdx.x;
  if (!seqs_ok(a)) return;
  const int64_t lo = a.rank_off[r], hi = a.rank_off[r + 1];
  const int64_t per = (hi - lo + blockDim.x - 1) / blockDim.x;
  const int64_t b0 = lo + (int64_t)threadIdx.x * per, b1 = b0 + per < hi ? b0 + per : hi;
  int64_t loc = 0;
  for (int64_t i = b0; i < b1; ++i) {
    const int64_t len = a.lens[i];
    loc += len < 0 ? 0 : len;
  }
  int64_t tot;
  int64_t run = block_excl_scan<int64_t>(loc, sh, &tot);
  for (int64_t i = b0; i < b1; ++i) {
    a.seq_off[i] = run;
    const int64_t len = a.lens[i];
    run += len < 0 ? 0 : len;
  }
  if (threadIdx.x == 0) {
    a.origin_rows[r] = tot;
    a.send_count[r] = 0;
  }
}

// ------------------------------------------------------------------ sort
// Per replica sort by (workload desc, sample_id asc) (balancer.cpp:37-40) as
// ascending (~bits(w), id, local index): w >= 0, so its IEEE bits are
// monotone in value; the index makes the order total, so the result does not
// depend on sort stability.  Multi-CTA: k_sort_tiles sorts 2048-record tiles
// in shared memory (one CTA per tile of every replica), then log2(n/2048)
// k_merge_pass launches merge run pairs by co-rank (each record's output
// slot = its rank in its own run + its rank in the partner run, one binary
// search per record, all CTAs busy); k_sort_finish emits the greedy order.

// Replica of gathered position g (replicas are contiguous in gather order).
__device__ __forceinline__ int replica_of(const PlanArgs& a, int64_t g) {
  int lo = 0, hi = a.R;  // rank_off[lo*U] <= g < rank_off[hi*U]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (a.rank_off[mid * a.U] <= g) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Sorted runs of kRunTile records, one record per thread: a 512-record
// register bitonic is ~4.5 us on one SM, so several small tiles on several
// SMs plus merge passes beat one 2048-record tile (48 us, issue-bound).
constexpr int kSortThreads = 512;
constexpr int kRunTile = kSortThreads;
static_assert(kRunTile <= kSortTile, "run tile fits the staging buffers");

template <int T, int RPT>
__device__ __forceinline__ void sort_tile_out(const PlanArgs& a, uint64_t* s_hi, uint64_t* s_lo, uint32_t* s_v, int cnt,
                                              int64_t base) {
  uint64_t h[RPT], l[RPT];
  uint32_t v[RPT];
  reg_bitonic<T, RPT, kSortThreads>(s_hi, s_lo, s_v, cnt, h, l, v);
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int x = threadIdx.x + r * kSortThreads;
    if (x < cnt) {
      a.sk_hi[base + x] = h[r];
      a.sk_lo[base + x] = l[r];
      a.sk_v[base + x] = v[r];
    }
  }
}

__global__ void __launch_bounds__(kSortThreads) k_sort_tiles(PlanArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (!seqs_ok(a)) return;
  int b = blockIdx.x, rep = -1;
  int64_t lo = 0, n = 0;
  for (int r = 0; r < a.R; ++r) {
    const int64_t rl = a.rank_off[r * a.U], rn = a.rank_off[r * a.U + a.U] - rl;
    const int tiles = (int)((rn + kRunTile - 1) / kRunTile);
    if (b < tiles) {
      rep = r;
      lo = rl;
      n = rn;
      break;
    }
    b -= tiles;
  }
  if (rep < 0) return;
  const int64_t t0 = (int64_t)b * kRunTile;
  const int cnt = (int)(n - t0 < kRunTile ? n - t0 : kRunTile);
  uint64_t* s_hi = reinterpret_cast<uint64_t*>(smem);
  uint64_t* s_lo = s_hi + kSortTile;
  uint32_t* s_v = reinterpret_cast<uint32_t*>(s_lo + kSortTile);
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const double wv = a.w[lo + t0 + i];
    s_hi[i] = ~(uint64_t)__double_as_longlong(wv == 0.0 ? 0.0 : wv);  // -0.0 ties +0.0
    s_lo[i] = a.ids[lo + t0 + i];
    s_v[i] = (uint32_t)(t0 + i);
  }
  __syncthreads();
  // register bitonic (block_sort.cuh), unrolled for the tile's power of two
  int tile = 64;
  while (tile < cnt) tile <<= 1;
  const int64_t base = lo + t0;
  switch (tile) {
    case 64: sort_tile_out<64, 1>(a, s_hi, s_lo, s_v, cnt, base); break;
    case 128: sort_tile_out<128, 1>(a, s_hi, s_lo, s_v, cnt, base); break;
    case 256: sort_tile_out<256, 1>(a, s_hi, s_lo, s_v, cnt, base); break;
    default: sort_tile_out<512, 1>(a, s_hi, s_lo, s_v, cnt, base); break;
  }
}

// One merge level: runs of `width` records (replica-relative) pairwise.
__global__ void __launch_bounds__(256) k_merge_pass(PlanArgs a, int64_t width, const uint64_t* __restrict__ shi,
                                                    const uint64_t* __restrict__ slo, const uint32_t* __restrict__ sv,
                                                    uint64_t* dhi, uint64_t* dlo, uint32_t* dv) {
  if (!seqs_ok(a)) return;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.rank_off[a.W]) return;
  const int rep = replica_of(a, g);
  const int64_t lo = a.rank_off[rep * a.U], n = a.rank_off[rep * a.U + a.U] - lo;
  const int64_t d = g - lo, run = d / width, base = run * width, pbase = (run ^ 1) * width;
  const uint64_t kh = shi[g], kl = slo[g];
  const uint32_t kv = sv[g];
  int64_t plen = n - pbase;
  plen = plen < 0 ? 0 : (plen > width ? width : plen);
  int64_t c = 0;  // partner records ordered before this one
  if (plen > 0) {
    int64_t l = 0, h = plen;
    const int64_t p0 = lo + pbase;
    while (l < h) {
      const int64_t m = (l + h) >> 1;
      if (rec_less(shi[p0 + m], slo[p0 + m], sv[p0 + m], kh, kl, kv)) l = m + 1;
      else h = m;
    }
    c = l;
  }
  const int64_t out = lo + (base < pbase ? base : pbase) + (d - base) + c;
  dhi[out] = kh;
  dlo[out] = kl;
  dv[out] = kv;
}

// All merge levels in one pass: a record's place in the replica's order is
// its index in its own 512-record run plus, for every other run, the number
// of that run's records ordered before it (the order is total, so the places
// are a permutation).  One thread per record; the binary searches over the
// other runs advance in lockstep, so each thread keeps one independent load
// per run in flight: ~10 dependent rounds in all instead of a dependent chain
// per merge level.  Replaces the k_merge_pass launches + k_sort_finish for
// replicas of up to kRankMergeMax records.  Measured on B200: 2K 27.8 -> 25.8
// us, 4K 38 -> 32 us; at 16K (32 runs) the divergent probes are L1-wavefront
// bound (320 probes x 3 loads per record) and the merge passes win (55 vs 81).
constexpr int64_t kRankMergeMax = 4096;

template <int G>
__global__ void __launch_bounds__(256) k_rank_merge(PlanArgs a) {
  if (!seqs_ok(a)) return;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.rank_off[a.W]) return;
  const int rep = replica_of(a, g);
  const int64_t lo = a.rank_off[rep * a.U], n = a.rank_off[rep * a.U + a.U] - lo;
  const int64_t d = g - lo;
  const int run = (int)(d / kRunTile), runs = (int)((n + kRunTile - 1) / kRunTile);
  const uint64_t kh = a.sk_hi[g], kl = a.sk_lo[g];
  const uint32_t kv = a.sk_v[g];
  const uint64_t* __restrict__ hi = a.sk_hi + lo;
  const uint64_t* __restrict__ lw = a.sk_lo + lo;
  const uint32_t* __restrict__ vv = a.sk_v + lo;
  int64_t rank = d - (int64_t)run * kRunTile;
  for (int r0 = 0; r0 < runs; r0 += G) {
    int l[G], h[G];
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const int r = r0 + k;
      const int64_t b = (int64_t)r * kRunTile;
      l[k] = 0;
      h[k] = (r < runs && r != run) ? (int)(n - b < kRunTile ? n - b : kRunTile) : 0;
    }
#pragma unroll
    for (int it = 0; it < 10; ++it) {  // ceil(log2(kRunTile + 1)) halvings
#pragma unroll
      for (int k = 0; k < G; ++k) {
        if (l[k] < h[k]) {
          const int m = (l[k] + h[k]) >> 1;
          const int64_t x = (int64_t)(r0 + k) * kRunTile + m;
          // the whole key at once: ties on the workload are common (equal
          // lengths), and a second dependent load would double the latency
          if (rec_less_bf(hi[x], lw[x], vv[x], kh, kl, kv)) l[k] = m + 1;
          else h[k] = m;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < G; ++k) rank += l[k];
  }
  const int64_t s = lo + kv;  // kv: replica-relative gather index
  a.sorted_idx[lo + rank] = (int32_t)s;
  a.sorted_w[lo + rank] = a.w[s];
}

__global__ void k_sort_finish(PlanArgs a, const uint32_t* __restrict__ sv) {
  if (!seqs_ok(a)) return;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.rank_off[a.W]) return;
  const int64_t lo = a.rank_off[replica_of(a, g) * a.U];
  const int64_t s = lo + sv[g];
  a.sorted_idx[g] = (int32_t)s;
  a.sorted_w[g] = a.w[s];
}

// Serial FP64 totals: per replica in gather order (balancer.cpp:24-25) and
// BalanceReport::total_workload over every replica (balancer.cpp:147).  One
// CTA per sum, computed by block_serial_sum (serial_sum.cuh): bit-identical
// to the one-thread DADD chain, ~log2(total / first) block scans instead of
// one ~8-cycle dependent add per sequence.  Workloads are recomputed from the
// lengths (bit-identical to k_prep_seq's), so the sums start with the plan.
// Runs on the planner's side stream, concurrently with the prep and the sort.
constexpr int kSumThreads = 512;  // measured: 512 beats 128 at 16K (fewer window restarts)
constexpr int kSumPerThread = 4;  // measured at 16K: 2 -> 55 us, 4 -> 47, 8 -> 48-52, 16 -> 59-70
constexpr int64_t kSumStage = 24576;  // workloads staged in shared memory (192 KB) up to this many

// Stage x_j = f(j), j < n, into dynamic shared memory when the launch gave
// room for them (every restart of block_serial_sum re-reads its window).
template <class F>
__device__ __forceinline__ bool sum_stage(double* stage, int64_t cap, int64_t n, F f) {
  if (n > cap) return false;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) stage[j] = f(j);
  __syncthreads();
  return true;
}

__global__ void __launch_bounds__(kSumThreads) k_totals(PlanArgs a, int64_t stage_cap) {
  extern __shared__ __align__(16) double stage[];
  if (!seqs_ok(a)) return;
  const int b = blockIdx.x;
  int64_t lo, hi;
  if (b < a.R) {
    lo = a.rank_off[b * a.U];
    hi = a.rank_off[b * a.U + a.U];
  } else {
    lo = 0;
    hi = a.rank_off[a.W];
  }
  auto f = [&](int64_t j) { return seq_workload(a, lo + j); };
  const bool st = sum_stage(stage, stage_cap, hi - lo, f);
  const double s = block_serial_sum<kSumThreads, kSumPerThread>(
      hi - lo, [&](int64_t j) { return st ? stage[j] : f(j); }, [](int64_t, double, double) {});
  if (threadIdx.x != 0) return;
  if (b < a.R) {
    a.rep_total[b] = s;
  } else {
    *a.total = s;
    *a.n_seqs = hi;
  }
}

// Large path: one warp per replica.  The sorted workloads stream through a
// two-chunk shared-memory ring: at the start of chunk k the warp loads chunk
// k+1 (coalesced, latency hidden under 1024 greedy steps), so the chain's
// three-step-ahead prefetch always hits shared memory.
// Replicas of up to kGreedyStage sequences are staged whole into dynamic
// shared memory first (k_greedy_staged: flat loop, 137 vs 158 cycles per
// sequence); larger ones stream through the ring.
constexpr int kGreedyStage = 24576;  // 192 KB of workloads

template <int BPL, bool QOUT = false>
__global__ void __launch_bounds__(32) k_greedy_staged(PlanArgs a) {
  extern __shared__ __align__(16) double stage_raw[];  // max_seqs + 6 doubles (+ max_seqs ints for QOUT)
  __shared__ __align__(8) uint64_t sbar;
  if (!seqs_ok(a)) return;
  const int rep = blockIdx.x, lane = threadIdx.x;
  const int64_t lo = a.rank_off[rep * a.U], hi = a.rank_off[rep * a.U + a.U];
  const int n = (int)(hi - lo);
  // greedy-order workloads into shared memory by bulk copy (one warp's
  // dependent load rounds took ~30 us at 16K sequences)
  const double* stage = stage_doubles_bulk(stage_raw, a.sorted_w + lo, n, &sbar);
  if (lane < 4) const_cast<double*>(stage)[n + lane] = 0.0;  // the unclamped prefetch reads 3 past the end
  __syncwarp();
  if constexpr (!QOUT) {
    greedy_warp<BPL, 0, false, true>(a, rep, n, a.rep_total[rep], [&](int p) { return stage[p]; }, [](int) {},
                                     a.pick + lo, nullptr, a.violations);
  } else {
    // hybrid path: the picks go to shared memory behind the workloads, then
    // one pass derives each position's rank inside its bag (the stable bag
    // partition, match_any per 32 positions) and writes both out coalesced.
    // Recording the rank inside the chain cost ~16 cycles per step.
    __shared__ int run[kMaxBags];
    int32_t* p_stage = reinterpret_cast<int32_t*>(stage_raw + a.max_seqs + 6);
    greedy_warp<BPL, 0, false, true>(a, rep, n, a.rep_total[rep], [&](int p) { return stage[p]; }, [](int) {},
                                     p_stage, nullptr, a.violations);
    for (int b = lane; b < a.M; b += 32) run[b] = 0;
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
    for (int p0 = 0; p0 < n; p0 += 32) {
      const int p = p0 + lane;
      const bool valid = p < n;
      const int b = valid ? p_stage[p] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      const int rank_in = __popc(peers & lt);
      const int base = valid ? run[b] : 0;
      __syncwarp();
      if (valid && rank_in == 0) run[b] = base + __popc(peers);
      __syncwarp();
      if (valid) {
        a.pick[lo + p] = b;
        a.greedy_q[lo + p] = base + rank_in;
      }
    }
  }
}

template <int BPL>
__global__ void __launch_bounds__(32) k_greedy(PlanArgs a) {
  __shared__ double ring[2][kGreedyChunk];
  if (!seqs_ok(a)) return;
  const int rep = blockIdx.x, lane = threadIdx.x;
  const int64_t lo = a.rank_off[rep * a.U], hi = a.rank_off[rep * a.U + a.U];
  const int n = (int)(hi - lo);
  const double* sw = a.sorted_w + lo;
  auto load = [&](int c) {
    const int b = c * kGreedyChunk;
    for (int i = lane; i < kGreedyChunk && b + i < n; i += 32) ring[c & 1][i] = sw[b + i];
  };
  auto hook = [&](int p0) {
    if (p0 == 0) load(0);
    load(p0 / kGreedyChunk + 1);
    __syncwarp();
  };
  greedy_warp<BPL, kGreedyChunk>(a, rep, n, a.rep_total[rep],
                   [&](int p) { return ring[(p / kGreedyChunk) & 1][p % kGreedyChunk]; }, hook, a.pick + lo,
                   nullptr, a.violations);
}

// More than kMaxBags bags per replica (up to kMaxBagsLarge): the same
// decision per step (balancer.cpp:44-62) without the register speculation --
// every lane walks its bags (j = lane, lane + 32, ...) in shared memory,
// forms key = (infeasible, bits(occupancy)) with the exact division, keeps the
// first minimum, and the warp takes the lexicographic (key, bag) minimum by
// three REDUX; the winner's lane adds the workload.  Same arithmetic as
// greedy_warp (occupancy_sel == __ddiv_rn, tests/test_gpu_parity.py), so the
// picks and the FP64 report are identical; ~BPL times slower per step.
__global__ void __launch_bounds__(32) k_greedy_many(PlanArgs a) {
  extern __shared__ __align__(16) double gm[];  // cap[M], asg[M], then cnt[M] (int)
  if (!seqs_ok(a)) return;
  const int rep = blockIdx.x, lane = threadIdx.x, M = a.M;
  double* cap = gm;
  double* asg = gm + M;
  int* cnt = reinterpret_cast<int*>(gm + 2 * M);
  const int64_t lo = a.rank_off[rep * a.U], hi = a.rank_off[rep * a.U + a.U];
  const int n = (int)(hi - lo);
  const double target = __ddiv_rn(a.rep_total[rep], (double)a.U);  // balancer.cpp:26
  for (int j = lane; j < M; j += 32) {
    cap[j] = __dmul_rn((double)a.bag_size[j], target);  // balancer.cpp:30
    asg[j] = 0.0;
    cnt[j] = 0;
  }
  __syncwarp();
  const double* sw = a.sorted_w + lo;
  int viol = 0;
  double w_next = n > 0 ? sw[0] : 0.0;
  for (int p = 0; p < n; ++p) {
    const double w = w_next;
    w_next = p + 1 < n ? sw[p + 1] : 0.0;  // prefetch under this step
    uint64_t best = ~0ull;
    uint32_t best_j = 0xffffffffu;
    for (int j = lane; j < M; j += 32) {
      const double o = occupancy(asg[j], cap[j]);
      const uint64_t key = greedy_key(__dsub_rn(cap[j], asg[j]) >= w, o);
      if (key < best) {  // strict: the lower bag of this lane keeps ties
        best = key;
        best_j = (uint32_t)j;
      }
    }
    const uint32_t khi = (uint32_t)(best >> 32), klo = (uint32_t)best;
    const uint32_t m1 = __reduce_min_sync(0xffffffffu, khi);
    const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
    const uint32_t pick = __reduce_min_sync(0xffffffffu, (khi == m1 && klo == m2) ? best_j : 0xffffffffu);
    viol += (int)(m1 >> 31);  // winner infeasible: fallback pick == capacity violation
    if ((int)(pick & 31u) == lane) {
      asg[pick] = __dadd_rn(asg[pick], w);
      cnt[pick] += 1;
    }
    if (lane == 0) a.pick[lo + p] = (int)pick;
    __syncwarp();
  }
  for (int j = lane; j < M; j += 32) {
    a.bag_count[rep * M + j] = cnt[j];
    a.per_bag_occ[rep * M + j] = occupancy(asg[j], cap[j]);  // balancer.cpp:170-175 (replay == greedy)
    const int g = a.bag_size[j];
    const double per = __ddiv_rn(asg[j], (double)g);  // balancer.cpp:199-202
    for (int k = 0; k < g; ++k) a.per_gpu[rep * a.U + a.bag_ranks[a.bag_off[j] + k]] = per;
  }
  if (lane == 0) atomicAdd(a.violations, viol);
}

// One bag per replica: the picks (all bag 0) and bag counts (replica sizes)
// are known before the serial FP64 prefix runs, so emission and the lists
// start at once while greedy_single_bag's chain runs on the side stream.
__global__ void __launch_bounds__(256) k_single_bag_fill(PlanArgs a) {
  if (!seqs_ok(a)) return;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < a.rank_off[a.W]) a.pick[p] = 0;
  if (p < a.R) a.bag_count[p] = (int32_t)(a.rank_off[p * a.U + a.U] - a.rank_off[p * a.U]);
}

// One bag per replica, large path: the occupancy replay (balancer.cpp:159-166)
// over the greedy order is a serial FP64 prefix of the sorted workloads;
// block_serial_sum yields every prefix exactly, so each sequence's
// `capacity - assigned >= w` test runs in parallel.  Outputs as greedy_warp.
__global__ void __launch_bounds__(kSumThreads) k_single_bag_chain(PlanArgs a, int64_t stage_cap) {
  extern __shared__ __align__(16) double stage[];
  __shared__ int s_viol;
  if (!seqs_ok(a)) return;
  const int rep = blockIdx.x;
  const int64_t lo = a.rank_off[rep * a.U], hi = a.rank_off[rep * a.U + a.U];
  const double target = __ddiv_rn(a.rep_total[rep], (double)a.U);  // balancer.cpp:26
  const int size = a.bag_size[0];
  const double cap = __dmul_rn((double)size, target);  // balancer.cpp:30
  if (threadIdx.x == 0) s_viol = 0;
  __syncthreads();
  int viol = 0;
  const double* sw = a.sorted_w + lo;
  const bool st = sum_stage(stage, stage_cap, hi - lo, [&](int64_t j) { return sw[j]; });
  const double asg = block_serial_sum<kSumThreads, kSumPerThread>(
      hi - lo, [&](int64_t j) { return st ? stage[j] : sw[j]; },
      [&](int64_t, double before, double w) { viol += __dsub_rn(cap, before) >= w ? 0 : 1; });
  viol = __reduce_add_sync(0xffffffffu, viol);
  if ((threadIdx.x & 31) == 0 && viol) atomicAdd(&s_viol, viol);
  __syncthreads();
  if (threadIdx.x != 0) return;
  a.per_bag_occ[rep] = occupancy(asg, cap);  // balancer.cpp:170-175
  const double per = __ddiv_rn(asg, (double)size);  // balancer.cpp:199-202
  for (int k = 0; k < size; ++k) a.per_gpu[rep * a.U + a.bag_ranks[a.bag_off[0] + k]] = per;
  if (s_viol) atomicAdd(a.violations, s_viol);
}

// Self-test of block_serial_sum against the one-thread chain: block b sums
// len_b generated values (mode picks the law: reals, integers and halves --
// frequent round-half-even ties --, zeros over 120 binades, workloads,
// power-of-two tie patterns, overflow to +inf) and checks the result and
// every emitted prefix bit-for-bit.
__device__ __forceinline__ double selftest_value(uint64_t seed, int mode, int b, int64_t j) {
  const uint64_t r = splitmix64(seed ^ ((uint64_t)b << 40) ^ (uint64_t)j);
  switch (mode) {
    case 0: return (double)(r >> 11) * 0x1.0p-53 * 1e15;
    case 1: return (double)(r % 1000000007ull);
    case 2: return (double)(r % 4096) * 0.5;
    case 3: return (r & 3) == 0 ? 0.0 : ldexp((double)(r >> 11) * 0x1.0p-53, (int)((r >> 3) % 120) - 60);
    case 4: {
      const double l = 64.0 + (double)(r % 4096);
      return __dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(24.0, l), 3072.0), 3072.0),
                       __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(0.49, 4.0), l), l), 3072.0));
    }
    case 5: return j < 5 ? 0.0 : ldexp(1.0, (int)(r % 40)) + (((r >> 20) & 1) ? ldexp(1.0, (int)(r % 40) - 53) : 0.0);
    default: return (r & 1) ? 1e300 * (double)((r >> 1) % 3) : 1.0;
  }
}

__global__ void __launch_bounds__(kSumThreads) k_selftest_sum(uint64_t seed, int mode, int64_t max_len,
                                                              double* prefix, unsigned long long* mismatches) {
  const int b = blockIdx.x;
  const int64_t n = 1 + (int64_t)(splitmix64(seed ^ 0xabcdefull ^ (uint64_t)b) % (uint64_t)max_len);
  double* pre = prefix + (int64_t)b * max_len;
  const double s = block_serial_sum<kSumThreads, kSumPerThread>(
      n, [&](int64_t j) { return selftest_value(seed, mode, b, j); },
      [&](int64_t j, double before, double) { pre[j] = before; });
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long bad = 0;
  double t = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    if (__double_as_longlong(pre[j]) != __double_as_longlong(t)) ++bad;
    t = __dadd_rn(t, selftest_value(seed, mode, b, j));
  }
  if (__double_as_longlong(s) != __double_as_longlong(t)) ++bad;
  if (bad) atomicAdd(mismatches, bad);
}

// ------------------------------------------------------------------ k_emit
// balancer.cpp:178-218.  Sequences of bag b in assignment order get index q
// (a stable partition of the greedy order by bag); chunk k of (b, q) is
// global chunk rep_base + bag_base[b] + q*G_b + k and targets the bag's k-th
// rank.

// Phase A1 (grid: tiles of kEmitTile greedy positions x replicas): per-tile
// bag counts of the picks.
constexpr int kEmitTile = 1024;

__global__ void __launch_bounds__(kEmitTile) k_emit_count(PlanArgs a) {
  extern __shared__ int cnt[];  // M counters
  if (!seqs_ok(a)) return;
  const int rep = blockIdx.y, tile = blockIdx.x;
  const int64_t lo = a.rank_off[rep * a.U], hi = a.rank_off[rep * a.U + a.U];
  if (tile == 0 && threadIdx.x == 0) {  // the replica's (bag -> first chunk, first bag_seq slot) bases
    int64_t c = 0, sq = lo;
    for (int b = 0; b < a.M; ++b) {
      const int64_t nb = a.bag_count[rep * a.M + b];
      a.bag_cbase[rep * a.M + b] = c;
      a.bag_sbase[rep * a.M + b] = sq;
      c += nb * a.bag_size[b];
      sq += nb;
    }
    a.rep_chunks[rep] = c;
  }
  const int64_t p0 = lo + (int64_t)tile * kEmitTile;
  if (p0 >= hi) return;
  for (int b = threadIdx.x; b < a.M; b += blockDim.x) cnt[b] = 0;
  __syncthreads();
  const int64_t p = p0 + threadIdx.x;
  if (p < hi) atomicAdd(&cnt[a.pick[p]], 1);
  __syncthreads();
  for (int b = threadIdx.x; b < a.M; b += blockDim.x)
    a.tile_cnt[((int64_t)rep * gridDim.x + tile) * a.M + b] = cnt[b];
}

// Phase A2 (same grid): q = rank of each pick among its bag's picks in
// greedy order -- a stable bag partition (balancer.cpp:178-218): earlier
// tiles' counts + match_any / per-warp counts inside the tile; then the
// per-sequence fields and the inverse map bag_seq[(bag, q)] = s that lets
// phase B emit chunks in parallel.
__global__ void __launch_bounds__(kEmitTile) k_emit(PlanArgs a) {
  extern __shared__ int wc[];  // per-warp bag counts: [kEmitTile / 32][M]
  auto warp_cnt = [&](int w, int b) -> int& { return wc[w * a.M + b]; };
  __shared__ int64_t rep_base;
  if (!seqs_ok(a)) return;
  const int rep = blockIdx.y, tile = blockIdx.x;
  const int64_t lo = a.rank_off[rep * a.U], hi = a.rank_off[rep * a.U + a.U];
  if (threadIdx.x == 0) {  // chunks of earlier replicas (rep_chunks from k_emit_count)
    int64_t acc = 0;
    for (int r = 0; r < rep; ++r) acc += a.rep_chunks[r];
    rep_base = acc;
    if (tile == 0) {  // also for empty replicas
      a.rep_cbase[rep] = acc;
      if (rep == a.R - 1) a.rep_cbase[a.R] = acc + a.rep_chunks[rep];
    }
  }
  const int64_t p0 = lo + (int64_t)tile * kEmitTile;
  if (p0 >= hi) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t p = p0 + tid;
  const bool valid = p < hi;
  const int b = valid ? a.pick[p] : -1;
  const unsigned peers = __match_any_sync(0xffffffffu, b);
  const int rank_in = __popc(peers & ((1u << lane) - 1u));
  for (int e = tid; e < (kEmitTile / 32) * a.M; e += blockDim.x) wc[e] = 0;
  __syncthreads();
  if (valid && rank_in == 0) warp_cnt(warp, b) = __popc(peers);
  __syncthreads();
  for (int bb = tid; bb < a.M; bb += blockDim.x) {  // exclusive prefix over earlier tiles, then over this tile's warps
    int run = 0;
    const int* tc = a.tile_cnt + (int64_t)rep * gridDim.x * a.M + bb;
    for (int t = 0; t < tile; ++t) run += tc[(int64_t)t * a.M];
    for (int w = 0; w < kEmitTile / 32; ++w) {
      const int c = warp_cnt(w, bb);
      warp_cnt(w, bb) = run;
      run += c;
    }
  }
  __syncthreads();
  if (!valid) return;
  const int q = warp_cnt(warp, b) + rank_in;
  const int s = a.sorted_idx[p];
  const int g = a.bag_size[b];
  a.bag_seq[a.bag_sbase[rep * a.M + b] + q] = s;
  a.seq_bag[s] = b;
  a.seq_G[s] = g;
  a.seq_chunk_base[s] = rep_base + a.bag_cbase[rep * a.M + b] + (int64_t)q * g;
  atomicAdd(&a.send_count[a.seq_rank[s]], (unsigned long long)g);
}

// Phase B (grid over chunk capacity): chunk c = (replica, bag b, q, k) ->
// sequence bag_seq[(b, q)]; every field written coalesced across threads
// (balancer.cpp:178-218 chunk emission).
__global__ void __launch_bounds__(256) k_emit_chunks(PlanArgs a) {
  if (!seqs_ok(a)) return;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.rep_cbase[a.R]) return;
  int rep = 0;
  {
    int l = 0, h = a.R;  // rep_cbase[l] <= c < rep_cbase[h]
    while (h - l > 1) {
      const int m = (l + h) >> 1;
      if (a.rep_cbase[m] <= c) l = m;
      else h = m;
    }
    rep = l;
  }
  int64_t rel = c - a.rep_cbase[rep];
  int b = 0;
  {
    // last bag whose replica-local chunk base is <= rel (an empty bag shares
    // its base with the next bag, so the search lands on the non-empty one)
    const int64_t* cbase = a.bag_cbase + (int64_t)rep * a.M;
    int l = 0, h = a.M;
    while (h - l > 1) {
      const int m = (l + h) >> 1;
      if (cbase[m] <= rel) l = m;
      else h = m;
    }
    b = l;
    rel -= cbase[b];
  }
  const int64_t sq = a.bag_sbase[rep * a.M + b];
  const int g = a.bag_size[b];
  const int64_t q = rel / g;
  const int k = (int)(rel - q * g);
  const int s = a.bag_seq[sq + q];
  const int64_t l = a.lens[s] < 0 ? 0 : a.lens[s];
  const int64_t st = chunk_start(l, g, k);
  a.c_id[c] = a.ids[s];
  a.c_idx[c] = k;
  a.c_start[c] = st;
  a.c_end[c] = st + chunk_len(l, g, k);
  a.c_src[c] = a.seq_rank[s];
  a.c_dst[c] = rep * a.U + a.bag_ranks[a.bag_off[b] + k];
  a.c_src_row[c] = a.seq_off[s] + st;
  a.c_seq[c] = s;
}

// reverse_plan's receive order for rank r (balancer.cpp:259-285) when its
// (segment, start) keys can tie -- a sequence shorter than its bag leaves
// several empty chunks at the same start.  Our O(C) order breaks ties by
// chunk index; the reference's std::sort breaks them however introsort
// happens to, so replay libstdc++'s algorithm on its input (the incoming
// chunks in index order == send[r]) with its comparator.  Single thread;
// lists of <= 16 entries are already identical (insertion sort is stable).
__device__ void fix_rev_ties(int32_t* rev_recv_idx, const int32_t* send_idx, const int32_t* seq, const int64_t* st,
                             int64_t off, int64_t n, stdsort::Frame* stack) {
  if (n <= stdsort::kThreshold) return;
  for (int64_t i = 0; i < n; ++i) rev_recv_idx[off + i] = send_idx[off + i];
  stdsort::sort(
      rev_recv_idx + off, n,
      [&](int32_t x, int32_t y) {
        if (seq[x] != seq[y]) return seq[x] < seq[y];
        return st[x] < st[y];
      },
      stack);
}

// ----------------------------------------------------------------- k_lists
// Per global rank r (grid: tiles of kListTile elements x ranks), four
// scans over r's domains:
//   recv[r]      = chunks (q, k) of r's bag member slot k, q ascending
//                  (finalize_manifests, balancer.cpp:84-91), plus the
//                  receive-side row offsets (target packing, :93-101);
//   c_seq_base   = row base of each sequence in its bag's full-sequence
//                  layout (member 0 only; pre_attn shells, exchange.cpp:291-295);
//   send[r]      = chunks with source r in chunk order: r's sequences sorted
//                  by their first chunk index, each expanded to G chunks --
//                  a stable filter of bag_seq (chunk order is (replica, bag,
//                  q, k)) by source rank;
//   rev_recv[r]  = reverse_plan's receive order (:259-285): r's sequences in
//                  buffer order, chunks by start (chunk index breaks the
//                  zero-length ties; libstdc++'s order replayed by k_finalize).
// k_lists_count sums each tile of each domain (and the rank offsets),
// k_lists adds the earlier tiles' sums to an in-tile block scan.
constexpr int kListTile = 1024;

struct ListDomains {
  int rep, b, k, g, n_b;
  int64_t cb0, rlo, rhi, lo, hi;
};

__device__ __forceinline__ ListDomains list_domains(const PlanArgs& a, int r) {
  ListDomains d;
  d.rep = r / a.U;
  const int u = r % a.U;
  d.b = a.rank_bag[u];
  d.k = a.rank_member[u];
  d.g = a.bag_size[d.b];
  d.n_b = a.bag_count[d.rep * a.M + d.b];
  d.cb0 = a.rep_cbase[d.rep] + a.bag_cbase[d.rep * a.M + d.b];
  d.rlo = a.rank_off[d.rep * a.U];
  d.rhi = a.rank_off[d.rep * a.U + a.U];
  d.lo = a.rank_off[r];
  d.hi = a.rank_off[r + 1];
  return d;
}

// The four per-element values of domain position o (0 when out of range).
__device__ __forceinline__ void list_values(const PlanArgs& a, const ListDomains& d, int r, int64_t o, int64_t v[4]) {
  v[0] = v[1] = v[2] = v[3] = 0;
  if (o < d.n_b) {
    const int64_t c = d.cb0 + o * d.g + d.k;
    v[0] = a.c_end[c] - a.c_start[c];
    if (d.k == 0) v[1] = a.c_end[c + d.g - 1];  // the last chunk ends at the sequence length
  }
  if (d.rlo + o < d.rhi) {
    const int s = a.bag_seq[d.rlo + o];
    v[2] = a.seq_rank[s] == r ? a.seq_G[s] : 0;
  }
  if (d.lo + o < d.hi) v[3] = a.seq_G[d.lo + o];
}

__global__ void __launch_bounds__(kListTile) k_lists_count(PlanArgs a) {
  __shared__ int64_t part[kListTile / 32][4];
  if (!seqs_ok(a)) return;
  const int r = blockIdx.y, t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const ListDomains d = list_domains(a, r);
  if (t == 0 && tid == 0) {  // manifest offsets (balancer.cpp:84-91)
    int64_t ro = 0, so = 0;
    for (int x = 0; x < r; ++x) {
      ro += a.bag_count[(x / a.U) * a.M + a.rank_bag[x % a.U]];
      so += (int64_t)a.send_count[x];
    }
    a.recv_off[r] = ro;
    a.send_off[r] = so;
    if (r == a.W - 1) {
      a.recv_off[a.W] = ro + d.n_b;
      a.send_off[a.W] = so + (int64_t)a.send_count[r];
    }
    a.list_tie[r] = 0;
  }
  const int64_t o0 = (int64_t)t * kListTile;
  if (o0 >= d.n_b && d.rlo + o0 >= d.rhi && d.lo + o0 >= d.hi) {
    // empty tile of this rank: its sums are zero (k_lists adds every tile's,
    // and the buffer may hold a previous plan's)
    if (tid < 4) a.list_sum[((int64_t)r * gridDim.x + t) * 4 + tid] = 0;
    return;
  }
  int64_t v[4];
  list_values(a, d, r, o0 + tid, v);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int64_t x = v[j];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) part[warp][j] = x;
  }
  __syncthreads();
  if (tid < 4) {
    int64_t x = 0;
    for (int w = 0; w < kListTile / 32; ++w) x += part[w][tid];
    a.list_sum[((int64_t)r * gridDim.x + t) * 4 + tid] = x;
  }
}

__global__ void __launch_bounds__(kListTile) k_lists(PlanArgs a) {
  __shared__ int64_t sh[33];
  __shared__ int64_t base[4];
  if (!seqs_ok(a)) return;
  const int r = blockIdx.y, t = blockIdx.x, tid = threadIdx.x;
  const int T = gridDim.x;
  const ListDomains d = list_domains(a, r);
  const int64_t* ts = a.list_sum + (int64_t)r * T * 4;
  if (t == 0 && tid == 32) {  // totals: target rows of r, full rows of its bag
    int64_t tr = 0, br = 0;
    for (int x = 0; x < T; ++x) {
      tr += ts[x * 4 + 0];
      br += ts[x * 4 + 1];
    }
    a.target_rows[r] = tr;
    if (d.k == 0) a.bag_rows[d.rep * a.M + d.b] = br;
  }
  const int64_t o0 = (int64_t)t * kListTile;
  if (o0 >= d.n_b && d.rlo + o0 >= d.rhi && d.lo + o0 >= d.hi) return;
  if (tid < 4) {
    int64_t x = 0;
    for (int y = 0; y < t; ++y) x += ts[y * 4 + tid];
    base[tid] = x;
  }
  const int64_t recv_off = a.recv_off[r], send_off = a.send_off[r];
  const int64_t o = o0 + tid;
  int64_t v[4];
  list_values(a, d, r, o, v);
  int64_t tot;
  __syncthreads();  // base
  if (o0 < d.n_b) {  // recv list + target rows
    const int64_t ex = block_excl_scan<int64_t>(v[0], sh, &tot);
    if (o < d.n_b) {
      const int64_t c = d.cb0 + o * d.g + d.k;
      a.c_dst_row[c] = base[0] + ex;
      a.recv_idx[recv_off + o] = (int32_t)c;
    }
    if (d.k == 0) {  // Ulysses: per-sequence base rows in the bag's full layout
      const int64_t ex1 = block_excl_scan<int64_t>(v[1], sh, &tot);
      if (o < d.n_b) a.c_seq_base[d.cb0 + o * d.g] = base[1] + ex1;
    }
  }
  if (d.rlo + o0 < d.rhi) {  // send list
    const int64_t ex = block_excl_scan<int64_t>(v[2], sh, &tot);
    if (v[2] > 0) {
      const int64_t cb = a.seq_chunk_base[a.bag_seq[d.rlo + o]];
      for (int kk = 0; kk < (int)v[2]; ++kk) a.send_idx[send_off + base[2] + ex + kk] = (int32_t)(cb + kk);
    }
  }
  if (d.lo + o0 < d.hi) {  // reverse receive order: sequences in buffer order, chunks ascending
    const int64_t ex = block_excl_scan<int64_t>(v[3], sh, &tot);
    int tie = 0;  // a sequence shorter than its bag: empty chunks with equal (segment, start)
    if (d.lo + o < d.hi) {
      const int gs = (int)v[3];
      tie = (gs > 1 && a.lens[d.lo + o] < gs) ? 1 : 0;
      const int64_t cb = a.seq_chunk_base[d.lo + o];
      for (int kk = 0; kk < gs; ++kk) a.rev_recv_idx[send_off + base[3] + ex + kk] = (int32_t)(cb + kk);
    }
    tie = __syncthreads_or(tie);
    if (tid == 0 && tie) atomicOr(&a.list_tie[r], 1);
  }
}


// -------------------------------------------------------------- k_finalize
__global__ void k_finalize(PlanArgs a) {
  if (!seqs_ok(a)) return;
  if (threadIdx.x == 0) {
    int64_t c = 0;
    for (int r = 0; r < a.R; ++r) c += a.rep_chunks[r];
    *a.n_chunks = c;
    // workload_imbalance_ratio (metrics.cpp:20-31)
    double lo = a.per_gpu[0], hi = a.per_gpu[0];
    for (int r = 0; r < a.W; ++r) {
      lo = fmin(lo, a.per_gpu[r]);
      hi = fmax(hi, a.per_gpu[r]);
    }
    double wir;
    if (hi == 0.0) wir = 1.0;
    else if (lo == 0.0) wir = __longlong_as_double(0x7ff0000000000000ll);
    else wir = __ddiv_rn(hi, lo);
    *a.wir = wir;
  }
  // ranks whose reverse receive order can tie: replay std::sort now that
  // send[r] (its input order) is complete; one lane per rank
  for (int r = threadIdx.x; r < a.W; r += blockDim.x)
    if (a.list_tie[r]) {
      stdsort::Frame stk[stdsort::kStackFrames];
      fix_rev_ties(a.rev_recv_idx, a.send_idx, a.c_seq, a.c_start, a.send_off[r], a.send_off[r + 1] - a.send_off[r],
                   stk);
    }
}

}  // namespace sb
#include "planner_small.cuh"
namespace sb {

// ------------------------------------------------ generic plan manifests
// For plans that did not come from k_emit (uploaded RoutingPlans):
// finalize_manifests (balancer.cpp:84-91) as ordered compactions by source
// and target rank, and reverse_plan's receive order (balancer.cpp:259-285):
// each incoming chunk's first containing segment in the origin layout, then
// a sort by (segment, start, chunk index).
struct GenericArgs {
  int W;
  const int64_t* n_chunks;
  const uint64_t* c_id;
  const int32_t *c_src, *c_dst;
  const int64_t *c_start, *c_end;
  const int64_t* seg_off;
  const uint64_t* seg_id;
  const int64_t *seg_first, *seg_len;
  unsigned long long *send_count, *recv_count;
  int64_t *send_off, *recv_off;
  int32_t *send_idx, *recv_idx, *rev_recv_idx;
  uint64_t *ck_hi, *ck_lo, *ck_thi, *ck_tlo;
  uint32_t *ck_v, *ck_tv;
  int32_t* status;
};

__global__ void k_generic_count(GenericArgs a) {
  const int64_t n = *a.n_chunks;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(&a.send_count[a.c_src[c]], 1ull);
    atomicAdd(&a.recv_count[a.c_dst[c]], 1ull);
  }
}

__global__ void __launch_bounds__(1024) k_generic_lists(GenericArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t sh[33];
  __shared__ int64_t s_so, s_ro;
  const int r = blockIdx.x, tid = threadIdx.x;
  const int64_t n = *a.n_chunks;
  if (tid == 0) {
    int64_t so = 0, ro = 0;
    for (int x = 0; x < r; ++x) {
      so += (int64_t)a.send_count[x];
      ro += (int64_t)a.recv_count[x];
    }
    s_so = so;
    s_ro = ro;
    a.send_off[r] = so;
    a.recv_off[r] = ro;
    if (r == a.W - 1) {
      a.send_off[a.W] = so + (int64_t)a.send_count[r];
      a.recv_off[a.W] = ro + (int64_t)a.recv_count[r];
    }
  }
  __syncthreads();
  int64_t cs = 0, cr = 0;
  for (int64_t t0 = 0; t0 < n; t0 += blockDim.x) {
    const int64_t c = t0 + tid;
    const bool fs = c < n && a.c_src[c] == r;
    const bool fr = c < n && a.c_dst[c] == r;
    int64_t ts, tr;
    const int64_t es = block_excl_scan<int64_t>(fs ? 1 : 0, sh, &ts);
    const int64_t er = block_excl_scan<int64_t>(fr ? 1 : 0, sh, &tr);
    if (fs) a.send_idx[s_so + cs + es] = (int32_t)c;
    if (fr) a.recv_idx[s_ro + cr + er] = (int32_t)c;
    cs += ts;
    cr += tr;
  }
  __syncthreads();
  // reverse receive order of rank r: its outgoing chunks, keyed by the
  // first origin segment containing them (balancer.cpp:267-277)
  const int64_t s0 = a.seg_off[r], s1 = a.seg_off[r + 1];
  for (int64_t i = tid; i < cs; i += blockDim.x) {
    const int32_t c = a.send_idx[s_so + i];
    int64_t seg = -1;
    for (int64_t q = s0; q < s1; ++q) {
      if (a.seg_id[q] == a.c_id[c] && a.c_start[c] >= a.seg_first[q] &&
          a.c_end[c] <= a.seg_first[q] + a.seg_len[q]) {
        seg = q - s0;
        break;
      }
    }
    if (seg < 0) atomicOr(a.status, 32);
    a.ck_hi[c] = (uint64_t)(seg < 0 ? 0 : seg);  // per chunk id: the comparator's segment
    a.rev_recv_idx[s_so + i] = c;                // std::sort's input: incoming in chunk order
  }
  __syncthreads();
  // balancer.cpp:278-283: the reference's std::sort on (segment, start),
  // replayed exactly (stdsort.cuh) so tied keys land where libstdc++ puts them
  if (tid == 0) {
    const uint64_t* seg = a.ck_hi;
    const int64_t* st = a.c_start;
    stdsort::Frame stk[stdsort::kStackFrames];
    stdsort::sort(a.rev_recv_idx + s_so, cs, [&](int32_t x, int32_t y) {
      if (seg[x] != seg[y]) return seg[x] < seg[y];
      return st[x] < st[y];
    }, stk);
  }
  (void)smem;
}

// -------------------------------------------------------- identity kernels
// identity_plan (balancer.cpp:227-240): chunk i = sequence i, src = dst.
__global__ void k_identity(PlanArgs a) {
  if (!seqs_ok(a)) return;
  const int64_t n = a.rank_off[a.W];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = a.lens[i] < 0 ? 0 : a.lens[i];
    const int r = a.seq_rank[i];
    a.c_id[i] = a.ids[i];
    a.c_idx[i] = 0;
    a.c_start[i] = 0;
    a.c_end[i] = l;
    a.c_src[i] = r;
    a.c_dst[i] = r;
    a.c_src_row[i] = a.seq_off[i];
    a.c_seq[i] = (int32_t)i;
    a.c_dst_row[i] = a.seq_off[i];
    a.send_idx[i] = (int32_t)i;
    a.recv_idx[i] = (int32_t)i;
    a.rev_recv_idx[i] = (int32_t)i;
    a.seq_G[i] = 1;
    a.seq_chunk_base[i] = i;
  }
  if (blockIdx.x == 0) {
    for (int r = threadIdx.x; r <= a.W; r += blockDim.x) {
      a.send_off[r] = a.rank_off[r];
      a.recv_off[r] = a.rank_off[r];
      if (r < a.W) a.target_rows[r] = a.origin_rows[r];
    }
  }
}

// Report for the no-balancer case, as simulator.cpp:76-86 computes it:
// per-rank sums in gather order, then WIR.
__global__ void k_identity_report(PlanArgs a) {
  if (!seqs_ok(a)) return;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < a.W) {
    double s = 0.0;
    for (int64_t i = a.rank_off[r]; i < a.rank_off[r + 1]; ++i) s = __dadd_rn(s, a.w[i]);
    a.per_gpu[r] = s;
  }
}

__global__ void k_identity_finalize(PlanArgs a) {
  if (!seqs_ok(a)) return;
  if (threadIdx.x == 0) {
    *a.n_chunks = a.rank_off[a.W];
    double lo = a.per_gpu[0], hi = a.per_gpu[0];
    for (int r = 0; r < a.W; ++r) {
      lo = fmin(lo, a.per_gpu[r]);
      hi = fmax(hi, a.per_gpu[r]);
    }
    *a.wir = hi == 0.0 ? 1.0 : (lo == 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : __ddiv_rn(hi, lo));
  }
}

// ------------------------------------------------------------------ host
template <typename T>
static void dalloc(T** p, int64_t n) {
  SB_CUDA(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (size_t)(n > 0 ? n : 1)));
}

static PlanArgs make_args(sb_planner* p) {
  PlanArgs a;
  a.W = p->W; a.U = p->U; a.M = p->M; a.R = p->R;
  a.d_model = (double)p->d_model; a.gamma = p->gamma; a.max_seqs = p->max_seqs;
  a.bag_off = p->d_bag_off; a.bag_ranks = p->d_bag_ranks; a.bag_size = p->d_bag_size;
  a.rank_bag = p->d_rank_bag; a.rank_member = p->d_rank_member;
  a.ids = p->ids; a.lens = p->lens; a.rank_off = p->rank_off; a.w_in = p->w_in;
  a.w = p->w; a.seq_rank = p->seq_rank; a.seq_off = p->seq_off; a.hash = p->hash;
  a.sk_hi = p->sk_hi; a.sk_lo = p->sk_lo; a.tk_hi = p->tk_hi; a.tk_lo = p->tk_lo;
  a.sk_v = p->sk_v; a.tk_v = p->tk_v;
  a.sorted_w = p->sorted_w; a.sorted_idx = p->sorted_idx; a.pick = p->pick;
  a.seq_bag = p->seq_bag; a.seq_G = p->seq_G; a.seq_chunk_base = p->seq_chunk_base;
  a.greedy_q = p->greedy_q;
  a.rep_total = p->rep_total; a.sentinel = p->sentinel; a.bag_count = p->bag_count;
  a.bag_rows = p->bag_rows; a.rep_chunks = p->rep_chunks; a.send_count = p->send_count;
  a.rep_cbase = p->rep_cbase; a.bag_seq = p->bag_seq;
  a.tile_cnt = p->tile_cnt; a.list_sum = p->list_sum; a.list_tie = p->list_tie; a.bag_cbase = p->bag_cbase; a.bag_sbase = p->bag_sbase;
  a.n_chunks = p->n_chunks; a.n_seqs = p->n_seqs;
  a.c_id = p->c_id; a.c_idx = p->c_idx; a.c_src = p->c_src; a.c_dst = p->c_dst;
  a.c_start = p->c_start; a.c_end = p->c_end; a.c_src_row = p->c_src_row; a.c_dst_row = p->c_dst_row;
  a.c_seq_base = p->c_seq_base;
  a.c_seq = p->c_seq;
  a.send_off = p->send_off; a.recv_off = p->recv_off; a.send_idx = p->send_idx;
  a.recv_idx = p->recv_idx; a.rev_recv_idx = p->rev_recv_idx;
  a.origin_rows = p->origin_rows; a.target_rows = p->target_rows;
  a.per_gpu = p->per_gpu; a.per_bag_occ = p->per_bag_occ; a.total = p->total; a.wir = p->wir;
  a.violations = p->violations; a.status = p->status;
  a.trace = p->trace;
  return a;
}

static void planner_alloc(sb_planner* p) {
  const int64_t N = p->max_seqs, C = p->max_chunks, W = p->W, R = p->R, M = p->M;
  SB_CUDA(cudaHostAlloc(&p->h_small, 4 * sizeof(int64_t), cudaHostAllocDefault));
  dalloc(&p->d_bag_off, M + 1); dalloc(&p->d_bag_ranks, p->U); dalloc(&p->d_bag_size, M);
  dalloc(&p->d_rank_bag, p->U); dalloc(&p->d_rank_member, p->U);
  dalloc(&p->w, N); dalloc(&p->seq_rank, N); dalloc(&p->seq_off, N); dalloc(&p->hash, 2 * N);
  dalloc(&p->sk_hi, N); dalloc(&p->sk_lo, N); dalloc(&p->tk_hi, N); dalloc(&p->tk_lo, N);
  dalloc(&p->sk_v, N); dalloc(&p->tk_v, N);
  dalloc(&p->sorted_w, N + 2);  // + bulk-copy alignment slack (k_greedy_staged)
  dalloc(&p->sorted_idx, N); dalloc(&p->pick, N);
  dalloc(&p->seq_bag, N); dalloc(&p->seq_G, N); dalloc(&p->seq_chunk_base, N); dalloc(&p->greedy_q, N);
  dalloc(&p->rep_total, R); dalloc(&p->sentinel, R); dalloc(&p->bag_count, R * M);
  dalloc(&p->bag_rows, R * M); dalloc(&p->rep_chunks, R); dalloc(&p->send_count, W);
  dalloc(&p->rep_cbase, R + 1); dalloc(&p->bag_seq, N);
  dalloc(&p->tile_cnt, R * ((N + 1023) / 1024) * M); dalloc(&p->list_sum, W * ((N + 1023) / 1024) * 4);
  dalloc(&p->list_tie, W); dalloc(&p->bag_cbase, R * M); dalloc(&p->bag_sbase, R * M);
  dalloc(&p->recv_count, W);
  dalloc(&p->n_chunks, 1); dalloc(&p->n_seqs, 1);
  dalloc(&p->c_id, C); dalloc(&p->c_idx, C); dalloc(&p->c_src, C); dalloc(&p->c_dst, C);
  dalloc(&p->c_start, C); dalloc(&p->c_end, C); dalloc(&p->c_src_row, C); dalloc(&p->c_dst_row, C);
  dalloc(&p->c_seq_base, C);
  dalloc(&p->c_seq, C);
  dalloc(&p->send_off, W + 1); dalloc(&p->recv_off, W + 1);
  dalloc(&p->send_idx, C); dalloc(&p->recv_idx, C); dalloc(&p->rev_recv_idx, C);
  dalloc(&p->origin_rows, W); dalloc(&p->target_rows, W);
  dalloc(&p->per_gpu, W); dalloc(&p->per_bag_occ, R * M); dalloc(&p->total, 1); dalloc(&p->wir, 1);
  dalloc(&p->violations, 1); dalloc(&p->status, 1);
  SB_CUDA(cudaMemcpy(p->d_bag_off, p->bag_off.data(), sizeof(int32_t) * (M + 1), cudaMemcpyHostToDevice));
  SB_CUDA(cudaMemcpy(p->d_bag_ranks, p->bag_ranks.data(), sizeof(int32_t) * p->U, cudaMemcpyHostToDevice));
  SB_CUDA(cudaMemcpy(p->d_bag_size, p->bag_size.data(), sizeof(int32_t) * M, cudaMemcpyHostToDevice));
  SB_CUDA(cudaMemcpy(p->d_rank_bag, p->rank_bag.data(), sizeof(int32_t) * p->U, cudaMemcpyHostToDevice));
  SB_CUDA(cudaMemcpy(p->d_rank_member, p->rank_member.data(), sizeof(int32_t) * p->U, cudaMemcpyHostToDevice));
  SB_CUDA(cudaFuncSetAttribute(k_sort_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSortSmemBytes));
  if (p->max_seqs <= kSmallSeqs && p->W <= 1024) {
    p->small_smem = small_layout((int)p->max_seqs, p->W, p->R * p->M, p->R, p->U, p->M).total;
    static size_t set_to = 0;  // attribute is per function: keep the largest requested
    if (p->small_smem > set_to) {
      SB_CUDA(cudaFuncSetAttribute(k_plan_small<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->small_smem));
      SB_CUDA(cudaFuncSetAttribute(k_plan_small<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->small_smem));
      SB_CUDA(cudaFuncSetAttribute(k_plan_small<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->small_smem));
      set_to = p->small_smem;
    }
  }
  if (const char* e = getenv("SEQBAL_PLANNER")) p->path = std::string(e) == "small" ? 1 : std::string(e) == "large" ? 2 : 0;
  for (int i = 0; i < 6; ++i) SB_CUDA(cudaEventCreate(&p->ev[i]));
  SB_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
  SB_CUDA(cudaEventCreateWithFlags(&p->fork_ev, cudaEventDisableTiming));
  SB_CUDA(cudaEventCreateWithFlags(&p->join_ev, cudaEventDisableTiming));
  SB_CUDA(cudaEventCreateWithFlags(&p->gfork_ev, cudaEventDisableTiming));
  SB_CUDA(cudaEventCreateWithFlags(&p->gjoin_ev, cudaEventDisableTiming));
  SB_CUDA(cudaEventCreateWithFlags(&p->dup_ev, cudaEventDisableTiming));
}

static void planner_free(sb_planner* p) {
  void* ptrs[] = {p->d_bag_off, p->d_bag_ranks, p->d_bag_size, p->d_rank_bag, p->d_rank_member,
                  p->w, p->seq_rank, p->seq_off, p->hash, p->sk_hi, p->sk_lo, p->tk_hi, p->tk_lo,
                  p->sk_v, p->tk_v, p->sorted_w, p->sorted_idx, p->pick, p->seq_bag, p->seq_G,
                  p->seq_chunk_base, p->rep_total, p->sentinel, p->bag_count, p->bag_rows,
                  p->rep_chunks, p->send_count, p->n_chunks, p->n_seqs, p->c_id, p->c_idx, p->c_src,
                  p->c_dst, p->c_start, p->c_end, p->c_src_row, p->c_dst_row, p->c_seq_base, p->c_seq,
                  p->send_off, p->recv_off, p->send_idx, p->recv_idx, p->rev_recv_idx,
                  p->origin_rows, p->target_rows, p->per_gpu, p->per_bag_occ, p->total, p->wir,
                  p->violations, p->status,
                  p->stage_ids, p->stage_lens, p->stage_w, p->stage_off,
                  p->seg_off, p->seg_id, p->seg_first, p->seg_len, p->recv_count, p->ck_hi, p->ck_lo,
                  p->ck_thi, p->ck_tlo, p->ck_v, p->ck_tv, p->rep_cbase, p->bag_seq, p->tile_cnt, p->list_sum, p->list_tie,
                  p->bag_cbase, p->bag_sbase, p->greedy_q};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (p->h_small) cudaFreeHost(p->h_small);
  for (int i = 0; i < 6; ++i)
    if (p->ev[i]) cudaEventDestroy(p->ev[i]);
  if (p->fork_ev) cudaEventDestroy(p->fork_ev);
  if (p->join_ev) cudaEventDestroy(p->join_ev);
  if (p->gfork_ev) cudaEventDestroy(p->gfork_ev);
  if (p->gjoin_ev) cudaEventDestroy(p->gjoin_ev);
  if (p->dup_ev) cudaEventDestroy(p->dup_ev);
  if (p->side) cudaStreamDestroy(p->side);
  for (cudaEvent_t e : p->copy_ev) cudaEventDestroy(e);
  if (p->x_owner) cudaFree(p->x_owner);
  if (p->unpack.jobs) cudaFree(p->unpack.jobs);
  if (p->unpack.piece_off) cudaFree(p->unpack.piece_off);
  if (p->unpack.n_jobs) cudaFree(p->unpack.n_jobs);
  for (auto& sl : p->slots) {
    if (sl.jobs) cudaFree(sl.jobs);
    if (sl.piece_off) cudaFree(sl.piece_off);
    if (sl.n_jobs) cudaFree(sl.n_jobs);
  }
}

static void plan_common_prologue(sb_planner* p, cudaStream_t s) {
  SB_CUDA(cudaMemsetAsync(p->hash, 0xff, sizeof(uint64_t) * 2 * (size_t)p->max_seqs, s));
  SB_CUDA(cudaMemsetAsync(p->sentinel, 0, sizeof(int32_t) * p->R, s));
  SB_CUDA(cudaMemsetAsync(p->status, 0, sizeof(int32_t), s));
  SB_CUDA(cudaMemsetAsync(p->violations, 0, sizeof(int32_t), s));
}

// Path choice.  The fused single-CTA planner wins while launches dominate;
// the multi-kernel path's fixed cost is ~50 us (a dozen launches) but its
// greedy runs in a 32-thread kernel (~102 cycles per step against ~150 inside
// the 512-thread fused CTA) and its sort / emission use many SMs; the hybrid
// (fused prefix, 32-thread greedy kernel, fused suffix) pays two kernel
// boundaries and a reload for the faster chain.  Measured by graph replay
// (tools/path_compare.py, profiles/r02/s3_planner/path_compare*.txt), g1n8:
// 256 sequences fused 34 / hybrid 36 / multi-kernel 67 us, 512 61 / 56 / 86,
// 768 91 / 82 / 100, 1024 116 / 102-113 / 114-117, 1536 multi-kernel ahead;
// one bag per replica 512 46 vs 61 fused ahead, 768 66 vs 61 behind.
constexpr int64_t kSmallChunks = 8192;

constexpr int64_t kSmallAutoSeqsOneBag = 640;   // one bag per replica (no greedy chain)
constexpr int64_t kHybridAutoSeqs = 256;        // hybrid from here (see choose_path) ...
constexpr int64_t kHybridAutoMaxSeqs = 1152;    // ... up to here, multi-kernel above

// 1 = fused single CTA, 2 = multi-kernel, 3 = hybrid (fused prefix, 32-thread
// greedy kernel, fused suffix).
static int choose_path(const sb_planner* p) {
  const bool fits = p->max_seqs <= kSmallSeqs && p->W <= 1024 && p->M <= kMaxBags;
  if (p->path == 2 || !fits) return 2;
  if (p->path == 1) return 1;
  if (p->path == 3) return 3;
  if (p->M == 1) return p->max_seqs <= kSmallAutoSeqsOneBag && p->max_chunks <= kSmallChunks ? 1 : 2;
  if (p->max_chunks > kSmallChunks || p->max_seqs > kHybridAutoMaxSeqs) return 2;
  return p->max_seqs < kHybridAutoSeqs ? 1 : 3;
}

// Shared-memory staging capacity of the serial-sum kernels (workloads of one
// replica / the whole gather); the attribute is raised once per process.
static int64_t sum_stage_cap(const sb_planner* p) {
  const int64_t cap = std::min<int64_t>(std::max<int64_t>(p->max_seqs, 1), kSumStage);
  static int64_t set_to = 0;
  if (cap > set_to) {
    const int bytes = (int)(cap * sizeof(double));
    SB_CUDA(cudaFuncSetAttribute(k_totals, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    SB_CUDA(cudaFuncSetAttribute(k_single_bag_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    set_to = cap;
  }
  return cap;
}

// The serial FP64 totals and the origin row offsets fork onto the planner's
// side stream as soon as the metadata is there (the totals recompute workloads
// from lengths) and join before the greedy: they overlap the per-sequence
// pass and the sort.
static void launch_totals(sb_planner* p, const PlanArgs& a, cudaStream_t s) {
  SB_CUDA(cudaEventRecord(p->fork_ev, s));
  SB_CUDA(cudaStreamWaitEvent(p->side, p->fork_ev, 0));
  const int64_t cap = sum_stage_cap(p);
  k_totals<<<p->R + 1, kSumThreads, (size_t)cap * sizeof(double), p->side>>>(a, cap);
  SB_CHECK_LAUNCH();
  k_prep_rows<<<p->W, kPrepRowsThreads, 0, p->side>>>(a);
  SB_CHECK_LAUNCH();
  SB_CUDA(cudaEventRecord(p->join_ev, p->side));
  k_prep_dup<<<(int)((p->max_seqs + 255) / 256), 256, 0, p->side>>>(a);  // joined by join_dup()
  SB_CHECK_LAUNCH();
  SB_CUDA(cudaEventRecord(p->dup_ev, p->side));
  count_launch(3);
}

static void join_dup(sb_planner* p, cudaStream_t s) { SB_CUDA(cudaStreamWaitEvent(s, p->dup_ev, 0)); }

static void launch_prep(sb_planner* p, const PlanArgs& a, cudaStream_t s) {
  k_prep_seq<<<(int)((p->max_seqs + 255) / 256), 256, 0, s>>>(a);
  SB_CHECK_LAUNCH();
  count_launch(1);
}

static void launch_sort(sb_planner* p, const PlanArgs& a, cudaStream_t s, bool order) {
  int launches = 0;
  if (order) {
    const int64_t N = p->max_seqs;
    const int tiles = (int)((N + kRunTile - 1) / kRunTile) + p->R;
    k_sort_tiles<<<tiles, kSortThreads, kSortSmemBytes, s>>>(a);
    SB_CHECK_LAUNCH();
    const int blocks = (int)((N + 255) / 256);
    if (N <= kRankMergeMax) {  // every replica fits: one rank pass writes the greedy order
      k_rank_merge<kRankMergeMax / kRunTile><<<blocks, 256, 0, s>>>(a);
      SB_CHECK_LAUNCH();
      SB_CUDA(cudaStreamWaitEvent(s, p->join_ev, 0));  // totals joined
      count_launch(2);
      return;
    }
    uint64_t *shi = p->sk_hi, *slo = p->sk_lo, *dhi = p->tk_hi, *dlo = p->tk_lo;
    uint32_t *sv = p->sk_v, *dv = p->tk_v;
    for (int64_t width = kRunTile; width < N; width <<= 1) {
      k_merge_pass<<<blocks, 256, 0, s>>>(a, width, shi, slo, sv, dhi, dlo, dv);
      SB_CHECK_LAUNCH();
      std::swap(shi, dhi);
      std::swap(slo, dlo);
      std::swap(sv, dv);
      ++launches;
    }
    k_sort_finish<<<blocks, 256, 0, s>>>(a, sv);
    SB_CHECK_LAUNCH();
    launches += 2;
  }
  SB_CUDA(cudaStreamWaitEvent(s, p->join_ev, 0));  // totals joined
  count_launch(launches);
}

// k_greedy_staged when every replica fits the staging buffer (the planner's
// sequence capacity bounds every replica), else the ring-fed k_greedy.
// fork: a single-bag chain runs on the side stream; the caller joins gjoin_ev
// (run_plan: before k_finalize).
static void launch_greedy(sb_planner* p, const PlanArgs& a, cudaStream_t s, bool fork) {
  if (p->M == 1) {  // picks and counts up front; the occupancy replay forks when asked
    k_single_bag_fill<<<(int)((std::max<int64_t>(p->max_seqs, p->R) + 255) / 256), 256, 0, s>>>(a);
    SB_CHECK_LAUNCH();
    cudaStream_t gs = s;
    if (fork) {
      SB_CUDA(cudaEventRecord(p->gfork_ev, s));
      SB_CUDA(cudaStreamWaitEvent(p->side, p->gfork_ev, 0));
      gs = p->side;
    }
    const int64_t cap = sum_stage_cap(p);
    k_single_bag_chain<<<p->R, kSumThreads, (size_t)cap * sizeof(double), gs>>>(a, cap);
    SB_CHECK_LAUNCH();
    if (fork) SB_CUDA(cudaEventRecord(p->gjoin_ev, p->side));
    count_launch(1);  // the callers count one greedy launch
    return;
  }
  if (p->M > kMaxBags) {
    const int smem = (int)((2 * sizeof(double) + sizeof(int)) * p->M);
    k_greedy_many<<<p->R, 32, smem, s>>>(a);
    SB_CHECK_LAUNCH();
    return;
  }
  const bool wide = (p->M + 31) / 32 > 1;
  if (p->max_seqs <= kGreedyStage) {
    const int smem = (int)(sizeof(double) * (std::max<int64_t>(1, p->max_seqs) + 6));
    static int set_to[2] = {0, 0};
    if (smem > set_to[wide]) {
      if (wide) SB_CUDA(cudaFuncSetAttribute(k_greedy_staged<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      else SB_CUDA(cudaFuncSetAttribute(k_greedy_staged<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      set_to[wide] = smem;
    }
    if (wide) k_greedy_staged<2><<<p->R, 32, smem, s>>>(a);
    else k_greedy_staged<1><<<p->R, 32, smem, s>>>(a);
  } else {
    if (wide) k_greedy<2><<<p->R, 32, 0, s>>>(a);
    else k_greedy<1><<<p->R, 32, 0, s>>>(a);
  }
  SB_CHECK_LAUNCH();
}

static void run_plan(sb_planner* p, cudaStream_t s) {
  PlanArgs a = make_args(p);
  p->last_path = choose_path(p);
  if (p->last_path == 1) {  // one launch: the kernel clears the status word itself
    if (p->timing) SB_CUDA(cudaEventRecord(p->ev[0], s));
    k_plan_small<0><<<1, kSmallThreads, p->small_smem, s>>>(a, (int)p->max_seqs);
    SB_CHECK_LAUNCH();
    if (p->timing)
      for (int i = 1; i < 6; ++i) SB_CUDA(cudaEventRecord(p->ev[i], s));
    count_launch(1);
    return;
  }
  if (p->last_path == 3) {
    // hybrid: the prefix (phases 0-2, then -- one replica -- the greedy on
    // warp 0 once the other warps have exited; several replicas: the 32-thread
    // greedy kernel), then the suffix (phases 3-6) as a programmatic dependent
    // launch: its prologue (tables, ids, the duplicate-id check) runs under the
    // greedy chain and it waits on the grid dependency before the rest.
    if (p->timing) SB_CUDA(cudaEventRecord(p->ev[0], s));
    k_plan_small<1><<<1, kSmallThreads, p->small_smem, s>>>(a, (int)p->max_seqs);
    SB_CHECK_LAUNCH();
    if (p->R > 1) {  // several replicas: the 32-thread greedy kernel, one CTA per replica
      const int smem = (int)(sizeof(double) * (std::max<int64_t>(1, p->max_seqs) + 6) +
                             sizeof(int32_t) * std::max<int64_t>(1, p->max_seqs));
      static int set_to[2] = {0, 0};
      const bool wide = p->M > 32;
      if (smem > set_to[wide]) {
        if (wide)
          SB_CUDA(cudaFuncSetAttribute(k_greedy_staged<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        else
          SB_CUDA(cudaFuncSetAttribute(k_greedy_staged<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        set_to[wide] = smem;
      }
      if (wide) k_greedy_staged<2, true><<<p->R, 32, smem, s>>>(a);
      else k_greedy_staged<1, true><<<p->R, 32, smem, s>>>(a);
      SB_CHECK_LAUNCH();
    }
    {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(1);
      cfg.blockDim = dim3(kSmallThreads);
      cfg.dynamicSmemBytes = p->small_smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      SB_CUDA(cudaLaunchKernelEx(&cfg, k_plan_small<2>, a, (int)p->max_seqs));
      SB_CHECK_LAUNCH();
    }
    if (p->timing)
      for (int i = 1; i < 6; ++i) SB_CUDA(cudaEventRecord(p->ev[i], s));
    count_launch(p->R > 1 ? 3 : 2);
    return;
  }
  plan_common_prologue(p, s);
  if (p->timing) SB_CUDA(cudaEventRecord(p->ev[0], s));
  launch_totals(p, a, s);
  launch_prep(p, a, s);
  if (p->timing) SB_CUDA(cudaEventRecord(p->ev[1], s));
  launch_sort(p, a, s, true);
  if (p->timing) SB_CUDA(cudaEventRecord(p->ev[2], s));
  launch_greedy(p, a, s, true);
  if (p->timing) SB_CUDA(cudaEventRecord(p->ev[3], s));
  const dim3 eg((unsigned)((p->max_seqs + kEmitTile - 1) / kEmitTile), (unsigned)p->R);
  const int emit_smem = (int)(sizeof(int) * (kEmitTile / 32) * p->M);
  if (emit_smem > 48 * 1024) {
    static int set_to = 0;
    if (emit_smem > set_to) {
      SB_CUDA(cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, emit_smem));
      set_to = emit_smem;
    }
  }
  k_emit_count<<<eg, kEmitTile, sizeof(int) * p->M, s>>>(a);
  SB_CHECK_LAUNCH();
  k_emit<<<eg, kEmitTile, emit_smem, s>>>(a);
  SB_CHECK_LAUNCH();
  k_emit_chunks<<<(int)((p->max_chunks + 255) / 256), 256, 0, s>>>(a);
  SB_CHECK_LAUNCH();
  if (p->timing) SB_CUDA(cudaEventRecord(p->ev[4], s));
  const dim3 lg((unsigned)((p->max_seqs + kListTile - 1) / kListTile), (unsigned)p->W);
  k_lists_count<<<lg, kListTile, 0, s>>>(a);
  SB_CHECK_LAUNCH();
  k_lists<<<lg, kListTile, 0, s>>>(a);
  SB_CHECK_LAUNCH();
  if (p->M == 1) SB_CUDA(cudaStreamWaitEvent(s, p->gjoin_ev, 0));  // single-bag occupancy replay joined
  k_finalize<<<1, 32, 0, s>>>(a);
  SB_CHECK_LAUNCH();
  join_dup(p, s);
  if (p->timing) SB_CUDA(cudaEventRecord(p->ev[5], s));
  count_launch(7);  // greedy, emit count, emit, emit chunks, lists count, lists, finalize (+ tie replay)
}

static void run_identity(sb_planner* p, cudaStream_t s) {
  PlanArgs a = make_args(p);
  plan_common_prologue(p, s);
  launch_totals(p, a, s);
  launch_prep(p, a, s);
  launch_sort(p, a, s, false);  // join the totals only (sorted order unused)
  k_identity<<<148, 256, 0, s>>>(a);
  SB_CHECK_LAUNCH();
  k_identity_report<<<(p->W + 127) / 128, 128, 0, s>>>(a);
  SB_CHECK_LAUNCH();
  k_identity_finalize<<<1, 32, 0, s>>>(a);
  SB_CHECK_LAUNCH();
  join_dup(p, s);
  count_launch(3);
}

}  // namespace sb

// ============================================================== C-ABI
using sb::Error;

#define SB_API_BEGIN try {
#define SB_API_END                              \
  return SB_OK;                                 \
  }                                             \
  catch (const Error& e) {                      \
    sb::set_error(e.msg);                       \
    return e.code;                              \
  }                                             \
  catch (const std::bad_alloc&) {               \
    sb::set_error("host allocation failed");    \
    return SB_ERR_CAPACITY;                     \
  }

extern "C" sb_status sb_planner_create(const sb_planner_desc* d, sb_planner** out) {
  SB_API_BEGIN
  if (!d || !out) throw Error{SB_ERR_CONFIG, "sb_planner_create: null argument"};
  *out = nullptr;
  // All four shape fields 0: an assignment-only planner (sb_assign_to_bags);
  // no workload model, no head check, sb_plan / sb_plan_identity refuse it.
  const bool assign_only = d->d_model == 0 && d->n_heads == 0 && d->d_head == 0 && d->n_blocks == 0;
  // WorkloadModel::validate (workload_model.cpp:15-31)
  if (!assign_only && (d->d_model < 1 || d->n_heads < 1 || d->d_head < 1 || d->n_blocks < 1))
    throw Error{SB_ERR_CONFIG, "model shape fields must be >= 1"};
  if ((int64_t)d->n_heads * d->d_head != d->d_model)
    throw Error{SB_ERR_CONFIG, "n_heads * d_head must equal d_model (" + std::to_string(d->n_heads) + " * " +
                                   std::to_string(d->d_head) + " != " + std::to_string(d->d_model) + ")"};
  if (!(d->gamma > 0.0)) throw Error{SB_ERR_CONFIG, "gamma must be positive"};
  if (!(d->k > 0.0)) throw Error{SB_ERR_CONFIG, "k must be positive"};
  if (d->n_bags < 1 || !d->bag_offsets || !d->bag_ranks) throw Error{SB_ERR_CONFIG, "topology has no GPUs"};
  if (d->unit_size < 1) throw Error{SB_ERR_CONFIG, "topology has no GPUs"};
  // replicate (topology.cpp:81-93)
  if (d->world_size < d->unit_size)
    throw Error{SB_ERR_CONFIG, "world_size " + std::to_string(d->world_size) +
                                   " is smaller than the sharding unit " + std::to_string(d->unit_size)};
  if (d->world_size % d->unit_size != 0)
    throw Error{SB_ERR_CONFIG, "world_size " + std::to_string(d->world_size) +
                                   " is not a multiple of the sharding unit " + std::to_string(d->unit_size)};
  if (d->n_bags > sb::kMaxBagsLarge)
    throw Error{SB_ERR_CONFIG, "more than " + std::to_string(sb::kMaxBagsLarge) + " bags per replica"};
  auto* p = new sb_planner();
  p->W = d->world_size;
  p->U = d->unit_size;
  p->M = d->n_bags;
  p->R = d->world_size / d->unit_size;
  p->d_model = d->d_model;
  p->n_heads = d->n_heads;
  p->d_head = d->d_head;
  p->n_blocks = d->n_blocks;
  p->gamma = d->gamma;
  p->k = d->k;
  p->bag_off.assign(d->bag_offsets, d->bag_offsets + d->n_bags + 1);
  if (p->bag_off[0] != 0 || p->bag_off[p->M] != p->U) {
    delete p;
    throw Error{SB_ERR_CONFIG, "bag ranks must cover the unit exactly once"};
  }
  p->bag_ranks.assign(d->bag_ranks, d->bag_ranks + p->U);
  p->rank_bag.assign(p->U, -1);
  p->rank_member.assign(p->U, -1);
  for (int b = 0; b < p->M; ++b) {
    const int g = p->bag_off[b + 1] - p->bag_off[b];
    if (g < 1) {
      delete p;
      throw Error{SB_ERR_CONFIG, "empty bag"};
    }
    // plan_routing head check (balancer.cpp:114-120)
    if (!assign_only && d->n_heads % g != 0) {
      delete p;
      throw Error{SB_ERR_CONFIG, "bag of " + std::to_string(g) + " GPUs does not divide n_heads " +
                                     std::to_string(d->n_heads)};
    }
    p->bag_size.push_back(g);
    p->max_bag = std::max(p->max_bag, g);
    if (g > 1) p->any_multi_bag = true;
    for (int k = 0; k < g; ++k) {
      const int u = p->bag_ranks[p->bag_off[b] + k];
      if (u < 0 || u >= p->U || p->rank_bag[u] != -1) {
        delete p;
        throw Error{SB_ERR_CONFIG, "bag ranks must cover the unit exactly once"};
      }
      p->rank_bag[u] = b;
      p->rank_member[u] = k;
    }
  }
  p->max_seqs = std::max<int64_t>(1, d->max_seqs);
  if (p->max_seqs > (int64_t)1 << 30) {
    delete p;
    throw Error{SB_ERR_CONFIG, "max_seqs too large"};
  }
  p->max_chunks = p->max_seqs * p->max_bag;
  try {
    sb::planner_alloc(p);
  } catch (...) {
    sb::planner_free(p);
    delete p;
    throw;
  }
  *out = p;
  SB_API_END
}

namespace sb {
sb_planner* planner_clone(const sb_planner* p) {
  sb_planner_desc d{};
  d.world_size = p->W;
  d.unit_size = p->U;
  d.n_bags = p->M;
  d.bag_offsets = p->bag_off.data();
  d.bag_ranks = p->bag_ranks.data();
  d.d_model = p->d_model;
  d.n_heads = p->n_heads;
  d.d_head = p->d_head;
  d.n_blocks = p->n_blocks;
  d.gamma = p->gamma;
  d.k = p->k;
  d.max_seqs = p->max_seqs;
  sb_planner* q = nullptr;
  const sb_status st = sb_planner_create(&d, &q);
  if (st != SB_OK) throw Error{st, sb_last_error()};
  q->path = p->path;
  return q;
}
}  // namespace sb

extern "C" sb_status sb_planner_destroy(sb_planner* p) {
  SB_API_BEGIN
  if (p) {
    sb::planner_free(p);
    delete p;
  }
  SB_API_END
}

extern "C" sb_status sb_plan(sb_planner* p, const uint64_t* d_ids, const int64_t* d_lens,
                             const int64_t* d_rank_off, sb_stream stream) {
  SB_API_BEGIN
  if (!p || !d_rank_off) throw Error{SB_ERR_CONFIG, "sb_plan: null argument"};
  if (p->n_heads == 0) throw Error{SB_ERR_CONFIG, "sb_plan: planner was created for assign_to_bags only"};
  p->ids = d_ids;
  p->lens = d_lens;
  p->rank_off = d_rank_off;
  p->w_in = nullptr;
  p->identity = false;
  p->uploaded = false;
  sb::run_plan(p, (cudaStream_t)stream);
  SB_API_END
}

extern "C" sb_status sb_selftest_div(int64_t n, uint64_t seed, int64_t* mismatches) {
  SB_API_BEGIN
  if (!mismatches || n < 0) throw Error{SB_ERR_CONFIG, "sb_selftest_div: bad arguments"};
  unsigned long long* d = nullptr;
  SB_CUDA(cudaMalloc(&d, sizeof *d));
  SB_CUDA(cudaMemset(d, 0, sizeof *d));
  sb::k_selftest_div<<<1184, 256>>>(seed, n, d);
  const cudaError_t e = cudaGetLastError();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) throw Error{SB_ERR_CUDA, cudaGetErrorString(e)};
  *mismatches = (int64_t)h;
  SB_API_END
}

extern "C" sb_status sb_selftest_serial_sum(int64_t blocks, int64_t max_len, uint64_t seed, int mode,
                                           int64_t* mismatches) {
  SB_API_BEGIN
  if (!mismatches || blocks < 1 || max_len < 1 || mode < 0 || mode > 6)
    throw Error{SB_ERR_CONFIG, "sb_selftest_serial_sum: bad arguments"};
  unsigned long long* d = nullptr;
  double* pre = nullptr;
  SB_CUDA(cudaMalloc(&d, sizeof *d));
  if (cudaMalloc(&pre, sizeof(double) * blocks * max_len) != cudaSuccess) {
    cudaFree(d);
    throw Error{SB_ERR_CUDA, "sb_selftest_serial_sum: scratch allocation"};
  }
  cudaMemset(d, 0, sizeof *d);
  sb::k_selftest_sum<<<(unsigned)blocks, sb::kSumThreads>>>(seed, mode, max_len, pre, d);
  const cudaError_t e = cudaGetLastError();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(pre);
  cudaFree(d);
  if (e != cudaSuccess) throw Error{SB_ERR_CUDA, cudaGetErrorString(e)};
  *mismatches = (int64_t)h;
  SB_API_END
}

extern "C" sb_status sb_planner_trace(sb_planner* p, int enable, int64_t* out16) {
  SB_API_BEGIN
  if (!p) throw Error{SB_ERR_CONFIG, "null planner"};
  if (enable && !p->trace) {
    SB_CUDA(cudaMalloc(&p->trace, sizeof(long long) * 16));
    SB_CUDA(cudaMemset(p->trace, 0, sizeof(long long) * 16));
  }
  if (!enable && p->trace) {
    cudaFree(p->trace);
    p->trace = nullptr;
  }
  if (out16 && p->trace) {
    SB_CUDA(cudaDeviceSynchronize());
    SB_CUDA(cudaMemcpy(out16, p->trace, sizeof(long long) * 16, cudaMemcpyDeviceToHost));
  }
  SB_API_END
}

extern "C" sb_status sb_planner_set_path(sb_planner* p, int path) {
  SB_API_BEGIN
  if (!p || path < 0 || path > 3) throw Error{SB_ERR_CONFIG, "sb_planner_set_path: path must be 0, 1, 2 or 3"};
  if ((path == 1 || path == 3) && !(p->max_seqs <= sb::kSmallSeqs && p->W <= 1024))
    throw Error{SB_ERR_CONFIG, "sb_planner_set_path: capacity too large for the single-CTA planner"};
  p->path = path;
  SB_API_END
}

extern "C" sb_status sb_planner_last_path(sb_planner* p, int* path) {
  SB_API_BEGIN
  if (!p || !path) throw Error{SB_ERR_CONFIG, "null argument"};
  *path = p->last_path;
  SB_API_END
}

// Manifests + reverse receive order for an uploaded plan (see k_generic_*).
extern "C" sb_status sb_plan_manifests(sb_planner* p, sb_stream stream) {
  SB_API_BEGIN
  if (!p) throw Error{SB_ERR_CONFIG, "null planner"};
  if (!p->uploaded || !p->seg_off) throw Error{SB_ERR_CONFIG, "sb_plan_manifests: no uploaded plan"};
  cudaStream_t s = (cudaStream_t)stream;
  if (!p->ck_hi) {
    sb::dalloc(&p->ck_hi, p->max_chunks); sb::dalloc(&p->ck_lo, p->max_chunks);
    sb::dalloc(&p->ck_thi, p->max_chunks); sb::dalloc(&p->ck_tlo, p->max_chunks);
    sb::dalloc(&p->ck_v, p->max_chunks); sb::dalloc(&p->ck_tv, p->max_chunks);
    SB_CUDA(cudaFuncSetAttribute(sb::k_generic_lists, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sb::kSortSmemBytes));
  }
  sb::GenericArgs g;
  g.W = p->W;
  g.n_chunks = p->n_chunks;
  g.c_id = p->c_id; g.c_src = p->c_src; g.c_dst = p->c_dst; g.c_start = p->c_start; g.c_end = p->c_end;
  g.seg_off = p->seg_off; g.seg_id = p->seg_id; g.seg_first = p->seg_first; g.seg_len = p->seg_len;
  g.send_count = p->send_count; g.recv_count = p->recv_count;
  g.send_off = p->send_off; g.recv_off = p->recv_off;
  g.send_idx = p->send_idx; g.recv_idx = p->recv_idx; g.rev_recv_idx = p->rev_recv_idx;
  g.ck_hi = p->ck_hi; g.ck_lo = p->ck_lo; g.ck_thi = p->ck_thi; g.ck_tlo = p->ck_tlo; g.ck_v = p->ck_v;
  g.ck_tv = p->ck_tv;
  g.status = p->status;
  SB_CUDA(cudaMemsetAsync(p->send_count, 0, sizeof(unsigned long long) * p->W, s));
  SB_CUDA(cudaMemsetAsync(p->recv_count, 0, sizeof(unsigned long long) * p->W, s));
  SB_CUDA(cudaMemsetAsync(p->status, 0, sizeof(int32_t), s));
  sb::k_generic_count<<<148, 256, 0, s>>>(g);
  SB_CHECK_LAUNCH();
  sb::k_generic_lists<<<p->W, 1024, sb::kSortSmemBytes, s>>>(g);
  SB_CHECK_LAUNCH();
  sb::count_launch(2);
  SB_CUDA(cudaStreamSynchronize(s));
  int32_t st = 0;
  SB_CUDA(cudaMemcpy(&st, p->status, sizeof st, cudaMemcpyDeviceToHost));
  if (st) throw Error{SB_ERR_INTEGRITY, "reverse_plan: a chunk does not fit any destination segment"};
  SB_API_END
}

// assign_to_bags (balancer.cpp:15-64) on caller workloads: k_prep_seq (workload
// validation) -> k_sort (order + total) -> k_greedy, then the assignment in
// sorted order is copied back.  Host arrays in and out; synchronises.
extern "C" sb_status sb_assign_to_bags(sb_planner* p, int64_t n, const uint64_t* ids, const double* workloads,
                                       uint64_t* out_ids, double* out_w, int32_t* out_bag, sb_stream stream) {
  SB_API_BEGIN
  if (!p || n < 0 || (n > 0 && (!ids || !workloads || !out_ids || !out_w || !out_bag)))
    throw Error{SB_ERR_CONFIG, "sb_assign_to_bags: bad arguments"};
  if (p->R != 1) throw Error{SB_ERR_CONFIG, "sb_assign_to_bags: planner must describe one replica"};
  if (n > p->max_seqs) throw Error{SB_ERR_CAPACITY, "sb_assign_to_bags: more sequences than planner capacity"};
  cudaStream_t s = (cudaStream_t)stream;
  if (!p->stage_ids) {
    sb::dalloc(&p->stage_ids, p->max_seqs);
    sb::dalloc(&p->stage_lens, p->max_seqs);
    sb::dalloc(&p->stage_w, p->max_seqs);
    sb::dalloc(&p->stage_off, p->W + 1);
    SB_CUDA(cudaMemset(p->stage_lens, 0, sizeof(int64_t) * p->max_seqs));
  }
  std::vector<int64_t> off(p->W + 1, n);
  off[0] = 0;
  if (n > 0) {
    SB_CUDA(cudaMemcpyAsync(p->stage_ids, ids, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, s));
    SB_CUDA(cudaMemcpyAsync(p->stage_w, workloads, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  }
  SB_CUDA(cudaMemcpyAsync(p->stage_off, off.data(), sizeof(int64_t) * (p->W + 1), cudaMemcpyHostToDevice, s));
  p->ids = p->stage_ids;
  p->lens = p->stage_lens;
  p->rank_off = p->stage_off;
  p->w_in = p->stage_w;
  p->identity = false;
  p->uploaded = false;
  sb::PlanArgs a = sb::make_args(p);
  sb::plan_common_prologue(p, s);
  sb::launch_totals(p, a, s);
  sb::launch_prep(p, a, s);
  sb::launch_sort(p, a, s, true);
  sb::launch_greedy(p, a, s, false);
  sb::join_dup(p, s);
  sb::count_launch(2);
  SB_CUDA(cudaStreamSynchronize(s));
  int32_t st = 0;
  SB_CUDA(cudaMemcpy(&st, p->status, sizeof st, cudaMemcpyDeviceToHost));
  p->w_in = nullptr;
  if (st & sb::ST_NEG_LENGTH) throw Error{SB_ERR_CONFIG, "assign_to_bags: negative workload"};
  if (st) throw Error{SB_ERR_INTEGRITY, "assign_to_bags: device status " + std::to_string(st)};
  if (n > 0) {
    std::vector<int32_t> idx(n);
    SB_CUDA(cudaMemcpy(idx.data(), p->sorted_idx, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    SB_CUDA(cudaMemcpy(out_w, p->sorted_w, sizeof(double) * n, cudaMemcpyDeviceToHost));
    SB_CUDA(cudaMemcpy(out_bag, p->pick, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) out_ids[i] = ids[idx[i]];
  }
  SB_API_END
}

extern "C" sb_status sb_plan_identity(sb_planner* p, const uint64_t* d_ids, const int64_t* d_lens,
                                      const int64_t* d_rank_off, sb_stream stream) {
  SB_API_BEGIN
  if (!p || !d_rank_off) throw Error{SB_ERR_CONFIG, "sb_plan_identity: null argument"};
  if (p->n_heads == 0) throw Error{SB_ERR_CONFIG, "sb_plan_identity: planner was created for assign_to_bags only"};
  p->ids = d_ids;
  p->lens = d_lens;
  p->rank_off = d_rank_off;
  p->w_in = nullptr;
  p->identity = true;
  p->uploaded = false;
  sb::run_identity(p, (cudaStream_t)stream);
  SB_API_END
}

extern "C" sb_status sb_plan_get(const sb_planner* p, sb_plan_dev* o) {
  SB_API_BEGIN
  if (!p || !o) throw Error{SB_ERR_CONFIG, "sb_plan_get: null argument"};
  o->world_size = p->W;
  o->max_chunks = p->max_chunks;
  o->n_chunks = p->n_chunks;
  o->chunk_id = p->c_id;
  o->chunk_index = p->c_idx;
  o->chunk_start = p->c_start;
  o->chunk_end = p->c_end;
  o->chunk_src = p->c_src;
  o->chunk_dst = p->c_dst;
  o->chunk_src_row = p->c_src_row;
  o->chunk_dst_row = p->c_dst_row;
  o->send_off = p->send_off;
  o->send_idx = p->send_idx;
  o->recv_off = p->recv_off;
  o->recv_idx = p->recv_idx;
  o->rev_recv_idx = p->rev_recv_idx;
  o->origin_rows = p->origin_rows;
  o->target_rows = p->target_rows;
  o->per_gpu_workload = p->per_gpu;
  o->per_bag_occupancy = p->per_bag_occ;
  o->capacity_violations = p->violations;
  o->total_workload = p->total;
  o->wir = p->wir;
  o->status = p->status;
  SB_API_END
}

// One read-back per call: status, chunk count and (for planned metadata) the
// sequence count land in pinned scalars with one stream synchronisation.
static void check_plan_status(sb_planner* p, cudaStream_t s) {
  int32_t* st_h = reinterpret_cast<int32_t*>(&p->h_small[0]);
  SB_CUDA(cudaMemcpyAsync(st_h, p->status, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SB_CUDA(cudaMemcpyAsync(&p->h_small[1], p->n_chunks, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  p->h_small[2] = 0;
  if (!p->uploaded && p->rank_off)  // uploaded plans carry no sequence metadata
    SB_CUDA(cudaMemcpyAsync(&p->h_small[2], p->rank_off + p->W, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SB_CUDA(cudaStreamSynchronize(s));
  const int32_t st = *st_h;
  if (st & sb::ST_CAPACITY)
    throw Error{SB_ERR_CAPACITY, "plan_routing: more sequences than the planner capacity"};
  if (st & sb::ST_NEG_LENGTH) throw Error{SB_ERR_CONFIG, "seq_len must be >= 0"};
  if (st & sb::ST_DUP_ID)
    throw Error{SB_ERR_CONFIG, "plan_routing: duplicate sample_id within a replica"};
  if (st) throw Error{SB_ERR_INTEGRITY, "plan_routing: device status " + std::to_string(st)};
}

extern "C" sb_status sb_plan_sizes(sb_planner* p, sb_stream stream, int64_t* n_chunks, int64_t* n_seqs) {
  SB_API_BEGIN
  if (!p) throw Error{SB_ERR_CONFIG, "sb_plan_sizes: null planner"};
  check_plan_status(p, (cudaStream_t)stream);
  if (n_chunks) *n_chunks = p->h_small[1];
  if (n_seqs) *n_seqs = p->h_small[2];
  SB_API_END
}

template <typename T>
static void d2h(T* dst, const T* src, int64_t n, cudaStream_t s) {
  if (dst && n > 0) SB_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * (size_t)n, cudaMemcpyDeviceToHost, s));
}

extern "C" sb_status sb_plan_download(sb_planner* p, sb_plan_host* o, sb_stream stream) {
  SB_API_BEGIN
  if (!p || !o) throw Error{SB_ERR_CONFIG, "sb_plan_download: null argument"};
  cudaStream_t s = (cudaStream_t)stream;
  check_plan_status(p, s);
  const int64_t c = p->h_small[1];
  d2h(o->chunk_id, p->c_id, c, s);
  d2h(o->chunk_index, p->c_idx, c, s);
  d2h(o->chunk_start, p->c_start, c, s);
  d2h(o->chunk_end, p->c_end, c, s);
  d2h(o->chunk_src, p->c_src, c, s);
  d2h(o->chunk_dst, p->c_dst, c, s);
  d2h(o->send_off, p->send_off, p->W + 1, s);
  d2h(o->send_idx, p->send_idx, c, s);
  d2h(o->recv_off, p->recv_off, p->W + 1, s);
  d2h(o->recv_idx, p->recv_idx, c, s);
  d2h(o->rev_recv_idx, p->rev_recv_idx, c, s);
  d2h(o->target_rows, p->target_rows, p->W, s);
  d2h(o->per_gpu_workload, p->per_gpu, p->W, s);
  if (!p->identity) d2h(o->per_bag_occupancy, p->per_bag_occ, (int64_t)p->R * p->M, s);
  SB_CUDA(cudaMemcpyAsync(&o->capacity_violations, p->violations, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SB_CUDA(cudaMemcpyAsync(&o->total_workload, p->total, sizeof(double), cudaMemcpyDeviceToHost, s));
  SB_CUDA(cudaMemcpyAsync(&o->wir, p->wir, sizeof(double), cudaMemcpyDeviceToHost, s));
  SB_CUDA(cudaStreamSynchronize(s));
  SB_API_END
}

extern "C" sb_status sb_planner_enable_timing(sb_planner* p, int enable) {
  SB_API_BEGIN
  if (!p) throw Error{SB_ERR_CONFIG, "null planner"};
  p->timing = enable != 0;
  SB_API_END
}

extern "C" sb_status sb_planner_timing(sb_planner* p, double* a, double* b, double* c, double* d, double* e) {
  SB_API_BEGIN
  if (!p) throw Error{SB_ERR_CONFIG, "null planner"};
  double* outs[5] = {a, b, c, d, e};
  for (int i = 0; i < 5; ++i) {
    float ms = 0.f;
    if (p->timing) SB_CUDA(cudaEventElapsedTime(&ms, p->ev[i], p->ev[i + 1]));
    if (outs[i]) *outs[i] = 1000.0 * ms;
  }
  SB_API_END
}
