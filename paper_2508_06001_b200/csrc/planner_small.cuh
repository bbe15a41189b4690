// Single-CTA planner for small batches (up to kSmallSeqs sequences).
//
// The multi-kernel pipeline in planner.cu is launch-latency bound when a
// step carries a few dozen sequences (C2: 30): many launches, each paying a
// kernel start and a cold read of what the previous one wrote.  Here one
// 512-thread CTA keeps every per-sequence array in shared memory and runs
// the phases back to back (listed above k_plan_small).  Results are
// bit-identical to the large path (tests/test_gpu_parity.py runs both on the
// same inputs).
#pragma once

namespace sb {

// Per-phase clock64() trace (thread 0) when the planner has a trace buffer.
#define SB_PHASE(k)                                   \
  do {                                                \
    if (a.trace && threadIdx.x == 0) a.trace[k] = clock64(); \
  } while (0)
// Sub-phase marks (diagnostics): thread 0's time / the latest warp's time.
#define SB_MARK(k) SB_PHASE(k)
#ifdef SB_TRACE_P3  // diagnostics: slots 7-9, 11, 12 mark phase 3's setup / epilogue instead of phases 1 and 5
#define SB_P3(k) SB_PHASE(k)
#define SB_P5(x)
#else
#define SB_P3(k)
#define SB_P5(x) x
#endif
#define SB_MARK_MAX(k)                                                                                   \
  do {                                                                                                   \
    if (a.trace && (threadIdx.x & 31) == 0)                                                              \
      atomicMax(reinterpret_cast<unsigned long long*>(a.trace + (k)), (unsigned long long)clock64()); \
  } while (0)

constexpr int kSmallSeqs = 2048;
constexpr int kSmallScanSeqs = 128;  // up to here one warp computes the origin offsets (phase 1)
constexpr int kSmallThreads = 512;  // a 256-thread block measured no faster greedy (same code generation)

__host__ __device__ inline int small_pow2(int n) {
  int t = 32;
  while (t < n) t <<= 1;
  return t;
}

struct SmallLayout {  // byte offsets into dynamic shared memory
  size_t ids, lens, w, soff, hi, lo, v, rank, sorted, pick, G, cb, bo, rank_off, rpre, bagcnt, bagcb, bagq,
      sendcnt, sendoff, reptot, repc, tie, t_boff, t_branks, t_bsize, t_rbag, t_rmem, pergpu, recvoff, q, qcnt, total;
  int T;
};

__host__ __device__ inline SmallLayout small_layout(int cap, int W, int RM, int R, int U, int M) {
  SmallLayout L;
  const int T = small_pow2(cap);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += (bytes + 15) & ~size_t(15);
    return at;
  };
  L.T = T;
  L.ids = take(8ull * cap);
  L.lens = take(8ull * cap);
  L.w = take(8ull * cap);
  L.soff = take(8ull * cap);
  L.hi = take(8ull * T);
  L.lo = take(8ull * T);
  L.v = take(4ull * T);
  L.rank = take(4ull * cap);
  L.sorted = take(4ull * cap);
  L.pick = take(4ull * cap);
  L.G = take(4ull * cap);
  L.cb = take(8ull * cap);
  L.bo = take(4ull * cap);
  L.rank_off = take(8ull * (W + 1));
  L.rpre = take(8ull * (W + 1));
  L.bagcnt = take(4ull * RM);
  L.bagcb = take(8ull * RM);
  L.bagq = take(4ull * RM);
  L.sendcnt = take(8ull * W);
  L.sendoff = take(8ull * (W + 1));
  L.tie = take(4ull * W);
  L.reptot = take(8ull * R);
  L.repc = take(8ull * R);
  L.t_boff = take(4ull * (M + 1));  // topology tables, staged once (read by every phase)
  L.t_branks = take(4ull * U);
  L.t_bsize = take(4ull * M);
  L.t_rbag = take(4ull * U);
  L.t_rmem = take(4ull * U);
  L.pergpu = take(8ull * W);  // per-GPU workload: the greedy writes it, WIR reads it
  L.recvoff = take(8ull * W);
  L.q = take(4ull * cap);  // rank of each greedy position inside its bag
  L.qcnt = take(4ull * M);  // bag counters of the split bag-rank pass (one replica)
  L.total = o;
  return L;
}

// Bitonic sort of n records already in shared memory (capacity t = pow2).
__device__ void smem_bitonic(uint64_t* hi, uint64_t* lo, uint32_t* v, int n, int t) {
  for (int i = n + threadIdx.x; i < t; i += blockDim.x) {
    hi[i] = ~0ull;
    lo[i] = ~0ull;
    v[i] = 0xffffffffu;
  }
  __syncthreads();
  for (int k = 2; k <= t; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < t / 2; i += blockDim.x) {
        const int a = 2 * j * (i / j) + (i % j), b = a + j;
        const bool up = (a & k) == 0;
        if (rec_less(hi[b], lo[b], v[b], hi[a], lo[a], v[a]) == up) {
          uint64_t x = hi[a]; hi[a] = hi[b]; hi[b] = x;
          uint64_t y = lo[a]; lo[a] = lo[b]; lo[b] = y;
          uint32_t z = v[a]; v[a] = v[b]; v[b] = z;
        }
      }
      __syncthreads();
    }
  }
}

template <int T, int RPT>
__device__ void reg_sort_emit(int32_t* sorted_idx, uint64_t* s_hi, uint64_t* s_lo, uint32_t* s_v, int32_t* s_sorted,
                              const double* s_w, double* s_wsorted, int64_t lo, int n) {
  uint64_t h[RPT], l[RPT];
  uint32_t v[RPT];
  reg_bitonic<T, RPT, kSmallThreads>(s_hi, s_lo, s_v, n, h, l, v);
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int x = threadIdx.x + r * kSmallThreads;
    if (x < n) {
      s_sorted[lo + x] = (int32_t)(lo + v[r]);
      s_wsorted[lo + x] = s_w[lo + v[r]];
      sorted_idx[lo + x] = (int32_t)(lo + v[r]);
    }
  }
}

// Each greedy position's rank inside its bag (the stable bag partition,
// balancer.cpp:178-192): one match_any pass over the picks, `cnt` (M bag
// counters, zero on entry) running.  Recording it inside the chain cost more
// per step.
__device__ __forceinline__ void bag_ranks_pass(const int32_t* pick, int n, int32_t* cnt, int32_t* q) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int p0 = 0; p0 < n; p0 += 32) {
    const int p = p0 + lane;
    const bool valid = p < n;
    const int b = valid ? pick[p] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    const int rank_in = __popc(peers & lt);
    const int base = valid ? cnt[b] : 0;
    __syncwarp();
    if (valid && rank_in == 0) cnt[b] = base + __popc(peers);
    __syncwarp();
    if (valid) q[p] = base + rank_in;
  }
}

// The greedy inlined (an out-of-line call gave the same ~150 cycles per step
// and a larger stack frame that lengthened every launch by ~4 us,
// tools/plan_latency.py).  `qsplit`: the bag ranks are another warp's (it
// waits on named barrier 4, which this warp arrives at once the picks are
// stored); else this warp derives them after the per-bag epilogue, with
// `bagcnt` (this replica's M counts, written by the greedy) as the running
// counters, restored at the end.
template <int BPL>
__device__ __forceinline__ void small_greedy(const PlanArgs& a, int rep, int64_t n, double total_rep, const double* ws,
                                          int32_t* pick, int32_t* bagcnt, int* viol, int32_t* q, bool qsplit) {
  auto handoff = [qsplit]() {
    if (qsplit) {
      __syncwarp();
      asm volatile("bar.arrive 4, 64;" ::: "memory");
    }
  };
  greedy_warp<BPL, 0>(a, rep, n, total_rep, [ws](int p) { return ws[p]; }, [](int) {}, pick, bagcnt, viol, nullptr,
                      handoff);
  if (qsplit) return;
  const int lane = threadIdx.x & 31, M = a.M;
  int32_t* cnt = bagcnt + rep * M;
  __syncwarp();
  int keep[BPL];
#pragma unroll
  for (int i = 0; i < BPL; ++i) {
    const int j = lane + 32 * i;
    keep[i] = j < M ? cnt[j] : 0;
    if (j < M) cnt[j] = 0;
  }
  __syncwarp();
  bag_ranks_pass(pick, (int)n, cnt, q);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < BPL; ++i)
    if (lane + 32 * i < M) cnt[lane + 32 * i] = keep[i];
  __syncwarp();
}

// Warp-level inclusive scan helper over int64.
__device__ __forceinline__ int64_t warp_scan_incl64(int64_t x) { return warp_incl_scan<int64_t>(x); }

// Single-CTA plan in seven barrier-separated phases.  Independent work shares
// a phase on different warps instead of taking its own (the kernel is a
// latency chain: a phase costs its slowest warp plus a barrier):
//   0 rank offsets + topology tables -> shared memory
//   1 per sequence: workload, rank, sort keys (warps 2..) | serial FP64 total
//     straight from the lengths (warp 0) | origin row offsets (warp 1)
//   2 sort by (workload desc, id asc); workloads gathered into greedy order
//   3 greedy, one warp per replica, which also records each sequence's rank
//     inside its bag and the bag bases | duplicate-id check (other warps)
//   4 per-sequence chunk emission (stable bag partition from those ranks) |
//     WIR (warp 0)
//   5 manifest offsets scanned by every warp, recv / Ulysses / reverse lists
//     per rank warp, send lists per sequence
//   6 libstdc++ tie-order replay of the reverse lists (rare)
//
// MODE 0 runs all of it.  The hybrid path (planner.cu run_plan) splits it
// around the 32-thread greedy kernel, whose chain runs ~100 cycles per step
// against ~150 inside this 512-thread kernel: MODE 1 runs
// phases 0-2 and leaves the greedy-order workloads in global memory,
// k_greedy_staged<.., true> picks, and MODE 2 reloads the per-sequence state
// and runs phases 3-6 with the bag bases in place of the greedy.
template <int MODE>
__global__ void __launch_bounds__(kSmallThreads, 1) k_plan_small(PlanArgs a_in, int cap) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int64_t sh[33];
  __shared__ int s_flag, s_viol, s_biglen;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  constexpr unsigned kFull = 0xffffffffu;
  PlanArgs a = a_in;  // topology tables and per_gpu redirected to shared memory after phase 0
  const int W = a.W, R = a.R, M = a.M, U = a.U;
  const SmallLayout L = small_layout(cap, W, R * M, R, U, M);
  uint64_t* s_ids = reinterpret_cast<uint64_t*>(sm + L.ids);
  int64_t* s_lens = reinterpret_cast<int64_t*>(sm + L.lens);
  double* s_w = reinterpret_cast<double*>(sm + L.w);
  int64_t* s_soff = reinterpret_cast<int64_t*>(sm + L.soff);
  uint64_t* s_hi = reinterpret_cast<uint64_t*>(sm + L.hi);
  uint64_t* s_lo = reinterpret_cast<uint64_t*>(sm + L.lo);
  uint32_t* s_v = reinterpret_cast<uint32_t*>(sm + L.v);
  int32_t* s_rank = reinterpret_cast<int32_t*>(sm + L.rank);
  int32_t* s_sorted = reinterpret_cast<int32_t*>(sm + L.sorted);
  int32_t* s_pick = reinterpret_cast<int32_t*>(sm + L.pick);
  int32_t* s_G = reinterpret_cast<int32_t*>(sm + L.G);
  int64_t* s_cb = reinterpret_cast<int64_t*>(sm + L.cb);
  double* s_wsorted = reinterpret_cast<double*>(sm + L.cb);  // greedy-order workloads; s_cb is written after the greedy
  int32_t* s_bo = reinterpret_cast<int32_t*>(sm + L.bo);
  int64_t* s_roff = reinterpret_cast<int64_t*>(sm + L.rank_off);
  int64_t* s_rpre = reinterpret_cast<int64_t*>(sm + L.rpre);
  int32_t* s_bagcnt = reinterpret_cast<int32_t*>(sm + L.bagcnt);
  int64_t* s_bagcb = reinterpret_cast<int64_t*>(sm + L.bagcb);
  int32_t* s_bagq = reinterpret_cast<int32_t*>(sm + L.bagq);
  int64_t* s_sendcnt = reinterpret_cast<int64_t*>(sm + L.sendcnt);
  int64_t* s_sendoff = reinterpret_cast<int64_t*>(sm + L.sendoff);
  int64_t* s_recvoff = reinterpret_cast<int64_t*>(sm + L.recvoff);
  int32_t* s_tie = reinterpret_cast<int32_t*>(sm + L.tie);
  double* s_reptot = reinterpret_cast<double*>(sm + L.reptot);
  int64_t* s_repc = reinterpret_cast<int64_t*>(sm + L.repc);
  int32_t* s_q = reinterpret_cast<int32_t*>(sm + L.q);

  // the hybrid prefix lets its suffix launch at once: the suffix's prologue
  // reads inputs only and waits on the grid dependency before the rest
  if constexpr (MODE == 1) asm volatile("griddepcontrol.launch_dependents;");
  if (MODE != 2) SB_PHASE(0);
  // ---- phase 0: rank offsets, topology tables
  for (int r = tid; r <= W; r += blockDim.x) s_roff[r] = a.rank_off[r];
  {
    int32_t* t_boff = reinterpret_cast<int32_t*>(sm + L.t_boff);
    int32_t* t_branks = reinterpret_cast<int32_t*>(sm + L.t_branks);
    int32_t* t_bsize = reinterpret_cast<int32_t*>(sm + L.t_bsize);
    int32_t* t_rbag = reinterpret_cast<int32_t*>(sm + L.t_rbag);
    int32_t* t_rmem = reinterpret_cast<int32_t*>(sm + L.t_rmem);
    // all loads first, then the shared stores (a generic source pointer may
    // alias shared memory, so interleaving would serialise the round trips)
    for (int i0 = 0; i0 <= (M > U ? M : U); i0 += blockDim.x) {
      const int i = i0 + tid;
      const int32_t bo = i <= M ? a.bag_off[i] : 0, bs = i < M ? a.bag_size[i] : 0;
      const int32_t br = i < U ? a.bag_ranks[i] : 0, rb = i < U ? a.rank_bag[i] : 0,
                    rm = i < U ? a.rank_member[i] : 0;
      if (i <= M) t_boff[i] = bo;
      if (i < M) t_bsize[i] = bs;
      if (i < U) {
        t_branks[i] = br;
        t_rbag[i] = rb;
        t_rmem[i] = rm;
      }
    }
    a.bag_off = t_boff;
    a.bag_ranks = t_branks;
    a.bag_size = t_bsize;
    a.rank_bag = t_rbag;
    a.rank_member = t_rmem;
    if (MODE == 0) a.per_gpu = reinterpret_cast<double*>(sm + L.pergpu);  // the hybrid's greedy writes it globally
  }
  for (int r = tid; r < W; r += blockDim.x) s_sendcnt[r] = 0;
  if (tid == 0) {
    s_flag = 0;
    s_viol = 0;
    s_biglen = 0;
    if (MODE != 2) *a.status = 0;  // no memset node before the launch; every atomicOr below follows this barrier
    if (MODE == 1) *a.violations = 0;  // the greedy kernel adds to it
  }
  __syncthreads();
  const int64_t N = s_roff[W];
  if (N > cap) {
    if (tid == 0) atomicOr(a.status, ST_CAPACITY);
    return;
  }
  auto rank_of = [&](int64_t i) {  // rank r with roff[r] <= i < roff[r+1]
    int lo = 0, hi = W;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_roff[mid] <= i) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  auto raw_workload = [&](int64_t i) {  // workload of gather index i (balancer.cpp:144)
    if (a.w_in) return a.w_in[i];
    const int64_t len = a.lens[i];
    return gamma_weighted_workload(len < 0 ? 0 : len, a.d_model, a.gamma);
  };
  // duplicate sample ids inside each replica (divergence):
  // open-addressing set in the sort scratch (s_hi and s_lo are contiguous,
  // 2T slots >= 2 * replica size, EMPTY = ~0) on threads [t0 .. t0 + nt) of
  // this CTA (named barrier 2); sets s_flag, reads s_ids and s_roff only
  auto dup_check = [&](int t, int nt) {
    auto bar = [nt]() { asm volatile("bar.sync 2, %0;" ::"r"(nt) : "memory"); };
    for (int rep = 0; rep < R; ++rep) {
      const int64_t lo = s_roff[rep * U], hi = s_roff[rep * U + U];
      const int tsz = 2 * L.T;
      for (int i = t; i < tsz; i += nt) s_hi[i] = ~0ull;
      if (t == 0) s_v[0] = 0;  // count of ids equal to the EMPTY marker
      bar();
      for (int64_t i = lo + t; i < hi; i += nt) {
        const uint64_t id = s_ids[i];
        if (id == ~0ull) {
          if (atomicAdd(&s_v[0], 1u) > 0) s_flag = 1;
          continue;
        }
        uint32_t slot = (uint32_t)(hash_slot(id) & (uint64_t)(tsz - 1));
        for (;;) {
          const unsigned long long old =
              atomicCAS(reinterpret_cast<unsigned long long*>(&s_hi[slot]), ~0ull, (unsigned long long)id);
          if (old == ~0ull) break;
          if (old == id) {
            s_flag = 1;
            break;
          }
          slot = (slot + 1) & (uint32_t)(tsz - 1);
        }
      }
      bar();
    }
  };
  if constexpr (MODE != 2) {  // phases 1-2 (fused, hybrid prefix)
    SB_PHASE(1);
    // ---- phase 1: metadata, workloads, ranks (balancer.cpp:139-149)
    auto seq_pass = [&](int t0, int nt, bool keys) {
      for (int64_t i = t0; i < N; i += nt) {
        const int r = rank_of(i);
        int64_t len = a.lens[i];
        if (len < 0) {
          atomicOr(a.status, ST_NEG_LENGTH);
          len = 0;
        }
        double wv;
        if (a.w_in) {
          wv = a.w_in[i];
          if (!(wv >= 0.0)) atomicOr(a.status, ST_NEG_LENGTH);
        } else {
          wv = gamma_weighted_workload(len, a.d_model, a.gamma);
        }
        if (len >= (int64_t)1 << 26) s_biglen = 1;  // 32 lengths no longer sum in 32 bits
        const uint64_t id = a.ids[i];
        s_ids[i] = id;
        s_lens[i] = len;
        s_w[i] = wv;
        s_rank[i] = r;
        a.w[i] = wv;
        a.seq_rank[i] = r;
        if (keys) {  // one replica: its sort records, indexed by gather position
          s_hi[i] = ~(uint64_t)__double_as_longlong(wv == 0.0 ? 0.0 : wv);
          s_lo[i] = id;
          s_v[i] = (uint32_t)i;
        }
      }
    };
    if (R == 1) {
      if (warp == 0) {
        // serial FP64 total in gather order (balancer.cpp:24-25; the replica
        // total of :147 is the same sum): the warp recomputes the workloads
        // from the lengths into the (not yet used) greedy-order scratch, lane 0
        // chains them
        const int n = (int)N;
        const double* wsrc = s_wsorted;
        if (N > kSmallScanSeqs) {
          // the sequence pass (warps 1..) writes s_w; wait for it on barrier 3
          // (producers only arrive) instead of reloading the lengths here
          asm volatile("bar.sync 3, %0;" ::"r"((int)blockDim.x) : "memory");
          wsrc = s_w;
        } else {
  #pragma unroll 4
          for (int i = lane; i < n; i += 32) s_wsorted[i] = raw_workload(i);
          __syncwarp();
        }
        double s = 0.0;
        if (lane == 0) {
          // 16-byte loads, the next group's issued before this group's DADDs
          // (the chain is the only serial part: ~8 cycles per element)
          const double2* v2 = reinterpret_cast<const double2*>(wsrc);
          int i = 0;
          if (n >= 8) {
            double2 c0 = v2[0], c1 = v2[1], c2 = v2[2], c3 = v2[3];
            for (i = 8; i + 8 <= n; i += 8) {
              const double2 d0 = v2[i / 2], d1 = v2[i / 2 + 1], d2 = v2[i / 2 + 2], d3 = v2[i / 2 + 3];
              s = __dadd_rn(s, c0.x); s = __dadd_rn(s, c0.y); s = __dadd_rn(s, c1.x); s = __dadd_rn(s, c1.y);
              s = __dadd_rn(s, c2.x); s = __dadd_rn(s, c2.y); s = __dadd_rn(s, c3.x); s = __dadd_rn(s, c3.y);
              c0 = d0; c1 = d1; c2 = d2; c3 = d3;
            }
            s = __dadd_rn(s, c0.x); s = __dadd_rn(s, c0.y); s = __dadd_rn(s, c1.x); s = __dadd_rn(s, c1.y);
            s = __dadd_rn(s, c2.x); s = __dadd_rn(s, c2.y); s = __dadd_rn(s, c3.x); s = __dadd_rn(s, c3.y);
          }
          for (; i < n; ++i) s = __dadd_rn(s, wsrc[i]);
        }
        if (MODE == 0) SB_P5(SB_MARK_MAX(11));  // diagnostics: totals chain done
        if (lane == 0) {
          *a.total = s;
          *a.n_seqs = N;
          s_reptot[0] = s;
          a.rep_total[0] = s;
        }
      } else if (N <= kSmallScanSeqs && warp == 1) {
        // origin packing offsets, few sequences: one warp scans the lengths in
        // gather order (32 per step) and rebases them per rank
        int64_t carry = 0;
        for (int64_t base = 0; base < N; base += 32) {
          const int64_t i = base + lane;
          int64_t v = i < N ? a.lens[i] : 0;
          v = v < 0 ? 0 : v;
          const int64_t inc = warp_incl_scan<int64_t>(v);
          if (i < N) s_soff[i] = carry + inc - v;
          carry += __shfl_sync(kFull, inc, 31);
        }
        __syncwarp();
        for (int r = lane; r <= W; r += 32) s_rpre[r] = s_roff[r] < N ? s_soff[s_roff[r]] : carry;
        __syncwarp();
        for (int64_t i = lane; i < N; i += 32) {
          s_soff[i] -= s_rpre[rank_of(i)];
          a.seq_off[i] = s_soff[i];
        }
        for (int r = lane; r < W; r += 32) a.origin_rows[r] = s_rpre[r + 1] - s_rpre[r];
        if (MODE == 0) SB_P5(SB_MARK_MAX(12));  // diagnostics: origin offsets done
      } else if (N <= kSmallScanSeqs) {
        seq_pass(tid - 64, (int)blockDim.x - 64, true);
      } else {
        // warps 1..: the per-sequence pass, then the origin packing offsets
        // (exclusive scan of the lengths in gather order, rebased per rank) as
        // a scan over these warps only, closed by named barrier 1 (one warp
        // walking 32 lengths per dependent step was the phase's critical path)
        const int t = tid - 32, nt = (int)blockDim.x - 32, tw = t >> 5, ntw = nt >> 5;
        auto bar = [nt]() { asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory"); };
        seq_pass(t, nt, true);
        asm volatile("bar.arrive 3, %0;" ::"r"((int)blockDim.x) : "memory");  // s_w ready for warp 0
        bar();
        const int n = (int)N;
        const int per = (n + nt - 1) / nt, b0 = t * per < n ? t * per : n, b1 = b0 + per < n ? b0 + per : n;
        int64_t loc = 0;
        for (int i = b0; i < b1; ++i) loc += s_lens[i];
        const int64_t inc = warp_incl_scan<int64_t>(loc);
        if (lane == 31) sh[tw] = inc;
        bar();
        if (tw == 0) {
          const int64_t x = lane < ntw ? sh[lane] : 0;
          const int64_t xi = warp_incl_scan<int64_t>(x);
          __syncwarp();
          if (lane < ntw) sh[lane] = xi - x;
          if (lane == ntw - 1) sh[32] = xi;
        }
        bar();
        int64_t run = sh[tw] + inc - loc;
        for (int i = b0; i < b1; ++i) {
          s_soff[i] = run;
          run += s_lens[i];
        }
        bar();
        for (int r = t; r <= W; r += nt) s_rpre[r] = s_roff[r] < N ? s_soff[s_roff[r]] : sh[32];
        bar();
        for (int i = t; i < n; i += nt) {
          s_soff[i] -= s_rpre[s_rank[i]];
          a.seq_off[i] = s_soff[i];
        }
        for (int r = t; r < W; r += nt) a.origin_rows[r] = s_rpre[r + 1] - s_rpre[r];
        if (MODE == 0) SB_P5(SB_MARK_MAX(12));  // diagnostics: origin offsets done
      }
      __syncthreads();
    } else {
      seq_pass(tid, (int)blockDim.x, false);
      __syncthreads();
      const int64_t per = (N + blockDim.x - 1) / blockDim.x;
      const int64_t b0 = tid * per, b1 = b0 + per < N ? b0 + per : N;
      int64_t loc = 0;
      for (int64_t i = b0; i < b1; ++i) loc += s_lens[i];
      int64_t tot;
      int64_t run = block_excl_scan<int64_t>(loc, sh, &tot);
      for (int64_t i = b0; i < b1; ++i) {
        s_soff[i] = run;
        run += s_lens[i];
      }
      __syncthreads();
      for (int r = tid; r <= W; r += blockDim.x) s_rpre[r] = s_roff[r] < N ? s_soff[s_roff[r]] : tot;
      __syncthreads();
      for (int64_t i = tid; i < N; i += blockDim.x) {
        s_soff[i] -= s_rpre[s_rank[i]];
        a.seq_off[i] = s_soff[i];
      }
      for (int r = tid; r < W; r += blockDim.x) a.origin_rows[r] = s_rpre[r + 1] - s_rpre[r];
      // serial totals (balancer.cpp:24-25, :147): global on warp 0, one
      // replica per lane of warp 1
      if (warp == 0 && lane == 0) {
        double s = 0.0;
        for (int64_t i = 0; i < N; ++i) s = __dadd_rn(s, s_w[i]);
        *a.total = s;
        *a.n_seqs = N;
      } else if (warp == 1) {
        for (int rep = lane; rep < R; rep += 32) {
          double s = 0.0;
          for (int64_t i = s_roff[rep * U]; i < s_roff[rep * U + U]; ++i) s = __dadd_rn(s, s_w[i]);
          s_reptot[rep] = s;
          a.rep_total[rep] = s;
        }
      }
      __syncthreads();
    }
    SB_PHASE(2);
    // ---- phase 2: per replica sort by (workload desc, id asc) (balancer.cpp:37-40);
    // each variant also gathers the workloads into greedy order
    for (int rep = 0; rep < R; ++rep) {
      const int64_t lo = s_roff[rep * U], n = s_roff[rep * U + U] - lo;
      if (R > 1) {
        for (int64_t i = tid; i < n; i += blockDim.x) {
          const double wv = s_w[lo + i];
          s_hi[i] = ~(uint64_t)__double_as_longlong(wv == 0.0 ? 0.0 : wv);
          s_lo[i] = s_ids[lo + i];
          s_v[i] = (uint32_t)i;
        }
        __syncthreads();
      }
      if (n > 32 && n <= 4 * kSmallThreads && blockDim.x == kSmallThreads) {
        const int nn = (int)n;
        int32_t* gs = a.sorted_idx;
        if (nn <= 64) reg_sort_emit<64, 1>(gs, s_hi, s_lo, s_v, s_sorted, s_w, s_wsorted, lo, nn);
        else if (nn <= 128) reg_sort_emit<128, 1>(gs, s_hi, s_lo, s_v, s_sorted, s_w, s_wsorted, lo, nn);
        else if (nn <= 256) reg_sort_emit<256, 1>(gs, s_hi, s_lo, s_v, s_sorted, s_w, s_wsorted, lo, nn);
        else if (nn <= 512) reg_sort_emit<512, 1>(gs, s_hi, s_lo, s_v, s_sorted, s_w, s_wsorted, lo, nn);
        else if (nn <= 1024) reg_sort_emit<1024, 2>(gs, s_hi, s_lo, s_v, s_sorted, s_w, s_wsorted, lo, nn);
      else reg_sort_emit<2048, 4>(gs, s_hi, s_lo, s_v, s_sorted, s_w, s_wsorted, lo, nn);
      } else if (n <= 1024) {
        // rank by counting: the key (~bits(w), id, index) is a total order.
        // k = blockDim/n lanes (power of two <= 32) share one record's count,
        // each over a slice of the candidates (broadcast smem reads), then a
        // shuffle reduction inside the k-lane group.
        const int nn = (int)n;
        int k = 1;
        while (k < 32 && 2 * k * nn <= (int)blockDim.x) k <<= 1;
        const int per = (nn + k - 1) / k;
        for (int base = 0; base < nn * k; base += blockDim.x) {
          const int x = base + tid;
          const int i = x / k, part = x % k;
          int pos = 0;
          if (i < nn) {
            const uint64_t hi_i = s_hi[i], lo_i = s_lo[i];
            const int j0 = part * per, j1 = j0 + per < nn ? j0 + per : nn;
  #pragma unroll 8
            for (int j = j0; j < j1; ++j) pos += rec_less(s_hi[j], s_lo[j], (uint32_t)j, hi_i, lo_i, (uint32_t)i);
          }
          for (int o = k >> 1; o > 0; o >>= 1) pos += __shfl_xor_sync(kFull, pos, o);
          if (i < nn && part == 0) {
            s_sorted[lo + pos] = (int32_t)(lo + i);
            s_wsorted[lo + pos] = s_w[lo + i];
            a.sorted_idx[lo + pos] = (int32_t)(lo + i);
          }
        }
      } else {
        smem_bitonic(s_hi, s_lo, s_v, (int)n, small_pow2((int)n));
        for (int64_t i = tid; i < n; i += blockDim.x) {
          s_sorted[lo + i] = (int32_t)(lo + s_v[i]);
          s_wsorted[lo + i] = s_w[lo + s_v[i]];
          a.sorted_idx[lo + i] = (int32_t)(lo + s_v[i]);
        }
      }
      __syncthreads();
    }
    if constexpr (MODE == 1) {
      // one replica: the greedy on warp 0 after every other warp has exited:
      // only then does ptxas prove the warp converged and schedule the
      // speculative FP64 work across the REDUX latencies (~107 cycles per step
      // instead of ~140-150 with live warps waiting, tools/micro/greedy_prod.cu)
      // Several replicas: the greedy-order workloads go to the 32-thread greedy
      // kernel, one CTA per replica (a replica loop here, with bounds ptxas
      // cannot prove warp-uniform, would bring the guard back).
      for (int64_t p = tid; p < N; p += blockDim.x) a.sorted_w[p] = s_wsorted[p];
      SB_PHASE(12);  // trace: phases 0-2 done
      if (R != 1 || warp != 0) return;
      const int rep = 0;
      const int64_t lo = 0;
      const int n = (int)(s_roff[rep * U + U] - lo);
      const double* ws = s_wsorted + lo;  // reads up to 3 past the replica's end: unused values
      int32_t* pk = s_pick + lo;
      if (M <= 32)
        greedy_warp<1, 0, false, true>(a, rep, n, s_reptot[rep], [ws](int p) { return ws[p]; }, [](int) {}, pk,
                                       nullptr, a.violations);
      else
        greedy_warp<2, 0, false, true>(a, rep, n, s_reptot[rep], [ws](int p) { return ws[p]; }, [](int) {}, pk,
                                       nullptr, a.violations);
      // each position's rank inside its bag (match_any pass), picks and ranks
      // out in the same pass (bag_ranks_pass plus a separate pick loop measured
      // 1-2 us slower per plan)
      int32_t* cnt = s_bagcnt + rep * M;
      for (int j = lane; j < M; j += 32) cnt[j] = 0;
      __syncwarp();
      const unsigned lt = (1u << lane) - 1u;
      for (int p0 = 0; p0 < n; p0 += 32) {
        const int p = p0 + lane;
        const bool valid = p < n;
        const int b = valid ? pk[p] : -1;
        const unsigned peers = __match_any_sync(kFull, b);
        const int rank_in = __popc(peers & lt);
        const int base = valid ? cnt[b] : 0;
        __syncwarp();
        if (valid && rank_in == 0) cnt[b] = base + __popc(peers);
        __syncwarp();
        if (valid) {
          a.pick[lo + p] = b;
          a.greedy_q[lo + p] = base + rank_in;
        }
      }
      return;
    }
  } else {  // hybrid suffix
    SB_PHASE(11);  // trace: suffix start
    // ---- MODE 2, launched as a programmatic dependent of the prefix (or of the
    // greedy kernel): until the grid dependency resolves it touches inputs only
    // -- phase 0 above, the ids and lengths, and the duplicate-id check, all
    // under the prefix's greedy chain
    for (int64_t i = tid; i < N; i += blockDim.x) {
      const int64_t len = a.lens[i] < 0 ? 0 : a.lens[i];
      if (len >= (int64_t)1 << 26) s_biglen = 1;
      s_ids[i] = a.ids[i];
      s_lens[i] = len;
    }
    __syncthreads();
    if (!a.w_in) dup_check(tid, (int)blockDim.x);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // then what phases 0-2 and the greedy left in global memory
    for (int64_t i = tid; i < N; i += blockDim.x) {
      s_rank[i] = a.seq_rank[i];
      s_soff[i] = a.seq_off[i];
      s_sorted[i] = a.sorted_idx[i];
      s_pick[i] = a.pick[i];
      s_q[i] = a.greedy_q[i];
    }
    for (int e = tid; e < R * M; e += blockDim.x) s_bagcnt[e] = a.bag_count[e];
    if (tid == 0 && s_flag) atomicOr(a.status, ST_DUP_ID);  // after the prefix reset the status word
    __syncthreads();
  }
  SB_PHASE(3);
  // ---- phase 3: greedy, one warp per replica (balancer.cpp:44-62), beside
  // the duplicate-id check inside each replica (divergence)
  const int ng = R < nw - 2 ? R : nw - 2;
  // one replica: warp 1 derives the bag ranks from the picks (handed over on
  // named barrier 4) while warp 0 finishes the per-bag epilogue and the bag
  // bases; the duplicate check then runs on warps 2..
  const bool qsplit = MODE == 0 && R == 1 && nw >= 4;
  if (warp < ng) {
    for (int rep = warp; rep < R; rep += ng) {
      const int64_t lo = s_roff[rep * U], n = s_roff[rep * U + U] - lo;
      if constexpr (MODE == 0) {
        const double* ws = s_wsorted + lo;
        if (M <= 32) small_greedy<1>(a, rep, n, s_reptot[rep], ws, s_pick + lo, s_bagcnt, &s_viol, s_q + lo, qsplit);
        else small_greedy<2>(a, rep, n, s_reptot[rep], ws, s_pick + lo, s_bagcnt, &s_viol, s_q + lo, qsplit);
        __syncwarp();
        if (rep == 0) SB_P3(8);
      }
      // replica-local chunk bases of the bags (chunk order: bag, q, k) and
      // the bags' first slots in the (replica, bag)-grouped sequence list
      int cb = 0, q = (int)lo;  // <= cap * kMaxBags chunks: 32 bits
      for (int x0 = 0; x0 < M; x0 += 32) {
        const int x = x0 + lane;
        const int nb = x < M ? s_bagcnt[rep * M + x] : 0;
        const int c = x < M ? nb * a.bag_size[x] : 0;
        const int ic = warp_incl_scan<int>(c), iq = warp_incl_scan<int>(nb);
        if (x < M) {
          s_bagcb[rep * M + x] = cb + ic - c;
          s_bagq[rep * M + x] = q + iq - nb;
        }
        cb += __shfl_sync(kFull, ic, 31);
        q += __shfl_sync(kFull, iq, 31);
      }
      if (lane == 0) {
        s_repc[rep] = cb;
        a.rep_chunks[rep] = cb;
        if (R == 1) *a.n_chunks = cb;
      }
      if (rep == 0) SB_P3(9);
    }
  } else if (qsplit && warp == 1) {
    int32_t* qc = reinterpret_cast<int32_t*>(sm + L.qcnt);
    for (int j = lane; j < M; j += 32) qc[j] = 0;
    __syncwarp();
    asm volatile("bar.sync 4, 64;" ::: "memory");
    bag_ranks_pass(s_pick, (int)N, qc, s_q);
  } else if (MODE == 0 && !a.w_in) {  // the hybrid's suffix runs it before its grid dependency
    const int w0 = ng + (qsplit ? 1 : 0);
    const int t = tid - 32 * w0;
    dup_check(t, (int)blockDim.x - 32 * w0);
    if (s_flag && t == 0) atomicOr(a.status, ST_DUP_ID);
  }
  __syncthreads();
  if (R > 1) {
    // replica chunk bases (chunk order: replica, bag, q, k)
    if (warp == 0) {
      int64_t carry = 0;
      for (int x0 = 0; x0 < R; x0 += 32) {
        const int x = x0 + lane;
        const int64_t c = x < R ? s_repc[x] : 0;
        const int64_t inc = warp_incl_scan<int64_t>(c);
        if (x < R) s_repc[x] = carry + inc - c;
        carry += __shfl_sync(kFull, inc, 31);
      }
      __syncwarp();
      for (int e = lane; e < R * M; e += 32) s_bagcb[e] += s_repc[e / M];
      if (lane == 0) *a.n_chunks = carry;
    }
    __syncthreads();
  }
  SB_PHASE(4);
  // ---- phase 4: stable bag partition (balancer.cpp:178-192), one thread per
  // sequence: the greedy recorded each sequence's rank q in its bag, so its
  // chunks are [bag base + q * g, + g) and its slot in the grouped list is
  // bag first slot + q.  Warp 0 computes the WIR beside it.
  if (warp == 0) {
    if (MODE == 0)
      for (int r = lane; r < W; r += 32) a_in.per_gpu[r] = a.per_gpu[r];
    // min and max are order-independent (no NaN) (metrics.cpp:20-31)
    double lo = a.per_gpu[0], hi = lo;
    for (int r = lane; r < W; r += 32) {
      const double v = a.per_gpu[r];
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(kFull, lo, o));
      hi = fmax(hi, __shfl_xor_sync(kFull, hi, o));
    }
    if (lane == 0) {
      *a.wir = hi == 0.0 ? 1.0 : (lo == 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : __ddiv_rn(hi, lo));
      if (MODE == 0) *a.violations = s_viol;
    }
  } else {
    for (int64_t p = tid - 32; p < N; p += (int)blockDim.x - 32) {
      const int s = s_sorted[p];
      const int b = s_pick[p], q = s_q[p];
      const int src = s_rank[s];
      const int rep = src / U;
      const int rb = rep * M + b;
      const int g = a.bag_size[b];
      const int64_t cb = s_bagcb[rb] + (int64_t)q * g;
      s_G[s] = g;
      s_cb[s] = cb;
      s_bo[s_bagq[rb] + q] = s;
      a.seq_G[s] = g;
      a.seq_chunk_base[s] = cb;
      atomicAdd(reinterpret_cast<unsigned long long*>(&s_sendcnt[src]), (unsigned long long)g);
    }
    SB_MARK_MAX(10);
  }
  __syncthreads();
  SB_PHASE(5);
  // ---- phase 5: manifests (balancer.cpp:84-101, reverse order :259-285)
  // recv list + receive-side rows (target packing) + Ulysses sequence bases
  // of rank r, and its reverse receive order: r's sequences in buffer order,
  // chunks ascending.  Warp-wide; ro / so = r's recv / send list offsets.
  auto rank_lists = [&](int r, int64_t ro, int64_t so) {
    const int rep = r / U, u = r % U;
    const int b = a.rank_bag[u], k = a.rank_member[u], g = a.bag_size[b];
    const int nb = s_bagcnt[rep * M + b];
    const int bq = s_bagq[rep * M + b];
    int64_t carry = 0, carry2 = 0;
    for (int q0 = 0; q0 < nb; q0 += 32) {
      const int q = q0 + lane;
      const bool valid = q < nb;
      const int s = valid ? s_bo[bq + q] : 0;
      const int64_t l = valid ? s_lens[s] : 0;
      const int64_t len = valid ? chunk_len(l, g, k) : 0;
      int64_t inc, inc2 = 0;
      if (!s_biglen) {  // block-uniform: every 32-lane partial sum fits in 32 bits
        inc = warp_incl_scan<int>((int)len);
        if (k == 0) inc2 = warp_incl_scan<int>((int)l);
      } else {
        inc = warp_scan_incl64(len);
        if (k == 0) inc2 = warp_scan_incl64(l);
      }
      if (valid) {
        const int64_t c = s_cb[s] + k;
        a.c_dst_row[c] = carry + inc - len;
        a.recv_idx[ro + q] = (int32_t)c;
        if (k == 0) a.c_seq_base[s_cb[s]] = carry2 + inc2 - l;
      }
      carry += __shfl_sync(kFull, inc, 31);
      if (k == 0) carry2 += __shfl_sync(kFull, inc2, 31);
    }
    if (lane == 0) {
      a.target_rows[r] = carry;
      if (k == 0) a.bag_rows[rep * M + b] = carry2;
    }
    const int64_t s0 = s_roff[r], s1 = s_roff[r + 1];
    int64_t c4 = 0;
    bool tie = false;  // a sequence shorter than its bag: equal (segment, start) keys
    for (int64_t i0 = s0; i0 < s1; i0 += 32) {
      const int64_t i = i0 + lane;
      const bool valid = i < s1;
      const int gs = valid ? s_G[i] : 0;
      tie |= gs > 1 && s_lens[i] < gs;
      const int64_t inc = warp_incl_scan<int>(gs);  // <= 32 * kMaxBags
      if (valid)
        for (int kk = 0; kk < gs; ++kk) a.rev_recv_idx[so + c4 + inc - gs + kk] = (int32_t)(s_cb[i] + kk);
      c4 += __shfl_sync(kFull, inc, 31);
    }
    tie = __any_sync(kFull, tie);
    if (lane == 0) s_tie[r] = tie ? 1 : 0;
  };
  // send list of the rank of sequence i: r's sequences ordered by first
  // chunk index (counting, no sort); so = the rank's send offset
  auto send_list = [&](int64_t i, int64_t so) {
    const int r = s_rank[i];
    const int64_t cb = s_cb[i];
    int64_t pos = 0;
    for (int64_t j = s_roff[r]; j < s_roff[r + 1]; ++j)
      if (s_cb[j] < cb) pos += s_G[j];
    for (int kk = 0; kk < s_G[i]; ++kk) a.send_idx[so + pos + kk] = (int32_t)(cb + kk);
  };
  // chunk emission (balancer.cpp:194-218), one thread per chunk (coalesced
  // stores): bag rb = (rep, b) holds chunks [bagcb[rb], bagcb[rb] + count * g)
  // in its sequences' bag order; a chunk finds its bag by binary search
  const int RM = R * M;
  const int64_t n_chunks = s_bagcb[RM - 1] + (int64_t)s_bagcnt[RM - 1] * a.bag_size[M - 1];
  auto emit_chunk = [&](int64_t c) -> int {  // returns the chunk's source rank
    int blo = 0, bhi = RM;  // last bag with base <= c (empty bags share the base of the next)
    while (bhi - blo > 1) {
      const int mid = (blo + bhi) >> 1;
      if (s_bagcb[mid] <= c) blo = mid;
      else bhi = mid;
    }
    const int rep = blo / M, b = blo - rep * M;
    const int g = a.bag_size[b];
    const uint32_t e = (uint32_t)(c - s_bagcb[blo]);
    const int q = (int)(e / (uint32_t)g), k = (int)(e - (uint32_t)q * (uint32_t)g);
    const int s = s_bo[s_bagq[blo] + q];
    int64_t cq;
    int cr;
    len_divmod(s_lens[s], g, cq, cr);
    const int64_t st = (int64_t)k * cq + (k < cr ? k : cr);
    a.c_id[c] = s_ids[s];
    a.c_idx[c] = k;
    a.c_start[c] = st;
    a.c_end[c] = st + cq + (k < cr ? 1 : 0);
    a.c_src[c] = s_rank[s];
    a.c_dst[c] = rep * U + a.bag_ranks[a.bag_off[b] + k];
    a.c_src_row[c] = s_soff[s] + st;
    a.c_seq[c] = s;
    return s_rank[s];
  };
  // chunk emission and send lists go to the highest threads first: warps
  // without a rank list take them while the rank warps scan
  const int rtid = (int)blockDim.x - 1 - tid;
  if (W <= 32) {
    // every warp scans the per-rank counts itself: lane r holds rank r's
    // send / recv offsets (no extra barrier)
    // 32-bit scans: counts are bounded by the plan's chunk capacity
    const int sc = lane < W ? (int)s_sendcnt[lane] : 0;
    const int rc = lane < W ? s_bagcnt[(lane / U) * M + a.rank_bag[lane % U]] : 0;
    const int is = warp_incl_scan<int>(sc), ir = warp_incl_scan<int>(rc);
    const int so_l = is - sc, ro_l = ir - rc;
    if (warp == 0) {
      if (lane < W) {
        s_sendoff[lane] = so_l;
        a.send_off[lane] = so_l;
        a.recv_off[lane] = ro_l;
      }
      if (lane == W - 1) {
        s_sendoff[W] = is;
        a.send_off[W] = is;
        a.recv_off[W] = ir;
      }
    }
    SB_P5(SB_MARK(7));
    if (N > kSmallScanSeqs && 2 * W <= nw) {
      // send[r] = the chunks of source r in chunk order (finalize_manifests,
      // balancer.cpp:84-91): a stable filter of the chunk array by source
      // rank, emitted tile by tile on warps [W, nw) (match_any + per-warp
      // counts, double-buffered, named barrier 1) while warps [0, W) build
      // the rank lists -- O(chunks) instead of counting over each rank's
      // sequences
      __shared__ int s_wcnt[2][kSmallThreads / 32][32];
      __shared__ int s_run[32];
      if (warp < W) {
        rank_lists(warp, __shfl_sync(kFull, ro_l, warp), __shfl_sync(kFull, so_l, warp));
        SB_P5(SB_MARK_MAX(8));
      } else {
        const int t0 = tid - 32 * W, nt = (int)blockDim.x - 32 * W, tw = warp - W, ntw = nw - W;
        auto bar = [nt]() { asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory"); };
        if (t0 < 32) s_run[t0] = 0;
        const unsigned lt = (1u << lane) - 1u;
        for (int64_t base = 0, t = 0; base < n_chunks; base += nt, ++t) {
          const int64_t c = base + t0;
          const bool valid = c < n_chunks;
          const int r = valid ? emit_chunk(c) : -1;
          const unsigned peers = __match_any_sync(kFull, r);
          const int rank_in = __popc(peers & lt);
          int* wc = &s_wcnt[t & 1][tw][0];
          if (lane < W) wc[lane] = 0;
          __syncwarp();
          if (valid && rank_in == 0) wc[r] = __popc(peers);
          bar();
          if (tw == 0 && lane < W) {  // exclusive prefix over the warps, after the earlier tiles
            int run = s_run[lane];
            for (int w = 0; w < ntw; ++w) {
              const int x = s_wcnt[t & 1][w][lane];
              s_wcnt[t & 1][w][lane] = run;
              run += x;
            }
            s_run[lane] = run;
          }
          bar();
          const int64_t so = __shfl_sync(kFull, so_l, valid ? r : 0);
          if (valid) a.send_idx[so + wc[r] + rank_in] = (int32_t)c;
        }
        SB_P5(SB_MARK_MAX(9));
      }
    } else {
      for (int r = warp; r < W; r += nw) rank_lists(r, __shfl_sync(kFull, ro_l, r), __shfl_sync(kFull, so_l, r));
      SB_P5(SB_MARK_MAX(8));
      for (int64_t c = rtid; c < n_chunks; c += blockDim.x) emit_chunk(c);
      for (int64_t b0 = 0; b0 < N; b0 += blockDim.x) {  // warp-uniform trip count (the shuffle below)
        const int64_t i = b0 + rtid;
        const int r = i < N ? s_rank[i] : 0;
        const int64_t so = __shfl_sync(kFull, so_l, r);
        if (i < N) send_list(i, so);
      }
      SB_P5(SB_MARK_MAX(9));
    }
  } else {
    if (warp == 0) {
      int64_t so = 0, ro = 0;
      for (int r0 = 0; r0 < W; r0 += 32) {
        const int r = r0 + lane;
        const int64_t sc = r < W ? s_sendcnt[r] : 0;
        const int64_t rc = r < W ? (int64_t)s_bagcnt[(r / U) * M + a.rank_bag[r % U]] : 0;
        const int64_t is = warp_incl_scan<int64_t>(sc), ir = warp_incl_scan<int64_t>(rc);
        if (r < W) {
          s_sendoff[r] = so + is - sc;
          a.send_off[r] = so + is - sc;
          a.recv_off[r] = ro + ir - rc;
          s_recvoff[r] = ro + ir - rc;
        }
        so += __shfl_sync(kFull, is, 31);
        ro += __shfl_sync(kFull, ir, 31);
      }
      if (lane == 0) {
        s_sendoff[W] = so;
        a.send_off[W] = so;
        a.recv_off[W] = ro;
      }
    }
    __syncthreads();
    for (int r = warp; r < W; r += nw) rank_lists(r, s_recvoff[r], s_sendoff[r]);
    for (int64_t c = rtid; c < n_chunks; c += blockDim.x) emit_chunk(c);
    for (int64_t i = rtid; i < N; i += blockDim.x) send_list(i, s_sendoff[s_rank[i]]);
  }
  __syncthreads();  // send lists complete: reverse-order tie replay reads them
  SB_PHASE(6);
  for (int r = warp; r < W; r += nw)
    if (lane == 0 && s_tie[r]) {
      stdsort::Frame stk[stdsort::kStackFrames];
      fix_rev_ties(a.rev_recv_idx, a.send_idx, a.c_seq, a.c_start, s_sendoff[r], s_sendoff[r + 1] - s_sendoff[r], stk);
    }
  SB_PHASE(13);
}

}  // namespace sb
