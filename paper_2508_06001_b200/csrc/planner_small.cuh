// Single-CTA planner for small batches (up to kSmallSeqs sequences).
//
// The multi-kernel pipeline in planner.cu is launch-latency bound when a
// step carries a few dozen sequences (C2: 30): six launches, each paying a
// kernel start and a cold read of what the previous one wrote.  Here one
// 1024-thread CTA keeps every per-sequence array in shared memory and runs
// the same phases back to back, separated by __syncthreads:
//   load + workload + origin offsets -> duplicate check (sort by id) ->
//   serial FP64 totals -> sort by (workload desc, id asc) -> greedy (warp
//   per replica) -> stable bag partition + chunk emission -> manifests,
//   receive rows, Ulysses bases, reverse order -> WIR.
// Results are bit-identical to the large path (tests/test_gpu_parity.py
// runs both on the same inputs).
#pragma once

namespace sb {

// Per-phase clock64() trace (thread 0) when the planner has a trace buffer.
#define SB_PHASE(k)                                   \
  do {                                                \
    if (a.trace && threadIdx.x == 0) a.trace[k] = clock64(); \
  } while (0)

constexpr int kSmallSeqs = 2048;
constexpr int kSmallThreads = 512;  // 128 registers per thread: the greedy keeps its speculation in registers

__host__ __device__ inline int small_pow2(int n) {
  int t = 32;
  while (t < n) t <<= 1;
  return t;
}

struct SmallLayout {  // byte offsets into dynamic shared memory
  size_t ids, lens, w, soff, hi, lo, v, rank, sorted, pick, G, cb, bo, rank_off, rpre, bagcnt, bagcb, bagq,
      sendcnt, sendoff, reptot, tie, t_boff, t_branks, t_bsize, t_rbag, t_rmem, pergpu, recvoff, total;
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
  L.t_boff = take(4ull * (M + 1));  // topology tables, staged once (read by every phase)
  L.t_branks = take(4ull * U);
  L.t_bsize = take(4ull * M);
  L.t_rbag = take(4ull * U);
  L.t_rmem = take(4ull * U);
  L.pergpu = take(8ull * W);  // per-GPU workload: the greedy writes it, WIR reads it
  L.recvoff = take(8ull * W);
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
__device__ void reg_sort_emit(const PlanArgs& a, uint64_t* s_hi, uint64_t* s_lo, uint32_t* s_v, int32_t* s_sorted,
                              int64_t lo, int n) {
  uint64_t h[RPT], l[RPT];
  uint32_t v[RPT];
  reg_bitonic<T, RPT, kSmallThreads>(s_hi, s_lo, s_v, n, h, l, v);
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int x = threadIdx.x + r * kSmallThreads;
    if (x < n) {
      s_sorted[lo + x] = (int32_t)(lo + v[r]);
      a.sorted_idx[lo + x] = (int32_t)(lo + v[r]);
    }
  }
}

// Warp-level inclusive scan helper over int64.
__device__ __forceinline__ int64_t warp_scan_incl64(int64_t x) { return warp_incl_scan<int64_t>(x); }

template <int BPL>
__device__ void small_greedy(const PlanArgs& a, int rep, int64_t lo, int64_t n, const double* s_w, const int32_t* s_sorted,
                             int32_t* s_pick, int32_t* s_bagcnt, double total_rep, int* viol_out) {
  const double* ws = s_w + lo;  // workloads already gathered into greedy order
  greedy_warp<BPL, 0>(a, rep, n, total_rep, [ws](int p) { return ws[p]; }, [](int) {}, s_pick + lo, s_bagcnt,
                      viol_out);
}

__global__ void __launch_bounds__(kSmallThreads) k_plan_small(PlanArgs a_in, int cap) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int64_t sh[33];
  __shared__ int s_flag, s_viol, s_biglen;
  __shared__ int warp_cnt[32][kMaxBags];
  __shared__ int running[kMaxBags];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
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
  int32_t* s_bo = reinterpret_cast<int32_t*>(sm + L.bo);
  int64_t* s_roff = reinterpret_cast<int64_t*>(sm + L.rank_off);
  int64_t* s_rpre = reinterpret_cast<int64_t*>(sm + L.rpre);
  int32_t* s_bagcnt = reinterpret_cast<int32_t*>(sm + L.bagcnt);
  int64_t* s_bagcb = reinterpret_cast<int64_t*>(sm + L.bagcb);
  int32_t* s_bagq = reinterpret_cast<int32_t*>(sm + L.bagq);
  int64_t* s_sendcnt = reinterpret_cast<int64_t*>(sm + L.sendcnt);
  int64_t* s_sendoff = reinterpret_cast<int64_t*>(sm + L.sendoff);
  int32_t* s_tie = reinterpret_cast<int32_t*>(sm + L.tie);
  double* s_reptot = reinterpret_cast<double*>(sm + L.reptot);

  SB_PHASE(0);
  // ---- phase 0: rank offsets, capacity, topology tables
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
    a.per_gpu = reinterpret_cast<double*>(sm + L.pergpu);
  }
  if (tid == 0) {
    s_flag = 0;
    s_viol = 0;
    s_biglen = 0;
    *a.status = 0;  // no memset node before the launch; every atomicOr below follows this barrier
  }
  __syncthreads();
  const int64_t N = s_roff[W];
  if (N > cap) {
    if (tid == 0) atomicOr(a.status, ST_CAPACITY);
    return;
  }
  SB_PHASE(1);
  // ---- phase 1: metadata, workloads, ranks (balancer.cpp:139-149)
  for (int64_t i = tid; i < N; i += blockDim.x) {
    int lo = 0, hi = W;  // rank r with roff[r] <= i < roff[r+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_roff[mid] <= i) lo = mid;
      else hi = mid;
    }
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
    s_ids[i] = a.ids[i];
    s_lens[i] = len;
    s_w[i] = wv;
    s_rank[i] = lo;
    a.w[i] = wv;
    a.seq_rank[i] = lo;
  }
  __syncthreads();
  SB_PHASE(2);
  // ---- phase 2: origin packing offsets (exclusive scan of lens in gather
  // order, rebased per rank).  One replica: warp 1 does it inside phases 3+4,
  // beside the totals and the duplicate check (origin_offsets_warp below)
  auto origin_offsets_warp = [&]() {
    int64_t carry = 0;
    for (int64_t base = 0; base < N; base += 32) {
      const int64_t i = base + lane;
      const int64_t v = i < N ? s_lens[i] : 0;
      const int64_t inc = warp_incl_scan<int64_t>(v);
      if (i < N) s_soff[i] = carry + inc - v;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    __syncwarp();
    for (int r = lane; r <= W; r += 32) s_rpre[r] = s_roff[r] < N ? s_soff[s_roff[r]] : carry;
    __syncwarp();
    for (int64_t i = lane; i < N; i += 32) {
      s_soff[i] -= s_rpre[s_rank[i]];
      a.seq_off[i] = s_soff[i];
    }
    for (int r = lane; r < W; r += 32) {
      a.origin_rows[r] = s_rpre[r + 1] - s_rpre[r];
      s_sendcnt[r] = 0;
    }
  };
  if (R > 1) {
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
    for (int r = tid; r < W; r += blockDim.x) {
      a.origin_rows[r] = s_rpre[r + 1] - s_rpre[r];
      s_sendcnt[r] = 0;
    }
    __syncthreads();
  }
  SB_PHASE(3);
  // ---- phases 3+4 side by side: warps 0-1 run the serial FP64 totals
  // (balancer.cpp:24-25, :147) while warps 2.. check for duplicate sample ids
  // inside each replica (divergence); named barrier 2 syncs
  // the checking warps only.  One replica: its total is the report total
  // (same additions, same order).
  if (warp == 0) {
    if (lane == 0) {
      double s = 0.0;
      for (int64_t i = 0; i < N; ++i) s = __dadd_rn(s, s_w[i]);
      *a.total = s;
      *a.n_seqs = N;
      if (R == 1) {
        s_reptot[0] = s;
        a.rep_total[0] = s;
      }
    }
  } else if (warp == 1) {
    if (R == 1) origin_offsets_warp();
    else
      for (int rep = lane; rep < R; rep += 32) {
        double s = 0.0;
        for (int64_t i = s_roff[rep * U]; i < s_roff[rep * U + U]; ++i) s = __dadd_rn(s, s_w[i]);
        s_reptot[rep] = s;
        a.rep_total[rep] = s;
      }
  } else if (!a.w_in) {
    // open-addressing set per replica in the (not yet used) sort scratch:
    // s_hi and s_lo are contiguous, 2T slots >= 2 * replica size, EMPTY = ~0
    const int t = tid - 64, nt = (int)blockDim.x - 64;
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
    if (s_flag && t == 0) atomicOr(a.status, ST_DUP_ID);
  }
  __syncthreads();
  SB_PHASE(4);
  SB_PHASE(5);
  // ---- phase 5: per replica sort by (workload desc, id asc) (balancer.cpp:37-40)
  for (int rep = 0; rep < R; ++rep) {
    const int64_t lo = s_roff[rep * U], n = s_roff[rep * U + U] - lo;
    for (int64_t i = tid; i < n; i += blockDim.x) {
      const double wv = s_w[lo + i];
      s_hi[i] = ~(uint64_t)__double_as_longlong(wv == 0.0 ? 0.0 : wv);
      s_lo[i] = s_ids[lo + i];
      s_v[i] = (uint32_t)i;
    }
    __syncthreads();
    if (n > 32 && n <= 2 * kSmallThreads && blockDim.x == kSmallThreads) {
      const int nn = (int)n;
      if (nn <= 64) reg_sort_emit<64, 1>(a, s_hi, s_lo, s_v, s_sorted, lo, nn);
      else if (nn <= 128) reg_sort_emit<128, 1>(a, s_hi, s_lo, s_v, s_sorted, lo, nn);
      else if (nn <= 256) reg_sort_emit<256, 1>(a, s_hi, s_lo, s_v, s_sorted, lo, nn);
      else if (nn <= 512) reg_sort_emit<512, 1>(a, s_hi, s_lo, s_v, s_sorted, lo, nn);
      else reg_sort_emit<1024, 2>(a, s_hi, s_lo, s_v, s_sorted, lo, nn);
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
        for (int o = k >> 1; o > 0; o >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, o);
        if (i < nn && part == 0) {
          s_sorted[lo + pos] = (int32_t)(lo + i);
          a.sorted_idx[lo + pos] = (int32_t)(lo + i);
        }
      }
    } else {
      smem_bitonic(s_hi, s_lo, s_v, (int)n, small_pow2((int)n));
      for (int64_t i = tid; i < n; i += blockDim.x) {
        s_sorted[lo + i] = (int32_t)(lo + s_v[i]);
        a.sorted_idx[lo + i] = (int32_t)(lo + s_v[i]);
      }
    }
    __syncthreads();
  }
  SB_PHASE(6);
  // ---- phase 6: greedy, one warp per replica (balancer.cpp:44-62), over the
  // workloads gathered into greedy order (the sort scratch is free now)
  double* s_wsorted = reinterpret_cast<double*>(s_hi);
  for (int64_t i = tid; i < N; i += blockDim.x) s_wsorted[i] = s_w[s_sorted[i]];
  __syncthreads();
  for (int rep = warp; rep < R; rep += nw) {
    const int64_t lo = s_roff[rep * U], n = s_roff[rep * U + U] - lo;
    if (M <= 32) small_greedy<1>(a, rep, lo, n, s_wsorted, nullptr, s_pick, s_bagcnt, s_reptot[rep], &s_viol);
    else small_greedy<2>(a, rep, lo, n, s_wsorted, nullptr, s_pick, s_bagcnt, s_reptot[rep], &s_viol);
  }
  __syncthreads();
  SB_PHASE(7);
  // ---- phase 7: chunk bases of every (replica, bag): warp 0 scans the
  // (replica, bag) counts 32 at a time
  if (warp == 0) {
    int64_t cb = 0, q = 0;
    for (int x0 = 0; x0 < R * M; x0 += 32) {
      const int x = x0 + lane;
      const int64_t n = x < R * M ? s_bagcnt[x] : 0;
      const int64_t c = x < R * M ? n * a.bag_size[x % M] : 0;
      const int64_t ic = warp_incl_scan<int64_t>(c), iq = warp_incl_scan<int64_t>(n);
      if (x < R * M) {
        s_bagcb[x] = cb + ic - c;
        s_bagq[x] = (int32_t)(q + iq - n);
      }
      cb += __shfl_sync(0xffffffffu, ic, 31);
      q += __shfl_sync(0xffffffffu, iq, 31);
    }
    __syncwarp();
    for (int rep = lane; rep < R; rep += 32) {
      const int64_t e = rep + 1 < R ? s_bagcb[(rep + 1) * M] : cb;
      a.rep_chunks[rep] = e - s_bagcb[rep * M];
    }
    if (lane == 0) {
      *a.n_chunks = cb;
      *a.violations = s_viol;
    }
  }
  __syncthreads();
  SB_PHASE(8);
  // ---- phase 8: stable bag partition + chunk emission (balancer.cpp:178-218)
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int rep = 0; rep < R; ++rep) {
    const int64_t lo = s_roff[rep * U], hi = s_roff[rep * U + U];
    for (int b = tid; b < M; b += blockDim.x) running[b] = 0;
    __syncthreads();
    for (int64_t tile = lo; tile < hi; tile += blockDim.x) {
      for (int e = tid; e < nw * M; e += blockDim.x) warp_cnt[e / M][e % M] = 0;
      __syncthreads();
      const int64_t p = tile + tid;
      const bool valid = p < hi;
      const int b = valid ? s_pick[p] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      const int rank_in = __popc(peers & lt_mask);
      if (valid && rank_in == 0) warp_cnt[warp][b] = __popc(peers);
      __syncthreads();
      for (int b2 = warp; b2 < M; b2 += nw) {  // warp b2 scans bag b2's per-warp counts
        const int c = lane < nw ? warp_cnt[lane][b2] : 0;
        const int inc = warp_incl_scan<int>(c);
        const int run = running[b2];
        __syncwarp();
        if (lane < nw) warp_cnt[lane][b2] = run + inc - c;
        if (lane == 31) running[b2] = run + inc;
      }
      __syncthreads();
      if (valid) {
        const int q = warp_cnt[warp][b] + rank_in;
        const int s = s_sorted[p];
        const int g = a.bag_size[b];
        const int64_t cb = s_bagcb[rep * M + b] + (int64_t)q * g;
        const int src = s_rank[s];
        s_G[s] = g;
        s_cb[s] = cb;
        s_bo[s_bagq[rep * M + b] + q] = s;
        a.seq_G[s] = g;
        a.seq_chunk_base[s] = cb;
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_sendcnt[src]), (unsigned long long)g);
      }
      __syncthreads();
    }
  }
  // chunk emission, one thread per chunk (coalesced stores): bag rb =
  // (rep, b) holds chunks [bagcb[rb], bagcb[rb] + count * g) in its
  // sequences' bag order; a chunk finds its bag by binary search
  {
    const int RM = R * M;
    const int64_t total = s_bagcb[RM - 1] + (int64_t)s_bagcnt[RM - 1] * a.bag_size[M - 1];
    for (int64_t c = tid; c < total; c += blockDim.x) {
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
    }
  }
  __syncthreads();
  SB_PHASE(9);
  // ---- phase 9: manifest offsets (balancer.cpp:84-91), warp 0 scans 32
  // ranks at a time
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
        reinterpret_cast<int64_t*>(sm + L.recvoff)[r] = ro + ir - rc;
      }
      so += __shfl_sync(0xffffffffu, is, 31);
      ro += __shfl_sync(0xffffffffu, ir, 31);
    }
    if (lane == 0) {
      s_sendoff[W] = so;
      a.send_off[W] = so;
      a.recv_off[W] = ro;
    }
  }
  __syncthreads();
  SB_PHASE(10);
  // ---- phase 10: per rank lists, one warp per rank
  for (int r = warp; r < W; r += nw) {
    const int rep = r / U, u = r % U;
    const int b = a.rank_bag[u], k = a.rank_member[u], g = a.bag_size[b];
    const int nb = s_bagcnt[rep * M + b];
    const int bq = s_bagq[rep * M + b];
    const int64_t ro = reinterpret_cast<const int64_t*>(sm + L.recvoff)[r];
    // recv list + receive-side rows (target packing, balancer.cpp:93-101)
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
      carry += __shfl_sync(0xffffffffu, inc, 31);
      if (k == 0) carry2 += __shfl_sync(0xffffffffu, inc2, 31);
    }
    if (lane == 0) {
      a.target_rows[r] = carry;
      if (k == 0) a.bag_rows[rep * M + b] = carry2;
    }
    // reverse receive order: r's sequences in buffer order, chunks ascending
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
        for (int kk = 0; kk < gs; ++kk) a.rev_recv_idx[s_sendoff[r] + c4 + inc - gs + kk] = (int32_t)(s_cb[i] + kk);
      c4 += __shfl_sync(0xffffffffu, inc, 31);
    }
    tie = __any_sync(0xffffffffu, tie);
    if (lane == 0) s_tie[r] = tie ? 1 : 0;
  }
  __syncthreads();
  SB_PHASE(11);
  // ---- phase 11: send lists -- r's sequences ordered by first chunk index
  // position of sequence i in send[r] = chunks of r's sequences with a
  // smaller first chunk index (counting, no sort, no barrier)
  for (int64_t i = tid; i < N; i += blockDim.x) {
    const int r = s_rank[i];
    const int64_t cb = s_cb[i];
    int64_t pos = 0;
    for (int64_t j = s_roff[r]; j < s_roff[r + 1]; ++j)
      if (s_cb[j] < cb) pos += s_G[j];
    for (int kk = 0; kk < s_G[i]; ++kk) a.send_idx[s_sendoff[r] + pos + kk] = (int32_t)(cb + kk);
  }
  __syncthreads();  // send lists complete: reverse-order tie replay reads them
  for (int r = warp; r < W; r += nw)
    if (lane == 0 && s_tie[r]) fix_rev_ties(a, r, s_sendoff[r], s_sendoff[r + 1] - s_sendoff[r]);
  SB_PHASE(12);
  // ---- phase 12: WIR (metrics.cpp:20-31); per_gpu written by the greedy
  __syncthreads();
  for (int r = tid; r < W; r += blockDim.x) a_in.per_gpu[r] = a.per_gpu[r];
  if (warp == 0) {  // min and max are order-independent (no NaN): one warp, loads in parallel
    double lo = a.per_gpu[0], hi = lo;
    for (int r = lane; r < W; r += 32) {
      const double v = a.per_gpu[r];
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0)
      *a.wir = hi == 0.0 ? 1.0 : (lo == 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : __ddiv_rn(hi, lo));
  }
  SB_PHASE(13);
}

}  // namespace sb
