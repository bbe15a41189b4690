// Block-cooperative sort of (hi:u64, lo:u64, val:u32) records, ascending
// lexicographically.  `val` is unique per record, so the order is total and
// the result deterministic (no reliance on sort stability).
//
// Phase 1 sorts tiles of up to 2048 records in shared memory with a bitonic
// network; phase 2 merges runs pairwise in global memory (L2-resident at the
// sizes the planner sees) using merge-path partitioning so every thread
// produces an equal share of each merged output.
#pragma once

#include <cstdint>

namespace sb {

constexpr int kSortTile = 2048;
constexpr size_t kSortSmemBytes = kSortTile * (8 + 8 + 4);

struct SortRec {
  uint64_t hi, lo;
  uint32_t v;
};

__device__ __forceinline__ bool rec_less(uint64_t ahi, uint64_t alo, uint32_t av, uint64_t bhi,
                                         uint64_t blo, uint32_t bv) {
  if (ahi != bhi) return ahi < bhi;
  if (alo != blo) return alo < blo;
  return av < bv;
}

// Branch-free (key, id, index) order for the register sort.
__device__ __forceinline__ bool rec_less_bf(uint64_t ahi, uint64_t alo, uint32_t av, uint64_t bhi, uint64_t blo,
                                            uint32_t bv) {
  return (ahi < bhi) | ((ahi == bhi) & ((alo < blo) | ((alo == blo) & (av < bv))));
}

// Bitonic sort with the records in registers: thread x holds records
// x + r * B (r < RPT, B = the block size) of T = pow2 >= n (slots >= n are
// +inf padding).  T is a template parameter, so all (log2 T)(log2 T + 1)/2
// stages unroll: partners at distance j < 32 are exchanged by shuffles,
// 32 <= j < B through shared memory (the only barriers: n = 256 has 6 of
// 36 stages), j >= B inside the thread.  Leaves the record of rank
// x + r * B in (h, l, v)[r].
template <int T, int RPT, int B>
__device__ void reg_bitonic(uint64_t* s_hi, uint64_t* s_lo, uint32_t* s_v, int n, uint64_t (&h)[RPT],
                            uint64_t (&l)[RPT], uint32_t (&v)[RPT]) {
  static_assert(T <= RPT * B && (RPT == 1 || T == RPT * B), "register bitonic shape");
  const int tid = threadIdx.x;
  const bool live = RPT > 1 || (tid & ~31) < T;  // warp-uniform
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int x = tid + r * B;
    h[r] = x < n ? s_hi[x] : ~0ull;
    l[r] = x < n ? s_lo[x] : ~0ull;
    v[r] = x < n ? s_v[x] : 0xffffffffu;
  }
#pragma unroll
  for (int k = 2; k <= T; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= B) {  // the partner of record r is this thread's record r ^ (j / B)
        const int d = j / B;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          if ((r & d) != 0) continue;
          const int r2 = r | d;
          const int x = tid + r * B;
          const bool up = (x & k) == 0;  // ascending half of the current bitonic merge
          const bool lt = rec_less_bf(h[r2], l[r2], v[r2], h[r], l[r], v[r]);
          if (lt == up) {  // ascending: smaller to r; descending: larger to r
            const uint64_t a = h[r], b = l[r];
            const uint32_t c = v[r];
            h[r] = h[r2]; l[r] = l[r2]; v[r] = v[r2];
            h[r2] = a; l[r2] = b; v[r2] = c;
          }
        }
        continue;
      }
      uint64_t ph[RPT], pl[RPT];
      uint32_t pv[RPT];
      if (j >= 32) {
        __syncthreads();  // the previous exchange's reads are done
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int x = tid + r * B;
          if (x < T) {
            s_hi[x] = h[r];
            s_lo[x] = l[r];
            s_v[x] = v[r];
          }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int x = tid + r * B;
          const int p = x < T ? (x ^ j) : x;  // x >= T: padding stays (never read back)
          ph[r] = x < T ? s_hi[p] : h[r];
          pl[r] = x < T ? s_lo[p] : l[r];
          pv[r] = x < T ? s_v[p] : v[r];
        }
      } else {
        if (!live) continue;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          ph[r] = __shfl_xor_sync(0xffffffffu, h[r], j);
          pl[r] = __shfl_xor_sync(0xffffffffu, l[r], j);
          pv[r] = __shfl_xor_sync(0xffffffffu, v[r], j);
        }
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int x = tid + r * B;
        const bool up = (x & k) == 0, lower = (x & j) == 0;
        const bool pless = rec_less_bf(ph[r], pl[r], pv[r], h[r], l[r], v[r]);
        const bool take = (lower == up) ? pless : !pless;  // records are unique; equal padding swaps to itself
        h[r] = take ? ph[r] : h[r];
        l[r] = take ? pl[r] : l[r];
        v[r] = take ? pv[r] : v[r];
      }
    }
  }
}

// Sorts a[0..n) in place (b is scratch of the same size).  All threads of the
// block must call it.  `smem` must hold kSortSmemBytes.
__device__ void block_sort(int64_t n, uint64_t* ahi, uint64_t* alo, uint32_t* av, uint64_t* bhi,
                           uint64_t* blo, uint32_t* bv, unsigned char* smem) {
  uint64_t* s_hi = reinterpret_cast<uint64_t*>(smem);
  uint64_t* s_lo = s_hi + kSortTile;
  uint32_t* s_v = reinterpret_cast<uint32_t*>(s_lo + kSortTile);
  const int tid = threadIdx.x, nt = blockDim.x;
  if (n <= 1) return;

  int tile = 64;
  while (tile < n && tile < kSortTile) tile <<= 1;

  // ---- phase 1: bitonic sort of each tile in shared memory
  for (int64_t t0 = 0; t0 < n; t0 += tile) {
    for (int i = tid; i < tile; i += nt) {
      const int64_t g = t0 + i;
      if (g < n) {
        s_hi[i] = ahi[g];
        s_lo[i] = alo[g];
        s_v[i] = av[g];
      } else {
        s_hi[i] = ~0ull;
        s_lo[i] = ~0ull;
        s_v[i] = 0xffffffffu;
      }
    }
    __syncthreads();
    for (int k = 2; k <= tile; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < tile / 2; i += nt) {
          const int lo = 2 * j * (i / j) + (i % j);
          const int hi = lo + j;
          const bool up = (lo & k) == 0;
          const bool sw = rec_less(s_hi[hi], s_lo[hi], s_v[hi], s_hi[lo], s_lo[lo], s_v[lo]);
          if (sw == up) {
            uint64_t x = s_hi[lo]; s_hi[lo] = s_hi[hi]; s_hi[hi] = x;
            uint64_t y = s_lo[lo]; s_lo[lo] = s_lo[hi]; s_lo[hi] = y;
            uint32_t z = s_v[lo]; s_v[lo] = s_v[hi]; s_v[hi] = z;
          }
        }
        __syncthreads();
      }
    }
    for (int i = tid; i < tile; i += nt) {
      const int64_t g = t0 + i;
      if (g < n) {
        ahi[g] = s_hi[i];
        alo[g] = s_lo[i];
        av[g] = s_v[i];
      }
    }
    __syncthreads();
  }
  if (n <= tile) return;

  // ---- phase 2: pairwise merges of sorted runs (global memory ping-pong)
  uint64_t *shi = ahi, *slo = alo, *dhi = bhi, *dlo = blo;
  uint32_t *sv = av, *dv = bv;
  const int64_t per = (n + nt - 1) / nt;
  for (int64_t width = tile; width < n; width <<= 1) {
    int64_t o = (int64_t)tid * per;
    const int64_t o_end = o + per < n ? o + per : n;
    while (o < o_end) {
      const int64_t pair = (o / (2 * width)) * (2 * width);
      const int64_t a0 = pair;
      const int64_t la = width < n - a0 ? width : n - a0;
      const int64_t b0 = a0 + la;
      const int64_t lb = (b0 < n) ? (width < n - b0 ? width : n - b0) : 0;
      const int64_t seg_end = (pair + la + lb) < o_end ? (pair + la + lb) : o_end;
      const int64_t d = o - pair;
      // merge path: i = number of A records among the first d outputs
      int64_t lo = d - lb > 0 ? d - lb : 0;
      int64_t hi = d < la ? d : la;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const int64_t bj = b0 + (d - 1 - mid);
        if (rec_less(shi[a0 + mid], slo[a0 + mid], sv[a0 + mid], shi[bj], slo[bj], sv[bj]))
          lo = mid + 1;
        else
          hi = mid;
      }
      int64_t i = lo, j = d - lo;
      for (; o < seg_end; ++o) {
        bool takeA;
        if (i >= la) takeA = false;
        else if (j >= lb) takeA = true;
        else takeA = rec_less(shi[a0 + i], slo[a0 + i], sv[a0 + i], shi[b0 + j], slo[b0 + j], sv[b0 + j]);
        if (takeA) {
          dhi[o] = shi[a0 + i]; dlo[o] = slo[a0 + i]; dv[o] = sv[a0 + i]; ++i;
        } else {
          dhi[o] = shi[b0 + j]; dlo[o] = slo[b0 + j]; dv[o] = sv[b0 + j]; ++j;
        }
      }
    }
    __syncthreads();
    uint64_t* t1 = shi; shi = dhi; dhi = t1;
    uint64_t* t2 = slo; slo = dlo; dlo = t2;
    uint32_t* t3 = sv; sv = dv; dv = t3;
  }
  if (shi != ahi) {
    for (int64_t i = tid; i < n; i += nt) {
      ahi[i] = shi[i];
      alo[i] = slo[i];
      av[i] = sv[i];
    }
    __syncthreads();
  }
}

}  // namespace sb
