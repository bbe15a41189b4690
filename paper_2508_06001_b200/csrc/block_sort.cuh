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
