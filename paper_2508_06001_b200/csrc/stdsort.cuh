// Exact replica of libstdc++'s std::sort (GCC 13, bits/stl_algo.h /
// stl_heap.h) for int32 chunk-index arrays and a strict-weak comparator.
//
// Why: reverse_plan orders each rank's receive list with
// std::sort(incoming, (segment, start)) (balancer.cpp:278-283).  The key is
// not unique when a sequence is shorter than its bag (its trailing chunks are
// empty and share (segment, start)), and std::sort is unstable, so the
// reference's order of those ties is whatever introsort's partitioning
// produces.  To keep RoutingPlan equality bit-exact even then, ranks whose
// receive list can tie re-run this single-threaded replica (introsort with
// median-of-three pivoting, heapsort fallback at depth 2*floor(log2 n),
// final insertion sort with a 16-element threshold) on the same input order.
// Lists without ties never reach it (their order is unique).
#pragma once

#include <cstdint>

namespace sb {
namespace stdsort {

constexpr int64_t kThreshold = 16;  // _S_threshold

template <typename Less>
__device__ void insertion_sort(int32_t* first, int64_t n, Less less) {
  for (int64_t i = 1; i < n; ++i) {
    const int32_t val = first[i];
    if (less(val, first[0])) {
      for (int64_t k = i; k > 0; --k) first[k] = first[k - 1];  // move_backward
      first[0] = val;
    } else {
      int64_t last = i, next = i - 1;  // __unguarded_linear_insert
      while (less(val, first[next])) {
        first[last] = first[next];
        last = next;
        --next;
      }
      first[last] = val;
    }
  }
}

template <typename Less>
__device__ void unguarded_insertion_sort(int32_t* first, int64_t from, int64_t to, Less less) {
  for (int64_t i = from; i < to; ++i) {
    const int32_t val = first[i];
    int64_t last = i, next = i - 1;
    while (less(val, first[next])) {
      first[last] = first[next];
      last = next;
      --next;
    }
    first[last] = val;
  }
}

template <typename Less>
__device__ void push_heap(int32_t* first, int64_t hole, int64_t top, int32_t value, Less less) {
  int64_t parent = (hole - 1) / 2;
  while (hole > top && less(first[parent], value)) {
    first[hole] = first[parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  first[hole] = value;
}

template <typename Less>
__device__ void adjust_heap(int32_t* first, int64_t hole, int64_t len, int32_t value, Less less) {
  const int64_t top = hole;
  int64_t child = hole;
  while (child < (len - 1) / 2) {
    child = 2 * (child + 1);
    if (less(first[child], first[child - 1])) child--;
    first[hole] = first[child];
    hole = child;
  }
  if ((len & 1) == 0 && child == (len - 2) / 2) {
    child = 2 * (child + 1);
    first[hole] = first[child - 1];
    hole = child - 1;
  }
  push_heap(first, hole, top, value, less);
}

template <typename Less>
__device__ void heap_sort(int32_t* first, int64_t len, Less less) {  // __partial_sort(first, last, last)
  if (len >= 2) {  // make_heap
    int64_t parent = (len - 2) / 2;
    for (;;) {
      adjust_heap(first, parent, len, first[parent], less);
      if (parent == 0) break;
      --parent;
    }
  }
  for (int64_t m = len; m > 1;) {  // __sort_heap
    --m;
    const int32_t value = first[m];
    first[m] = first[0];
    adjust_heap(first, 0, m, value, less);
  }
}

template <typename Less>
__device__ void move_median_to_first(int32_t* result, int32_t* a, int32_t* b, int32_t* c, Less less) {
  auto swp = [](int32_t* x, int32_t* y) {
    const int32_t t = *x;
    *x = *y;
    *y = t;
  };
  if (less(*a, *b)) {
    if (less(*b, *c)) swp(result, b);
    else if (less(*a, *c)) swp(result, c);
    else swp(result, a);
  } else if (less(*a, *c)) {
    swp(result, a);
  } else if (less(*b, *c)) {
    swp(result, c);
  } else {
    swp(result, b);
  }
}

template <typename Less>
__device__ int64_t unguarded_partition(int32_t* base, int64_t first, int64_t last, int64_t pivot, Less less) {
  for (;;) {
    while (less(base[first], base[pivot])) ++first;
    --last;
    while (less(base[pivot], base[last])) --last;
    if (!(first < last)) return first;
    const int32_t t = base[first];
    base[first] = base[last];
    base[last] = t;
    ++first;
  }
}

__device__ __forceinline__ int64_t lg(int64_t n) { return 63 - __clzll((unsigned long long)n); }

// __introsort_loop with an explicit stack in place of the tail recursion on
// the right part (the visiting order, and therefore every swap, is kept).
struct Frame {
  int64_t first, last, depth;
};
constexpr int kStackFrames = 64;  // > 2 log2(n) + 1 for any n < 2^31

// `stack` holds kStackFrames frames (the caller's local array; shared memory
// measured no faster in the fused planner)
template <typename Less>
__device__ void introsort_loop(int32_t* base, int64_t first, int64_t last, int64_t depth, Less less, Frame* stack) {
  int sp = 0;
  stack[sp++] = {first, last, depth};
  while (sp > 0) {
    Frame f = stack[--sp];
    while (f.last - f.first > kThreshold) {
      if (f.depth == 0) {
        heap_sort(base + f.first, f.last - f.first, less);
        break;
      }
      --f.depth;
      const int64_t mid = f.first + (f.last - f.first) / 2;
      move_median_to_first(base + f.first, base + f.first + 1, base + mid, base + f.last - 1, less);
      const int64_t cut = unguarded_partition(base, f.first + 1, f.last, f.first, less);
      // libstdc++ recurses on [cut, last) first, then loops on [first, cut):
      // process the right part completely before the left one.
      stack[sp++] = {f.first, cut, f.depth};  // resumed after the right part
      f.first = cut;
    }
  }
}

// std::sort(v, v + n, less)
template <typename Less>
__device__ void sort(int32_t* v, int64_t n, Less less, Frame* stack) {
  if (n <= 1) return;
  introsort_loop(v, 0, n, 2 * lg(n), less, stack);
  if (n > kThreshold) {
    insertion_sort(v, kThreshold, less);
    unguarded_insertion_sort(v, kThreshold, n, less);
  } else {
    insertion_sort(v, n, less);
  }
}

}  // namespace stdsort
}  // namespace sb
