// TEST INFRASTRUCTURE ONLY (part of liboracle.so).
//
// reverse_plan orders each rank's receive list with std::sort on
// (segment index, start) (balancer.cpp:278-283).  That key ties for the
// zero-length chunks of a sequence shorter than its bag, and std::sort is
// unstable, so the reference's tie order is libstdc++'s.  The oracle calls
// the very same std::sort (same compiler/runtime as oracle/_ref) so it
// reproduces the reference exactly; the device replica lives in
// paper_2508_06001_b200/csrc/stdsort.cuh and is checked against this.
#include <algorithm>
#include <cstdint>

extern "C" void or_std_sort_chunks(int32_t* v, int64_t n, const int64_t* seg, const int64_t* start) {
  std::sort(v, v + n, [&](int32_t a, int32_t b) {
    if (seg[a] != seg[b]) return seg[a] < seg[b];
    return start[a] < start[b];
  });
}
