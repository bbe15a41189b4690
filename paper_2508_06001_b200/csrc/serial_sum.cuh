// Serial FP64 sums computed by a whole CTA, bit-identical to the one-thread
// chain  s_0 = 0, s_{j+1} = RN(s_j + x_j)  over non-negative x_j.
//
// The reference sums workloads serially in several places: the replica and
// report totals (balancer.cpp:24-25, :147) and the occupancy replay of a
// one-bag replica (balancer.cpp:159-166, where every sequence lands in bag 0
// and `capacity - assigned >= w` needs every prefix).  On one thread that is
// a DADD latency chain (~8 cycles per element); at 16K sequences it was the
// planner's critical path.
//
// Exactness argument.  While s stays inside one binade [2^e, 2^(e+1)), it is
// an integer multiple K of q = ulp(s) = 2^(e-52), and
//     RN(K q + x) = (K + m + t) q,   m = floor(x / q),  f = x / q - m,
// with t = 1 if f > 1/2, 0 if f < 1/2 and, on an exact tie, whichever makes
// K + m + t even (round half to even).  x / q is exact (q is a power of two),
// so every increment is an integer known up front except for the tie bit,
// which depends on the parity of the running K.  The parity dependence is a
// two-state automaton, so each element becomes a pair (increment if the
// running sum is even, increment if odd), pairs compose associatively, and a
// block scan gives every element its exact prefix -- as long as the result
// stays in the binade.  The first element whose sum would leave the binade
// (K + inc >= 2^53) is added with one real DADD and the scan restarts in the
// new binade; s only grows, so there are about log2(total / x_first) restarts.
// Zero and tiny (< 2^-960) running sums take scalar steps.  Validated against
// the serial chain on adversarial inputs (integers and halves, i.e. frequent
// ties; zeros; 120-binade ranges; overflow) by sb_selftest_serial_sum.
#pragma once

#include <cstdint>

namespace sb {

constexpr int64_t kSumSat = int64_t(1) << 60;  // saturated increment: the sum leaves the binade
constexpr int64_t kSumLim = int64_t(1) << 53;  // K + increments must stay below this

struct SumPair {
  int64_t a0, a1;  // cumulative increment if the running K starts even / odd
};

__device__ __forceinline__ int64_t sum_sat(int64_t v) { return v > kSumSat ? kSumSat : v; }

__device__ __forceinline__ SumPair sum_combine(SumPair l, SumPair r) {
  return {sum_sat(l.a0 + ((l.a0 & 1) ? r.a1 : r.a0)), sum_sat(l.a1 + (((1 + l.a1) & 1) ? r.a1 : r.a0))};
}

struct SumElem {
  int64_t m;  // floor(x / q), saturated
  int rb;     // 1: round up (f > 1/2)
  int tie;    // f == 1/2 exactly
};

__device__ __forceinline__ SumElem sum_elem(double x, double rq) {
  const double y = __dmul_rn(x, rq);  // exact: rq is a power of two
  SumElem e{0, 0, 0};
  if (!(y < 9007199254740992.0)) {  // >= 2^53 q: leaves the binade on its own
    e.m = kSumSat;
    return e;
  }
  const double fm = floor(y), f = __dsub_rn(y, fm);
  e.m = (int64_t)fm;
  e.rb = f > 0.5;
  e.tie = f == 0.5;
  return e;
}

// increment of one element when the running K before it has parity `par`
__device__ __forceinline__ int64_t sum_inc(const SumElem& e, int64_t par) {
  if (e.m >= kSumSat) return kSumSat;
  return e.m + (e.tie ? ((par + e.m) & 1) : e.rb);
}

// Named barrier 1 over threads [0, NT): the sum can run on the first warps of a
// larger CTA (the fused planner) while the others wait at their next barrier.
template <int NT>
__device__ __forceinline__ void sum_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

// Serial sum of x_j = load(j), j in [0, n), by threads [0, NT) of the CTA
// (whole warps; all of them call with the same n and get the same result).
// emit(j, s_j, x_j) runs exactly once for every j (on some thread) with the
// serially-rounded sum of x_0..x_{j-1}.  Every restart (one per binade
// crossing and per NT*E-element window) costs several thousand cycles, so a
// one-thread chain (~10 cycles per element) stays cheaper below a few thousand
// elements: the planner uses this on its large path only.
template <int NT, int E, class Load, class Emit>
__device__ double block_serial_sum(int64_t n, Load load, Emit emit) {
  static_assert(NT % 32 == 0 && NT <= 1024, "whole warps");
  constexpr int NW = NT / 32;
  constexpr int64_t WIN = (int64_t)NT * E;
  __shared__ SumPair s_wp[NW + 1];
  __shared__ unsigned long long s_jstar;
  __shared__ double s_next;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double s = 0.0;
  int64_t i = 0;
  // serial head: the running sum crosses a binade roughly every doubling of
  // the element count, so the first ~log2(kHead) restarts cost more than
  // kHead dependent adds on one thread
  constexpr int64_t kHead = 128;
  if (n > 0) {
    const int64_t h = n < kHead ? n : kHead;
    if (tid == 0) {
      double t = 0.0;
      for (int64_t j = 0; j < h; ++j) {
        const double x = load(j);
        emit(j, t, x);
        t = __dadd_rn(t, x);
      }
      s_next = t;
    }
    sum_bar<NT>();
    s = s_next;
    i = h;
    sum_bar<NT>();
  }
  while (i < n) {
    if (!(s < __longlong_as_double(0x7ff0000000000000ll))) {  // +inf absorbs everything that follows
      for (int64_t j = i + tid; j < n; j += NT) emit(j, s, load(j));
      break;
    }
    if (s == 0.0) {  // RN(0 + x) = x: skip the leading zeros of the window, take the first non-zero
      const int64_t w1 = i + WIN < n ? i + WIN : n;
      if (tid == 0) s_jstar = ~0ull;
      sum_bar<NT>();
      for (int64_t j = i + tid; j < w1; j += NT)
        if (load(j) != 0.0) atomicMin(&s_jstar, (unsigned long long)j);
      sum_bar<NT>();
      const unsigned long long js = s_jstar;
      const int64_t last = js == ~0ull ? w1 : (int64_t)js + 1;
      for (int64_t j = i + tid; j < last; j += NT) emit(j, 0.0, load(j));
      if (js != ~0ull) s = load((int64_t)js);
      i = last;
      sum_bar<NT>();  // s_jstar reuse
      continue;
    }
    if (s < 0x1p-960) {  // tiny running sum (its ulp would be subnormal): one scalar step
      const double x = load(i);
      if (tid == 0) emit(i, s, x);
      s = __dadd_rn(s, x);
      ++i;
      continue;
    }
    const uint64_t sbits = (uint64_t)__double_as_longlong(s);
    const int eb = (int)(sbits >> 52);                                          // biased exponent, 63..2046
    const double q = __longlong_as_double((long long)((uint64_t)(eb - 52) << 52));   // 2^(eb-1075)
    const double rq = __longlong_as_double((long long)((uint64_t)(2098 - eb) << 52));  // 1 / q
    const int64_t K = (int64_t)((sbits & ((uint64_t(1) << 52) - 1)) | (uint64_t(1) << 52));
    const int64_t p0 = K & 1;
    // this thread's E consecutive elements of the window
    const int64_t j0 = i + (int64_t)tid * E;
    double xv[E];
    SumElem ev[E];
    SumPair loc{0, 0};
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int64_t j = j0 + k;
      xv[k] = j < n ? load(j) : 0.0;
      ev[k] = sum_elem(xv[k], rq);
      loc.a0 = sum_sat(loc.a0 + sum_inc(ev[k], loc.a0 & 1));
      loc.a1 = sum_sat(loc.a1 + sum_inc(ev[k], (1 + loc.a1) & 1));
    }
    // block exclusive scan of the pairs (composition, in element order)
    SumPair inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      SumPair u;
      u.a0 = __shfl_up_sync(0xffffffffu, inc.a0, o);
      u.a1 = __shfl_up_sync(0xffffffffu, inc.a1, o);
      if (lane >= o) inc = sum_combine(u, inc);
    }
    if (lane == 31) s_wp[warp] = inc;
    if (tid == 0) s_jstar = ~0ull;
    sum_bar<NT>();
    if (warp == 0) {
      SumPair x = lane < NW ? s_wp[lane] : SumPair{0, 0};
      SumPair xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        SumPair u;
        u.a0 = __shfl_up_sync(0xffffffffu, xi.a0, o);
        u.a1 = __shfl_up_sync(0xffffffffu, xi.a1, o);
        if (lane >= o) xi = sum_combine(u, xi);
      }
      SumPair ex;  // exclusive = inclusive of the previous lane
      ex.a0 = __shfl_up_sync(0xffffffffu, xi.a0, 1);
      ex.a1 = __shfl_up_sync(0xffffffffu, xi.a1, 1);
      if (lane == 0) ex = SumPair{0, 0};
      if (lane < NW) s_wp[lane] = ex;
      if (lane == NW - 1) s_wp[NW] = xi;
    }
    sum_bar<NT>();
    // exclusive prefix of this thread = (warp prefix) o (lanes before it in the warp)
    SumPair lex;
    lex.a0 = __shfl_up_sync(0xffffffffu, inc.a0, 1);
    lex.a1 = __shfl_up_sync(0xffffffffu, inc.a1, 1);
    SumPair ex = s_wp[warp];
    if (lane > 0) ex = sum_combine(ex, lex);
    const SumPair tot = s_wp[NW];
    // walk: exact prefixes until the first element that leaves the binade
    int64_t P = p0 ? ex.a1 : ex.a0;
    int64_t before[E];
    int cross = E;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      before[k] = K + P;
      if (cross == E && j0 + k < n) {
        const int64_t d = sum_inc(ev[k], (p0 + P) & 1);
        if (K + P + d >= kSumLim) cross = k;
        else P += d;
      }
    }
    if (cross < E) atomicMin(&s_jstar, (unsigned long long)(j0 + cross));
    sum_bar<NT>();
    const unsigned long long js = s_jstar;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int64_t j = j0 + k;
      if (j < n && (unsigned long long)j <= js) {
        const double sb4 = __dmul_rn((double)before[k], q);  // exact: K + P < 2^53, q a power of two
        emit(j, sb4, xv[k]);
        if ((unsigned long long)j == js) s_next = __dadd_rn(sb4, xv[k]);
      }
    }
    sum_bar<NT>();
    if (js != ~0ull) {
      s = s_next;
      i = (int64_t)js + 1;
    } else {
      s = __dmul_rn((double)(K + (p0 ? tot.a1 : tot.a0)), q);
      i = i + WIN < n ? i + WIN : n;
    }
    sum_bar<NT>();  // s_next / s_wp / s_jstar reuse
  }
  return s;
}

}  // namespace sb
