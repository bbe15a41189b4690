// Microbenchmarks for the greedy's critical path on sm_100a (diagnostics).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o greedy_micro greedy_micro.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <type_traits>
#include <cuda_runtime.h>

__global__ void lat_redux(int iters, unsigned* out, long long* cyc) {
  unsigned x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __reduce_min_sync(0xffffffffu, x + threadIdx.x) ;
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_shfl(int iters, unsigned* out, long long* cyc) {
  unsigned x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (x + 1) & 31);
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_ballot(int iters, unsigned* out, long long* cyc) {
  unsigned x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __ffs(__ballot_sync(0xffffffffu, (x & 31) == threadIdx.x)) ;
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_dfma(int iters, double a, double* out, long long* cyc) {
  double y = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) y = __fma_rn(y, a, 0.5);
  long long t1 = clock64();
  out[threadIdx.x] = y; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_dadd(int iters, double a, double* out, long long* cyc) {
  double y = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) y = __dadd_rn(y, a);
  long long t1 = clock64();
  out[threadIdx.x] = y; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_dsetp(int iters, double a, double* out, long long* cyc) {
  double y = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) y = (y >= a) ? y - 1.0 : y + 2.0;
  long long t1 = clock64();
  out[threadIdx.x] = y; if (threadIdx.x == 0) *cyc = t1 - t0;
}

__device__ __forceinline__ double div_m(double a, double b, double r) {
  double y = __dmul_rn(a, r);
  double e = __fma_rn(-b, y, a);
  y = __fma_rn(r, e, y);
  e = __fma_rn(-b, y, a);
  return __fma_rn(r, e, y);
}
__device__ __forceinline__ double occf(double asg, double cap, double rcap) {
  if (cap > 0.0) return div_m(asg, cap, rcap);
  return asg > 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0;
}
__device__ __forceinline__ uint32_t argmin_lane(uint64_t key) {
  const uint32_t khi = (uint32_t)(key >> 32), klo = (uint32_t)key;
  const uint32_t m1 = __reduce_min_sync(0xffffffffu, khi);
  const unsigned eq = __ballot_sync(0xffffffffu, khi == m1);
  if (__popc(eq) == 1) return (uint32_t)(__ffs(eq) - 1);
  const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
  return (uint32_t)(__ffs(__ballot_sync(0xffffffffu, khi == m1 && klo == m2)) - 1);
}

// V0: the production greedy (k_greedy<1>) inner loop.
__global__ void g_v0(const double* w_sorted, int n, int M, const double* caps, int* pick, long long* cyc) {
  const int lane = threadIdx.x;
  const double cap = lane < M ? caps[lane] : 0.0;
  const double rcap = cap > 0.0 ? __drcp_rn(cap) : 0.0;
  double asg = 0.0, occ = occf(0.0, cap, rcap), rem = __dsub_rn(cap, 0.0);
  long long t0 = clock64();
  for (int p0 = 0; p0 < n; p0 += 32) {
    const double w_lane = (p0 + lane < n) ? w_sorted[p0 + lane] : 0.0;
    const int steps = (n - p0) < 32 ? (n - p0) : 32;
    int my = 0;
    for (int t = 0; t < steps; ++t) {
      const double w = __shfl_sync(0xffffffffu, w_lane, t);
      const double nasg = __dadd_rn(asg, w);
      const double nocc = occf(nasg, cap, rcap);
      const double nrem = __dsub_rn(cap, nasg);
      uint64_t key = ~0ull;
      if (lane < M) key = ((rem >= w) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ);
      const uint32_t pk = argmin_lane(key);
      if ((uint32_t)lane == pk) { asg = nasg; occ = nocc; rem = nrem; }
      if (lane == t) my = (int)pk;
    }
    if (p0 + lane < n) pick[p0 + lane] = my;
  }
  long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// V1: keys for step t+1 speculated during step t for both outcomes of
// step t (this lane wins / does not win); the state after a win is computed
// one step ahead, so the loop-carried chain is select -> REDUX -> pick.
__global__ void g_v1(const double* w_sorted, int n, int M, const double* caps, int* pick, long long* cyc) {
  const int lane = threadIdx.x;
  const bool act = lane < M;
  const double cap = act ? caps[lane] : 0.0;
  const double rcap = cap > 0.0 ? __drcp_rn(cap) : 0.0;
  // state at the start of step t
  double asg = 0.0, occ = occf(0.0, cap, rcap), rem = __dsub_rn(cap, 0.0);
  long long t0 = clock64();
  // w for step 0 and lookahead
  __shared__ double ws[32 + 1];
  int my = 0;
  // key for step 0 (no previous pick)
  double w0 = n > 0 ? w_sorted[0] : 0.0;
  uint64_t key = act ? (((rem >= w0) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) : ~0ull;
  double w_lane = (lane < n) ? w_sorted[lane] : 0.0;
  for (int p0 = 0; p0 < n; p0 += 32) {
    const int steps = (n - p0) < 32 ? (n - p0) : 32;
    const double w_next_blk = (p0 + 32 + lane < n) ? w_sorted[p0 + 32 + lane] : 0.0;
    for (int t = 0; t < steps; ++t) {
      const double w = __shfl_sync(0xffffffffu, w_lane, t);
      double wn = __shfl_sync(0xffffffffu, w_lane, (t + 1) & 31);
      const double wn2 = __shfl_sync(0xffffffffu, w_next_blk, 0);
      if (t == 31) wn = wn2;
      // if this lane wins step t:
      const double nasg = __dadd_rn(asg, w);
      const double nocc = occf(nasg, cap, rcap);
      const double nrem = __dsub_rn(cap, nasg);
      // speculative keys for step t+1
      const uint64_t kWin = act ? (((nrem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(nocc)) : ~0ull;
      const uint64_t kNot = act ? (((rem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) : ~0ull;
      const uint32_t pk = argmin_lane(key);
      const bool won = (uint32_t)lane == pk;
      key = won ? kWin : kNot;
      if (won) { asg = nasg; occ = nocc; rem = nrem; }
      if (lane == t) my = (int)pk;
    }
    if (p0 + lane < n) pick[p0 + lane] = my;
    w_lane = w_next_blk;
  }
  long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// REDUX-only lexicographic argmin of (key, lane): three dependent REDUX, no
// vote / branch.
__device__ __forceinline__ uint32_t argmin_redux(uint64_t key) {
  const uint32_t khi = (uint32_t)(key >> 32), klo = (uint32_t)key;
  const uint32_t m1 = __reduce_min_sync(0xffffffffu, khi);
  const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
  return __reduce_min_sync(0xffffffffu, (khi == m1 && klo == m2) ? (uint32_t)threadIdx.x : 31u);
}

// V2: V1's speculation + REDUX-only argmin; w for the block staged in smem.
__global__ void g_v2(const double* w_sorted, int n, int M, const double* caps, int* pick, long long* cyc) {
  const int lane = threadIdx.x;
  const bool act = lane < M;
  const double cap = act ? caps[lane] : 0.0;
  const double rcap = cap > 0.0 ? __drcp_rn(cap) : 0.0;
  double asg = 0.0, occ = occf(0.0, cap, rcap), rem = __dsub_rn(cap, 0.0);
  __shared__ double ws[2][33];
  long long t0 = clock64();
  ws[0][lane] = (lane < n) ? w_sorted[lane] : 0.0;
  ws[0][32] = (32 < n) ? w_sorted[32] : 0.0;
  __syncwarp();
  const double w0 = ws[0][0];
  uint64_t key = act ? (((rem >= w0) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) : ~0ull;
  int buf = 0;
  for (int p0 = 0; p0 < n; p0 += 32) {
    const int steps = (n - p0) < 32 ? (n - p0) : 32;
    // prefetch the next block (+1 lookahead element)
    ws[buf ^ 1][lane] = (p0 + 32 + lane < n) ? w_sorted[p0 + 32 + lane] : 0.0;
    if (lane == 0) ws[buf ^ 1][32] = (p0 + 64 < n) ? w_sorted[p0 + 64] : 0.0;
    int my = 0;
    const double* wb = ws[buf];
    for (int t = 0; t < steps; ++t) {
      const double w = wb[t];
      const double wn = wb[t + 1];
      const double nasg = __dadd_rn(asg, w);
      const double nocc = occf(nasg, cap, rcap);
      const double nrem = __dsub_rn(cap, nasg);
      const uint64_t kWin = act ? (((nrem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(nocc)) : ~0ull;
      const uint64_t kNot = act ? (((rem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) : ~0ull;
      const uint32_t pk = argmin_redux(key);
      const bool won = (uint32_t)lane == pk;
      key = won ? kWin : kNot;
      if (won) { asg = nasg; occ = nocc; rem = nrem; }
      if (lane == t) my = (int)pk;
    }
    if (p0 + lane < n) pick[p0 + lane] = my;
    __syncwarp();
    buf ^= 1;
  }
  long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// V3: V0 with the REDUX-only argmin (no speculation).
__global__ void g_v3(const double* w_sorted, int n, int M, const double* caps, int* pick, long long* cyc) {
  const int lane = threadIdx.x;
  const double cap = lane < M ? caps[lane] : 0.0;
  const double rcap = cap > 0.0 ? __drcp_rn(cap) : 0.0;
  double asg = 0.0, occ = occf(0.0, cap, rcap), rem = __dsub_rn(cap, 0.0);
  long long t0 = clock64();
  for (int p0 = 0; p0 < n; p0 += 32) {
    const double w_lane = (p0 + lane < n) ? w_sorted[p0 + lane] : 0.0;
    const int steps = (n - p0) < 32 ? (n - p0) : 32;
    int my = 0;
    for (int t = 0; t < steps; ++t) {
      const double w = __shfl_sync(0xffffffffu, w_lane, t);
      const double nasg = __dadd_rn(asg, w);
      const double nocc = occf(nasg, cap, rcap);
      const double nrem = __dsub_rn(cap, nasg);
      uint64_t key = ~0ull;
      if (lane < M) key = ((rem >= w) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ);
      const uint32_t pk = argmin_redux(key);
      if ((uint32_t)lane == pk) { asg = nasg; occ = nocc; rem = nrem; }
      if (lane == t) my = (int)pk;
    }
    if (p0 + lane < n) pick[p0 + lane] = my;
  }
  long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// Branch-free occupancy: both arms computed, selected (no BSSY/BSYNC).
__device__ __forceinline__ double occ_sel(double asg, double cap, double rcap) {
  const double q = div_m(asg, cap, rcap);
  const double z = asg > 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0;
  return cap > 0.0 ? q : z;
}

// V5: V2 with branch-free occupancy.
__global__ void g_v5(const double* w_sorted, int n, int M, const double* caps, int* pick, long long* cyc) {
  const int lane = threadIdx.x;
  const bool act = lane < M;
  const double cap = act ? caps[lane] : 0.0;
  const double rcap = cap > 0.0 ? __drcp_rn(cap) : 0.0;
  double asg = 0.0, occ = occ_sel(0.0, cap, rcap), rem = __dsub_rn(cap, 0.0);
  __shared__ double ws[2][33];
  long long t0 = clock64();
  ws[0][lane] = (lane < n) ? w_sorted[lane] : 0.0;
  ws[0][32] = (32 < n) ? w_sorted[32] : 0.0;
  __syncwarp();
  const double w0 = ws[0][0];
  const uint64_t inact = act ? 0ull : ~0ull;
  uint64_t key = (((rem >= w0) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) | inact;
  int buf = 0;
  for (int p0 = 0; p0 < n; p0 += 32) {
    const int steps = (n - p0) < 32 ? (n - p0) : 32;
    ws[buf ^ 1][lane] = (p0 + 32 + lane < n) ? w_sorted[p0 + 32 + lane] : 0.0;
    if (lane == 0) ws[buf ^ 1][32] = (p0 + 64 < n) ? w_sorted[p0 + 64] : 0.0;
    int my = 0;
    const double* wb = ws[buf];
#pragma unroll 4
    for (int t = 0; t < steps; ++t) {
      const double w = wb[t];
      const double wn = wb[t + 1];
      const double nasg = __dadd_rn(asg, w);
      const double nocc = occ_sel(nasg, cap, rcap);
      const double nrem = __dsub_rn(cap, nasg);
      const uint64_t kWin = (((nrem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(nocc)) | inact;
      const uint64_t kNot = (((rem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) | inact;
      const uint32_t pk = argmin_redux(key);
      const bool won = (uint32_t)lane == pk;
      key = won ? kWin : kNot;
      asg = won ? nasg : asg;
      occ = won ? nocc : occ;
      rem = won ? nrem : rem;
      my = (lane == t) ? (int)pk : my;
    }
    if (p0 + lane < n) pick[p0 + lane] = my;
    __syncwarp();
    buf ^= 1;
  }
  long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// 27-bit monotone image of the exact key (infeasible, occ): occupancy in
// fixed point with 25 fractional bits, saturated at 2.  f(a) < f(b) implies
// key(a) < key(b); equal images are the only ambiguity (detected).
__device__ __forceinline__ uint32_t key27(bool infeasible, double occ) {
  const double q = occ < 1.999999 ? occ : 1.999999;
  const uint32_t fx = (uint32_t)__double2uint_rz(__dmul_rn(q, 33554432.0));  // 2^25
  return (infeasible ? (1u << 26) : 0u) | fx;
}

// V6: one REDUX per step on (key27 << 5 | lane); a lane whose key27 equals
// the winner's flags a conflict; a block with a conflict is replayed from
// its checkpoint with the exact three-REDUX loop.
__global__ void g_v6(const double* w_sorted, int n, int M, const double* caps, int* pick, long long* cyc,
                     int* replays) {
  const int lane = threadIdx.x;
  const bool act = lane < M;
  const double cap = act ? caps[lane] : 0.0;
  const double rcap = cap > 0.0 ? __drcp_rn(cap) : 0.0;
  double asg = 0.0, occ = occ_sel(0.0, cap, rcap), rem = __dsub_rn(cap, 0.0);
  __shared__ double ws[2][33];
  long long t0 = clock64();
  ws[0][lane] = (lane < n) ? w_sorted[lane] : 0.0;
  ws[0][32] = (32 < n) ? w_sorted[32] : 0.0;
  __syncwarp();
  const uint64_t inact = act ? 0ull : ~0ull;
  const uint32_t inact32 = act ? 0u : ~0u;
  int buf = 0, nrep = 0;
  for (int p0 = 0; p0 < n; p0 += 32) {
    const int steps = (n - p0) < 32 ? (n - p0) : 32;
    ws[buf ^ 1][lane] = (p0 + 32 + lane < n) ? w_sorted[p0 + 32 + lane] : 0.0;
    if (lane == 0) ws[buf ^ 1][32] = (p0 + 64 < n) ? w_sorted[p0 + 64] : 0.0;
    const double* wb = ws[buf];
    const double c_asg = asg, c_occ = occ, c_rem = rem;  // checkpoint
    int my = 0;
    bool conflict = false;
    uint32_t key = (key27(!(rem >= wb[0]), occ) << 5 | (uint32_t)lane) | inact32;
#pragma unroll 4
    for (int t = 0; t < steps; ++t) {
      const double w = wb[t];
      const double wn = wb[t + 1];
      const double nasg = __dadd_rn(asg, w);
      const double nocc = occ_sel(nasg, cap, rcap);
      const double nrem = __dsub_rn(cap, nasg);
      const uint32_t kWin = (key27(!(nrem >= wn), nocc) << 5 | (uint32_t)lane) | inact32;
      const uint32_t kNot = (key27(!(rem >= wn), occ) << 5 | (uint32_t)lane) | inact32;
      const uint32_t m = __reduce_min_sync(0xffffffffu, key);
      const bool won = key == m;
      // exact 64-bit keys of this lane and of the winner: an equal image
      // with a different exact key is a near tie the image cannot order.
      const uint64_t k64 = (((rem >= w) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) | inact;
      const uint32_t whi = __shfl_sync(0xffffffffu, (uint32_t)(k64 >> 32), (int)(m & 31u));
      const uint32_t wlo = __shfl_sync(0xffffffffu, (uint32_t)k64, (int)(m & 31u));
      conflict |= ((key ^ m) >> 5) == 0 && k64 != (((uint64_t)whi << 32) | wlo);
      key = won ? kWin : kNot;
      asg = won ? nasg : asg;
      occ = won ? nocc : occ;
      rem = won ? nrem : rem;
      my = (lane == t) ? (int)(m & 31u) : my;
    }
    if (__any_sync(0xffffffffu, conflict)) {
      ++nrep;
      asg = c_asg; occ = c_occ; rem = c_rem;
      uint64_t k64 = (((rem >= wb[0]) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) | inact;
      for (int t = 0; t < steps; ++t) {
        const double w = wb[t];
        const double wn = wb[t + 1];
        const double nasg = __dadd_rn(asg, w);
        const double nocc = occ_sel(nasg, cap, rcap);
        const double nrem = __dsub_rn(cap, nasg);
        const uint64_t kWin = (((nrem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(nocc)) | inact;
        const uint64_t kNot = (((rem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) | inact;
        const uint32_t pk = argmin_redux(k64);
        const bool won = (uint32_t)lane == pk;
        k64 = won ? kWin : kNot;
        asg = won ? nasg : asg;
        occ = won ? nocc : occ;
        rem = won ? nrem : rem;
        my = (lane == t) ? (int)pk : my;
      }
    }
    if (p0 + lane < n) pick[p0 + lane] = my;
    __syncwarp();
    buf ^= 1;
  }
  long long t1 = clock64();
  if (lane == 0) { *cyc = t1 - t0; *replays = nrep; }
}

// Exact 64-bit key with the lane folded in: [infeasible:1][exp-992:6]
// [mantissa:52][lane:5].  Exact for occupancies 0, +inf and normal values
// with biased exponent in [993, 1054]; `oor` flags anything else.
__device__ __forceinline__ uint64_t key_lane(bool infeasible, double occ, uint32_t lane, bool& oor) {
  const uint64_t b = (uint64_t)__double_as_longlong(occ);
  const uint32_t e = (uint32_t)(b >> 52);  // sign is 0
  const uint64_t mant = b & ((1ull << 52) - 1);
  // e == 0 (zero / subnormal) keeps ep 0 and its mantissa order; occ is
  // never NaN, so e == 2047 is +inf.
  uint32_t ep = e - 992u;
  ep = (e == 2047u) ? 63u : ep;
  ep = (e == 0u) ? 0u : ep;
  const uint32_t bad = (uint32_t)(e != 0u) & (uint32_t)(e != 2047u) & (uint32_t)((e - 993u) > 61u);
  oor = (bool)((uint32_t)oor | bad);
  return ((uint64_t)infeasible << 63) | ((uint64_t)(ep & 63u) << 57) | (mant << 5) | lane;
}

// V7: exact two-REDUX greedy on lane-folded keys; blocks with an
// out-of-range occupancy are replayed with the three-REDUX loop.
__global__ void g_v7(const double* w_sorted, int n, int M, const double* caps, int* pick, long long* cyc,
                     int* replays) {
  const int lane = threadIdx.x;
  const bool act = lane < M;
  const double cap = act ? caps[lane] : 0.0;
  const double rcap = cap > 0.0 ? __drcp_rn(cap) : 0.0;
  double asg = 0.0, occ = occ_sel(0.0, cap, rcap), rem = __dsub_rn(cap, 0.0);
  __shared__ double ws[2][33];
  long long t0 = clock64();
  ws[0][lane] = (lane < n) ? w_sorted[lane] : 0.0;
  ws[0][32] = (32 < n) ? w_sorted[32] : 0.0;
  __syncwarp();
  const uint64_t inact = act ? 0ull : ~0ull;
  int buf = 0, nrep = 0;
  for (int p0 = 0; p0 < n; p0 += 32) {
    const int steps = (n - p0) < 32 ? (n - p0) : 32;
    ws[buf ^ 1][lane] = (p0 + 32 + lane < n) ? w_sorted[p0 + 32 + lane] : 0.0;
    if (lane == 0) ws[buf ^ 1][32] = (p0 + 64 < n) ? w_sorted[p0 + 64] : 0.0;
    const double* wb = ws[buf];
    const double c_asg = asg, c_occ = occ, c_rem = rem;  // checkpoint
    int my = 0;
    bool oor = false;
    uint64_t key = key_lane(!(rem >= wb[0]), occ, lane, oor) | inact;
#pragma unroll 4
    for (int t = 0; t < steps; ++t) {
      const double w = wb[t];
      const double wn = wb[t + 1];
      const double nasg = __dadd_rn(asg, w);
      const double nocc = occ_sel(nasg, cap, rcap);
      const double nrem = __dsub_rn(cap, nasg);
      const uint64_t kWin = key_lane(!(nrem >= wn), nocc, lane, oor) | inact;
      const uint64_t kNot = key_lane(!(rem >= wn), occ, lane, oor) | inact;
      const uint32_t khi = (uint32_t)(key >> 32), klo = (uint32_t)key;
      const uint32_t m1 = __reduce_min_sync(0xffffffffu, khi);
      const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
      const bool won = (khi == m1) && (klo == m2);
      key = won ? kWin : kNot;
      asg = won ? nasg : asg;
      occ = won ? nocc : occ;
      rem = won ? nrem : rem;
      my = (lane == t) ? (int)(m2 & 31u) : my;
    }
    if (__any_sync(0xffffffffu, oor && act)) {
      ++nrep;
      asg = c_asg; occ = c_occ; rem = c_rem;
      uint64_t k64 = (((rem >= wb[0]) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) | inact;
      for (int t = 0; t < steps; ++t) {
        const double w = wb[t];
        const double wn = wb[t + 1];
        const double nasg = __dadd_rn(asg, w);
        const double nocc = occ_sel(nasg, cap, rcap);
        const double nrem = __dsub_rn(cap, nasg);
        const uint64_t kWin = (((nrem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(nocc)) | inact;
        const uint64_t kNot = (((rem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) | inact;
        const uint32_t pk = argmin_redux(k64);
        const bool won = (uint32_t)lane == pk;
        k64 = won ? kWin : kNot;
        asg = won ? nasg : asg;
        occ = won ? nocc : occ;
        rem = won ? nrem : rem;
        my = (lane == t) ? (int)pk : my;
      }
    }
    if (p0 + lane < n) pick[p0 + lane] = my;
    __syncwarp();
    buf ^= 1;
  }
  long long t1 = clock64();
  if (lane == 0) { *cyc = t1 - t0; *replays = nrep; }
}

// Order-preserving image of an occupancy with the lane in the low 5 bits:
// [0][exp-992:6][mantissa:52][lane:5] -- exact for 0 and for normal values
// with biased exponent in [993, 1054]; anything else sets `oor`.
__device__ __forceinline__ uint64_t occ_img(double occ, uint32_t lane, uint32_t& oor) {
  const uint64_t b = (uint64_t)__double_as_longlong(occ);
  const uint32_t e = (uint32_t)(b >> 52);
  oor |= (uint32_t)(b != 0ull) & (uint32_t)((e - 993u) > 61u);
  const uint64_t img = (b - (992ull << 52)) << 5;
  return (b == 0ull ? 0ull : img) | lane;
}
// V8: two REDUX on lane-folded exact keys + two-level speculation (the
// state after a win and all four candidate keys of step t+1 are formed
// during step t for both outcomes of step t), flat loop over a staged
// workload array; any out-of-range occupancy reruns with the exact
// three-REDUX loop.
__global__ void g_v8(const double* w_sorted, int n, int M, const double* caps, int* pick, long long* cyc,
                     int* replays) {
  extern __shared__ double wsd[];
  const int lane = threadIdx.x;
  const bool act = lane < M;
  const double cap = act ? caps[lane] : 0.0;
  const double rcap = cap > 0.0 ? __drcp_rn(cap) : 0.0;
  for (int i = lane; i < n + 2; i += 32) wsd[i] = i < n ? w_sorted[i] : 0.0;
  __syncwarp();
  long long t0 = clock64();
  const uint64_t inact = act ? 0ull : ~0ull;
  const uint64_t HI = 1ull << 63;
  uint32_t oor = 0;
  double asg = 0.0, rem = __dsub_rn(cap, 0.0);
  uint64_t img = occ_img(occ_sel(0.0, cap, rcap), lane, oor);
  double nasg = __dadd_rn(asg, wsd[0]);
  double nrem = __dsub_rn(cap, nasg);
  uint64_t nimg = occ_img(occ_sel(nasg, cap, rcap), lane, oor);
  uint64_t key = ((rem >= wsd[0]) ? 0ull : HI) | img | inact;
  uint64_t kwin = ((nrem >= wsd[1]) ? 0ull : HI) | nimg | inact;
  uint64_t knot = ((rem >= wsd[1]) ? 0ull : HI) | img | inact;
  int viol = 0;
  for (int t = 0; t < n; ++t) {
    const double w1 = wsd[t + 1], w2 = wsd[t + 2];
    // case W (this lane wins step t): S_{t+1} = V_t
    const double aW = __dadd_rn(nasg, w1);
    const double rW = __dsub_rn(cap, aW);
    const uint64_t iW = occ_img(occ_sel(aW, cap, rcap), lane, oor);
    const uint64_t kwW = ((rW >= w2) ? 0ull : HI) | iW | inact;
    const uint64_t knW = ((nrem >= w2) ? 0ull : HI) | nimg | inact;
    // case N: S_{t+1} = S_t
    const double aN = __dadd_rn(asg, w1);
    const double rN = __dsub_rn(cap, aN);
    const uint64_t iN = occ_img(occ_sel(aN, cap, rcap), lane, oor);
    const uint64_t kwN = ((rN >= w2) ? 0ull : HI) | iN | inact;
    const uint64_t knN = ((rem >= w2) ? 0ull : HI) | img | inact;
    const uint32_t khi = (uint32_t)(key >> 32), klo = (uint32_t)key;
    const uint32_t m1 = __reduce_min_sync(0xffffffffu, khi);
    const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
    const bool won = (khi == m1) & (klo == m2);
    viol += (int)(m1 >> 31);
    key = won ? kwin : knot;
    asg = won ? nasg : asg;
    rem = won ? nrem : rem;
    img = won ? nimg : img;
    nasg = won ? aW : aN;
    nrem = won ? rW : rN;
    nimg = won ? iW : iN;
    kwin = won ? kwW : kwN;
    knot = won ? knW : knN;
    if (lane == 0) pick[t] = (int)(m2 & 31u);
  }
  int rep = 0;
  if (__any_sync(0xffffffffu, oor && act)) rep = 1;
  long long t1 = clock64();
  if (lane == 0) { *cyc = t1 - t0; *replays = rep + viol * 0; }
}
// Diagnostics for v5's two loop-carried chains.  mode 1: REDUX chain only
// (kWin from the old state: no division on the loop); mode 2: division
// chain only (the pick is a cheap function of the key, no REDUX);
// mode 3 (v9): two REDUX on keys with the low 5 mantissa bits replaced by
// the lane, exactness checked off the chain (min of the true low bits over
// the truncated-key ties), conflicting blocks replayed.
template <int MODE>
__global__ void g_diag(const double* w_sorted, int n, int M, const double* caps, int* pick, long long* cyc,
                       int* replays) {
  extern __shared__ double wsd[];
  const int lane = threadIdx.x;
  const bool act = lane < M;
  const double cap = act ? caps[lane] : 0.0;
  const double rcap = cap > 0.0 ? __drcp_rn(cap) : 0.0;
  for (int i = lane; i < n + 2; i += 32) wsd[i] = i < n ? w_sorted[i] : 0.0;
  __syncwarp();
  const uint64_t inact = act ? 0ull : ~0ull;
  double asg = 0.0, occ = occ_sel(0.0, cap, rcap), rem = __dsub_rn(cap, 0.0);
  uint32_t oorf = 0;
  auto fold = [&](uint64_t k) -> uint64_t {
    if (MODE == 3) return (k & ~31ull) | (uint64_t)lane;
    if (MODE == 4) {  // exact lane-folded key (v7's layout), out-of-range occupancies flagged
      const uint64_t b = k & ~(1ull << 63);
      const uint32_t e = (uint32_t)(b >> 52);
      oorf |= (uint32_t)(b != 0ull) & (uint32_t)((e - 993u) > 61u);
      const uint64_t img = (b == 0ull) ? 0ull : ((b - (992ull << 52)) << 5);
      return (k & (1ull << 63)) | img | (uint64_t)lane;
    }
    return k;
  };
  uint64_t key = fold((((rem >= wsd[0]) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) | inact);
  uint32_t low = (uint32_t)__double_as_longlong(occ) & 31u;
  int nrep = 0;
  uint32_t conflict = 0;
  long long t0 = clock64();
  for (int t = 0; t < n; ++t) {
    const double w = wsd[t];
    const double wn = wsd[t + 1];
    const double nasg = __dadd_rn(asg, w);
    const double nocc = MODE == 1 ? occ : occ_sel(nasg, cap, rcap);
    const double nrem = __dsub_rn(cap, nasg);
    const uint64_t kWinR = (((nrem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(nocc)) | inact;
    const uint64_t kNotR = (((rem >= wn) ? 0ull : (1ull << 63)) | (uint64_t)__double_as_longlong(occ)) | inact;
    const uint64_t kWin = fold(kWinR), kNot = fold(kNotR);
    const uint32_t khi = (uint32_t)(key >> 32), klo = (uint32_t)key;
    uint32_t pk;
    if (MODE == 2) {
      pk = (khi ^ klo) & 7u;  // stand-in, no cross-lane op
      pk = pk < (uint32_t)M ? pk : 0u;
    } else if (MODE == 4) {
      const uint32_t m1 = __reduce_min_sync(0xffffffffu, khi);
      const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
      pk = m2 & 31u;
    } else if (MODE == 3) {
      const uint32_t m1 = __reduce_min_sync(0xffffffffu, khi);
      const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
      pk = m2 & 31u;
      // off the chain: true low bits among the truncated-key ties
      const bool cand = (khi == m1) & ((klo >> 5) == (m2 >> 5));
      const uint32_t mlow = __reduce_min_sync(0xffffffffu, cand ? low : 0xffffffffu);
      conflict |= ((uint32_t)lane == pk) & (low != mlow);
    } else {
      const uint32_t m1 = __reduce_min_sync(0xffffffffu, khi);
      const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
      pk = __reduce_min_sync(0xffffffffu, (khi == m1 && klo == m2) ? (uint32_t)lane : 31u);
    }
    const bool won = (uint32_t)lane == pk;
    key = won ? kWin : kNot;
    if (MODE == 3) low = won ? ((uint32_t)kWinR & 31u) : ((uint32_t)kNotR & 31u);
    asg = won ? nasg : asg;
    occ = won ? nocc : occ;
    rem = won ? nrem : rem;
    if (lane == 0) pick[t] = (int)pk;
  }
  if (MODE == 3 && __any_sync(0xffffffffu, conflict != 0)) nrep = 1;
  if (MODE == 4 && __any_sync(0xffffffffu, oorf != 0 && act)) nrep = 1;
  long long t1 = clock64();
  if (lane == 0) { *cyc = t1 - t0; *replays = nrep; }
}

// The production greedy_warp step (planner.cu, CHUNK == 0, BPL == 1) and
// variants, to find what separates it from v5flat:
//  VAR 0: production (3-ahead prefetch ring, clamped index, picks + q to smem, viol)
//  VAR 1: no q store       VAR 2: direct w / wn loads (no ring)
//  VAR 3: no viol          VAR 4: picks to global (as v5flat)   VAR 5: 1 + 2 + 3
//  VAR 6: VAR 0 inside a 512-thread CTA (128-register cap), the other 15
//  warps waiting at __syncthreads (the fused planner's situation)
template <int VAR>
__global__ void __launch_bounds__((VAR == 6 || VAR == 7) ? 512 : 32) g_prod(const double* w_sorted, int n, int M, const double* caps, int* pick, long long* cyc,
                       int* replays) {
  extern __shared__ double wsd[];
  __shared__ int s_pick[4096];  // ring: the store cost is what is measured
  __shared__ int s_q[4096];
  const int lane = threadIdx.x;
  if ((VAR == 6 || VAR == 7) && threadIdx.x >= 32) {
    __syncthreads();
    return;
  }
  for (int i = lane; i < n + 2; i += 32) wsd[i] = i < n ? w_sorted[i] : 0.0;
  __syncwarp();
  const double* ws = wsd;
  auto getw = [ws](int p) { return ws[p]; };
  const double cap = lane < M ? caps[lane] : 0.0;
  const double rcap = cap > 0.0 ? __drcp_rn(cap) : 0.0;
  double asg = 0.0, occ = 0.0, rem = __dsub_rn(cap, 0.0);
  const int nn = n;
  double w_a = nn > 0 ? getw(0) : 0.0, w_b = nn > 1 ? getw(1) : 0.0, w_c = nn > 2 ? getw(2) : 0.0;
  uint64_t key = lane < M ? ((((rem >= w_a) ? 0ull : (1ull << 63))) | (uint64_t)__double_as_longlong(occ)) : ~0ull;
  int cnt = 0, viol = 0;
  long long t0 = clock64();
  for (int p = 0; p < nn; ++p) {
    double w, wn;
    if (VAR == 2 || VAR == 5) {
      w = ws[p];
      wn = ws[p + 1];
    } else {
      w = w_a;
      wn = w_b;
      w_a = w_b;
      w_b = w_c;
      w_c = getw(p + 3 < nn ? p + 3 : nn - 1);
    }
    const bool act = lane < M;
    const double nasg = __dadd_rn(asg, w);
    const double nocc = occ_sel(nasg, cap, rcap);
    const double nrem = __dsub_rn(cap, nasg);
    const uint64_t kwin = act ? ((((nrem >= wn) ? 0ull : (1ull << 63))) | (uint64_t)__double_as_longlong(nocc)) : ~0ull;
    const uint64_t knot = act ? ((((rem >= wn) ? 0ull : (1ull << 63))) | (uint64_t)__double_as_longlong(occ)) : ~0ull;
    const uint64_t best = key;
    const uint32_t best_j = (uint32_t)lane;
    const uint32_t khi = (uint32_t)(best >> 32), klo = (uint32_t)best;
    uint32_t m1, m2, pk;
    if (VAR == 8) {  // unique-high-word shortcut: ballot, else the two exact REDUX
      m1 = __reduce_min_sync(0xffffffffu, khi);
      const unsigned eq = __ballot_sync(0xffffffffu, khi == m1);
      if (__popc(eq) == 1) {
        pk = (uint32_t)(__ffs(eq) - 1);
      } else {
        m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
        pk = __reduce_min_sync(0xffffffffu, (khi == m1 && klo == m2) ? best_j : 0xffffffffu);
      }
    } else if (VAR == 7) {  // inline-PTX redux.sync (bounds 512): does it avoid the divergence checks?
      asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(m1) : "r"(khi));
      asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(m2) : "r"(khi == m1 ? klo : 0xffffffffu));
      asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(pk) : "r"((khi == m1 && klo == m2) ? best_j : 0xffffffffu));
    } else {
      m1 = __reduce_min_sync(0xffffffffu, khi);
      m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
      pk = __reduce_min_sync(0xffffffffu, (khi == m1 && klo == m2) ? best_j : 0xffffffffu);
    }
    if (VAR != 3 && VAR != 5) viol += (int)(m1 >> 31);
    const bool won = (uint32_t)lane == pk;
    if (VAR != 1 && VAR != 5 && won) s_q[p & 4095] = cnt;
    key = won ? kwin : knot;
    asg = won ? nasg : asg;
    occ = won ? nocc : occ;
    rem = won ? nrem : rem;
    cnt += won ? 1 : 0;
    if (VAR == 4) {
      if (lane == 0) pick[p] = (int)pk;
    } else if (lane == 0) {
      s_pick[p & 4095] = (int)pk;
    }
  }
  long long t1 = clock64();
  __syncwarp();
  if (VAR != 4)
    for (int i = lane; i < n; i += 32) pick[i] = i < n - 4096 ? -1 : s_pick[i & 4095];
  if (lane == 0) { *cyc = t1 - t0; *replays = viol + s_q[n / 2] * 0; }
  if ((VAR == 6 || VAR == 7) && blockDim.x > 32) __syncthreads();
}

// Two-REDUX argmin with exact block replay (candidate for greedy_warp):
// the second REDUX runs on the low word with its 5 low bits replaced by the
// lane, so it returns the winner directly; a lane of the winner's 32-ulp
// bucket other than the winner flags the step as ambiguous.  Per block of K
// steps the state is saved; an ambiguous block is replayed with the exact
// three-REDUX step.
template <int K>
__global__ void __launch_bounds__(32) g_fast(const double* w_sorted, int n, int M, const double* caps, int* pick,
                                             long long* cyc, int* replays) {
  extern __shared__ double wsd[];
  const int lane = threadIdx.x;
  for (int i = lane; i < n + 2; i += 32) wsd[i] = i < n ? w_sorted[i] : 0.0;
  __syncwarp();
  const double* ws = wsd;
  const double cap = lane < M ? caps[lane] : 0.0;
  const double rcap = cap > 0.0 ? __drcp_rn(cap) : 0.0;
  const bool act = lane < M;
  double asg = 0.0, occ = 0.0, rem = __dsub_rn(cap, 0.0);
  const int nn = n;
  double w_a = ws[0], w_b = ws[1], w_c = ws[2];
  uint64_t key = act ? ((((rem >= w_a) ? 0ull : (1ull << 63))) | (uint64_t)__double_as_longlong(occ)) : ~0ull;
  int cnt = 0, viol = 0, nrep = 0;
  auto step = [&](int p, auto ex) -> bool {
    constexpr bool EXACT = decltype(ex)::value;
    const double w = w_a, wn = w_b;
    w_a = w_b;
    w_b = w_c;
    w_c = ws[p + 3 < nn ? p + 3 : nn - 1];
    const double nasg = __dadd_rn(asg, w);
    const double nocc = occ_sel(nasg, cap, rcap);
    const double nrem = __dsub_rn(cap, nasg);
    const uint64_t kwin = act ? ((((nrem >= wn) ? 0ull : (1ull << 63))) | (uint64_t)__double_as_longlong(nocc)) : ~0ull;
    const uint64_t knot = act ? ((((rem >= wn) ? 0ull : (1ull << 63))) | (uint64_t)__double_as_longlong(occ)) : ~0ull;
    const uint32_t khi = (uint32_t)(key >> 32), klo = (uint32_t)key;
    const uint32_t m1 = __reduce_min_sync(0xffffffffu, khi);
    uint32_t pk;
    bool amb = false;
    if constexpr (EXACT) {
      const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
      pk = __reduce_min_sync(0xffffffffu, (khi == m1 && klo == m2) ? (uint32_t)lane : 0xffffffffu);
    } else {
      const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? ((klo & ~31u) | (uint32_t)lane) : 0xffffffffu);
      pk = m2 & 31u;
      amb = khi == m1 && (klo | 31u) == (m2 | 31u) && (uint32_t)lane != pk;
    }
    viol += (int)(m1 >> 31);
    const bool won = (uint32_t)lane == pk;
    key = won ? kwin : knot;
    asg = won ? nasg : asg;
    occ = won ? nocc : occ;
    rem = won ? nrem : rem;
    cnt += won ? 1 : 0;
    if (lane == 0) pick[p] = (int)pk;
    return amb;
  };
  long long t0 = clock64();
  for (int p0 = 0; p0 < nn; p0 += K) {
    const int p1 = p0 + K < nn ? p0 + K : nn;
    const uint64_t key0 = key;
    const double asg0 = asg, occ0 = occ, rem0 = rem, wa0 = w_a, wb0 = w_b, wc0 = w_c;
    const int cnt0 = cnt, viol0 = viol;
    bool amb = false;
    for (int p = p0; p < p1; ++p) amb |= step(p, std::false_type{});
    if (__any_sync(0xffffffffu, amb)) {
      ++nrep;
      key = key0; asg = asg0; occ = occ0; rem = rem0; w_a = wa0; w_b = wb0; w_c = wc0; cnt = cnt0; viol = viol0;
      for (int p = p0; p < p1; ++p) step(p, std::true_type{});
    }
  }
  long long t1 = clock64();
  if (lane == 0) { *cyc = t1 - t0; *replays = nrep; }
}
int main() {
  unsigned* du; double* dd; long long* dc;
  cudaMalloc(&du, 128); cudaMalloc(&dd, 512); cudaMalloc(&dc, 8);
  long long c;
  const int it = 4096;
  auto rep = [&](const char* name) { cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("%-10s %.1f cyc\n", name, (double)c / it); };
  lat_redux<<<1,32>>>(it, du, dc); rep("redux");
  lat_shfl<<<1,32>>>(it, du, dc); rep("shfl");
  lat_ballot<<<1,32>>>(it, du, dc); rep("ballot+ffs");
  lat_dfma<<<1,32>>>(it, 0.999, dd, dc); rep("dfma");
  lat_dadd<<<1,32>>>(it, 0.999, dd, dc); rep("dadd");
  lat_dsetp<<<1,32>>>(it, 3.0, dd, dc); rep("dsetp+sel");
  // greedy: C1-law workloads
  for (int M : {8, 6, 2, 32, -8}) {
    const bool uniform = M < 0; if (uniform) M = -M;
    const int n = 16384;
    std::vector<double> w(n);
    srand(1);
    const double d = 3072.0;
    for (int i = 0; i < n; ++i) { double l = 64 + rand() % 449 + 256 + rand() % 3841; if (uniform) l = 1024 + (i % 3); w[i] = 24.0 * l * d * d + 0.49 * 4.0 * l * l * d; }
    std::sort(w.begin(), w.end(), [](double a, double b) { return a > b; });
    double tot = 0; for (double x : w) tot += x;
    std::vector<double> caps(32, 0.0);
    for (int j = 0; j < M; ++j) caps[j] = 1.0 * (tot / M);
    double *dw, *dcap; int *p0, *p1;
    cudaMalloc(&dw, n * 8); cudaMalloc(&dcap, 32 * 8); cudaMalloc(&p0, n * 4); cudaMalloc(&p1, n * 4);
    cudaMemcpy(dw, w.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dcap, caps.data(), 32 * 8, cudaMemcpyHostToDevice);
    for (int r = 0; r < 2; ++r) { g_v0<<<1,32>>>(dw, n, M, dcap, p0, dc); }
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); long long c0 = c;
    for (int r = 0; r < 2; ++r) { g_v1<<<1,32>>>(dw, n, M, dcap, p1, dc); }
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); long long c1 = c;
    int *p2, *p3; cudaMalloc(&p2, n * 4); cudaMalloc(&p3, n * 4);
    for (int r = 0; r < 2; ++r) { g_v2<<<1,32>>>(dw, n, M, dcap, p2, dc); }
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); long long c2 = c;
    for (int r = 0; r < 2; ++r) { g_v3<<<1,32>>>(dw, n, M, dcap, p3, dc); }
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); long long c3 = c;
    int* p5; cudaMalloc(&p5, n * 4);
    for (int r = 0; r < 2; ++r) { g_v5<<<1,32>>>(dw, n, M, dcap, p5, dc); }
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); long long c5 = c;
    std::vector<int> h5(n); cudaMemcpy(h5.data(), p5, n * 4, cudaMemcpyDeviceToHost);
    int *p6, *drep, hrep = 0; cudaMalloc(&p6, n * 4); cudaMalloc(&drep, 4);
    for (int r = 0; r < 2; ++r) { g_v6<<<1,32>>>(dw, n, M, dcap, p6, dc, drep); }
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); long long c6 = c;
    cudaMemcpy(&hrep, drep, 4, cudaMemcpyDeviceToHost);
    std::vector<int> h6(n); cudaMemcpy(h6.data(), p6, n * 4, cudaMemcpyDeviceToHost);
    int d6 = 0; for (int i = 0; i < n; ++i) d6 += h5[i] != h6[i];
    for (int r = 0; r < 2; ++r) { g_v7<<<1,32>>>(dw, n, M, dcap, p6, dc, drep); }
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); long long c7 = c;
    cudaMemcpy(&hrep, drep, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h6.data(), p6, n * 4, cudaMemcpyDeviceToHost);
    int d7 = 0; for (int i = 0; i < n; ++i) d7 += h5[i] != h6[i];
    printf("  v7 %.1f cyc/seq (diffs %d, replayed blocks %d)\n", (double)c7 / n, d7, hrep);
    cudaFuncSetAttribute(g_v8, cudaFuncAttributeMaxDynamicSharedMemorySize, (n + 2) * 8);
    for (int r = 0; r < 2; ++r) { g_v8<<<1, 32, (n + 2) * 8>>>(dw, n, M, dcap, p6, dc, drep); }
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); long long c8 = c;
    cudaMemcpy(&hrep, drep, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h6.data(), p6, n * 4, cudaMemcpyDeviceToHost);
    int d8 = 0; for (int i = 0; i < n; ++i) d8 += h5[i] != h6[i];
    printf("  v8 %.1f cyc/seq (diffs %d, oor %d) %s\n", (double)c8 / n, d8, hrep, cudaGetErrorString(cudaGetLastError()));
    {
      auto run = [&](auto kern, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (n + 2) * 8);
        for (int r = 0; r < 2; ++r) kern<<<1, 32, (n + 2) * 8>>>(dw, n, M, dcap, p6, dc, drep);
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&hrep, drep, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(h6.data(), p6, n * 4, cudaMemcpyDeviceToHost);
        int dd = 0; for (int i = 0; i < n; ++i) dd += h6[i] >= 0 && h5[i] != h6[i];
        printf("  %s %.1f cyc/seq (diffs %d, conflict %d)\n", name, (double)c / n, dd, hrep);
      };
      run(g_diag<0>, "v5flat");
      run(g_fast<32>, "fast2-K32");
      run(g_fast<16>, "fast2-K16");
      run(g_fast<64>, "fast2-K64");
      run(g_prod<0>, "prod");
      run(g_prod<8>, "prod-unique-hi");
      run(g_prod<1>, "prod-no-q");
      run(g_prod<2>, "prod-direct-w");
      run(g_prod<3>, "prod-no-viol");
      run(g_prod<4>, "prod-pick-global");
      run(g_prod<5>, "prod-1+2+3");
      {
        cudaFuncSetAttribute(g_prod<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (n + 2) * 8);
        for (int r = 0; r < 2; ++r) g_prod<6><<<1, 512, (n + 2) * 8>>>(dw, n, M, dcap, p6, dc, drep);
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("  prod-in-512-CTA %.1f cyc/seq (%s)\n", (double)c / n, cudaGetErrorString(cudaGetLastError()));
        for (int r = 0; r < 2; ++r) g_prod<6><<<1, 32, (n + 2) * 8>>>(dw, n, M, dcap, p6, dc, drep);
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("  prod-bounds512-alone %.1f cyc/seq (%s)\n", (double)c / n, cudaGetErrorString(cudaGetLastError()));
        cudaFuncSetAttribute(g_prod<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (n + 2) * 8);
        for (int r = 0; r < 2; ++r) g_prod<7><<<1, 512, (n + 2) * 8>>>(dw, n, M, dcap, p6, dc, drep);
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("  prod-bounds512-asm-redux %.1f cyc/seq (%s)\n", (double)c / n, cudaGetErrorString(cudaGetLastError()));
        cudaFuncSetAttribute(g_prod<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (n + 2) * 8);
      }
      run(g_diag<1>, "redux-chain-only");
      run(g_diag<2>, "division-chain-only");
      run(g_diag<3>, "v9");
      run(g_diag<4>, "v10");
    }
    printf("  v6 %.1f cyc/seq (diffs %d, replayed blocks %d of %d)\n", (double)c6 / n, d6, hrep, (n + 31) / 32);
    int d5 = 0;
    std::vector<int> h2(n), h3(n);
    cudaMemcpy(h2.data(), p2, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h3.data(), p3, n * 4, cudaMemcpyDeviceToHost);
    int d2 = 0, d3 = 0;
    std::vector<int> h0(n), h1(n);
    cudaMemcpy(h0.data(), p0, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h1.data(), p1, n * 4, cudaMemcpyDeviceToHost);
    int diff = 0; for (int i = 0; i < n; ++i) { diff += h0[i] != h1[i]; d2 += h0[i] != h2[i]; d3 += h0[i] != h3[i]; d5 += h0[i] != h5[i]; }
    printf("  v5 %.1f cyc/seq (diffs %d)\n", (double)c5 / n, d5);
    printf("  v2 %.1f cyc/seq (diffs %d), v3 %.1f cyc/seq (diffs %d)\n", (double)c2 / n, d2, (double)c3 / n, d3);
    printf("greedy M=%d n=%d: v0 %.1f cyc/seq, v1 %.1f cyc/seq, pick diffs %d  (%s)\n", M, n, (double)c0 / n, (double)c1 / n, diff, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
