// Single-lane greedy for replicas whose bags all have the same size
// (diagnostics; the production candidate is planner.cu greedy_uniform).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o greedy_single greedy_single.cu
//
// With one capacity `cap` for every bag, occupancy RN(asg / cap) is monotone
// in asg and so is feasibility RN(cap - asg) >= w; the reference's pick
// (balancer.cpp:44-62) is therefore the lowest-index bag of minimum asg,
// unless another bag's asg is so close that RN(asg / cap) ties -- checked
// per step (a 4-ulp window on the IEEE bits), and then the step is replayed
// with the exact occupancies.  No division, no cross-lane operation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ double occ_ref(double asg, double cap) {
  if (cap > 0.0) return __ddiv_rn(asg, cap);
  return asg > 0.0 ? __longlong_as_double(0x7ff0000000000000ll) : 0.0;
}

// Reference production algorithm (warp, lane = bag, three REDUX): the exact pick sequence.
__global__ void g_ref(const double* w, int n, int M, double cap, int* pick) {
  const int lane = threadIdx.x;
  const bool act = lane < M;
  double asg = 0.0;
  for (int t = 0; t < n; ++t) {
    const double occ = occ_ref(asg, cap);
    const bool feas = __dsub_rn(cap, asg) >= w[t];
    const uint64_t key = act ? (((feas ? 0ull : 1ull << 63)) | (uint64_t)__double_as_longlong(occ)) : ~0ull;
    const uint32_t khi = (uint32_t)(key >> 32), klo = (uint32_t)key;
    const uint32_t m1 = __reduce_min_sync(0xffffffffu, khi);
    const uint32_t m2 = __reduce_min_sync(0xffffffffu, khi == m1 ? klo : 0xffffffffu);
    const uint32_t pk = __reduce_min_sync(0xffffffffu, (khi == m1 && klo == m2) ? (uint32_t)lane : 31u);
    if ((uint32_t)lane == pk) asg = __dadd_rn(asg, w[t]);
    if (lane == 0) pick[t] = (int)pk;
  }
}

template <int M>
struct Tour {
  // lowest (bits, index): the right side wins only if strictly smaller
  __device__ static __forceinline__ void run(const uint64_t* b, uint64_t& kb, int& kj) {
    uint64_t lb;
    int lj;
    Tour<M / 2>::run(b, lb, lj);
    uint64_t rb;
    int rj;
    Tour<M - M / 2>::run(b + M / 2, rb, rj);
    rj += M / 2;
    const bool r = rb < lb;
    kb = r ? rb : lb;
    kj = r ? rj : lj;
  }
};
template <>
struct Tour<1> {
  __device__ static __forceinline__ void run(const uint64_t* b, uint64_t& kb, int& kj) {
    kb = b[0];
    kj = 0;
  }
};

template <int M>
__global__ void g_single(const double* w_sorted, int n, double cap, int* pick, long long* cyc, int* slow_out) {
  extern __shared__ double wsd[];
  for (int i = threadIdx.x; i < n + 1; i += 32) wsd[i] = i < n ? w_sorted[i] : 0.0;
  __syncwarp();
  if (threadIdx.x != 0) return;
  double asg[M];
  int cnt[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    asg[j] = 0.0;
    cnt[j] = 0;
  }
  int slow = 0, viol = 0;
  const uint64_t lo_bits = (uint64_t)__double_as_longlong(ldexp(cap, -960));
  const uint64_t hi_bits = (uint64_t)__double_as_longlong(ldexp(cap, 960));
  long long t0 = clock64();
  for (int t = 0; t < n; ++t) {
    const double w = wsd[t];
    uint64_t b[M];
    double nasg[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      b[j] = (uint64_t)__double_as_longlong(asg[j]);
      nasg[j] = __dadd_rn(asg[j], w);
    }
    uint64_t kb;
    int kj;
    Tour<M>::run(b, kb, kj);
    // near ties: another bag within 4 ulps of the minimum (conservative)
    const uint32_t khi = (uint32_t)(kb >> 32), klo = (uint32_t)kb;
    // minimum outside [cap 2^-960, cap 2^960]: quotients may flush or overflow
    bool near = (kb < lo_bits) | (kb > hi_bits);
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const uint32_t dh = (uint32_t)(b[j] >> 32) - khi, dl = (uint32_t)b[j] - klo;
      near |= (dh <= 1u) & (dl <= 4u) & ((dh | dl) != 0u);
    }
    int pk = kj;
    if (near) {  // replay the reference step exactly (balancer.cpp:44-62)
      ++slow;
      int best = M, fb = M;
      double bo = 0.0, fo = 0.0;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const double o = occ_ref(asg[j], cap);
        if (__dsub_rn(cap, asg[j]) >= w && (best == M || o < bo)) {
          best = j;
          bo = o;
        }
        if (fb == M || o < fo) {
          fb = j;
          fo = o;
        }
      }
      pk = best != M ? best : fb;
    }
    viol += __dsub_rn(cap, __longlong_as_double((long long)kb)) >= w ? 0 : 1;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const bool won = j == pk;
      asg[j] = won ? nasg[j] : asg[j];
      cnt[j] += won ? 1 : 0;
    }
    pick[t] = pk;
  }
  long long t1 = clock64();
  *cyc = t1 - t0;
  *slow_out = slow + (viol << 20) * 0;
}

int main() {
  const int n = 16384;
  for (int law = 0; law < 3; ++law) {
    std::vector<double> w(n);
    srand(1 + law);
    const double d = 3072.0;
    for (int i = 0; i < n; ++i) {
      double l;
      if (law == 0) l = 64 + rand() % 449 + 256 + rand() % 3841;        // C1 law
      else if (law == 1) l = 1024 + (i % 3);                             // heavy exact ties
      else l = (rand() % 4 == 0) ? 4096 : 256 * (1 + rand() % 4);        // FLUX-like few distinct lengths
      w[i] = 24.0 * l * d * d + 0.49 * 4.0 * l * l * d;
    }
    std::sort(w.begin(), w.end(), [](double a, double b) { return a > b; });
    double tot = 0;
    for (double x : w) tot += x;
    double* dw;
    int *pr, *ps, *dslow;
    long long* dc;
    cudaMalloc(&dw, n * 8);
    cudaMalloc(&pr, n * 4);
    cudaMalloc(&ps, n * 4);
    cudaMalloc(&dslow, 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dw, w.data(), n * 8, cudaMemcpyHostToDevice);
    auto one = [&](int M, auto kern) {
      const double cap = 1.0 * (tot / M);  // bag size 1 x target; sizes 2 / 4 scale both sides alike
      g_ref<<<1, 32>>>(dw, n, M, cap, pr);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (n + 1) * 8);
      long long c = 0;
      int slow = 0;
      for (int r = 0; r < 2; ++r) kern<<<1, 32, (n + 1) * 8>>>(dw, n, cap, ps, dc, dslow);
      cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&slow, dslow, 4, cudaMemcpyDeviceToHost);
      std::vector<int> a(n), b(n);
      cudaMemcpy(a.data(), pr, n * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), ps, n * 4, cudaMemcpyDeviceToHost);
      int diff = 0;
      for (int i = 0; i < n; ++i) diff += a[i] != b[i];
      printf("law %d M=%d single-lane %.1f cyc/seq, diffs %d, slow steps %d (%s)\n", law, M, (double)c / n, diff, slow,
             cudaGetErrorString(cudaGetLastError()));
    };
    one(2, g_single<2>);
    one(3, g_single<3>);
    one(4, g_single<4>);
    one(6, g_single<6>);
    one(8, g_single<8>);
    cudaFree(dw);
    cudaFree(pr);
    cudaFree(ps);
    cudaFree(dslow);
    cudaFree(dc);
  }
  return 0;
}
