// The production greedy (csrc/greedy.cuh greedy_warp, as k_greedy_staged
// runs it) timed beside greedy_micro.cu's hand copy of its step on the same
// sorted workloads (diagnostics).
//   nvcc -O3 -std=c++17 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a \
//        -I../../paper_2508_06001_b200/csrc -I../../include -o greedy_prod greedy_prod.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "greedy.cuh"

using namespace sb;

// production code path: PlanArgs in the parameter space, workloads staged in
// shared memory, picks to global memory (k_greedy_staged)
__global__ void __launch_bounds__(32) k_prod(PlanArgs a, const double* sw, int n, long long* cyc) {
  extern __shared__ __align__(16) double stage[];
  const int lane = threadIdx.x;
  for (int i = lane; i < n; i += 32) stage[i] = sw[i];
  __syncwarp();
  const long long t0 = clock64();
  greedy_warp<1, 0>(a, 0, n, *a.total, [&](int p) { return stage[p]; }, [](int) {}, a.pick, nullptr, a.violations);
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// same, with the bag count and topology passed as plain scalars in registers
__global__ void __launch_bounds__(32) k_prod_regs(PlanArgs a, const double* sw, int n, long long* cyc) {
  extern __shared__ __align__(16) double stage[];
  const int lane = threadIdx.x;
  for (int i = lane; i < n; i += 32) stage[i] = sw[i];
  __syncwarp();
  PlanArgs b = a;
  const long long t0 = clock64();
  greedy_warp<1, 0>(b, 0, n, *a.total, [&](int p) { return stage[p]; }, [](int) {}, a.pick, nullptr, a.violations);
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// lengths file (int64, written by the driver script): the planner's own C4
// inputs; workloads as the planner computes them (workload_model.cpp:65-70)
static double host_workload(int64_t len, double d, double gamma) {
  const double l = (double)len;
  double lin = 24.0 * l;
  lin = lin * d;
  lin = lin * d;
  double att = gamma * 4.0;
  att = att * l;
  att = att * l;
  att = att * d;
  return lin + att;
}

// production code with the unclamped prefetch (PADDED: stage has 3 spare slots)
__global__ void __launch_bounds__(32) k_prod_pad(PlanArgs a, const double* sw, int n, long long* cyc) {
  extern __shared__ __align__(16) double stage[];
  const int lane = threadIdx.x;
  for (int i = lane; i < n + 4; i += 32) stage[i] = i < n ? sw[i] : 0.0;
  __syncwarp();
  const long long t0 = clock64();
  greedy_warp<1, 0, false, true>(a, 0, n, *a.total, [&](int p) { return stage[p]; }, [](int) {}, a.pick, nullptr,
                                 a.violations);
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// register budget probes: the same kernel as k_prod_pad under a 128- and a
// 64-register cap (the fused planner's 512-thread CTA allows 128), and a
// 512-thread CTA whose warp 0 runs it (warps 1.. exit)
template <int MINB>
__global__ void __launch_bounds__(32, MINB) k_prod_cap(PlanArgs a, const double* sw, int n, long long* cyc) {
  extern __shared__ __align__(16) double stage[];
  const int lane = threadIdx.x;
  for (int i = lane; i < n + 4; i += 32) stage[i] = i < n ? sw[i] : 0.0;
  __syncwarp();
  const long long t0 = clock64();
  greedy_warp<1, 0, false, true>(a, 0, n, *a.total, [&](int p) { return stage[p]; }, [](int) {}, a.pick, nullptr,
                                 a.violations);
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}
__global__ void __launch_bounds__(512, 1) k_prod_512(PlanArgs a, const double* sw, int n, long long* cyc) {
  extern __shared__ __align__(16) double stage[];
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  for (int i = lane; i < n + 4; i += 32) stage[i] = i < n ? sw[i] : 0.0;
  __syncwarp();
  const long long t0 = clock64();
  greedy_warp<1, 0, false, true>(a, 0, n, *a.total, [&](int p) { return stage[p]; }, [](int) {}, a.pick, nullptr,
                                 a.violations);
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// the fused planner's shape: warps 1.. wait at a CTA barrier while warp 0
// runs the greedy (SYNC); plus the warp-strided replica loop that makes ptxas
// guard the REDUX chain with BRA.DIV (STRIDED)
template <bool STRIDED>
__global__ void __launch_bounds__(512, 1) k_prod_512sync(PlanArgs a, const double* sw, int n, long long* cyc) {
  extern __shared__ __align__(16) double stage[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < n + 4; i += blockDim.x) stage[i] = i < n ? sw[i] : 0.0;
  __syncthreads();
  const int R = a.R, ng = R < 14 ? R : 14;
  if (warp < ng) {
    for (int rep = STRIDED ? warp : 0; rep < (STRIDED ? R : 1); rep += ng) {
      const long long t0 = clock64();
      greedy_warp<1, 0, false, true>(a, rep, n, *a.total, [&](int p) { return stage[p]; }, [](int) {}, a.pick,
                                     nullptr, a.violations);
      const long long t1 = clock64();
      if (lane == 0) *cyc = t1 - t0;
    }
  }
  __syncthreads();
}

// warp 0 by a constant test (ptxas proves convergence: no BRA.DIV) while the
// others wait at the CTA barrier (W0) / the others exit early (EXIT: control)
template <int V>
__global__ void __launch_bounds__(512, 1) k_prod_512w0(PlanArgs a, const double* sw, int n, long long* cyc) {
  extern __shared__ __align__(16) double stage[];
  __shared__ int flag;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < n + 4; i += blockDim.x) stage[i] = i < n ? sw[i] : 0.0;
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  if (warp == 0) {
    const long long t0 = clock64();
    greedy_warp<1, 0, false, true>(a, 0, n, *a.total, [&](int p) { return stage[p]; }, [](int) {}, a.pick, nullptr,
                                   a.violations);
    const long long t1 = clock64();
    if (lane == 0) *cyc = t1 - t0;
    if (V == 1 && lane == 0) atomicExch(&flag, 1);
  } else if (V == 1) {  // the others sleep-poll a shared flag instead of a barrier
    while (atomicAdd(&flag, 0) == 0) __nanosleep(2000);
  }
  if (V == 0) __syncthreads();
}

// divergent block-wide work and a barrier first, then warps 1.. exit and
// warp 0 runs the greedy (a prefix kernel that keeps the greedy)
__global__ void __launch_bounds__(512, 1) k_prod_512late(PlanArgs a, const double* sw, int n, long long* cyc) {
  extern __shared__ __align__(16) double stage[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < n + 4; i += blockDim.x) stage[i] = i < n ? sw[i] : 0.0;
  if (lane < (threadIdx.x % 7)) stage[n + 3] = 0.0;  // lane-divergent store
  __syncthreads();
  if (warp != 0) return;
  const long long t0 = clock64();
  greedy_warp<1, 0, false, true>(a, 0, n, *a.total, [&](int p) { return stage[p]; }, [](int) {}, a.pick, nullptr,
                                 a.violations);
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// warps 1.. do other work and exit while warp 0 runs the greedy (the hybrid
// prefix with the greedy and the duplicate check side by side)
__global__ void __launch_bounds__(512, 1) k_prod_512work(PlanArgs a, const double* sw, int n, long long* cyc) {
  extern __shared__ __align__(16) double stage[];
  __shared__ unsigned long long table[1024];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < n + 4; i += blockDim.x) stage[i] = i < n ? sw[i] : 0.0;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) table[i] = ~0ull;
  __syncthreads();
  if (warp != 0) {  // open-addressing inserts (the duplicate check's shape)
    for (int i = threadIdx.x - 32; i < (n < 512 ? n : 512); i += blockDim.x - 32) {
      const unsigned long long id = __double_as_longlong(stage[i]);
      unsigned slot = (unsigned)(id * 0x9E3779B97F4A7C15ull >> 54);
      for (;;) {
        const unsigned long long old = atomicCAS(&table[slot], ~0ull, id);
        if (old == ~0ull || old == id) break;
        slot = (slot + 1) & 1023u;
      }
    }
    if (threadIdx.x == 32 && table[0] == 12345ull) a.pick[0] = -1;
    return;
  }
  const long long t0 = clock64();
  greedy_warp<1, 0, false, true>(a, 0, n, *a.total, [&](int p) { return stage[p]; }, [](int) {}, a.pick, nullptr,
                                 a.violations);
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

int main(int argc, char** argv) {
  std::vector<int64_t> lens;
  if (argc > 1) {
    FILE* f = fopen(argv[1], "rb");
    int64_t x;
    while (f && fread(&x, 8, 1, f) == 1) lens.push_back(x);
    if (f) fclose(f);
  }
  const int n = lens.empty() ? 16384 : (int)lens.size();
  for (int M : {8, 4, 2}) {
    std::vector<double> w(n);
    srand(1);
    const double d = 3072.0;
    for (int i = 0; i < n; ++i) {
      const double l = lens.empty() ? 64 + rand() % 449 + 256 + rand() % 3841 : (double)lens[i];
      w[i] = lens.empty() ? 24.0 * l * d * d + 0.49 * 4.0 * l * l * d : host_workload(lens[i], d, 0.49);
    }
    std::sort(w.begin(), w.end(), [](double x, double y) { return x > y; });
    double tot = 0;
    for (double x : w) tot += x;
    std::vector<int32_t> bag_off(M + 1), bag_size(M), bag_ranks(M);
    for (int j = 0; j <= M; ++j) bag_off[j] = j;
    for (int j = 0; j < M; ++j) {
      bag_size[j] = 1;
      bag_ranks[j] = j;
    }
    PlanArgs a{};
    a.W = a.U = a.M = M;
    a.R = 1;
    double *dw, *dtot, *per_gpu, *occ;
    int32_t *dboff, *dbsize, *dbranks, *pick, *bag_count, *viol;
    long long* dc;
    cudaMalloc(&dw, n * 8);
    cudaMalloc(&dtot, 8);
    cudaMalloc(&per_gpu, 64 * 8);
    cudaMalloc(&occ, 64 * 8);
    cudaMalloc(&dboff, 65 * 4);
    cudaMalloc(&dbsize, 64 * 4);
    cudaMalloc(&dbranks, 64 * 4);
    cudaMalloc(&pick, n * 4);
    cudaMalloc(&bag_count, 64 * 4);
    cudaMalloc(&viol, 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dw, w.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dtot, &tot, 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dboff, bag_off.data(), (M + 1) * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dbsize, bag_size.data(), M * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dbranks, bag_ranks.data(), M * 4, cudaMemcpyHostToDevice);
    a.bag_off = dboff;
    a.bag_size = dbsize;
    a.bag_ranks = dbranks;
    a.total = dtot;
    a.per_gpu = per_gpu;
    a.per_bag_occ = occ;
    a.bag_count = bag_count;
    a.pick = pick;
    a.violations = viol;
    a.trace = nullptr;
    auto run = [&](auto kern, const char* name, int threads = 32) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (n + 4) * 8);
      long long c = 0;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int r = 0; r < 3; ++r) kern<<<1, threads, (n + 4) * 8>>>(a, dw, n, dc);
      cudaEventRecord(e0);
      kern<<<1, threads, (n + 4) * 8>>>(a, dw, n, dc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      printf("M=%d %-10s %.1f cyc/seq, kernel %.1f us = %.1f ns/seq -> %.0f MHz (%s)\n", M, name, (double)c / n,
             ms * 1e3, ms * 1e6 / n, (double)c / (ms * 1e-3) / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    run(k_prod, "prod");
    run(k_prod_regs, "prod-regs");
    run(k_prod_pad, "prod-padded");
    run(k_prod_cap<16>, "cap-128reg");
    run(k_prod_cap<32>, "cap-64reg");
    run(k_prod_512, "cta-512", 512);
    run(k_prod_512sync<false>, "512-sync", 512);
    run(k_prod_512sync<true>, "512-strided", 512);
    run(k_prod_512w0<0>, "512-w0-bar", 512);
    run(k_prod_512w0<1>, "512-w0-sleep", 512);
    run(k_prod_512late, "512-late-exit", 512);
    run(k_prod_512work, "512-work-exit", 512);
  }
  return 0;
}
