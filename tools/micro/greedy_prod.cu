// The production greedy (csrc/greedy.cuh greedy_warp, as k_greedy_staged
// runs it) timed beside greedy_micro.cu's hand copy of its step on the same
// sorted workloads (diagnostics).
//   nvcc -O3 -std=c++17 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a \
//        -I../../paper_2508_06001_b200/csrc -o greedy_prod greedy_prod.cu
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
    auto run = [&](auto kern, const char* name) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (n + 4) * 8);
      long long c = 0;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int r = 0; r < 3; ++r) kern<<<1, 32, (n + 4) * 8>>>(a, dw, n, dc);
      cudaEventRecord(e0);
      kern<<<1, 32, (n + 4) * 8>>>(a, dw, n, dc);
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
  }
  return 0;
}
