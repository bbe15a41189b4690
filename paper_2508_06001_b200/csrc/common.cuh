// Shared device/host helpers for libseqbal_cuda.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "seqbal_capi.h"

namespace sb {

// ------------------------------------------------------------ error state
void set_error(const std::string& msg);
extern thread_local std::string g_last_error;

struct Error {
  sb_status code;
  std::string msg;
};

#define SB_CUDA(expr)                                                                 \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) {                                                          \
      cudaGetLastError(); /* clear the non-sticky error so later calls start clean */ \
      throw ::sb::Error{SB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
    }                                                                                 \
  } while (0)

#define SB_CHECK_LAUNCH() SB_CUDA(cudaGetLastError())

void count_launch(int n = 1);

// Status bits in the device status word.
enum : int32_t {
  ST_NEG_LENGTH = 1,    // ConfigError: seq_len must be >= 0 (workload_model.cpp:66)
  ST_DUP_ID = 2,        // ConfigError: duplicate sample_id inside a replica
  ST_CAPACITY = 4,      // capacity exceeded
  ST_BAG_CAP = 8,       // bag count above the compiled limit
  ST_LAYOUT = 16,       // world arena too small for the requested layout
  ST_MISMATCH = 32,     // IntegrityError: source world layout differs from the plan (exchange.cpp:96-123)
};

// ---------------------------------------------------------- device helpers
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// rng.hpp:20-24 derive_key for a fixed list of parts.
__host__ __device__ __forceinline__ uint64_t derive_key4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  uint64_t k = 0x8f51a7c0c0c0f5a3ULL;
  k = splitmix64(k ^ a);
  k = splitmix64(k ^ b);
  k = splitmix64(k ^ c);
  k = splitmix64(k ^ d);
  return k;
}
__host__ __device__ __forceinline__ uint64_t derive_key3(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t k = 0x8f51a7c0c0c0f5a3ULL;
  k = splitmix64(k ^ a);
  k = splitmix64(k ^ b);
  k = splitmix64(k ^ c);
  return k;
}

// Reference gamma-weighted workload (workload_model.cpp:65-70):
//   24.0*l*d*d + gamma*4.0*l*l*d, left-associative, every product rounded.
// The _rn intrinsics forbid FMA contraction so the bits equal the
// reference's default x86-64 build.
__device__ __forceinline__ double gamma_weighted_workload(int64_t len, double d, double gamma) {
  const double l = (double)len;
  double lin = __dmul_rn(24.0, l);
  lin = __dmul_rn(lin, d);
  lin = __dmul_rn(lin, d);
  double att = __dmul_rn(gamma, 4.0);
  att = __dmul_rn(att, l);
  att = __dmul_rn(att, l);
  att = __dmul_rn(att, d);
  return __dadd_rn(lin, att);
}

// l = q * g + r for a sequence length l >= 0 and a bag size g >= 1: 32-bit
// division whenever l fits (every realistic length; the 64-bit divide is a
// ~70-instruction subroutine).
__device__ __forceinline__ void len_divmod(int64_t l, int g, int64_t& q, int& r) {
  if ((uint64_t)l <= 0xffffffffull) {
    const uint32_t l32 = (uint32_t)l, q32 = l32 / (uint32_t)g;
    q = q32;
    r = (int)(l32 - q32 * (uint32_t)g);
  } else {
    q = l / g;
    r = (int)(l - q * g);
  }
}
// chunk_lengths (balancer.cpp:66-82): chunk k of a length-l sequence split g ways
__device__ __forceinline__ int64_t chunk_len(int64_t l, int g, int k) {
  int64_t q;
  int r;
  len_divmod(l, g, q, r);
  return q + (k < r ? 1 : 0);
}
__device__ __forceinline__ int64_t chunk_start(int64_t l, int g, int k) {
  int64_t q;
  int r;
  len_divmod(l, g, q, r);
  return (int64_t)k * q + (k < r ? k : r);
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan (blockDim.x multiple of 32, <= 1024); returns the
// exclusive prefix and writes the block total to *total.  `sh` >= 33 slots.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* sh, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) sh[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T x = lane < nw ? sh[lane] : T(0);
    T xi = warp_incl_scan(x);
    if (lane < nw) sh[lane] = xi - x;
    if (lane == nw - 1) sh[32] = xi;
  }
  __syncthreads();
  T ex = inc - v + sh[warp];
  *total = sh[32];
  __syncthreads();
  return ex;
}

}  // namespace sb
