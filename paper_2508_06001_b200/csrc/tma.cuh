// mbarrier + bulk-copy (TMA, cp.async.bulk) helpers shared by the copy
// engines (exchange.cu) and the planner's shared-memory staging (planner.cu).
#pragma once

#include <cstdint>

namespace sb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}

// Stage `n` doubles from global `src` into shared memory with bulk copies
// (one warp; lane 0 issues, every lane waits).  The 16-byte alignment the
// bulk engine needs is met by copying from the aligned address below `src`
// into `raw` (>= n + 2 doubles); returns where element 0 landed.  Reads up to
// 8 bytes on either side of [src, src + n): the caller's allocation pads them.
__device__ __forceinline__ const double* stage_doubles_bulk(double* raw, const double* src, int n, uint64_t* bar) {
  const uintptr_t s0 = reinterpret_cast<uintptr_t>(src);
  const uintptr_t a0 = s0 & ~uintptr_t(15);
  const int shift = (int)((s0 - a0) / 8);
  const uint32_t bytes = (uint32_t)((((uint64_t)(n + shift) * 8) + 15) & ~uint64_t(15));
  if ((threadIdx.x & 31) == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bar, bytes);
    for (uint32_t off = 0; off < bytes; off += 32768u) {
      const uint32_t len = bytes - off < 32768u ? bytes - off : 32768u;
      bulk_g2s(reinterpret_cast<char*>(raw) + off, reinterpret_cast<const char*>(a0) + off, len, bar);
    }
  }
  __syncwarp();
  mbar_wait(bar, 0);
  return raw + shift;
}

}  // namespace sb
