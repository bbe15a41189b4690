// Multi-process plumbing over peer memory (one process per GPU, NVLink 5 /
// NVSwitch): CUDA IPC export/import of arenas, the metadata all-gather as
// peer stores (replaces gather_sequence_info, exchange.cpp:68-77, which in
// the reference is an in-process vector copy), and a device-side barrier on
// system-scope flags so exchange phases close without a host round trip.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

struct sb_gather {
  int W = 0, n_local = 0, first_local = 0, n_procs = 1;
  int64_t cap = 0;          // records per rank
  void* buf = nullptr;      // [W] counts (i64) + [W*cap] ids (u64) + [W*cap] lens (i64)
  int64_t bytes = 0;
  uint64_t* d_peers = nullptr;  // n_procs buffer bases (peer-mapped)
  int32_t* d_status = nullptr;
};

struct sb_barrier {
  int n_procs = 1, me = 0;
  uint64_t* flags = nullptr;    // [n_procs] epochs written by peers into this process
  uint64_t* d_peers = nullptr;  // n_procs flag bases (peer-mapped)
  uint64_t* d_state = nullptr;  // [0] epoch of the last barrier (device counter: graph-replayable)
                                // [1] status: 0 ok, else 1 + the first process that did not arrive
                                // [2] epoch at which the timeout fired
  uint64_t timeout_ns = 0;
};

namespace sb {

struct GatherArgs {
  int W, n_local, first_local, n_procs;
  int64_t cap;
  const uint64_t* peers;
  int32_t* status;
};

__device__ __forceinline__ int64_t* g_cnt(uint64_t base) { return reinterpret_cast<int64_t*>(base); }
__device__ __forceinline__ uint64_t* g_ids(uint64_t base, int W) {
  return reinterpret_cast<uint64_t*>(base + sizeof(int64_t) * W);
}
__device__ __forceinline__ int64_t* g_lens(uint64_t base, int W, int64_t cap) {
  return reinterpret_cast<int64_t*>(base + sizeof(int64_t) * W + sizeof(uint64_t) * W * cap);
}

// grid: (n_procs destination processes) x blocks; pushes this process's
// local ranks' records into slot [rank] of every destination buffer.  A rank
// with more records than the slot holds is pushed as a poison count (-1), so
// every process -- not only the sender -- sees the overflow in its compact.
__global__ void k_gather_push(GatherArgs a, const uint64_t* ids, const int64_t* lens, const int64_t* local_off) {
  const int dst = blockIdx.y;
  const uint64_t base = a.peers[dst];
  if (!base) return;  // unmapped peer: the collective transport all-gathers the slots instead
  for (int lr = 0; lr < a.n_local; ++lr) {
    const int r = a.first_local + lr;
    const int64_t lo = local_off[lr], n = local_off[lr + 1] - local_off[lr];
    if (n > a.cap || n < 0) {
      if (threadIdx.x == 0 && blockIdx.x == 0) g_cnt(base)[r] = -1;
      continue;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) g_cnt(base)[r] = n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      g_ids(base, a.W)[r * a.cap + i] = ids[lo + i];
      g_lens(base, a.W, a.cap)[r * a.cap + i] = lens[lo + i];
    }
  }
  __threadfence_system();
}

// After the barrier: compact slots into gather order (rank-major).
__global__ void k_gather_compact(GatherArgs a, uint64_t own, uint64_t* ids, int64_t* lens, int64_t* rank_off) {
  __shared__ int64_t off[1025];
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int r = 0; r < a.W; ++r) {
      off[r] = acc;
      const int64_t c = g_cnt(own)[r];
      if (c < 0 || c > a.cap) {  // poisoned by the sender: report, plan nothing from that rank
        atomicOr(a.status, ST_CAPACITY);
        continue;
      }
      acc += c;
    }
    off[a.W] = acc;
  }
  __syncthreads();
  for (int r = threadIdx.x; r <= a.W; r += blockDim.x) rank_off[r] = off[r];
  for (int r = 0; r < a.W; ++r) {
    const int64_t n = off[r + 1] - off[r];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      ids[off[r] + i] = g_ids(own, a.W)[r * a.cap + i];
      lens[off[r] + i] = g_lens(own, a.W, a.cap)[r * a.cap + i];
    }
  }
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// One block, n_procs threads: thread q publishes our epoch into process q's
// flag array (system-scope release), then waits until every process has
// published the epoch into ours (system-scope acquire).  The epoch lives on
// the device (state[0]) so a captured graph replays correctly.  The wait is
// bounded: after timeout_ns without process q arriving the barrier records
// status 1+q and returns, and sb_barrier_status reports SB_ERR_COMM (a dead
// or stalled peer no longer hangs every rank).  Once the status is set,
// later barriers return at once (the epoch sequence is broken).
__global__ void k_barrier(const uint64_t* peers, uint64_t* own_flags, uint64_t* state, int n_procs, int me,
                          uint64_t timeout_ns) {
  __shared__ uint64_t s_epoch;
  const int q = threadIdx.x;
  if (q == 0) s_epoch = state[0] + 1;
  __syncthreads();
  const uint64_t epoch = s_epoch;
  const bool failed = *reinterpret_cast<volatile uint64_t*>(&state[1]) != 0;
  if (q < n_procs && !failed) {
    __threadfence_system();
    uint64_t* flag = reinterpret_cast<uint64_t*>(peers[q]) + me;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(epoch) : "memory");
    uint64_t v = 0;
    const uint64_t t0 = globaltimer_ns();
    uint32_t spins = 0;
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(own_flags + q) : "memory");
      if (v >= epoch) break;
      if ((++spins & 255) == 0) {
        if (globaltimer_ns() - t0 > timeout_ns) {
          atomicCAS(reinterpret_cast<unsigned long long*>(&state[1]), 0ull, (unsigned long long)(1 + q));
          state[2] = epoch;
          break;
        }
        __nanosleep(64);
      }
    }
  }
  __syncthreads();
  if (q == 0) state[0] = epoch;
  __threadfence_system();
}

}  // namespace sb

using sb::Error;

#define SB_API_BEGIN try {
#define SB_API_END                              \
  return SB_OK;                                 \
  }                                             \
  catch (const Error& e) {                      \
    sb::set_error(e.msg);                       \
    return e.code;                              \
  }                                             \
  catch (const std::bad_alloc&) {               \
    sb::set_error("host allocation failed");    \
    return SB_ERR_CAPACITY;                     \
  }

extern "C" sb_status sb_ipc_export(const void* dptr, void* handle) {
  SB_API_BEGIN
  if (!dptr || !handle) throw Error{SB_ERR_CONFIG, "sb_ipc_export: null argument"};
  cudaIpcMemHandle_t h;
  SB_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
  static_assert(sizeof(h) == SB_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof h);
  SB_API_END
}

extern "C" sb_status sb_ipc_import(const void* handle, void** dptr) {
  SB_API_BEGIN
  if (!dptr || !handle) throw Error{SB_ERR_CONFIG, "sb_ipc_import: null argument"};
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  cudaError_t e = cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error{SB_ERR_COMM, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e)};
  }
  SB_API_END
}

extern "C" sb_status sb_ipc_close(void* dptr) {
  SB_API_BEGIN
  if (dptr) SB_CUDA(cudaIpcCloseMemHandle(dptr));
  SB_API_END
}

extern "C" sb_status sb_gather_create(int world_size, int n_local, int first_local, int64_t cap_per_rank,
                                      sb_gather** out) {
  SB_API_BEGIN
  if (!out || world_size < 1 || n_local < 1 || world_size % n_local || first_local % n_local ||
      first_local + n_local > world_size || cap_per_rank < 1 || world_size > 1024)
    throw Error{SB_ERR_CONFIG, "sb_gather_create: bad arguments"};
  auto* g = new sb_gather();
  g->W = world_size;
  g->n_local = n_local;
  g->first_local = first_local;
  g->n_procs = world_size / n_local;
  g->cap = cap_per_rank;
  g->bytes = (int64_t)sizeof(int64_t) * world_size + (int64_t)(sizeof(uint64_t) + sizeof(int64_t)) * world_size * cap_per_rank;
  try {
    SB_CUDA(cudaMalloc(&g->buf, (size_t)g->bytes));
    SB_CUDA(cudaMemset(g->buf, 0, (size_t)g->bytes));
    SB_CUDA(cudaMalloc(&g->d_peers, sizeof(uint64_t) * g->n_procs));
    SB_CUDA(cudaMalloc(&g->d_status, sizeof(int32_t)));
    SB_CUDA(cudaMemset(g->d_status, 0, sizeof(int32_t)));
    std::vector<uint64_t> p(g->n_procs, 0);
    p[first_local / n_local] = (uint64_t)g->buf;
    SB_CUDA(cudaMemcpy(g->d_peers, p.data(), sizeof(uint64_t) * p.size(), cudaMemcpyHostToDevice));
  } catch (...) {
    if (g->buf) cudaFree(g->buf);
    delete g;
    throw;
  }
  *out = g;
  SB_API_END
}

extern "C" sb_status sb_gather_destroy(sb_gather* g) {
  SB_API_BEGIN
  if (g) {
    cudaFree(g->buf);
    cudaFree(g->d_peers);
    cudaFree(g->d_status);
    delete g;
  }
  SB_API_END
}

extern "C" sb_status sb_gather_buffer(const sb_gather* g, void** buf, int64_t* bytes) {
  SB_API_BEGIN
  if (!g) throw Error{SB_ERR_CONFIG, "null gather"};
  if (buf) *buf = g->buf;
  if (bytes) *bytes = g->bytes;
  SB_API_END
}

extern "C" sb_status sb_gather_set_peers(sb_gather* g, const uint64_t* bases, int n_procs) {
  SB_API_BEGIN
  if (!g || !bases || n_procs != g->n_procs) throw Error{SB_ERR_CONFIG, "sb_gather_set_peers: bad arguments"};
  SB_CUDA(cudaMemcpy(g->d_peers, bases, sizeof(uint64_t) * n_procs, cudaMemcpyHostToDevice));
  SB_API_END
}

extern "C" sb_status sb_gather_push(sb_gather* g, const uint64_t* d_ids, const int64_t* d_lens,
                                    const int64_t* d_local_off, sb_stream stream) {
  SB_API_BEGIN
  if (!g || !d_ids || !d_lens || !d_local_off) throw Error{SB_ERR_CONFIG, "sb_gather_push: null argument"};
  sb::GatherArgs a{g->W, g->n_local, g->first_local, g->n_procs, g->cap, g->d_peers, g->d_status};
  // the status describes the latest gather (sb_gather_status after compact)
  SB_CUDA(cudaMemsetAsync(g->d_status, 0, sizeof(int32_t), (cudaStream_t)stream));
  sb::k_gather_push<<<dim3(4, g->n_procs), 256, 0, (cudaStream_t)stream>>>(a, d_ids, d_lens, d_local_off);
  SB_CHECK_LAUNCH();
  sb::count_launch();
  SB_API_END
}

extern "C" sb_status sb_gather_compact(sb_gather* g, uint64_t* d_ids, int64_t* d_lens, int64_t* d_rank_off,
                                       sb_stream stream) {
  SB_API_BEGIN
  if (!g || !d_ids || !d_lens || !d_rank_off) throw Error{SB_ERR_CONFIG, "sb_gather_compact: null argument"};
  sb::GatherArgs a{g->W, g->n_local, g->first_local, g->n_procs, g->cap, g->d_peers, g->d_status};
  sb::k_gather_compact<<<1, 1024, 0, (cudaStream_t)stream>>>(a, (uint64_t)g->buf, d_ids, d_lens, d_rank_off);
  SB_CHECK_LAUNCH();
  sb::count_launch();
  SB_API_END
}

extern "C" sb_status sb_gather_status(sb_gather* g, sb_stream stream) {
  SB_API_BEGIN
  if (!g) throw Error{SB_ERR_CONFIG, "null gather"};
  SB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  int32_t st = 0;
  SB_CUDA(cudaMemcpy(&st, g->d_status, sizeof st, cudaMemcpyDeviceToHost));
  if (st) throw Error{SB_ERR_CAPACITY, "metadata all-gather: more sequences on a rank than cap_per_rank "
                                     "(reported by every process; that rank's sequences were not planned)"};
  SB_API_END
}

extern "C" sb_status sb_barrier_create(int n_procs, int me, sb_barrier** out) {
  SB_API_BEGIN
  if (!out || n_procs < 1 || me < 0 || me >= n_procs || n_procs > 1024)
    throw Error{SB_ERR_CONFIG, "sb_barrier_create: bad arguments"};
  auto* b = new sb_barrier();
  b->n_procs = n_procs;
  b->me = me;
  try {
    SB_CUDA(cudaMalloc(&b->flags, sizeof(uint64_t) * n_procs));
    SB_CUDA(cudaMemset(b->flags, 0, sizeof(uint64_t) * n_procs));
    SB_CUDA(cudaMalloc(&b->d_peers, sizeof(uint64_t) * n_procs));
    SB_CUDA(cudaMalloc(&b->d_state, sizeof(uint64_t) * 4));
    SB_CUDA(cudaMemset(b->d_state, 0, sizeof(uint64_t) * 4));
    const char* tv = getenv("SEQBAL_BARRIER_TIMEOUT_MS");
    b->timeout_ns = (uint64_t)(tv ? std::max(1.0, atof(tv)) : 60000.0) * 1000000ull;
    std::vector<uint64_t> p(n_procs, 0);
    p[me] = (uint64_t)b->flags;
    SB_CUDA(cudaMemcpy(b->d_peers, p.data(), sizeof(uint64_t) * n_procs, cudaMemcpyHostToDevice));
  } catch (...) {
    delete b;
    throw;
  }
  *out = b;
  SB_API_END
}

extern "C" sb_status sb_barrier_destroy(sb_barrier* b) {
  SB_API_BEGIN
  if (b) {
    cudaFree(b->flags);
    cudaFree(b->d_peers);
    cudaFree(b->d_state);
    delete b;
  }
  SB_API_END
}

extern "C" sb_status sb_barrier_buffer(const sb_barrier* b, void** buf, int64_t* bytes) {
  SB_API_BEGIN
  if (!b) throw Error{SB_ERR_CONFIG, "null barrier"};
  if (buf) *buf = b->flags;
  if (bytes) *bytes = (int64_t)sizeof(uint64_t) * b->n_procs;
  SB_API_END
}

extern "C" sb_status sb_barrier_set_peers(sb_barrier* b, const uint64_t* bases, int n_procs) {
  SB_API_BEGIN
  if (!b || !bases || n_procs != b->n_procs) throw Error{SB_ERR_CONFIG, "sb_barrier_set_peers: bad arguments"};
  SB_CUDA(cudaMemcpy(b->d_peers, bases, sizeof(uint64_t) * n_procs, cudaMemcpyHostToDevice));
  SB_API_END
}

extern "C" sb_status sb_barrier_wait(sb_barrier* b, sb_stream stream) {
  SB_API_BEGIN
  if (!b) throw Error{SB_ERR_CONFIG, "null barrier"};
  sb::k_barrier<<<1, 32 * ((b->n_procs + 31) / 32), 0, (cudaStream_t)stream>>>(b->d_peers, b->flags, b->d_state,
                                                                               b->n_procs, b->me, b->timeout_ns);
  SB_CHECK_LAUNCH();
  sb::count_launch();
  SB_API_END
}

extern "C" sb_status sb_barrier_set_timeout(sb_barrier* b, double timeout_ms) {
  SB_API_BEGIN
  if (!b || !(timeout_ms > 0)) throw Error{SB_ERR_CONFIG, "sb_barrier_set_timeout: bad arguments"};
  b->timeout_ns = (uint64_t)(timeout_ms * 1e6);
  SB_API_END
}

extern "C" sb_status sb_barrier_status(sb_barrier* b, uint64_t* epoch, sb_stream stream) {
  SB_API_BEGIN
  if (!b) throw Error{SB_ERR_CONFIG, "null barrier"};
  SB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  uint64_t st[4] = {0, 0, 0, 0};
  SB_CUDA(cudaMemcpy(st, b->d_state, sizeof st, cudaMemcpyDeviceToHost));
  if (epoch) *epoch = st[0];
  if (st[1])
    throw Error{SB_ERR_COMM, "peer barrier timed out: process " + std::to_string(st[1] - 1) +
                                 " did not arrive at barrier epoch " + std::to_string(st[2]) + " (process " +
                                 std::to_string(b->me) + " of " + std::to_string(b->n_procs) + ")"};
  SB_API_END
}
