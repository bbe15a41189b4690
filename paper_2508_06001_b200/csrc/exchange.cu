// Exchange engine: device worlds, plan -> copy-job builders for route /
// reverse_route / pre_attn / post_attn, and the batched strided copy kernel
// that moves the rows (the pack, the all-to-all and the unpack fused into one
// pass: each row is read once from its source buffer and written once into
// its final slot, local or peer-mapped).
//
// Reference data movement being replaced: exchange.cpp:127-198 (route),
// :255-436 (pre_attn / post_attn), exchange_kernels.cpp:15-56 (the
// OpenMP memcpy of BlockMoves).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "common.cuh"
#include "tma.cuh"
#include "internal.hpp"

namespace sb {

thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch(int n) { g_launches += n; }

constexpr int64_t kPieceBytes = 32768;  // work unit of the copy kernel
constexpr int kCopyThreads = 256;

// --------------------------------------------------------------- layouts
struct WorldArgs {
  int W, T, n_local, first_local, n_procs;
  uint64_t* base;     // T*W
  int64_t* pitch;     // T*W
  int64_t* rows;      // W
  int32_t* headcol;   // W
  const uint64_t* peer_arena;  // T*n_procs
  const int64_t* arena_bytes;  // T
  int32_t* status;
};

static WorldArgs wargs(sb_world* w) {
  WorldArgs a;
  a.W = w->W; a.T = w->T; a.n_local = w->n_local; a.first_local = w->first_local; a.n_procs = w->n_procs;
  a.base = w->d_base; a.pitch = w->d_pitch; a.rows = w->d_rows; a.headcol = w->d_headcol;
  a.peer_arena = w->d_peer_arena; a.arena_bytes = w->d_arena_bytes; a.status = w->d_status;
  return a;
}

struct TensorInfo {
  int64_t row_bytes[16];
  int kind[16];  // 0 meta, 1 payload (head-sliced), 2 aux
};

static TensorInfo tinfo(sb_world* w) {
  TensorInfo t;
  for (int i = 0; i < w->T && i < 16; ++i) {
    t.row_bytes[i] = w->row_bytes[i];
    t.kind[i] = (int)w->tensor_desc[i];
  }
  return t;
}

// Packs ranks back to back per owner process.  mode 0: every rank gets
// rows_src[r] full-width rows (route / reverse_route / origin).  mode 1:
// ranks of multi-GPU bags get the Ulysses (full sequence, H/G heads) layout,
// others alias `src`.  mode 2: ranks of multi-GPU bags get the chunk layout
// again (post_attn), others alias `src`.
struct LayoutPlan {
  const int64_t* rows_src;  // mode 0: rows per rank
  const int64_t* expect_rows;  // mode 0: rows the SOURCE must hold per rank (origin / target layout)
  const int32_t* rank_bag;  // U
  const int32_t* rank_member;
  const int32_t* bag_size;
  const int64_t* bag_rows;  // R*M
  const int64_t* target_rows;
  int U, M;
  int no_check;  // standalone layout (sb_world_layout_plan): no source to validate
};

// check_world_matches_layout (exchange.cpp:96-123) / check_bag_chunk_layout
// (:210-251) restated on row counts: every local source rank must hold the
// rows the plan expects for this exchange -- origin (route), target
// (reverse_route, pre_attn) or the Ulysses full-sequence rows (post_attn on
// multi-GPU bags).  A mismatch raises ST_MISMATCH on the destination and the
// job builders then emit empty jobs, so a stale or foreign world is reported
// as IntegrityError by sb_world_status instead of being read out of bounds.
__device__ __forceinline__ bool rank_matches_plan(const WorldArgs& s, const LayoutPlan& lp, int mode, int r) {
  int64_t want;
  if (mode == 0) {
    want = lp.expect_rows[r];
  } else {
    const int u = r % lp.U, rep = r / lp.U;
    const int b = lp.rank_bag[u];
    want = (mode == 2 && lp.bag_size[b] > 1) ? lp.bag_rows[rep * lp.M + b] : lp.target_rows[r];
  }
  return s.rows[r] == want;
}

// Layout of tensor t, computed by ONE WARP (lane = rank, 32 ranks at a time):
// rows and pitch per rank by mode, then each rank's byte offset inside its
// owner process's arena by a segmented exclusive scan (owners hold
// contiguous blocks of n_local ranks; a segment restarts at every owner's
// first rank).  Aliased ranks (one-GPU bags under pre/post_attn) take the
// source's tables and no arena bytes.  All per-rank loads are independent
// across lanes, so the layout costs a few memory round trips instead of a
// dependent chain over the world's ranks.
__device__ void layout_tensor(const WorldArgs& d, const WorldArgs& s, const LayoutPlan& lp, const TensorInfo& ti,
                              int mode, int t) {
  if (t >= d.T) return;
  const int lane = threadIdx.x & 31;
  if (t == 0 && !lp.no_check) {  // the status reflects the latest exchange into d
    bool bad = false;
    for (int r = s.first_local + lane; r < s.first_local + s.n_local; r += 32) bad |= !rank_matches_plan(s, lp, mode, r);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      if (bad) atomicOr(d.status, ST_MISMATCH);
      else atomicAnd(d.status, ~ST_MISMATCH);
    }
  }
  int64_t carry = 0;
  bool overflow = false;
  for (int r0 = 0; r0 < d.W; r0 += 32) {
    const int r = r0 + lane;
    const bool valid = r < d.W;
    int64_t rows = 0, pitch = ti.row_bytes[t];
    int32_t headcol = 0;
    bool alias = false;
    if (valid) {
      if (mode == 0) {
        rows = lp.rows_src[r];
      } else {
        const int u = r % lp.U, rep = r / lp.U;
        const int b = lp.rank_bag[u];
        const int g = lp.bag_size[b];
        if (g == 1 && mode == 3) {  // standalone Ulysses layout: one-GPU bags keep their chunk rows
          rows = lp.target_rows[r];
        } else if (g == 1) {  // alias the source world's buffers (pre/post are no-ops)
          alias = true;
        } else {
          const bool sliced = mode == 1 || mode == 3;
          rows = sliced ? lp.bag_rows[rep * lp.M + b] : lp.target_rows[r];
          if (sliced && ti.kind[t] == 1) pitch = ti.row_bytes[t] / g;
          if (sliced) headcol = (int32_t)(lp.rank_member[u] * (ti.row_bytes[1] / 8 / g));
        }
      }
    }
    const int64_t bytes = valid && !alias ? rows * pitch : 0;
    bool f = valid && r % d.n_local == 0;  // segment head: first rank of an owner
    int64_t x = bytes;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {  // segmented inclusive scan
      const int64_t nx = __shfl_up_sync(0xffffffffu, x, o);
      const bool nf = __shfl_up_sync(0xffffffffu, f, o);
      if (lane >= o && !f) {
        x += nx;
        f = nf;
      }
    }
    const int64_t incl = f ? x : x + carry;
    if (valid) {
      if (alias) {
        d.base[t * d.W + r] = s.base[t * s.W + r];
        d.pitch[t * d.W + r] = s.pitch[t * s.W + r];
        if (t == 0) {
          d.rows[r] = s.rows[r];
          d.headcol[r] = s.headcol[r];
        }
      } else {
        const int owner = r / d.n_local;
        d.base[t * d.W + r] = d.peer_arena[t * d.n_procs + owner] + (uint64_t)(incl - bytes);
        d.pitch[t * d.W + r] = pitch;
        overflow |= incl > d.arena_bytes[t];
        if (t == 0) {
          d.rows[r] = rows;
          d.headcol[r] = headcol;
        }
      }
    }
    carry = __shfl_sync(0xffffffffu, incl, 31);
  }
  if (__any_sync(0xffffffffu, overflow) && lane == 0) atomicOr(d.status, ST_LAYOUT);
}

__global__ void k_layout(WorldArgs d, WorldArgs s, LayoutPlan lp, TensorInfo ti, int mode) {
  layout_tensor(d, s, lp, ti, mode, threadIdx.x >> 5);  // one warp per tensor
}

// ----------------------------------------------------------- job builders
struct JobArgs {
  const int64_t* n_chunks;
  const int32_t *c_idx, *c_src, *c_dst, *bag_of_rank, *bag_size;
  const int64_t *c_start, *c_end, *c_src_row, *c_dst_row, *c_seq_base;
  int U;
  int max_bag;
  SbJob* jobs;
  int64_t* n_jobs;
  int32_t* owner;  // collective transport: every chunk's jobs, owner[x] = src proc << 16 | dst proc (-1: none)
};

__device__ __forceinline__ bool is_local(const WorldArgs& w, int r) {
  return r >= w.first_local && r < w.first_local + w.n_local;
}

__device__ __forceinline__ void route_job(const JobArgs& j, const WorldArgs& s, const WorldArgs& d,
                                          const TensorInfo& ti, int reverse, int64_t x) {
  const int T = s.T;
  {
    const int64_t c = x / T;
    const int t = (int)(x % T);
    const int sr = reverse ? j.c_dst[c] : j.c_src[c];
    const int dr = reverse ? j.c_src[c] : j.c_dst[c];
    const int64_t srow = reverse ? j.c_dst_row[c] : j.c_src_row[c];
    const int64_t drow = reverse ? j.c_src_row[c] : j.c_dst_row[c];
    SbJob job;
    const int64_t sp = s.pitch[t * s.W + sr], dp = d.pitch[t * d.W + dr];
    job.src = s.base[t * s.W + sr] + (uint64_t)(srow * sp);
    job.dst = d.base[t * d.W + dr] + (uint64_t)(drow * dp);
    const bool coll = j.owner != nullptr;
    job.n_rows = (coll || (is_local(s, sr) && !(*d.status & ST_MISMATCH))) ? j.c_end[c] - j.c_start[c] : 0;
    job.width = ti.row_bytes[t];
    job.spitch = sp;
    job.dpitch = dp;
    j.jobs[x] = job;
    if (coll) j.owner[x] = ((sr / s.n_local) << 16) | (dr / d.n_local);
  }
}

__global__ void k_jobs_route(JobArgs j, WorldArgs s, WorldArgs d, TensorInfo ti, int reverse) {
  const int64_t n = *j.n_chunks * s.T;
  if (blockIdx.x == 0 && threadIdx.x == 0) *j.n_jobs = n;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
    route_job(j, s, d, ti, reverse, x);
}

// pre_attn (exchange.cpp:298-325): chunk c = (seq q, member m) held by bag
// rank m moves, for each destination member d, its column slice d (payload)
// or its whole rows (metadata / aux) to row seq_base(q) + start on rank d.
// post_attn (exchange.cpp:406-431) is the transpose: destination chunk
// c = (q, d) gathers slice m from every member m; metadata from m = 0 only.
__device__ __forceinline__ void ulysses_job(const JobArgs& j, const WorldArgs& s, const WorldArgs& d,
                                            const TensorInfo& ti, int post, int64_t x) {
  const int T = s.T, G = j.max_bag;
  {
    const int t = (int)(x % T);
    const int64_t y = x / T;
    const int other = (int)(y % G);  // d for pre, m for post
    const int64_t c = y / G;
    SbJob job;
    job.src = job.dst = 0;
    job.n_rows = 0;
    job.width = 16;
    job.spitch = job.dpitch = 16;
    const bool coll = j.owner != nullptr;
    int32_t own = -1;
    const int dst_rank_of_chunk = j.c_dst[c];
    const int g = j.bag_size[j.bag_of_rank[dst_rank_of_chunk % j.U]];
    const int mine = j.c_idx[c];
    if (g > 1 && other < g) {
      const int64_t cq0 = c - mine;
      const int64_t full_row = j.c_seq_base[cq0] + j.c_start[c];
      const int64_t n = j.c_end[c] - j.c_start[c];
      const int kind = ti.kind[t];
      const int64_t slice = ti.row_bytes[t] / g;
      int sr, dr;
      int64_t srow, drow, scol = 0, dcol = 0, width;
      bool active = true;
      if (!post) {
        sr = dst_rank_of_chunk;               // member m = mine holds chunk c
        dr = j.c_dst[cq0 + other];            // member d
        srow = j.c_dst_row[c];
        drow = full_row;
        if (kind == 1) {
          scol = other * slice;
          width = slice;
        } else {
          width = ti.row_bytes[t];
        }
      } else {
        sr = j.c_dst[cq0 + other];            // member m holds slice m of the full seq
        dr = dst_rank_of_chunk;               // member d = mine gets chunk c back
        srow = full_row;
        drow = j.c_dst_row[c];
        if (kind == 1) {
          dcol = other * slice;
          width = slice;
        } else {
          width = ti.row_bytes[t];
          active = other == 0;  // metadata once per destination row (exchange.cpp:424)
        }
      }
      if (active && (coll || (is_local(s, sr) && !(*d.status & ST_MISMATCH)))) {
        own = ((sr / s.n_local) << 16) | (dr / d.n_local);
        const int64_t sp = s.pitch[t * s.W + sr], dp = d.pitch[t * d.W + dr];
        job.src = s.base[t * s.W + sr] + (uint64_t)(srow * sp + scol);
        job.dst = d.base[t * d.W + dr] + (uint64_t)(drow * dp + dcol);
        job.n_rows = n;
        job.width = width;
        job.spitch = sp;
        job.dpitch = dp;
      }
    }
    j.jobs[x] = job;
    if (coll) j.owner[x] = own;
  }
}

__global__ void k_jobs_ulysses(JobArgs j, WorldArgs s, WorldArgs d, TensorInfo ti, int post) {
  const int64_t total = *j.n_chunks * j.max_bag * s.T;
  if (blockIdx.x == 0 && threadIdx.x == 0) *j.n_jobs = total;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x)
    ulysses_job(j, s, d, ti, post, x);
}

// Piece decomposition + exclusive scan (single CTA).  A job whose rows are
// contiguous on both sides is split into kPieceBytes spans of the flat byte
// range; otherwise into groups of kPieceBytes/width rows.
__device__ __forceinline__ bool job_flat(const SbJob& j) { return j.width == j.spitch && j.width == j.dpitch; }
__device__ __forceinline__ int64_t job_rows_per_piece(const SbJob& j) {
  const int64_t r = kPieceBytes / (j.width > 0 ? j.width : 1);
  return r > 0 ? r : 1;
}
__device__ __forceinline__ int64_t job_pieces(const SbJob& j) {
  if (j.n_rows <= 0 || j.width <= 0) return 0;
  if (job_flat(j)) return (j.n_rows * j.width + kPieceBytes - 1) / kPieceBytes;
  const int64_t rp = job_rows_per_piece(j);
  return (j.n_rows + rp - 1) / rp;
}

__device__ void pieces_body(const SbJob* jobs, const int64_t* n_jobs_p, int64_t* piece_off, int64_t* bytes_moved) {
  __shared__ int64_t sh[33];
  const int64_t n = *n_jobs_p;
  const int nt = blockDim.x, tid = threadIdx.x;
  const int64_t per = (n + nt - 1) / nt;
  const int64_t b = tid * per, e = b + per < n ? b + per : n;
  int64_t cnt = 0, bytes = 0;
  for (int64_t i = b; i < e; ++i) {
    const SbJob jb = jobs[i];
    cnt += job_pieces(jb);
    if (jb.n_rows > 0) bytes += jb.n_rows * jb.width;
  }
  int64_t tot, tb;
  const int64_t ex = block_excl_scan<int64_t>(cnt, sh, &tot);
  block_excl_scan<int64_t>(bytes, sh, &tb);
  int64_t run = ex;
  for (int64_t i = b; i < e; ++i) {
    piece_off[i] = run;
    run += job_pieces(jobs[i]);
  }
  if (tid == 0) {
    piece_off[n] = tot;
    *bytes_moved = tb;
  }
}

__global__ void __launch_bounds__(1024) k_pieces(const SbJob* jobs, const int64_t* n_jobs_p, int64_t* piece_off,
                                                 int64_t* bytes_moved) {
  pieces_body(jobs, n_jobs_p, piece_off, bytes_moved);
}

// Fused exchange preparation for plans of modest size: destination layout,
// copy jobs and the piece scan in ONE CTA (three launches become one; the
// phases hand over through global memory inside the block).  op: 0 route,
// 1 reverse_route, 2 pre_attn, 3 post_attn.
__global__ void __launch_bounds__(1024) k_exchange_prep(JobArgs j, WorldArgs s, WorldArgs d, TensorInfo ti,
                                                        LayoutPlan lp, int op, int64_t* piece_off,
                                                        int64_t* bytes_moved) {
  const int mode = op < 2 ? 0 : (op == 2 ? 1 : 2);
  layout_tensor(d, s, lp, ti, mode, threadIdx.x >> 5);
  __syncthreads();
  const int64_t n = op < 2 ? *j.n_chunks * s.T : *j.n_chunks * j.max_bag * s.T;
  if (threadIdx.x == 0) *j.n_jobs = n;
  for (int64_t x = threadIdx.x; x < n; x += blockDim.x) {
    if (op < 2) route_job(j, s, d, ti, op, x);
    else ulysses_job(j, s, d, ti, op == 3, x);
  }
  __syncthreads();
  pieces_body(j.jobs, j.n_jobs, piece_off, bytes_moved);
}

// ------------------------------------------- collective transport split
// The NCCL baseline transport (sb_exchange_pack / sb_exchange_unpack): no
// peer mappings.  Every process builds the FULL job list of the exchange
// (all processes hold the same plan, so the lists are identical) and splits
// it: a job whose source rank is local and destination remote is packed, in
// job order, into the destination process's contiguous segment of a send
// buffer; a job whose destination is local and source remote is unpacked
// from the source process's segment of the receive buffer.  Sender and
// receiver walk the same list in the same order, so every byte offset is
// known on both sides without exchanging any layout.  Local-to-local jobs
// copy directly in the pack pass.  Between the two passes the caller runs one
// all-to-all-v (grouped ncclSend/ncclRecv) with the byte counts written to
// counts[0, P) (sent to each process) and counts[P, 2P) (received).
constexpr int kMaxCollProcs = 16;

__global__ void __launch_bounds__(1024) k_collective_split(SbJob* jobs, const int32_t* owner, const int64_t* n_jobs_p,
                                                           int me, int P, uint64_t send, int64_t send_cap,
                                                           uint64_t recv, int64_t recv_cap, int32_t* status,
                                                           int64_t* piece_off, int64_t* bytes_moved, SbJob* ujobs,
                                                           int64_t* u_n_jobs, int64_t* u_piece_off, int64_t* counts) {
  __shared__ int64_t sh[33];
  __shared__ int64_t s_tot[2 * kMaxCollProcs];
  const int64_t n = *n_jobs_p;
  const int nt = blockDim.x, tid = threadIdx.x;
  const int64_t per = (n + nt - 1) / nt;
  const int64_t b = tid * per, e = b + per < n ? b + per : n;
  int64_t cs[kMaxCollProcs], cr[kMaxCollProcs];
  for (int q = 0; q < kMaxCollProcs; ++q) cs[q] = cr[q] = 0;
  for (int64_t i = b; i < e; ++i) {
    const int32_t o = owner[i];
    const SbJob jb = jobs[i];
    if (o < 0 || jb.n_rows <= 0) continue;
    const int so = o >> 16, dd = o & 0xffff;
    const int64_t nb = jb.n_rows * jb.width;
    if (so == me && dd != me) cs[dd] += nb;
    else if (dd == me && so != me) cr[so] += nb;
  }
  for (int q = 0; q < P; ++q) {
    int64_t tot;
    cs[q] = block_excl_scan<int64_t>(cs[q], sh, &tot);
    if (tid == 0) s_tot[q] = tot;
    cr[q] = block_excl_scan<int64_t>(cr[q], sh, &tot);
    if (tid == 0) s_tot[kMaxCollProcs + q] = tot;
  }
  __syncthreads();
  int64_t sd[kMaxCollProcs], rd[kMaxCollProcs], st = 0, rt = 0;
  for (int q = 0; q < P; ++q) {
    sd[q] = st;
    rd[q] = rt;
    st += s_tot[q];
    rt += s_tot[kMaxCollProcs + q];
  }
  const bool fits = st <= send_cap && rt <= recv_cap;
  const bool copy = fits && !(*status & ST_MISMATCH);
  if (tid == 0 && !fits) atomicOr(status, ST_CAPACITY);
  for (int64_t i = b; i < e; ++i) {
    const int32_t o = owner[i];
    SbJob pk = jobs[i], up;
    up.src = up.dst = 0;
    up.n_rows = 0;
    up.width = up.spitch = up.dpitch = 16;
    if (o < 0 || pk.n_rows <= 0) {
      pk.n_rows = 0;
    } else {
      const int so = o >> 16, dd = o & 0xffff;
      const int64_t nb = pk.n_rows * pk.width;
      if (so == me) {
        if (dd != me) {
          pk.dst = send + (uint64_t)(sd[dd] + cs[dd]);
          pk.dpitch = pk.width;
          cs[dd] += nb;
        }
      } else {
        if (dd == me) {
          up = pk;
          up.src = recv + (uint64_t)(rd[so] + cr[so]);
          up.spitch = up.width;
          cr[so] += nb;
        }
        pk.n_rows = 0;
      }
    }
    if (!copy) pk.n_rows = up.n_rows = 0;
    jobs[i] = pk;
    ujobs[i] = up;
  }
  if (tid == 0) {
    *u_n_jobs = n;
    for (int q = 0; q < P; ++q) {
      counts[q] = s_tot[q];
      counts[P + q] = s_tot[kMaxCollProcs + q];
    }
  }
  __syncthreads();
  pieces_body(jobs, n_jobs_p, piece_off, bytes_moved);
  __syncthreads();
  pieces_body(ujobs, u_n_jobs, u_piece_off, u_n_jobs + 1);
}

// ------------------------------------------------------------ copy kernel
// Cache-policy variants of the 128-bit streaming load/store (HINT):
//  0: ld.global.nc.L1::no_allocate.L2::256B / st.global.L1::no_allocate
//  1: ld.global.nc.L1::no_allocate          / st.global.L1::no_allocate
//  2: ld.global.cs (evict-first)            / st.global.cs
//  3: as 0, stores with an L2 evict_first policy
//  4: loads with an L2 evict_first policy, stores as 0
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <int HINT>
__device__ __forceinline__ int4 ld_stream(const void* p) {
  int4 r;
  if (HINT == 4)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(l2_evict_first()));
  else if (HINT == 0 || HINT == 3)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  else if (HINT == 1)
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  else
    asm volatile("ld.global.cs.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
template <int HINT>
__device__ __forceinline__ void st_stream(void* p, const int4& v) {
  if (HINT == 2)
    asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  else if (HINT == 3)
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w), "l"(l2_evict_first())
                 : "memory");
  else
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

constexpr int kUnroll = 8;

// Warp copies `len` contiguous bytes (16-B aligned) with kUnroll 128-bit
// loads in flight per lane before the matching stores.
template <int HINT>
__device__ __forceinline__ void warp_copy_flat(const char* src, char* dst, int64_t len, int lane) {
  const int64_t step = 32 * 16 * kUnroll;
  int64_t off = (int64_t)lane * 16;
  for (; off + (kUnroll - 1) * 512 < len; off += step) {
    int4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream<HINT>(src + off + u * 512);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) st_stream<HINT>(dst + off + u * 512, v[u]);
  }
  int4 v[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u)
    if (off + u * 512 < len) v[u] = ld_stream<HINT>(src + off + u * 512);
#pragma unroll
  for (int u = 0; u < kUnroll; ++u)
    if (off + u * 512 < len) st_stream<HINT>(dst + off + u * 512, v[u]);
}

// Warp copies rows [r0, r1) of a strided job: flat index over (row, vec).
template <int HINT>
__device__ __forceinline__ void warp_copy_rows(const SbJob& j, int64_t r0, int64_t r1, int lane) {
  const int vpr = (int)(j.width >> 4);
  const int total = (int)(r1 - r0) * vpr;
  const float inv = 1.0f / (float)vpr;
  const char* src = reinterpret_cast<const char*>(j.src) + r0 * j.spitch;
  char* dst = reinterpret_cast<char*>(j.dst) + r0 * j.dpitch;
  for (int base = 0; base < total; base += 32 * kUnroll) {
    int4 v[kUnroll];
    int rr[kUnroll], cc[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int f = base + u * 32 + lane;
      int row = (int)((float)f * inv);
      if (row * vpr > f) --row;
      else if ((row + 1) * vpr <= f) ++row;
      rr[u] = row;
      cc[u] = f - row * vpr;
      if (f < total) v[u] = ld_stream<HINT>(src + rr[u] * j.spitch + cc[u] * 16);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int f = base + u * 32 + lane;
      if (f < total) st_stream<HINT>(dst + rr[u] * j.dpitch + cc[u] * 16, v[u]);
    }
  }
}

// Unaligned fallback (never hit by the bench layouts; kept for generality).
__device__ void warp_copy_bytes(const SbJob& j, int64_t r0, int64_t r1, int lane) {
  for (int64_t r = r0; r < r1; ++r) {
    const char* s = reinterpret_cast<const char*>(j.src) + r * j.spitch;
    char* d = reinterpret_cast<char*>(j.dst) + r * j.dpitch;
    for (int64_t b = lane; b < j.width; b += 32) d[b] = s[b];
  }
}

template <int MINB, int HINT = 0>
__global__ void __launch_bounds__(kCopyThreads, MINB) k_copy(const SbJob* __restrict__ jobs,
                                                       const int64_t* __restrict__ piece_off,
                                                       const int64_t* __restrict__ n_jobs_p, int fence_sys) {
  const int64_t n_jobs = *n_jobs_p;
  const int64_t total = piece_off[n_jobs];
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (kCopyThreads / 32);
  const int64_t wid = (int64_t)blockIdx.x * (kCopyThreads / 32) + (threadIdx.x >> 5);
  // contiguous block of pieces per warp: one job search, then walk
  const int64_t g0 = total * wid / nwarps, g1 = total * (wid + 1) / nwarps;
  if (g0 >= g1) return;
  int64_t lo = 0, hi = n_jobs;  // find last job with piece_off[j] <= g0
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (piece_off[mid] <= g0) lo = mid;
    else hi = mid;
  }
  int64_t jb = lo;
  for (int64_t g = g0; g < g1; ++g) {
    while (piece_off[jb + 1] <= g) ++jb;
    const SbJob j = jobs[jb];
    const int64_t k = g - piece_off[jb];
    const bool aligned = ((j.src | j.dst | (uint64_t)j.width | (uint64_t)j.spitch | (uint64_t)j.dpitch) & 15) == 0;
    if (job_flat(j)) {
      const int64_t len = j.n_rows * j.width;
      const int64_t b = k * kPieceBytes;
      const int64_t e = b + kPieceBytes < len ? b + kPieceBytes : len;
      if (aligned) {
        warp_copy_flat<HINT>(reinterpret_cast<const char*>(j.src) + b, reinterpret_cast<char*>(j.dst) + b, e - b, lane);
      } else {
        const char* s = reinterpret_cast<const char*>(j.src);
        char* d = reinterpret_cast<char*>(j.dst);
        for (int64_t x = b + lane; x < e; x += 32) d[x] = s[x];
      }
    } else {
      const int64_t rp = job_rows_per_piece(j);
      const int64_t r0 = k * rp, r1 = r0 + rp < j.n_rows ? r0 + rp : j.n_rows;
      if (aligned) warp_copy_rows<HINT>(j, r0, r1, lane);
      else warp_copy_bytes(j, r0, r1, lane);
    }
  }
  // Peer (NVLink) stores must be visible system-wide before the barrier
  // kernel that follows publishes this phase as complete.
  if (fence_sys) __threadfence_system();
}

// rows per rank = sum of its sequence lengths (origin packing).
__global__ void k_rank_rows(const int64_t* lens, const int64_t* off, int64_t* rows) {
  __shared__ int64_t sh[33];
  const int r = blockIdx.x;
  int64_t local = 0;
  for (int64_t i = off[r] + threadIdx.x; i < off[r + 1]; i += blockDim.x) local += lens[i] > 0 ? lens[i] : 0;
  int64_t tot;
  block_excl_scan<int64_t>(local, sh, &tot);
  if (threadIdx.x == 0) rows[r] = tot;
}

// ------------------------------------------------- TMA bulk copy engine
// The same piece decomposition as k_copy, moved by the Tensor Memory
// Accelerator instead of the LSU: one elected lane per CTA streams each
// piece global -> shared (cp.async.bulk ... mbarrier::complete_tx) and
// shared -> global (cp.async.bulk.global.shared::cta.bulk_group) through a
// kTmaStages-deep ring of 32 KB stages.  Registers and issue slots stay
// free, and a few hundred bytes of instructions keep ~200 KB per SM in
// flight.  Used when every job is 16-byte aligned and pieces fit a stage
// (always true for the route/Ulysses layouts here) and the destination is
// local HBM.
// Default ring: 2 stages x 3 CTAs per SM (192 KB of stages per SM).  C2 DiT
// step, profiles/r02/tma_ring_sweep: 2x3 0.3126 ms, 3x2 0.315, 4x1 / 6x1
// 0.3155 (pre_attn alone faster, 112 vs 116 us, but one 128-192 KB CTA per SM
// leaves the side-stream plan / prepare kernels less room), 2x2 0.325, 3x1
// 0.328, 2x1 0.396.  SEQBAL_TMA_RING=stages,ctas_per_sm overrides.
constexpr int kTmaStages = 2;
constexpr int kTmaCtasPerSm = 3;
constexpr int kTmaMaxStages = 6;

// L2 eviction-priority variants of the bulk copies (SEQBAL_TMA_HINT bits:
// 1 = stores evict_first, 2 = loads evict_first, 4 = stores evict_last,
// 8 = loads evict_last); the policy word comes from createpolicy.
__device__ __forceinline__ uint64_t l2_policy(int evict_last) {
  uint64_t pol;
  if (evict_last) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* gdst, const void* smem_src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct PieceRef {
  const char* src;
  char* dst;
  int64_t rows;    // rows in this piece (flat: 1)
  int64_t width;   // bytes per row (flat: span bytes)
  int64_t spitch, dpitch;
};

__device__ __forceinline__ PieceRef piece_of(const SbJob& j, int64_t k) {
  PieceRef p;
  if (job_flat(j)) {
    const int64_t len = j.n_rows * j.width;
    const int64_t b = k * kPieceBytes;
    p.src = reinterpret_cast<const char*>(j.src) + b;
    p.dst = reinterpret_cast<char*>(j.dst) + b;
    p.rows = 1;
    p.width = (b + kPieceBytes < len ? kPieceBytes : len - b);
    p.spitch = p.dpitch = 0;
  } else {
    const int64_t rp = job_rows_per_piece(j);
    const int64_t r0 = k * rp, r1 = r0 + rp < j.n_rows ? r0 + rp : j.n_rows;
    p.src = reinterpret_cast<const char*>(j.src) + r0 * j.spitch;
    p.dst = reinterpret_cast<char*>(j.dst) + r0 * j.dpitch;
    p.rows = r1 - r0;
    p.width = j.width;
    p.spitch = j.spitch;
    p.dpitch = j.dpitch;
  }
  return p;
}

__global__ void __launch_bounds__(32) k_copy_tma(const SbJob* __restrict__ jobs, const int64_t* __restrict__ piece_off,
                                                 const int64_t* __restrict__ n_jobs_p, int hint, int stages) {
  extern __shared__ __align__(128) unsigned char stage_mem[];
  __shared__ __align__(8) uint64_t bars[kTmaMaxStages];
  const int ns = stages;
  const int64_t n_jobs = *n_jobs_p;
  const int64_t total = piece_off[n_jobs];
  const int64_t g0 = total * blockIdx.x / gridDim.x, g1 = total * (blockIdx.x + 1) / gridDim.x;
  if (g0 >= g1 || threadIdx.x != 0) return;  // one elected lane drives the DMA ring
  for (int s = 0; s < ns; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  int64_t lo = 0, hi = n_jobs;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (piece_off[mid] <= g0) lo = mid;
    else hi = mid;
  }
  const uint64_t spol = (hint & 5) ? l2_policy(hint & 4) : 0, lpol = (hint & 10) ? l2_policy(hint & 8) : 0;
  int64_t jl = lo, js = lo;  // job cursors of the load and the store streams
  auto load = [&](int64_t g, int s) {
    while (piece_off[jl + 1] <= g) ++jl;
    const PieceRef p = piece_of(jobs[jl], g - piece_off[jl]);
    char* sm = reinterpret_cast<char*>(stage_mem) + (size_t)s * kPieceBytes;
    mbar_expect_tx(&bars[s], (uint32_t)(p.rows * p.width));
    if (lpol)
      for (int64_t r = 0; r < p.rows; ++r)
        bulk_g2s_hint(sm + r * p.width, p.src + r * p.spitch, (uint32_t)p.width, &bars[s], lpol);
    else
      for (int64_t r = 0; r < p.rows; ++r) bulk_g2s(sm + r * p.width, p.src + r * p.spitch, (uint32_t)p.width, &bars[s]);
  };
  auto store = [&](int64_t g, int s) {
    while (piece_off[js + 1] <= g) ++js;
    const PieceRef p = piece_of(jobs[js], g - piece_off[js]);
    const char* sm = reinterpret_cast<const char*>(stage_mem) + (size_t)s * kPieceBytes;
    if (spol)
      for (int64_t r = 0; r < p.rows; ++r) bulk_s2g_hint(p.dst + r * p.dpitch, sm + r * p.width, (uint32_t)p.width, spol);
    else
      for (int64_t r = 0; r < p.rows; ++r) bulk_s2g(p.dst + r * p.dpitch, sm + r * p.width, (uint32_t)p.width);
    bulk_commit();
  };
  const int64_t n = g1 - g0;
  for (int64_t k = 0; k < ns && k < n; ++k) load(g0 + k, (int)k);
  for (int64_t k = 0; k < n; ++k) {
    const int s = (int)(k % ns);
    mbar_wait(&bars[s], (uint32_t)((k / ns) & 1));
    store(g0 + k, s);
    // refill the stage whose store was issued one step ago, once it has
    // been read out of shared memory
    if (k >= 1 && k - 1 + ns < n) {
      bulk_wait_read<1>();
      load(g0 + k - 1 + ns, (int)((k - 1) % ns));
    }
  }
  bulk_wait_all();
}

static int g_num_sms = 0;
static int copy_grid() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  static int per_sm = -1;  // CTAs per SM of the LSU copy grid (SEQBAL_COPY_CTAS_PER_SM)
  if (per_sm < 0) {
    const char* v = getenv("SEQBAL_COPY_CTAS_PER_SM");
    per_sm = v ? std::max(1, atoi(v)) : 8;
  }
  return g_num_sms * per_sm;
}

// ----------------------------------------------------- witness / checksum
// Witness fill for hosted ranks (exchange.cpp:18-23, 52-63): one warp per
// row; metadata {id, pos} and payload doubles payload_value(id, pos, col).
template <bool PAYLOAD>
__global__ void k_witness(WorldArgs w, TensorInfo ti, const uint64_t* ids, const int64_t* rank_off,
                          const int64_t* lens) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int lr = 0; lr < w.n_local; ++lr) {
    const int r = w.first_local + lr;
    const int64_t rows = w.rows[r];
    const int64_t s0 = rank_off[r], s1 = rank_off[r + 1];
    for (int64_t row = warp; row < rows; row += nwarps) {
      // sequence containing `row` (fixture path: linear walk over the rank's lengths)
      int64_t acc = 0, s = s0;
      for (; s < s1; ++s) {
        const int64_t l = lens[s] > 0 ? lens[s] : 0;
        if (row < acc + l) break;
        acc += l;
      }
      const uint64_t id = ids[s];
      const int64_t pos = row - acc;
      if (lane == 0) {
        uint64_t* m = reinterpret_cast<uint64_t*>(w.base[r] + row * w.pitch[r]);
        m[0] = id;
        m[1] = (uint64_t)pos;
      }
      for (int t = 1; PAYLOAD && t < w.T; ++t) {
        if (ti.kind[t] != 1) continue;
        double* pl = reinterpret_cast<double*>(w.base[t * w.W + r] + row * w.pitch[t * w.W + r]);
        const int wd = (int)(ti.row_bytes[t] / 8);
        for (int c = lane; c < wd; c += 32) {
          const uint64_t h = derive_key4(0x7061796c6f6164ULL, id, (uint64_t)pos, (uint64_t)c);
          pl[c] = (double)(h >> 11) * 0x1.0p-53;
        }
      }
    }
  }
}

// Row metadata {sample_id, position} of the origin layout: one CTA per hosted
// rank scans the rank's lengths in shared memory, then each warp writes
// whole sequences (coalesced 16-B stores, no per-row search).
__global__ void __launch_bounds__(1024) k_fill_meta(WorldArgs w, const uint64_t* ids, const int64_t* rank_off,
                                                    const int64_t* lens) {
  __shared__ int64_t sh[33];
  __shared__ int64_t s_off[1024];
  const int r = w.first_local + blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t s0 = rank_off[r], s1 = rank_off[r + 1];
  int64_t carry = 0;
  for (int64_t b = s0; b < s1; b += blockDim.x) {
    const int64_t s = b + threadIdx.x;
    const int64_t l = s < s1 ? (lens[s] > 0 ? lens[s] : 0) : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan<int64_t>(l, sh, &tot);
    s_off[threadIdx.x] = carry + ex;
    __syncthreads();
    for (int64_t q = b + warp; q < s1 && q < b + blockDim.x; q += nw) {
      const int64_t first = s_off[q - b];
      const int64_t l2 = lens[q] > 0 ? lens[q] : 0;
      const uint64_t id = ids[q];
      for (int64_t pos = lane; pos < l2; pos += 32) {
        uint64_t* m = reinterpret_cast<uint64_t*>(w.base[r] + (first + pos) * w.pitch[r]);
        m[0] = id;
        m[1] = (uint64_t)pos;
      }
    }
    carry += tot;
    __syncthreads();
  }
}

// simulator.cpp:128-136 on hosted full-width ranks.
__global__ void k_perturb(WorldArgs w, TensorInfo ti) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int lr = 0; lr < w.n_local; ++lr) {
    const int r = w.first_local + lr;
    const int64_t rows = w.rows[r];
    for (int64_t row = warp; row < rows; row += nwarps) {
      const uint64_t* m = reinterpret_cast<const uint64_t*>(w.base[r] + row * w.pitch[r]);
      const uint64_t h = derive_key3(0x706572747572ULL, m[0], m[1]);
      const double delta = (double)(h >> 11) * 0x1.0p-53;
      for (int t = 1; t < w.T; ++t) {
        if (ti.kind[t] != 1) continue;
        double* pl = reinterpret_cast<double*>(w.base[t * w.W + r] + row * w.pitch[t * w.W + r]);
        const int wd = (int)(w.pitch[t * w.W + r] / 8);
        for (int c = lane; c < wd; c += 32) pl[c] = __dadd_rn(pl[c], delta);
      }
    }
  }
}

// content_checksum (exchange.cpp:438-457) over payload tensor 1.
__global__ void k_checksum(WorldArgs w, unsigned long long* acc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long sum = 0;
  for (int lr = 0; lr < w.n_local; ++lr) {
    const int r = w.first_local + lr;
    const int64_t rows = w.rows[r];
    const int wd = (int)(w.pitch[1 * w.W + r] / 8);
    const int hc = w.headcol[r];
    for (int64_t row = warp; row < rows; row += nwarps) {
      const uint64_t* m = reinterpret_cast<const uint64_t*>(w.base[r] + row * w.pitch[r]);
      const uint64_t id = m[0], pos = m[1];
      const uint64_t* pl = reinterpret_cast<const uint64_t*>(w.base[1 * w.W + r] + row * w.pitch[1 * w.W + r]);
      for (int c = lane; c < wd; c += 32) sum += derive_key4(id, pos, (uint64_t)(hc + c), pl[c]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0 && sum) atomicAdd(acc, sum);
}

// worlds_bitwise_equal (exchange.cpp:459-480) on hosted ranks: per rank the
// row counts must match, then every byte of every tensor (16-B words).
// Adds the number of differing words (+1 per rank whose rows differ) to
// *count; 0 means bitwise equal.
__global__ void k_world_compare(WorldArgs a, WorldArgs b, TensorInfo ti, unsigned long long* count) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  unsigned long long bad = 0;
  for (int lr = 0; lr < a.n_local; ++lr) {
    const int r = a.first_local + lr;
    const int64_t rows = a.rows[r];
    if (rows != b.rows[r]) {
      if (tid == 0) ++bad;
      continue;
    }
    for (int t = 0; t < a.T; ++t) {
      const int64_t ap = a.pitch[t * a.W + r], bp = b.pitch[t * b.W + r];
      if (ap != bp) {
        if (tid == 0) ++bad;
        continue;
      }
      const int64_t words = rows * ap / 16;  // row bytes are multiples of 16 on the compared layouts
      const int4* x = reinterpret_cast<const int4*>(a.base[t * a.W + r]);
      const int4* y = reinterpret_cast<const int4*>(b.base[t * b.W + r]);
      for (int64_t i = tid; i < words; i += nthreads) {
        const int4 u = x[i], v = y[i];
        bad += (u.x != v.x) | (u.y != v.y) | (u.z != v.z) | (u.w != v.w);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(count, bad);
}

static void select_slot(sb_planner* p, int slot) {
  if (slot < 0 || slot >= sb_planner::kSlots) throw Error{SB_ERR_CONFIG, "exchange slot out of range"};
  p->cur_slot = slot;
  sb_planner::Slot& sl = p->slots[slot];
  p->jobs = sl.jobs;
  p->piece_off = sl.piece_off;
  p->n_jobs = sl.n_jobs;
  p->job_cap = sl.cap;
}

void ensure_jobs(sb_planner* p, int64_t cap) {
  sb_planner::Slot& sl = p->slots[p->cur_slot];
  if (cap > sl.cap) {
    if (sl.jobs) cudaFree(sl.jobs);
    if (sl.piece_off) cudaFree(sl.piece_off);
    sl.jobs = nullptr;
    sl.piece_off = nullptr;
    SB_CUDA(cudaMalloc(&sl.jobs, sizeof(SbJob) * (size_t)cap));
    SB_CUDA(cudaMalloc(&sl.piece_off, sizeof(int64_t) * (size_t)(cap + 1)));
    sl.cap = cap;
  }
  if (!sl.n_jobs) {
    SB_CUDA(cudaMalloc(&sl.n_jobs, sizeof(int64_t) * 2));
    SB_CUDA(cudaMemset(sl.n_jobs, 0, sizeof(int64_t) * 2));
  }
  select_slot(p, p->cur_slot);
}

static JobArgs jargs(sb_planner* p) {
  JobArgs j;
  j.n_chunks = p->n_chunks;
  j.c_idx = p->c_idx; j.c_src = p->c_src; j.c_dst = p->c_dst;
  j.bag_of_rank = p->d_rank_bag; j.bag_size = p->d_bag_size;
  j.c_start = p->c_start; j.c_end = p->c_end; j.c_src_row = p->c_src_row; j.c_dst_row = p->c_dst_row;
  j.c_seq_base = p->c_seq_base;
  j.U = p->U;
  j.max_bag = p->max_bag;
  j.jobs = p->jobs;
  j.n_jobs = p->n_jobs;
  j.owner = p->coll_mode ? p->x_owner : nullptr;
  return j;
}

static void check_compatible(sb_planner* p, sb_world* a, sb_world* b) {
  if (a->W != p->W || b->W != p->W)
    throw Error{SB_ERR_INTEGRITY, "route: plan world size " + std::to_string(p->W) + " != world ranks " +
                                      std::to_string(a->W)};
  if (a->T != b->T || a->row_bytes != b->row_bytes || a->n_local != b->n_local || a->first_local != b->first_local)
    throw Error{SB_ERR_CONFIG, "exchange: source and destination worlds have different tensors"};
  if (a->T > 16) throw Error{SB_ERR_CONFIG, "at most 16 tensors per world"};
}

// Copy engines: 0 = LSU (128-bit LDG/STG, 8 loads in flight per lane),
// 2 = LSU capped at 3 CTAs/SM worth of registers, 1 = TMA bulk.  Peer
// (multi-process) destinations always use the LSU path.  Defaults from the
// B200 measurements in profiles/: contiguous route spans -> LSU, strided
// Ulysses head slices -> TMA.  SEQBAL_ROUTE_ENGINE / SEQBAL_ULYSSES_ENGINE =
// ldg|ldg3|tma override.
static int engine_from_env(const char* var, int dflt) {
  const char* v = getenv(var);
  if (!v) return dflt;
  const std::string e(v);
  return e == "tma" ? 1 : e == "ldg3" ? 2 : e == "ldg" ? 0 : dflt;
}
static int route_engine() {
  static int e = engine_from_env("SEQBAL_ROUTE_ENGINE", 0);
  return e;
}
// Ulysses copies move head slices of row_bytes / G bytes.  Measured on B200
// (profiles/r01b): the TMA bulk ring wins for wide slices (C2, G = 2,
// 3072 B: 45 vs 59 us) and loses for narrow ones (C3, G = 8, 768 B: 341 vs
// 237 us -- one issuing thread per CTA cannot keep enough small bulk copies
// in flight); at G = 4 (1536 B) they tie.  Default: TMA when every payload
// slice is >= 2 KB, else the LSU engine.  SEQBAL_ULYSSES_ENGINE overrides.
static int ulysses_engine(int64_t min_slice_bytes) {
  static int e = engine_from_env("SEQBAL_ULYSSES_ENGINE", -1);
  if (e >= 0) return e;
  return min_slice_bytes >= 2048 ? 1 : 0;
}

constexpr int64_t kFusedPrepMaxJobs = 1 << 16;  // single-CTA prep up to this many jobs

static void launch_copy(SbJob* jobs, int64_t* piece_off, int64_t* n_jobs, cudaStream_t s, int fence_sys,
                        bool tma_ok, int engine);

static void run_copy(sb_planner* p, cudaStream_t s, int fence_sys, bool tma_ok, int engine, bool pieces_done) {
  if (!pieces_done) {
    k_pieces<<<1, 1024, 0, s>>>(p->jobs, p->n_jobs, p->piece_off, p->n_jobs + 1);
    SB_CHECK_LAUNCH();
    count_launch(1);
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p->timing) {
    if (p->copy_used + 2 > p->copy_ev.size()) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        SB_CUDA(cudaEventCreate(&e));
        p->copy_ev.push_back(e);
      }
      p->copy_op.resize(p->copy_ev.size() / 2);
    }
    e0 = p->copy_ev[p->copy_used];
    e1 = p->copy_ev[p->copy_used + 1];
    p->copy_op[p->copy_used / 2] = p->current_op;
    p->copy_used += 2;
    SB_CUDA(cudaEventRecord(e0, s));
  }
  launch_copy(p->jobs, p->piece_off, p->n_jobs, s, fence_sys, tma_ok, engine);
  if (e1) SB_CUDA(cudaEventRecord(e1, s));
}

// The copy engines over a prepared job list (pieces already scanned).
static void launch_copy(SbJob* jobs, int64_t* piece_off, int64_t* n_jobs, cudaStream_t s, int fence_sys,
                        bool tma_ok, int engine) {
  if (!fence_sys && tma_ok && engine == 1) {
    static int stages = 0, per_sm = 0;  // ring depth x CTAs per SM
    if (!stages) {
      stages = kTmaStages;
      per_sm = kTmaCtasPerSm;
      if (const char* v = getenv("SEQBAL_TMA_RING")) {
        int a = 0, b = 0;
        if (sscanf(v, "%d,%d", &a, &b) == 2 && a >= 2 && a <= kTmaMaxStages && b >= 1 && b <= 8) {
          stages = a;
          per_sm = b;
        }
      }
      SB_CUDA(cudaFuncSetAttribute(k_copy_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(stages * kPieceBytes)));
      SB_CUDA(cudaFuncSetAttribute(k_copy_tma, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    copy_grid();
    static int tma_hint = -1;  // SEQBAL_TMA_HINT (see l2_policy)
    if (tma_hint < 0) {
      const char* v = getenv("SEQBAL_TMA_HINT");
      tma_hint = v ? atoi(v) : 0;
    }
    k_copy_tma<<<g_num_sms * per_sm, 32, stages * kPieceBytes, s>>>(jobs, piece_off, n_jobs, tma_hint, stages);
  } else if (engine == 2) {
    k_copy<3><<<copy_grid(), kCopyThreads, 0, s>>>(jobs, piece_off, n_jobs, fence_sys);
  } else {
    static int hint = -1;  // SEQBAL_COPY_HINT=0..4 (see ld_stream)
    if (hint < 0) {
      const char* v = getenv("SEQBAL_COPY_HINT");
      hint = v ? atoi(v) : 0;
    }
    if (hint == 1) k_copy<1, 1><<<copy_grid(), kCopyThreads, 0, s>>>(jobs, piece_off, n_jobs, fence_sys);
    else if (hint == 2) k_copy<1, 2><<<copy_grid(), kCopyThreads, 0, s>>>(jobs, piece_off, n_jobs, fence_sys);
    else if (hint == 3) k_copy<1, 3><<<copy_grid(), kCopyThreads, 0, s>>>(jobs, piece_off, n_jobs, fence_sys);
    else if (hint == 4) k_copy<1, 4><<<copy_grid(), kCopyThreads, 0, s>>>(jobs, piece_off, n_jobs, fence_sys);
    else k_copy<1, 0><<<copy_grid(), kCopyThreads, 0, s>>>(jobs, piece_off, n_jobs, fence_sys);
  }
  SB_CHECK_LAUNCH();
  count_launch(1);
}

}  // namespace sb

// ============================================================== C-ABI
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

extern "C" const char* sb_last_error(void) { return sb::g_last_error.c_str(); }
extern "C" int sb_abi_version(void) { return 1; }
extern "C" int64_t sb_kernel_launches(void) { return sb::g_launches.load(); }

extern "C" sb_status sb_world_create(const sb_world_desc* d, sb_world** out) {
  SB_API_BEGIN
  if (!d || !out) throw Error{SB_ERR_CONFIG, "sb_world_create: null argument"};
  *out = nullptr;
  if (d->world_size < 1 || d->n_local < 1 || d->world_size % d->n_local != 0 || d->first_local % d->n_local != 0 ||
      d->first_local + d->n_local > d->world_size)
    throw Error{SB_ERR_CONFIG, "sb_world_create: hosted ranks must be a contiguous block dividing the world"};
  if (d->n_payload < 1 || d->n_aux < 0 || d->n_heads < 1 || 1 + d->n_payload + d->n_aux > 16)
    throw Error{SB_ERR_CONFIG, "sb_world_create: need 1..15 tensors and n_heads >= 1"};
  auto* w = new sb_world();
  w->W = d->world_size;
  w->n_local = d->n_local;
  w->first_local = d->first_local;
  w->n_heads = d->n_heads;
  w->n_payload = d->n_payload;
  w->n_aux = d->n_aux;
  w->T = 1 + d->n_payload + d->n_aux;
  w->max_bag = std::max(1, d->max_bag);
  w->n_procs = d->world_size / d->n_local;
  w->capacity_rows = std::max<int64_t>(1, d->capacity_rows);
  w->row_bytes.push_back(16);
  w->tensor_desc.push_back(0);
  for (int i = 0; i < d->n_payload + d->n_aux; ++i) {
    const int64_t rb = d->row_bytes[i];
    if (rb < 1) {
      delete w;
      throw Error{SB_ERR_CONFIG, "row bytes must be >= 1"};
    }
    if (i < d->n_payload && rb % d->n_heads != 0) {
      delete w;
      throw Error{SB_ERR_CONFIG, "payload width must be a positive multiple of n_heads"};
    }
    w->row_bytes.push_back(rb);
    w->tensor_desc.push_back(i < d->n_payload ? 1 : 2);
  }
  try {
    w->arena.assign(w->T, nullptr);
    w->arena_bytes.assign(w->T, 0);
    for (int t = 0; t < w->T; ++t) {
      // metadata is replicated G-fold in the Ulysses layout
      int64_t bytes = w->capacity_rows * w->row_bytes[t];
      if (t == 0 || w->tensor_desc[t] == 2) bytes *= w->max_bag;
      w->arena_bytes[t] = bytes;
      SB_CUDA(cudaMalloc(&w->arena[t], (size_t)bytes));
    }
    SB_CUDA(cudaMalloc(&w->d_base, sizeof(uint64_t) * w->T * w->W));
    SB_CUDA(cudaMalloc(&w->d_pitch, sizeof(int64_t) * w->T * w->W));
    SB_CUDA(cudaMalloc(&w->d_rows, sizeof(int64_t) * w->W));
    SB_CUDA(cudaMalloc(&w->d_headcol, sizeof(int32_t) * w->W));
    SB_CUDA(cudaMalloc(&w->d_peer_arena, sizeof(uint64_t) * w->T * w->n_procs));
    SB_CUDA(cudaMalloc(&w->d_arena_bytes, sizeof(int64_t) * w->T));
    SB_CUDA(cudaMalloc(&w->d_status, sizeof(int32_t)));
    SB_CUDA(cudaMemset(w->d_status, 0, sizeof(int32_t)));
    SB_CUDA(cudaMemset(w->d_rows, 0, sizeof(int64_t) * w->W));
    SB_CUDA(cudaMemset(w->d_headcol, 0, sizeof(int32_t) * w->W));
    SB_CUDA(cudaMemset(w->d_base, 0, sizeof(uint64_t) * w->T * w->W));
    SB_CUDA(cudaMemset(w->d_pitch, 0, sizeof(int64_t) * w->T * w->W));
    SB_CUDA(cudaMemcpy(w->d_arena_bytes, w->arena_bytes.data(), sizeof(int64_t) * w->T, cudaMemcpyHostToDevice));
    // single process: every "peer" slot is this process's arena
    std::vector<uint64_t> pa((size_t)w->T * w->n_procs, 0);
    const int me = w->first_local / w->n_local;
    for (int t = 0; t < w->T; ++t) pa[(size_t)t * w->n_procs + me] = (uint64_t)w->arena[t];
    SB_CUDA(cudaMemcpy(w->d_peer_arena, pa.data(), sizeof(uint64_t) * pa.size(), cudaMemcpyHostToDevice));
  } catch (...) {
    for (void* q : w->arena)
      if (q) cudaFree(q);
    delete w;
    throw;
  }
  *out = w;
  SB_API_END
}

extern "C" sb_status sb_world_destroy(sb_world* w) {
  SB_API_BEGIN
  if (w) {
    for (void* q : w->arena)
      if (q) cudaFree(q);
    void* ptrs[] = {w->d_base, w->d_pitch, w->d_rows, w->d_headcol, w->d_peer_arena, w->d_arena_bytes, w->d_status};
    for (void* q : ptrs)
      if (q) cudaFree(q);
    delete w;
  }
  SB_API_END
}

extern "C" sb_status sb_world_arena(const sb_world* w, int t, void** base, int64_t* bytes) {
  SB_API_BEGIN
  if (!w || t < 0 || t >= w->T) throw Error{SB_ERR_CONFIG, "sb_world_arena: bad tensor"};
  if (base) *base = w->arena[t];
  if (bytes) *bytes = w->arena_bytes[t];
  SB_API_END
}

extern "C" sb_status sb_world_tables(const sb_world* w, int t, const uint64_t** b, const int64_t** pitch,
                                     const int64_t** rows) {
  SB_API_BEGIN
  if (!w || t < 0 || t >= w->T) throw Error{SB_ERR_CONFIG, "sb_world_tables: bad tensor"};
  if (b) *b = w->d_base + (size_t)t * w->W;
  if (pitch) *pitch = w->d_pitch + (size_t)t * w->W;
  if (rows) *rows = w->d_rows;
  SB_API_END
}

extern "C" sb_status sb_world_set_peers(sb_world* w, int t, const uint64_t* host_bases, int n_procs) {
  SB_API_BEGIN
  if (!w || t < 0 || t >= w->T || n_procs != w->n_procs || !host_bases)
    throw Error{SB_ERR_CONFIG, "sb_world_set_peers: bad arguments"};
  SB_CUDA(cudaMemcpy(w->d_peer_arena + (size_t)t * w->n_procs, host_bases, sizeof(uint64_t) * n_procs,
                     cudaMemcpyHostToDevice));
  SB_API_END
}

extern "C" sb_status sb_world_layout_origin(sb_world* w, const int64_t* d_lens, const int64_t* d_rank_off,
                                            sb_stream stream) {
  SB_API_BEGIN
  if (!w || !d_lens || !d_rank_off) throw Error{SB_ERR_CONFIG, "sb_world_layout_origin: null argument"};
  (void)d_lens;
  cudaStream_t s = (cudaStream_t)stream;
  sb::k_rank_rows<<<w->W, 256, 0, s>>>(d_lens, d_rank_off, w->d_rows);
  SB_CHECK_LAUNCH();
  sb::LayoutPlan lp{};
  lp.rows_src = w->d_rows;
  lp.expect_rows = w->d_rows;
  sb::WorldArgs a = sb::wargs(w);
  sb::k_layout<<<1, 32 * 16, 0, s>>>(a, a, lp, sb::tinfo(w), 0);
  SB_CHECK_LAUNCH();
  sb::count_launch(2);
  SB_API_END
}

// Layout of a world that no exchange produced (e.g. q/k/v written by a
// projection in the chunk layout, or an attention output in the Ulysses
// layout): per-rank tables from the current plan, on the device.
extern "C" sb_status sb_world_layout_plan(sb_world* w, const sb_planner* p, int layout, sb_stream stream) {
  SB_API_BEGIN
  if (!w || !p) throw Error{SB_ERR_CONFIG, "sb_world_layout_plan: null argument"};
  if (w->W != p->W)
    throw Error{SB_ERR_INTEGRITY, "layout: plan world size " + std::to_string(p->W) + " != world ranks " +
                                      std::to_string(w->W)};
  if (layout < 0 || layout > 2) throw Error{SB_ERR_CONFIG, "sb_world_layout_plan: layout must be 0, 1 or 2"};
  if (!p->origin_rows || !p->target_rows) throw Error{SB_ERR_CONFIG, "sb_world_layout_plan: no plan"};
  sb::LayoutPlan lp{};
  lp.no_check = 1;
  int mode = 0;
  if (layout == 0 || layout == 1) {
    lp.rows_src = layout == 0 ? p->origin_rows : p->target_rows;
  } else {
    if (p->identity || p->uploaded)
      throw Error{SB_ERR_CONFIG, "Ulysses layout needs a device-built plan (sb_plan)"};
    for (int b = 0; b < p->M; ++b)
      if (w->n_heads % p->bag_size[b] != 0)
        throw Error{SB_ERR_CONFIG, "pre_attn: bag of " + std::to_string(p->bag_size[b]) +
                                       " GPUs does not divide n_heads " + std::to_string(w->n_heads)};
    if (w->max_bag < p->max_bag) throw Error{SB_ERR_CONFIG, "world max_bag smaller than the topology's bags"};
    lp.rank_bag = p->d_rank_bag;
    lp.rank_member = p->d_rank_member;
    lp.bag_size = p->d_bag_size;
    lp.bag_rows = p->bag_rows;
    lp.target_rows = p->target_rows;
    lp.U = p->U;
    lp.M = p->M;
    mode = 3;
  }
  sb::WorldArgs a = sb::wargs(w);
  sb::k_layout<<<1, 32 * 16, 0, (cudaStream_t)stream>>>(a, a, lp, sb::tinfo(w), mode);
  SB_CHECK_LAUNCH();
  sb::count_launch();
  SB_API_END
}

extern "C" sb_status sb_world_fill_witness(sb_world* w, const uint64_t* d_ids, const int64_t* d_lens,
                                           const int64_t* d_rank_off, sb_stream stream) {
  SB_API_BEGIN
  if (!w || !d_ids || !d_lens || !d_rank_off) throw Error{SB_ERR_CONFIG, "sb_world_fill_witness: null argument"};
  for (int t = 1; t < w->T; ++t)
    if (w->tensor_desc[t] == 1 && w->row_bytes[t] % 8 != 0)
      throw Error{SB_ERR_CONFIG, "witness payload must be whole doubles"};
  sb::k_witness<true><<<sb::copy_grid(), 256, 0, (cudaStream_t)stream>>>(sb::wargs(w), sb::tinfo(w), d_ids,
                                                                         d_rank_off, d_lens);
  SB_CHECK_LAUNCH();
  sb::count_launch();
  SB_API_END
}

extern "C" sb_status sb_world_fill_meta(sb_world* w, const uint64_t* d_ids, const int64_t* d_lens,
                                        const int64_t* d_rank_off, sb_stream stream) {
  SB_API_BEGIN
  if (!w || !d_ids || !d_lens || !d_rank_off) throw Error{SB_ERR_CONFIG, "sb_world_fill_meta: null argument"};
  sb::k_fill_meta<<<w->n_local, 1024, 0, (cudaStream_t)stream>>>(sb::wargs(w), d_ids, d_rank_off, d_lens);
  SB_CHECK_LAUNCH();
  sb::count_launch();
  SB_API_END
}

extern "C" sb_status sb_world_perturb(sb_world* w, sb_stream stream) {
  SB_API_BEGIN
  if (!w) throw Error{SB_ERR_CONFIG, "null world"};
  sb::k_perturb<<<sb::copy_grid(), 256, 0, (cudaStream_t)stream>>>(sb::wargs(w), sb::tinfo(w));
  SB_CHECK_LAUNCH();
  sb::count_launch();
  SB_API_END
}

extern "C" sb_status sb_world_compare(sb_world* a, sb_world* b, uint64_t* d_count, sb_stream stream) {
  SB_API_BEGIN
  if (!a || !b || !d_count) throw Error{SB_ERR_CONFIG, "sb_world_compare: null argument"};
  if (a->W != b->W || a->T != b->T || a->n_local != b->n_local || a->first_local != b->first_local)
    throw Error{SB_ERR_CONFIG, "sb_world_compare: worlds of different shape"};
  for (int t = 0; t < a->T; ++t)
    if (a->row_bytes[t] % 16 != 0) throw Error{SB_ERR_CONFIG, "sb_world_compare: row bytes must be multiples of 16"};
  sb::k_world_compare<<<sb::copy_grid(), 256, 0, (cudaStream_t)stream>>>(
      sb::wargs(a), sb::wargs(b), sb::tinfo(a), reinterpret_cast<unsigned long long*>(d_count));
  SB_CHECK_LAUNCH();
  sb::count_launch();
  SB_API_END
}

extern "C" sb_status sb_world_checksum(sb_world* w, uint64_t* d_acc, sb_stream stream) {
  SB_API_BEGIN
  if (!w || !d_acc) throw Error{SB_ERR_CONFIG, "null argument"};
  sb::k_checksum<<<sb::copy_grid(), 256, 0, (cudaStream_t)stream>>>(sb::wargs(w),
                                                                    reinterpret_cast<unsigned long long*>(d_acc));
  SB_CHECK_LAUNCH();
  sb::count_launch();
  SB_API_END
}

// ------------------------------------------------------ prepare / run
// prepare: destination layout + copy jobs + piece scan into `slot`;
// run: the copy kernel over the slot.  sb_route & co. do both back to back;
// sb_exchange_prepare/run let a caller prepare on a side stream while an
// earlier exchange is still copying (the preparations chain only through
// the world tables, never through the payload).
static void prepare_route(sb_planner* p, int slot, int reverse, sb_world* src, sb_world* dst, cudaStream_t s) {
  if (src == dst) throw Error{SB_ERR_CONFIG, "sb_route is out-of-place: src and dst must differ"};
  sb::check_compatible(p, src, dst);
  sb::select_slot(p, slot);
  sb::ensure_jobs(p, p->max_chunks * src->T);
  sb::LayoutPlan lp{};
  lp.rows_src = reverse ? p->origin_rows : p->target_rows;
  lp.expect_rows = reverse ? p->target_rows : p->origin_rows;
  const bool fused = p->max_chunks * src->T <= sb::kFusedPrepMaxJobs;
  if (fused) {
    sb::k_exchange_prep<<<1, 1024, 0, s>>>(sb::jargs(p), sb::wargs(src), sb::wargs(dst), sb::tinfo(src), lp,
                                           reverse ? 1 : 0, p->piece_off, p->n_jobs + 1);
    SB_CHECK_LAUNCH();
    sb::count_launch(1);
  } else {
    sb::k_layout<<<1, 32 * 16, 0, s>>>(sb::wargs(dst), sb::wargs(src), lp, sb::tinfo(dst), 0);
    SB_CHECK_LAUNCH();
    sb::k_jobs_route<<<std::min<int64_t>(1184, (p->max_chunks * src->T + 255) / 256), 256, 0, s>>>(
        sb::jargs(p), sb::wargs(src), sb::wargs(dst), sb::tinfo(src), reverse);
    SB_CHECK_LAUNCH();
    sb::count_launch(2);
  }
  bool tma_ok = true;  // every row size a multiple of 16 B: all spans are TMA-legal
  for (int64_t rb : src->row_bytes) tma_ok &= rb % 16 == 0;
  sb_planner::Slot& sl = p->slots[slot];
  sl.prepared = true;
  sl.pieces_done = fused;
  sl.tma_ok = tma_ok;
  sl.fence_sys = dst->n_procs > 1;
  sl.engine = sb::route_engine();
  sl.op = reverse ? 1 : 0;
}

static void prepare_ulysses(sb_planner* p, int slot, int post, sb_world* src, sb_world* dst, cudaStream_t s) {
  if (p->identity) throw Error{SB_ERR_CONFIG, "Ulysses transforms need a balanced plan (not identity_plan)"};
  if (p->uploaded)
    throw Error{SB_ERR_CONFIG, "Ulysses transforms need a device-built plan (sb_plan); use sb_apply_moves"};
  sb::check_compatible(p, src, dst);
  if (src == dst) throw Error{SB_ERR_CONFIG, "Ulysses transforms are out-of-place: src and dst must differ"};
  for (int b = 0; b < p->M; ++b)
    if (src->n_heads % p->bag_size[b] != 0)
      throw Error{SB_ERR_CONFIG, "pre_attn: bag of " + std::to_string(p->bag_size[b]) +
                                     " GPUs does not divide n_heads " + std::to_string(src->n_heads)};
  if (dst->max_bag < p->max_bag) throw Error{SB_ERR_CONFIG, "world max_bag smaller than the topology's bags"};
  sb::select_slot(p, slot);
  sb::ensure_jobs(p, p->max_chunks * p->max_bag * src->T);
  sb::LayoutPlan lp{};
  lp.rank_bag = p->d_rank_bag;
  lp.rank_member = p->d_rank_member;
  lp.bag_size = p->d_bag_size;
  lp.bag_rows = p->bag_rows;
  lp.target_rows = p->target_rows;
  lp.U = p->U;
  lp.M = p->M;
  const int64_t total = p->max_chunks * p->max_bag * src->T;
  const bool fused = total <= sb::kFusedPrepMaxJobs;
  if (fused) {
    sb::k_exchange_prep<<<1, 1024, 0, s>>>(sb::jargs(p), sb::wargs(src), sb::wargs(dst), sb::tinfo(src), lp,
                                           post ? 3 : 2, p->piece_off, p->n_jobs + 1);
    SB_CHECK_LAUNCH();
    sb::count_launch(1);
  } else {
    sb::k_layout<<<1, 32 * 16, 0, s>>>(sb::wargs(dst), sb::wargs(src), lp, sb::tinfo(dst), post ? 2 : 1);
    SB_CHECK_LAUNCH();
    sb::k_jobs_ulysses<<<std::min<int64_t>(1184, (total + 255) / 256), 256, 0, s>>>(
        sb::jargs(p), sb::wargs(src), sb::wargs(dst), sb::tinfo(src), post);
    SB_CHECK_LAUNCH();
    sb::count_launch(2);
  }
  bool tma_ok = true;  // row and head-slice sizes multiples of 16 B, slices within a stage
  int64_t min_slice = INT64_MAX;
  for (int t = 0; t < src->T; ++t) {
    tma_ok &= src->row_bytes[t] % 16 == 0;
    if (src->tensor_desc[t] == 1)
      for (int b = 0; b < p->M; ++b) {
        const int64_t slice = src->row_bytes[t] / p->bag_size[b];
        tma_ok &= slice % 16 == 0 && slice <= sb::kPieceBytes;
        if (p->bag_size[b] > 1) min_slice = std::min(min_slice, slice);
      }
  }
  sb_planner::Slot& sl = p->slots[slot];
  sl.prepared = true;
  sl.pieces_done = fused;
  sl.tma_ok = tma_ok;
  sl.fence_sys = dst->n_procs > 1;
  sl.engine = sb::ulysses_engine(min_slice);
  sl.op = post ? 3 : 2;
}

static void run_slot(sb_planner* p, int slot, cudaStream_t s) {
  sb::select_slot(p, slot);
  sb_planner::Slot& sl = p->slots[slot];
  if (!sl.prepared) throw Error{SB_ERR_CONFIG, "exchange slot " + std::to_string(slot) + " was not prepared"};
  p->current_op = sl.op;
  p->last_run_slot = slot;
  sb::run_copy(p, s, sl.fence_sys, sl.tma_ok, sl.engine, sl.pieces_done);
}

extern "C" sb_status sb_exchange_prepare(sb_planner* p, int op, sb_world* src, sb_world* dst, int slot,
                                         sb_stream stream) {
  SB_API_BEGIN
  if (!p || !src || !dst) throw Error{SB_ERR_CONFIG, "sb_exchange_prepare: null argument"};
  cudaStream_t s = (cudaStream_t)stream;
  if (op == 0 || op == 1) prepare_route(p, slot, op, src, dst, s);
  else if (op == 2 || op == 3) prepare_ulysses(p, slot, op == 3, src, dst, s);
  else throw Error{SB_ERR_CONFIG, "sb_exchange_prepare: op must be 0..3"};
  SB_API_END
}

extern "C" sb_status sb_exchange_run(sb_planner* p, int slot, sb_stream stream) {
  SB_API_BEGIN
  if (!p) throw Error{SB_ERR_CONFIG, "sb_exchange_run: null planner"};
  run_slot(p, slot, (cudaStream_t)stream);
  SB_API_END
}

extern "C" sb_status sb_route(sb_planner* p, int reverse, sb_world* src, sb_world* dst, sb_stream stream) {
  SB_API_BEGIN
  if (!p || !src || !dst) throw Error{SB_ERR_CONFIG, "sb_route: null argument"};
  prepare_route(p, reverse ? 1 : 0, reverse ? 1 : 0, src, dst, (cudaStream_t)stream);
  run_slot(p, reverse ? 1 : 0, (cudaStream_t)stream);
  SB_API_END
}

extern "C" sb_status sb_pre_attn(sb_planner* p, sb_world* src, sb_world* dst, sb_stream stream) {
  SB_API_BEGIN
  if (!p || !src || !dst) throw Error{SB_ERR_CONFIG, "sb_pre_attn: null argument"};
  prepare_ulysses(p, 2, 0, src, dst, (cudaStream_t)stream);
  run_slot(p, 2, (cudaStream_t)stream);
  SB_API_END
}

extern "C" sb_status sb_post_attn(sb_planner* p, sb_world* src, sb_world* dst, sb_stream stream) {
  SB_API_BEGIN
  if (!p || !src || !dst) throw Error{SB_ERR_CONFIG, "sb_post_attn: null argument"};
  prepare_ulysses(p, 3, 1, src, dst, (cudaStream_t)stream);
  run_slot(p, 3, (cudaStream_t)stream);
  SB_API_END
}

// Collective transport (the NCCL baseline; see k_collective_split): pack
// this process's outbound jobs of exchange `op` (0 route, 1 reverse_route,
// 2 pre_attn, 3 post_attn) into per-destination segments of send_buf and
// copy local-to-local jobs directly; write the all-to-all-v byte counts to
// d_counts[0, 2P).  The caller moves send_buf -> recv_buf (ncclSend/ncclRecv
// grouped, or any all-to-all-v) on the same stream, then calls
// sb_exchange_unpack.  Worlds need no peer mappings (sb_world_set_peers).
extern "C" sb_status sb_exchange_pack(sb_planner* p, int op, sb_world* src, sb_world* dst, void* send_buf,
                                      int64_t send_cap, void* recv_buf, int64_t recv_cap, int64_t* d_counts,
                                      sb_stream stream) {
  SB_API_BEGIN
  if (!p || !src || !dst || !d_counts) throw Error{SB_ERR_CONFIG, "sb_exchange_pack: null argument"};
  if (op < 0 || op > 3) throw Error{SB_ERR_CONFIG, "sb_exchange_pack: op must be 0..3"};
  if ((send_cap > 0 && !send_buf) || (recv_cap > 0 && !recv_buf) || send_cap < 0 || recv_cap < 0)
    throw Error{SB_ERR_CONFIG, "sb_exchange_pack: bad transport buffers"};
  if (dst->n_procs > sb::kMaxCollProcs)
    throw Error{SB_ERR_CONFIG, "collective transport supports at most " + std::to_string(sb::kMaxCollProcs) +
                                   " processes"};
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t cap = op < 2 ? p->max_chunks * src->T : p->max_chunks * p->max_bag * src->T;
  if (cap > p->x_owner_cap) {
    if (p->x_owner) cudaFree(p->x_owner);
    p->x_owner = nullptr;
    p->x_owner_cap = 0;
    SB_CUDA(cudaMalloc(&p->x_owner, sizeof(int32_t) * (size_t)std::max<int64_t>(1, cap)));
    p->x_owner_cap = cap;
  }
  sb_planner::Slot& u = p->unpack;
  if (cap > u.cap) {
    if (u.jobs) cudaFree(u.jobs);
    if (u.piece_off) cudaFree(u.piece_off);
    u.jobs = nullptr;
    u.piece_off = nullptr;
    u.cap = 0;
    SB_CUDA(cudaMalloc(&u.jobs, sizeof(SbJob) * (size_t)std::max<int64_t>(1, cap)));
    SB_CUDA(cudaMalloc(&u.piece_off, sizeof(int64_t) * (size_t)(cap + 1)));
    u.cap = cap;
  }
  if (!u.n_jobs) {
    SB_CUDA(cudaMalloc(&u.n_jobs, sizeof(int64_t) * 2));
    SB_CUDA(cudaMemset(u.n_jobs, 0, sizeof(int64_t) * 2));
  }
  u.prepared = false;
  p->coll_mode = true;
  try {
    if (op < 2) prepare_route(p, op, op, src, dst, s);
    else prepare_ulysses(p, op, op == 3, src, dst, s);
  } catch (...) {
    p->coll_mode = false;
    throw;
  }
  p->coll_mode = false;
  sb_planner::Slot& sl = p->slots[op];
  const int me = dst->first_local / dst->n_local;
  sb::k_collective_split<<<1, 1024, 0, s>>>(sl.jobs, p->x_owner, sl.n_jobs, me, dst->n_procs, (uint64_t)send_buf,
                                             send_cap, (uint64_t)recv_buf, recv_cap, dst->d_status, sl.piece_off,
                                             sl.n_jobs + 1, u.jobs, u.n_jobs, u.piece_off, d_counts);
  SB_CHECK_LAUNCH();
  sb::count_launch(1);
  sl.pieces_done = true;
  sl.fence_sys = 0;  // every store is local: the send buffer or this process's arena
  u.prepared = true;
  u.pieces_done = true;
  u.tma_ok = sl.tma_ok;
  u.engine = sl.engine;
  u.fence_sys = 0;
  u.op = sl.op;
  run_slot(p, op, s);
  SB_API_END
}

extern "C" sb_status sb_exchange_unpack(sb_planner* p, sb_stream stream) {
  SB_API_BEGIN
  if (!p) throw Error{SB_ERR_CONFIG, "sb_exchange_unpack: null planner"};
  sb_planner::Slot& u = p->unpack;
  if (!u.prepared) throw Error{SB_ERR_CONFIG, "sb_exchange_unpack: no packed exchange"};
  p->current_op = u.op;
  sb::launch_copy(u.jobs, u.piece_off, u.n_jobs, (cudaStream_t)stream, 0, u.tma_ok, u.engine);
  u.prepared = false;
  SB_API_END
}

extern "C" sb_status sb_world_status(sb_world* w, sb_stream stream) {
  SB_API_BEGIN
  if (!w) throw Error{SB_ERR_CONFIG, "null world"};
  SB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  int32_t st = 0;
  SB_CUDA(cudaMemcpy(&st, w->d_status, sizeof st, cudaMemcpyDeviceToHost));
  if (st & sb::ST_LAYOUT) throw Error{SB_ERR_CAPACITY, "world arena too small for the requested layout"};
  if (st & sb::ST_CAPACITY) throw Error{SB_ERR_CAPACITY, "collective transport buffers too small for the exchange"};
  if (st & sb::ST_MISMATCH)
    throw Error{SB_ERR_INTEGRITY, "exchange source world does not match the plan's layout (rows per rank differ); "
                                  "nothing was copied"};
  if (st) throw Error{SB_ERR_INTEGRITY, "world status " + std::to_string(st)};
  SB_API_END
}

extern "C" sb_status sb_world_upload(sb_world* w, void* const* host, const int64_t* bytes, sb_stream stream) {
  SB_API_BEGIN
  if (!w || !host || !bytes) throw Error{SB_ERR_CONFIG, "sb_world_upload: null argument"};
  for (int t = 0; t < w->T; ++t) {
    if (bytes[t] > w->arena_bytes[t]) throw Error{SB_ERR_CAPACITY, "sb_world_upload: image larger than arena"};
    if (host[t] && bytes[t] > 0)
      SB_CUDA(cudaMemcpyAsync(w->arena[t], host[t], (size_t)bytes[t], cudaMemcpyHostToDevice, (cudaStream_t)stream));
  }
  SB_API_END
}

extern "C" sb_status sb_world_download(sb_world* w, void* const* host, const int64_t* bytes, sb_stream stream) {
  SB_API_BEGIN
  if (!w || !host || !bytes) throw Error{SB_ERR_CONFIG, "sb_world_download: null argument"};
  for (int t = 0; t < w->T; ++t) {
    if (bytes[t] > w->arena_bytes[t]) throw Error{SB_ERR_CAPACITY, "sb_world_download: image larger than arena"};
    if (host[t] && bytes[t] > 0)
      SB_CUDA(cudaMemcpyAsync(host[t], w->arena[t], (size_t)bytes[t], cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  }
  SB_API_END
}

extern "C" sb_status sb_world_shape(sb_world* w, int t, int64_t* rows, int64_t* pitch, sb_stream stream) {
  SB_API_BEGIN
  if (!w || t < 0 || t >= w->T) throw Error{SB_ERR_CONFIG, "sb_world_shape: bad tensor"};
  SB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (rows) SB_CUDA(cudaMemcpy(rows, w->d_rows, sizeof(int64_t) * w->W, cudaMemcpyDeviceToHost));
  if (pitch) SB_CUDA(cudaMemcpy(pitch, w->d_pitch + (size_t)t * w->W, sizeof(int64_t) * w->W, cudaMemcpyDeviceToHost));
  SB_API_END
}

static void rank_span(sb_world* w, int t, int rank, cudaStream_t s, uint64_t* base, int64_t* bytes) {
  if (!w || t < 0 || t >= w->T || rank < 0 || rank >= w->W) throw Error{SB_ERR_CONFIG, "bad tensor or rank"};
  SB_CUDA(cudaStreamSynchronize(s));
  int64_t rows = 0, pitch = 0;
  SB_CUDA(cudaMemcpy(&rows, w->d_rows + rank, sizeof rows, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(&pitch, w->d_pitch + (size_t)t * w->W + rank, sizeof pitch, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(base, w->d_base + (size_t)t * w->W + rank, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  *bytes = rows * pitch;
}

extern "C" sb_status sb_world_read_rank(sb_world* w, int t, int rank, void* host, int64_t capacity, int64_t* bytes,
                                        sb_stream stream) {
  SB_API_BEGIN
  uint64_t base = 0;
  int64_t n = 0;
  rank_span(w, t, rank, (cudaStream_t)stream, &base, &n);
  if (bytes) *bytes = n;
  if (host) {
    if (capacity < n) throw Error{SB_ERR_CAPACITY, "sb_world_read_rank: host buffer too small"};
    if (n > 0) SB_CUDA(cudaMemcpy(host, reinterpret_cast<void*>(base), (size_t)n, cudaMemcpyDeviceToHost));
  }
  SB_API_END
}

extern "C" sb_status sb_world_write_rank(sb_world* w, int t, int rank, const void* host, int64_t bytes,
                                         sb_stream stream) {
  SB_API_BEGIN
  uint64_t base = 0;
  int64_t n = 0;
  rank_span(w, t, rank, (cudaStream_t)stream, &base, &n);
  if (bytes != n) throw Error{SB_ERR_INTEGRITY, "sb_world_write_rank: byte count does not match the layout"};
  if (n > 0) SB_CUDA(cudaMemcpy(reinterpret_cast<void*>(base), host, (size_t)n, cudaMemcpyHostToDevice));
  SB_API_END
}

extern "C" sb_status sb_copy_timing(sb_planner* p, int op, int64_t* count, double* total_us) {
  SB_API_BEGIN
  if (!p) throw Error{SB_ERR_CONFIG, "null planner"};
  int64_t n = 0;
  double us = 0;
  for (size_t i = 0; i + 1 < p->copy_used; i += 2) {
    if (op >= 0 && p->copy_op[i / 2] != op) continue;
    SB_CUDA(cudaEventSynchronize(p->copy_ev[i + 1]));
    float ms = 0.f;
    SB_CUDA(cudaEventElapsedTime(&ms, p->copy_ev[i], p->copy_ev[i + 1]));
    us += 1000.0 * ms;
    ++n;
  }
  if (count) *count = n;
  if (total_us) *total_us = us;
  SB_API_END
}

extern "C" sb_status sb_copy_timing_reset(sb_planner* p) {
  SB_API_BEGIN
  if (!p) throw Error{SB_ERR_CONFIG, "null planner"};
  p->copy_used = 0;
  SB_API_END
}

extern "C" sb_status sb_last_exchange_bytes(const sb_planner* p, int64_t* bytes_read, int64_t* bytes_written) {
  SB_API_BEGIN
  if (!p) throw Error{SB_ERR_CONFIG, "null planner"};
  int64_t b = 0;
  const int64_t* nj = p->slots[p->last_run_slot].n_jobs;
  if (nj) SB_CUDA(cudaMemcpy(&b, nj + 1, sizeof b, cudaMemcpyDeviceToHost));
  if (bytes_read) *bytes_read = b;
  if (bytes_written) *bytes_written = b;
  SB_API_END
}

// ====================================================================
// Host-buffer entry points used by the C++ drop-in API (include/seqbal/):
// a RoutingPlan that did not come from sb_plan (e.g. user-built or
// deserialised) is uploaded and its chunk rows located on the device; a
// world layout can be set from host row counts; and the reference's
// BlockMove lists (exchange.hpp:86-105) run on the same copy engine.
// ====================================================================
namespace sb {

struct UploadArgs {
  int W;
  int64_t n;
  const int64_t *o_off, *t_off;      // W+1 segment CSR (origin, target)
  const uint64_t *o_id, *t_id;
  const int64_t *o_first, *o_len, *t_first, *t_len;
  const int64_t *o_row, *t_row;      // per-segment row offsets (prefix of lens within rank)
  const uint64_t* c_id;
  const int32_t *c_src, *c_dst;
  const int64_t *c_start, *c_end;
  int64_t *c_src_row, *c_dst_row;
  unsigned long long* first_bad;     // smallest failing chunk index
  int32_t* status;
};

// route's locate (exchange.cpp:156-167): the first segment of the holding
// rank that contains the chunk's token range, on both sides.
__device__ __forceinline__ int64_t locate_row(const int64_t* off, const uint64_t* id, const int64_t* first,
                                              const int64_t* len, const int64_t* row, int rank, uint64_t cid,
                                              int64_t st, int64_t en) {
  for (int64_t s = off[rank]; s < off[rank + 1]; ++s)
    if (id[s] == cid && st >= first[s] && en <= first[s] + len[s]) return row[s] + (st - first[s]);
  return -1;
}

__global__ void k_locate(UploadArgs a) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < a.n; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t st = a.c_start[c], en = a.c_end[c];
    if (en == st) {  // empty transfers are skipped (exchange.cpp:172)
      a.c_src_row[c] = 0;
      a.c_dst_row[c] = 0;
      continue;
    }
    const int64_t sr = locate_row(a.o_off, a.o_id, a.o_first, a.o_len, a.o_row, a.c_src[c], a.c_id[c], st, en);
    const int64_t dr = locate_row(a.t_off, a.t_id, a.t_first, a.t_len, a.t_row, a.c_dst[c], a.c_id[c], st, en);
    if (sr < 0 || dr < 0) {
      atomicOr(a.status, sr < 0 ? 32 : 64);
      atomicMin(a.first_bad, (unsigned long long)c);
    }
    a.c_src_row[c] = sr < 0 ? 0 : sr;
    a.c_dst_row[c] = dr < 0 ? 0 : dr;
  }
}

struct Scratch {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t n) {
    if (n > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      SB_CUDA(cudaMalloc(&p, n));
      cap = n;
    }
    return p;
  }
};

static thread_local Scratch g_move_jobs, g_move_pieces, g_move_n, g_upload, g_bad;

}  // namespace sb

extern "C" sb_status sb_plan_upload(sb_planner* p, int64_t n, const uint64_t* c_id, const int32_t* c_idx,
                                    const int64_t* c_start, const int64_t* c_end, const int32_t* c_src,
                                    const int32_t* c_dst, const int64_t* origin_off, const uint64_t* origin_id,
                                    const int64_t* origin_first, const int64_t* origin_len, const int64_t* target_off,
                                    const uint64_t* target_id, const int64_t* target_first, const int64_t* target_len,
                                    sb_stream stream) {
  SB_API_BEGIN
  if (!p || n < 0) throw Error{SB_ERR_CONFIG, "sb_plan_upload: bad arguments"};
  if (n > p->max_chunks) throw Error{SB_ERR_CAPACITY, "sb_plan_upload: more chunks than planner capacity"};
  const int W = p->W;
  cudaStream_t s = (cudaStream_t)stream;
  for (int64_t c = 0; c < n; ++c)
    if (c_src[c] < 0 || c_src[c] >= W || c_dst[c] < 0 || c_dst[c] >= W || c_end[c] < c_start[c])
      throw Error{SB_ERR_INTEGRITY, "route: chunk " + std::to_string(c) + " has an invalid rank or range"};
  const int64_t so = origin_off[W], sd = target_off[W];
  // per-segment row offsets and per-rank rows, host side (cheap prefix sums)
  std::vector<int64_t> o_row(so), t_row(sd), orows(W), trows(W);
  for (int r = 0; r < W; ++r) {
    int64_t acc = 0;
    for (int64_t q = origin_off[r]; q < origin_off[r + 1]; ++q) { o_row[q] = acc; acc += origin_len[q]; }
    orows[r] = acc;
    acc = 0;
    for (int64_t q = target_off[r]; q < target_off[r + 1]; ++q) { t_row[q] = acc; acc += target_len[q]; }
    trows[r] = acc;
  }
  // one staging allocation for the segment tables
  const size_t segb = sizeof(int64_t) * (size_t)(2 * (W + 1) + 4 * (so + sd)) + sizeof(uint64_t) * (size_t)(so + sd) + 64;
  char* st = static_cast<char*>(sb::g_upload.get(segb));
  auto put = [&](const void* src, size_t bytes) {
    char* at = st;
    if (bytes) SB_CUDA(cudaMemcpyAsync(at, src, bytes, cudaMemcpyHostToDevice, s));
    st += (bytes + 7) & ~size_t(7);
    return at;
  };
  sb::UploadArgs a;
  a.W = W;
  a.n = n;
  a.o_off = (const int64_t*)put(origin_off, sizeof(int64_t) * (W + 1));
  a.t_off = (const int64_t*)put(target_off, sizeof(int64_t) * (W + 1));
  a.o_id = (const uint64_t*)put(origin_id, sizeof(uint64_t) * so);
  a.t_id = (const uint64_t*)put(target_id, sizeof(uint64_t) * sd);
  a.o_first = (const int64_t*)put(origin_first, sizeof(int64_t) * so);
  a.o_len = (const int64_t*)put(origin_len, sizeof(int64_t) * so);
  a.t_first = (const int64_t*)put(target_first, sizeof(int64_t) * sd);
  a.t_len = (const int64_t*)put(target_len, sizeof(int64_t) * sd);
  a.o_row = (const int64_t*)put(o_row.data(), sizeof(int64_t) * so);
  a.t_row = (const int64_t*)put(t_row.data(), sizeof(int64_t) * sd);
  if (n > 0) {
    SB_CUDA(cudaMemcpyAsync(p->c_id, c_id, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, s));
    SB_CUDA(cudaMemcpyAsync(p->c_idx, c_idx, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    SB_CUDA(cudaMemcpyAsync(p->c_start, c_start, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    SB_CUDA(cudaMemcpyAsync(p->c_end, c_end, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    SB_CUDA(cudaMemcpyAsync(p->c_src, c_src, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    SB_CUDA(cudaMemcpyAsync(p->c_dst, c_dst, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
  }
  // keep the origin layout for reverse_plan's receive order (sb_plan_manifests)
  if (so > p->seg_cap || !p->seg_off) {
    cudaFree(p->seg_id);
    cudaFree(p->seg_first);
    cudaFree(p->seg_len);
    if (!p->seg_off) SB_CUDA(cudaMalloc(&p->seg_off, sizeof(int64_t) * (W + 1)));
    const int64_t cap = std::max<int64_t>(1, so);
    SB_CUDA(cudaMalloc(&p->seg_id, sizeof(uint64_t) * cap));
    SB_CUDA(cudaMalloc(&p->seg_first, sizeof(int64_t) * cap));
    SB_CUDA(cudaMalloc(&p->seg_len, sizeof(int64_t) * cap));
    p->seg_cap = cap;
  }
  SB_CUDA(cudaMemcpyAsync(p->seg_off, origin_off, sizeof(int64_t) * (W + 1), cudaMemcpyHostToDevice, s));
  if (so) {
    SB_CUDA(cudaMemcpyAsync(p->seg_id, origin_id, sizeof(uint64_t) * so, cudaMemcpyHostToDevice, s));
    SB_CUDA(cudaMemcpyAsync(p->seg_first, origin_first, sizeof(int64_t) * so, cudaMemcpyHostToDevice, s));
    SB_CUDA(cudaMemcpyAsync(p->seg_len, origin_len, sizeof(int64_t) * so, cudaMemcpyHostToDevice, s));
  }
  SB_CUDA(cudaMemcpyAsync(p->n_chunks, &n, sizeof n, cudaMemcpyHostToDevice, s));
  SB_CUDA(cudaMemcpyAsync(p->origin_rows, orows.data(), sizeof(int64_t) * W, cudaMemcpyHostToDevice, s));
  SB_CUDA(cudaMemcpyAsync(p->target_rows, trows.data(), sizeof(int64_t) * W, cudaMemcpyHostToDevice, s));
  SB_CUDA(cudaMemsetAsync(p->status, 0, sizeof(int32_t), s));
  unsigned long long* bad = static_cast<unsigned long long*>(sb::g_bad.get(sizeof(unsigned long long)));
  SB_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
  a.c_id = p->c_id;
  a.c_src = p->c_src;
  a.c_dst = p->c_dst;
  a.c_start = p->c_start;
  a.c_end = p->c_end;
  a.c_src_row = p->c_src_row;
  a.c_dst_row = p->c_dst_row;
  a.first_bad = bad;
  a.status = p->status;
  if (n > 0) {
    sb::k_locate<<<(int)std::min<int64_t>(1184, (n + 255) / 256), 256, 0, s>>>(a);
    SB_CHECK_LAUNCH();
    sb::count_launch();
  }
  SB_CUDA(cudaStreamSynchronize(s));  // staging tables are reused by the next call
  int32_t stt = 0;
  unsigned long long fb = 0;
  SB_CUDA(cudaMemcpy(&stt, p->status, sizeof stt, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(&fb, bad, sizeof fb, cudaMemcpyDeviceToHost));
  if (stt) {
    const int64_t c = (int64_t)fb;
    throw Error{SB_ERR_INTEGRITY, "route: sample " + std::to_string(c_id[c]) + " chunk [" +
                                      std::to_string(c_start[c]) + "," + std::to_string(c_end[c]) +
                                      ") has no containing " + ((stt & 32) ? "origin" : "target") + " segment"};
  }
  p->identity = false;
  p->uploaded = true;
  SB_API_END
}

extern "C" sb_status sb_world_set_layout(sb_world* w, const int64_t* rows, const int64_t* pitch, sb_stream stream) {
  SB_API_BEGIN
  if (!w || !rows || !pitch) throw Error{SB_ERR_CONFIG, "sb_world_set_layout: null argument"};
  if (w->n_procs != 1) throw Error{SB_ERR_CONFIG, "sb_world_set_layout: single-process worlds only"};
  const int W = w->W, T = w->T;
  std::vector<uint64_t> base((size_t)T * W);
  for (int t = 0; t < T; ++t) {
    int64_t off = 0;
    for (int r = 0; r < W; ++r) {
      const int64_t pt = pitch[(size_t)t * W + r];
      if (rows[r] < 0 || pt < 0) throw Error{SB_ERR_CONFIG, "sb_world_set_layout: negative size"};
      base[(size_t)t * W + r] = (uint64_t)w->arena[t] + (uint64_t)off;
      off += rows[r] * pt;
      if (off > w->arena_bytes[t]) throw Error{SB_ERR_CAPACITY, "world arena too small for the requested layout"};
    }
  }
  std::vector<int32_t> hc(W, 0);
  cudaStream_t s = (cudaStream_t)stream;
  SB_CUDA(cudaMemcpyAsync(w->d_base, base.data(), sizeof(uint64_t) * base.size(), cudaMemcpyHostToDevice, s));
  SB_CUDA(cudaMemcpyAsync(w->d_pitch, pitch, sizeof(int64_t) * (size_t)T * W, cudaMemcpyHostToDevice, s));
  SB_CUDA(cudaMemcpyAsync(w->d_rows, rows, sizeof(int64_t) * W, cudaMemcpyHostToDevice, s));
  SB_CUDA(cudaMemcpyAsync(w->d_headcol, hc.data(), sizeof(int32_t) * W, cudaMemcpyHostToDevice, s));
  SB_CUDA(cudaStreamSynchronize(s));
  SB_API_END
}

extern "C" sb_status sb_world_set_headcol(sb_world* w, const int32_t* headcol, sb_stream stream) {
  SB_API_BEGIN
  if (!w || !headcol) throw Error{SB_ERR_CONFIG, "null argument"};
  SB_CUDA(cudaMemcpyAsync(w->d_headcol, headcol, sizeof(int32_t) * w->W, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  SB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  SB_API_END
}

extern "C" sb_status sb_apply_moves(sb_world* src, sb_world* dst, const sb_block_move* moves, int64_t n,
                                    sb_stream stream) {
  SB_API_BEGIN
  if (!src || !dst || (n > 0 && !moves)) throw Error{SB_ERR_CONFIG, "sb_apply_moves: bad arguments"};
  if (src->W != dst->W || src->T < 2 || dst->T < 2) throw Error{SB_ERR_CONFIG, "sb_apply_moves: incompatible worlds"};
  cudaStream_t s = (cudaStream_t)stream;
  const int W = src->W;
  std::vector<uint64_t> sb0(W), sb1(W), db0(W), db1(W);
  std::vector<int64_t> sp0(W), sp1(W), dp0(W), dp1(W), srows(W), drows(W);
  SB_CUDA(cudaStreamSynchronize(s));
  SB_CUDA(cudaMemcpy(sb0.data(), src->d_base, sizeof(uint64_t) * W, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(sb1.data(), src->d_base + W, sizeof(uint64_t) * W, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(db0.data(), dst->d_base, sizeof(uint64_t) * W, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(db1.data(), dst->d_base + W, sizeof(uint64_t) * W, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(sp0.data(), src->d_pitch, sizeof(int64_t) * W, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(sp1.data(), src->d_pitch + W, sizeof(int64_t) * W, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(dp0.data(), dst->d_pitch, sizeof(int64_t) * W, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(dp1.data(), dst->d_pitch + W, sizeof(int64_t) * W, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(srows.data(), src->d_rows, sizeof(int64_t) * W, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(drows.data(), dst->d_rows, sizeof(int64_t) * W, cudaMemcpyDeviceToHost));
  std::vector<SbJob> jobs;
  jobs.reserve((size_t)n * 2);
  for (int64_t i = 0; i < n; ++i) {
    const sb_block_move& m = moves[i];
    if (m.src_rank < 0 || m.src_rank >= W || m.dst_rank < 0 || m.dst_rank >= W || m.n_rows < 0 ||
        m.src_row < 0 || m.dst_row < 0 || m.src_row + m.n_rows > srows[m.src_rank] ||
        m.dst_row + m.n_rows > drows[m.dst_rank] || m.src_col_bytes < 0 || m.dst_col_bytes < 0 ||
        m.src_col_bytes + m.n_col_bytes > sp1[m.src_rank] || m.dst_col_bytes + m.n_col_bytes > dp1[m.dst_rank])
      throw Error{SB_ERR_INTEGRITY, "apply_block_moves: move " + std::to_string(i) + " outside its buffers"};
    SbJob j;
    j.src = sb1[m.src_rank] + (uint64_t)(m.src_row * sp1[m.src_rank] + m.src_col_bytes);
    j.dst = db1[m.dst_rank] + (uint64_t)(m.dst_row * dp1[m.dst_rank] + m.dst_col_bytes);
    j.n_rows = m.n_rows;
    j.width = m.n_col_bytes;
    j.spitch = sp1[m.src_rank];
    j.dpitch = dp1[m.dst_rank];
    jobs.push_back(j);
    if (m.copy_meta) {
      SbJob k;
      k.src = sb0[m.src_rank] + (uint64_t)(m.src_row * sp0[m.src_rank]);
      k.dst = db0[m.dst_rank] + (uint64_t)(m.dst_row * dp0[m.dst_rank]);
      k.n_rows = m.n_rows;
      k.width = 16;
      k.spitch = sp0[m.src_rank];
      k.dpitch = dp0[m.dst_rank];
      jobs.push_back(k);
    }
  }
  const int64_t nj = (int64_t)jobs.size();
  SbJob* dj = static_cast<SbJob*>(sb::g_move_jobs.get(sizeof(SbJob) * (size_t)std::max<int64_t>(1, nj)));
  int64_t* dpo = static_cast<int64_t*>(sb::g_move_pieces.get(sizeof(int64_t) * (size_t)(nj + 1)));
  int64_t* dn = static_cast<int64_t*>(sb::g_move_n.get(sizeof(int64_t) * 2));
  if (nj) SB_CUDA(cudaMemcpyAsync(dj, jobs.data(), sizeof(SbJob) * nj, cudaMemcpyHostToDevice, s));
  SB_CUDA(cudaMemcpyAsync(dn, &nj, sizeof nj, cudaMemcpyHostToDevice, s));
  sb::k_pieces<<<1, 1024, 0, s>>>(dj, dn, dpo, dn + 1);
  SB_CHECK_LAUNCH();
  sb::k_copy<1><<<sb::copy_grid(), sb::kCopyThreads, 0, s>>>(dj, dpo, dn, 0);
  SB_CHECK_LAUNCH();
  sb::count_launch(2);
  SB_CUDA(cudaStreamSynchronize(s));  // host job vector and staging are reused
  SB_API_END
}

// =============================================== uniform (T5) balancer
// balance_uniform_items / reverse_uniform_plan (balancer.cpp:411-462): the
// appendix's balancer for identical-cost items (T5 text strings).  Plan on
// the device (one CTA), then the items move with the same copy engines as
// route.  The reference defines counts and moves only; the item layout the
// exchange realises (documented in DESIGN.md): a surplus rank keeps its
// first final_count items and sends the rest, in order, along its moves in
// move order; a deficit rank appends what it receives after its own items in
// move order.  The reverse exchange is the exact inverse.
struct sb_uniform {
  int W = 0;
  int64_t* counts = nullptr;  // W   (copy of the planned counts)
  int64_t* final_ = nullptr;  // W
  int64_t* mv = nullptr;      // 5 * 2W: src, dst, count, src item offset, dst item offset
  int64_t* hdr = nullptr;     // [0] moves, [1] total moved, [2] status
  int64_t* rows = nullptr;    // 2W: destination / expected source rows of the current exchange
  SbJob* jobs = nullptr;
  int64_t* piece_off = nullptr;
  int64_t* n_jobs = nullptr;  // [0] jobs, [1] bytes
  int64_t job_cap = 0;
};

namespace sb {

__global__ void __launch_bounds__(1024) k_uniform_plan(const int64_t* __restrict__ counts_in, int W, int64_t* counts,
                                                       int64_t* fin, int64_t* mv, int64_t* hdr) {
  __shared__ int64_t sh[33];
  __shared__ int64_t s_base, s_rem;
  int64_t local = 0;
  int neg = 0;
  for (int r = threadIdx.x; r < W; r += blockDim.x) {
    const int64_t c = counts_in[r];
    counts[r] = c;
    neg |= c < 0;
    local += c;
  }
  int64_t total;
  block_excl_scan<int64_t>(local, sh, &total);
  neg = __syncthreads_or(neg);
  if (threadIdx.x == 0) {
    s_base = total / W;
    s_rem = total % W;
    hdr[2] = neg;  // ConfigError: balance_uniform_items: negative count
  }
  __syncthreads();
  // +1 slots to the largest counts, ties toward the lower rank
  // (std::stable_sort by count desc): rank r's position in that order
  for (int r = threadIdx.x; r < W; r += blockDim.x) {
    const int64_t c = counts[r];
    int pos = 0;
    for (int q = 0; q < W; ++q) pos += (counts[q] > c) || (counts[q] == c && q < r);
    fin[r] = s_base + (pos < s_rem ? 1 : 0);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // pair surpluses with deficits in rank order (two cursors)
  int si = 0, di = 0, n = 0;
  int64_t moved_total = 0, s_left = 0, d_left = 0, s_sent = 0, d_got = 0;
  auto next_s = [&](int from) {
    for (int r = from; r < W; ++r)
      if (counts[r] - fin[r] > 0) return r;
    return W;
  };
  auto next_d = [&](int from) {
    for (int r = from; r < W; ++r)
      if (counts[r] - fin[r] < 0) return r;
    return W;
  };
  si = next_s(0);
  di = next_d(0);
  if (si < W) s_left = counts[si] - fin[si];
  if (di < W) d_left = fin[di] - counts[di];
  while (si < W && di < W) {
    const int64_t m = s_left < d_left ? s_left : d_left;
    mv[5 * n + 0] = si;
    mv[5 * n + 1] = di;
    mv[5 * n + 2] = m;
    mv[5 * n + 3] = fin[si] + s_sent;   // first item leaving si
    mv[5 * n + 4] = counts[di] + d_got;  // first free slot on di
    ++n;
    moved_total += m;
    s_left -= m;
    d_left -= m;
    s_sent += m;
    d_got += m;
    if (s_left == 0) {
      si = next_s(si + 1);
      s_sent = 0;
      if (si < W) s_left = counts[si] - fin[si];
    }
    if (d_left == 0) {
      di = next_d(di + 1);
      d_got = 0;
      if (di < W) d_left = fin[di] - counts[di];
    }
  }
  hdr[0] = n;
  hdr[1] = moved_total;
}

// One CTA prepares a uniform exchange: destination rows, the destination
// layout (with the source-layout check), the item jobs and the piece scan.
__global__ void __launch_bounds__(1024) k_uniform_prep(const int64_t* counts, const int64_t* fin, const int64_t* mv,
                                                       const int64_t* hdr, int W, int64_t rpi, int reverse,
                                                       WorldArgs s, WorldArgs d, TensorInfo ti, int64_t* rows,
                                                       SbJob* jobs, int64_t* n_jobs, int64_t* piece_off) {
  for (int r = threadIdx.x; r < W; r += blockDim.x) {
    rows[r] = (reverse ? counts[r] : fin[r]) * rpi;      // destination
    rows[W + r] = (reverse ? fin[r] : counts[r]) * rpi;  // expected source
  }
  __syncthreads();
  LayoutPlan lp{};
  lp.rows_src = rows;
  lp.expect_rows = rows + W;
  layout_tensor(d, s, lp, ti, 0, threadIdx.x >> 5);
  __syncthreads();
  const int T = s.T;
  const int64_t total = (int64_t)3 * W * T;
  if (threadIdx.x == 0) *n_jobs = total;
  const bool bad = (*d.status & ST_MISMATCH) != 0;
  for (int64_t x = threadIdx.x; x < total; x += blockDim.x) {
    const int t = (int)(x % T);
    const int64_t e = x / T;
    SbJob j;
    j.src = j.dst = 0;
    j.n_rows = 0;
    j.width = ti.row_bytes[t];
    int sr = 0, dr = 0;
    int64_t srow = 0, drow = 0, n = 0;
    if (e < W) {  // items that stay: the first min(count, final) of the rank
      sr = dr = (int)e;
      const int64_t keep = counts[e] < fin[e] ? counts[e] : fin[e];
      n = keep * rpi;
    } else if (e - W < hdr[0]) {
      const int64_t* m = mv + 5 * (e - W);
      if (!reverse) {
        sr = (int)m[0];
        dr = (int)m[1];
        srow = m[3] * rpi;
        drow = m[4] * rpi;
      } else {
        sr = (int)m[1];
        dr = (int)m[0];
        srow = m[4] * rpi;
        drow = m[3] * rpi;
      }
      n = m[2] * rpi;
    }
    if (n > 0 && !bad && is_local(s, sr)) {
      const int64_t sp = s.pitch[t * s.W + sr], dp = d.pitch[t * d.W + dr];
      j.src = s.base[t * s.W + sr] + (uint64_t)(srow * sp);
      j.dst = d.base[t * d.W + dr] + (uint64_t)(drow * dp);
      j.n_rows = n;
      j.spitch = sp;
      j.dpitch = dp;
    } else {
      j.spitch = j.dpitch = j.width;
    }
    jobs[x] = j;
  }
  __syncthreads();
  pieces_body(jobs, n_jobs, piece_off, n_jobs + 1);
}

}  // namespace sb

extern "C" sb_status sb_uniform_create(int world, sb_uniform** out) {
  SB_API_BEGIN
  if (!out || world < 1) throw Error{SB_ERR_CONFIG, "sb_uniform_create: world must be >= 1"};
  *out = nullptr;
  sb_uniform* u = new sb_uniform();
  u->W = world;
  try {
    SB_CUDA(cudaMalloc(&u->counts, sizeof(int64_t) * world));
    SB_CUDA(cudaMalloc(&u->final_, sizeof(int64_t) * world));
    SB_CUDA(cudaMalloc(&u->mv, sizeof(int64_t) * 5 * 2 * world));
    SB_CUDA(cudaMalloc(&u->hdr, sizeof(int64_t) * 3));
    SB_CUDA(cudaMemset(u->hdr, 0, sizeof(int64_t) * 3));
    SB_CUDA(cudaMalloc(&u->rows, sizeof(int64_t) * 2 * world));
    SB_CUDA(cudaMalloc(&u->n_jobs, sizeof(int64_t) * 2));
  } catch (...) {
    sb_uniform_destroy(u);
    throw;
  }
  *out = u;
  SB_API_END
}

extern "C" sb_status sb_uniform_destroy(sb_uniform* u) {
  if (!u) return SB_OK;
  void* ptrs[] = {u->counts, u->final_, u->mv, u->hdr, u->rows, u->jobs, u->piece_off, u->n_jobs};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  delete u;
  return SB_OK;
}

extern "C" sb_status sb_uniform_plan(sb_uniform* u, const int64_t* d_counts, sb_stream stream) {
  SB_API_BEGIN
  if (!u || !d_counts) throw Error{SB_ERR_CONFIG, "sb_uniform_plan: null argument"};
  sb::k_uniform_plan<<<1, 1024, 0, (cudaStream_t)stream>>>(d_counts, u->W, u->counts, u->final_, u->mv, u->hdr);
  SB_CHECK_LAUNCH();
  sb::count_launch();
  SB_API_END
}

extern "C" sb_status sb_uniform_download(sb_uniform* u, int64_t* final_counts, int64_t* moves3, int64_t* n_moves,
                                         int64_t* total_moved, sb_stream stream) {
  SB_API_BEGIN
  if (!u) throw Error{SB_ERR_CONFIG, "null uniform plan"};
  cudaStream_t s = (cudaStream_t)stream;
  SB_CUDA(cudaStreamSynchronize(s));
  int64_t hdr[3];
  SB_CUDA(cudaMemcpy(hdr, u->hdr, sizeof hdr, cudaMemcpyDeviceToHost));
  if (hdr[2]) throw Error{SB_ERR_CONFIG, "balance_uniform_items: negative count"};
  if (final_counts) SB_CUDA(cudaMemcpy(final_counts, u->final_, sizeof(int64_t) * u->W, cudaMemcpyDeviceToHost));
  if (moves3 && hdr[0] > 0) {
    std::vector<int64_t> mv((size_t)(5 * hdr[0]));
    SB_CUDA(cudaMemcpy(mv.data(), u->mv, sizeof(int64_t) * mv.size(), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < hdr[0]; ++i)
      for (int k = 0; k < 3; ++k) moves3[3 * i + k] = mv[(size_t)(5 * i + k)];
  }
  if (n_moves) *n_moves = hdr[0];
  if (total_moved) *total_moved = hdr[1];
  SB_API_END
}

// Moves the items of the current uniform plan: forward (reverse == 0) from
// the counts layout to the balanced one, or back (reverse_uniform_plan).
// Every rank's tensor rows are items x rows_per_item.
extern "C" sb_status sb_uniform_route(sb_uniform* u, int reverse, int64_t rows_per_item, sb_world* src, sb_world* dst,
                                      sb_stream stream) {
  SB_API_BEGIN
  if (!u || !src || !dst) throw Error{SB_ERR_CONFIG, "sb_uniform_route: null argument"};
  if (src == dst) throw Error{SB_ERR_CONFIG, "sb_uniform_route is out-of-place: src and dst must differ"};
  if (rows_per_item < 1) throw Error{SB_ERR_CONFIG, "rows_per_item must be >= 1"};
  if (src->W != u->W || dst->W != u->W || src->T != dst->T)
    throw Error{SB_ERR_CONFIG, "sb_uniform_route: world shape differs from the plan"};
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t cap = (int64_t)3 * u->W * src->T;
  if (cap > u->job_cap) {
    if (u->jobs) cudaFree(u->jobs);
    if (u->piece_off) cudaFree(u->piece_off);
    u->jobs = nullptr;
    u->piece_off = nullptr;
    SB_CUDA(cudaMalloc(&u->jobs, sizeof(SbJob) * (size_t)cap));
    SB_CUDA(cudaMalloc(&u->piece_off, sizeof(int64_t) * (size_t)(cap + 1)));
    u->job_cap = cap;
  }
  sb::k_uniform_prep<<<1, 1024, 0, s>>>(u->counts, u->final_, u->mv, u->hdr, u->W, rows_per_item, reverse ? 1 : 0,
                                        sb::wargs(src), sb::wargs(dst), sb::tinfo(src), u->rows, u->jobs, u->n_jobs,
                                        u->piece_off);
  SB_CHECK_LAUNCH();
  sb::count_launch(1);
  bool tma_ok = true;
  for (int64_t rb : src->row_bytes) tma_ok &= rb % 16 == 0;
  sb::launch_copy(u->jobs, u->piece_off, u->n_jobs, s, dst->n_procs > 1, tma_ok, sb::route_engine());
  SB_API_END
}
