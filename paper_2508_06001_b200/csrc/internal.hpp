// Host-side objects behind the opaque C-ABI handles.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"
#include "seqbal_capi.h"

// One copy job: n_rows rows of `width` bytes from src (row pitch spitch) to
// dst (row pitch dpitch).  Built on the device from a plan.
struct SbJob {
  uint64_t src;
  uint64_t dst;
  int64_t n_rows;
  int64_t width;
  int64_t spitch;
  int64_t dpitch;
};

struct sb_planner {
  int W = 0, U = 0, M = 0, R = 0;
  int d_model = 0, n_heads = 0, d_head = 0, n_blocks = 0;
  double gamma = 0, k = 0;
  int64_t max_seqs = 0, max_chunks = 0;
  int max_bag = 1;
  std::vector<int32_t> bag_off, bag_ranks, bag_size, rank_bag, rank_member;
  bool identity = false;
  bool any_multi_bag = false;
  bool uploaded = false;  // current plan came from sb_plan_upload (no bag tables)
  int path = 0;           // planner pipeline: 0 auto, 1 single-CTA small, 2 multi-kernel, 3 hybrid
  int last_path = 0;      // what the last sb_plan ran: 1 single-CTA, 2 multi-kernel, 3 hybrid
  long long* trace = nullptr;  // per-phase clock64 stamps of the fused planner (diagnostics)
  size_t small_smem = 0;  // dynamic shared memory of the small path
  // origin layout of an uploaded plan (segment CSR), kept for reverse_plan
  int64_t seg_cap = 0;
  int64_t* seg_off = nullptr;  // W+1
  uint64_t* seg_id = nullptr;
  int64_t* seg_first = nullptr;
  int64_t* seg_len = nullptr;

  // constant topology tables (device)
  int32_t *d_bag_off = nullptr, *d_bag_ranks = nullptr, *d_bag_size = nullptr;
  int32_t *d_rank_bag = nullptr, *d_rank_member = nullptr;

  // inputs of the last plan (device, caller-owned)
  const uint64_t* ids = nullptr;
  const int64_t* lens = nullptr;
  const int64_t* rank_off = nullptr;
  const double* w_in = nullptr;  // assign_to_bags mode: caller workloads
  uint64_t* stage_ids = nullptr;  // staging for host-array entry points
  int64_t* stage_lens = nullptr;
  double* stage_w = nullptr;
  int64_t* stage_off = nullptr;

  // per-sequence scratch (max_seqs)
  double* w = nullptr;
  int32_t* seq_rank = nullptr;
  int64_t* seq_off = nullptr;
  uint64_t* hash = nullptr;  // 2*max_seqs
  uint64_t *sk_hi = nullptr, *sk_lo = nullptr, *tk_hi = nullptr, *tk_lo = nullptr;
  uint32_t *sk_v = nullptr, *tk_v = nullptr;
  double* sorted_w = nullptr;
  int32_t* sorted_idx = nullptr;
  int32_t* pick = nullptr;
  int32_t* seq_bag = nullptr;
  int32_t* greedy_q = nullptr;  // hybrid path: rank of each greedy position inside its bag
  int32_t* seq_G = nullptr;
  int64_t* seq_chunk_base = nullptr;

  // per replica / bag / rank
  double* rep_total = nullptr;       // R
  int32_t* sentinel = nullptr;       // R
  int32_t* bag_count = nullptr;      // R*M
  int64_t* bag_rows = nullptr;       // R*M
  int64_t* rep_chunks = nullptr;     // R
  int64_t* rep_cbase = nullptr;      // R+1
  int32_t* bag_seq = nullptr;        // max_seqs
  int32_t* tile_cnt = nullptr;       // R * ceil(max_seqs / 1024) * M: emission tile bag counts
  int64_t* list_sum = nullptr;       // W * ceil(max_seqs / 1024) * 4: manifest tile sums
  int32_t* list_tie = nullptr;       // W: reverse-order tie flags
  int64_t* bag_cbase = nullptr;      // R*M: first chunk of (replica, bag) within the replica
  int64_t* bag_sbase = nullptr;      // R*M: first bag_seq slot of (replica, bag)
  unsigned long long* send_count = nullptr;  // W
  unsigned long long* recv_count = nullptr;  // W (generic manifests)
  // chunk-sized sort scratch for the generic reverse order (lazy)
  uint64_t *ck_hi = nullptr, *ck_lo = nullptr, *ck_thi = nullptr, *ck_tlo = nullptr;
  uint32_t *ck_v = nullptr, *ck_tv = nullptr;

  // pinned host scalars for read-backs: [0] status (int32), [1] n_chunks, [2] n_seqs
  int64_t* h_small = nullptr;

  // plan (device)
  int64_t* n_chunks = nullptr;
  int64_t* n_seqs = nullptr;
  uint64_t* c_id = nullptr;
  int32_t *c_idx = nullptr, *c_src = nullptr, *c_dst = nullptr;
  int64_t *c_start = nullptr, *c_end = nullptr, *c_src_row = nullptr, *c_dst_row = nullptr;
  int64_t* c_seq_base = nullptr;  // per chunk (q,0): row base of the sequence in its bag's full layout
  int32_t* c_seq = nullptr;       // per chunk: gather index of its sequence (reverse-order ties)
  int64_t *send_off = nullptr, *recv_off = nullptr;
  int32_t *send_idx = nullptr, *recv_idx = nullptr, *rev_recv_idx = nullptr;
  int64_t *origin_rows = nullptr, *target_rows = nullptr;
  double *per_gpu = nullptr, *per_bag_occ = nullptr, *total = nullptr, *wir = nullptr;
  int32_t* violations = nullptr;
  int32_t* status = nullptr;

  // Exchange slots: a prepared exchange (destination layout written, copy
  // jobs + piece scan in the slot's buffers) waiting to run.  Preparation can
  // run on another stream ahead of the copy (sb_exchange_prepare/run).
  struct Slot {
    SbJob* jobs = nullptr;
    int64_t* piece_off = nullptr;
    int64_t* n_jobs = nullptr;  // [0] jobs, [1] bytes moved (one way)
    int64_t cap = 0;
    bool prepared = false, pieces_done = false, tma_ok = false;
    int fence_sys = 0, engine = 0, op = 0;
  };
  static constexpr int kSlots = 8;
  Slot slots[kSlots];
  // collective transport (sb_exchange_pack / _unpack): the full job list's
  // (source process << 16 | destination process) per job, and the unpack list
  bool coll_mode = false;  // job builders emit every chunk's jobs + owners
  int32_t* x_owner = nullptr;
  int64_t x_owner_cap = 0;
  Slot unpack;
  int unpack_op = -1;
  int cur_slot = 0, last_run_slot = 0;
  // current slot's buffers (aliases of slots[cur_slot])
  SbJob* jobs = nullptr;
  int64_t* piece_off = nullptr;
  int64_t* n_jobs = nullptr;
  int64_t job_cap = 0;
  int64_t last_bytes_read = 0, last_bytes_written = 0;

  // copy-kernel event pairs recorded while timing is on: (start, stop, op)
  std::vector<cudaEvent_t> copy_ev;
  std::vector<int> copy_op;
  size_t copy_used = 0;
  int current_op = 0;

  // side stream for work that overlaps the main planner chain (serial totals)
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  cudaEvent_t gfork_ev = nullptr, gjoin_ev = nullptr;  // single-bag greedy chain (overlaps emission)
  cudaEvent_t dup_ev = nullptr;                         // multi-kernel duplicate-id check (side stream)

  // timing
  bool timing = false;
  cudaEvent_t ev[6] = {};
  float last_ms[5] = {};
};

struct sb_world {
  int W = 0, n_local = 0, first_local = 0, n_heads = 0, n_payload = 0, n_aux = 0, T = 0, max_bag = 1;
  int n_procs = 1;
  int64_t capacity_rows = 0;
  std::vector<int64_t> row_bytes;    // T (tensor 0 = 16-byte metadata)
  std::vector<void*> arena;          // T
  std::vector<int64_t> arena_bytes;  // T
  uint64_t* d_base = nullptr;        // T*W
  int64_t* d_pitch = nullptr;        // T*W
  int64_t* d_rows = nullptr;         // W
  int32_t* d_headcol = nullptr;      // W: first global payload column held (doubles)
  uint64_t* d_peer_arena = nullptr;  // T*n_procs
  int64_t* d_arena_bytes = nullptr;  // T
  int32_t* d_status = nullptr;
  std::vector<int64_t> tensor_desc;  // flags: 0 meta, 1 payload, 2 aux
};

namespace sb {
void ensure_jobs(sb_planner* p, int64_t cap);
// A second planner with p's topology, model and capacity (fresh device
// scratch; the plan-ahead driver alternates two of them).
sb_planner* planner_clone(const sb_planner* p);
}
