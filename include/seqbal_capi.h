/*
 * seqbal_capi.h -- C-ABI of libseqbal_cuda.so, the B200-native
 * balance-and-redistribute path (KnapFormer, arXiv 2508.06001).
 *
 * Plain C: integers, pointers and sizes only; no CUDA, torch or C++ types in
 * any signature (a stream is passed as an opaque pointer, i.e. a
 * cudaStream_t).  Every call returns an sb_status; on failure
 * sb_last_error() holds a thread-local message.  Status values mirror the
 * reference's exception classes (/root/reference/proj/include/seqbal/error.hpp)
 * and the CLI exit-code mapping (proj/tools/main.cpp:369-387):
 *   SB_ERR_CONFIG    <-> ConfigError    (error.hpp:24-27)
 *   SB_ERR_INTEGRITY <-> IntegrityError (error.hpp:31-34)
 *   SB_ERR_PARSE     <-> ParseError     (error.hpp:10-21)
 *
 * The C++ host API in include/seqbal/*.hpp (same names and signatures as the
 * reference headers) is layered on these entry points; INTEGRATION.md shows
 * the binding a reference maintainer would add.
 *
 * Everything device-side is asynchronous and stream-ordered: a plan computed
 * by sb_plan() lives in device memory owned by the planner and is consumed by
 * sb_route()/sb_pre_attn()/... without a host round trip, so a whole step
 * can be captured in one CUDA graph.  Only the *_download / *_status calls
 * synchronise.
 */
#ifndef SEQBAL_CAPI_H
#define SEQBAL_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SB_API __attribute__((visibility("default")))
#else
#define SB_API
#endif

typedef int sb_status;
enum {
  SB_OK = 0,
  SB_ERR_CONFIG = 1,    /* ConfigError */
  SB_ERR_INTEGRITY = 2, /* IntegrityError */
  SB_ERR_PARSE = 3,     /* ParseError */
  SB_ERR_CAPACITY = 4,  /* a caller-sized buffer/capacity was too small */
  SB_ERR_CUDA = 5,      /* CUDA runtime failure (no device, launch failure, ...) */
  SB_ERR_COMM = 6       /* peer-memory / multi-process exchange failure */
};

typedef void* sb_stream; /* cudaStream_t; NULL = legacy default stream */

SB_API const char* sb_last_error(void);
SB_API int sb_abi_version(void);
/* Number of CUDA kernels this library has launched in this process (the
 * bench's gpu_launches evidence). */
SB_API int64_t sb_kernel_launches(void);

/* ------------------------------------------------------------ planner -- */
/* Replaces plan_routing / identity_plan / reverse_plan
 * (proj/include/seqbal/balancer.hpp:95-104) and gamma_weighted_workload
 * (workload_model.hpp:63).  One planner per (model, topology, world).       */
typedef struct sb_planner sb_planner;

typedef struct sb_planner_desc {
  int world_size;            /* W: global ranks (WorldLayout::world_size)          */
  int unit_size;             /* ranks per replica (Topology::unit_size)            */
  int n_bags;                /* bags per replica (Topology::bags.size())           */
  const int32_t* bag_offsets;/* host, n_bags+1: CSR into bag_ranks                 */
  const int32_t* bag_ranks;  /* host, unit-local ranks of each bag (ComputeBag)    */
  int d_model, n_heads, d_head, n_blocks; /* ModelShape (workload_model.hpp:13-24) */
  double gamma;              /* WorkloadModel::gamma                               */
  double k;                  /* WorkloadModel::k (validated only)                  */
  int64_t max_seqs;          /* capacity: sequences over all ranks                 */
} sb_planner_desc;

/* Validates like WorkloadModel::validate (workload_model.cpp:15-31),
 * replicate (topology.cpp:81-93) and plan_routing's head check
 * (balancer.cpp:114-120); SB_ERR_CONFIG with the reference's message.
 * Limits: at most 1024 bags per replica (SB_ERR_CONFIG "more than 1024 bags
 * per replica"; the reference has none; above 64 the multi-kernel path runs).  All four shape fields 0 create an
 * assignment-only planner for sb_assign_to_bags (no model, no head check);
 * sb_plan / sb_plan_identity refuse it. */
SB_API sb_status sb_planner_create(const sb_planner_desc* desc, sb_planner** out);
SB_API sb_status sb_planner_destroy(sb_planner* p);

/* Metadata all-gather result in gather order (exchange.cpp:68-77): rank r's
 * sequences are [rank_off[r], rank_off[r+1]).  All three arrays are DEVICE
 * pointers.  Computes the plan on the device (no host synchronisation). */
SB_API sb_status sb_plan(sb_planner* p, const uint64_t* d_ids, const int64_t* d_lens,
                  const int64_t* d_rank_off, sb_stream stream);
/* identity_plan (balancer.cpp:227-240) into the same planner slots. */
SB_API sb_status sb_plan_identity(sb_planner* p, const uint64_t* d_ids, const int64_t* d_lens,
                           const int64_t* d_rank_off, sb_stream stream);

/* Device view of the current plan.  Counts live in device memory; arrays are
 * sized for the planner's capacity. */
typedef struct sb_plan_dev {
  int world_size;
  int64_t max_chunks;
  const int64_t* n_chunks;      /* device scalar                                   */
  const uint64_t* chunk_id;     /* ChunkAssignment SoA (balancer.hpp:38-47)        */
  const int32_t* chunk_index;
  const int64_t* chunk_start;
  const int64_t* chunk_end;
  const int32_t* chunk_src;
  const int32_t* chunk_dst;
  const int64_t* chunk_src_row; /* row of the chunk's first token in origin packing */
  const int64_t* chunk_dst_row; /* row in target packing                           */
  const int64_t* send_off;      /* W+1: RoutingPlan::send as CSR                   */
  const int32_t* send_idx;
  const int64_t* recv_off;      /* W+1: RoutingPlan::recv                          */
  const int32_t* recv_idx;
  const int32_t* rev_recv_idx;  /* reverse_plan(plan).recv; offsets = send_off     */
  const int64_t* origin_rows;   /* W: rows per rank before the exchange            */
  const int64_t* target_rows;   /* W: rows per rank after                          */
  const double* per_gpu_workload;  /* BalanceReport (balancer.hpp:78-84)           */
  const double* per_bag_occupancy; /* replicas * n_bags                            */
  const int32_t* capacity_violations;
  const double* total_workload;
  const double* wir;
  const int32_t* status;        /* device error word (0 = ok)                      */
} sb_plan_dev;
SB_API sb_status sb_plan_get(const sb_planner* p, sb_plan_dev* out);

/* Synchronises `stream`, checks the device status word and returns the plan
 * sizes.  n_seqs is the sequence count the plan was built from. */
SB_API sb_status sb_plan_sizes(sb_planner* p, sb_stream stream, int64_t* n_chunks, int64_t* n_seqs);

/* Host copy of the plan (caller-allocated arrays; NULL entries are skipped). */
typedef struct sb_plan_host {
  uint64_t* chunk_id;
  int32_t* chunk_index;
  int64_t* chunk_start;
  int64_t* chunk_end;
  int32_t* chunk_src;
  int32_t* chunk_dst;
  int64_t* send_off;     /* W+1 */
  int32_t* send_idx;     /* n_chunks */
  int64_t* recv_off;     /* W+1 */
  int32_t* recv_idx;     /* n_chunks */
  int32_t* rev_recv_idx; /* n_chunks */
  int64_t* target_rows;  /* W */
  double* per_gpu_workload;  /* W */
  double* per_bag_occupancy; /* replicas * n_bags */
  int32_t capacity_violations;
  double total_workload;
  double wir;
} sb_plan_host;
SB_API sb_status sb_plan_download(sb_planner* p, sb_plan_host* out, sb_stream stream);

/* Planner pipeline: 0 = auto (by capacity: the single-CTA fused planner for
 * small batches, the hybrid -- fused prefix with the greedy (one replica) or
 * the 32-thread greedy kernel (several), fused suffix as a programmatic
 * dependent launch -- for 256-1152
 * sequences, else the multi-kernel pipeline), 1 = force
 * the fused planner, 2 = force the multi-kernel pipeline, 3 = force the
 * hybrid.  All are bit-exact. */
SB_API sb_status sb_planner_set_path(sb_planner* p, int path);
/* The pipeline the last sb_plan ran: 1 fused, 2 multi-kernel, 3 hybrid. */
SB_API sb_status sb_planner_last_path(sb_planner* p, int* path);
/* Self-test: the planner's fast correctly-rounded division against
 * __ddiv_rn on n random operand pairs; *mismatches must be 0. */
SB_API sb_status sb_selftest_div(int64_t n, uint64_t seed, int64_t* mismatches);
/* Self-test: the planner's block-parallel serial FP64 sum (serial_sum.cuh)
 * against the one-thread chain, `blocks` sums of 1..max_len generated values
 * of law `mode` (0..6), result and every prefix; *mismatches must be 0. */
SB_API sb_status sb_selftest_serial_sum(int64_t blocks, int64_t max_len, uint64_t seed, int mode,
                                        int64_t* mismatches);
/* Diagnostics: per-phase clock64() stamps of the fused planner (16 slots). */
SB_API sb_status sb_planner_trace(sb_planner* p, int enable, int64_t* out16);

/* Plan latency breakdown of the last sb_plan (device time, microseconds,
 * measured with events when timing is enabled; zeros otherwise). */
SB_API sb_status sb_planner_enable_timing(sb_planner* p, int enable);
SB_API sb_status sb_planner_timing(sb_planner* p, double* us_prep, double* us_sort, double* us_greedy,
                            double* us_emit, double* us_lists);

/* -------------------------------------------------------------- world -- */
/* Device-resident rank buffers (RankBuffer, exchange.hpp:22-44) laid out for
 * HBM: one arena per tensor, ranks packed back to back, plus per-rank tables
 * (row count, base pointer, row pitch) that the kernels read.  Tensor 0 is
 * the 16-byte row metadata {uint64 sample_id, int64 position}; tensors
 * 1..n_payload are head-sliced payloads (hidden states, q/k/v ...); the
 * remaining n_aux tensors are whole-row auxiliaries (e.g. RoPE ids). */
typedef struct sb_world sb_world;

typedef struct sb_world_desc {
  int world_size;          /* global ranks W                                    */
  int n_local;             /* ranks hosted by this process                      */
  int first_local;         /* global rank of the first hosted rank              */
  int n_heads;             /* World::n_heads                                    */
  int n_payload;           /* >= 1 head-sliced tensors                          */
  int n_aux;               /* whole-row tensors besides the metadata            */
  const int64_t* row_bytes;/* n_payload + n_aux full-width row sizes            */
  int64_t capacity_rows;   /* rows per tensor arena (all hosted ranks)          */
  int max_bag;             /* largest bag size (sizes the metadata arena)       */
} sb_world_desc;

SB_API sb_status sb_world_create(const sb_world_desc* desc, sb_world** out);
SB_API sb_status sb_world_destroy(sb_world* w);
/* Arena base of tensor t (0 = metadata) -- for peer export / host copies. */
SB_API sb_status sb_world_arena(const sb_world* w, int tensor, void** base, int64_t* bytes);
/* Per-rank tables (device pointers, W entries). */
SB_API sb_status sb_world_tables(const sb_world* w, int tensor, const uint64_t** d_base,
                          const int64_t** d_pitch, const int64_t** d_rows);
/* Multi-process: arena bases of every process's world for tensor t
 * (peer-mapped device pointers), index = process; n_procs = W / n_local.   */
SB_API sb_status sb_world_set_peers(sb_world* w, int tensor, const uint64_t* host_bases, int n_procs);

/* Origin layout from gathered metadata: rank r holds its sequences packed in
 * gather order (exchange.cpp:31-66 shells).  Device arrays as in sb_plan. */
SB_API sb_status sb_world_layout_origin(sb_world* w, const int64_t* d_lens, const int64_t* d_rank_off,
                                 sb_stream stream);
/* Layout from the current plan of `p` (no data moved): 0 origin packing,
 * 1 target (chunk) packing -- what route writes --, 2 Ulysses packing --
 * what pre_attn writes: multi-GPU bags hold full sequences x H/G heads,
 * one-GPU bags their chunk rows.  For tensors an exchange did not produce:
 * q/k/v written by a projection in the chunk layout (the source of a
 * 3-tensor pre_attn), an attention output in the Ulysses layout (the source
 * of post_attn) -- the DiT pattern of metrics.cpp:85-121.                  */
SB_API sb_status sb_world_layout_plan(sb_world* w, const sb_planner* p, int layout, sb_stream stream);
/* Fill hosted ranks with the reference witness: metadata (id, pos) and
 * payload doubles payload_value(id, pos, col) (exchange.cpp:18-23,52-63).
 * Fixture generator for tests/bench; payload tensors must be 8*W_d bytes. */
SB_API sb_status sb_world_fill_witness(sb_world* w, const uint64_t* d_ids, const int64_t* d_lens,
                                const int64_t* d_rank_off, sb_stream stream);
/* Row metadata only ({sample_id, position} of every origin row), payload
 * untouched: the input side of a timed step whose payload is produced
 * elsewhere (the step driver without verification). */
SB_API sb_status sb_world_fill_meta(sb_world* w, const uint64_t* d_ids, const int64_t* d_lens,
                                    const int64_t* d_rank_off, sb_stream stream);
/* payload[r][c] += block_perturbation(id, pos) on hosted ranks
 * (simulator.cpp:128-136) -- stands in for a transformer block. */
SB_API sb_status sb_world_perturb(sb_world* w, sb_stream stream);
/* content_checksum (exchange.cpp:438-457) over the hosted ranks' payload
 * tensor 1, accumulated into *d_acc (device uint64, caller zeroes it). */
SB_API sb_status sb_world_checksum(sb_world* w, uint64_t* d_acc, sb_stream stream);

/* worlds_bitwise_equal (exchange.cpp:459-480) on the hosted ranks: adds the
 * number of differing 16-byte words (+1 per rank/tensor whose shape differs)
 * to *d_count (device uint64, caller zeroes it); 0 == bitwise equal. */
SB_API sb_status sb_world_compare(sb_world* a, sb_world* b, uint64_t* d_count, sb_stream stream);

/* ------------------------------------------------------------ exchange -- */
/* route (exchange.cpp:127-194): every chunk of the current plan moves to its
 * target rank, packed in receive order; out-of-place from `src` to `dst`.
 * reverse != 0 executes reverse_route (exchange.cpp:196-198), i.e. the plan
 * with source and target swapped.  Each process pushes the chunks whose
 * source it hosts (peer stores when the target is remote).                */
SB_API sb_status sb_route(sb_planner* p, int reverse, sb_world* src, sb_world* dst, sb_stream stream);
/* Ulysses seq->head all-to-all for every multi-GPU bag of every replica
 * (pre_attn, exchange.cpp:255-331); ranks in single-GPU bags alias `src`.  */
SB_API sb_status sb_pre_attn(sb_planner* p, sb_world* src, sb_world* dst, sb_stream stream);
/* Inverse (post_attn, exchange.cpp:333-436).                               */
SB_API sb_status sb_post_attn(sb_planner* p, sb_world* src, sb_world* dst, sb_stream stream);
/* Split form of the four calls above.  op: 0 route, 1 reverse_route,
 * 2 pre_attn, 3 post_attn.  prepare writes the destination layout tables
 * and the copy jobs into `slot` (0..7); run launches the copy.  Preparations
 * depend only on the plan and on the world tables written by the previous
 * preparation, so all of a step's preparations may run on a side stream
 * while earlier copies are still moving data (sb_route & co. use slots
 * 0..3 and prepare + run back to back). */
SB_API sb_status sb_exchange_prepare(sb_planner* p, int op, sb_world* src, sb_world* dst, int slot,
                                     sb_stream stream);
SB_API sb_status sb_exchange_run(sb_planner* p, int slot, sb_stream stream);
/* Collective transport (the NCCL baseline of the four exchanges above; the
 * reference's simulated all-to-all is exchange.cpp:127-198 / :255-436).  No
 * peer mappings: every process builds the exchange's full job list from the
 * shared plan and packs the jobs whose source it hosts and whose target it
 * does not into one segment per destination process of `send_buf` (in job
 * order; local->local jobs copy directly).  d_counts (device, 2P int64)
 * receives the bytes sent to each process [0, P) and received from each
 * [P, 2P).  The caller then runs ONE all-to-all-v send_buf -> recv_buf on the
 * same stream (grouped ncclSend/ncclRecv; NCCL skips zero counts, so the
 * Ulysses exchanges stay inside each bag) and calls sb_exchange_unpack, which
 * scatters recv_buf into the destination world.  A plan needing more than
 * send_cap / recv_cap bytes copies nothing and sb_world_status(dst) reports
 * SB_ERR_CAPACITY; at most 16 processes. */
SB_API sb_status sb_exchange_pack(sb_planner* p, int op, sb_world* src, sb_world* dst, void* send_buf,
                                  int64_t send_cap, void* recv_buf, int64_t recv_cap, int64_t* d_counts,
                                  sb_stream stream);
SB_API sb_status sb_exchange_unpack(sb_planner* p, sb_stream stream);
/* Synchronises and returns the world's device status (layout capacity). */
SB_API sb_status sb_world_status(sb_world* w, sb_stream stream);

/* Copy the hosted ranks' packed image of every tensor between host and
 * device (pinned host memory is fastest): bytes[t] from/to the start of
 * tensor t's arena, where k_layout packs the hosted ranks back to back in
 * rank order.  Asynchronous; NULL host[t] skips tensor t. */
SB_API sb_status sb_world_upload(sb_world* w, void* const* host, const int64_t* bytes, sb_stream stream);
SB_API sb_status sb_world_download(sb_world* w, void* const* host, const int64_t* bytes, sb_stream stream);
/* One rank's tensor t (rows x pitch bytes, current layout) to/from host
 * memory; synchronises.  *bytes returns the rank's byte size (pass
 * host == NULL to query). */
SB_API sb_status sb_world_read_rank(sb_world* w, int tensor, int rank, void* host, int64_t capacity,
                                    int64_t* bytes, sb_stream stream);
SB_API sb_status sb_world_write_rank(sb_world* w, int tensor, int rank, const void* host, int64_t bytes,
                                     sb_stream stream);
/* Current per-rank rows/pitch as host arrays (synchronises). */
SB_API sb_status sb_world_shape(sb_world* w, int tensor, int64_t* rows, int64_t* pitch, sb_stream stream);

/* ------------------------------------------- uniform (T5) balancer -- */
/* balance_uniform_items / reverse_uniform_plan (balancer.hpp:122-144,
 * balancer.cpp:411-462) for identical-cost items: post-counts differ by at
 * most 1, moves minimal, +1 slots to the largest counts (ties toward the
 * lower rank), surpluses paired with deficits in rank order.  The plan is
 * computed on the device from device counts[world]; sb_uniform_route moves
 * the items (rows_per_item rows each, every tensor of the world) with the
 * route copy engines: a surplus rank keeps its first final_count items and
 * sends the rest in move order; a deficit rank appends received items in
 * move order.  reverse != 0 sends every relocated item home. */
typedef struct sb_uniform sb_uniform;
SB_API sb_status sb_uniform_create(int world, sb_uniform** out);
SB_API sb_status sb_uniform_destroy(sb_uniform* u);
SB_API sb_status sb_uniform_plan(sb_uniform* u, const int64_t* d_counts, sb_stream stream);
/* Synchronises; moves3 = n_moves x {src_rank, dst_rank, count} (<= 2*world). */
SB_API sb_status sb_uniform_download(sb_uniform* u, int64_t* final_counts, int64_t* moves3, int64_t* n_moves,
                                     int64_t* total_moved, sb_stream stream);
SB_API sb_status sb_uniform_route(sb_uniform* u, int reverse, int64_t rows_per_item, sb_world* src, sb_world* dst,
                                  sb_stream stream);

/* ------------------------------------- upstream generator (data_sim) -- */
/* A sharding-group scenario: g{G}b{B}i{R}f{F}s{S} data streams
 * (parse_data_code, data_sim.cpp:39-76 -- same grammar, ParseError messages
 * and byte offsets), a scenario file (parse_scenario, :95-129) or a preset
 * (:152-170).  group_size 0 = the sum of the streams' GPU counts. */
typedef struct sb_scenario sb_scenario;
SB_API sb_status sb_scenario_create(const char* const* codes, int n_codes, int group_size, sb_scenario** out);
SB_API sb_status sb_scenario_parse(const char* text, sb_scenario** out);
SB_API sb_status sb_scenario_preset(const char* name, sb_scenario** out);
SB_API sb_status sb_scenario_destroy(sb_scenario* sc);
/* specs5 (optional): n_streams x {gpus, batch, resolution, frames, smooth}. */
SB_API sb_status sb_scenario_info(const sb_scenario* sc, int* group_size, int* n_streams, int32_t* specs5);

/* K scenarios on the device for a world of `world` ranks: step s draws
 * every rank's batch from scenario s mod K with next_batch
 * (data_sim.cpp:225-248) -- ids make_sample_id(step, rank, i), lengths
 * text U[0,392] + visual_tokens(stream, aspect multiplier) -- bit-exactly.
 * bounds: the largest sequence count / total rows any step can produce. */
typedef struct sb_schedule sb_schedule;
SB_API sb_status sb_schedule_create(const sb_scenario* const* scenarios, int K, int world, uint64_t seed,
                                    sb_schedule** out);
SB_API sb_status sb_schedule_destroy(sb_schedule* s);
SB_API sb_status sb_schedule_bounds(const sb_schedule* s, int64_t* max_seqs, int64_t* max_rows);
/* Writes the gathered metadata of step (step + (d_step ? *d_step : 0)):
 * ids/lens in gather order and rank_off[world + 1].  One kernel. */
SB_API sb_status sb_schedule_generate(const sb_schedule* s, int64_t step, const int64_t* d_step, uint64_t* d_ids,
                                      int64_t* d_lens, int64_t* d_rank_off, sb_stream stream);

/* ---------------------------------------------- step driver (simulator) -- */
/* simulate_step (simulator.cpp:45-178) on the device path: generate the
 * step's batches -> origin layout + witness payload -> plan_routing ->
 * route -> pre_attn/post_attn (multi-GPU bags) -> reverse_route.  With
 * verify, the reference's inline checks run on the device: content
 * checksum conserved by route and pre_attn, post_attn(pre_attn(x)) == x
 * bitwise, and a perturbed payload (block_perturbation) returns home
 * bitwise.  The step index lives in device memory and advances per step,
 * so sb_driver_step is graph-capturable; records land in a device ring of
 * record_cap entries indexed by step. */
enum {
  SB_CHECK_ROUTE_CONSERVED = 1,
  SB_CHECK_PRE_CONSERVED = 2,
  SB_CHECK_POST_INVERTS_PRE = 4,
  SB_CHECK_REVERSE_RESTORES = 8,
  SB_CHECK_ALL = 15
};
typedef struct sb_step_record {
  int64_t step;
  int64_t tokens;
  int64_t sequences;
  int64_t chunks;
  double wir;             /* BalanceReport::wir (metrics.cpp:20-31)            */
  double max_over_mean;   /* max(per_gpu_workload) / mean                       */
  double total_workload;  /* BalanceReport::total_workload                      */
  uint64_t checksum;      /* content_checksum of the step's input (verify)      */
  int32_t scenario;       /* s mod K                                            */
  int32_t capacity_violations;
  int32_t checks;         /* SB_CHECK_* bits that held (verify)                 */
  int32_t verified;
} sb_step_record;
typedef struct sb_driver sb_driver;
SB_API sb_status sb_driver_create(sb_planner* p, const sb_schedule* s, int n_heads, int64_t payload_row_bytes,
                                  int verify, int64_t record_cap, sb_driver** out);
SB_API sb_status sb_driver_destroy(sb_driver* d);
SB_API sb_status sb_driver_set_step(sb_driver* d, int64_t step, sb_stream stream);  /* synchronises */
/* Plan-ahead schedule (on != 0): the driver keeps a second slot (a clone of
 * the planner + five worlds + metadata) and, while step s's copies run,
 * generates, plans and prepares step s+1 on a side stream; results are
 * identical to the serial schedule.  Step s+1 is prepared before step s
 * returns, so a captured graph must hold an even number of steps.
 * Synchronises; prepares the step the device counter names. */
SB_API sb_status sb_driver_set_pipeline(sb_driver* d, int on, sb_stream stream);
SB_API sb_status sb_driver_step(sb_driver* d, sb_stream stream);
SB_API sb_status sb_driver_run(sb_driver* d, int64_t n_steps, sb_stream stream);
/* next step index, steps run since set_step, steps whose checks failed (synchronises). */
SB_API sb_status sb_driver_progress(sb_driver* d, int64_t* next_step, int64_t* steps_run, int64_t* failed,
                                    sb_stream stream);
SB_API sb_status sb_driver_records(sb_driver* d, sb_step_record* host, int64_t capacity, int64_t* n_out,
                                   sb_stream stream);
/* Worlds / metadata of the most recently issued step.
 * which: 0 origin (A), 1 routed (B), 2 Ulysses (C), 3 post_attn (D), 4 returned (E). */
SB_API sb_status sb_driver_world(const sb_driver* d, int which, sb_world** out);
SB_API sb_status sb_driver_meta(const sb_driver* d, const uint64_t** ids, const int64_t** lens,
                                const int64_t** rank_off);

/* ------------------------------------- host-buffer drop-in entry points -- */
/* assign_to_bags (balancer.hpp:30-31, balancer.cpp:15-64) on caller
 * workloads; the planner must describe exactly one replica.  Host arrays;
 * outputs in assignment (sorted) order; out_bag = bag INDEX.  Synchronises. */
SB_API sb_status sb_assign_to_bags(sb_planner* p, int64_t n, const uint64_t* ids, const double* workloads,
                                   uint64_t* out_ids, double* out_w, int32_t* out_bag, sb_stream stream);

/* A RoutingPlan that did not come from sb_plan (host arrays): chunks plus
 * the origin/target layouts as per-rank segment CSR.  Chunk rows are located
 * on the device (route's locate, exchange.cpp:156-167); SB_ERR_INTEGRITY
 * names the sample when a chunk has no containing segment.  The uploaded
 * plan drives sb_route (both directions).  Synchronises. */
SB_API sb_status sb_plan_upload(sb_planner* p, int64_t n_chunks, const uint64_t* chunk_id, const int32_t* chunk_index,
                                const int64_t* chunk_start, const int64_t* chunk_end, const int32_t* chunk_src,
                                const int32_t* chunk_dst, const int64_t* origin_off, const uint64_t* origin_id,
                                const int64_t* origin_first, const int64_t* origin_len, const int64_t* target_off,
                                const uint64_t* target_id, const int64_t* target_first, const int64_t* target_len,
                                sb_stream stream);

/* finalize_manifests (balancer.cpp:84-91) and reverse_plan's receive order
 * (balancer.cpp:259-285) for the uploaded plan, on the device; results in
 * the planner's send/recv/rev_recv arrays (sb_plan_download).  Synchronises. */
SB_API sb_status sb_plan_manifests(sb_planner* p, sb_stream stream);

/* Host-chosen layout: rows[W] and pitch[T*W] (bytes per row per tensor);
 * ranks packed back to back in each arena.  Single-process worlds. */
SB_API sb_status sb_world_set_layout(sb_world* w, const int64_t* rows, const int64_t* pitch, sb_stream stream);
/* First global payload column (in doubles) held per rank (checksum). */
SB_API sb_status sb_world_set_headcol(sb_world* w, const int32_t* headcol, sb_stream stream);

/* BlockMove (exchange.hpp:86-96) with columns in bytes of payload tensor 1;
 * copy_meta also moves the 16-byte metadata rows. */
typedef struct sb_block_move {
  int32_t src_rank, dst_rank;
  int64_t src_row, dst_row, n_rows;
  int64_t src_col_bytes, dst_col_bytes, n_col_bytes;
  int32_t copy_meta, reserved;
} sb_block_move;
/* apply_block_moves (exchange.hpp:98-105, exchange_kernels.cpp:35-56) on
 * the device copy engine; destinations must be disjoint (as the reference
 * requires), so the result equals the serial reference bit for bit. */
SB_API sb_status sb_apply_moves(sb_world* src, sb_world* dst, const sb_block_move* moves, int64_t n,
                                sb_stream stream);

/* ------------------------------------------------- multi-process / peer -- */
/* One process per GPU.  Device buffers are shared once through CUDA IPC
 * (handles travel over the caller's control plane, e.g. torch.distributed);
 * the exchange kernels then store straight into peer memory over NVLink.  */
#define SB_IPC_HANDLE_BYTES 64
SB_API sb_status sb_ipc_export(const void* dptr, void* handle /* SB_IPC_HANDLE_BYTES */);
SB_API sb_status sb_ipc_import(const void* handle, void** dptr);
SB_API sb_status sb_ipc_close(void* dptr);

/* Metadata all-gather (gather_sequence_info, exchange.cpp:68-77, made a real
 * collective): every process pushes its hosted ranks' (id, len) records into
 * slot [rank] of every process's gather buffer (peer stores), then -- after a
 * barrier -- compacts its own buffer into gather order for sb_plan.
 * Without sb_gather_set_peers only this process's slots are written; the
 * collective transport then all-gathers the buffer's three sections (counts
 * [W] i64, ids [W*cap] u64, lens [W*cap] i64; each process owns the
 * contiguous slots of its ranks) with ncclAllGather before compacting.    */
typedef struct sb_gather sb_gather;
SB_API sb_status sb_gather_create(int world_size, int n_local, int first_local, int64_t cap_per_rank,
                                  sb_gather** out);
SB_API sb_status sb_gather_destroy(sb_gather* g);
SB_API sb_status sb_gather_buffer(const sb_gather* g, void** buf, int64_t* bytes);
SB_API sb_status sb_gather_set_peers(sb_gather* g, const uint64_t* bases, int n_procs);
/* d_local_off: n_local+1 offsets of the hosted ranks' records in d_ids/d_lens. */
SB_API sb_status sb_gather_push(sb_gather* g, const uint64_t* d_ids, const int64_t* d_lens,
                                const int64_t* d_local_off, sb_stream stream);
SB_API sb_status sb_gather_compact(sb_gather* g, uint64_t* d_ids, int64_t* d_lens, int64_t* d_rank_off,
                                   sb_stream stream);
SB_API sb_status sb_gather_status(sb_gather* g, sb_stream stream);

/* Device-side barrier over system-scope flags in peer memory: closes an
 * exchange phase on every process without a host round trip.            */
typedef struct sb_barrier sb_barrier;
SB_API sb_status sb_barrier_create(int n_procs, int me, sb_barrier** out);
SB_API sb_status sb_barrier_destroy(sb_barrier* b);
SB_API sb_status sb_barrier_buffer(const sb_barrier* b, void** buf, int64_t* bytes);
SB_API sb_status sb_barrier_set_peers(sb_barrier* b, const uint64_t* bases, int n_procs);
SB_API sb_status sb_barrier_wait(sb_barrier* b, sb_stream stream);
/* Bounded wait: a barrier that does not complete within the timeout
 * (default 60 s, env SEQBAL_BARRIER_TIMEOUT_MS) records which process did
 * not arrive; sb_barrier_status synchronises the stream and returns
 * SB_ERR_COMM with that process and epoch (failure detection).
 * The epoch counter is device-resident, so barriers replay inside CUDA
 * graphs; *epoch (optional) receives the last completed epoch. */
SB_API sb_status sb_barrier_set_timeout(sb_barrier* b, double timeout_ms);
SB_API sb_status sb_barrier_status(sb_barrier* b, uint64_t* epoch, sb_stream stream);

/* Device time of the copy kernels launched while timing was enabled
 * (sb_planner_enable_timing): op 0 route, 1 reverse_route, 2 pre_attn,
 * 3 post_attn, -1 all.  Synchronises on the recorded events. */
SB_API sb_status sb_copy_timing(sb_planner* p, int op, int64_t* count, double* total_us);
SB_API sb_status sb_copy_timing_reset(sb_planner* p);

/* Bytes the last exchange call moved (algorithmic, read + write) and the
 * number of copy jobs it issued; for roofline accounting. */
SB_API sb_status sb_last_exchange_bytes(const sb_planner* p, int64_t* bytes_read, int64_t* bytes_written);

#ifdef __cplusplus
}
#endif
#endif
