/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the balance-and-redistribute
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load this library, and only as a checker.  The product path
 * (paper_2508_06001_b200/, libseqbal_cuda.so) never links or calls it.
 *
 * A plain-C restatement of the reference `seqbal` algorithm
 * (/root/reference/proj).  Every function cites the reference file:line it
 * follows.  Parity is pinned by tests/test_oracle_golden.py against golden
 * fixtures produced by the unmodified reference (oracle/_ref/ref_harness,
 * tests/golden/make_golden.py) and against the reference tests' known-answer
 * values.
 *
 * Deliberate, documented divergence:
 * duplicate sample ids inside one replica are rejected (return 1); the
 * reference silently mis-plans them (balancer.cpp:183-192 lower_bound).
 * reverse_plan's receive order uses libstdc++'s std::sort exactly like the
 * reference (oracle/stdsort_ref.cpp), including the order of tied keys.
 */
#ifndef SEQBAL_ORACLE_H
#define SEQBAL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:12-55 */
uint64_t or_splitmix64(uint64_t x);
uint64_t or_derive_key(const uint64_t* parts, int n);
uint64_t or_rng_u64(uint64_t key, uint64_t counter);
int64_t or_rng_int(uint64_t key, uint64_t counter, int64_t lo, int64_t hi);
double or_rng_real(uint64_t key, uint64_t counter, double lo, double hi);

/* data_sim.cpp:219-223 */
uint64_t or_make_sample_id(int64_t step, int rank, int index);
/* data_sim.cpp:198-203, 177-191, 225-248 */
double or_aspect_multiplier(uint64_t seed, int64_t step, int stream_index);
int64_t or_visual_tokens(int resolution, int frames, int smooth, double mult);
/* next_batch for one rank of a scenario; streams given as parallel arrays.
 * Writes batch_per_gpu entries of ids / text / visual.  Returns count or -1. */
int or_next_batch(int n_streams, const int* gpus, const int* batch, const int* res,
                  const int* frames, const int* smooth, int rank, int64_t step, uint64_t seed,
                  uint64_t* ids, int64_t* text, int64_t* visual);
/* SURVEY.md 8(d) C1 generator: CounterRng({seed, step, rank}); text U[64,512]
 * then image U[256,4096]; id make_sample_id(step, rank, i). */
void or_c1_batch(uint64_t seed, int64_t step, int rank, int per_rank, uint64_t* ids,
                 int64_t* lens);

/* exchange.cpp:18-29 */
double or_payload_value(uint64_t sample_id, int64_t position, int col);
double or_block_perturbation(uint64_t sample_id, int64_t position);

/* Byte digest shared with oracle/ref_harness.cpp digest_bytes(). */
uint64_t or_digest(const void* data, size_t n, uint64_t h);
#define OR_DIGEST_SEED 0x6469676573740000ULL

/* workload_model.cpp:65-70 */
double or_gamma_weighted_workload(int64_t seq_len, int d_model, double gamma);
/* balancer.cpp:66-73 */
void or_chunk_lengths(int64_t total_len, int parts, int64_t* out);
/* metrics.cpp:20-31 */
double or_wir(const double* w, int n);

/* balancer.cpp:15-64.  Output in assignment (sorted) order.  bag_ids[j] is
 * returned for a pick of bag index j.  Returns 0, or 1 on ConfigError. */
int or_assign_to_bags(int n, const uint64_t* ids, const double* w, int m, const int* bag_sizes,
                      const int* bag_ids, uint64_t* out_ids, double* out_w, int* out_bag);

typedef struct or_plan_in {
  int world_size;          /* W */
  const int64_t* rank_off; /* W+1 offsets into ids/lens (gather order) */
  const uint64_t* ids;
  const int64_t* lens;
  int unit_size;
  int n_bags;
  const int* bag_off;   /* n_bags+1 offsets into bag_ranks */
  const int* bag_ranks; /* unit-local ranks in textual order */
  int d_model;
  int n_heads;
  double gamma;
} or_plan_in;

typedef struct or_plan_out {
  int64_t cap_chunks;
  int64_t n_chunks;
  uint64_t* c_id;
  int32_t* c_idx;
  int64_t* c_start;
  int64_t* c_end;
  int32_t* c_src;
  int32_t* c_dst;
  int64_t* send_off; /* W+1 */
  int32_t* send_idx; /* cap_chunks */
  int64_t* recv_off; /* W+1 */
  int32_t* recv_idx; /* cap_chunks */
  double* per_gpu;     /* W */
  double* per_bag_occ; /* replicas * n_bags */
  int32_t violations;
  double total_workload;
  double wir;
} or_plan_out;

/* balancer.cpp:105-225.  0 OK, 1 ConfigError, 4 capacity too small. */
int or_plan_routing(const or_plan_in* in, or_plan_out* out);
/* balancer.cpp:227-240 */
int or_identity_plan(int world_size, const int64_t* rank_off, const uint64_t* ids,
                     const int64_t* lens, or_plan_out* out);

/* balancer.cpp:242-287 for a general plan.  Inputs: the forward plan's chunks
 * and its ORIGIN layout (rev.target) as per-rank segment CSR.  Output chunks
 * are swapped copies; send/recv CSR per the reference rules.
 * 0 OK, 2 IntegrityError (a chunk fits no destination segment). */
int or_reverse_plan(int world_size, int64_t n_chunks, const uint64_t* c_id, const int64_t* c_start,
                    const int64_t* c_end, const int32_t* c_src, const int32_t* c_dst,
                    const int64_t* seg_off, const uint64_t* seg_id, const int64_t* seg_first,
                    const int64_t* seg_len, int64_t* send_off, int32_t* send_idx,
                    int64_t* recv_off, int32_t* recv_idx);

/* std::sort (libstdc++, oracle/stdsort_ref.cpp) of chunk indices by
 * (seg[c], start[c]) -- the reference's receive-order sort including its
 * tie order (balancer.cpp:278-283). */
void or_std_sort_chunks(int32_t* v, int64_t n, const int64_t* seg, const int64_t* start);

/* exchange.cpp:31-66 payload rows: fill rows x width doubles for
 * (ids[i], pos[i]) from payload_value. */
void or_fill_witness(int64_t rows, const uint64_t* ids, const int64_t* pos, int width, double* out);
/* simulator.cpp:128-136: payload[r][c] += block_perturbation(id, pos). */
void or_perturb(int64_t rows, const uint64_t* ids, const int64_t* pos, int width, double* payload);
/* exchange.cpp:438-457, one rank's contribution. */
uint64_t or_checksum_rank(int64_t rows, const uint64_t* ids, const int64_t* pos, int width,
                          int head_cols, const double* payload);

#ifdef __cplusplus
}
#endif
#endif
