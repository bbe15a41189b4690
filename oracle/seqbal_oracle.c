/*
 * TEST INFRASTRUCTURE ONLY -- see seqbal_oracle.h.  Never linked into the
 * product library.  Plain-C restatement of /root/reference/proj; compiled
 * with -ffp-contract=off semantics enforced below so every FP64 expression
 * rounds exactly as the reference's default x86-64 build (no FMA).
 */
#pragma STDC FP_CONTRACT OFF
#include "seqbal_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.hpp */

/* rng.hpp:12-17 */
uint64_t or_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* rng.hpp:20-24 */
uint64_t or_derive_key(const uint64_t* parts, int n) {
  uint64_t k = 0x8f51a7c0c0c0f5a3ULL;
  for (int i = 0; i < n; ++i) k = or_splitmix64(k ^ parts[i]);
  return k;
}

/* rng.hpp:34 -- draw `counter` of the stream keyed by `key`. */
uint64_t or_rng_u64(uint64_t key, uint64_t counter) {
  return or_splitmix64(key ^ or_splitmix64(counter));
}

/* rng.hpp:45-50 (Lemire fixed-point multiply) */
int64_t or_rng_int(uint64_t key, uint64_t counter, int64_t lo, int64_t hi) {
  const uint64_t span = (uint64_t)(hi - lo) + 1;
  const uint64_t r = (uint64_t)(((unsigned __int128)or_rng_u64(key, counter) * span) >> 64);
  return lo + (int64_t)r;
}

/* rng.hpp:37-40 */
double or_rng_real(uint64_t key, uint64_t counter, double lo, double hi) {
  const double u = (double)(or_rng_u64(key, counter) >> 11) * 0x1.0p-53;
  const double span = hi - lo;
  const double scaled = u * span;
  return lo + scaled;
}

/* ----------------------------------------------------------- data_sim.cpp */

/* data_sim.cpp:219-223 */
uint64_t or_make_sample_id(int64_t step, int rank, int index) {
  return ((uint64_t)step << 32) | ((uint64_t)(rank & 0xffff) << 16) | (uint64_t)(index & 0xffff);
}

static const uint64_t kTextDomain = 0x7465787421ULL;   /* data_sim.cpp:195 */
static const uint64_t kAspectDomain = 0x6173706563ULL; /* data_sim.cpp:196 */

/* data_sim.cpp:198-203 */
double or_aspect_multiplier(uint64_t seed, int64_t step, int stream_index) {
  const uint64_t parts[4] = {kAspectDomain, seed, (uint64_t)step, (uint64_t)stream_index};
  return or_rng_real(or_derive_key(parts, 4), 0, 0.96, 1.04);
}

/* data_sim.cpp:177-191 (latent_frames + visual_tokens) */
int64_t or_visual_tokens(int resolution, int frames, int smooth, double mult) {
  const int64_t side = resolution / 16;
  const int64_t spatial = side * side;
  const int64_t scaled = llround((double)spatial * mult);
  int64_t latent = frames;
  if (smooth) {
    const double f = (double)frames * 5;
    latent = llround(f / 17);
  }
  const int64_t tokens = scaled * latent;
  return tokens < 1 ? 1 : tokens;
}

/* data_sim.cpp:225-248 */
int or_next_batch(int n_streams, const int* gpus, const int* batch, const int* res,
                  const int* frames, const int* smooth, int rank, int64_t step, uint64_t seed,
                  uint64_t* ids, int64_t* text, int64_t* visual) {
  int group = 0;
  for (int i = 0; i < n_streams; ++i) group += gpus[i];
  if (group < 1 || rank < 0) return -1;
  const int group_rank = rank % group;
  int stream = -1, cursor = 0;
  for (int i = 0; i < n_streams; ++i) {
    cursor += gpus[i];
    if (group_rank < cursor) {
      stream = i;
      break;
    }
  }
  if (stream < 0) return -1;
  const double mult = or_aspect_multiplier(seed, step, stream);
  const uint64_t parts[4] = {kTextDomain, seed, (uint64_t)step, (uint64_t)rank};
  const uint64_t key = or_derive_key(parts, 4);
  for (int i = 0; i < batch[stream]; ++i) {
    ids[i] = or_make_sample_id(step, rank, i);
    text[i] = or_rng_int(key, (uint64_t)i, 0, 392);
    visual[i] = or_visual_tokens(res[stream], frames[stream], smooth[stream], mult);
  }
  return batch[stream];
}

void or_c1_batch(uint64_t seed, int64_t step, int rank, int per_rank, uint64_t* ids,
                 int64_t* lens) {
  const uint64_t parts[3] = {seed, (uint64_t)step, (uint64_t)rank};
  const uint64_t key = or_derive_key(parts, 3);
  for (int i = 0; i < per_rank; ++i) {
    const int64_t text = or_rng_int(key, 2 * (uint64_t)i, 64, 512);
    const int64_t image = or_rng_int(key, 2 * (uint64_t)i + 1, 256, 4096);
    ids[i] = or_make_sample_id(step, rank, i);
    lens[i] = text + image;
  }
}

/* ----------------------------------------------------------- exchange.cpp */

static const uint64_t kPayloadDomain = 0x7061796c6f6164ULL; /* exchange.cpp:14 */
static const uint64_t kPerturbDomain = 0x706572747572ULL;   /* exchange.cpp:15 */

/* exchange.cpp:18-23 */
double or_payload_value(uint64_t sample_id, int64_t position, int col) {
  const uint64_t parts[4] = {kPayloadDomain, sample_id, (uint64_t)position, (uint64_t)col};
  return (double)(or_derive_key(parts, 4) >> 11) * 0x1.0p-53;
}

/* exchange.cpp:25-29 */
double or_block_perturbation(uint64_t sample_id, int64_t position) {
  const uint64_t parts[3] = {kPerturbDomain, sample_id, (uint64_t)position};
  return (double)(or_derive_key(parts, 3) >> 11) * 0x1.0p-53;
}

uint64_t or_digest(const void* data, size_t n, uint64_t h) {
  const unsigned char* p = (const unsigned char*)data;
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    memcpy(&w, p + i, 8);
    h = or_splitmix64(h ^ w);
  }
  if (i < n) {
    uint64_t w = 0;
    memcpy(&w, p + i, n - i);
    h = or_splitmix64(h ^ w);
  }
  return h;
}

/* exchange.cpp:52-63 (payload part of make_world) */
void or_fill_witness(int64_t rows, const uint64_t* ids, const int64_t* pos, int width, double* out) {
  for (int64_t r = 0; r < rows; ++r)
    for (int c = 0; c < width; ++c) out[r * width + c] = or_payload_value(ids[r], pos[r], c);
}

/* simulator.cpp:128-136 */
void or_perturb(int64_t rows, const uint64_t* ids, const int64_t* pos, int width, double* payload) {
  for (int64_t r = 0; r < rows; ++r) {
    const double delta = or_block_perturbation(ids[r], pos[r]);
    for (int c = 0; c < width; ++c) payload[r * width + c] += delta;
  }
}

/* exchange.cpp:438-457, contribution of one rank buffer */
uint64_t or_checksum_rank(int64_t rows, const uint64_t* ids, const int64_t* pos, int width,
                          int head_cols, const double* payload) {
  uint64_t acc = 0;
  for (int64_t r = 0; r < rows; ++r) {
    for (int c = 0; c < width; ++c) {
      uint64_t bits;
      memcpy(&bits, &payload[r * width + c], 8);
      const uint64_t parts[4] = {ids[r], (uint64_t)pos[r], (uint64_t)(head_cols + c), bits};
      acc += or_derive_key(parts, 4);
    }
  }
  return acc;
}

/* ----------------------------------------------------- workload / metrics */

/* workload_model.cpp:65-70: 24*l*d*d + gamma*4*l*l*d, left-associative,
 * each product rounded (the reference build has no FMA). */
double or_gamma_weighted_workload(int64_t seq_len, int d_model, double gamma) {
  const double l = (double)seq_len;
  const double d = (double)d_model;
  double lin = 24.0 * l;
  lin = lin * d;
  lin = lin * d;
  double att = gamma * 4.0;
  att = att * l;
  att = att * l;
  att = att * d;
  return lin + att;
}

/* balancer.cpp:66-73 */
void or_chunk_lengths(int64_t total_len, int parts, int64_t* out) {
  const int64_t rem = total_len % parts;
  for (int i = 0; i < parts; ++i) out[i] = total_len / parts + (i < rem ? 1 : 0);
}

/* metrics.cpp:20-31 */
double or_wir(const double* w, int n) {
  double lo = w[0], hi = w[0];
  for (int i = 0; i < n; ++i) {
    if (w[i] < lo) lo = w[i];
    if (w[i] > hi) hi = w[i];
  }
  if (hi == 0.0) return 1.0;
  if (lo == 0.0) return INFINITY;
  return hi / lo;
}

/* ------------------------------------------------------------ balancer.cpp */

typedef struct {
  double w;
  uint64_t id;
  int64_t src; /* index of the sequence in the caller's array */
} sw_t;

/* balancer.cpp:37-40: descending workload, ascending sample_id. */
static int cmp_sw(const void* a, const void* b) {
  const sw_t* x = (const sw_t*)a;
  const sw_t* y = (const sw_t*)b;
  if (x->w != y->w) return x->w > y->w ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return 0;
}

static double occupancy(double asg, double cap) { /* balancer.cpp:32-35 */
  if (cap > 0.0) return asg / cap;
  return asg > 0.0 ? INFINITY : 0.0;
}

/* balancer.cpp:15-64 on a pre-sorted list; writes the bag INDEX per entry. */
static void greedy_sorted(int64_t n, const sw_t* s, int m, const int* bag_sizes, int* pick_out,
                          double* cap, double* asg) {
  int total_gpus = 0;
  for (int j = 0; j < m; ++j) total_gpus += bag_sizes[j];
  /* total is summed in the caller's (gather) order: balancer.cpp:24-25 */
  (void)total_gpus;
  for (int64_t i = 0; i < n; ++i) {
    int best = m, fallback = m;
    double best_occ = 0.0, fallback_occ = 0.0;
    for (int j = 0; j < m; ++j) {
      const double occ = occupancy(asg[j], cap[j]);
      if (cap[j] - asg[j] >= s[i].w && (best == m || occ < best_occ)) {
        best = j;
        best_occ = occ;
      }
      if (fallback == m || occ < fallback_occ) {
        fallback = j;
        fallback_occ = occ;
      }
    }
    const int pick = best != m ? best : fallback;
    asg[pick] += s[i].w;
    pick_out[i] = pick;
  }
}

static void capacities(const double* w_gather, int64_t n, int m, const int* bag_sizes, double* cap) {
  int total_gpus = 0;
  for (int j = 0; j < m; ++j) total_gpus += bag_sizes[j];
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += w_gather[i]; /* balancer.cpp:24-25 */
  const double target = total / total_gpus;              /* balancer.cpp:26 */
  for (int j = 0; j < m; ++j) cap[j] = bag_sizes[j] * target; /* balancer.cpp:30 */
}

int or_assign_to_bags(int n, const uint64_t* ids, const double* w, int m, const int* bag_sizes,
                      const int* bag_ids, uint64_t* out_ids, double* out_w, int* out_bag) {
  if (m < 1) return 1; /* balancer.cpp:17 */
  for (int i = 0; i < n; ++i)
    if (!(w[i] >= 0.0)) return 1; /* balancer.cpp:18-20 */
  double* cap = (double*)calloc((size_t)m, sizeof(double));
  double* asg = (double*)calloc((size_t)m, sizeof(double));
  sw_t* s = (sw_t*)malloc(sizeof(sw_t) * (size_t)(n > 0 ? n : 1));
  int* pick = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  capacities(w, n, m, bag_sizes, cap);
  for (int i = 0; i < n; ++i) {
    s[i].w = w[i];
    s[i].id = ids[i];
    s[i].src = i;
  }
  qsort(s, (size_t)n, sizeof(sw_t), cmp_sw);
  greedy_sorted(n, s, m, bag_sizes, pick, cap, asg);
  for (int i = 0; i < n; ++i) {
    out_ids[i] = s[i].id;
    out_w[i] = s[i].w;
    out_bag[i] = bag_ids[pick[i]];
  }
  free(cap);
  free(asg);
  free(s);
  free(pick);
  return 0;
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* balancer.cpp:84-91: stable partition of chunk indices by rank. */
static void manifests(int world, int64_t n, const int32_t* key, int64_t* off, int32_t* idx) {
  for (int r = 0; r <= world; ++r) off[r] = 0;
  for (int64_t i = 0; i < n; ++i) off[key[i] + 1]++;
  for (int r = 0; r < world; ++r) off[r + 1] += off[r];
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(world + 1));
  memcpy(cur, off, sizeof(int64_t) * (size_t)(world + 1));
  for (int64_t i = 0; i < n; ++i) idx[cur[key[i]]++] = (int32_t)i;
  free(cur);
}

int or_plan_routing(const or_plan_in* in, or_plan_out* out) {
  const int W = in->world_size;
  const int unit = in->unit_size;
  const int M = in->n_bags;
  if (unit < 1 || W < unit || W % unit != 0) return 1; /* topology.cpp:81-93 */
  for (int j = 0; j < M; ++j) {                          /* balancer.cpp:114-120 */
    const int g = in->bag_off[j + 1] - in->bag_off[j];
    if (g < 1 || in->n_heads % g != 0) return 1;
  }
  const int64_t N = in->rank_off[W];
  for (int64_t i = 0; i < N; ++i)
    if (in->lens[i] < 0) return 1; /* workload_model.cpp:66 */

  int* bag_sizes = (int*)malloc(sizeof(int) * (size_t)M);
  for (int j = 0; j < M; ++j) bag_sizes[j] = in->bag_off[j + 1] - in->bag_off[j];

  for (int r = 0; r < W; ++r) out->per_gpu[r] = 0.0;
  out->total_workload = 0.0;
  out->violations = 0;
  out->n_chunks = 0;
  int status = 0;

  const int reps = W / unit;
  double* w = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
  int32_t* origin = (int32_t*)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
  sw_t* s = (sw_t*)malloc(sizeof(sw_t) * (size_t)(N > 0 ? N : 1));
  int* pick = (int*)malloc(sizeof(int) * (size_t)(N > 0 ? N : 1));
  uint64_t* idsort = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(N > 0 ? N : 1));
  double* cap = (double*)malloc(sizeof(double) * (size_t)M);
  double* asg = (double*)malloc(sizeof(double) * (size_t)M);

  for (int r = 0; r < W; ++r)
    for (int64_t i = in->rank_off[r]; i < in->rank_off[r + 1]; ++i) origin[i] = r;

  for (int rep = 0; rep < reps && status == 0; ++rep) {
    const int base = rep * unit;
    const int64_t lo = in->rank_off[base], hi = in->rank_off[base + unit];
    const int64_t n = hi - lo;
    /* balancer.cpp:139-149: workloads in gather order, global running total */
    for (int64_t i = lo; i < hi; ++i) {
      w[i] = or_gamma_weighted_workload(in->lens[i], in->d_model, in->gamma);
      out->total_workload += w[i];
    }
    /* divergence: reject duplicate ids inside a replica */
    for (int64_t i = 0; i < n; ++i) idsort[i] = in->ids[lo + i];
    qsort(idsort, (size_t)n, sizeof(uint64_t), cmp_u64);
    for (int64_t i = 1; i < n; ++i)
      if (idsort[i] == idsort[i - 1]) status = 1;
    if (status) break;

    /* balancer.cpp:151 -> assign_to_bags */
    capacities(w + lo, n, M, bag_sizes, cap);
    for (int j = 0; j < M; ++j) asg[j] = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      s[i].w = w[lo + i];
      s[i].id = in->ids[lo + i];
      s[i].src = lo + i;
    }
    qsort(s, (size_t)n, sizeof(sw_t), cmp_sw);
    /* balancer.cpp:156-176: the replay counts a violation exactly when the
     * pick had less remaining capacity than the sequence, i.e. when the
     * feasible set was empty; recomputed here the same way. */
    {
      double* asg2 = (double*)calloc((size_t)M, sizeof(double));
      greedy_sorted(n, s, M, bag_sizes, pick, cap, asg);
      for (int64_t i = 0; i < n; ++i) {
        const int b = pick[i];
        if (cap[b] - asg2[b] < s[i].w) out->violations++;
        asg2[b] += s[i].w;
      }
      for (int j = 0; j < M; ++j) out->per_bag_occ[rep * M + j] = occupancy(asg2[j], cap[j]);
      free(asg2);
    }
    /* balancer.cpp:178-218: by_bag in assignment order, chunk emission */
    for (int b = 0; b < M; ++b) {
      const int g = bag_sizes[b];
      double bag_load = 0.0;
      for (int64_t i = 0; i < n; ++i)
        if (pick[i] == b) bag_load += s[i].w;
      for (int k = 0; k < g; ++k) out->per_gpu[base + in->bag_ranks[in->bag_off[b] + k]] = bag_load / g;
      for (int64_t i = 0; i < n; ++i) {
        if (pick[i] != b) continue;
        const int64_t seq = s[i].src;
        const int64_t len = in->lens[seq];
        int64_t cursor = 0;
        for (int k = 0; k < g; ++k) {
          const int64_t cl = len / g + (k < len % g ? 1 : 0);
          const int64_t c = out->n_chunks;
          if (c >= out->cap_chunks) {
            status = 4;
            break;
          }
          out->c_id[c] = in->ids[seq];
          out->c_idx[c] = k;
          out->c_start[c] = cursor;
          out->c_end[c] = cursor + cl;
          out->c_src[c] = origin[seq];
          out->c_dst[c] = base + in->bag_ranks[in->bag_off[b] + k];
          cursor += cl;
          out->n_chunks++;
        }
        if (status) break;
      }
      if (status) break;
    }
  }
  if (status == 0) {
    manifests(W, out->n_chunks, out->c_src, out->send_off, out->send_idx); /* balancer.cpp:84-91 */
    manifests(W, out->n_chunks, out->c_dst, out->recv_off, out->recv_idx);
    out->wir = or_wir(out->per_gpu, W); /* balancer.cpp:223 */
  }
  free(bag_sizes);
  free(w);
  free(origin);
  free(s);
  free(pick);
  free(idsort);
  free(cap);
  free(asg);
  return status;
}

/* balancer.cpp:227-240 */
int or_identity_plan(int world_size, const int64_t* rank_off, const uint64_t* ids,
                     const int64_t* lens, or_plan_out* out) {
  out->n_chunks = 0;
  for (int r = 0; r < world_size; ++r) {
    for (int64_t i = rank_off[r]; i < rank_off[r + 1]; ++i) {
      const int64_t c = out->n_chunks++;
      if (c >= out->cap_chunks) return 4;
      out->c_id[c] = ids[i];
      out->c_idx[c] = 0;
      out->c_start[c] = 0;
      out->c_end[c] = lens[i];
      out->c_src[c] = r;
      out->c_dst[c] = r;
    }
  }
  manifests(world_size, out->n_chunks, out->c_src, out->send_off, out->send_idx);
  manifests(world_size, out->n_chunks, out->c_dst, out->recv_off, out->recv_idx);
  return 0;
}

typedef struct {
  int64_t seg;
  int64_t start;
  int32_t chunk;
} rk_t;

static int cmp_rk(const void* a, const void* b) {
  const rk_t* x = (const rk_t*)a;
  const rk_t* y = (const rk_t*)b;
  if (x->seg != y->seg) return x->seg < y->seg ? -1 : 1;
  if (x->start != y->start) return x->start < y->start ? -1 : 1;
  return x->chunk < y->chunk ? -1 : (x->chunk > y->chunk ? 1 : 0);
}

typedef struct {
  uint64_t id;
  int64_t idx;
} si_t;

static int cmp_si(const void* a, const void* b) {
  const si_t* x = (const si_t*)a;
  const si_t* y = (const si_t*)b;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

/* balancer.cpp:242-287 */
int or_reverse_plan(int world_size, int64_t n_chunks, const uint64_t* c_id, const int64_t* c_start,
                    const int64_t* c_end, const int32_t* c_src, const int32_t* c_dst,
                    const int64_t* seg_off, const uint64_t* seg_id, const int64_t* seg_first,
                    const int64_t* seg_len, int64_t* send_off, int32_t* send_idx,
                    int64_t* recv_off, int32_t* recv_idx) {
  /* rev.send[r] = chunks whose reversed source (forward target) is r, in
   * chunk order (balancer.cpp:256-258). */
  manifests(world_size, n_chunks, c_dst, send_off, send_idx);
  /* rev.recv[r]: chunks whose forward source is r, sorted by (index of the
   * first containing segment of rev.target[r] = plan.origin[r], start). */
  int status = 0;
  for (int r = 0; r <= world_size; ++r) recv_off[r] = 0;
  for (int64_t i = 0; i < n_chunks; ++i) recv_off[c_src[i] + 1]++;
  for (int r = 0; r < world_size; ++r) recv_off[r + 1] += recv_off[r];
  rk_t* buf = (rk_t*)malloc(sizeof(rk_t) * (size_t)(n_chunks > 0 ? n_chunks : 1));
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(world_size + 1));
  int64_t* segc = (int64_t*)calloc((size_t)(n_chunks > 0 ? n_chunks : 1), sizeof(int64_t));
  memcpy(fill, recv_off, sizeof(int64_t) * (size_t)(world_size + 1));
  for (int64_t i = 0; i < n_chunks; ++i) buf[fill[c_src[i]]++].chunk = (int32_t)i;
  for (int r = 0; r < world_size && status == 0; ++r) {
    const int64_t s0 = seg_off[r], ns = seg_off[r + 1] - seg_off[r];
    si_t* idx = (si_t*)malloc(sizeof(si_t) * (size_t)(ns > 0 ? ns : 1));
    for (int64_t s = 0; s < ns; ++s) {
      idx[s].id = seg_id[s0 + s];
      idx[s].idx = s;
    }
    qsort(idx, (size_t)ns, sizeof(si_t), cmp_si);
    for (int64_t k = recv_off[r]; k < recv_off[r + 1]; ++k) {
      const int32_t c = buf[k].chunk;
      /* lower_bound on id, then the first segment (by index) containing it */
      int64_t a = 0, b = ns;
      while (a < b) {
        const int64_t mid = (a + b) / 2;
        if (idx[mid].id < c_id[c]) a = mid + 1;
        else b = mid;
      }
      int64_t found = -1;
      for (int64_t q = a; q < ns && idx[q].id == c_id[c]; ++q) {
        const int64_t s = idx[q].idx;
        if (c_start[c] >= seg_first[s0 + s] && c_end[c] <= seg_first[s0 + s] + seg_len[s0 + s]) {
          found = s;
          break;
        }
      }
      if (found < 0) {
        status = 2; /* balancer.cpp:274-276 */
        break;
      }
      buf[k].seg = found;
      buf[k].start = c_start[c];
      segc[c] = found;
    }
    free(idx);
    if (status) break;
    /* balancer.cpp:278-283: the reference's std::sort, ties included */
    for (int64_t k = recv_off[r]; k < recv_off[r + 1]; ++k) recv_idx[k] = buf[k].chunk;
    or_std_sort_chunks(recv_idx + recv_off[r], recv_off[r + 1] - recv_off[r], segc, c_start);
  }
  free(buf);
  free(fill);
  free(segc);
  return status;
}
