// Upstream generator and step driver: the reference's data simulator
// (data_sim.cpp) as a device batch generator, and its training-step driver
// (simulator.cpp:45-178 simulate_step) re-built on the device path.
//
//   sb_scenario  one sharding-group config: g{G}b{B}i{R}f{F}s{S} streams
//                (parse_data_code data_sim.cpp:39-76, parse_scenario
//                :95-129, presets :152-165), parsed on the host with the
//                reference's error classes and messages;
//   sb_schedule  K scenarios on the device; step s draws every rank's batch
//                from scenario s mod K (next_batch :225-248) -- the C5
//                dynamic stream -- with a kernel, no host work per step;
//   sb_driver    one step = generate -> origin layout + witness -> plan ->
//                route -> Ulysses pre/post -> reverse_route, optionally with
//                simulate_step's inline checks (token conservation through
//                route and pre_attn, post_attn(pre_attn(x)) == x, mutated
//                payload returns home bit-exactly, simulator.cpp:106-159).
//                Every step appends a record (WIR, max/mean, tokens, check
//                bits) to a device ring; the step index lives in device
//                memory, so a step is graph-capturable and replays advance it.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "seqbal_capi.h"

namespace sb {

// ------------------------------------------------------------ host parse
constexpr int64_t kMaxFieldValue = 1 << 20;  // data_sim.cpp:16
constexpr int kSpatialStride = 16;           // data_sim.hpp:15

struct Spec {
  int32_t gpus, batch, res, frames, smooth;
};

static std::string parse_msg(const std::string& what, size_t at) {
  return what + " (at offset " + std::to_string(at) + ")";  // ParseError::what (error.hpp:10-21)
}

// parse_data_code (data_sim.cpp:39-76): same grammar, messages and offsets.
static Spec parse_code(const std::string& code) {
  if (code.empty()) throw Error{SB_ERR_PARSE, parse_msg("empty data code", 0)};
  size_t pos = 0;
  auto tag = [&](char t) {
    if (pos >= code.size() || code[pos] != t) throw Error{SB_ERR_PARSE, parse_msg(std::string("expected '") + t + "'", pos)};
    ++pos;
  };
  auto field = [&](const char* what) {
    const size_t start = pos;
    int64_t v = 0;
    while (pos < code.size() && code[pos] >= '0' && code[pos] <= '9') {
      v = v * 10 + (code[pos] - '0');
      if (v > kMaxFieldValue) throw Error{SB_ERR_PARSE, parse_msg(std::string(what) + " value too large", start)};
      ++pos;
    }
    if (pos == start) throw Error{SB_ERR_PARSE, parse_msg(std::string("expected digits for ") + what, start)};
    return v;
  };
  Spec s{};
  tag('g');
  size_t at = pos;
  s.gpus = (int32_t)field("gpu count");
  if (s.gpus < 1) throw Error{SB_ERR_PARSE, parse_msg("gpu count must be >= 1", at)};
  tag('b');
  at = pos;
  s.batch = (int32_t)field("batch size");
  if (s.batch < 1) throw Error{SB_ERR_PARSE, parse_msg("batch size must be >= 1", at)};
  tag('i');
  at = pos;
  s.res = (int32_t)field("resolution");
  if (s.res < 1) throw Error{SB_ERR_PARSE, parse_msg("resolution must be >= 1", at)};
  if (s.res % kSpatialStride != 0)
    throw Error{SB_ERR_PARSE, parse_msg("resolution must be a multiple of " + std::to_string(kSpatialStride), at)};
  tag('f');
  at = pos;
  s.frames = (int32_t)field("frame count");
  if (s.frames < 1) throw Error{SB_ERR_PARSE, parse_msg("frame count must be >= 1", at)};
  tag('s');
  if (pos >= code.size() || (code[pos] != '0' && code[pos] != '1'))
    throw Error{SB_ERR_PARSE, parse_msg("smoothness flag must be 0 or 1", pos)};
  s.smooth = code[pos] == '1';
  ++pos;
  if (pos != code.size()) throw Error{SB_ERR_PARSE, parse_msg("trailing characters after data code", pos)};
  return s;
}

}  // namespace sb

struct sb_scenario {
  int group_size = 0;
  std::vector<sb::Spec> streams;
};

struct sb_schedule {
  int world = 0, K = 0;
  uint64_t seed = 0;
  int64_t max_seqs = 0, max_rows = 0;
  int32_t* d_spec = nullptr;  // [sum streams][5]
  int32_t* d_meta = nullptr;  // per scenario: {first stream, n streams, group size}
};

namespace sb {

static void validate(const sb_scenario& sc) {  // ShardingGroupConfig::validate (data_sim.cpp:86-93)
  if (sc.group_size < 1) throw Error{SB_ERR_CONFIG, "group_size must be >= 1"};
  if (sc.streams.empty()) throw Error{SB_ERR_CONFIG, "scenario has no data streams"};
  int total = 0;
  for (const Spec& s : sc.streams) total += s.gpus;
  if (total != sc.group_size)
    throw Error{SB_ERR_CONFIG, "stream GPU counts sum to " + std::to_string(total) + " but group_size is " +
                                   std::to_string(sc.group_size)};
}

static int stream_of_rank(const sb_scenario& sc, int group_rank) {  // data_sim.cpp:193-203
  int cursor = 0;
  for (size_t i = 0; i < sc.streams.size(); ++i) {
    cursor += sc.streams[i].gpus;
    if (group_rank < cursor) return (int)i;
  }
  throw Error{SB_ERR_CONFIG, "rank not covered by any stream"};
}

static int64_t llround_host(double x) { return std::llround(x); }

// Upper bound of visual_tokens over aspect multipliers in [0.96, 1.04]
// (data_sim.cpp:184-191): monotone in the multiplier.
static int64_t max_visual(const Spec& s) {
  const int64_t side = s.res / kSpatialStride;
  const int64_t scaled = llround_host((double)(side * side) * 1.04);
  const int64_t latent = s.smooth ? llround_host((double)s.frames * 5 / 17) : s.frames;
  const int64_t t = scaled * latent;
  return t < 1 ? 1 : t;
}

// ---------------------------------------------------------- device gen
struct GenArgs {
  const int32_t* spec;
  const int32_t* meta;
  int K, world;
  uint64_t seed;
};

__device__ __forceinline__ int dev_stream_of(const int32_t* spec, int first, int n, int group_rank) {
  int cursor = 0;
  for (int i = 0; i < n; ++i) {
    cursor += spec[(first + i) * 5 + 0];
    if (group_rank < cursor) return i;
  }
  return n - 1;
}

// One CTA per rank: rank offset (prefix over earlier ranks' batch sizes),
// then next_batch's samples in parallel -- text U[0, 392] from
// CounterRng({kTextDomain, seed, step, rank}) draw i, visual tokens from the
// stream's spec and aspect_multiplier(seed, step, stream) (data_sim.cpp:
// 184-248, rng.hpp:30-55); every FP operation in the reference's order.
__global__ void k_generate(GenArgs g, int64_t step_base, const int64_t* d_step, uint64_t* ids, int64_t* lens,
                           int64_t* rank_off, int32_t* scen_out) {
  const int64_t step = step_base + (d_step ? *d_step : 0);
  const int k = (int)(step % g.K);
  const int first = g.meta[3 * k], ns = g.meta[3 * k + 1], G = g.meta[3 * k + 2];
  const int r = blockIdx.x;
  int64_t off = 0;
  for (int x = threadIdx.x; x < r; x += blockDim.x)
    off += g.spec[(first + dev_stream_of(g.spec, first, ns, x % G)) * 5 + 1];
  for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(0xffffffffu, off, o);
  __shared__ int64_t part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = off;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    part[0] = t;
  }
  __syncthreads();
  off = part[0];
  const int si = dev_stream_of(g.spec, first, ns, r % G);
  const int32_t* sp = g.spec + (first + si) * 5;
  const int batch = sp[1], res = sp[2], frames = sp[3], smooth = sp[4];
  if (threadIdx.x == 0) {
    rank_off[r] = off;
    if (r == g.world - 1) rank_off[g.world] = off + batch;
    if (r == 0 && scen_out) *scen_out = k;
  }
  // aspect_multiplier: CounterRng({kAspectDomain, seed, step, stream}).next_real(0.96, 1.04)
  const uint64_t akey = derive_key4(0x6173706563ULL, g.seed, (uint64_t)step, (uint64_t)si);
  const uint64_t adraw = splitmix64(akey ^ splitmix64(0));
  const double u = __dmul_rn((double)(adraw >> 11), 0x1.0p-53);
  const double mult = __dadd_rn(0.96, __dmul_rn(u, __dsub_rn(1.04, 0.96)));
  // visual_tokens (data_sim.cpp:184-191)
  const int64_t side = res / kSpatialStride;
  const int64_t scaled = llround(__dmul_rn((double)(side * side), mult));
  const int64_t latent = smooth ? llround(__ddiv_rn(__dmul_rn((double)frames, 5.0), 17.0)) : (int64_t)frames;
  int64_t vis = scaled * latent;
  vis = vis < 1 ? 1 : vis;
  const uint64_t tkey = derive_key4(0x7465787421ULL, g.seed, (uint64_t)step, (uint64_t)r);
  for (int i = threadIdx.x; i < batch; i += blockDim.x) {
    const uint64_t draw = splitmix64(tkey ^ splitmix64((uint64_t)i));
    const int64_t text = (int64_t)__umul64hi(draw, 393ull);  // next_int(0, kMaxTextTokens = 392)
    ids[off + i] = ((uint64_t)step << 32) | ((uint64_t)(r & 0xffff) << 16) | (uint64_t)(i & 0xffff);
    lens[off + i] = text + vis;
  }
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

// ------------------------------------------------------------- scenarios
extern "C" sb_status sb_scenario_create(const char* const* codes, int n_codes, int group_size, sb_scenario** out) {
  SB_API_BEGIN
  if (!out || (n_codes > 0 && !codes)) throw Error{SB_ERR_CONFIG, "sb_scenario_create: null argument"};
  *out = nullptr;
  sb_scenario sc;
  int sum = 0;
  for (int i = 0; i < n_codes; ++i) {
    sc.streams.push_back(sb::parse_code(codes[i] ? codes[i] : ""));
    sum += sc.streams.back().gpus;
  }
  sc.group_size = group_size > 0 ? group_size : sum;
  sb::validate(sc);
  *out = new sb_scenario(sc);
  SB_API_END
}

// parse_scenario (data_sim.cpp:95-129): '#' comments, CR and trailing
// blanks stripped, blank lines skipped, a 'group_size <N>' header, one data
// code per line; errors carry the line number.
extern "C" sb_status sb_scenario_parse(const char* text, sb_scenario** out) {
  SB_API_BEGIN
  if (!text || !out) throw Error{SB_ERR_CONFIG, "sb_scenario_parse: null argument"};
  *out = nullptr;
  sb_scenario sc;
  std::istringstream in(text);
  std::string line;
  size_t line_no = 0;
  bool have_header = false;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    while (!line.empty() && (line.back() == ' ' || line.back() == '\t')) line.pop_back();
    if (line.empty()) continue;
    if (!have_header) {
      std::istringstream ls(line);
      std::string key;
      ls >> key;
      if (key != "group_size" || !(ls >> sc.group_size) || !(ls >> std::ws).eof())
        throw Error{SB_ERR_PARSE, sb::parse_msg("line " + std::to_string(line_no) + ": expected 'group_size <N>' header",
                                                line_no)};
      have_header = true;
      continue;
    }
    try {
      sc.streams.push_back(sb::parse_code(line));
    } catch (const Error& e) {
      throw Error{SB_ERR_PARSE, sb::parse_msg("line " + std::to_string(line_no) + ": " + e.msg, line_no)};
    }
  }
  if (!have_header) throw Error{SB_ERR_PARSE, sb::parse_msg("scenario file missing 'group_size' header", 0)};
  sb::validate(sc);
  *out = new sb_scenario(sc);
  SB_API_END
}

extern "C" sb_status sb_scenario_preset(const char* name, sb_scenario** out) {  // data_sim.cpp:152-170
  SB_API_BEGIN
  if (!name || !out) throw Error{SB_ERR_CONFIG, "sb_scenario_preset: null argument"};
  const std::string n = name;
  std::vector<const char*> codes;
  if (n == "lowres_image") codes = {"g32b32i256f1s0"};
  else if (n == "mixed_image") codes = {"g16b4i256f1s0", "g4b5i512f1s0", "g4b5i1024f1s0", "g8b1i2048f1s0"};
  else if (n == "joint_image_video")
    codes = {"g8b4i256f1s0", "g2b5i512f1s0", "g2b5i1024f1s0", "g4b1i2048f1s0",
             "g1b10i256f4s0", "g3b1i512f4s0", "g8b2i256f85s1", "g4b1i512f85s1"};
  else
    throw Error{SB_ERR_CONFIG, "unknown scenario preset '" + n + "'; known: lowres_image, mixed_image, joint_image_video"};
  return sb_scenario_create(codes.data(), (int)codes.size(), 0, out);
  SB_API_END
}

extern "C" sb_status sb_scenario_destroy(sb_scenario* sc) {
  delete sc;
  return SB_OK;
}

extern "C" sb_status sb_scenario_info(const sb_scenario* sc, int* group_size, int* n_streams, int32_t* specs5) {
  SB_API_BEGIN
  if (!sc) throw Error{SB_ERR_CONFIG, "null scenario"};
  if (group_size) *group_size = sc->group_size;
  if (n_streams) *n_streams = (int)sc->streams.size();
  if (specs5)
    for (size_t i = 0; i < sc->streams.size(); ++i) {
      const sb::Spec& s = sc->streams[i];
      const int32_t v[5] = {s.gpus, s.batch, s.res, s.frames, s.smooth};
      std::memcpy(specs5 + 5 * i, v, sizeof v);
    }
  SB_API_END
}

extern "C" sb_status sb_schedule_create(const sb_scenario* const* sc, int K, int world, uint64_t seed,
                                        sb_schedule** out) {
  SB_API_BEGIN
  if (!sc || K < 1 || !out) throw Error{SB_ERR_CONFIG, "sb_schedule_create: need >= 1 scenario"};
  if (world < 1) throw Error{SB_ERR_CONFIG, "world_size must be >= 1"};
  *out = nullptr;
  std::vector<int32_t> spec, meta;
  int64_t max_seqs = 0, max_rows = 0;
  for (int k = 0; k < K; ++k) {
    if (!sc[k]) throw Error{SB_ERR_CONFIG, "null scenario"};
    sb::validate(*sc[k]);
    if (world % sc[k]->group_size != 0)  // ScenarioConfig::validate (simulator.cpp:15-21)
      throw Error{SB_ERR_CONFIG, "world_size " + std::to_string(world) +
                                     " is not a multiple of the data sharding group " +
                                     std::to_string(sc[k]->group_size)};
    meta.push_back((int32_t)(spec.size() / 5));
    meta.push_back((int32_t)sc[k]->streams.size());
    meta.push_back(sc[k]->group_size);
    for (const sb::Spec& s : sc[k]->streams) spec.insert(spec.end(), {s.gpus, s.batch, s.res, s.frames, s.smooth});
    int64_t seqs = 0, rows = 0;
    for (int r = 0; r < world; ++r) {
      const sb::Spec& s = sc[k]->streams[sb::stream_of_rank(*sc[k], r % sc[k]->group_size)];
      seqs += s.batch;
      rows += (int64_t)s.batch * (392 + sb::max_visual(s));
    }
    max_seqs = std::max(max_seqs, seqs);
    max_rows = std::max(max_rows, rows);
  }
  sb_schedule* s = new sb_schedule();
  s->world = world;
  s->K = K;
  s->seed = seed;
  s->max_seqs = max_seqs;
  s->max_rows = max_rows;
  try {
    SB_CUDA(cudaMalloc(&s->d_spec, sizeof(int32_t) * spec.size()));
    SB_CUDA(cudaMalloc(&s->d_meta, sizeof(int32_t) * meta.size()));
    SB_CUDA(cudaMemcpy(s->d_spec, spec.data(), sizeof(int32_t) * spec.size(), cudaMemcpyHostToDevice));
    SB_CUDA(cudaMemcpy(s->d_meta, meta.data(), sizeof(int32_t) * meta.size(), cudaMemcpyHostToDevice));
  } catch (...) {
    cudaFree(s->d_spec);
    cudaFree(s->d_meta);
    delete s;
    throw;
  }
  *out = s;
  SB_API_END
}

extern "C" sb_status sb_schedule_destroy(sb_schedule* s) {
  if (s) {
    cudaFree(s->d_spec);
    cudaFree(s->d_meta);
    delete s;
  }
  return SB_OK;
}

extern "C" sb_status sb_schedule_bounds(const sb_schedule* s, int64_t* max_seqs, int64_t* max_rows) {
  SB_API_BEGIN
  if (!s) throw Error{SB_ERR_CONFIG, "null schedule"};
  if (max_seqs) *max_seqs = s->max_seqs;
  if (max_rows) *max_rows = s->max_rows;
  SB_API_END
}

static sb::GenArgs gen_args(const sb_schedule* s) {
  sb::GenArgs g;
  g.spec = s->d_spec;
  g.meta = s->d_meta;
  g.K = s->K;
  g.world = s->world;
  g.seed = s->seed;
  return g;
}

extern "C" sb_status sb_schedule_generate(const sb_schedule* s, int64_t step, const int64_t* d_step, uint64_t* d_ids,
                                          int64_t* d_lens, int64_t* d_rank_off, sb_stream stream) {
  SB_API_BEGIN
  if (!s || !d_ids || !d_lens || !d_rank_off) throw Error{SB_ERR_CONFIG, "sb_schedule_generate: null argument"};
  if (step < 0) throw Error{SB_ERR_CONFIG, "step must be >= 0"};
  sb::k_generate<<<s->world, 256, 0, (cudaStream_t)stream>>>(gen_args(s), step, d_step, d_ids, d_lens, d_rank_off,
                                                             nullptr);
  SB_CHECK_LAUNCH();
  sb::count_launch();
  SB_API_END
}

// ---------------------------------------------------------------- driver
// One step's device state: its gathered metadata, planner and the five
// worlds of simulate_step (A origin, B routed, C Ulysses, D post, E returned).
struct DriverSlot {
  sb_planner* p = nullptr;
  bool own_p = false;
  sb_world* w[5] = {};
  uint64_t* ids = nullptr;
  int64_t* lens = nullptr;
  int64_t* rank_off = nullptr;
  int32_t* scen = nullptr;
  sb_step_record* stage = nullptr;  // the step's record until its copies (and checks) are done
};

struct sb_driver {
  sb_schedule* s = nullptr;
  int verify = 0, uly = 0;
  int n_heads = 0;
  int64_t row_bytes = 0;
  // slot 0 plans with the caller's planner; slot 1 (plan-ahead only) with a clone
  DriverSlot slot[2];
  int cur = 0;    // slot of the next step
  int last = 0;   // slot of the most recently issued step
  bool pipeline = false, primed = false;
  int64_t* d_step = nullptr;  // [0] next step; [1] steps run; [2] failed checks; [3] next step to generate
  uint64_t* d_acc = nullptr;  // [0..2] checksums, [3..4] compare counts
  sb_step_record* d_rec = nullptr;
  int64_t rec_cap = 0;
  // plan + exchange preparations run on a side stream: under the witness
  // fill and the earlier copies (serial schedule), or a whole step ahead
  // (plan-ahead); ev[0] fork, ev[1..4] slot prepared
  cudaStream_t side = nullptr;
  cudaEvent_t ev[5] = {};
};

namespace sb {

// Step record from the device plan + the meta (balancer.hpp:78-89 report,
// the reference harness's max/mean).  The step index is the generator's
// counter, which this kernel advances.
__global__ void k_record(sb_step_record* stage, int64_t* d_gen, const int32_t* scen, const int64_t* lens,
                         const int64_t* rank_off, int W, const int64_t* n_chunks, const double* per_gpu,
                         const double* wir, const double* total, const int32_t* viol) {
  __shared__ int64_t part[32];
  const int64_t n = rank_off[W];
  int64_t t = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) t += lens[i];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x != 0) return;
  int64_t tokens = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tokens += part[w];
  const int64_t step = *d_gen;
  sb_step_record& r = *stage;
  r.step = step;
  r.tokens = tokens;
  r.sequences = n;
  r.chunks = *n_chunks;
  r.wir = *wir;
  double mx = 0.0, sum = 0.0;
  for (int q = 0; q < W; ++q) {
    mx = fmax(mx, per_gpu[q]);
    sum = __dadd_rn(sum, per_gpu[q]);
  }
  r.max_over_mean = sum > 0.0 ? __ddiv_rn(mx, __ddiv_rn(sum, (double)W)) : 1.0;
  r.total_workload = *total;
  r.checksum = 0;
  r.scenario = *scen;
  r.capacity_violations = *viol;
  r.checks = 0;
  r.verified = 0;
  *d_gen = step + 1;
}

// Closes a step: its record (plus the inline check bits) enters the ring.
__global__ void k_record_checks(sb_step_record* rec, int64_t cap, int64_t* d_step, const sb_step_record* stage,
                                const uint64_t* acc, int uly, int verify) {
  if (threadIdx.x != 0) return;
  sb_step_record r = *stage;
  if (verify) {
    int c = 0;
    c |= acc[1] == acc[0] ? SB_CHECK_ROUTE_CONSERVED : 0;
    c |= (!uly || acc[2] == acc[0]) ? SB_CHECK_PRE_CONSERVED : 0;
    c |= acc[3] == 0 ? SB_CHECK_POST_INVERTS_PRE : 0;
    c |= acc[4] == 0 ? SB_CHECK_REVERSE_RESTORES : 0;
    r.checks = c;
    r.verified = 1;
    r.checksum = acc[0];
    if (c != SB_CHECK_ALL) d_step[2] += 1;
  }
  rec[r.step % cap] = r;
  d_step[0] = r.step + 1;
  d_step[1] += 1;
}

static void ck(sb_status st) {
  if (st != SB_OK) throw Error{st, sb_last_error()};
}

static void slot_alloc(sb_driver* d, DriverSlot& x, sb_planner* p, bool own) {
  x.p = p;
  x.own_p = own;
  const int64_t rb[1] = {d->row_bytes};
  sb_world_desc wd{};
  wd.world_size = p->W;
  wd.n_local = p->W;
  wd.first_local = 0;
  wd.n_heads = d->n_heads;
  wd.n_payload = 1;
  wd.n_aux = 0;
  wd.row_bytes = rb;
  wd.capacity_rows = d->s->max_rows;
  wd.max_bag = p->max_bag;
  for (auto& w : x.w) ck(sb_world_create(&wd, &w));
  SB_CUDA(cudaMalloc(&x.ids, sizeof(uint64_t) * (size_t)std::max<int64_t>(1, d->s->max_seqs)));
  SB_CUDA(cudaMalloc(&x.lens, sizeof(int64_t) * (size_t)std::max<int64_t>(1, d->s->max_seqs)));
  SB_CUDA(cudaMalloc(&x.rank_off, sizeof(int64_t) * (size_t)(p->W + 1)));
  SB_CUDA(cudaMalloc(&x.scen, sizeof(int32_t)));
  SB_CUDA(cudaMalloc(&x.stage, sizeof(sb_step_record)));
  SB_CUDA(cudaMemset(x.stage, 0, sizeof(sb_step_record)));
}

static void slot_free(DriverSlot& x) {
  for (auto& w : x.w)
    if (w) sb_world_destroy(w);
  void* ptrs[] = {x.ids, x.lens, x.rank_off, x.scen, x.stage};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (x.own_p && x.p) sb_planner_destroy(x.p);
  x = DriverSlot{};
}

static void launch_generate(sb_driver* d, DriverSlot& x, cudaStream_t st) {
  k_generate<<<d->s->world, 256, 0, st>>>(gen_args(d->s), 0, d->d_step + 3, x.ids, x.lens, x.rank_off, x.scen);
  SB_CHECK_LAUNCH();
  count_launch();
}

static void launch_record(sb_driver* d, DriverSlot& x, cudaStream_t st) {
  k_record<<<1, 1024, 0, st>>>(x.stage, d->d_step + 3, x.scen, x.lens, x.rank_off, x.p->W, x.p->n_chunks,
                               x.p->per_gpu, x.p->wir, x.p->total, x.p->violations);
  SB_CHECK_LAUNCH();
  count_launch();
}

static void fill_origin(sb_driver* d, DriverSlot& x, sb_stream st) {
  // With verification the origin payload is the reference witness (the
  // checks need it); timed steps write the row metadata only -- the payload
  // stands for hidden states produced upstream, as the reference's CPU
  // timing excludes make_world.
  if (d->verify) ck(sb_world_fill_witness(x.w[0], x.ids, x.lens, x.rank_off, st));
  else ck(sb_world_fill_meta(x.w[0], x.ids, x.lens, x.rank_off, st));
}

// Everything of a step that precedes its data movement -- generate, origin
// layout + rows, plan, record, the four exchange preparations -- on one
// stream (the plan-ahead schedule runs it a step early on the side stream).
static void prepare_step(sb_driver* d, DriverSlot& x, cudaStream_t st) {
  const sb_stream sst = (sb_stream)st;
  sb_world *A = x.w[0], *B = x.w[1], *C = x.w[2], *D = x.w[3], *E = x.w[4];
  launch_generate(d, x, st);
  ck(sb_world_layout_origin(A, x.lens, x.rank_off, sst));
  fill_origin(d, x, sst);
  ck(sb_plan(x.p, x.ids, x.lens, x.rank_off, sst));
  ck(sb_exchange_prepare(x.p, 0, A, B, 0, sst));
  if (d->uly) {
    ck(sb_exchange_prepare(x.p, 2, B, C, 2, sst));
    ck(sb_exchange_prepare(x.p, 3, C, D, 3, sst));
  }
  ck(sb_exchange_prepare(x.p, 1, d->uly ? D : B, E, 1, sst));
  launch_record(d, x, st);
}

// The data movement of a prepared step, with simulate_step's checks under
// verify.  `wait` (serial schedule): slot k's copy first waits for ev[k].
static void move_step(sb_driver* d, DriverSlot& x, cudaStream_t s, bool wait) {
  const sb_stream st = (sb_stream)s;
  sb_world *A = x.w[0], *B = x.w[1], *C = x.w[2], *D = x.w[3], *E = x.w[4];
  sb_world* back_src = d->uly ? D : B;
  if (d->verify) {
    SB_CUDA(cudaMemsetAsync(d->d_acc, 0, sizeof(uint64_t) * 5, s));
    ck(sb_world_checksum(A, d->d_acc + 0, st));
  }
  if (wait) SB_CUDA(cudaStreamWaitEvent(s, d->ev[1], 0));
  ck(sb_exchange_run(x.p, 0, st));
  if (d->verify) ck(sb_world_checksum(B, d->d_acc + 1, st));
  if (d->uly) {
    if (wait) SB_CUDA(cudaStreamWaitEvent(s, d->ev[2], 0));
    ck(sb_exchange_run(x.p, 2, st));
    if (d->verify) ck(sb_world_checksum(C, d->d_acc + 2, st));
    if (wait) SB_CUDA(cudaStreamWaitEvent(s, d->ev[3], 0));
    ck(sb_exchange_run(x.p, 3, st));
    if (d->verify) ck(sb_world_compare(D, B, d->d_acc + 3, st));
  }
  // simulated transformer output: every row shifts by block_perturbation
  // (simulator.cpp:128-136); the reverse route must carry it home
  if (d->verify) ck(sb_world_perturb(back_src, st));
  if (wait) SB_CUDA(cudaStreamWaitEvent(s, d->ev[4], 0));  // also joins the side stream (record, plan)
  ck(sb_exchange_run(x.p, 1, st));
  if (d->verify) {
    ck(sb_world_perturb(A, st));  // expected: the original world, perturbed
    ck(sb_world_compare(E, A, d->d_acc + 4, st));
  }
}

static void close_step(sb_driver* d, DriverSlot& x, cudaStream_t s) {
  k_record_checks<<<1, 32, 0, s>>>(d->d_rec, d->rec_cap, d->d_step, x.stage, d->d_acc, d->uly, d->verify);
  SB_CHECK_LAUNCH();
  count_launch();
}

}  // namespace sb

extern "C" sb_status sb_driver_create(sb_planner* p, const sb_schedule* s, int n_heads, int64_t payload_row_bytes,
                                      int verify, int64_t record_cap, sb_driver** out) {
  SB_API_BEGIN
  if (!p || !s || !out) throw Error{SB_ERR_CONFIG, "sb_driver_create: null argument"};
  *out = nullptr;
  if (p->W != s->world) throw Error{SB_ERR_CONFIG, "planner world size differs from the schedule's"};
  if (p->max_seqs < s->max_seqs)
    throw Error{SB_ERR_CAPACITY, "planner max_seqs " + std::to_string(p->max_seqs) + " below the schedule's bound " +
                                     std::to_string(s->max_seqs)};
  if (payload_row_bytes <= 0 || payload_row_bytes % 16 != 0 || payload_row_bytes % 8 != 0)
    throw Error{SB_ERR_CONFIG, "payload row bytes must be a positive multiple of 16"};
  sb_driver* d = new sb_driver();
  d->s = const_cast<sb_schedule*>(s);
  d->verify = verify ? 1 : 0;
  d->uly = p->any_multi_bag ? 1 : 0;
  d->n_heads = n_heads;
  d->row_bytes = payload_row_bytes;
  d->rec_cap = record_cap > 0 ? record_cap : 1;
  try {
    sb::slot_alloc(d, d->slot[0], p, false);
    SB_CUDA(cudaMalloc(&d->d_step, sizeof(int64_t) * 4));
    SB_CUDA(cudaMemset(d->d_step, 0, sizeof(int64_t) * 4));
    SB_CUDA(cudaMalloc(&d->d_acc, sizeof(uint64_t) * 5));
    SB_CUDA(cudaMalloc(&d->d_rec, sizeof(sb_step_record) * (size_t)d->rec_cap));
    SB_CUDA(cudaMemset(d->d_rec, 0, sizeof(sb_step_record) * (size_t)d->rec_cap));
    int least = 0, greatest = 0;  // high priority: plan / prepare kernels jump the copy kernel's later waves
    SB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    SB_CUDA(cudaStreamCreateWithPriority(&d->side, cudaStreamNonBlocking, greatest));
    for (auto& e : d->ev) SB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  } catch (...) {
    sb_driver_destroy(d);
    throw;
  }
  *out = d;
  SB_API_END
}

extern "C" sb_status sb_driver_destroy(sb_driver* d) {
  if (!d) return SB_OK;
  for (auto& x : d->slot) sb::slot_free(x);
  void* ptrs[] = {d->d_step, d->d_acc, d->d_rec};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  for (auto& e : d->ev)
    if (e) cudaEventDestroy(e);
  if (d->side) cudaStreamDestroy(d->side);
  delete d;
  return SB_OK;
}

extern "C" sb_status sb_driver_set_step(sb_driver* d, int64_t step, sb_stream stream) {
  SB_API_BEGIN
  if (!d || step < 0) throw Error{SB_ERR_CONFIG, "sb_driver_set_step: bad argument"};
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t v[4] = {step, 0, 0, step};
  SB_CUDA(cudaMemcpyAsync(d->d_step, v, sizeof v, cudaMemcpyHostToDevice, s));
  d->primed = false;
  if (d->pipeline) {  // plan-ahead: the first step is prepared now
    sb::prepare_step(d, d->slot[d->cur], s);
    d->primed = true;
  }
  SB_CUDA(cudaStreamSynchronize(s));
  SB_API_END
}

extern "C" sb_status sb_driver_set_pipeline(sb_driver* d, int on, sb_stream stream) {
  SB_API_BEGIN
  if (!d) throw Error{SB_ERR_CONFIG, "null driver"};
  cudaStream_t s = (cudaStream_t)stream;
  SB_CUDA(cudaStreamSynchronize(s));
  if (on && !d->slot[1].p) {
    sb_planner* q = sb::planner_clone(d->slot[0].p);
    try {
      sb::slot_alloc(d, d->slot[1], q, true);
    } catch (...) {
      if (!d->slot[1].p) sb_planner_destroy(q);
      sb::slot_free(d->slot[1]);
      throw;
    }
  }
  d->pipeline = on != 0;
  d->cur = 0;
  d->last = 0;
  d->primed = false;
  // resume at the step the device counter names (a prepared-ahead step is dropped)
  SB_CUDA(cudaMemcpyAsync(d->d_step + 3, d->d_step, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  if (d->pipeline) {
    sb::prepare_step(d, d->slot[0], s);
    d->primed = true;
  }
  SB_CUDA(cudaStreamSynchronize(s));
  SB_API_END
}

// One step (simulate_step, simulator.cpp:45-178, on the device path).
// Stream-ordered, no host synchronisation: capturable into a CUDA graph
// whose replays advance the device step counter.
// Serial schedule:
//   main: generate -> origin layout -> origin fill -> route copy -> pre copy
//         -> post copy -> reverse copy -> close
//   side: plan -> prepare route / pre / post / reverse -> record
// (preparations touch only the plan and world tables, never payload, so the
// plan and every layout + job build run under the fill and the earlier
// copies; each copy waits for its own preparation).
// Plan-ahead schedule (sb_driver_set_pipeline): two slots alternate; while
// step s's copies run on the main stream, the side stream generates, lays
// out, fills, plans and prepares step s+1 in the other slot, joining before
// step s closes.  A graph must therefore hold an even number of steps.
extern "C" sb_status sb_driver_step(sb_driver* d, sb_stream stream) {
  SB_API_BEGIN
  if (!d) throw Error{SB_ERR_CONFIG, "null driver"};
  cudaStream_t s = (cudaStream_t)stream;
  sb_stream side = (sb_stream)d->side;
  if (d->pipeline) {
    DriverSlot& x = d->slot[d->cur];
    DriverSlot& y = d->slot[d->cur ^ 1];
    if (!d->primed) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      SB_CUDA(cudaStreamIsCapturing(s, &cs));
      if (cs != cudaStreamCaptureStatusNone)
        throw Error{SB_ERR_CONFIG, "plan-ahead driver: run set_step or one eager step before graph capture"};
      sb::prepare_step(d, x, s);
      d->primed = true;
    }
    SB_CUDA(cudaEventRecord(d->ev[0], s));
    SB_CUDA(cudaStreamWaitEvent(d->side, d->ev[0], 0));
    sb::prepare_step(d, y, d->side);
    SB_CUDA(cudaEventRecord(d->ev[1], d->side));
    sb::move_step(d, x, s, false);
    SB_CUDA(cudaStreamWaitEvent(s, d->ev[1], 0));
    sb::close_step(d, x, s);
    d->last = d->cur;
    d->cur ^= 1;
    return SB_OK;
  }
  DriverSlot& x = d->slot[0];
  sb_world *A = x.w[0], *B = x.w[1], *C = x.w[2], *D = x.w[3], *E = x.w[4];
  sb::launch_generate(d, x, s);
  sb::ck(sb_world_layout_origin(A, x.lens, x.rank_off, stream));
  SB_CUDA(cudaEventRecord(d->ev[0], s));
  SB_CUDA(cudaStreamWaitEvent(d->side, d->ev[0], 0));
  // side: plan, preparations, record
  sb::ck(sb_plan(x.p, x.ids, x.lens, x.rank_off, side));
  sb::ck(sb_exchange_prepare(x.p, 0, A, B, 0, side));
  SB_CUDA(cudaEventRecord(d->ev[1], d->side));
  if (d->uly) {
    sb::ck(sb_exchange_prepare(x.p, 2, B, C, 2, side));
    SB_CUDA(cudaEventRecord(d->ev[2], d->side));
    sb::ck(sb_exchange_prepare(x.p, 3, C, D, 3, side));
    SB_CUDA(cudaEventRecord(d->ev[3], d->side));
  }
  sb::ck(sb_exchange_prepare(x.p, 1, d->uly ? D : B, E, 1, side));
  sb::launch_record(d, x, d->side);
  SB_CUDA(cudaEventRecord(d->ev[4], d->side));
  // main: input synthesis, then the copies as their preparations land
  sb::fill_origin(d, x, stream);
  sb::move_step(d, x, s, true);
  sb::close_step(d, x, s);
  d->last = 0;
  SB_API_END
}

extern "C" sb_status sb_driver_run(sb_driver* d, int64_t n_steps, sb_stream stream) {
  SB_API_BEGIN
  if (!d || n_steps < 0) throw Error{SB_ERR_CONFIG, "sb_driver_run: bad argument"};
  for (int64_t i = 0; i < n_steps; ++i) {
    const sb_status st = sb_driver_step(d, stream);
    if (st != SB_OK) return st;
  }
  SB_API_END
}

extern "C" sb_status sb_driver_progress(sb_driver* d, int64_t* next_step, int64_t* steps_run, int64_t* failed,
                                        sb_stream stream) {
  SB_API_BEGIN
  if (!d) throw Error{SB_ERR_CONFIG, "null driver"};
  int64_t v[3];
  SB_CUDA(cudaMemcpyAsync(v, d->d_step, sizeof v, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  SB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (next_step) *next_step = v[0];
  if (steps_run) *steps_run = v[1];
  if (failed) *failed = v[2];
  SB_API_END
}

extern "C" sb_status sb_driver_records(sb_driver* d, sb_step_record* host, int64_t capacity, int64_t* n_out,
                                       sb_stream stream) {
  SB_API_BEGIN
  if (!d || !n_out) throw Error{SB_ERR_CONFIG, "sb_driver_records: null argument"};
  const int64_t n = std::min(capacity, d->rec_cap);
  if (host && n > 0) {
    SB_CUDA(cudaMemcpyAsync(host, d->d_rec, sizeof(sb_step_record) * (size_t)n, cudaMemcpyDeviceToHost,
                            (cudaStream_t)stream));
    SB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  }
  *n_out = d->rec_cap;
  SB_API_END
}

extern "C" sb_status sb_driver_world(const sb_driver* d, int which, sb_world** out) {
  SB_API_BEGIN
  if (!d || !out || which < 0 || which > 4) throw Error{SB_ERR_CONFIG, "sb_driver_world: bad argument"};
  *out = d->slot[d->last].w[which];
  SB_API_END
}

extern "C" sb_status sb_driver_meta(const sb_driver* d, const uint64_t** ids, const int64_t** lens,
                                    const int64_t** rank_off) {
  SB_API_BEGIN
  if (!d) throw Error{SB_ERR_CONFIG, "null driver"};
  const DriverSlot& x = d->slot[d->last];
  if (ids) *ids = x.ids;
  if (lens) *lens = x.lens;
  if (rank_off) *rank_off = x.rank_off;
  SB_API_END
}
