// SPDX-License-Identifier: Apache-2.0
//
// libseqbal.so: the reference's data-simulator and uniform-balancer API
// (data_sim.hpp:11-102, balancer.hpp:122-144) over the C-ABI.  The grammar
// and presets parse in sb_scenario_* (host), next_batch runs the device
// generator (sb_schedule_generate), balance_uniform_items the device planner
// (sb_uniform_plan).  The scalar helpers (visual_tokens, aspect_multiplier,
// ...) are the reference formulas, used to split a generated length into its
// text / visual parts.
#include <cmath>
#include <cstring>
#include <fstream>
#include <istream>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "seqbal/seqbal.hpp"
#include "seqbal_capi.h"

namespace seqbal {
namespace {

// C-ABI error -> reference exception; a ParseError's message ends in
// " (at offset N)" (error.hpp:10-21), which the C++ constructor re-appends.
[[noreturn]] void raise_ext(sb_status st, const char* where) {
  std::string msg = sb_last_error();
  switch (st) {
    case SB_ERR_PARSE: {
      std::size_t off = 0;
      const auto at = msg.rfind(" (at offset ");
      if (at != std::string::npos && msg.back() == ')') {
        off = std::stoull(msg.substr(at + 12, msg.size() - at - 13));
        msg.erase(at);
      }
      throw ParseError(msg, off);
    }
    case SB_ERR_CONFIG: throw ConfigError(msg);
    case SB_ERR_INTEGRITY: throw IntegrityError(msg);
    default: throw std::runtime_error(std::string(where) + ": " + msg);
  }
}

void ckx(sb_status st, const char* where) {
  if (st != SB_OK) raise_ext(st, where);
}

struct ScenarioHandle {
  sb_scenario* p = nullptr;
  ~ScenarioHandle() {
    if (p) sb_scenario_destroy(p);
  }
};

ShardingGroupConfig from_handle(sb_scenario* sc) {
  int g = 0, n = 0;
  ckx(sb_scenario_info(sc, &g, &n, nullptr), "scenario");
  std::vector<int32_t> spec(5 * static_cast<size_t>(n));
  ckx(sb_scenario_info(sc, nullptr, nullptr, spec.data()), "scenario");
  ShardingGroupConfig cfg;
  cfg.group_size = g;
  for (int i = 0; i < n; ++i)
    cfg.streams.push_back({spec[5 * i], spec[5 * i + 1], spec[5 * i + 2], spec[5 * i + 3], spec[5 * i + 4] != 0});
  return cfg;
}

void to_handle(const ShardingGroupConfig& cfg, ScenarioHandle& h) {
  std::vector<std::string> codes;
  for (const StreamSpec& s : cfg.streams) codes.push_back(format_data_code(s));
  std::vector<const char*> ptrs;
  for (const auto& c : codes) ptrs.push_back(c.c_str());
  ckx(sb_scenario_create(ptrs.data(), static_cast<int>(ptrs.size()), cfg.group_size, &h.p), "scenario");
}

// Device int64 buffers carved from a staging world's arenas.
struct DevI64 {
  sb_world* w = nullptr;
  void* a[3] = {};
  int64_t cap = 0;
  ~DevI64() {
    if (w) sb_world_destroy(w);
  }
  void ensure(int64_t n) {
    if (cap >= n) return;
    if (w) sb_world_destroy(w);
    w = nullptr;
    sb_world_desc d{};
    const int64_t rb[2] = {8, 8};
    d.world_size = 1;
    d.n_local = 1;
    d.n_heads = 1;
    d.n_payload = 2;
    d.row_bytes = rb;
    d.capacity_rows = n;
    d.max_bag = 1;
    ckx(sb_world_create(&d, &w), "device staging");
    int64_t bytes = 0;
    for (int t = 0; t < 3; ++t) ckx(sb_world_arena(w, t, &a[t], &bytes), "device staging");
    cap = n;
  }
  void download(void* const* host, const int64_t* bytes) { ckx(sb_world_download(w, host, bytes, nullptr), "download"); }
  void upload(void* const* host, const int64_t* bytes) { ckx(sb_world_upload(w, host, bytes, nullptr), "upload"); }
};

std::mutex& ext_mu() {
  static std::mutex* m = new std::mutex();
  return *m;
}

constexpr std::uint64_t kAspectDomain = 0x6173706563ULL;  // data_sim.cpp:207-208

std::uint64_t sm64(std::uint64_t x) {  // rng.hpp:12-17
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

}  // namespace

StreamSpec parse_data_code(std::string_view code) {
  const std::string c(code);
  const char* a[1] = {c.c_str()};
  ScenarioHandle h;
  ckx(sb_scenario_create(a, 1, 0, &h.p), "parse_data_code");
  return from_handle(h.p).streams.at(0);
}

std::string format_data_code(const StreamSpec& spec) {  // data_sim.cpp:78-82
  return "g" + std::to_string(spec.gpus) + "b" + std::to_string(spec.batch_per_gpu) + "i" +
         std::to_string(spec.resolution) + "f" + std::to_string(spec.frames) + "s" + (spec.smooth ? "1" : "0");
}

void ShardingGroupConfig::validate() const {  // data_sim.cpp:84-93
  if (group_size < 1) throw ConfigError("group_size must be >= 1");
  if (streams.empty()) throw ConfigError("scenario has no data streams");
  int total = 0;
  for (const StreamSpec& s : streams) total += s.gpus;
  if (total != group_size)
    throw ConfigError("stream GPU counts sum to " + std::to_string(total) + " but group_size is " +
                      std::to_string(group_size));
}

ShardingGroupConfig parse_scenario(std::istream& in) {
  std::stringstream ss;
  ss << in.rdbuf();
  ScenarioHandle h;
  ckx(sb_scenario_parse(ss.str().c_str(), &h.p), "parse_scenario");
  return from_handle(h.p);
}

ShardingGroupConfig parse_scenario_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open scenario file: " + path);
  return parse_scenario(in);
}

ShardingGroupConfig scenario_preset(std::string_view name) {
  const std::string n(name);
  ScenarioHandle h;
  ckx(sb_scenario_preset(n.c_str(), &h.p), "scenario_preset");
  return from_handle(h.p);
}

ShardingGroupConfig preset_lowres_image() { return scenario_preset("lowres_image"); }
ShardingGroupConfig preset_mixed_image() { return scenario_preset("mixed_image"); }
ShardingGroupConfig preset_joint_image_video() { return scenario_preset("joint_image_video"); }
std::vector<std::string> scenario_preset_names() { return {"lowres_image", "mixed_image", "joint_image_video"}; }

std::int64_t latent_frames(const StreamSpec& spec) {  // data_sim.cpp:179-182
  if (!spec.smooth) return spec.frames;
  return std::llround(static_cast<double>(spec.frames) * kTemporalNum / kTemporalDen);
}

std::int64_t visual_tokens(const StreamSpec& spec, double mult) {  // data_sim.cpp:184-191
  const std::int64_t side = spec.resolution / kSpatialStride;
  const std::int64_t scaled = std::llround(static_cast<double>(side * side) * mult);
  const std::int64_t tokens = scaled * latent_frames(spec);
  return tokens < 1 ? 1 : tokens;
}

int stream_of_rank(const ShardingGroupConfig& config, int group_rank) {  // data_sim.cpp:193-203
  if (group_rank < 0 || group_rank >= config.group_size)
    throw ConfigError("rank " + std::to_string(group_rank) + " outside sharding group of " +
                      std::to_string(config.group_size));
  int cursor = 0;
  for (std::size_t i = 0; i < config.streams.size(); ++i) {
    cursor += config.streams[i].gpus;
    if (group_rank < cursor) return static_cast<int>(i);
  }
  throw ConfigError("rank not covered by any stream");
}

double aspect_multiplier(std::uint64_t seed, std::int64_t step, int stream_index) {  // data_sim.cpp:210-214
  std::uint64_t k = 0x8f51a7c0c0c0f5a3ULL;  // derive_key (rng.hpp:20-24)
  for (std::uint64_t part : {kAspectDomain, seed, static_cast<std::uint64_t>(step),
                             static_cast<std::uint64_t>(stream_index)})
    k = sm64(k ^ part);
  const double u = static_cast<double>(sm64(k ^ sm64(0)) >> 11) * 0x1.0p-53;  // CounterRng::next_real
  return kAspectMultMin + u * (kAspectMultMax - kAspectMultMin);
}

std::uint64_t make_sample_id(std::int64_t step, int rank, int index) {  // data_sim.cpp:219-223
  return (static_cast<std::uint64_t>(step) << 32) | (static_cast<std::uint64_t>(rank & 0xffff) << 16) |
         static_cast<std::uint64_t>(index & 0xffff);
}

SampleMeta dummy_sample(int rank, std::int64_t step) {  // data_sim.cpp:250-257
  SampleMeta s;
  s.sample_id = make_sample_id(step, rank, 0);
  s.text_len = 0;
  s.visual_len = 1;
  s.origin_rank = rank;
  return s;
}

std::vector<SampleMeta> next_batch(const ShardingGroupConfig& config, int rank, std::int64_t step,
                                   std::uint64_t seed) {
  config.validate();
  if (rank < 0) throw ConfigError("rank must be >= 0");
  if (step < 0) throw ConfigError("step must be >= 0");
  const int G = config.group_size;
  const int world = (rank / G + 1) * G;
  std::lock_guard<std::mutex> lock(ext_mu());
  ScenarioHandle h;
  to_handle(config, h);
  sb_schedule* sch = nullptr;
  const sb_scenario* one[1] = {h.p};
  ckx(sb_schedule_create(one, 1, world, seed, &sch), "next_batch");
  struct Guard {
    sb_schedule* s;
    ~Guard() { sb_schedule_destroy(s); }
  } guard{sch};
  int64_t max_seqs = 0;
  ckx(sb_schedule_bounds(sch, &max_seqs, nullptr), "next_batch");
  static DevI64* buf = new DevI64();
  buf->ensure(std::max<int64_t>(max_seqs, world + 1) + 1);
  ckx(sb_schedule_generate(sch, step, nullptr, static_cast<uint64_t*>(buf->a[1]), static_cast<int64_t*>(buf->a[2]),
                           static_cast<int64_t*>(buf->a[0]), nullptr),
      "next_batch");
  std::vector<int64_t> off(static_cast<size_t>(world) + 1);
  std::vector<uint64_t> ids(static_cast<size_t>(max_seqs));
  std::vector<int64_t> lens(static_cast<size_t>(max_seqs));
  void* host[3] = {off.data(), ids.data(), lens.data()};
  const int64_t bytes[3] = {static_cast<int64_t>(off.size() * 8), static_cast<int64_t>(ids.size() * 8),
                            static_cast<int64_t>(lens.size() * 8)};
  buf->download(host, bytes);
  const int si = stream_of_rank(config, rank % G);
  const std::int64_t vis = visual_tokens(config.streams[si], aspect_multiplier(seed, step, si));
  std::vector<SampleMeta> out;
  for (int64_t i = off[rank]; i < off[rank + 1]; ++i) {
    SampleMeta m;
    m.sample_id = ids[i];
    m.visual_len = vis;
    m.text_len = lens[i] - vis;
    m.origin_rank = rank;
    out.push_back(m);
  }
  return out;
}

UniformPlan balance_uniform_items(const std::vector<std::int64_t>& counts) {
  UniformPlan plan;
  const int n = static_cast<int>(counts.size());
  if (n == 0) return plan;
  for (std::int64_t c : counts)
    if (c < 0) throw ConfigError("balance_uniform_items: negative count");
  std::lock_guard<std::mutex> lock(ext_mu());
  static DevI64* buf = new DevI64();
  buf->ensure(n);
  void* host[3] = {nullptr, const_cast<std::int64_t*>(counts.data()), nullptr};
  const int64_t bytes[3] = {0, static_cast<int64_t>(n) * 8, 0};
  buf->upload(host, bytes);
  sb_uniform* u = nullptr;
  ckx(sb_uniform_create(n, &u), "balance_uniform_items");
  struct Guard {
    sb_uniform* u;
    ~Guard() { sb_uniform_destroy(u); }
  } guard{u};
  ckx(sb_uniform_plan(u, static_cast<const int64_t*>(buf->a[1]), nullptr), "balance_uniform_items");
  plan.final_counts.resize(n);
  std::vector<int64_t> mv(6 * static_cast<size_t>(n));
  int64_t nm = 0, tot = 0;
  ckx(sb_uniform_download(u, plan.final_counts.data(), mv.data(), &nm, &tot, nullptr), "balance_uniform_items");
  for (int64_t i = 0; i < nm; ++i)
    plan.moves.push_back({static_cast<int>(mv[3 * i]), static_cast<int>(mv[3 * i + 1]), mv[3 * i + 2]});
  plan.total_moved = tot;
  return plan;
}

UniformPlan reverse_uniform_plan(const UniformPlan& plan, const std::vector<std::int64_t>& original_counts) {
  UniformPlan rev;  // balancer.cpp:450-460
  rev.final_counts = original_counts;
  rev.total_moved = plan.total_moved;
  for (const UniformMove& m : plan.moves) rev.moves.push_back({m.dst_rank, m.src_rank, m.count});
  return rev;
}

}  // namespace seqbal
