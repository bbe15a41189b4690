// Test infrastructure only (never shipped, never on the product path).
//
// A small harness that drives the UNMODIFIED reference `seqbal` library
// (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/) through its public C++ API.  Two jobs:
//
//   ref_harness dump  < case.json  > result.json
//       Runs plan_routing / reverse_plan / identity_plan / route /
//       reverse_route / pre_attn / post_attn on one case and prints the
//       results (full arrays for small cases, digests for large ones).
//       tests/golden/make_golden.py uses this to write the committed
//       golden fixtures that pin oracle/seqbal_oracle.c and the CUDA path.
//
//   ref_harness bench < config.json
//       Times the reference CPU path (plan + route + Ulysses round trip per
//       multi-GPU bag + reverse_route) on a bench config; bench.py's
//       `--impl reference` arm and `cpu_baseline` leg read its JSON line.
//
// Reference API used (all under /root/reference/proj/include/seqbal/):
//   balancer.hpp:95-104 plan_routing / identity_plan / reverse_plan
//   exchange.hpp:56-81  make_world / gather_sequence_info / route /
//                       reverse_route / pre_attn / post_attn
//   data_sim.hpp:95-101 next_batch / make_sample_id
//   rng.hpp:12-55       derive_key / CounterRng
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include <omp.h>

#include "json.hpp"
#include "seqbal/balancer.hpp"
#include "seqbal/data_sim.hpp"
#include "seqbal/error.hpp"
#include "seqbal/exchange.hpp"
#include "seqbal/rng.hpp"
#include "seqbal/topology.hpp"
#include "seqbal/workload_model.hpp"

using nlohmann::json;
using namespace seqbal;

namespace {

// Byte digest shared with oracle/seqbal_oracle.c (or_digest): fold every
// little-endian 8-byte word (zero-padded tail) through splitmix64.
std::uint64_t digest_bytes(const void* data, std::size_t n, std::uint64_t h = 0x6469676573740000ULL) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  std::size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    std::uint64_t w;
    std::memcpy(&w, p + i, 8);
    h = splitmix64(h ^ w);
  }
  if (i < n) {
    std::uint64_t w = 0;
    std::memcpy(&w, p + i, n - i);
    h = splitmix64(h ^ w);
  }
  return h;
}

std::string hex64(std::uint64_t v) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(v));
  return buf;
}

std::string dbits(double d) {
  std::uint64_t b;
  std::memcpy(&b, &d, 8);
  return hex64(b);
}

WorkloadModel model_from(const json& j) {
  WorkloadModel m;
  m.shape.d_model = j.value("d_model", 3072);
  m.shape.n_heads = j.value("n_heads", 24);
  m.shape.d_head = j.value("d_head", 128);
  m.shape.n_blocks = j.value("n_blocks", 57);
  m.gamma = j.value("gamma", 0.49);
  return m;
}

// Per-rank sample metadata for a case.  Generators follow SURVEY.md 8(d).
std::vector<std::vector<SampleMeta>> samples_from(const json& meta, int world) {
  std::vector<std::vector<SampleMeta>> out(world);
  const std::string kind = meta.at("kind");
  if (kind == "explicit") {
    const auto& lens = meta.at("lens");
    const bool have_ids = meta.contains("ids");
    std::uint64_t next = 1;
    for (int r = 0; r < world; ++r) {
      for (std::size_t i = 0; i < lens[r].size(); ++i) {
        SampleMeta s;
        s.sample_id = have_ids ? meta["ids"][r][i].get<std::uint64_t>() : next++;
        s.text_len = 0;
        s.visual_len = lens[r][i].get<std::int64_t>();
        s.origin_rank = r;
        out[r].push_back(s);
      }
    }
  } else if (kind == "c1") {
    // C1: one CounterRng({seed, step, rank}) per rank; text U[64,512] then
    // image U[256,4096]; id make_sample_id(step, rank, i).
    const std::uint64_t seed = meta.at("seed");
    const std::int64_t step = meta.at("step");
    const int per_rank = meta.at("per_rank");
    for (int r = 0; r < world; ++r) {
      CounterRng rng({seed, static_cast<std::uint64_t>(step), static_cast<std::uint64_t>(r)});
      for (int i = 0; i < per_rank; ++i) {
        SampleMeta s;
        s.sample_id = make_sample_id(step, r, i);
        s.text_len = rng.next_int(64, 512);
        s.visual_len = rng.next_int(256, 4096);
        s.origin_rank = r;
        out[r].push_back(s);
      }
    }
  } else if (kind == "scenario") {
    ShardingGroupConfig cfg;
    cfg.group_size = meta.at("group_size");
    for (const auto& c : meta.at("codes")) cfg.streams.push_back(parse_data_code(c.get<std::string>()));
    cfg.validate();
    const std::uint64_t seed = meta.at("seed");
    const std::int64_t step = meta.at("step");
    for (int r = 0; r < world; ++r) out[r] = next_batch(cfg, r, step, seed);
  } else {
    throw ConfigError("unknown meta kind " + kind);
  }
  return out;
}

json plan_json(const RoutingPlan& p, bool full) {
  json j;
  j["world_size"] = p.world_size;
  j["n_chunks"] = p.chunks.size();
  // Digests always; full arrays for small cases.
  std::vector<std::uint64_t> words;
  words.reserve(p.chunks.size() * 6);
  for (const auto& c : p.chunks) {
    words.push_back(c.sample_id);
    words.push_back(static_cast<std::uint64_t>(c.chunk_index));
    words.push_back(static_cast<std::uint64_t>(c.start));
    words.push_back(static_cast<std::uint64_t>(c.end));
    words.push_back(static_cast<std::uint64_t>(c.source_rank));
    words.push_back(static_cast<std::uint64_t>(c.target_rank));
  }
  j["chunks_digest"] = hex64(digest_bytes(words.data(), words.size() * 8));
  auto lists_digest = [](const std::vector<std::vector<int>>& v) {
    std::vector<std::uint64_t> w;
    for (const auto& l : v) {
      w.push_back(l.size());
      for (int x : l) w.push_back(static_cast<std::uint64_t>(x));
    }
    return hex64(digest_bytes(w.data(), w.size() * 8));
  };
  auto segs_digest = [](const std::vector<std::vector<Segment>>& v) {
    std::vector<std::uint64_t> w;
    for (const auto& l : v) {
      w.push_back(l.size());
      for (const auto& s : l) {
        w.push_back(s.sample_id);
        w.push_back(static_cast<std::uint64_t>(s.first_pos));
        w.push_back(static_cast<std::uint64_t>(s.length));
      }
    }
    return hex64(digest_bytes(w.data(), w.size() * 8));
  };
  j["send_digest"] = lists_digest(p.send);
  j["recv_digest"] = lists_digest(p.recv);
  j["origin_digest"] = segs_digest(p.origin);
  j["target_digest"] = segs_digest(p.target);
  if (full) {
    j["chunks"] = json::array();
    for (const auto& c : p.chunks) {
      j["chunks"].push_back({c.sample_id, c.chunk_index, c.start, c.end, c.source_rank, c.target_rank});
    }
    j["send"] = p.send;
    j["recv"] = p.recv;
    auto segs = [](const std::vector<std::vector<Segment>>& v) {
      json a = json::array();
      for (const auto& l : v) {
        json r = json::array();
        for (const auto& s : l) r.push_back({s.sample_id, s.first_pos, s.length});
        a.push_back(r);
      }
      return a;
    };
    j["origin"] = segs(p.origin);
    j["target"] = segs(p.target);
  }
  return j;
}

json report_json(const BalanceReport& r) {
  json j;
  j["per_gpu_workload"] = json::array();
  for (double d : r.per_gpu_workload) j["per_gpu_workload"].push_back(dbits(d));
  j["per_bag_occupancy"] = json::array();
  for (double d : r.per_bag_occupancy) j["per_bag_occupancy"].push_back(dbits(d));
  j["capacity_violations"] = r.capacity_violations;
  j["total_workload"] = dbits(r.total_workload);
  j["wir"] = dbits(r.wir);
  return j;
}

json world_json(const World& w) {
  json ranks = json::array();
  for (const auto& b : w.ranks) {
    json r;
    r["rows"] = b.num_rows();
    r["width"] = b.width;
    r["head_lo"] = b.head_lo;
    r["head_hi"] = b.head_hi;
    r["mode"] = b.mode == LayoutMode::ChunkFullHeads ? 0 : 1;
    r["ids_digest"] = hex64(digest_bytes(b.sample_ids.data(), b.sample_ids.size() * 8));
    r["pos_digest"] = hex64(digest_bytes(b.positions.data(), b.positions.size() * 8));
    r["payload_digest"] = hex64(digest_bytes(b.payload.data(), b.payload.size() * 8));
    json segs = json::array();
    for (const auto& s : b.segments) segs.push_back({s.sample_id, s.first_pos, s.length});
    r["segments"] = segs;
    ranks.push_back(r);
  }
  json j;
  j["ranks"] = ranks;
  j["checksum"] = hex64(content_checksum(w));
  return j;
}

int cmd_dump() {
  std::stringstream ss;
  ss << std::cin.rdbuf();
  const json c = json::parse(ss.str());
  const int world = c.at("world");
  const bool full = c.value("full", true);
  const WorkloadModel model = model_from(c.at("model"));
  const WorldLayout layout = replicate(parse_topology(c.at("topology").get<std::string>()), world);
  const auto samples = samples_from(c.at("meta"), world);
  const auto info = gather_sequence_info(samples);

  json out;
  json meta = json::array();
  for (const auto& r : info) {
    json l = json::array();
    for (const auto& s : r) l.push_back({s.sample_id, s.length});
    meta.push_back(l);
  }
  out["meta"] = meta;

  PlanResult pr;
  try {
    pr = plan_routing(info, model, layout);
  } catch (const ConfigError& e) {
    out["error"] = std::string("ConfigError: ") + e.what();
    std::cout << out.dump() << "\n";
    return 0;
  }
  out["plan"] = plan_json(pr.plan, full);
  out["report"] = report_json(pr.report);
  const RoutingPlan rev = reverse_plan(pr.plan);
  out["reverse"] = plan_json(rev, full);
  out["identity"] = plan_json(identity_plan(info), full);

  if (c.value("route", false)) {
    const int width = c.at("payload_width");
    const World w0 = make_world(samples, width, model.shape.n_heads);
    out["world0"] = world_json(w0);
    World routed = route(w0, pr.plan, Exec::Serial);
    out["routed"] = world_json(routed);
    if (c.value("ulysses", false)) {
      json uly = json::array();
      for (int rep = 0; rep < layout.num_replicas(); ++rep) {
        for (const auto& ub : layout.unit.bags) {
          if (ub.size() < 2) continue;
          const ComputeBag bag = global_bag(layout, rep, ub.bag_id);
          World staged = routed;
          const auto lens = pre_attn(staged, bag, Exec::Serial);
          json u;
          u["replica"] = rep;
          u["bag"] = ub.bag_id;
          u["full_lens"] = lens;
          u["pre"] = world_json(staged);
          post_attn(staged, bag, Exec::Serial);
          u["post_identity"] = worlds_bitwise_equal(staged, routed);
          uly.push_back(u);
        }
      }
      out["ulysses"] = uly;
    }
    // Mutate like simulator.cpp:128-136, then reverse.
    World mutated = routed;
    for (RankBuffer& buf : mutated.ranks) {
      for (std::int64_t r = 0; r < buf.num_rows(); ++r) {
        const double delta = block_perturbation(buf.sample_ids[r], buf.positions[r]);
        for (int col = 0; col < buf.width; ++col) buf.payload[r * buf.width + col] += delta;
      }
    }
    out["mutated"] = world_json(mutated);
    const World back = reverse_route(mutated, pr.plan, Exec::Serial);
    out["returned"] = world_json(back);
    out["roundtrip_identity"] = worlds_bitwise_equal(reverse_route(routed, pr.plan, Exec::Serial), w0);
  }
  std::cout << out.dump() << "\n";
  return 0;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// CPU baseline: one "step" = plan_routing + route + (pre_attn+post_attn per
// multi-GPU bag) + reverse_route, Exec::Parallel on all OpenMP threads.
// make_world (the fixture generator) is outside the timed region.
int cmd_bench() {
  std::stringstream ss;
  ss << std::cin.rdbuf();
  const json c = json::parse(ss.str());
  const int world = c.at("world");
  const WorkloadModel model = model_from(c.at("model"));
  const WorldLayout layout = replicate(parse_topology(c.at("topology").get<std::string>()), world);
  const auto samples = samples_from(c.at("meta"), world);
  const auto info = gather_sequence_info(samples);
  const int width = c.at("payload_width");
  const int steps = c.value("steps", 1);
  const int warmup = c.value("warmup", 0);
  const bool ulysses = c.value("ulysses", true);
  // DiT attention pattern (metrics.cpp:85-121): pre_attn on q, k and v, then
  // post_attn on the attention output o, and o is what reverse_route brings
  // home.  q/k/v (chunk layout) and o (Ulysses layout) are produced by the
  // model between the phases, so their images are prepared untimed.
  const bool qkv = c.value("qkv", false);
  const Exec exec = c.value("serial", false) ? Exec::Serial : Exec::Parallel;

  const World w0 = make_world(samples, width, model.shape.n_heads);
  std::int64_t tokens = 0;
  for (const auto& r : info)
    for (const auto& s : r) tokens += s.length;

  const double budget_s = c.value("budget_s", 1e30);  // bound the sample's wall time
  double t_plan = 0, t_route = 0, t_uly = 0, t_rev = 0;
  std::vector<double> step_s;
  const double t_begin = now_s();
  for (int it = 0; it < warmup + steps; ++it) {
    if (it > warmup && now_s() - t_begin > budget_s) break;
    const double a = now_s();
    const PlanResult pr = plan_routing(info, model, layout);
    const double b = now_s();
    World routed = route(w0, pr.plan, exec);
    const double cc = now_s();
    double untimed = 0;
    if (ulysses && qkv) {
      const double u0 = now_s();
      std::vector<World> q3{routed, routed, routed};
      World o = routed;
      for (int rep = 0; rep < layout.num_replicas(); ++rep)
        for (const auto& ub : layout.unit.bags)
          if (ub.size() >= 2) pre_attn(o, global_bag(layout, rep, ub.bag_id), exec);
      untimed = now_s() - u0;
      for (int rep = 0; rep < layout.num_replicas(); ++rep) {
        for (const auto& ub : layout.unit.bags) {
          if (ub.size() < 2) continue;
          const ComputeBag bag = global_bag(layout, rep, ub.bag_id);
          for (World& t : q3) pre_attn(t, bag, exec);
        }
      }
      for (int rep = 0; rep < layout.num_replicas(); ++rep) {
        for (const auto& ub : layout.unit.bags) {
          if (ub.size() < 2) continue;
          post_attn(o, global_bag(layout, rep, ub.bag_id), exec);
        }
      }
      routed = std::move(o);
    } else if (ulysses) {
      for (int rep = 0; rep < layout.num_replicas(); ++rep) {
        for (const auto& ub : layout.unit.bags) {
          if (ub.size() < 2) continue;
          const ComputeBag bag = global_bag(layout, rep, ub.bag_id);
          pre_attn(routed, bag, exec);
          post_attn(routed, bag, exec);
        }
      }
    }
    const double d = now_s();
    World back = reverse_route(routed, pr.plan, exec);
    const double e = now_s();
    if (it >= warmup) {
      t_plan += b - a;
      t_route += cc - b;
      t_uly += d - cc - untimed;
      t_rev += e - d;
      step_s.push_back(e - a - untimed);
    }
    if (back.ranks.size() != w0.ranks.size()) return 2;
  }
  json out;
  double total = 0;
  for (double s : step_s) total += s;
  const double ns = step_s.empty() ? 1.0 : static_cast<double>(step_s.size());
  out["steps"] = step_s.size();
  out["tokens_per_step"] = tokens;
  out["s_per_step"] = total / ns;
  out["tokens_per_s"] = tokens / (total / ns);
  out["plan_s"] = t_plan / ns;
  out["route_s"] = t_route / ns;
  out["ulysses_s"] = t_uly / ns;
  out["reverse_s"] = t_rev / ns;
  out["threads"] = omp_get_max_threads();
  out["bytes_per_row"] = width * 8;
  std::cout << out.dump() << "\n";
  return 0;
}

// C4 plan-latency sweep: for each case, plan_routing timed best-of-`reps`
// (bounded by budget_s per case) and reverse_plan timed once (it is
// O(W*C*S) in the reference, balancer.cpp:262-283).  Input:
//   {"world": W, "model": {...}, "reps": k, "budget_s": s,
//    "cases": [{"topology": "...", "meta": {...}, "reverse": true}, ...]}
int cmd_plan_bench() {
  std::stringstream ss;
  ss << std::cin.rdbuf();
  const json c = json::parse(ss.str());
  const int world = c.at("world");
  const WorkloadModel model = model_from(c.value("model", json::object()));
  const int reps = c.value("reps", 5);
  const double budget_s = c.value("budget_s", 5.0);
  json out = json::array();
  for (const auto& cs : c.at("cases")) {
    const WorldLayout layout = replicate(parse_topology(cs.at("topology").get<std::string>()), world);
    const auto info = gather_sequence_info(samples_from(cs.at("meta"), world));
    std::size_t n = 0;
    for (const auto& r : info) n += r.size();
    double best = 1e30;
    int done = 0;
    PlanResult pr;
    const double t_begin = now_s();
    for (int it = 0; it < reps; ++it) {
      if (it > 0 && now_s() - t_begin > budget_s) break;
      const double a = now_s();
      pr = plan_routing(info, model, layout);
      const double b = now_s();
      best = std::min(best, b - a);
      ++done;
    }
    json r;
    r["topology"] = cs.at("topology");
    r["sequences"] = n;
    r["chunks"] = pr.plan.chunks.size();
    r["plan_s"] = best;
    r["plan_reps"] = done;
    r["wir"] = pr.report.wir;
    if (cs.value("reverse", true)) {
      const double a = now_s();
      const RoutingPlan rp = reverse_plan(pr.plan);
      r["reverse_plan_s"] = now_s() - a;
      if (rp.chunks.size() != pr.plan.chunks.size()) return 2;
    }
    out.push_back(r);
  }
  std::cout << out.dump() << "\n";
  return 0;
}

// Scenario (sharding-group) config from JSON: {"codes": [...], "group_size": G}
// (group_size defaults to the sum of the streams' GPU counts), {"preset":
// name} or {"text": scenario-file text} (data_sim.cpp:95-165).
ShardingGroupConfig scenario_from(const json& j) {
  if (j.contains("preset")) return scenario_preset(j.at("preset").get<std::string>());
  if (j.contains("text")) {
    std::istringstream in(j.at("text").get<std::string>());
    return parse_scenario(in);
  }
  ShardingGroupConfig cfg;
  int sum = 0;
  for (const auto& c : j.at("codes")) {
    cfg.streams.push_back(parse_data_code(c.get<std::string>()));
    sum += cfg.streams.back().gpus;
  }
  cfg.group_size = j.value("group_size", sum);
  cfg.validate();
  return cfg;
}

// Upstream generator goldens: next_batch per rank for several steps, and the
// parser's verdict (ParseError offset / ConfigError) on data codes.
int cmd_batches() {
  std::stringstream ss;
  ss << std::cin.rdbuf();
  const json c = json::parse(ss.str());
  json out;
  out["cases"] = json::array();
  for (const auto& cs : c.value("cases", json::array())) {
    const ShardingGroupConfig cfg = scenario_from(cs);
    const int world = cs.at("world");
    const std::uint64_t seed = cs.at("seed");
    json jc;
    jc["group_size"] = cfg.group_size;
    jc["streams"] = json::array();
    for (const auto& st : cfg.streams) jc["streams"].push_back(format_data_code(st));
    jc["steps"] = json::array();
    for (const auto& stv : cs.at("steps")) {
      const std::int64_t step = stv.get<std::int64_t>();
      json js;
      js["step"] = step;
      js["ranks"] = json::array();
      for (int r = 0; r < world; ++r) {
        json jr = json::array();
        for (const SampleMeta& m : next_batch(cfg, r, step, seed)) jr.push_back({m.sample_id, m.text_len, m.visual_len});
        js["ranks"].push_back(jr);
      }
      jc["steps"].push_back(js);
    }
    out["cases"].push_back(jc);
  }
  out["parse"] = json::array();
  for (const auto& code : c.value("parse", json::array())) {
    json jp;
    jp["code"] = code;
    try {
      jp["format"] = format_data_code(parse_data_code(code.get<std::string>()));
    } catch (const ParseError& e) {
      jp["error"] = "ParseError";
      jp["offset"] = e.offset();
      jp["what"] = e.what();
    }
    out["parse"].push_back(jp);
  }
  std::cout << out.dump() << "\n";
  return 0;
}

// C5 dynamic stream on the reference: step s draws every rank's batch from
// scenario s mod K (next_batch, seed), plans it (plan_routing, timed each
// step) and, every `full_every` steps while the budget lasts, runs the full
// data path (make_world untimed; route + pre/post_attn per multi-GPU bag +
// reverse_route timed, Exec::Parallel).  Emits per-step WIR / max-over-mean
// bits (golden for the device driver) and the timings (CPU baseline).
int cmd_stream() {
  std::stringstream ss;
  ss << std::cin.rdbuf();
  const json c = json::parse(ss.str());
  const int world = c.at("world");
  const WorkloadModel model = model_from(c.value("model", json::object()));
  const WorldLayout layout = replicate(parse_topology(c.at("topology").get<std::string>()), world);
  std::vector<ShardingGroupConfig> scen;
  for (const auto& j : c.at("scenarios")) scen.push_back(scenario_from(j));
  const std::uint64_t seed = c.at("seed");
  const std::int64_t first = c.value("first_step", 0);
  const std::int64_t steps = c.at("steps");
  const int full_every = c.value("full_every", 50);
  const int width = c.value("payload_width", 768);
  const double budget_s = c.value("budget_s", 1e30);
  const Exec exec = Exec::Parallel;
  json per = json::array();
  double t_plan = 0, t_full = 0;
  std::int64_t full_tokens = 0, full_steps = 0, tokens_all = 0;
  const double t_begin = now_s();
  std::int64_t done = 0;
  for (std::int64_t s = first; s < first + steps; ++s) {
    if (s > first && now_s() - t_begin > budget_s) break;
    const ShardingGroupConfig& cfg = scen[static_cast<std::size_t>(s % static_cast<std::int64_t>(scen.size()))];
    std::vector<std::vector<SampleMeta>> batches(world);
    for (int r = 0; r < world; ++r) batches[r] = next_batch(cfg, r, s, seed);
    const auto info = gather_sequence_info(batches);
    std::int64_t tokens = 0, nseq = 0;
    for (const auto& r : info)
      for (const auto& q : r) {
        tokens += q.length;
        ++nseq;
      }
    const double a = now_s();
    const PlanResult pr = plan_routing(info, model, layout);
    t_plan += now_s() - a;
    tokens_all += tokens;
    double mx = 0, sum = 0;
    for (double v : pr.report.per_gpu_workload) {
      mx = std::max(mx, v);
      sum += v;
    }
    json js;
    js["step"] = s;
    js["tokens"] = tokens;
    js["sequences"] = nseq;
    js["chunks"] = pr.plan.chunks.size();
    js["wir"] = dbits(pr.report.wir);
    js["total_workload"] = dbits(pr.report.total_workload);
    js["violations"] = pr.report.capacity_violations;
    js["max_over_mean"] = sum > 0 ? mx / (sum / static_cast<double>(world)) : 1.0;
    per.push_back(js);
    if (full_every > 0 && (s - first) % full_every == 0 && now_s() - t_begin <= budget_s) {
      const World w0 = make_world(batches, width, model.shape.n_heads);
      const double b = now_s();
      World routed = route(w0, pr.plan, exec);
      for (int rep = 0; rep < layout.num_replicas(); ++rep)
        for (const auto& ub : layout.unit.bags) {
          if (ub.size() < 2) continue;
          const ComputeBag bag = global_bag(layout, rep, ub.bag_id);
          pre_attn(routed, bag, exec);
          post_attn(routed, bag, exec);
        }
      World back = reverse_route(routed, pr.plan, exec);
      t_full += now_s() - b;
      full_tokens += tokens;
      ++full_steps;
      if (back.ranks.size() != w0.ranks.size()) return 2;
    }
    ++done;
  }
  json out;
  out["steps"] = done;
  out["per_step"] = per;
  out["plan_s_per_step"] = done ? t_plan / static_cast<double>(done) : 0.0;
  out["tokens_per_step"] = done ? static_cast<double>(tokens_all) / static_cast<double>(done) : 0.0;
  out["full_steps"] = full_steps;
  out["roundtrip_tokens_per_s"] = t_full > 0 ? static_cast<double>(full_tokens) / t_full : 0.0;
  out["roundtrip_s_per_step"] = full_steps ? t_full / static_cast<double>(full_steps) : 0.0;
  out["threads"] = omp_get_max_threads();
  std::cout << out.dump() << "\n";
  return 0;
}

// balance_uniform_items / reverse_uniform_plan goldens: {"counts": [[...], ...]}
int cmd_uniform() {
  std::stringstream ss;
  ss << std::cin.rdbuf();
  const json c = json::parse(ss.str());
  json out = json::array();
  for (const auto& cv : c.at("counts")) {
    const std::vector<std::int64_t> counts = cv.get<std::vector<std::int64_t>>();
    json r;
    r["counts"] = counts;
    try {
      const UniformPlan p = balance_uniform_items(counts);
      r["final_counts"] = p.final_counts;
      r["total_moved"] = p.total_moved;
      r["moves"] = json::array();
      for (const UniformMove& m : p.moves) r["moves"].push_back({m.src_rank, m.dst_rank, m.count});
      const UniformPlan q = reverse_uniform_plan(p, counts);
      r["reverse_moves"] = json::array();
      for (const UniformMove& m : q.moves) r["reverse_moves"].push_back({m.src_rank, m.dst_rank, m.count});
      r["reverse_final_counts"] = q.final_counts;
    } catch (const ConfigError& e) {
      r["error"] = std::string("ConfigError: ") + e.what();
    }
    out.push_back(r);
  }
  std::cout << out.dump() << "\n";
  return 0;
}

// nlohmann::json's text for doubles given as IEEE bit patterns (hex).
int cmd_dtoa() {
  std::stringstream ss;
  ss << std::cin.rdbuf();
  const json c = json::parse(ss.str());
  json out = json::array();
  for (const auto& h : c.at("bits")) {
    const std::uint64_t b = std::stoull(h.get<std::string>(), nullptr, 16);
    double d;
    std::memcpy(&d, &b, 8);
    out.push_back(json(d).dump());
  }
  std::cout << out.dump() << "\n";
  return 0;
}

// The CLI's `plan` subcommand (tools/main.cpp:200-230) on in-memory inputs:
// sequential ids, ModelShape{d_model, n_heads, d_model / n_heads, 1}.
int cmd_cli_plan() {
  std::stringstream ss;
  ss << std::cin.rdbuf();
  const json c = json::parse(ss.str());
  json out = json::array();
  for (const auto& cs : c.at("cases")) {
    json r;
    try {
      std::vector<std::vector<SequenceInfo>> per_rank;
      std::uint64_t id = 0;
      for (const auto& rank_lens : cs.at("lens")) {
        std::vector<SequenceInfo> seqs;
        for (const auto& l : rank_lens) {
          const std::int64_t len = l.get<std::int64_t>();
          if (len < 0) throw ConfigError("sequence lengths must be >= 0");  // main.cpp:212
          seqs.push_back({id++, len});
        }
        per_rank.push_back(std::move(seqs));
      }
      const int d_model = cs.value("d_model", 3072), n_heads = cs.value("n_heads", 24);
      WorkloadModel model;
      if (d_model % n_heads != 0) throw ConfigError("d_model must be divisible by n_heads");  // main.cpp:220
      model.shape = ModelShape{d_model, n_heads, d_model / n_heads, 1};
      model.gamma = cs.value("gamma", kGammaH100);
      const Topology topology = parse_topology(cs.at("topology").get<std::string>());
      const WorldLayout layout = replicate(topology, static_cast<int>(per_rank.size()));
      const PlanResult result = plan_routing(per_rank, model, layout);
      r["json"] = plan_to_json(result.plan, result.report);
    } catch (const std::exception& e) {
      r["error"] = e.what();
    }
    out.push_back(r);
  }
  std::cout << out.dump() << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_harness dump|bench|plan_bench|batches|stream|uniform|dtoa|cli_plan < json\n");
    return 1;
  }
  try {
    if (std::strcmp(argv[1], "dump") == 0) return cmd_dump();
    if (std::strcmp(argv[1], "bench") == 0) return cmd_bench();
    if (std::strcmp(argv[1], "plan_bench") == 0) return cmd_plan_bench();
    if (std::strcmp(argv[1], "batches") == 0) return cmd_batches();
    if (std::strcmp(argv[1], "stream") == 0) return cmd_stream();
    if (std::strcmp(argv[1], "uniform") == 0) return cmd_uniform();
    if (std::strcmp(argv[1], "dtoa") == 0) return cmd_dtoa();
    if (std::strcmp(argv[1], "cli_plan") == 0) return cmd_cli_plan();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_harness: %s\n", e.what());
    return 3;
  }
  std::fprintf(stderr, "unknown command %s\n", argv[1]);
  return 1;
}
