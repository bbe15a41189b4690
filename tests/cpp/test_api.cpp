// C++ drop-in API (include/seqbal/seqbal.hpp -> libseqbal.so -> GPU) checked
// the way the reference's own GTest suites check the reference
// (balancer_test.cpp, exchange_test.cpp), plus direct comparisons with the
// C oracle (oracle/seqbal_oracle.c, test infrastructure) on random inputs.
// Built by tests/test_cpp_api.py; needs a CUDA device.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../oracle/seqbal_oracle.h"
#include "seqbal/seqbal.hpp"

using namespace seqbal;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);                \
    }                                                                            \
  } while (0)
#define CHECK_THROWS(expr, Type)                                                 \
  do {                                                                           \
    bool _t = false;                                                             \
    try {                                                                        \
      (void)(expr);                                                              \
    } catch (const Type&) {                                                      \
      _t = true;                                                                 \
    }                                                                            \
    CHECK(_t);                                                                   \
  } while (0)

static uint64_t bits(double d) {
  uint64_t b;
  std::memcpy(&b, &d, 8);
  return b;
}

// CounterRng equivalent through the oracle's restatement (test-side only).
struct Rng {
  uint64_t key, ctr = 0;
  explicit Rng(uint64_t seed) {
    key = or_derive_key(&seed, 1);
  }
  int64_t next_int(int64_t lo, int64_t hi) { return or_rng_int(key, ctr++, lo, hi); }
};

static std::vector<ComputeBag> single_bags(int m) {
  std::vector<ComputeBag> b(m);
  for (int i = 0; i < m; ++i) b[i] = ComputeBag{i, {i}};
  return b;
}

static WorkloadModel small_model() {  // exchange_test.cpp:17-22
  WorkloadModel m;
  m.shape = ModelShape{64, 4, 16, 2};
  m.gamma = 0.49;
  return m;
}

static std::vector<std::vector<SampleMeta>> samples(const std::vector<std::vector<int64_t>>& lens) {
  std::vector<std::vector<SampleMeta>> out(lens.size());
  uint64_t id = 1;
  for (size_t r = 0; r < lens.size(); ++r)
    for (int64_t l : lens[r]) out[r].push_back(SampleMeta{id++, 0, l, static_cast<int>(r)});
  return out;
}

static void test_assign() {
  // balancer_test.cpp:33-49 hand trace with fallback
  auto res = assign_to_bags({{0, 10}, {1, 8}, {2, 5}, {3, 1}}, single_bags(2));
  CHECK(res.size() == 4);
  CHECK(res[0].sample_id == 0 && res[0].assigned_bag == 0);
  CHECK(res[1].assigned_bag == 1 && res[2].assigned_bag == 1 && res[3].assigned_bag == 0);
  // :67-73 descending order with id tie-break
  auto t = assign_to_bags({{7, 5}, {3, 5}, {9, 8}}, single_bags(1));
  CHECK(t[0].sample_id == 9 && t[1].sample_id == 3 && t[2].sample_id == 7);
  // :75-78 rejects
  CHECK_THROWS(assign_to_bags({{0, 1}}, {}), ConfigError);
  CHECK_THROWS(assign_to_bags({{0, -1}}, single_bags(1)), ConfigError);
  // bag sizes whose product overflows int (the first ten primes): no head
  // check applies to assign_to_bags, so this must plan like the oracle
  {
    const int primes[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29};
    std::vector<ComputeBag> bags;
    std::vector<int> sizes, bid;
    int next = 0;
    for (int j = 0; j < 10; ++j) {
      ComputeBag b{j, {}};
      for (int k = 0; k < primes[j]; ++k) b.gpu_ranks.push_back(next++);
      bags.push_back(b);
      sizes.push_back(primes[j]);
      bid.push_back(j);
    }
    std::vector<SequenceWorkload> w;
    std::vector<uint64_t> ids;
    std::vector<double> ws;
    for (int i = 0; i < 60; ++i) {
      w.push_back({static_cast<uint64_t>(i * 7 + 1), static_cast<double>((i * 37) % 101)});
      ids.push_back(w.back().sample_id);
      ws.push_back(w.back().workload);
    }
    auto got = assign_to_bags(w, bags);
    std::vector<uint64_t> oi(60);
    std::vector<double> ow(60);
    std::vector<int> ob(60);
    or_assign_to_bags(60, ids.data(), ws.data(), 10, sizes.data(), bid.data(), oi.data(), ow.data(), ob.data());
    bool same = got.size() == 60;
    for (int i = 0; same && i < 60; ++i) same = got[i].sample_id == oi[i] && got[i].assigned_bag == ob[i];
    CHECK(same);
  }
  // more than 64 bags (the multi-kernel path's k_greedy_many) vs the oracle;
  // documented limit: at most 1024 bags per replica
  {
    const int m = 100, n = 700;
    std::vector<SequenceWorkload> w;
    std::vector<uint64_t> ids, oi(n);
    std::vector<double> ws, ow(n);
    std::vector<int> sizes(m, 1), bid(m), ob(n);
    for (int j = 0; j < m; ++j) bid[j] = j;
    for (int i = 0; i < n; ++i) {
      w.push_back({static_cast<uint64_t>(i * 13 + 5), static_cast<double>((i * 7919) % 997 + (i % 3 == 0 ? 0 : 1000))});
      ids.push_back(w.back().sample_id);
      ws.push_back(w.back().workload);
    }
    auto got = assign_to_bags(w, single_bags(m));
    or_assign_to_bags(n, ids.data(), ws.data(), m, sizes.data(), bid.data(), oi.data(), ow.data(), ob.data());
    bool same = got.size() == static_cast<size_t>(n);
    for (int i = 0; same && i < n; ++i) same = got[i].sample_id == oi[i] && got[i].assigned_bag == ob[i];
    CHECK(same);
  }
  CHECK_THROWS(assign_to_bags({{0, 1}}, single_bags(1025)), ConfigError);
  // random instances vs the oracle, heterogeneous bags
  Rng rng(99);
  for (int trial = 0; trial < 50; ++trial) {
    const int m = static_cast<int>(rng.next_int(1, 5));
    std::vector<ComputeBag> bags;
    std::vector<int> sizes, ids_b;
    int next = 0;
    for (int j = 0; j < m; ++j) {
      const int g = static_cast<int>(rng.next_int(1, 3));
      ComputeBag b{j, {}};
      for (int k = 0; k < g; ++k) b.gpu_ranks.push_back(next++);
      bags.push_back(b);
      sizes.push_back(g);
      ids_b.push_back(j);
    }
    const int n = static_cast<int>(rng.next_int(0, 40));
    std::vector<SequenceWorkload> w;
    std::vector<uint64_t> ids;
    std::vector<double> ws;
    for (int i = 0; i < n; ++i) {
      w.push_back({static_cast<uint64_t>(rng.next_int(0, 1000000)), static_cast<double>(rng.next_int(0, 100))});
      ids.push_back(w.back().sample_id);
      ws.push_back(w.back().workload);
    }
    auto got = assign_to_bags(w, bags);
    std::vector<uint64_t> oi(n);
    std::vector<double> ow(n);
    std::vector<int> ob(n);
    or_assign_to_bags(n, ids.data(), ws.data(), m, sizes.data(), ids_b.data(), oi.data(), ow.data(), ob.data());
    bool same = static_cast<int>(got.size()) == n;
    for (int i = 0; same && i < n; ++i)
      same = got[i].sample_id == oi[i] && bits(got[i].workload) == bits(ow[i]) && got[i].assigned_bag == ob[i];
    CHECK(same);
  }
}

static void compare_with_oracle(const std::vector<std::vector<SequenceInfo>>& seqs, const char* topo,
                                const WorkloadModel& model) {
  const WorldLayout layout = replicate(parse_topology(topo), static_cast<int>(seqs.size()));
  const PlanResult pr = plan_routing(seqs, model, layout);
  std::vector<int64_t> off{0}, lens;
  std::vector<uint64_t> ids;
  for (const auto& r : seqs) {
    for (const auto& s : r) {
      ids.push_back(s.sample_id);
      lens.push_back(s.length);
    }
    off.push_back(static_cast<int64_t>(ids.size()));
  }
  std::vector<int> boff{0}, branks;
  for (const auto& b : layout.unit.bags) {
    for (int r : b.gpu_ranks) branks.push_back(r);
    boff.push_back(static_cast<int>(branks.size()));
  }
  const int W = layout.world_size;
  const int64_t cap = std::max<int64_t>(1, static_cast<int64_t>(ids.size()) * 8);
  std::vector<uint64_t> cid(cap);
  std::vector<int32_t> cidx(cap), csrc(cap), cdst(cap), sidx(cap), ridx(cap);
  std::vector<int64_t> cs(cap), ce(cap), soff(W + 1), roff(W + 1);
  std::vector<double> per(W), occ(layout.num_replicas() * layout.unit.bags.size() + 1);
  or_plan_in in{W, off.data(), ids.data(), lens.data(), layout.unit.unit_size,
                static_cast<int>(layout.unit.bags.size()), boff.data(), branks.data(), model.shape.d_model,
                model.shape.n_heads, model.gamma};
  or_plan_out o{cap, 0, cid.data(), cidx.data(), cs.data(), ce.data(), csrc.data(), cdst.data(), soff.data(),
                sidx.data(), roff.data(), ridx.data(), per.data(), occ.data(), 0, 0.0, 0.0};
  CHECK(or_plan_routing(&in, &o) == 0);
  bool same = static_cast<int64_t>(pr.plan.chunks.size()) == o.n_chunks;
  for (int64_t c = 0; same && c < o.n_chunks; ++c) {
    const auto& ch = pr.plan.chunks[c];
    same = ch.sample_id == cid[c] && ch.chunk_index == cidx[c] && ch.start == cs[c] && ch.end == ce[c] &&
           ch.source_rank == csrc[c] && ch.target_rank == cdst[c];
  }
  CHECK(same);
  for (int r = 0; r < W; ++r) {
    CHECK(static_cast<int64_t>(pr.plan.send[r].size()) == soff[r + 1] - soff[r]);
    CHECK(static_cast<int64_t>(pr.plan.recv[r].size()) == roff[r + 1] - roff[r]);
    for (int64_t k = soff[r]; k < soff[r + 1]; ++k) CHECK(pr.plan.send[r][k - soff[r]] == sidx[k]);
    for (int64_t k = roff[r]; k < roff[r + 1]; ++k) CHECK(pr.plan.recv[r][k - roff[r]] == ridx[k]);
    CHECK(bits(pr.report.per_gpu_workload[r]) == bits(per[r]));
  }
  for (size_t j = 0; j < pr.report.per_bag_occupancy.size(); ++j)
    CHECK(bits(pr.report.per_bag_occupancy[j]) == bits(occ[j]));
  CHECK(pr.report.capacity_violations == o.violations);
  CHECK(bits(pr.report.total_workload) == bits(o.total_workload));
  CHECK(bits(pr.report.wir) == bits(o.wir));
}

static void test_plan_routing() {
  // balancer_test.cpp:120-128 already balanced -> no movement
  {
    std::vector<std::vector<SequenceInfo>> s{{{0, 500}}, {{1, 500}}, {{2, 500}}, {{3, 500}}};
    const PlanResult r = plan_routing(s, WorkloadModel{}, replicate(parse_topology("g1n4"), 4));
    CHECK(r.report.wir == 1.0);
    for (const auto& c : r.plan.chunks) CHECK(c.source_rank == c.target_rank);
  }
  // :145-153 replicas are independent
  {
    std::vector<std::vector<SequenceInfo>> s{{{0, 1000}}, {{1, 10}}, {{2, 2000}}, {{3, 20}}};
    const PlanResult r = plan_routing(s, WorkloadModel{}, replicate(parse_topology("g1n2"), 4));
    for (const auto& c : r.plan.chunks) CHECK(c.source_rank / 2 == c.target_rank / 2);
  }
  // :205-214 head divisibility rejected
  {
    WorkloadModel m;
    m.shape = ModelShape{3072, 12, 256, 57};
    std::vector<std::vector<SequenceInfo>> s(8);
    s[0].push_back({1, 10});
    CHECK_THROWS(plan_routing(s, m, replicate(parse_topology("g8n1"), 8)), ConfigError);
  }
  // world size mismatch
  CHECK_THROWS(plan_routing(std::vector<std::vector<SequenceInfo>>(3), WorkloadModel{},
                            replicate(parse_topology("g1n4"), 4)),
               ConfigError);
  // random worlds vs the oracle (ragged, empty ranks, heterogeneous bags)
  Rng rng(31);
  const char* topos[] = {"g1n8", "g2n4", "g4n2", "g8n1", "g1n2+g2n1+g4n1"};
  uint64_t id = 0;
  for (int trial = 0; trial < 40; ++trial) {
    const char* t = topos[trial % 5];
    const int W = trial % 5 == 4 ? 16 : 8;
    std::vector<std::vector<SequenceInfo>> s(W);
    for (auto& r : s) {
      const int n = static_cast<int>(rng.next_int(0, 6));
      for (int i = 0; i < n; ++i) r.push_back({id++, rng.next_int(0, 5000)});
    }
    compare_with_oracle(s, t, WorkloadModel{});
  }
}

static void test_reverse_plan() {
  // balancer_test.cpp:226-235 involution and identity
  std::vector<std::vector<SequenceInfo>> s{{{0, 900}, {1, 30}}, {{2, 64}}, {{3, 4096}}, {{4, 128}, {5, 128}}};
  const PlanResult r = plan_routing(s, WorkloadModel{}, replicate(parse_topology("g1n2+g2n1"), 4));
  const RoutingPlan rev = reverse_plan(r.plan);
  CHECK(reverse_plan(rev) == r.plan);  // generic device path (rev is not cached)
  const RoutingPlan ident = identity_plan(s);
  CHECK(reverse_plan(ident) == ident);
  // identity_plan for worlds beyond 64 ranks (simulator.cpp:77 'none' baseline)
  {
    std::vector<std::vector<SequenceInfo>> big(100);
    uint64_t id = 1000;
    for (int r = 0; r < 100; ++r)
      for (int i = 0; i < r % 3; ++i) big[r].push_back({id++, static_cast<int64_t>(10 * r + i)});
    const RoutingPlan ip = identity_plan(big);
    bool ok = ip.world_size == 100;
    size_t n = 0;
    for (const auto& c : ip.chunks) ok = ok && c.source_rank == c.target_rank && c.start == 0;
    for (const auto& r : big) n += r.size();
    CHECK(ok && ip.chunks.size() == n);
    CHECK(reverse_plan(ip) == ip);
  }
  // documented limit: plan_routing with more than 1024 bags per replica
  {
    std::vector<std::vector<SequenceInfo>> s1025(1025);
    s1025[0].push_back({1, 10});
    CHECK_THROWS(plan_routing(s1025, WorkloadModel{}, replicate(parse_topology("g1n1025"), 1025)), ConfigError);
  }
}

static void test_route_split_and_mismatch() {
  // exchange_test.cpp:72-87
  const auto smp = samples({{10}, {}});
  const World world = make_world(smp, 8, 4);
  for (int64_t r = 0; r < 3; ++r)
    for (int c = 0; c < 8; ++c) CHECK(world.ranks[0].payload[r * 8 + c] == payload_value(1, r, c));
  const PlanResult pr = plan_routing(gather_sequence_info(smp), small_model(), replicate(parse_topology("g2n1"), 2));
  const World routed = route(world, pr.plan);
  CHECK(routed.ranks[0].num_rows() == 5 && routed.ranks[1].num_rows() == 5);
  CHECK((routed.ranks[1].positions == std::vector<int64_t>{5, 6, 7, 8, 9}));
  for (int64_t r = 0; r < 5; ++r)
    for (int c = 0; c < 8; ++c) CHECK(routed.ranks[1].payload[r * 8 + c] == payload_value(1, 5 + r, c));
  CHECK(routed.ranks[1].segments.front().first_pos == 5);
  // :89-105 plan/buffer mismatch names the sample
  auto wrong = gather_sequence_info(smp);
  wrong[0][0].length = 9;
  bool named = false;
  try {
    route(world, identity_plan(wrong));
  } catch (const IntegrityError& e) {
    named = std::string(e.what()).find('1') != std::string::npos;
  }
  CHECK(named);
  auto missing = gather_sequence_info(smp);
  missing[0][0].sample_id = 999;
  CHECK_THROWS(route(world, identity_plan(missing)), IntegrityError);
  // identity route keeps the world bit-exact (:62-70)
  const auto s2 = samples({{5, 2}, {3}});
  const World w2 = make_world(s2, 8, 4);
  CHECK(worlds_bitwise_equal(route(w2, identity_plan(gather_sequence_info(s2))), w2));
}

static void test_round_trips() {
  // exchange_test.cpp:118-137 (60 trials) + checksum invariance
  Rng rng(404);
  for (int trial = 0; trial < 60; ++trial) {
    std::vector<std::vector<int64_t>> lens(4);
    for (auto& r : lens) {
      const int n = static_cast<int>(rng.next_int(0, 4));
      for (int i = 0; i < n; ++i) r.push_back(rng.next_int(1, 200));
    }
    const auto smp = samples(lens);
    const World world = make_world(smp, 8, 4);
    const PlanResult pr =
        plan_routing(gather_sequence_info(smp), small_model(), replicate(parse_topology("g1n1+g2n1+g1n1"), 4));
    const World routed = route(world, pr.plan);
    CHECK(worlds_bitwise_equal(reverse_route(routed, pr.plan), world));
    CHECK(content_checksum(routed) == content_checksum(world));
  }
  // :139-168 mutated payload returns home
  const auto smp = samples({{40, 7}, {11}});
  const World world = make_world(smp, 8, 4);
  const PlanResult pr = plan_routing(gather_sequence_info(smp), small_model(), replicate(parse_topology("g2n1"), 2));
  World routed = route(world, pr.plan);
  for (RankBuffer& b : routed.ranks)
    for (int64_t r = 0; r < b.num_rows(); ++r) {
      const double d = block_perturbation(b.sample_ids[r], b.positions[r]);
      for (int c = 0; c < b.width; ++c) b.payload[r * b.width + c] += d;
    }
  const World back = reverse_route(routed, pr.plan);
  bool ok = true;
  for (size_t r = 0; r < back.ranks.size(); ++r) {
    const RankBuffer &b = back.ranks[r], &o = world.ranks[r];
    ok &= b.sample_ids == o.sample_ids && b.positions == o.positions;
    for (int64_t i = 0; i < b.num_rows(); ++i)
      for (int c = 0; c < b.width; ++c)
        ok &= b.payload[i * b.width + c] == o.payload[i * b.width + c] + block_perturbation(b.sample_ids[i], b.positions[i]);
  }
  CHECK(ok);
}

static World routed_bag_world(const std::vector<int64_t>& lens, const WorldLayout& layout) {
  std::vector<std::vector<int64_t>> per(layout.world_size);
  per[0] = lens;
  const auto smp = samples(per);
  const World w = make_world(smp, 8, 4);
  return route(w, plan_routing(gather_sequence_info(smp), small_model(), layout).plan);
}

static void test_ulysses() {
  // exchange_test.cpp:195-216 two-GPU bag holds the full sequence, half heads
  {
    const WorldLayout layout = replicate(parse_topology("g2n1"), 2);
    World w = routed_bag_world({10}, layout);
    const auto lens = pre_attn(w, global_bag(layout, 0, 0));
    CHECK((lens == std::vector<int64_t>{10}));
    for (int m = 0; m < 2; ++m) {
      const RankBuffer& b = w.ranks[m];
      CHECK(b.mode == LayoutMode::FullSeqPartialHeads && b.num_rows() == 10 && b.width == 4);
      CHECK(b.head_lo == m * 2 && b.head_hi == (m + 1) * 2);
      for (int64_t r = 0; r < 10; ++r)
        for (int c = 0; c < 4; ++c) CHECK(b.payload[r * 4 + c] == payload_value(1, r, m * 4 + c));
    }
  }
  // :245-260 post(pre(x)) == x over 30 trials, checksum invariant
  Rng rng(777);
  const WorldLayout layout = replicate(parse_topology("g4n1"), 4);
  for (int trial = 0; trial < 30; ++trial) {
    std::vector<int64_t> lens;
    const int n = static_cast<int>(rng.next_int(1, 5));
    for (int i = 0; i < n; ++i) lens.push_back(rng.next_int(1, 64));
    World w = routed_bag_world(lens, layout);
    const World before = w;
    pre_attn(w, global_bag(layout, 0, 0));
    CHECK(content_checksum(w) == content_checksum(before));
    post_attn(w, global_bag(layout, 0, 0));
    CHECK(worlds_bitwise_equal(before, w));
  }
  // :233-243 indivisible head split; :288-292 wrong layout
  {
    auto w = make_world(samples({{6}, {}, {}}), 8, 4);
    CHECK_THROWS(pre_attn(w, ComputeBag{0, {0, 1, 2}}), ConfigError);
    auto w2 = make_world(samples({{6}, {6}}), 8, 4);
    CHECK_THROWS(post_attn(w2, ComputeBag{0, {0, 1}}), IntegrityError);
  }
  // single-GPU bag is a no-op (:183-193)
  {
    auto w = make_world(samples({{9, 4}}), 8, 4);
    const World before = w;
    CHECK((pre_attn(w, ComputeBag{0, {0}}) == std::vector<int64_t>{9, 4}));
    CHECK(worlds_bitwise_equal(before, w));
  }
}

static void test_block_moves() {
  // exchange_kernels.cpp:1-6: serial == parallel bit for bit
  const auto smp = samples({{100, 3}, {57}, {13, 13, 13}, {}});
  const World world = make_world(smp, 8, 4);
  const PlanResult pr = plan_routing(gather_sequence_info(smp), small_model(), replicate(parse_topology("g2n2"), 4));
  CHECK(worlds_bitwise_equal(route(world, pr.plan, Exec::Serial), route(world, pr.plan, Exec::Parallel)));
  World dst = world;
  for (auto& b : dst.ranks) std::fill(b.payload.begin(), b.payload.end(), 0.0);
  std::vector<BlockMove> moves{{0, 10, 2, 2, 1, 4, 5, 4, false}, {1, 0, 0, 0, 50, 0, 7, 8, true}};
  World a = dst, b = dst;
  apply_block_moves_serial(world, moves, a);
  apply_block_moves_parallel(world, moves, b);
  CHECK(worlds_bitwise_equal(a, b));
  for (int64_t r = 0; r < 5; ++r)
    for (int c = 0; c < 4; ++c) CHECK(a.ranks[2].payload[(1 + r) * 8 + 4 + c] == world.ranks[0].payload[(10 + r) * 8 + 2 + c]);
  CHECK(a.ranks[0].sample_ids[50] == world.ranks[1].sample_ids[0]);
}

// data_sim_test.cpp:15-166 on the device generator (next_batch) and the
// host grammar.
static void test_data_sim() {
  CHECK((parse_data_code("g32b32i256f1s0") == StreamSpec{32, 32, 256, 1, false}));
  CHECK((parse_data_code("g8b2i256f85s1") == StreamSpec{8, 2, 256, 85, true}));
  CHECK((parse_data_code("g1b1i16f1s0") == StreamSpec{1, 1, 16, 1, false}));
  for (const auto& name : scenario_preset_names()) {
    const ShardingGroupConfig config = scenario_preset(name);
    CHECK(config.group_size == 32);
    for (const StreamSpec& s : config.streams) CHECK(parse_data_code(format_data_code(s)) == s);
  }
  const std::pair<const char*, std::size_t> bad[] = {{"", 0}, {"b32g32i256f1s0", 0}, {"g32b32i256f1", 12},
                                                     {"g32b32i256f1s2", 13}, {"g32b32i255f1s0", 7},
                                                     {"g0b32i256f1s0", 1}, {"g32b32i256f1s0x", 14},
                                                     {"g32b0i256f1s0", 4}, {"g32b32i256f0s0", 11}};
  for (const auto& [text, off] : bad) {
    bool thrown = false;
    try {
      parse_data_code(text);
    } catch (const ParseError& e) {
      thrown = true;
      CHECK(e.offset() == off);
    }
    CHECK(thrown);
  }
  CHECK(visual_tokens(StreamSpec{1, 1, 256, 1, false}, 1.0) == 256);
  CHECK(visual_tokens(StreamSpec{1, 1, 512, 85, true}, 1.0) == 25600);
  CHECK(latent_frames(StreamSpec{1, 1, 512, 85, true}) == 25);
  CHECK(latent_frames(StreamSpec{1, 1, 512, 17, true}) == 5);
  CHECK(visual_tokens(StreamSpec{1, 1, 256, 4, false}, 1.0) == 1024);
  CHECK(visual_tokens(StreamSpec{1, 1, 16, 1, true}, 1.0) == 1);
  CHECK(visual_tokens(StreamSpec{1, 1, 256, 1, false}, 0.96) == 246);
  CHECK(visual_tokens(StreamSpec{1, 1, 256, 1, false}, 1.04) == 266);
  const ShardingGroupConfig mixed = preset_mixed_image();
  CHECK(stream_of_rank(mixed, 0) == 0 && stream_of_rank(mixed, 15) == 0 && stream_of_rank(mixed, 16) == 1);
  CHECK(stream_of_rank(mixed, 19) == 1 && stream_of_rank(mixed, 20) == 2 && stream_of_rank(mixed, 24) == 3);
  CHECK(stream_of_rank(mixed, 31) == 3);
  CHECK_THROWS(stream_of_rank(mixed, 32), ConfigError);
  ShardingGroupConfig wrong;
  wrong.group_size = 8;
  wrong.streams.push_back(parse_data_code("g4b1i256f1s0"));
  CHECK_THROWS(wrong.validate(), ConfigError);
  // next_batch: deterministic, rank/step/seed sensitive, stream-shaped
  const auto a = next_batch(mixed, 5, 3, 42), b = next_batch(mixed, 5, 3, 42);
  CHECK(a.size() == b.size());
  bool same = a.size() == b.size(), diff = false;
  const auto r6 = next_batch(mixed, 6, 3, 42), s4 = next_batch(mixed, 5, 4, 42), z = next_batch(mixed, 5, 3, 43);
  for (size_t i = 0; i < a.size() && same; ++i) {
    same &= a[i].sample_id == b[i].sample_id && a[i].text_len == b[i].text_len && a[i].visual_len == b[i].visual_len;
    diff |= a[i].text_len != r6[i].text_len || a[i].text_len != s4[i].text_len || a[i].text_len != z[i].text_len;
  }
  CHECK(same && diff);
  const auto r17 = next_batch(mixed, 17, 0, 7);
  CHECK(r17.size() == 5);
  for (const SampleMeta& sm : r17) CHECK(sm.origin_rank == 17 && sm.text_len >= 0 && sm.text_len <= kMaxTextTokens);
  for (int rank : {0, 3, 16, 20, 24}) {
    const int si = stream_of_rank(mixed, rank);
    const double mult = aspect_multiplier(7, 11, si);
    for (const SampleMeta& sm : next_batch(mixed, rank, 11, 7))
      CHECK(sm.visual_len == visual_tokens(mixed.streams[si], mult));
  }
  const ShardingGroupConfig lowres = preset_lowres_image();
  for (int step = 0; step < 40; ++step) {
    const auto batch = next_batch(lowres, 0, step, 1234);
    CHECK(batch.size() == 32);
    for (const SampleMeta& sm : batch) CHECK(sm.visual_len >= 246 && sm.visual_len <= 266);
  }
  const auto r33 = next_batch(mixed, 33, 0, 7);
  CHECK(r33.size() == 4 && r33.front().origin_rank == 33);
  std::istringstream sc("# x\ngroup_size 4\ng2b1i512f1s0\n\ng2b4i256f1s1 # y\n");
  const ShardingGroupConfig parsed = parse_scenario(sc);
  CHECK(parsed.group_size == 4 && parsed.streams.size() == 2 && parsed.streams[1].smooth);
  std::istringstream nohdr("g2b1i512f1s0\n");
  CHECK_THROWS(parse_scenario(nohdr), ParseError);
  const SampleMeta d = dummy_sample(3, 9);
  CHECK(d.sample_id == make_sample_id(9, 3, 0) && d.visual_len == 1 && d.text_len == 0);
}

// balancer_test.cpp:298-370 on the device uniform balancer.
static std::int64_t min_moves_oracle(const std::vector<std::int64_t>& counts) {
  const int n = static_cast<int>(counts.size());
  std::int64_t total = 0;
  for (auto c : counts) total += c;
  const std::int64_t base = total / n;
  const int rem = static_cast<int>(total % n);
  std::int64_t best = INT64_MAX;
  for (int mask = 0; mask < (1 << n); ++mask) {
    if (__builtin_popcount(mask) != rem) continue;
    std::int64_t moved = 0;
    for (int r = 0; r < n; ++r) moved += std::max<std::int64_t>(0, counts[r] - (base + ((mask >> r) & 1)));
    best = std::min(best, moved);
  }
  return best;
}

static void test_uniform() {
  const UniformPlan p = balance_uniform_items({4, 0});
  CHECK((p.final_counts == std::vector<std::int64_t>{2, 2}) && p.total_moved == 2);
  const UniformPlan q = balance_uniform_items({3, 3, 3});
  CHECK((q.final_counts == std::vector<std::int64_t>{3, 3, 3}) && q.total_moved == 0 && q.moves.empty());
  const UniformPlan r = balance_uniform_items({5, 0, 0});
  CHECK((r.final_counts == std::vector<std::int64_t>{2, 2, 1}) && r.total_moved == 3);
  CHECK_THROWS(balance_uniform_items({1, -1}), ConfigError);
  uint64_t state = 55;
  for (int trial = 0; trial < 300; ++trial) {
    auto next = [&](int lo, int hi) {
      state = state * 6364136223846793005ULL + 1442695040888963407ULL;
      return lo + static_cast<int>((state >> 33) % static_cast<uint64_t>(hi - lo + 1));
    };
    const int n = next(1, 8);
    std::vector<std::int64_t> counts(n);
    for (auto& c : counts) c = next(0, 12);
    const UniformPlan u = balance_uniform_items(counts);
    std::int64_t total = 0, ftotal = 0, lo = INT64_MAX, hi = INT64_MIN;
    for (int k = 0; k < n; ++k) {
      total += counts[k];
      ftotal += u.final_counts[k];
      lo = std::min(lo, u.final_counts[k]);
      hi = std::max(hi, u.final_counts[k]);
    }
    CHECK(total == ftotal && hi - lo <= 1);
    CHECK(u.total_moved == min_moves_oracle(counts));
    std::vector<std::int64_t> sim = counts;
    for (const UniformMove& m : u.moves) {
      sim[m.src_rank] -= m.count;
      sim[m.dst_rank] += m.count;
    }
    CHECK(sim == u.final_counts);
    for (const UniformMove& m : reverse_uniform_plan(u, counts).moves) {
      sim[m.src_rank] -= m.count;
      sim[m.dst_rank] += m.count;
    }
    CHECK(sim == counts);
  }
}

// balancer.cpp:289-352 wire format through the drop-in API: a device plan
// serialises and re-reads to an equal plan.
static void test_plan_json() {
  std::vector<std::vector<SequenceInfo>> seqs = {{{1, 900}, {2, 30}, {3, 0}}, {{4, 64}}, {{5, 4096}, {6, 7}}, {}};
  WorkloadModel m;
  const PlanResult pr = plan_routing(seqs, m, replicate(parse_topology("g1n2+g2n1"), 4));
  const std::string js = plan_to_json(pr.plan, pr.report);
  const PlanResult back = plan_from_json(js);
  CHECK(back.plan == pr.plan);
  CHECK(plan_to_json(back.plan, back.report) == js);
  CHECK(js.rfind("{\"chunks\":[{\"chunk_index\":0,", 0) == 0);
  CHECK_THROWS(plan_from_json("{\"world_size\":2,\"chunks\":[],\"origins\":[[]]}"), ConfigError);
  CHECK_THROWS(plan_from_json("{\"world_size\":"), ParseError);
}

int main() {
  const std::pair<const char*, std::function<void()>> tests[] = {
      {"assign_to_bags", test_assign},        {"plan_routing", test_plan_routing},
      {"reverse_plan", test_reverse_plan},    {"route", test_route_split_and_mismatch},
      {"round_trips", test_round_trips},      {"ulysses", test_ulysses},
      {"block_moves", test_block_moves},      {"data_sim", test_data_sim},
      {"uniform", test_uniform},              {"plan_json", test_plan_json}};
  for (const auto& [name, fn] : tests) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("FAIL %s: exception %s\n", name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
