// SPDX-License-Identifier: Apache-2.0
//
// libseqbal.so: the reference-compatible C++ API (include/seqbal/seqbal.hpp)
// layered on the C-ABI of libseqbal_cuda.so.  Host work here is limited to
// argument validation with the reference's messages, container reshaping
// (std::vector <-> packed device images) and the small integer utilities the
// headers expose; planning and every byte of data movement run on the GPU.
#include <cstring>
#include <initializer_list>
#include <limits>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "seqbal/seqbal.hpp"
#include "seqbal_capi.h"

namespace seqbal {

ParseError::ParseError(const std::string& what, std::size_t offset)
    : std::invalid_argument(what + " (at offset " + std::to_string(offset) + ")"), offset_(offset) {}

namespace {

[[noreturn]] void raise(sb_status st, const char* where) {
  const std::string msg = std::string(sb_last_error());
  switch (st) {
    case SB_ERR_CONFIG: throw ConfigError(msg);
    case SB_ERR_INTEGRITY: throw IntegrityError(msg);
    case SB_ERR_PARSE: throw ParseError(msg, 0);
    default: throw std::runtime_error(std::string(where) + ": " + msg);
  }
}

inline void ck(sb_status st, const char* where) {
  if (st != SB_OK) raise(st, where);
}

// ------------------------------------------------------------- device ctx
// One process-wide context: planners cached per configuration, a device
// staging area for metadata, and the host copy of the last device-built plan
// so route/reverse_plan can reuse it without an upload.
struct PlannerKey {
  int W, U;
  std::vector<int32_t> bag_off, bag_ranks;
  int d_model, n_heads, d_head, n_blocks;
  double gamma, k;
  bool operator==(const PlannerKey&) const = default;
};

struct Entry {
  PlannerKey key;
  int64_t cap = 0;
  sb_planner* p = nullptr;
};

struct Device {
  std::mutex mu;
  std::vector<Entry> planners;
  sb_planner* last = nullptr;  // planner holding the last device-built plan
  RoutingPlan last_plan;
  bool last_valid = false;
  std::vector<uint64_t> rev_recv_of_last;  // flattened reverse receive lists
  std::vector<int64_t> rev_off_of_last;
};

Device& dev() {
  static Device* d = new Device();
  return *d;
}

struct DevBuf {  // minimal device allocation helper via the C-ABI worlds
  void* p = nullptr;
};

sb_planner* planner_for(const PlannerKey& key, int64_t need) {
  Device& d = dev();
  for (Entry& e : d.planners) {
    if (e.key == key && e.cap >= need) return e.p;
  }
  for (auto it = d.planners.begin(); it != d.planners.end(); ++it) {
    if (it->key == key) {  // grow: replace the smaller planner
      if (d.last == it->p) d.last_valid = false, d.last = nullptr;
      sb_planner_destroy(it->p);
      d.planners.erase(it);
      break;
    }
  }
  sb_planner_desc desc{};
  desc.world_size = key.W;
  desc.unit_size = key.U;
  desc.n_bags = static_cast<int>(key.bag_off.size()) - 1;
  desc.bag_offsets = key.bag_off.data();
  desc.bag_ranks = key.bag_ranks.data();
  desc.d_model = key.d_model;
  desc.n_heads = key.n_heads;
  desc.d_head = key.d_head;
  desc.n_blocks = key.n_blocks;
  desc.gamma = key.gamma;
  desc.k = key.k;
  const int64_t cap = std::max<int64_t>(need, 1024);
  desc.max_seqs = cap;
  sb_planner* p = nullptr;
  ck(sb_planner_create(&desc, &p), "sb_planner_create");
  d.planners.push_back({key, cap, p});
  return p;
}

PlannerKey key_for(const WorldLayout& layout, const WorkloadModel& model) {
  PlannerKey k;
  k.W = layout.world_size;
  k.U = layout.unit.unit_size;
  k.bag_off.push_back(0);
  for (std::size_t b = 0; b < layout.unit.bags.size(); ++b) {
    const ComputeBag& bag = layout.unit.bags[b];
    if (bag.bag_id != static_cast<int>(b))
      throw ConfigError("plan_routing: bag ids must equal their position in the topology");
    for (int r : bag.gpu_ranks) k.bag_ranks.push_back(r);
    k.bag_off.push_back(static_cast<int32_t>(k.bag_ranks.size()));
  }
  k.d_model = model.shape.d_model;
  k.n_heads = model.shape.n_heads;
  k.d_head = model.shape.d_head;
  k.n_blocks = model.shape.n_blocks;
  k.gamma = model.gamma;
  k.k = model.k;
  return k;
}

// Metadata staged in device memory through a 1-rank-per-entry "world" of
// 16-byte rows: we reuse sb_world arenas as generic device buffers.
struct DeviceMeta {
  sb_world* w = nullptr;  // tensor 0 (16 B rows) holds ids, tensor 1 lens, tensor 2 rank_off
  void* ids = nullptr;
  void* lens = nullptr;
  void* off = nullptr;
  int64_t cap = 0;
  ~DeviceMeta() {
    if (w) sb_world_destroy(w);
  }
};

DeviceMeta& meta_buf(int64_t n, int W) {
  static DeviceMeta* m = new DeviceMeta();
  const int64_t need = std::max<int64_t>(n, W + 1) + 1;
  if (m->cap < need) {
    if (m->w) sb_world_destroy(m->w);
    m->w = nullptr;
    sb_world_desc d{};
    const int64_t rb[2] = {8, 8};
    d.world_size = 1;
    d.n_local = 1;
    d.first_local = 0;
    d.n_heads = 1;
    d.n_payload = 2;
    d.n_aux = 0;
    d.row_bytes = rb;
    d.capacity_rows = need;
    d.max_bag = 1;
    ck(sb_world_create(&d, &m->w), "metadata staging");
    int64_t bytes = 0;
    ck(sb_world_arena(m->w, 0, &m->off, &bytes), "metadata staging");
    ck(sb_world_arena(m->w, 1, &m->ids, &bytes), "metadata staging");
    ck(sb_world_arena(m->w, 2, &m->lens, &bytes), "metadata staging");
    m->cap = need;
  }
  return *m;
}

struct FlatMeta {
  std::vector<uint64_t> ids;
  std::vector<int64_t> lens, off;
};

FlatMeta flatten(const std::vector<std::vector<SequenceInfo>>& per_rank) {
  FlatMeta f;
  f.off.push_back(0);
  for (const auto& r : per_rank) {
    for (const auto& s : r) {
      f.ids.push_back(s.sample_id);
      f.lens.push_back(s.length);
    }
    f.off.push_back(static_cast<int64_t>(f.ids.size()));
  }
  return f;
}

void upload_meta(const FlatMeta& f, DeviceMeta& m) {
  void* host[3] = {const_cast<int64_t*>(f.off.data()), const_cast<uint64_t*>(f.ids.data()),
                   const_cast<int64_t*>(f.lens.data())};
  const int64_t bytes[3] = {static_cast<int64_t>(f.off.size() * 8), static_cast<int64_t>(f.ids.size() * 8),
                            static_cast<int64_t>(f.lens.size() * 8)};
  ck(sb_world_upload(m.w, host, bytes, nullptr), "metadata upload");
}

// Host copy of a device plan.
struct HostPlan {
  std::vector<uint64_t> id;
  std::vector<int32_t> idx, src, dst, send_idx, recv_idx, rev_idx;
  std::vector<int64_t> start, end, send_off, recv_off, target_rows;
  std::vector<double> per_gpu, occ;
  int32_t violations = 0;
  double total = 0, wir = 1;
};

HostPlan download(sb_planner* p, int W, int64_t n_bag_slots) {
  int64_t nc = 0, ns = 0;
  ck(sb_plan_sizes(p, nullptr, &nc, &ns), "plan");
  HostPlan h;
  h.id.resize(nc);
  h.idx.resize(nc);
  h.src.resize(nc);
  h.dst.resize(nc);
  h.send_idx.resize(nc);
  h.recv_idx.resize(nc);
  h.rev_idx.resize(nc);
  h.start.resize(nc);
  h.end.resize(nc);
  h.send_off.resize(W + 1);
  h.recv_off.resize(W + 1);
  h.target_rows.resize(W);
  h.per_gpu.resize(W);
  h.occ.resize(n_bag_slots);
  sb_plan_host o{};
  o.chunk_id = h.id.data();
  o.chunk_index = h.idx.data();
  o.chunk_start = h.start.data();
  o.chunk_end = h.end.data();
  o.chunk_src = h.src.data();
  o.chunk_dst = h.dst.data();
  o.send_off = h.send_off.data();
  o.send_idx = h.send_idx.data();
  o.recv_off = h.recv_off.data();
  o.recv_idx = h.recv_idx.data();
  o.rev_recv_idx = h.rev_idx.data();
  o.target_rows = h.target_rows.data();
  o.per_gpu_workload = h.per_gpu.data();
  o.per_bag_occupancy = n_bag_slots ? h.occ.data() : nullptr;
  ck(sb_plan_download(p, &o, nullptr), "plan download");
  h.violations = o.capacity_violations;
  h.total = o.total_workload;
  h.wir = o.wir;
  return h;
}

std::vector<std::vector<int>> lists(const std::vector<int64_t>& off, const std::vector<int32_t>& idx, int W) {
  std::vector<std::vector<int>> out(W);
  for (int r = 0; r < W; ++r) out[r].assign(idx.begin() + off[r], idx.begin() + off[r + 1]);
  return out;
}

RoutingPlan to_plan(const HostPlan& h, const std::vector<std::vector<SequenceInfo>>& seqs) {
  RoutingPlan plan;
  const int W = static_cast<int>(seqs.size());
  plan.world_size = W;
  plan.chunks.resize(h.id.size());
  for (std::size_t c = 0; c < h.id.size(); ++c)
    plan.chunks[c] = {h.id[c], h.idx[c], h.start[c], h.end[c], h.src[c], h.dst[c]};
  plan.send = lists(h.send_off, h.send_idx, W);
  plan.recv = lists(h.recv_off, h.recv_idx, W);
  plan.origin.resize(W);
  for (int r = 0; r < W; ++r)
    for (const SequenceInfo& s : seqs[r]) plan.origin[r].push_back({s.sample_id, 0, s.length});
  plan.target.resize(W);
  for (int r = 0; r < W; ++r)
    for (int c : plan.recv[r]) {
      const ChunkAssignment& ch = plan.chunks[c];
      plan.target[r].push_back({ch.sample_id, ch.start, ch.end - ch.start});
    }
  return plan;
}

void remember(sb_planner* p, const RoutingPlan& plan, const HostPlan& h) {
  Device& d = dev();
  d.last = p;
  d.last_plan = plan;
  d.last_valid = true;
  d.rev_off_of_last = h.send_off;
  d.rev_recv_of_last.assign(h.rev_idx.begin(), h.rev_idx.end());
}

// Upload an arbitrary plan to a planner sized for it; returns the planner.
sb_planner* device_plan(const RoutingPlan& plan) {
  Device& d = dev();
  if (d.last_valid && d.last && plan == d.last_plan) return d.last;
  const int W = plan.world_size;
  PlannerKey k;
  k.W = W;
  k.U = W;
  k.bag_off = {0, W};
  k.bag_ranks.resize(W);
  std::iota(k.bag_ranks.begin(), k.bag_ranks.end(), 0);
  k.d_model = 64;
  k.n_heads = W;  // any bag of W divides W heads
  k.d_head = 64 % W == 0 ? 64 / W : 0;
  if (k.d_head == 0) {
    k.d_model = W;
    k.d_head = 1;
  }
  k.n_blocks = 1;
  k.gamma = 1.0;
  k.k = 1.0;
  const int64_t n = static_cast<int64_t>(plan.chunks.size());
  sb_planner* p = planner_for(k, std::max<int64_t>(1, (n + W - 1) / W));
  std::vector<uint64_t> cid(n);
  std::vector<int32_t> cidx(n), csrc(n), cdst(n);
  std::vector<int64_t> cs(n), ce(n);
  for (int64_t c = 0; c < n; ++c) {
    const ChunkAssignment& ch = plan.chunks[c];
    cid[c] = ch.sample_id;
    cidx[c] = ch.chunk_index;
    cs[c] = ch.start;
    ce[c] = ch.end;
    csrc[c] = ch.source_rank;
    cdst[c] = ch.target_rank;
  }
  auto segs = [&](const std::vector<std::vector<Segment>>& L, std::vector<int64_t>& off, std::vector<uint64_t>& id,
                  std::vector<int64_t>& first, std::vector<int64_t>& len) {
    off.assign(1, 0);
    for (const auto& r : L) {
      for (const Segment& s : r) {
        id.push_back(s.sample_id);
        first.push_back(s.first_pos);
        len.push_back(s.length);
      }
      off.push_back(static_cast<int64_t>(id.size()));
    }
    while (static_cast<int>(off.size()) < W + 1) off.push_back(off.back());
  };
  std::vector<int64_t> ooff, ofirst, olen, toff, tfirst, tlen;
  std::vector<uint64_t> oid, tid;
  segs(plan.origin, ooff, oid, ofirst, olen);
  segs(plan.target, toff, tid, tfirst, tlen);
  ck(sb_plan_upload(p, n, cid.data(), cidx.data(), cs.data(), ce.data(), csrc.data(), cdst.data(), ooff.data(),
                    oid.data(), ofirst.data(), olen.data(), toff.data(), tid.data(), tfirst.data(), tlen.data(),
                    nullptr),
     "route");
  d.last = nullptr;
  d.last_valid = false;
  return p;
}

// ------------------------------------------------------------ device worlds
// Worlds of doubles: tensor 0 = 16-byte {id, pos} rows, tensor 1 = payload.
struct DevWorld {
  sb_world* w = nullptr;
  explicit DevWorld(int W, int n_heads, int width_doubles, int64_t rows, int max_bag) {
    sb_world_desc d{};
    const int64_t rb[1] = {static_cast<int64_t>(width_doubles) * 8};
    d.world_size = W;
    d.n_local = W;
    d.first_local = 0;
    d.n_heads = n_heads;
    d.n_payload = 1;
    d.n_aux = 0;
    d.row_bytes = rb;
    d.capacity_rows = std::max<int64_t>(rows, 1);
    d.max_bag = std::max(1, max_bag);
    ck(sb_world_create(&d, &w), "world");
  }
  ~DevWorld() {
    if (w) sb_world_destroy(w);
  }
  DevWorld(const DevWorld&) = delete;
  DevWorld& operator=(const DevWorld&) = delete;
};

struct Image {
  std::vector<uint64_t> meta;   // 2 words per row
  std::vector<double> payload;  // packed rows
};

// Host world -> packed image + layout (rows, pitches per rank).
void pack(const World& world, const std::vector<int>& ranks, Image& img, std::vector<int64_t>& rows,
          std::vector<int64_t>& pitch, std::vector<int32_t>& headcol) {
  const int W = static_cast<int>(world.ranks.size());
  rows.assign(W, 0);
  pitch.assign(2 * W, 0);
  headcol.assign(W, 0);
  for (int r = 0; r < W; ++r) {
    pitch[r] = 16;
    pitch[W + r] = static_cast<int64_t>(world.ranks[r].width) * 8;
  }
  for (int r : ranks) {
    const RankBuffer& b = world.ranks[r];
    rows[r] = b.num_rows();
    if (static_cast<int64_t>(b.positions.size()) != b.num_rows() ||
        static_cast<int64_t>(b.payload.size()) != b.num_rows() * b.width)
      throw IntegrityError("rank " + std::to_string(r) + " buffer sizes do not match its row count");
    for (int64_t i = 0; i < b.num_rows(); ++i) {
      img.meta.push_back(b.sample_ids[i]);
      img.meta.push_back(static_cast<uint64_t>(b.positions[i]));
    }
    img.payload.insert(img.payload.end(), b.payload.begin(), b.payload.end());
    if (b.width != world.payload_width && world.n_heads > 0)
      headcol[r] = b.head_lo * (world.payload_width / world.n_heads);
  }
}

void upload_world(DevWorld& dw, const World& world, const std::vector<int>& ranks) {
  Image img;
  std::vector<int64_t> rows, pitch;
  std::vector<int32_t> hc;
  pack(world, ranks, img, rows, pitch, hc);
  ck(sb_world_set_layout(dw.w, rows.data(), pitch.data(), nullptr), "world layout");
  ck(sb_world_set_headcol(dw.w, hc.data(), nullptr), "world layout");
  void* host[2] = {img.meta.data(), img.payload.data()};
  const int64_t bytes[2] = {static_cast<int64_t>(img.meta.size() * 8), static_cast<int64_t>(img.payload.size() * 8)};
  ck(sb_world_upload(dw.w, host, bytes, nullptr), "world upload");
}

// Read ranks back from a device world into host RankBuffers (rows/payload).
void read_rank(DevWorld& dw, int r, RankBuffer& b) {
  int64_t nb = 0;
  ck(sb_world_read_rank(dw.w, 0, r, nullptr, 0, &nb, nullptr), "world read");
  std::vector<uint64_t> meta(nb / 8);
  ck(sb_world_read_rank(dw.w, 0, r, meta.data(), nb, &nb, nullptr), "world read");
  const int64_t rows = nb / 16;
  b.sample_ids.resize(rows);
  b.positions.resize(rows);
  for (int64_t i = 0; i < rows; ++i) {
    b.sample_ids[i] = meta[2 * i];
    b.positions[i] = static_cast<int64_t>(meta[2 * i + 1]);
  }
  ck(sb_world_read_rank(dw.w, 1, r, nullptr, 0, &nb, nullptr), "world read");
  b.payload.resize(nb / 8);
  ck(sb_world_read_rank(dw.w, 1, r, b.payload.data(), nb, &nb, nullptr), "world read");
}

int64_t total_rows(const World& w) {
  int64_t n = 0;
  for (const auto& b : w.ranks) n += b.num_rows();
  return n;
}

void check_world_matches_layout(const World& world, const std::vector<std::vector<Segment>>& layout,
                                const char* op) {  // exchange.cpp:96-123
  if (world.ranks.size() != layout.size()) {
    throw IntegrityError(std::string(op) + ": plan world size " + std::to_string(layout.size()) +
                         " != world ranks " + std::to_string(world.ranks.size()));
  }
  for (std::size_t r = 0; r < layout.size(); ++r) {
    const RankBuffer& buf = world.ranks[r];
    if (buf.mode != LayoutMode::ChunkFullHeads || buf.width != world.payload_width) {
      throw IntegrityError(std::string(op) + ": rank " + std::to_string(r) +
                           " is not in (partial sequences, full heads) layout");
    }
    if (buf.segments.size() != layout[r].size()) {
      throw IntegrityError(std::string(op) + ": rank " + std::to_string(r) + " holds " +
                           std::to_string(buf.segments.size()) + " sequences, plan expects " +
                           std::to_string(layout[r].size()));
    }
    for (std::size_t s = 0; s < layout[r].size(); ++s) {
      if (!(buf.segments[s] == layout[r][s])) {
        throw IntegrityError(std::string(op) + ": rank " + std::to_string(r) + " segment mismatch for sample " +
                             std::to_string(layout[r][s].sample_id));
      }
    }
  }
}

World run_route(const World& world, const RoutingPlan& plan, bool reverse) {
  const std::vector<std::vector<Segment>>& from = reverse ? plan.target : plan.origin;
  const std::vector<std::vector<Segment>>& to = reverse ? plan.origin : plan.target;
  check_world_matches_layout(world, from, "route");
  std::lock_guard<std::mutex> lock(dev().mu);
  sb_planner* p = device_plan(plan);
  const int W = plan.world_size;
  const int64_t rows = std::max<int64_t>(total_rows(world), 1);
  DevWorld src(W, world.n_heads, world.payload_width, rows, 1), dst(W, world.n_heads, world.payload_width, rows, 1);
  std::vector<int> all(W);
  std::iota(all.begin(), all.end(), 0);
  upload_world(src, world, all);
  ck(sb_route(p, reverse ? 1 : 0, src.w, dst.w, nullptr), "route");
  ck(sb_world_status(dst.w, nullptr), "route");
  World out;
  out.payload_width = world.payload_width;
  out.n_heads = world.n_heads;
  out.ranks.resize(W);
  for (int r = 0; r < W; ++r) {
    RankBuffer& b = out.ranks[r];
    b.rank = r;
    b.mode = LayoutMode::ChunkFullHeads;
    b.head_lo = 0;
    b.head_hi = world.n_heads;
    b.width = world.payload_width;
    b.segments = to[r];
    read_rank(dst, r, b);
  }
  return out;
}

std::vector<sb_block_move> to_device_moves(const std::vector<BlockMove>& moves) {
  std::vector<sb_block_move> out(moves.size());
  for (std::size_t i = 0; i < moves.size(); ++i) {
    const BlockMove& m = moves[i];
    out[i] = sb_block_move{m.src_rank, m.dst_rank, m.src_row, m.dst_row, m.n_rows,
                           static_cast<int64_t>(m.src_col) * 8, static_cast<int64_t>(m.dst_col) * 8,
                           static_cast<int64_t>(m.n_cols) * 8, m.copy_meta ? 1 : 0, 0};
  }
  return out;
}

// Runs a move list on the device: src ranks `sr` uploaded from `src`, the
// destination world pre-filled from `dst` (moves may write partial rows), and
// the touched destination ranks `dr` read back.
void device_moves(const World& src, const std::vector<int>& sr, const std::vector<BlockMove>& moves, World& dst,
                  const std::vector<int>& dr) {
  const int W = static_cast<int>(src.ranks.size());
  if (static_cast<int>(dst.ranks.size()) != W) throw ConfigError("apply_block_moves: world sizes differ");
  int max_bag = 1;
  for (const auto& b : dst.ranks)
    if (b.width > 0 && dst.payload_width % b.width == 0) max_bag = std::max(max_bag, dst.payload_width / b.width);
  DevWorld s(W, src.n_heads, src.payload_width, std::max<int64_t>(total_rows(src), 1), max_bag);
  DevWorld d(W, dst.n_heads, dst.payload_width, std::max<int64_t>(total_rows(dst), 1), max_bag);
  upload_world(s, src, sr);
  upload_world(d, dst, dr);
  const auto dm = to_device_moves(moves);
  ck(sb_apply_moves(s.w, d.w, dm.data(), static_cast<int64_t>(dm.size()), nullptr), "apply_block_moves");
  for (int r : dr) read_rank(d, r, dst.ranks[r]);
}

}  // namespace

// ================================================================ topology
namespace {
constexpr int kMaxUnitSize = 1 << 20;
int parse_int(std::string_view s, std::size_t& pos, const char* what) {
  const std::size_t start = pos;
  long long v = 0;
  while (pos < s.size() && s[pos] >= '0' && s[pos] <= '9') {
    v = v * 10 + (s[pos] - '0');
    if (v > kMaxUnitSize) throw ParseError(std::string(what) + " value too large", start);
    ++pos;
  }
  if (pos == start) throw ParseError(std::string("expected digits for ") + what, start);
  if (v < 1) throw ParseError(std::string(what) + " must be >= 1", start);
  return static_cast<int>(v);
}
}  // namespace

Topology parse_topology(std::string_view spec) {  // topology.cpp:31-65 grammar
  if (spec.empty()) throw ParseError("empty topology spec", 0);
  std::vector<BagSpec> terms;
  std::size_t pos = 0;
  for (;;) {
    if (pos >= spec.size() || spec[pos] != 'g') throw ParseError("expected 'g'", pos);
    ++pos;
    BagSpec t;
    t.gpus_per_bag = parse_int(spec, pos, "bag size");
    if (pos >= spec.size() || spec[pos] != 'n') throw ParseError("expected 'n'", pos);
    ++pos;
    t.num_bags = parse_int(spec, pos, "bag count");
    terms.push_back(t);
    if (pos == spec.size()) break;
    if (spec[pos] != '+') throw ParseError("expected '+' or end of spec", pos);
    ++pos;
  }
  Topology topo;
  int next = 0;
  for (const BagSpec& t : terms) {
    for (int i = 0; i < t.num_bags; ++i) {
      ComputeBag bag;
      bag.bag_id = static_cast<int>(topo.bags.size());
      for (int k = 0; k < t.gpus_per_bag; ++k) bag.gpu_ranks.push_back(next + k);
      next += t.gpus_per_bag;
      if (next > kMaxUnitSize) throw ParseError("unit size too large", 0);
      topo.bags.push_back(std::move(bag));
    }
  }
  topo.unit_size = next;
  return topo;
}

std::string format_topology(const Topology& topo) {
  std::string out;
  for (std::size_t i = 0; i < topo.bags.size();) {
    std::size_t j = i;
    while (j < topo.bags.size() && topo.bags[j].size() == topo.bags[i].size()) ++j;
    if (!out.empty()) out += '+';
    out += "g" + std::to_string(topo.bags[i].size()) + "n" + std::to_string(j - i);
    i = j;
  }
  return out;
}

WorldLayout replicate(const Topology& topo, int world_size) {
  if (topo.unit_size < 1) throw ConfigError("topology has no GPUs");
  if (world_size < topo.unit_size)
    throw ConfigError("world_size " + std::to_string(world_size) + " is smaller than the sharding unit " +
                      std::to_string(topo.unit_size));
  if (world_size % topo.unit_size != 0)
    throw ConfigError("world_size " + std::to_string(world_size) + " is not a multiple of the sharding unit " +
                      std::to_string(topo.unit_size));
  return WorldLayout{topo, world_size};
}

BagLocation bag_of_rank(const WorldLayout& layout, int rank) {
  if (rank < 0 || rank >= layout.world_size)
    throw ConfigError("rank " + std::to_string(rank) + " outside world of " + std::to_string(layout.world_size));
  BagLocation loc;
  loc.replica_id = rank / layout.unit.unit_size;
  const int local = rank % layout.unit.unit_size, base = loc.replica_id * layout.unit.unit_size;
  for (const ComputeBag& bag : layout.unit.bags) {
    for (int r : bag.gpu_ranks) {
      if (r == local) {
        loc.bag_id = bag.bag_id;
        for (int q : bag.gpu_ranks)
          if (q + base != rank) loc.peer_ranks.push_back(q + base);
        return loc;
      }
    }
  }
  throw ConfigError("rank not covered by any bag");
}

ComputeBag global_bag(const WorldLayout& layout, int replica_id, int bag_id) {
  if (replica_id < 0 || replica_id >= layout.num_replicas())
    throw ConfigError("replica " + std::to_string(replica_id) + " out of range");
  if (bag_id < 0 || bag_id >= static_cast<int>(layout.unit.bags.size()))
    throw ConfigError("bag " + std::to_string(bag_id) + " out of range");
  ComputeBag bag = layout.unit.bags[bag_id];
  for (int& r : bag.gpu_ranks) r += replica_id * layout.unit.unit_size;
  return bag;
}

// ================================================================== model
void ModelShape::validate() const {  // workload_model.cpp:15-24
  if (d_model < 1 || n_heads < 1 || d_head < 1 || n_blocks < 1) throw ConfigError("model shape fields must be >= 1");
  if (static_cast<std::int64_t>(n_heads) * d_head != d_model)
    throw ConfigError("n_heads * d_head must equal d_model (" + std::to_string(n_heads) + " * " +
                      std::to_string(d_head) + " != " + std::to_string(d_model) + ")");
}

ModelShape ModelShape::flux() { return ModelShape{3072, 24, 128, 57}; }

void WorkloadModel::validate() const {
  shape.validate();
  if (!(gamma > 0.0)) throw ConfigError("gamma must be positive");
  if (!(k > 0.0)) throw ConfigError("k must be positive");
}

// Scalar form of the planner's device workload (same operation order).
double gamma_weighted_workload(std::int64_t seq_len, const WorkloadModel& model) {
  if (seq_len < 0) throw ConfigError("seq_len must be >= 0");
  const volatile double l = static_cast<double>(seq_len), d = static_cast<double>(model.shape.d_model);
  volatile double lin = 24.0 * l;
  lin = lin * d;
  lin = lin * d;
  volatile double att = model.gamma * 4.0;
  att = att * l;
  att = att * l;
  att = att * d;
  return lin + att;
}

double per_gpu_workload(std::int64_t seq_len, int bag_size, const WorkloadModel& model) {
  if (bag_size < 1) throw ConfigError("bag_size must be >= 1");
  if (model.shape.n_heads % bag_size != 0)
    throw ConfigError("bag size " + std::to_string(bag_size) + " does not divide n_heads " +
                      std::to_string(model.shape.n_heads) + "; the attention head split is infeasible");
  return gamma_weighted_workload(seq_len, model) / static_cast<double>(bag_size);
}

double workload_imbalance_ratio(const std::vector<double>& w) {  // metrics.cpp:20-31
  if (w.empty()) throw ConfigError("WIR of empty workload list");
  double lo = w.front(), hi = w.front();
  for (double x : w) {
    if (!(x >= 0.0)) throw ConfigError("negative per-GPU workload");
    lo = std::min(lo, x);
    hi = std::max(hi, x);
  }
  if (hi == 0.0) return 1.0;
  if (lo == 0.0) return std::numeric_limits<double>::infinity();
  return hi / lo;
}

std::vector<std::int64_t> chunk_lengths(std::int64_t total_len, int parts) {
  if (parts < 1) throw ConfigError("chunk_lengths: parts must be >= 1");
  if (total_len < 0) throw ConfigError("chunk_lengths: negative length");
  std::vector<std::int64_t> lens(parts, total_len / parts);
  for (std::int64_t i = 0; i < total_len % parts; ++i) ++lens[i];
  return lens;
}

// =============================================================== balancer
std::vector<SequenceAssignment> assign_to_bags(std::vector<SequenceWorkload> workloads,
                                               const std::vector<ComputeBag>& bags) {
  if (bags.empty()) throw ConfigError("assign_to_bags: no bags");
  for (const auto& w : workloads)
    if (!(w.workload >= 0.0)) throw ConfigError("assign_to_bags: negative workload");
  PlannerKey k;
  k.bag_off.push_back(0);
  int g_all = 0;
  for (const ComputeBag& b : bags) {
    // Divergence (documented in DESIGN.md): the reference gives an empty bag
    // capacity 0 and occupancy 0/inf; the device planner rejects it.
    if (b.size() < 1) throw ConfigError("assign_to_bags: empty bag");
    for (int i = 0; i < b.size(); ++i) k.bag_ranks.push_back(g_all + i);
    g_all += b.size();
    k.bag_off.push_back(g_all);
  }
  k.W = k.U = g_all;
  // assignment-only planner (all shape fields 0): the greedy never reads the
  // model, so there is no head-divisibility check to satisfy
  k.n_heads = k.d_head = k.d_model = k.n_blocks = 0;
  k.gamma = 1.0;
  k.k = 1.0;
  std::lock_guard<std::mutex> lock(dev().mu);
  const int64_t n = static_cast<int64_t>(workloads.size());
  sb_planner* p = planner_for(k, std::max<int64_t>(n, 1));
  std::vector<uint64_t> ids(n), oid(n);
  std::vector<double> w(n), ow(n);
  std::vector<int32_t> ob(n);
  for (int64_t i = 0; i < n; ++i) {
    ids[i] = workloads[i].sample_id;
    w[i] = workloads[i].workload;
  }
  ck(sb_assign_to_bags(p, n, ids.data(), w.data(), oid.data(), ow.data(), ob.data(), nullptr), "assign_to_bags");
  if (dev().last == p) dev().last_valid = false;
  std::vector<SequenceAssignment> out(n);
  for (int64_t i = 0; i < n; ++i) out[i] = {oid[i], ow[i], bags[ob[i]].bag_id};
  return out;
}

PlanResult plan_routing(const std::vector<std::vector<SequenceInfo>>& per_rank_seqs, const WorkloadModel& model,
                        const WorldLayout& layout) {
  model.validate();
  const int world = layout.world_size;
  if (static_cast<int>(per_rank_seqs.size()) != world)
    throw ConfigError("plan_routing: sequence metadata for " + std::to_string(per_rank_seqs.size()) +
                      " ranks, world is " + std::to_string(world));
  for (const ComputeBag& bag : layout.unit.bags)
    if (model.shape.n_heads % bag.size() != 0)
      throw ConfigError("bag of " + std::to_string(bag.size()) + " GPUs does not divide n_heads " +
                        std::to_string(model.shape.n_heads));
  std::lock_guard<std::mutex> lock(dev().mu);
  const FlatMeta f = flatten(per_rank_seqs);
  const int64_t n = static_cast<int64_t>(f.ids.size());
  sb_planner* p = planner_for(key_for(layout, model), std::max<int64_t>(n, 1));
  DeviceMeta& m = meta_buf(n, world);
  upload_meta(f, m);
  ck(sb_plan(p, static_cast<const uint64_t*>(m.ids), static_cast<const int64_t*>(m.lens),
             static_cast<const int64_t*>(m.off), nullptr),
     "plan_routing");
  const HostPlan h = download(p, world, static_cast<int64_t>(layout.num_replicas()) * layout.unit.bags.size());
  PlanResult res;
  res.plan = to_plan(h, per_rank_seqs);
  res.report.per_gpu_workload = h.per_gpu;
  res.report.per_bag_occupancy = h.occ;
  res.report.capacity_violations = h.violations;
  res.report.total_workload = h.total;
  res.report.wir = h.wir;
  remember(p, res.plan, h);
  return res;
}

RoutingPlan identity_plan(const std::vector<std::vector<SequenceInfo>>& per_rank_seqs) {
  const int W = static_cast<int>(per_rank_seqs.size());
  if (W < 1) {
    RoutingPlan empty;
    return empty;
  }
  // identity planning never reads the bag tables: one 1-rank bag replicated
  // W times keeps the planner at one bag per replica for any world size
  Topology t;
  t.bags.push_back(ComputeBag{0, {0}});
  t.unit_size = 1;
  WorkloadModel model;
  std::lock_guard<std::mutex> lock(dev().mu);
  const FlatMeta f = flatten(per_rank_seqs);
  const int64_t n = static_cast<int64_t>(f.ids.size());
  sb_planner* p = planner_for(key_for(WorldLayout{t, W}, model), std::max<int64_t>(n, 1));
  DeviceMeta& m = meta_buf(n, W);
  upload_meta(f, m);
  ck(sb_plan_identity(p, static_cast<const uint64_t*>(m.ids), static_cast<const int64_t*>(m.lens),
                      static_cast<const int64_t*>(m.off), nullptr),
     "identity_plan");
  const HostPlan h = download(p, W, 0);
  RoutingPlan plan = to_plan(h, per_rank_seqs);
  remember(p, plan, h);
  return plan;
}

RoutingPlan reverse_plan(const RoutingPlan& plan) {
  RoutingPlan rev;
  rev.world_size = plan.world_size;
  rev.origin = plan.target;
  rev.target = plan.origin;
  rev.chunks.reserve(plan.chunks.size());
  for (const ChunkAssignment& c : plan.chunks) {
    ChunkAssignment r = c;
    std::swap(r.source_rank, r.target_rank);
    rev.chunks.push_back(r);
  }
  const int W = plan.world_size;
  std::lock_guard<std::mutex> lock(dev().mu);
  Device& d = dev();
  std::vector<int64_t> off;
  std::vector<int32_t> idx;
  if (d.last_valid && d.last && plan == d.last_plan) {
    off = d.rev_off_of_last;
    idx.assign(d.rev_recv_of_last.begin(), d.rev_recv_of_last.end());
  } else {
    sb_planner* p = device_plan(plan);
    ck(sb_plan_manifests(p, nullptr), "reverse_plan");
    const HostPlan h = download(p, W, 0);
    off = h.send_off;
    idx = h.rev_idx;
  }
  rev.send = plan.recv;  // balancer.cpp:256-258: reversed sources are forward targets
  rev.recv = lists(off, idx, W);
  return rev;
}

// =============================================================== exchange
double payload_value(std::uint64_t sample_id, std::int64_t position, int col) {
  auto mix = [](std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  };
  std::uint64_t k = 0x8f51a7c0c0c0f5a3ULL;
  for (std::uint64_t p : std::initializer_list<std::uint64_t>{0x7061796c6f6164ULL, sample_id, static_cast<std::uint64_t>(position),
                          static_cast<std::uint64_t>(col)})
    k = mix(k ^ p);
  return static_cast<double>(k >> 11) * 0x1.0p-53;
}

double block_perturbation(std::uint64_t sample_id, std::int64_t position) {
  auto mix = [](std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  };
  std::uint64_t k = 0x8f51a7c0c0c0f5a3ULL;
  for (std::uint64_t p : std::initializer_list<std::uint64_t>{0x706572747572ULL, sample_id, static_cast<std::uint64_t>(position)})
    k = mix(k ^ p);
  return static_cast<double>(k >> 11) * 0x1.0p-53;
}

std::vector<std::vector<SequenceInfo>> gather_sequence_info(
    const std::vector<std::vector<SampleMeta>>& per_rank_samples) {
  std::vector<std::vector<SequenceInfo>> info(per_rank_samples.size());
  for (std::size_t r = 0; r < per_rank_samples.size(); ++r)
    for (const SampleMeta& s : per_rank_samples[r]) info[r].push_back({s.sample_id, s.total_len()});
  return info;
}

World make_world(const std::vector<std::vector<SampleMeta>>& per_rank_samples, int payload_width, int n_heads) {
  if (payload_width < 1 || n_heads < 1 || payload_width % n_heads != 0)
    throw ConfigError("payload width must be a positive multiple of n_heads");
  const int W = static_cast<int>(per_rank_samples.size());
  World world;
  world.payload_width = payload_width;
  world.n_heads = n_heads;
  world.ranks.resize(W);
  if (W == 0) return world;
  const auto info = gather_sequence_info(per_rank_samples);
  const FlatMeta f = flatten(info);
  int64_t rows = 0;
  for (int64_t l : f.lens) rows += l;
  std::lock_guard<std::mutex> lock(dev().mu);
  DeviceMeta& m = meta_buf(static_cast<int64_t>(f.ids.size()), W);
  upload_meta(f, m);
  DevWorld dw(W, n_heads, payload_width, std::max<int64_t>(rows, 1), 1);
  ck(sb_world_layout_origin(dw.w, static_cast<const int64_t*>(m.lens), static_cast<const int64_t*>(m.off), nullptr),
     "make_world");
  ck(sb_world_fill_witness(dw.w, static_cast<const uint64_t*>(m.ids), static_cast<const int64_t*>(m.lens),
                           static_cast<const int64_t*>(m.off), nullptr),
     "make_world");
  for (int r = 0; r < W; ++r) {
    RankBuffer& b = world.ranks[r];
    b.rank = r;
    b.mode = LayoutMode::ChunkFullHeads;
    b.head_lo = 0;
    b.head_hi = n_heads;
    b.width = payload_width;
    for (const SequenceInfo& s : info[r]) b.segments.push_back({s.sample_id, 0, s.length});
    read_rank(dw, r, b);
  }
  return world;
}

World route(const World& world, const RoutingPlan& plan, Exec) { return run_route(world, plan, false); }

World reverse_route(const World& world, const RoutingPlan& plan, Exec) { return run_route(world, plan, true); }

namespace {
struct BagView {
  std::vector<std::uint64_t> ids;
  std::vector<std::int64_t> full;
};

BagView check_bag_chunk_layout(const World& world, const ComputeBag& bag) {  // exchange.cpp:210-251
  BagView v;
  const int g = bag.size();
  const RankBuffer& first = world.ranks.at(bag.gpu_ranks.front());
  for (const Segment& s : first.segments) v.ids.push_back(s.sample_id);
  for (int m = 0; m < g; ++m) {
    const RankBuffer& buf = world.ranks.at(bag.gpu_ranks[m]);
    if (buf.mode != LayoutMode::ChunkFullHeads)
      throw IntegrityError("pre_attn: rank " + std::to_string(bag.gpu_ranks[m]) + " is not in chunk layout");
    if (buf.segments.size() != v.ids.size()) throw IntegrityError("pre_attn: bag members disagree on sequence count");
    for (std::size_t s = 0; s < buf.segments.size(); ++s)
      if (buf.segments[s].sample_id != v.ids[s])
        throw IntegrityError("pre_attn: bag members disagree on sample " + std::to_string(v.ids[s]));
  }
  for (std::size_t s = 0; s < v.ids.size(); ++s) {
    std::int64_t full = 0;
    for (int m = 0; m < g; ++m) full += world.ranks.at(bag.gpu_ranks[m]).segments[s].length;
    const auto lens = chunk_lengths(full, g);
    std::int64_t start = 0;
    for (int m = 0; m < g; ++m) {
      const Segment& seg = world.ranks.at(bag.gpu_ranks[m]).segments[s];
      if (seg.first_pos != start || seg.length != lens[m])
        throw IntegrityError("pre_attn: sample " + std::to_string(v.ids[s]) +
                             " is not split by the canonical chunk rule");
      start += lens[m];
    }
    v.full.push_back(full);
  }
  return v;
}
}  // namespace

std::vector<std::int64_t> pre_attn(World& world, const ComputeBag& bag, Exec) {
  const int g = bag.size();
  if (g == 1) {
    std::vector<std::int64_t> lens;
    for (const Segment& s : world.ranks.at(bag.gpu_ranks[0]).segments) lens.push_back(s.length);
    return lens;
  }
  if (world.n_heads % g != 0)
    throw ConfigError("pre_attn: bag of " + std::to_string(g) + " GPUs does not divide n_heads " +
                      std::to_string(world.n_heads));
  const BagView v = check_bag_chunk_layout(world, bag);
  const int slice = world.payload_width / g, hpr = world.n_heads / g;
  std::int64_t total = 0;
  for (std::int64_t l : v.full) total += l;
  // staged (full sequence, H/G heads) shells for the bag members
  World staged;
  staged.payload_width = world.payload_width;
  staged.n_heads = world.n_heads;
  staged.ranks.resize(world.ranks.size());
  for (std::size_t r = 0; r < world.ranks.size(); ++r) staged.ranks[r].width = world.payload_width;
  for (int m = 0; m < g; ++m) {
    RankBuffer& b = staged.ranks[bag.gpu_ranks[m]];
    b.rank = bag.gpu_ranks[m];
    b.mode = LayoutMode::FullSeqPartialHeads;
    b.head_lo = m * hpr;
    b.head_hi = (m + 1) * hpr;
    b.width = slice;
    b.sample_ids.assign(total, 0);
    b.positions.assign(total, 0);
    b.payload.assign(total * slice, 0.0);
    for (std::size_t s = 0; s < v.ids.size(); ++s) b.segments.push_back({v.ids[s], 0, v.full[s]});
  }
  std::vector<BlockMove> moves;  // exchange.cpp:298-325 move construction
  for (int sm = 0; sm < g; ++sm) {
    const RankBuffer& src = world.ranks[bag.gpu_ranks[sm]];
    std::int64_t row = 0, base = 0;
    for (std::size_t s = 0; s < v.ids.size(); ++s) {
      const Segment& seg = src.segments[s];
      if (seg.length > 0)
        for (int dm = 0; dm < g; ++dm)
          moves.push_back({bag.gpu_ranks[sm], row, dm * slice, bag.gpu_ranks[dm], base + seg.first_pos, 0, seg.length,
                           slice, true});
      row += seg.length;
      base += v.full[s];
    }
  }
  device_moves(world, bag.gpu_ranks, moves, staged, bag.gpu_ranks);
  for (int m = 0; m < g; ++m) world.ranks[bag.gpu_ranks[m]] = std::move(staged.ranks[bag.gpu_ranks[m]]);
  return v.full;
}

void post_attn(World& world, const ComputeBag& bag, Exec) {
  const int g = bag.size();
  if (g == 1) return;
  std::vector<std::uint64_t> ids;
  std::vector<std::int64_t> full;
  const RankBuffer& first = world.ranks.at(bag.gpu_ranks.front());
  if (first.mode != LayoutMode::FullSeqPartialHeads)
    throw IntegrityError("post_attn: bag is not in (full sequences, partial heads) layout");
  for (const Segment& s : first.segments) {
    ids.push_back(s.sample_id);
    full.push_back(s.length);
  }
  const int slice = world.payload_width / g, hpr = world.n_heads / g;
  for (int m = 0; m < g; ++m) {  // exchange.cpp:351-369 validation
    const RankBuffer& b = world.ranks.at(bag.gpu_ranks[m]);
    if (b.mode != LayoutMode::FullSeqPartialHeads || b.width != slice || b.head_lo != m * hpr ||
        b.head_hi != (m + 1) * hpr)
      throw IntegrityError("post_attn: rank " + std::to_string(bag.gpu_ranks[m]) +
                           " head slice does not match its bag position");
    if (b.segments.size() != ids.size()) throw IntegrityError("post_attn: bag members disagree on sequence count");
    for (std::size_t s = 0; s < ids.size(); ++s)
      if (b.segments[s].sample_id != ids[s] || b.segments[s].length != full[s] || b.segments[s].first_pos != 0)
        throw IntegrityError("post_attn: bag members disagree on sample " + std::to_string(ids[s]));
  }
  std::vector<std::vector<std::int64_t>> lens(ids.size()), starts(ids.size());
  for (std::size_t s = 0; s < ids.size(); ++s) {
    lens[s] = chunk_lengths(full[s], g);
    std::int64_t st = 0;
    for (int m = 0; m < g; ++m) {
      starts[s].push_back(st);
      st += lens[s][m];
    }
  }
  World staged;
  staged.payload_width = world.payload_width;
  staged.n_heads = world.n_heads;
  staged.ranks.resize(world.ranks.size());
  for (std::size_t r = 0; r < world.ranks.size(); ++r) staged.ranks[r].width = world.payload_width;
  for (int m = 0; m < g; ++m) {
    RankBuffer& b = staged.ranks[bag.gpu_ranks[m]];
    b.rank = bag.gpu_ranks[m];
    b.mode = LayoutMode::ChunkFullHeads;
    b.head_lo = 0;
    b.head_hi = world.n_heads;
    b.width = world.payload_width;
    std::int64_t rows = 0;
    for (std::size_t s = 0; s < ids.size(); ++s) {
      b.segments.push_back({ids[s], starts[s][m], lens[s][m]});
      rows += lens[s][m];
    }
    b.sample_ids.assign(rows, 0);
    b.positions.assign(rows, 0);
    b.payload.assign(rows * world.payload_width, 0.0);
  }
  std::vector<BlockMove> moves;  // exchange.cpp:406-431
  for (int dm = 0; dm < g; ++dm) {
    std::int64_t row = 0, base = 0;
    for (std::size_t s = 0; s < ids.size(); ++s) {
      const std::int64_t len = lens[s][dm];
      if (len > 0)
        for (int sm = 0; sm < g; ++sm)
          moves.push_back({bag.gpu_ranks[sm], base + starts[s][dm], 0, bag.gpu_ranks[dm], row, sm * slice, len,
                           slice, sm == 0});
      row += len;
      base += full[s];
    }
  }
  device_moves(world, bag.gpu_ranks, moves, staged, bag.gpu_ranks);
  for (int m = 0; m < g; ++m) world.ranks[bag.gpu_ranks[m]] = std::move(staged.ranks[bag.gpu_ranks[m]]);
}

void apply_block_moves(const World& src, const std::vector<BlockMove>& moves, World& dst, Exec) {
  std::vector<int> sr, dr;
  for (std::size_t r = 0; r < src.ranks.size(); ++r) sr.push_back(static_cast<int>(r));
  for (std::size_t r = 0; r < dst.ranks.size(); ++r) dr.push_back(static_cast<int>(r));
  device_moves(src, sr, moves, dst, dr);
}

void apply_block_moves_serial(const World& src, const std::vector<BlockMove>& moves, World& dst) {
  apply_block_moves(src, moves, dst, Exec::Serial);
}

void apply_block_moves_parallel(const World& src, const std::vector<BlockMove>& moves, World& dst) {
  apply_block_moves(src, moves, dst, Exec::Parallel);
}

std::uint64_t content_checksum(const World& world) {
  const int W = static_cast<int>(world.ranks.size());
  if (W == 0) return 0;
  int max_bag = 1;
  for (const auto& b : world.ranks)
    if (b.width > 0 && world.payload_width % b.width == 0) max_bag = std::max(max_bag, world.payload_width / b.width);
  DevWorld dw(W, world.n_heads, world.payload_width, std::max<int64_t>(total_rows(world), 1), max_bag);
  std::vector<int> all(W);
  std::iota(all.begin(), all.end(), 0);
  upload_world(dw, world, all);
  std::lock_guard<std::mutex> lock(dev().mu);  // meta_buf is the process-wide staging buffer
  DeviceMeta& m = meta_buf(1, 1);
  std::uint64_t zero = 0, acc = 0;
  void* host0[3] = {&zero, nullptr, nullptr};
  const int64_t b0[3] = {8, 0, 0};
  ck(sb_world_upload(m.w, host0, b0, nullptr), "checksum");
  ck(sb_world_checksum(dw.w, static_cast<uint64_t*>(m.off), nullptr), "checksum");
  void* host1[3] = {&acc, nullptr, nullptr};
  ck(sb_world_download(m.w, host1, b0, nullptr), "checksum");
  ck(sb_world_status(m.w, nullptr), "checksum");
  return acc;
}

bool worlds_bitwise_equal(const World& a, const World& b) {  // exchange.cpp:459-480
  if (a.payload_width != b.payload_width || a.n_heads != b.n_heads || a.ranks.size() != b.ranks.size()) return false;
  for (std::size_t r = 0; r < a.ranks.size(); ++r) {
    const RankBuffer& x = a.ranks[r];
    const RankBuffer& y = b.ranks[r];
    if (x.mode != y.mode || x.head_lo != y.head_lo || x.head_hi != y.head_hi || x.width != y.width ||
        x.segments != y.segments || x.sample_ids != y.sample_ids || x.positions != y.positions)
      return false;
    if (x.payload.size() != y.payload.size()) return false;
    if (!x.payload.empty() && std::memcmp(x.payload.data(), y.payload.data(), x.payload.size() * sizeof(double)) != 0)
      return false;
  }
  return true;
}

}  // namespace seqbal
