// SPDX-License-Identifier: Apache-2.0
//
// seqbal -- C++ host API of the B200-native balance-and-redistribute path.
//
// Drop-in for the reference library's public headers
// (/root/reference/proj/include/seqbal/{error,topology,workload_model,
// balancer,exchange,metrics}.hpp): the same namespace, type names, field
// names and function signatures for everything on the plan -> route ->
// Ulysses -> reverse path, so code that calls only those (the CLI's `plan`,
// the exchange benches, the balancer/exchange/topology tests) recompiles
// against libseqbal.so unchanged.  simulator.cpp and the CLI's other
// subcommands also use the modelled-cost layer (flops_per_block, CostModel,
// estimate_fbl, tokens_per_second, hardware_flops_utilization, fit_gamma,
// FitError, ScenarioConfig), which is off the hot path and NOT declared here
// (INTEGRATION.md section 1).
//
// Every planning step and every byte of data movement runs in
// libseqbal_cuda.so (sm_100a) through the C-ABI in seqbal_capi.h; this layer
// converts between the reference's host containers and device buffers and
// re-throws the reference's exception classes.  There is no CPU fallback:
// without a CUDA device the calls throw.
//
// Per-name headers (balancer.hpp, exchange.hpp, ...) include this file.
#pragma once

#include <cstdint>
#include <iosfwd>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace seqbal {

// ---------------------------------------------------------------- errors
// Mirrors error.hpp:10-40 (class names, bases, ParseError's byte offset).
class ParseError : public std::invalid_argument {
 public:
  ParseError(const std::string& what, std::size_t offset);
  std::size_t offset() const { return offset_; }

 private:
  std::size_t offset_;
};

class ConfigError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};

class IntegrityError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// --------------------------------------------------------------- topology
// topology.hpp:10-69.
struct BagSpec {
  int gpus_per_bag = 1;
  int num_bags = 1;
};

struct ComputeBag {
  int bag_id = 0;
  std::vector<int> gpu_ranks;
  int size() const { return static_cast<int>(gpu_ranks.size()); }
  bool operator==(const ComputeBag&) const = default;
};

struct Topology {
  std::vector<ComputeBag> bags;
  int unit_size = 0;
  bool operator==(const Topology&) const = default;
};

Topology parse_topology(std::string_view spec);
std::string format_topology(const Topology& topo);

struct WorldLayout {
  Topology unit;
  int world_size = 0;
  int num_replicas() const { return unit.unit_size ? world_size / unit.unit_size : 0; }
};

WorldLayout replicate(const Topology& topo, int world_size);

struct BagLocation {
  int replica_id = 0;
  int bag_id = 0;
  std::vector<int> peer_ranks;
};

BagLocation bag_of_rank(const WorldLayout& layout, int rank);
ComputeBag global_bag(const WorldLayout& layout, int replica_id, int bag_id);

// --------------------------------------------------------- workload model
// workload_model.hpp:13-80.
struct ModelShape {
  int d_model = 3072;
  int n_heads = 24;
  int d_head = 128;
  int n_blocks = 57;
  void validate() const;
  static ModelShape flux();
};

inline constexpr double kGammaH100 = 0.49;
inline constexpr double kGammaH100LatencyFit = 0.385;

struct WorkloadModel {
  ModelShape shape;
  double gamma = kGammaH100;
  double k = 4.0e-15;
  void validate() const;
};

double gamma_weighted_workload(std::int64_t seq_len, const WorkloadModel& model);
double per_gpu_workload(std::int64_t seq_len, int bag_size, const WorkloadModel& model);

// --------------------------------------------------------------- balancer
// balancer.hpp:13-104.
struct SequenceWorkload {
  std::uint64_t sample_id = 0;
  double workload = 0.0;
};

struct SequenceAssignment {
  std::uint64_t sample_id = 0;
  double workload = 0.0;
  int assigned_bag = 0;
};

std::vector<SequenceAssignment> assign_to_bags(std::vector<SequenceWorkload> workloads,
                                               const std::vector<ComputeBag>& bags);
std::vector<std::int64_t> chunk_lengths(std::int64_t total_len, int parts);

struct ChunkAssignment {
  std::uint64_t sample_id = 0;
  int chunk_index = 0;
  std::int64_t start = 0;
  std::int64_t end = 0;
  int source_rank = 0;
  int target_rank = 0;
  bool operator==(const ChunkAssignment&) const = default;
};

struct SequenceInfo {
  std::uint64_t sample_id = 0;
  std::int64_t length = 0;
};

struct Segment {
  std::uint64_t sample_id = 0;
  std::int64_t first_pos = 0;
  std::int64_t length = 0;
  bool operator==(const Segment&) const = default;
};

struct RoutingPlan {
  int world_size = 0;
  std::vector<ChunkAssignment> chunks;
  std::vector<std::vector<int>> send;
  std::vector<std::vector<int>> recv;
  std::vector<std::vector<Segment>> origin;
  std::vector<std::vector<Segment>> target;
  bool operator==(const RoutingPlan&) const = default;
};

struct BalanceReport {
  std::vector<double> per_gpu_workload;
  std::vector<double> per_bag_occupancy;
  int capacity_violations = 0;
  double total_workload = 0.0;
  double wir = 1.0;
};

struct PlanResult {
  RoutingPlan plan;
  BalanceReport report;
};

PlanResult plan_routing(const std::vector<std::vector<SequenceInfo>>& per_rank_seqs, const WorkloadModel& model,
                        const WorldLayout& layout);
RoutingPlan identity_plan(const std::vector<std::vector<SequenceInfo>>& per_rank_seqs);
RoutingPlan reverse_plan(const RoutingPlan& plan);

// Plan wire format (balancer.hpp:105-109, balancer.cpp:289-352): byte-identical
// to the reference's nlohmann::json output; plan_from_json rebuilds the
// manifests and target layout from chunks + origins.
std::string plan_to_json(const RoutingPlan& plan, const BalanceReport& report);
PlanResult plan_from_json(const std::string& text);

// ---------------------------------------------------------------- metrics
double workload_imbalance_ratio(const std::vector<double>& per_gpu_workloads);  // metrics.hpp:29

// --------------------------------------------------------------- data sim
// data_sim.hpp:11-102.  Grammar and presets parse on the host with the
// reference's messages; next_batch runs the device generator
// (sb_schedule_generate) and downloads the rank's samples.
inline constexpr int kSpatialStride = 16;
inline constexpr int kTemporalNum = 5;
inline constexpr int kTemporalDen = 17;
inline constexpr int kMaxTextTokens = 392;
inline constexpr double kAspectMultMin = 0.96;
inline constexpr double kAspectMultMax = 1.04;

struct StreamSpec {
  int gpus = 1;
  int batch_per_gpu = 1;
  int resolution = 256;
  int frames = 1;
  bool smooth = false;
  bool operator==(const StreamSpec&) const = default;
};

StreamSpec parse_data_code(std::string_view code);  // throws ParseError
std::string format_data_code(const StreamSpec& spec);

struct ShardingGroupConfig {
  std::vector<StreamSpec> streams;
  int group_size = 0;
  void validate() const;  // throws ConfigError
};

ShardingGroupConfig parse_scenario(std::istream& in);
ShardingGroupConfig parse_scenario_file(const std::string& path);
ShardingGroupConfig preset_lowres_image();
ShardingGroupConfig preset_mixed_image();
ShardingGroupConfig preset_joint_image_video();
ShardingGroupConfig scenario_preset(std::string_view name);
std::vector<std::string> scenario_preset_names();

struct SampleMeta {  // data_sim.hpp:61-68 (the record make_world consumes)
  std::uint64_t sample_id = 0;
  std::int64_t text_len = 0;
  std::int64_t visual_len = 1;
  int origin_rank = 0;
  std::int64_t total_len() const { return text_len + visual_len; }
};

std::int64_t latent_frames(const StreamSpec& spec);
std::int64_t visual_tokens(const StreamSpec& spec, double aspect_multiplier);
int stream_of_rank(const ShardingGroupConfig& config, int group_rank);
double aspect_multiplier(std::uint64_t seed, std::int64_t step, int stream_index);
std::vector<SampleMeta> next_batch(const ShardingGroupConfig& config, int rank, std::int64_t step,
                                   std::uint64_t seed);
SampleMeta dummy_sample(int rank, std::int64_t step);
std::uint64_t make_sample_id(std::int64_t step, int rank, int index);

// ---------------------------------------------------- uniform (T5) balancer
// balancer.hpp:122-144; planned on the device (sb_uniform_plan).
struct UniformMove {
  int src_rank = 0;
  int dst_rank = 0;
  std::int64_t count = 0;
  bool operator==(const UniformMove&) const = default;
};

struct UniformPlan {
  std::vector<std::int64_t> final_counts;
  std::vector<UniformMove> moves;
  std::int64_t total_moved = 0;
};

UniformPlan balance_uniform_items(const std::vector<std::int64_t>& counts);
UniformPlan reverse_uniform_plan(const UniformPlan& plan, const std::vector<std::int64_t>& original_counts);

// --------------------------------------------------------------- exchange
// exchange.hpp:14-114.
enum class Exec { Serial, Parallel };
enum class LayoutMode { ChunkFullHeads, FullSeqPartialHeads };

struct RankBuffer {
  int rank = 0;
  LayoutMode mode = LayoutMode::ChunkFullHeads;
  int head_lo = 0;
  int head_hi = 0;
  int width = 0;
  std::vector<std::uint64_t> sample_ids;
  std::vector<std::int64_t> positions;
  std::vector<double> payload;
  std::vector<Segment> segments;
  std::int64_t num_rows() const { return static_cast<std::int64_t>(sample_ids.size()); }
};

struct World {
  int payload_width = 0;
  int n_heads = 0;
  std::vector<RankBuffer> ranks;
};

double payload_value(std::uint64_t sample_id, std::int64_t position, int col);
double block_perturbation(std::uint64_t sample_id, std::int64_t position);
World make_world(const std::vector<std::vector<SampleMeta>>& per_rank_samples, int payload_width, int n_heads);
std::vector<std::vector<SequenceInfo>> gather_sequence_info(
    const std::vector<std::vector<SampleMeta>>& per_rank_samples);

// Exec is accepted for signature compatibility.  Both values run the same
// device copy engine: destinations are disjoint, so the result equals the
// reference's serial kernel bit for bit (exchange_kernels.cpp:1-6).
World route(const World& world, const RoutingPlan& plan, Exec exec = Exec::Parallel);
World reverse_route(const World& world, const RoutingPlan& plan, Exec exec = Exec::Parallel);
std::vector<std::int64_t> pre_attn(World& world, const ComputeBag& bag, Exec exec = Exec::Parallel);
void post_attn(World& world, const ComputeBag& bag, Exec exec = Exec::Parallel);

struct BlockMove {
  int src_rank = 0;
  std::int64_t src_row = 0;
  int src_col = 0;
  int dst_rank = 0;
  std::int64_t dst_row = 0;
  int dst_col = 0;
  std::int64_t n_rows = 0;
  int n_cols = 0;
  bool copy_meta = true;
};

void apply_block_moves_serial(const World& src, const std::vector<BlockMove>& moves, World& dst);
void apply_block_moves_parallel(const World& src, const std::vector<BlockMove>& moves, World& dst);
void apply_block_moves(const World& src, const std::vector<BlockMove>& moves, World& dst, Exec exec);

std::uint64_t content_checksum(const World& world);
bool worlds_bitwise_equal(const World& a, const World& b);

}  // namespace seqbal
