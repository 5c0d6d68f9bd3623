// API declarations derived from the `shardplan` reference headers
// (proj/include/shardplan/*.hpp), Copyright 2026 The Shardplan Authors,
// Apache License 2.0; see NOTICE.
//
// amsp/plan.hpp — the planner-side API of the AMSP model-state pipeline.
//
// Drop-in for the reference `shardplan` library (arXiv 2311.00257 artifact,
// /root/reference/proj/include/shardplan/*.hpp): same namespace, same value
// types, same free functions, same exceptions, so code written against the
// reference headers compiles unchanged against include/shardplan/*.hpp (which
// forward here) and links against libamsp.so instead. Results are bit-exact
// with the reference (tests/test_plan_golden.py diffs every entry point
// against golden output of the compiled reference).
//
// Everything here is host-side, pure and thread-safe. The B200 data plane
// that *executes* the plans chosen here lives behind include/amsp_c.h.
#pragma once

#include <compare>
#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace shardplan {

// ============================================================== errors
// Reference: domain.hpp:26-35, planner.hpp:44-52.

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};

/// A preset (or one of its meshes) cannot be placed on the cluster.
class InfeasibleError : public Error {
 public:
  explicit InfeasibleError(const std::string& what) : Error(what) {}
};

// ============================================================== domain
// Reference: domain.hpp:39-147, domain.cpp.

/// A group of GPUs laid out as `per_node` GPUs on each of `nodes` nodes
/// (the paper's p^0 x p^1).
struct DeviceMesh {
  int per_node = 1;
  int nodes = 1;

  constexpr int size() const { return per_node * nodes; }
  constexpr bool operator==(const DeviceMesh&) const = default;
  constexpr auto operator<=>(const DeviceMesh&) const = default;
};

std::string to_string(const DeviceMesh& m);

/// Leaf-spine fabric description (only used by placement).
struct Topology {
  int leaf_count = 1;
  int nodes_per_leaf = 1;
  double inter_leaf_penalty = 1.0;
};

struct ClusterSpec {
  int gpus_per_node = 8;                  // R
  int node_count = 1;                     // N
  std::uint64_t gpu_memory_capacity = 0;  // bytes per GPU
  DeviceMesh dp_mesh;                     // s_dp
  Topology topology;

  int gpu_count() const { return gpus_per_node * node_count; }
  void check() const;
};

/// Uniform-layer transformer: L layers of K modules with Phi_i params each;
/// total_params minus L*sum(Phi_i) is the embedding/head remainder.
struct ModelSpec {
  std::uint64_t total_params = 0;             // Phi
  int layer_count = 1;                        // L
  int modules_per_layer = 1;                  // K
  std::vector<std::uint64_t> module_params;   // Phi_i
  int hidden = 1;                             // H
  int seq_len = 1;                            // S
  int micro_batch = 1;                        // B
  int micro_batch_count = 1;                  // M
  int vocab = 1;                              // V
  int bytes_per_param = 2;
  int bytes_per_grad = 2;
  int bytes_per_os_per_param = 12;

  std::uint64_t layer_template_params() const;
  void check() const;
};

/// Sharding factors of parameters / gradients / optimizer states, each as a
/// device mesh; `secondary_params` is the ZeRO++ hierarchical copy.
struct ShardingPlan {
  DeviceMesh p;
  DeviceMesh g;
  DeviceMesh os;
  std::optional<DeviceMesh> secondary_params;

  int sp() const { return p.size(); }
  int sg() const { return g.size(); }
  int sos() const { return os.size(); }

  bool operator==(const ShardingPlan& o) const {
    return p == o.p && g == o.g && os == o.os &&
           secondary_params == o.secondary_params;
  }
  /// (s_p0, s_p1, s_g0, s_g1, s_os0, s_os1): candidate order and tie-break.
  auto lex_key() const {
    return std::tuple(p.per_node, p.nodes, g.per_node, g.nodes, os.per_node,
                      os.nodes);
  }
};

std::string to_string(const ShardingPlan& plan);

struct Violation {
  std::string constraint;
  std::string detail;
};

struct ValidationResult {
  std::vector<Violation> violations;
  bool ok() const { return violations.empty(); }
};

/// Dependency chain R >= s_dp >= s_os >= s_g >= s_p >= 1 per axis, the
/// divisibility and nesting rules, the fewer-nodes rule and s_g in
/// {s_p, s_os}. Every violation is listed.
ValidationResult validate_plan(const ShardingPlan& plan,
                               const ClusterSpec& cluster);

const std::vector<std::string>& preset_names();

/// Table III strategies instantiated on the cluster's DP mesh.
ShardingPlan preset(const std::string& name, const ClusterSpec& cluster);

// ========================================================== comm model
// Reference: comm_model.hpp:25-109, comm_model.cpp.

enum class CollectiveKind { AllGather, ReduceScatter, AllReduce, Broadcast };

const char* to_string(CollectiveKind kind);
CollectiveKind collective_from_string(const std::string& name);

struct AlphaBetaParams {
  double alpha = 0.0;
  double link_bandwidth = 1;
};

/// Ring alpha-beta time; AllReduce costs two passes.
double ring_time(CollectiveKind kind, double size_bytes, int participants,
                 const AlphaBetaParams& ab);

/// Profiled effective bandwidth w(op, size, mesh); t = size / w.
class BandwidthProfile {
 public:
  struct Point {
    std::uint64_t size = 0;
    double bandwidth = 0.0;
  };
  using Key = std::tuple<CollectiveKind, int, int>;

  void add_series(CollectiveKind kind, DeviceMesh mesh,
                  std::vector<Point> points);
  bool has_series(CollectiveKind kind, DeviceMesh mesh) const;
  bool empty() const { return table_.empty(); }

  double effective_bandwidth(CollectiveKind kind, std::uint64_t size_bytes,
                             DeviceMesh mesh) const;
  double collective_time(CollectiveKind kind, std::uint64_t size_bytes,
                         DeviceMesh mesh) const;

  const std::map<Key, std::vector<Point>>& series() const { return table_; }

 private:
  const std::vector<Point>& lookup(CollectiveKind kind, DeviceMesh mesh) const;
  std::map<Key, std::vector<Point>> table_;
};

BandwidthProfile synthetic_profile(const AlphaBetaParams& ab_intra,
                                   const AlphaBetaParams& ab_inter,
                                   const std::vector<DeviceMesh>& meshes,
                                   const std::vector<std::uint64_t>& sizes);

BandwidthProfile profile_from_csv(const std::string& csv_text);
BandwidthProfile load_profile_csv(const std::string& path);
std::string profile_to_canonical_json(const BandwidthProfile& profile);
BandwidthProfile profile_from_json(const std::string& json_text);
BandwidthProfile load_profile_json(const std::string& path);
BandwidthProfile load_profile(const std::string& path);

// ========================================================== cost model
// Reference: cost_model.hpp:24-131, cost_model.cpp.

enum class ActivationMode { None, FullRecompute };

struct CostConfig {
  std::uint64_t bucket_size = std::uint64_t{1} << 27;  // U
  ActivationMode activation_mode = ActivationMode::None;
  double activation_coeff_full = 34.0;
  double activation_coeff_recompute = 2.0;
  int tmp_in_flight_buckets = 2;
  bool tmp_include_gather_buffer = true;
  bool exact_residual_buckets = false;
  double flops_coeff_param = 6.0;
  double flops_coeff_attn = 12.0;
};

struct TimeBreakdown {
  double t_p = 0.0;
  double t_g = 0.0;
  double t_os_allreduce = 0.0;
  double t_os_broadcast = 0.0;
  double total = 0.0;
};

struct MemoryBreakdown {
  double d_params = 0.0;
  double d_grads = 0.0;
  double d_os = 0.0;
  double d_modelstate = 0.0;
  double d_activation = 0.0;
  double d_tmp = 0.0;
  double d_total = 0.0;
};

struct TensorPartition {
  std::vector<int> assignment;
  std::vector<std::uint64_t> shard_sizes;
};

double time_params_sharding(const ModelSpec& model, const ShardingPlan& plan,
                            const BandwidthProfile& profile);
std::uint64_t grad_bucket_count(const ModelSpec& model,
                                const ShardingPlan& plan,
                                const CostConfig& cfg);
double time_os_allreduce(const ModelSpec& model, const ClusterSpec& cluster,
                         const ShardingPlan& plan,
                         const BandwidthProfile& profile,
                         const CostConfig& cfg);
double time_os_broadcast(const ModelSpec& model, const ShardingPlan& plan,
                         const BandwidthProfile& profile);
double time_grads_sharding(const ModelSpec& model, const ShardingPlan& plan,
                           const BandwidthProfile& profile,
                           const CostConfig& cfg);
TimeBreakdown total_comm_time(const ModelSpec& model,
                              const ClusterSpec& cluster,
                              const ShardingPlan& plan,
                              const BandwidthProfile& profile,
                              const CostConfig& cfg);
MemoryBreakdown memory_breakdown(const ModelSpec& model,
                                 const ShardingPlan& plan,
                                 const CostConfig& cfg);
double flops_per_step(const ModelSpec& model, const CostConfig& cfg);
double mfu(const ModelSpec& model, double step_time_s,
           double peak_flops_per_gpu, int gpu_count, const CostConfig& cfg);

/// LPT greedy inter-tensor layout of the optimizer-state shards.
TensorPartition partition_tensors_greedy(
    const std::vector<std::uint64_t>& tensor_sizes, int shard_count);

// ============================================================= planner
// Reference: planner.hpp:25-104, planner.cpp.

struct PlanResult {
  ShardingPlan plan;
  TimeBreakdown time;
  MemoryBreakdown memory;
  bool feasible = false;
  int rank = -1;
};

struct SearchReport {
  PlanResult best;
  std::uint64_t candidates_evaluated = 0;
  std::uint64_t candidates_filtered = 0;
  std::optional<std::vector<PlanResult>> all_results;
};

/// Raised when no candidate fits in memory; carries the leanest candidate.
class NoFeasiblePlanError : public Error {
 public:
  NoFeasiblePlanError(const std::string& what, PlanResult closest)
      : Error(what), closest_(std::move(closest)) {}
  const PlanResult& closest() const { return closest_; }

 private:
  PlanResult closest_;
};

enum class ExecPolicy { Serial, Parallel };

struct SolveOptions {
  bool keep_all_results = false;
  ExecPolicy policy = ExecPolicy::Parallel;
};

std::vector<ShardingPlan> enumerate_candidates(const ClusterSpec& cluster);
PlanResult evaluate_plan(const ModelSpec& model, const ClusterSpec& cluster,
                         const ShardingPlan& plan,
                         const BandwidthProfile& profile,
                         const CostConfig& cfg);
SearchReport solve(const ModelSpec& model, const ClusterSpec& cluster,
                   const BandwidthProfile& profile, const CostConfig& cfg,
                   const SolveOptions& options = {});
SearchReport brute_force_oracle(const ModelSpec& model,
                                const ClusterSpec& cluster,
                                const BandwidthProfile& profile,
                                const CostConfig& cfg,
                                std::uint64_t max_raw_tuples = 1000000);

struct PresetResult {
  std::string name;
  std::optional<PlanResult> result;
  std::string error;
};

std::vector<PresetResult> compare_presets(const ModelSpec& model,
                                          const ClusterSpec& cluster,
                                          const BandwidthProfile& profile,
                                          const CostConfig& cfg);

// ========================================================= overlap sim
// Reference: overlap_sim.hpp:24-133, overlap_sim.cpp.

enum class OverlapTier { None, AgRs, AgRsAr, AgRsArBc };

const char* to_string(OverlapTier tier);
OverlapTier tier_from_string(const std::string& name);

enum class EventKind {
  FwdCompute,
  BwdGradInput,
  BwdGradWeight,
  RecomputeFwd,
  AllGather,
  ReduceScatter,
  AllReduceBucket,
  BroadcastShard,
};

const char* to_string(EventKind kind);

struct Event {
  int id = -1;
  EventKind kind = EventKind::FwdCompute;
  int layer = -1;
  int module = -1;
  double duration = 0.0;
  std::vector<int> depends_on;
  int stream = 0;
};

struct EventGraph {
  std::vector<Event> events;
  int stream_count = 1;
};

enum class ComputeTimeSource { Flops, Table };

struct SimConfig {
  OverlapTier overlap_tier = OverlapTier::AgRsArBc;
  bool recompute = false;
  int comm_streams = 2;
  ComputeTimeSource compute_time_source = ComputeTimeSource::Flops;
  double peak_flops_per_gpu = 312e12;
  double compute_efficiency = 0.6;
  std::vector<double> fwd_times;
  std::vector<double> bwd_grad_weight_times;
  std::vector<double> bwd_grad_input_times;
  double head_fwd_time = 0.0;
  double head_bwd_time = 0.0;
};

struct ScheduledEvent {
  int event_id = -1;
  double start = 0.0;
  double end = 0.0;
};

struct Timeline {
  std::vector<Event> events;
  std::vector<std::vector<ScheduledEvent>> streams;
  double step_time = 0.0;
  std::vector<double> busy;
  std::vector<double> idle;
};

struct IdleInterval {
  double start = 0.0;
  double end = 0.0;
};

struct BubbleReport {
  double compute_idle_total = 0.0;
  std::vector<IdleInterval> compute_intervals;
  std::vector<double> stream_idle;
};

/// One step of one rank as an event graph on 1 compute + 1..2 comm streams.
EventGraph build_schedule(const ModelSpec& model, const ClusterSpec& cluster,
                          const ShardingPlan& plan,
                          const BandwidthProfile& profile,
                          const CostConfig& cfg, const SimConfig& sim);
Timeline simulate_step(const EventGraph& graph);
BubbleReport bubble_report(const Timeline& timeline);
std::string render_trace(const Timeline& timeline);
void export_trace(const Timeline& timeline, const std::string& path);

// =========================================================== placement
// Reference: placement.hpp:23-54, placement.cpp.

struct GroupAssignment {
  std::vector<int> group_of;
  std::vector<int> leaf_of;
  int group_size = 1;
  int cross_leaf_groups = 0;
};

GroupAssignment assign_nodes(const Topology& topology,
                             const ClusterSpec& cluster,
                             const ShardingPlan& plan);
int count_cross_leaf_groups(const std::vector<int>& group_of, int group_count,
                            const std::vector<int>& leaf_of);
double placed_collective_time(const Topology& topology,
                              const GroupAssignment& assignment,
                              const BandwidthProfile& profile,
                              CollectiveKind kind, std::uint64_t size_bytes,
                              DeviceMesh mesh);

}  // namespace shardplan
