// B200 roofline of one AMSP step, and a solver that ranks plans by it (host
// only; no GPU needed).
//
// The reference solver (shardplan::solve, planner.cpp:144-166) ranks plans
// by communication time alone. On B200 the step is bounded by HBM or NVLink
// bytes, and the optimizer's HBM traffic (24 B of fp32 state per owned
// param) weighs as much as the collectives. The r01 strategy sweep measured
// the reference objective's pick 12% slower than the best plan
// (profiles/r01_sweep_1b_4gpu_v2.jsonl). solve_roofline keeps the
// reference's candidate set, memory model and feasibility rule, and orders
// candidates by this step time instead (T_comm, then the plan's lex key,
// break ties). shardplan::solve stays bit-exact with the reference.
#pragma once

#include <cstdint>
#include <vector>

#include "amsp/plan.hpp"

namespace amsp {

// Algorithmic bytes one rank moves in one step of the engine (DESIGN.md §4,
// the same formulas as bench.step_bytes):
//   HBM     = 24*owned + 2*Phi*R + 2*Phi/s_p  (+ gathers * 4*Phi when s_p > 1)
//   NVL in  = 2*owned*(W-1) + 2*(Phi/s_p - owned)
//   NVL out = 2*(R*Phi - owned) + 2*owned*(k-1)
//             (+ gathers * 2*Phi*(s_p-1)/s_p per direction when s_p > 1)
// with owned from the engine's own shard layout, R = W/s_os, k = s_os/s_p.
struct StepTraffic {
  std::uint64_t owned = 0, hbm = 0, nvl_in = 0, nvl_out = 0;
  double t_hbm = 0.0, t_nvlink = 0.0, t_step = 0.0;  // seconds
};

StepTraffic step_traffic(const std::vector<std::uint64_t>& tensor_sizes,
                         const shardplan::ShardingPlan& plan, shardplan::DeviceMesh dp,
                         int rank, int layout, int gathers, double hbm_bw, double nvlink_bw);

// The slowest rank of the group (the step ends when it does).
StepTraffic step_traffic_max(const std::vector<std::uint64_t>& tensor_sizes,
                             const shardplan::ShardingPlan& plan, shardplan::DeviceMesh dp,
                             int layout, int gathers, double hbm_bw, double nvlink_bw,
                             int* slowest_rank);

// The engine's flat tensor list of a LLaMA-style ModelSpec: embed (V*H),
// L x module_params, final norm (H), lm_head (V*H) when the head parameters
// are exactly that, else one head tensor first.
std::vector<std::uint64_t> model_tensors(const shardplan::ModelSpec& model);

struct RooflineResult {
  shardplan::PlanResult result;  // reference cost and memory of the plan
  StepTraffic step;              // slowest rank
  bool runnable = false;         // the engine can run it (s_p divides every tensor)
};

// All reference candidates that fit in memory and that the engine can run,
// fastest roofline step first. Throws shardplan::NoFeasiblePlanError when
// none qualifies.
std::vector<RooflineResult> solve_roofline(const shardplan::ModelSpec& model,
                                           const shardplan::ClusterSpec& cluster,
                                           const shardplan::BandwidthProfile& profile,
                                           const shardplan::CostConfig& cfg, double hbm_bw,
                                           double nvlink_bw, int layout);

}  // namespace amsp
