// B200 roofline of one AMSP step and the roofline-ordered solver (see
// roofline.h). Host only.
#include "roofline.h"

#include <algorithm>
#include <numeric>
#include <string>

#include "kernels.h"
#include "layout.h"

namespace amsp {

using shardplan::DeviceMesh;
using shardplan::Error;
using shardplan::ShardingPlan;

StepTraffic step_traffic(const std::vector<std::uint64_t>& tensor_sizes, const ShardingPlan& plan,
                         DeviceMesh dp, int rank, int layout, int gathers, double hbm_bw,
                         double nvlink_bw) {
  const int W = dp.size();
  if (rank < 0 || rank >= W) throw Error("roofline: rank out of range");
  if (hbm_bw <= 0.0 || nvlink_bw <= 0.0) throw Error("roofline: bandwidths must be > 0");
  if (gathers < 0) throw Error("roofline: gathers must be >= 0");
  const int sp = plan.sp(), sos = plan.sos();
  if (sp < 1 || sos < sp || sos % sp != 0 || W % sos != 0)
    throw Error("roofline: plan " + shardplan::to_string(plan) + " does not nest in dp " +
                shardplan::to_string(dp));
  for (auto t : tensor_sizes)
    if (t == 0 || t % static_cast<std::uint64_t>(sp) != 0)
      throw Error("roofline: every tensor must be a positive multiple of s_p");
  // The engine's groups and shard (engine.cpp create_engine).
  const MeshGroup pg = mesh_group(dp, plan.p, rank);
  const MeshGroup og = mesh_group(dp, plan.os, rank);
  int k = 0, my_k = 0;
  for (int m : og.members)
    if (mesh_group(dp, plan.p, m).position == pg.position) {
      if (m == rank) my_k = k;
      ++k;
    }
  const ShardLayout L = pshard_layout(tensor_sizes, sp, pg.position, k, my_k, layout);
  const std::uint64_t phi =
      std::accumulate(tensor_sizes.begin(), tensor_sizes.end(), std::uint64_t{0});
  const std::uint64_t R = static_cast<std::uint64_t>(W / sos), usp = static_cast<std::uint64_t>(sp);
  StepTraffic s;
  s.owned = L.owned;
  s.hbm = 24 * s.owned + 2 * phi * R + 2 * (phi / usp);
  s.nvl_in = 2 * s.owned * static_cast<std::uint64_t>(W - 1) + 2 * (phi / usp - s.owned);
  s.nvl_out = 2 * (R * phi - s.owned) + 2 * s.owned * static_cast<std::uint64_t>(k - 1);
  if (sp > 1) {
    const std::uint64_t g = static_cast<std::uint64_t>(gathers);
    // ZeRO++: the backward pass (the second of the two) gathers over the
    // secondary group, and the forward pass refreshes the Phi/s2 slice
    const std::uint64_t u2 =
        plan.secondary_params ? static_cast<std::uint64_t>(plan.secondary_params->size()) : 0;
    const std::uint64_t gs = (u2 > 1 && g >= 2) ? 1 : 0;
    s.hbm += g * 4 * phi + (gs ? 4 * (phi / u2) : 0);
    const std::uint64_t nvl = (g - gs) * 2 * phi * (usp - 1) / usp +
                              (gs ? 2 * phi * (u2 - 1) / u2 : 0);
    s.nvl_in += nvl;
    s.nvl_out += nvl;
  }
  if (W == 1) s.nvl_in = s.nvl_out = 0;
  s.t_hbm = static_cast<double>(s.hbm) / hbm_bw;
  s.t_nvlink = static_cast<double>(std::max(s.nvl_in, s.nvl_out)) / nvlink_bw;
  s.t_step = std::max(s.t_hbm, s.t_nvlink);
  return s;
}

StepTraffic step_traffic_max(const std::vector<std::uint64_t>& tensor_sizes,
                             const ShardingPlan& plan, DeviceMesh dp, int layout, int gathers,
                             double hbm_bw, double nvlink_bw, int* slowest_rank) {
  StepTraffic worst;
  int who = 0;
  for (int r = 0; r < dp.size(); ++r) {
    const StepTraffic s =
        step_traffic(tensor_sizes, plan, dp, r, layout, gathers, hbm_bw, nvlink_bw);
    if (r == 0 || s.t_step > worst.t_step) {
      worst = s;
      who = r;
    }
  }
  if (slowest_rank) *slowest_rank = who;
  return worst;
}

std::vector<std::uint64_t> model_tensors(const shardplan::ModelSpec& model) {
  model.check();
  const std::uint64_t layers = static_cast<std::uint64_t>(model.layer_count);
  const std::uint64_t body = layers * model.layer_template_params();
  const std::uint64_t head = model.total_params - body;
  const std::uint64_t vh =
      static_cast<std::uint64_t>(model.vocab) * static_cast<std::uint64_t>(model.hidden);
  std::vector<std::uint64_t> t;
  const bool llama = head == 2 * vh + static_cast<std::uint64_t>(model.hidden);
  if (llama) t.push_back(vh);
  else if (head > 0) t.push_back(head);
  for (int l = 0; l < model.layer_count; ++l)
    t.insert(t.end(), model.module_params.begin(), model.module_params.end());
  if (llama) {
    t.push_back(static_cast<std::uint64_t>(model.hidden));
    t.push_back(vh);
  }
  return t;
}

std::vector<RooflineResult> solve_roofline(const shardplan::ModelSpec& model,
                                           const shardplan::ClusterSpec& cluster,
                                           const shardplan::BandwidthProfile& profile,
                                           const shardplan::CostConfig& cfg, double hbm_bw,
                                           double nvlink_bw, int layout) {
  const std::vector<std::uint64_t> tensors = model_tensors(model);
  const DeviceMesh dp = cluster.dp_mesh;
  if (dp.size() > kMaxRanks)
    throw Error("roofline: dp mesh " + shardplan::to_string(dp) +
                " outside the 1..8 GPU NVSwitch domain of one node");
  std::vector<RooflineResult> out;
  shardplan::PlanResult leanest;
  bool any = false;
  // The reference's candidates, plus (our extension) the ZeRO++ variants of
  // every parameter-sharded one: a secondary mesh strictly inside the P mesh
  // for the backward all-gathers (domain.hpp:90-97; the engine runs them).
  std::vector<ShardingPlan> candidates;
  for (const ShardingPlan& plan : shardplan::enumerate_candidates(cluster)) {
    candidates.push_back(plan);
    if (plan.sp() == 1 || plan.secondary_params) continue;
    for (int a = 1; a <= plan.p.per_node; ++a)
      for (int b = 1; b <= plan.p.nodes; ++b)
        if (plan.p.per_node % a == 0 && plan.p.nodes % b == 0 && a * b > 1 &&
            a * b < plan.sp()) {
          ShardingPlan z = plan;
          z.secondary_params = DeviceMesh{a, b};
          candidates.push_back(z);
        }
  }
  for (const ShardingPlan& plan : candidates) {
    RooflineResult r;
    r.result = shardplan::evaluate_plan(model, cluster, plan, profile, cfg);
    if (!any || r.result.memory.d_total < leanest.memory.d_total) leanest = r.result;
    any = true;
    r.runnable = std::all_of(tensors.begin(), tensors.end(), [&](std::uint64_t t) {
      return t % static_cast<std::uint64_t>(plan.sp()) == 0 &&
             (!plan.secondary_params ||
              t % static_cast<std::uint64_t>(plan.secondary_params->size()) == 0);
    });
    if (!r.result.feasible || !r.runnable) continue;
    r.step = step_traffic_max(tensors, plan, dp, layout, 2, hbm_bw, nvlink_bw, nullptr);
    out.push_back(r);
  }
  if (out.empty())
    throw shardplan::NoFeasiblePlanError(
        "no feasible plan the engine can run: minimal-memory candidate " +
            (any ? shardplan::to_string(leanest.plan) : std::string("<none>")),
        leanest);
  std::stable_sort(out.begin(), out.end(), [](const RooflineResult& a, const RooflineResult& b) {
    if (a.step.t_step != b.step.t_step) return a.step.t_step < b.step.t_step;
    if (a.result.time.total != b.result.time.total)
      return a.result.time.total < b.result.time.total;
    return a.result.plan.lex_key() < b.result.plan.lex_key();
  });
  for (std::size_t i = 0; i < out.size(); ++i) out[i].result.rank = static_cast<int>(i);
  return out;
}

}  // namespace amsp
