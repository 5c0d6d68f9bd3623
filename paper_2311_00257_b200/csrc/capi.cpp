// C-ABI of the planner half (include/amsp_c.h): POD <-> shardplan types and
// exception -> status translation. Host only; loads without a GPU.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "amsp/plan.hpp"
#include "amsp_c.h"
#include "engine/layout.h"
#include "engine/roofline.h"
#include "convert.h"
#include "status.h"

using namespace shardplan;

namespace amsp {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

}  // namespace amsp

namespace {

using namespace amsp::conv;

amsp_time_t time_out(const TimeBreakdown& t) {
  return {t.t_p, t.t_g, t.t_os_allreduce, t.t_os_broadcast, t.total};
}

amsp_memory_t mem_out(const MemoryBreakdown& m) {
  return {m.d_params, m.d_grads, m.d_os, m.d_modelstate, m.d_activation, m.d_tmp, m.d_total};
}

amsp_step_roofline_t step_out(const amsp::StepTraffic& t) {
  return {t.owned, t.hbm, t.nvl_in, t.nvl_out, t.t_hbm, t.t_nvlink, t.t_step};
}

amsp_plan_result_t result_out(const PlanResult& r) {
  amsp_plan_result_t o{};
  o.plan = plan_out(r.plan);
  o.time = time_out(r.time);
  o.memory = mem_out(r.memory);
  o.feasible = r.feasible;
  o.rank = r.rank;
  return o;
}

CollectiveKind kind_in(int k) {
  if (k < 0 || k > 3) throw Error("unknown collective kind " + std::to_string(k));
  return static_cast<CollectiveKind>(k);
}

void write_text(const std::string& s, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = s.size();
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
}

}  // namespace

extern "C" {

int amsp_abi_version(void) { return AMSP_ABI_VERSION; }

const char* amsp_last_error(void) { return amsp::g_last_error.c_str(); }

void amsp_cost_config_default(amsp_cost_config_t* c) {
  if (!c) return;
  const CostConfig d;
  c->bucket_size = d.bucket_size;
  c->activation_mode = 0;
  c->activation_coeff_full = d.activation_coeff_full;
  c->activation_coeff_recompute = d.activation_coeff_recompute;
  c->tmp_in_flight_buckets = d.tmp_in_flight_buckets;
  c->tmp_include_gather_buffer = d.tmp_include_gather_buffer;
  c->exact_residual_buckets = d.exact_residual_buckets;
  c->flops_coeff_param = d.flops_coeff_param;
  c->flops_coeff_attn = d.flops_coeff_attn;
}

void amsp_sim_config_default(amsp_sim_config_t* c) {
  if (!c) return;
  const SimConfig d;
  std::memset(c, 0, sizeof(*c));
  c->overlap_tier = static_cast<int>(d.overlap_tier);
  c->recompute = d.recompute;
  c->comm_streams = d.comm_streams;
  c->compute_time_source = 0;
  c->peak_flops_per_gpu = d.peak_flops_per_gpu;
  c->compute_efficiency = d.compute_efficiency;
}

int amsp_profile_synthetic(double ai, double bi, double ao, double bo,
                           const amsp_mesh_t* meshes, int n_meshes, const uint64_t* sizes,
                           int n_sizes, amsp_profile_t** out) {
  return amsp::guarded([&] {
    if (!out || n_meshes < 0 || n_sizes < 0) throw Error("null argument");
    std::vector<DeviceMesh> ms;
    for (int i = 0; i < n_meshes; ++i) ms.push_back(mesh_in(meshes[i]));
    std::vector<std::uint64_t> sz(sizes, sizes + n_sizes);
    auto p = new amsp_profile{synthetic_profile({ai, bi}, {ao, bo}, ms, sz)};
    *out = p;
  });
}

int amsp_profile_from_csv(const char* text, amsp_profile_t** out) {
  return amsp::guarded([&] {
    if (!text || !out) throw Error("null argument");
    *out = new amsp_profile{profile_from_csv(text)};
  });
}

int amsp_profile_from_json(const char* text, amsp_profile_t** out) {
  return amsp::guarded([&] {
    if (!text || !out) throw Error("null argument");
    *out = new amsp_profile{profile_from_json(text)};
  });
}

int amsp_profile_load(const char* path, amsp_profile_t** out) {
  return amsp::guarded([&] {
    if (!path || !out) throw Error("null argument");
    *out = new amsp_profile{load_profile(path)};
  });
}

int amsp_profile_to_json(const amsp_profile_t* p, char* buf, size_t cap, size_t* needed) {
  return amsp::guarded([&] {
    if (!p) throw Error("null profile");
    write_text(profile_to_canonical_json(p->p), buf, cap, needed);
  });
}

int amsp_collective_time(const amsp_profile_t* p, int kind, uint64_t size_bytes,
                         amsp_mesh_t mesh, double* seconds) {
  return amsp::guarded([&] {
    if (!p || !seconds) throw Error("null argument");
    *seconds = p->p.collective_time(kind_in(kind), size_bytes, mesh_in(mesh));
  });
}

void amsp_profile_free(amsp_profile_t* p) { delete p; }

int amsp_ring_time(int kind, double size_bytes, int participants, double alpha,
                   double link_bandwidth, double* seconds) {
  return amsp::guarded([&] {
    if (!seconds) throw Error("null argument");
    *seconds = ring_time(kind_in(kind), size_bytes, participants, {alpha, link_bandwidth});
  });
}

int amsp_validate_plan(const amsp_plan_t* plan, const amsp_cluster_t* cluster,
                       int* n_violations, char* buf, size_t cap) {
  return amsp::guarded([&] {
    const ValidationResult v = validate_plan(plan_in(plan), cluster_in(cluster));
    if (n_violations) *n_violations = static_cast<int>(v.violations.size());
    std::string text;
    for (const auto& x : v.violations) text += x.constraint + ":" + x.detail + "\n";
    write_text(text, buf, cap, nullptr);
  });
}

int amsp_preset(const char* name, const amsp_cluster_t* cluster, amsp_plan_t* out) {
  return amsp::guarded([&] {
    if (!name || !out) throw Error("null argument");
    *out = plan_out(preset(name, cluster_in(cluster)));
  });
}

int amsp_memory_breakdown(const amsp_model_t* model, const amsp_plan_t* plan,
                          const amsp_cost_config_t* cfg, amsp_memory_t* out) {
  return amsp::guarded([&] {
    if (!out) throw Error("null argument");
    *out = mem_out(memory_breakdown(model_in(model), plan_in(plan), cost_in(cfg)));
  });
}

int amsp_total_comm_time(const amsp_model_t* model, const amsp_cluster_t* cluster,
                         const amsp_plan_t* plan, const amsp_profile_t* profile,
                         const amsp_cost_config_t* cfg, amsp_time_t* out) {
  return amsp::guarded([&] {
    if (!out || !profile) throw Error("null argument");
    *out = time_out(total_comm_time(model_in(model), cluster_in(cluster), plan_in(plan),
                                    profile->p, cost_in(cfg)));
  });
}

int amsp_grad_bucket_count(const amsp_model_t* model, const amsp_plan_t* plan,
                           const amsp_cost_config_t* cfg, uint64_t* out) {
  return amsp::guarded([&] {
    if (!out) throw Error("null argument");
    *out = grad_bucket_count(model_in(model), plan_in(plan), cost_in(cfg));
  });
}

int amsp_partition_greedy(const uint64_t* sizes, int n, int shard_count, int* assignment,
                          uint64_t* shard_sizes) {
  return amsp::guarded([&] {
    if (n < 0 || (n > 0 && !sizes)) throw Error("null argument");
    const TensorPartition p =
        partition_tensors_greedy(std::vector<std::uint64_t>(sizes, sizes + n), shard_count);
    if (assignment) std::copy(p.assignment.begin(), p.assignment.end(), assignment);
    if (shard_sizes) std::copy(p.shard_sizes.begin(), p.shard_sizes.end(), shard_sizes);
  });
}

int amsp_enumerate_candidates(const amsp_cluster_t* cluster, amsp_plan_t* plans, int cap,
                              int* n) {
  return amsp::guarded([&] {
    const auto v = enumerate_candidates(cluster_in(cluster));
    if (n) *n = static_cast<int>(v.size());
    for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i) plans[i] = plan_out(v[i]);
  });
}

int amsp_solve(const amsp_model_t* model, const amsp_cluster_t* cluster,
               const amsp_profile_t* profile, const amsp_cost_config_t* cfg,
               amsp_plan_result_t* best, uint64_t* evaluated, uint64_t* filtered,
               amsp_plan_result_t* all, int cap, int* n_all) {
  return amsp::guarded([&] {
    if (!profile) throw Error("null profile");
    SolveOptions o;
    o.keep_all_results = all != nullptr || n_all != nullptr;
    try {
      const SearchReport r = solve(model_in(model), cluster_in(cluster), profile->p,
                                   cost_in(cfg), o);
      if (best) *best = result_out(r.best);
      if (evaluated) *evaluated = r.candidates_evaluated;
      if (filtered) *filtered = r.candidates_filtered;
      if (r.all_results) {
        if (n_all) *n_all = static_cast<int>(r.all_results->size());
        for (int i = 0; all && i < cap && i < static_cast<int>(r.all_results->size()); ++i)
          all[i] = result_out((*r.all_results)[i]);
      }
    } catch (const NoFeasiblePlanError& e) {
      if (best) *best = result_out(e.closest());
      throw;
    }
  });
}

int amsp_simulate(const amsp_model_t* model, const amsp_cluster_t* cluster,
                  const amsp_plan_t* plan, const amsp_profile_t* profile,
                  const amsp_cost_config_t* cfg, const amsp_sim_config_t* sim,
                  double* step_time, double* compute_idle, int* n_events, char* trace,
                  size_t trace_cap, size_t* trace_needed) {
  return amsp::guarded([&] {
    if (!profile || !model) throw Error("null argument");
    const ModelSpec m = model_in(model);
    const EventGraph g = build_schedule(m, cluster_in(cluster), plan_in(plan), profile->p,
                                        cost_in(cfg), sim_in(sim, m.modules_per_layer));
    const Timeline t = simulate_step(g);
    if (step_time) *step_time = t.step_time;
    if (compute_idle) *compute_idle = bubble_report(t).compute_idle_total;
    if (n_events) *n_events = static_cast<int>(g.events.size());
    if (trace || trace_needed) write_text(render_trace(t), trace, trace_cap, trace_needed);
  });
}

int amsp_layout_segments(const uint64_t* tensor_sizes, int n_tensors, int shard_count,
                         int shard, int layout, uint64_t* flat, uint64_t* os, uint64_t* len,
                         int cap, int* n_segments, uint64_t* owned) {
  return amsp::guarded([&] {
    if (n_tensors < 0 || (n_tensors > 0 && !tensor_sizes)) throw Error("null argument");
    const amsp::ShardLayout L = amsp::shard_layout(
        std::vector<std::uint64_t>(tensor_sizes, tensor_sizes + n_tensors), shard_count,
        shard, layout);
    if (n_segments) *n_segments = static_cast<int>(L.segs.size());
    if (owned) *owned = L.owned;
    for (int i = 0; i < cap && i < static_cast<int>(L.segs.size()); ++i) {
      if (flat) flat[i] = L.segs[i].flat;
      if (os) os[i] = L.segs[i].os;
      if (len) len[i] = L.segs[i].len;
    }
  });
}

int amsp_pshard_layout(const uint64_t* tensor_sizes, int n_tensors, int sp, int p_pos, int k,
                       int os_pos, int layout, uint64_t* flat, uint64_t* os, uint64_t* dst,
                       uint64_t* len, int cap, int* n_segments, uint64_t* owned) {
  return amsp::guarded([&] {
    if (n_tensors < 0 || (n_tensors > 0 && !tensor_sizes)) throw Error("null argument");
    const amsp::ShardLayout L = amsp::pshard_layout(
        std::vector<std::uint64_t>(tensor_sizes, tensor_sizes + n_tensors), sp, p_pos, k,
        os_pos, layout);
    if (n_segments) *n_segments = static_cast<int>(L.segs.size());
    if (owned) *owned = L.owned;
    for (int i = 0; i < cap && i < static_cast<int>(L.segs.size()); ++i) {
      if (flat) flat[i] = L.segs[i].flat;
      if (os) os[i] = L.segs[i].os;
      if (dst) dst[i] = L.segs[i].dst;
      if (len) len[i] = L.segs[i].len;
    }
  });
}

int amsp_step_roofline(const uint64_t* tensor_sizes, int n_tensors, const amsp_plan_t* plan,
                       amsp_mesh_t dp, int rank, int layout, int gathers, double hbm_bw,
                       double nvlink_bw, int* slowest, amsp_step_roofline_t* out) {
  return amsp::guarded([&] {
    if (n_tensors < 1 || !tensor_sizes || !plan || !out) throw Error("null argument");
    const std::vector<std::uint64_t> t(tensor_sizes, tensor_sizes + n_tensors);
    const ShardingPlan p = plan_in(plan);
    int who = rank;
    const amsp::StepTraffic s =
        rank < 0 ? amsp::step_traffic_max(t, p, mesh_in(dp), layout, gathers, hbm_bw,
                                          nvlink_bw, &who)
                 : amsp::step_traffic(t, p, mesh_in(dp), rank, layout, gathers, hbm_bw,
                                      nvlink_bw);
    if (slowest) *slowest = who;
    *out = step_out(s);
  });
}

int amsp_model_tensors(const amsp_model_t* model, uint64_t* sizes, int cap, int* n) {
  return amsp::guarded([&] {
    const std::vector<std::uint64_t> t = amsp::model_tensors(model_in(model));
    if (n) *n = static_cast<int>(t.size());
    for (int i = 0; sizes && i < cap && i < static_cast<int>(t.size()); ++i) sizes[i] = t[i];
  });
}

int amsp_solve_roofline(const amsp_model_t* model, const amsp_cluster_t* cluster,
                        const amsp_profile_t* profile, const amsp_cost_config_t* cfg,
                        double hbm_bw, double nvlink_bw, int layout, amsp_plan_result_t* best,
                        amsp_step_roofline_t* best_step, amsp_plan_result_t* all,
                        amsp_step_roofline_t* all_steps, int cap, int* n_all) {
  return amsp::guarded([&] {
    if (!profile) throw Error("null profile");
    try {
      const auto r = amsp::solve_roofline(model_in(model), cluster_in(cluster), profile->p,
                                          cost_in(cfg), hbm_bw, nvlink_bw, layout);
      if (best) *best = result_out(r.front().result);
      if (best_step) *best_step = step_out(r.front().step);
      if (n_all) *n_all = static_cast<int>(r.size());
      for (int i = 0; i < cap && i < static_cast<int>(r.size()); ++i) {
        if (all) all[i] = result_out(r[i].result);
        if (all_steps) all_steps[i] = step_out(r[i].step);
      }
    } catch (const NoFeasiblePlanError& e) {
      if (best) *best = result_out(e.closest());
      throw;
    }
  });
}

int amsp_mesh_group(amsp_mesh_t dp, amsp_mesh_t mesh, int rank, int* block, int* position,
                    int* members, int cap, int* n_members) {
  return amsp::guarded([&] {
    const amsp::MeshGroup g = amsp::mesh_group(mesh_in(dp), mesh_in(mesh), rank);
    if (block) *block = g.block;
    if (position) *position = g.position;
    if (n_members) *n_members = static_cast<int>(g.members.size());
    for (int i = 0; members && i < cap && i < static_cast<int>(g.members.size()); ++i)
      members[i] = g.members[i];
  });
}

}  // extern "C"
