// Internal POD <-> shardplan conversions shared by the C-ABI (capi.cpp)
// and the overlap scheduler (engine/sched.cpp).
#pragma once

#include <vector>

#include "amsp/plan.hpp"
#include "amsp_c.h"

struct amsp_profile {
  shardplan::BandwidthProfile p;
};

namespace amsp::conv {

using namespace shardplan;

inline DeviceMesh mesh_in(amsp_mesh_t m) { return {m.per_node, m.nodes}; }
inline amsp_mesh_t mesh_out(DeviceMesh m) { return {m.per_node, m.nodes}; }

inline ShardingPlan plan_in(const amsp_plan_t* p) {
  if (!p) throw Error("null plan");
  ShardingPlan s{mesh_in(p->p), mesh_in(p->g), mesh_in(p->os), std::nullopt};
  if (p->has_secondary) s.secondary_params = mesh_in(p->secondary);
  return s;
}

inline amsp_plan_t plan_out(const ShardingPlan& s) {
  amsp_plan_t p{};
  p.p = mesh_out(s.p);
  p.g = mesh_out(s.g);
  p.os = mesh_out(s.os);
  p.has_secondary = s.secondary_params.has_value();
  if (s.secondary_params) p.secondary = mesh_out(*s.secondary_params);
  return p;
}

inline ClusterSpec cluster_in(const amsp_cluster_t* c) {
  if (!c) throw Error("null cluster");
  ClusterSpec s;
  s.gpus_per_node = c->gpus_per_node;
  s.node_count = c->node_count;
  s.gpu_memory_capacity = c->gpu_memory_capacity;
  s.dp_mesh = mesh_in(c->dp_mesh);
  s.topology = {c->leaf_count, c->nodes_per_leaf, c->inter_leaf_penalty};
  return s;
}

inline ModelSpec model_in(const amsp_model_t* m) {
  if (!m) throw Error("null model");
  ModelSpec s;
  s.total_params = m->total_params;
  s.layer_count = m->layer_count;
  s.modules_per_layer = m->modules_per_layer;
  if (m->modules_per_layer > 0 && m->module_params)
    s.module_params.assign(m->module_params, m->module_params + m->modules_per_layer);
  s.hidden = m->hidden;
  s.seq_len = m->seq_len;
  s.micro_batch = m->micro_batch;
  s.micro_batch_count = m->micro_batch_count;
  s.vocab = m->vocab;
  s.bytes_per_param = m->bytes_per_param;
  s.bytes_per_grad = m->bytes_per_grad;
  s.bytes_per_os_per_param = m->bytes_per_os_per_param;
  return s;
}

inline CostConfig cost_in(const amsp_cost_config_t* c) {
  CostConfig s;
  if (!c) return s;
  s.bucket_size = c->bucket_size;
  s.activation_mode = c->activation_mode ? ActivationMode::FullRecompute : ActivationMode::None;
  s.activation_coeff_full = c->activation_coeff_full;
  s.activation_coeff_recompute = c->activation_coeff_recompute;
  s.tmp_in_flight_buckets = c->tmp_in_flight_buckets;
  s.tmp_include_gather_buffer = c->tmp_include_gather_buffer != 0;
  s.exact_residual_buckets = c->exact_residual_buckets != 0;
  s.flops_coeff_param = c->flops_coeff_param;
  s.flops_coeff_attn = c->flops_coeff_attn;
  return s;
}

inline SimConfig sim_in(const amsp_sim_config_t* c, int k) {
  SimConfig s;
  if (!c) return s;
  if (c->overlap_tier < 0 || c->overlap_tier > 3) throw Error("sim: bad overlap tier");
  s.overlap_tier = static_cast<OverlapTier>(c->overlap_tier);
  s.recompute = c->recompute != 0;
  s.comm_streams = c->comm_streams;
  s.compute_time_source = c->compute_time_source ? ComputeTimeSource::Table : ComputeTimeSource::Flops;
  s.peak_flops_per_gpu = c->peak_flops_per_gpu;
  s.compute_efficiency = c->compute_efficiency;
  auto take = [k](const double* v) {
    return v ? std::vector<double>(v, v + k) : std::vector<double>{};
  };
  s.fwd_times = take(c->fwd_times);
  s.bwd_grad_weight_times = take(c->bwd_grad_weight_times);
  s.bwd_grad_input_times = take(c->bwd_grad_input_times);
  s.head_fwd_time = c->head_fwd_time;
  s.head_bwd_time = c->head_bwd_time;
  return s;
}

}  // namespace amsp::conv
