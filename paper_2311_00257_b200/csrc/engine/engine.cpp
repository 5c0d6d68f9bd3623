// The AMSP step engine: owns one rank's model-state buffers on its B200,
// maps the peers' buffers over NVLink (cudaIpc), and runs the step on a
// CUDA stream. One engine per GPU / process.
//
// Step (paper Fig 7 / SURVEY.md §3 call stack 5, pipeline-only form):
//   [s_p > 1] AG of every gather unit (forward order) then again (backward
//             order): NVLink pulls of the P-group's P shards;
//   barrier  -> fused reduce + AdamW + gather kernel ->  barrier.
//
// Memory layout per rank:
//   shared allocation (exported to peers):
//     grads  bf16 [Phi]      this rank's local gradient (backward output)
//     params bf16 [Phi/s_p]  this rank's P shard (= all params when s_p = 1),
//                            written by the OS owners of its elements
//     flags  u32 [8192 x 8]  cross-GPU barrier words ([id][r] written by rank r)
//     acc    bf16 [Phi/s_g]  G-shard micro-batch accumulator (M > 1, s_g > 1)
//   private allocation:
//     master, exp_avg, exp_avg_sq fp32 [owned]  the rank's OS shard
//     segment tables, 2 gathered-unit slots (s_p > 1), stats, error flag
// LLaMA-7B at s_p = 1: 27 GB shared + 81 GB / s_os private (fits 180 GB).
#include "engine_impl.h"

namespace {

void plan_groups(amsp_engine* e, const DeviceMesh& dp, const shardplan::ShardingPlan& plan) {
  e->sp = plan.sp();
  e->p_group = amsp::mesh_group(dp, plan.p, e->rank);
  e->os_group = amsp::mesh_group(dp, plan.os, e->rank);
  int my_k = -1;
  for (int m : e->os_group.members) {
    if (amsp::mesh_group(dp, plan.p, m).position == e->p_group.position) {
      if (m == e->rank) my_k = static_cast<int>(e->dst_members.size());
      e->dst_members.push_back(m);
    }
  }
  if (my_k < 0) throw Error("engine: rank missing from its own OS group");
  e->replicas = e->world / plan.sos();
  e->pmap = amsp::pshard_map(e->tensor_sizes, e->sp);
  e->param_elems = e->pmap.pshard_elems;
  e->layout = amsp::pshard_layout(e->tensor_sizes, e->sp, e->p_group.position,
                                  static_cast<int>(e->dst_members.size()), my_k,
                                  e->cfg.layout);
}

// Gradient accumulation over micro-batches. s_g = 1:
// every rank's full gradient buffer accumulates in place, nothing moves
// until the last micro-batch. s_g > 1 and M > 1 ("staged"): the ranks of a
// G-mesh block jointly accumulate, each holding the bf16 G shard of its
// elements; the last micro-batch sums the holders of every G block (block
// order) before the raw gradients.
void plan_accumulation(amsp_engine* e, const DeviceMesh& dp,
                       const shardplan::ShardingPlan& plan) {
  e->staged = e->sg > 1 && e->micro > 1;
  e->acc_by_dst = e->sg == e->sp;
  if (!e->staged) return;
  const amsp::MeshGroup mine = amsp::mesh_group(dp, plan.g, e->rank);
  e->acc_sources = mine.members;
  std::sort(e->acc_sources.begin(), e->acc_sources.end());
  e->acc_holders.assign(static_cast<std::size_t>(e->world / e->sg), -1);
  for (int r = 0; r < e->world; ++r) {
    const amsp::MeshGroup g = amsp::mesh_group(dp, plan.g, r);
    if (g.position == mine.position) e->acc_holders[static_cast<std::size_t>(g.block)] = r;
  }
  for (int h : e->acc_holders)
    if (h < 0) throw Error("engine: G mesh blocks do not tile the DP mesh");
  // s_g = s_p: the G shard is the P shard; s_g = s_os > s_p: the OS shard
  e->acc_elems = e->acc_by_dst ? e->param_elems : e->layout.owned;
}

// Gather units: consecutive tensors up to max(largest tensor, 2^27 elems).
void plan_units(amsp_engine* e, std::vector<amsp::CopySeg>& copy) {
  if (e->sp == 1) return;
  const std::size_t n = e->tensor_sizes.size();
  const std::uint64_t biggest =
      *std::max_element(e->tensor_sizes.begin(), e->tensor_sizes.end());
  const std::uint64_t cap = std::max<std::uint64_t>(biggest, std::uint64_t{1} << 27);
  std::size_t t = 0;
  while (t < n) {
    GatherUnit u;
    u.first_tensor = static_cast<int>(t);
    while (t < n && (u.n_tensors == 0 || u.elems + e->tensor_sizes[t] <= cap)) {
      u.elems += e->tensor_sizes[t];
      ++u.n_tensors;
      ++t;
    }
    std::vector<amsp::CopySeg> segs;
    const std::uint64_t base = e->pmap.tensor_offset[u.first_tensor];
    for (int i = 0; i < u.n_tensors; ++i) {
      const std::size_t ti = static_cast<std::size_t>(u.first_tensor + i);
      // One entry per tensor; the kernel interleaves the s_p sources tile by
      // tile (kernels.h CopySeg), rotated by this rank's P position.
      amsp::CopySeg c{};
      c.dst = e->pmap.tensor_offset[ti] - base;
      c.src = e->pmap.pshard_offset[ti];
      c.len = e->pmap.slice_len[ti];
      segs.push_back(c);
    }
    long long tiles = 0;
    for (auto& c : segs) {
      c.tile0 = static_cast<unsigned long long>(tiles);
      tiles += static_cast<long long>((c.len + amsp::kTile - 1) / amsp::kTile) * e->sp;
    }
    if (tiles > 0x7fffffffLL) throw Error("engine: gather unit too large");
    u.ntiles = static_cast<int>(tiles);
    u.seg_begin = static_cast<int>(copy.size());
    u.nseg = static_cast<int>(segs.size());
    copy.insert(copy.end(), segs.begin(), segs.end());
    e->slot_elems = std::max(e->slot_elems, u.elems);
    e->units.push_back(u);
  }
}

// Push all-gather tables: each rank handles only its own slice of every
// tensor of a unit (tile0 counts ceil(len / kTile) tiles per tensor) and
// stores it into all s_p members' slots.
void plan_push(amsp_engine* e, std::vector<amsp::CopySeg>& copy) {
  for (const auto& u : e->units) {
    GatherUnit v = u;
    v.seg_begin = static_cast<int>(copy.size());
    long long tiles = 0;
    for (int i = 0; i < u.n_tensors; ++i) {
      amsp::CopySeg c = copy[static_cast<std::size_t>(u.seg_begin + i)];
      c.tile0 = static_cast<unsigned long long>(tiles);
      tiles += static_cast<long long>((c.len + amsp::kTile - 1) / amsp::kTile);
      copy.push_back(c);
    }
    v.ntiles = static_cast<int>(tiles);
    e->units_push.push_back(v);
  }
}

// ZeRO++ secondary parameter shard (hpZ; plan.secondary_params, domain.hpp:
// 90-97): every rank keeps slice `position` of each tensor over its
// secondary group (Phi/s2 bf16, cost_model.cpp:148-150), refreshed from the
// forward all-gather; the backward all-gathers read the secondary group's
// slices instead of the primary P shards (overlap_sim.cpp:222-230,
// cost_model.cpp:41). Same gather units, a second copy table.
void plan_secondary(amsp_engine* e, const DeviceMesh& dp, const shardplan::ShardingPlan& plan,
                    std::vector<amsp::CopySeg>& copy) {
  if (!plan.secondary_params) return;
  if (e->sp == 1)
    throw Error("engine: a secondary parameter mesh needs parameter sharding (s_p > 1)");
  e->s2 = plan.secondary_params->size();
  if (e->s2 > e->world) throw Error("engine: secondary parameter mesh larger than the DP mesh");
  e->sec_group = amsp::mesh_group(dp, *plan.secondary_params, e->rank);
  e->smap = amsp::pshard_map(e->tensor_sizes, e->s2);
  // the forward gathers write the secondary slice as they go (GatherArgs::sec)
  // when every primary and secondary slice is 8-element aligned
  e->sec_fused = true;
  for (std::size_t t = 0; t < e->tensor_sizes.size(); ++t)
    if ((e->pmap.slice_len[t] | e->smap.slice_len[t]) & 7u) e->sec_fused = false;
  for (const auto& u : e->units)
    for (int i = 0; i < u.n_tensors; ++i)
      copy[static_cast<std::size_t>(u.seg_begin + i)].sec =
          e->smap.pshard_offset[static_cast<std::size_t>(u.first_tensor + i)];
  for (auto& u : e->units) {
    GatherUnit v = u;
    const std::uint64_t base = e->pmap.tensor_offset[u.first_tensor];
    long long tiles = 0;
    v.seg_begin = static_cast<int>(copy.size());
    for (int i = 0; i < u.n_tensors; ++i) {
      const std::size_t ti = static_cast<std::size_t>(u.first_tensor + i);
      amsp::CopySeg c{};
      c.dst = e->pmap.tensor_offset[ti] - base;
      c.src = e->smap.pshard_offset[ti];
      c.len = e->smap.slice_len[ti];
      c.tile0 = static_cast<unsigned long long>(tiles);
      tiles += static_cast<long long>((c.len + amsp::kTile - 1) / amsp::kTile) * e->s2;
      copy.push_back(c);
    }
    if (tiles > 0x7fffffffLL) throw Error("engine: gather unit too large");
    v.ntiles = static_cast<int>(tiles);
    v.nseg = u.n_tensors;
    e->units2.push_back(v);
  }
}

void create_engine(const amsp_engine_config_t* cfg, amsp_engine_t** out) {
  if (!cfg || !out) throw Error("engine: null argument");
  auto e = std::make_unique<amsp_engine>();
  e->cfg = *cfg;
  if (cfg->n_tensors < 1 || !cfg->tensor_sizes) throw Error("engine: no tensors");
  e->tensor_sizes.assign(cfg->tensor_sizes, cfg->tensor_sizes + cfg->n_tensors);
  for (auto s : e->tensor_sizes) {
    if (s == 0) throw Error("engine: tensor sizes must be positive");
    e->phi += s;
  }
  e->cfg.tensor_sizes = nullptr;
  const DeviceMesh dp = to_mesh(cfg->dp_mesh);
  e->world = dp.size();
  e->rank = cfg->rank;
  if (e->world < 1 || e->world > amsp::kMaxRanks)
    throw Error("engine: dp mesh " + shardplan::to_string(dp) +
                " outside the 1..8 GPU NVSwitch domain of one node");
  if (e->rank < 0 || e->rank >= e->world) throw Error("engine: rank out of range");

  // Plan semantics come from the planner's own validator.
  shardplan::ShardingPlan plan{to_mesh(cfg->plan.p), to_mesh(cfg->plan.g),
                               to_mesh(cfg->plan.os), std::nullopt};
  shardplan::ClusterSpec cl;
  cl.gpus_per_node = dp.per_node;
  cl.node_count = dp.nodes;
  cl.gpu_memory_capacity = 1;
  cl.dp_mesh = dp;
  cl.topology = {dp.nodes, 1, 1.0};
  const auto v = shardplan::validate_plan(plan, cl);
  if (!v.ok())
    throw Error("engine: plan " + shardplan::to_string(plan) + " violates " +
                v.violations.front().constraint);
  if (cfg->plan.has_secondary) {
    plan.secondary_params = to_mesh(cfg->plan.secondary);
    if (plan.secondary_params->per_node > dp.per_node || plan.secondary_params->nodes > dp.nodes)
      throw Error("engine: secondary parameter mesh " +
                  shardplan::to_string(*plan.secondary_params) + " does not fit dp mesh " +
                  shardplan::to_string(dp));
  }
  plan_groups(e.get(), dp, plan);
  e->micro = cfg->micro_batches > 0 ? cfg->micro_batches : 1;
  if (e->micro > 16) throw Error("engine: at most 16 micro-batches per step");
  e->sg = plan.sg();
  plan_accumulation(e.get(), dp, plan);
  e->ring = cfg->grad_ring_elems > 0;
  if (e->ring && e->sg == 1)
    throw Error("engine: a gradient ring needs s_g > 1 (s_g = 1 keeps the full gradient "
                "replica, D_g = 2*Phi)");
  e->grad_elems = e->ring ? (cfg->grad_ring_elems + 63) / 64 * 64 : e->phi;
  std::vector<amsp::CopySeg> copy;
  plan_units(e.get(), copy);
  plan_secondary(e.get(), dp, plan, copy);
  plan_push(e.get(), copy);
  // In-step all-gathers default to the TMA bulk-copy push kernel when every P
  // slice is 8-element aligned: on 13B ZeRO-3 the two passes take 57.7 ms
  // pushing vs 61.1 ms pulling at W = 4 (39.1 vs 40.8 at W = 2,
  // profiles/r02_gather_push_ab_13b.jsonl); the TMA pull kernel had beaten
  // the SM kernel (640 vs 608 GB/s) and the copy engines (357,
  // profiles/r01_tune_gather_tma.jsonl). Single gathers (and the ZeRO++
  // secondary passes) pull.
  if (e->sp > 1 && e->copies_aligned()) e->gather_grid = amsp_engine::kGatherPush;

  e->use_device();
  ck(cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking), "stream");

  // Shared region.
  e->off_grads = 0;
  e->off_params = align_up(e->grad_elems * 2);
  e->off_flags = e->off_params + align_up(e->param_elems * 2);
  e->off_sec = e->off_flags + align_up(kFlagBytes);
  // gather slots in the peer-exported region: the push all-gather stores
  // every rank's P slice straight into its peers' slots
  e->off_slots = e->off_sec + align_up(e->s2 > 1 ? e->smap.pshard_elems * 2 : 0);
  e->slot_bytes = align_up(e->slot_elems * 2);
  e->off_acc = e->off_slots + 2 * e->slot_bytes;
  // (the accumulator last: its size may differ per rank)
  e->shared_bytes = e->off_acc + align_up(e->acc_elems * 2);
  ck(cudaMalloc(&e->shared, e->shared_bytes), "cudaMalloc shared");
  ck(cudaMemset(e->shared + e->off_flags, 0, kFlagBytes), "zero flags");
  // a ring's slots are read before the scheduler first writes some of them
  // (tensors no backward event produces in compute='gemm' mode): keep them finite
  if (e->ring) ck(cudaMemset(e->shared + e->off_grads, 0, e->grad_elems * 2), "zero ring");
  for (int r = 0; r < e->world; ++r) e->peer_base[r] = e->shared;

  // Segment tables: the OS shard, and the whole P shard (for init).
  std::vector<amsp::Seg> segs, psegs;
  for (const auto& s : e->layout.segs) segs.push_back({s.flat, s.os, s.dst, s.len, 0});
  e->ntiles = tile_prefix(segs);
  e->nseg = static_cast<int>(segs.size());
  for (const auto& s : amsp::pshard_layout(e->tensor_sizes, e->sp, e->p_group.position, 1, 0,
                                           amsp::kLayoutContiguous).segs)
    psegs.push_back({s.flat, s.os, s.dst, s.len, 0});
  e->nptiles = tile_prefix(psegs);
  e->npseg = static_cast<int>(psegs.size());
  // Accumulation table: Seg::os = offset in the bf16 G-shard accumulator.
  std::vector<amsp::Seg> asegs;
  if (e->staged) {
    if (e->acc_by_dst)
      for (const auto& s : psegs) asegs.push_back({s.flat, s.dst, s.dst, s.len, 0});
    else
      asegs = segs;
    e->nacc_tiles = tile_prefix(asegs);
    e->nacc_seg = static_cast<int>(asegs.size());
  }

  // Private region.
  const std::size_t n = e->layout.owned;
  std::size_t off = 0;
  auto carve = [&off](std::size_t bytes) {
    const std::size_t at = off;
    off += align_up(std::max<std::size_t>(bytes, 1));
    return at;
  };
  const std::size_t o_master = carve(n * 4), o_m = carve(n * 4), o_v = carve(n * 4);
  const std::size_t o_seg = carve(segs.size() * sizeof(amsp::Seg));
  const std::size_t o_pseg = carve(psegs.size() * sizeof(amsp::Seg));
  const std::size_t o_copy = carve(copy.size() * sizeof(amsp::CopySeg));
  const std::size_t o_aseg = carve(asegs.size() * sizeof(amsp::Seg));
  const std::size_t o_stats = carve(kAlign), o_err = carve(kAlign), o_tab = carve(kAlign);
  ck(cudaMalloc(&e->priv, off), "cudaMalloc optimizer state");
  e->master = reinterpret_cast<float*>(e->priv + o_master);
  e->exp_avg = reinterpret_cast<float*>(e->priv + o_m);
  e->exp_avg_sq = reinterpret_cast<float*>(e->priv + o_v);
  e->d_segs = reinterpret_cast<amsp::Seg*>(e->priv + o_seg);
  e->d_psegs = reinterpret_cast<amsp::Seg*>(e->priv + o_pseg);
  e->d_copy = reinterpret_cast<amsp::CopySeg*>(e->priv + o_copy);
  e->d_acc_segs = reinterpret_cast<amsp::Seg*>(e->priv + o_aseg);
  e->slots[0] = e->slot_of(e->rank, 0);
  e->slots[1] = e->slot_of(e->rank, 1);
  e->stats = reinterpret_cast<float*>(e->priv + o_stats);
  e->err = reinterpret_cast<int*>(e->priv + o_err);
  e->d_peer_flags = reinterpret_cast<uint32_t**>(e->priv + o_tab);
  auto upload = [](void* dst, const void* src, std::size_t bytes, const char* what) {
    if (bytes) ck(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), what);
  };
  upload(e->d_segs, segs.data(), segs.size() * sizeof(amsp::Seg), "copy segments");
  upload(e->d_psegs, psegs.data(), psegs.size() * sizeof(amsp::Seg), "copy P segments");
  upload(e->d_copy, copy.data(), copy.size() * sizeof(amsp::CopySeg), "copy gather table");
  upload(e->d_acc_segs, asegs.data(), asegs.size() * sizeof(amsp::Seg), "copy accumulation table");
  ck(cudaMemset(e->priv + o_stats, 0, 2 * kAlign), "zero stats/err");
  e->publish_peer_flags();
  e->device_bytes = e->shared_bytes + off;

  int sms = 148;
  ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device), "sm count");
  e->sms = sms;
  e->retune(0, 0);
  *out = e.release();
}

void* buffer_ptr(amsp_engine_t* e, int which, std::size_t* elem, std::uint64_t* count) {
  switch (which) {
    case 0: *elem = 2; *count = e->grad_elems; return e->grads_of(e->rank);
    case 1: *elem = 2; *count = e->param_elems; return e->params_of(e->rank);
    case 2: *elem = 4; *count = e->layout.owned; return e->master;
    case 3: *elem = 4; *count = e->layout.owned; return e->exp_avg;
    case 4: *elem = 4; *count = e->layout.owned; return e->exp_avg_sq;
    case 5: *elem = 2; *count = e->slot_elems; return e->slots[0];
    case 6: *elem = 2; *count = e->slot_elems; return e->slots[1];
    case 7: *elem = 2; *count = e->acc_elems; return e->acc_of(e->rank);
    default: throw Error("engine: unknown buffer id " + std::to_string(which));
  }
}

// Single-GPU emulation of a group: every engine maps the others' buffers as
// its peers (amsp_engine_link_local / _sync).
void link_local(amsp_engine_t* const* engines, int n, bool sync) {
  if (!engines || n < 1) throw Error("engine: null argument");
  for (int r = 0; r < n; ++r) {
    const amsp_engine* e = engines[r];
    if (!e || e->world != n || e->rank != r || e->cfg.device != engines[0]->cfg.device ||
        e->phi != engines[0]->phi)
      throw Error("engine: link_local needs ranks 0..n-1 of one group on one device");
  }
  for (int r = 0; r < n; ++r) {
    amsp_engine* e = engines[r];
    for (int q = 0; q < n; ++q) e->peer_base[q] = engines[q]->shared;
    e->use_device();
    e->publish_peer_flags();
    e->imported = true;
    e->local_linked = true;
    e->local_sync = sync;
    // unsynchronised emulation: one stream orders the ranks' calls;
    // synchronised: every rank on its own stream, the barriers order them
    e->shared_default = sync ? nullptr : engines[0]->own_stream;
  }
}

}  // namespace

extern "C" {

int amsp_engine_create(const amsp_engine_config_t* cfg, amsp_engine_t** out) {
  return amsp::guarded([&] { create_engine(cfg, out); });
}

int amsp_engine_info(const amsp_engine_t* e, amsp_engine_info_t* info) {
  return amsp::guarded([&] {
    if (!e || !info) throw Error("engine: null argument");
    info->total_params = e->phi;
    info->owned = e->layout.owned;
    info->n_segments = e->nseg;
    info->world = e->world;
    info->os_block = e->os_group.block;
    info->os_position = e->os_group.position;
    info->os_group_size = static_cast<int>(e->dst_members.size());
    info->replica_count = e->replicas;
    info->ntiles = e->ntiles;
    info->grid = e->grid;
    info->block = amsp::kBlock;
    info->grads = e->grads_of(e->rank);
    info->params = e->params_of(e->rank);
    info->master = e->master;
    info->exp_avg = e->exp_avg;
    info->exp_avg_sq = e->exp_avg_sq;
    info->device_bytes = e->device_bytes;
    info->sp = e->sp;
    info->p_position = e->p_group.position;
    info->param_elems = e->param_elems;
    info->n_units = static_cast<int>(e->units.size());
    info->slot_elems = e->slot_elems;
    info->variant = e->variant;
    info->micro_batches = e->micro;
    info->grad_shards = e->sg;
    info->acc_elems = e->acc_elems;
    info->acc_sources = static_cast<int>(e->acc_sources.size());
    info->acc_holders = static_cast<int>(e->acc_holders.size());
    info->grad_elems = e->grad_elems;
    info->secondary_shards = e->s2;
    info->secondary_elems = e->s2 > 1 ? e->smap.pshard_elems : 0;
  });
}

int amsp_engine_unit(const amsp_engine_t* e, int unit, int* first_tensor, int* n_tensors,
                     uint64_t* elems) {
  return amsp::guarded([&] {
    if (!e) throw Error("engine: null argument");
    if (unit < 0 || unit >= static_cast<int>(e->units.size()))
      throw Error("engine: gather unit out of range");
    const GatherUnit& u = e->units[unit];
    if (first_tensor) *first_tensor = u.first_tensor;
    if (n_tensors) *n_tensors = u.n_tensors;
    if (elems) *elems = u.elems;
  });
}

int amsp_engine_gather(amsp_engine_t* e, int unit, int slot, void* stream) {
  return amsp::guarded([&] {
    if (!e) throw Error("engine: null argument");
    e->use_device();
    e->gather(unit, slot, e->pick(stream));
  });
}

int amsp_engine_gather_secondary(amsp_engine_t* e, int unit, int slot, void* stream) {
  return amsp::guarded([&] {
    if (!e) throw Error("engine: null argument");
    e->use_device();
    e->gather(unit, slot, e->pick(stream), true);
  });
}

int amsp_engine_export_handle(amsp_engine_t* e, void* handle64) {
  return amsp::guarded([&] {
    if (!e || !handle64) throw Error("engine: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == AMSP_IPC_HANDLE_BYTES);
    e->use_device();
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, e->shared), "cudaIpcGetMemHandle");
    std::memcpy(handle64, &h, sizeof(h));
  });
}

int amsp_engine_import_handles(amsp_engine_t* e, const void* handles, int world) {
  return amsp::guarded([&] {
    if (!e || !handles) throw Error("engine: null argument");
    if (world != e->world)
      throw Error("engine: got " + std::to_string(world) + " handles for a world of " +
                  std::to_string(e->world));
    e->use_device();
    for (int r = 0; r < world; ++r) {
      if (r == e->rank) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const char*>(handles) + r * AMSP_IPC_HANDLE_BYTES, sizeof(h));
      void* p = nullptr;
      ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      e->peer_base[r] = p;
    }
    e->publish_peer_flags();
    e->imported = true;
  });
}


int amsp_engine_link_local(amsp_engine_t* const* engines, int n) {
  return amsp::guarded([&] { link_local(engines, n, false); });
}

int amsp_engine_link_local_sync(amsp_engine_t* const* engines, int n) {
  return amsp::guarded([&] { link_local(engines, n, true); });
}

int amsp_engine_init_state(amsp_engine_t* e, void* stream) {
  return amsp::guarded([&] {
    if (!e) throw Error("engine: null argument");
    e->use_device();
    cudaStream_t s = e->pick(stream);
    ck(amsp::launch_init_params(e->d_psegs, e->npseg, e->nptiles, e->params_of(e->rank),
                                e->cfg.seed, s),
       "init params");
    ck(amsp::launch_init_state(e->d_segs, e->nseg, e->ntiles, e->master, e->exp_avg,
                               e->exp_avg_sq, e->cfg.seed, std::max(e->grid, 1), s),
       "init state");
    e->launches += 2;
  });
}

int amsp_engine_synth_grads(amsp_engine_t* e, int step, void* stream) {
  return amsp::guarded([&] {
    if (!e) throw Error("engine: null argument");
    e->require_full_grads("synth_grads");
    e->use_device();
    ck(amsp::launch_synth_grad(e->grads_of(e->rank), 0, e->phi, e->cfg.seed, step,
                               e->rank, e->pick(stream)),
       "synth grads");
    ++e->launches;
  });
}

int amsp_engine_synth_grads_mb(amsp_engine_t* e, int step, int mb, void* stream) {
  return amsp::guarded([&] {
    if (!e) throw Error("engine: null argument");
    e->check_micro_batch(mb);
    e->require_full_grads("synth_grads");
    e->use_device();
    // s_g = 1 accumulates micro-batches in the gradient buffer itself
    const bool in_place = e->sg == 1 && mb > 0;
    ck(amsp::launch_synth_grad(e->grads_of(e->rank), 0, e->phi, e->cfg.seed, step, e->rank,
                               e->pick(stream), mb, in_place),
       "synth grads");
    ++e->launches;
  });
}

int amsp_engine_accumulate(amsp_engine_t* e, int step, int mb, void* stream) {
  return amsp::guarded([&] {
    if (!e) throw Error("engine: null argument");
    if (step < 1) throw Error("engine: step index must be >= 1");
    e->require_full_grads("accumulate");
    e->use_device();
    e->accumulate(mb, e->pick(stream));
  });
}

int amsp_engine_step(amsp_engine_t* e, int step, void* stream) {
  return amsp::guarded([&] {
    if (!e) throw Error("engine: null argument");
    e->require_full_grads("step");
    e->use_device();
    e->step(step, e->pick(stream));
  });
}

int amsp_engine_step_host(amsp_engine_t* e, int step, const void* host_grads,
                          float* host_stats, void* stream) {
  return amsp::guarded([&] {
    if (!e || !host_grads) throw Error("engine: null argument");
    e->require_full_grads("step_host");
    e->use_device();
    cudaStream_t s = e->pick(stream);
    if (step < 1) throw Error("engine: step index must be >= 1");
    // Linked (emulated) engines upload on their own copy streams and skip the
    // per-chunk barriers, so a rank could update chunk c before a peer's
    // chunk c has landed: the host-buffer step needs real peers.
    if (e->local_linked && e->world > 1)
      throw Error("engine: step_host needs real peers (not link_local emulation)");
    if (e->micro > 1) throw Error("engine: step_host runs one micro-batch per step (M = 1)");
    if (e->sp == 1) {
      e->step_host_pipelined(step, host_grads, s);
    } else {
      // Parameter sharding: upload first, then the barrier-bracketed step
      // (its all-gathers run before the fused update).
      const std::size_t total = e->phi * 2, chunk = std::size_t{1} << 30;
      char* dst = reinterpret_cast<char*>(e->grads_of(e->rank));
      const char* src = static_cast<const char*>(host_grads);
      for (std::size_t off = 0; off < total; off += chunk)
        ck(cudaMemcpyAsync(dst + off, src + off, std::min(chunk, total - off),
                           cudaMemcpyHostToDevice, s),
           "H2D gradients");
      e->step(step, s);
    }
    if (host_stats)
      ck(cudaMemcpyAsync(host_stats, e->stats, 2 * sizeof(float), cudaMemcpyDeviceToHost, s),
         "D2H stats");
    ck(cudaStreamSynchronize(s), "step sync");
    e->check_err();
  });
}

int amsp_engine_stats(amsp_engine_t* e, float* stats2) {
  return amsp::guarded([&] {
    if (!e || !stats2) throw Error("engine: null argument");
    e->use_device();
    ck(cudaDeviceSynchronize(), "sync");
    e->check_err();
    ck(cudaMemcpy(stats2, e->stats, 2 * sizeof(float), cudaMemcpyDeviceToHost), "read stats");
  });
}

int amsp_engine_read(amsp_engine_t* e, int which, uint64_t offset, uint64_t count,
                     void* host_dst) {
  return amsp::guarded([&] {
    if (!e || (!host_dst && count)) throw Error("engine: null argument");
    std::size_t elem = 0;
    std::uint64_t n = 0;
    char* p = static_cast<char*>(buffer_ptr(e, which, &elem, &n));
    if (offset > n || count > n - offset) throw Error("engine: read out of range");
    e->use_device();
    ck(cudaDeviceSynchronize(), "sync");
    e->check_err();
    if (count) ck(cudaMemcpy(host_dst, p + offset * elem, count * elem, cudaMemcpyDeviceToHost), "D2H");
  });
}

int amsp_engine_write(amsp_engine_t* e, int which, uint64_t offset, uint64_t count,
                      const void* host_src) {
  return amsp::guarded([&] {
    if (!e || (!host_src && count)) throw Error("engine: null argument");
    std::size_t elem = 0;
    std::uint64_t n = 0;
    char* p = static_cast<char*>(buffer_ptr(e, which, &elem, &n));
    if (offset > n || count > n - offset) throw Error("engine: write out of range");
    e->use_device();
    ck(cudaDeviceSynchronize(), "sync");
    if (count) ck(cudaMemcpy(p + offset * elem, host_src, count * elem, cudaMemcpyHostToDevice), "H2D");
  });
}

int amsp_engine_tune_gather(amsp_engine_t* e, int grid) {
  return amsp::guarded([&] {
    if (!e || grid < -3) throw Error("engine: bad argument");
    if ((grid == amsp_engine::kGatherTma || grid == amsp_engine::kGatherPush) &&
        !e->copies_aligned())
      throw Error("engine: the TMA all-gathers need 8-element-aligned P slices");
    e->gather_grid = grid;
  });
}

int amsp_engine_tune(amsp_engine_t* e, int variant, int grid) {
  return amsp::guarded([&] {
    if (!e) throw Error("engine: null argument");
    if (variant < 0 || variant > 12) throw Error("engine: unknown kernel variant");
    if (variant >= 5) {
      for (const auto& s : e->layout.segs)
        if ((s.flat | s.os | s.dst | s.len) & 7u)
          throw Error("engine: the TMA variant needs 8-element-aligned segments");
    }
    e->use_device();
    e->retune(variant, grid);
  });
}

int amsp_engine_time_kernel(amsp_engine_t* e, int enable) {
  return amsp::guarded([&] {
    if (!e) throw Error("engine: null argument");
    e->time_kernel = enable != 0;
    e->kernel_events_used = 0;
    e->gather_events_used = 0;
    e->accum_events_used = 0;
  });
}

int amsp_engine_kernel_ms(amsp_engine_t* e, double* total_ms, int* launches) {
  return amsp::guarded([&] {
    if (!e || !total_ms) throw Error("engine: null argument");
    e->use_device();
    *total_ms = amsp_engine::sum_ms(e->kernel_events, e->kernel_events_used);
    if (launches) *launches = static_cast<int>(e->kernel_events_used);
    e->kernel_events_used = 0;
  });
}

int amsp_engine_gather_ms(amsp_engine_t* e, double* total_ms, int* steps) {
  return amsp::guarded([&] {
    if (!e || !total_ms) throw Error("engine: null argument");
    e->use_device();
    *total_ms = amsp_engine::sum_ms(e->gather_events, e->gather_events_used);
    if (steps) *steps = static_cast<int>(e->gather_events_used);
    e->gather_events_used = 0;
  });
}

int amsp_engine_accum_ms(amsp_engine_t* e, double* total_ms, int* launches) {
  return amsp::guarded([&] {
    if (!e || !total_ms) throw Error("engine: null argument");
    e->use_device();
    *total_ms = amsp_engine::sum_ms(e->accum_events, e->accum_events_used);
    if (launches) *launches = static_cast<int>(e->accum_events_used);
    e->accum_events_used = 0;
  });
}

int amsp_engine_nvlink_probe(amsp_engine_t* e, uint64_t bytes, int pattern, int iters,
                             double* ms_per_iter) {
  return amsp::guarded([&] {
    if (!e || !ms_per_iter) throw Error("engine: null argument");
    if (e->world < 2) throw Error("engine: the NVLink probe needs peers");
    if (pattern < 0 || pattern > 1 || iters < 1) throw Error("engine: bad probe arguments");
    e->require_peers();
    e->use_device();
    amsp::PullArgs a{};
    if (pattern == 0) {  // ring: pull everything from the next rank
      a.nsrc = 1;
      a.src[0] = reinterpret_cast<const uint4*>(e->grads_of((e->rank + 1) % e->world));
    } else {  // all-to-all: an equal share from every peer
      for (int j = 1; j < e->world; ++j)
        a.src[a.nsrc++] = reinterpret_cast<const uint4*>(e->grads_of((e->rank + j) % e->world));
    }
    a.rot = 0;
    const std::uint64_t per_src = std::min<std::uint64_t>(bytes / a.nsrc, e->grad_elems * 2) / 16;
    if (per_src == 0) throw Error("engine: probe size too small");
    a.vecs_per_src = per_src;
    const std::uint64_t total = per_src * 16 * a.nsrc;
    void* dst = nullptr;
    ck(cudaMalloc(&dst, total), "cudaMalloc probe buffer");
    a.dst = static_cast<uint4*>(dst);
    cudaStream_t s = e->own_stream;
    cudaEvent_t x, y;
    ck(cudaEventCreate(&x), "event");
    ck(cudaEventCreate(&y), "event");
    try {
      ck(amsp::launch_p2p_pull(a, 0, s), "probe warm-up");
      e->barrier(s);  // every rank pulls at the same time
      ck(cudaEventRecord(x, s), "event record");
      for (int i = 0; i < iters; ++i) ck(amsp::launch_p2p_pull(a, 0, s), "probe");
      ck(cudaEventRecord(y, s), "event record");
      e->barrier(s);
      ck(cudaEventSynchronize(y), "event sync");
      float ms = 0.0f;
      ck(cudaEventElapsedTime(&ms, x, y), "event elapsed");
      *ms_per_iter = ms / iters;
      e->launches += static_cast<std::uint64_t>(iters) + 1;
    } catch (...) {
      cudaEventDestroy(x);
      cudaEventDestroy(y);
      cudaFree(dst);
      throw;
    }
    cudaEventDestroy(x);
    cudaEventDestroy(y);
    cudaFree(dst);
    e->check_err();
  });
}

int amsp_engine_launch_count(const amsp_engine_t* e, uint64_t* n) {
  return amsp::guarded([&] {
    if (!e || !n) throw Error("engine: null argument");
    *n = e->launches;
  });
}

void amsp_engine_destroy(amsp_engine_t* e) {
  if (!e) return;
  cudaSetDevice(e->cfg.device);
  cudaDeviceSynchronize();
  for (int r = 0; r < e->world; ++r)
    if (!e->local_linked && r != e->rank && e->peer_base[r] && e->peer_base[r] != e->shared)
      cudaIpcCloseMemHandle(e->peer_base[r]);
  cudaFree(e->shared);
  cudaFree(e->priv);
  cudaFree(e->d_chunk_segs);
  for (auto ev : e->chunk_events) cudaEventDestroy(ev);
  if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
  if (e->own_stream) cudaStreamDestroy(e->own_stream);
  for (auto* pairs : {&e->kernel_events, &e->gather_events, &e->accum_events})
    for (auto& ev : *pairs) {
      cudaEventDestroy(ev.first);
      cudaEventDestroy(ev.second);
    }
  delete e;
  cudaGetLastError();  // teardown must not leave a sticky error for the next call
}

// ------------------------------------------------------------ raw kernels

int amsp_k_synth_grad(void* dst_bf16, uint64_t start, uint64_t n, uint64_t seed,
                      int step, int rank, void* stream) {
  return amsp::guarded([&] {
    ck(amsp::launch_synth_grad(static_cast<uint16_t*>(dst_bf16), start, n, seed, step,
                               rank, static_cast<cudaStream_t>(stream)),
       "synth grad");
  });
}

int amsp_k_spin(int ctas, uint64_t ns, void* stream) {
  return amsp::guarded([&] {
    if (ctas < 1 || ctas > 65535) throw Error("spin: 1..65535 CTAs");
    ck(amsp::launch_spin(ctas, ns, static_cast<cudaStream_t>(stream)), "spin");
  });
}

int amsp_k_adamw(const void* grad, int grad_is_bf16, float* master, float* m, float* v,
                 void* param_out_bf16, uint64_t n, int step, double lr, double beta1,
                 double beta2, double eps, double weight_decay, double grad_scale,
                 void* stream) {
  return amsp::guarded([&] {
    if (step < 1) throw Error("adamw: step index must be >= 1");
    const amsp::AdamScalars s =
        amsp::make_adam_scalars(lr, beta1, beta2, eps, weight_decay, step, grad_scale);
    ck(amsp::launch_adamw_flat(grad, grad_is_bf16 != 0, master, m, v,
                               static_cast<uint16_t*>(param_out_bf16), n, s,
                               static_cast<cudaStream_t>(stream)),
       "adamw");
  });
}

int amsp_k_upcast_scale(const void* src_bf16, float* dst, uint64_t n, float scale,
                        void* stream) {
  return amsp::guarded([&] {
    ck(amsp::launch_upcast_scale(static_cast<const uint16_t*>(src_bf16), dst, n, scale,
                                 static_cast<cudaStream_t>(stream)),
       "upcast");
  });
}

int amsp_k_rs_upcast_scale(const void* const* srcs_bf16, int nsrc, uint64_t offset,
                           float* dst, uint64_t n, float scale, void* stream) {
  return amsp::guarded([&] {
    if (!srcs_bf16 || (n && !dst)) throw Error("rs_upcast_scale: null argument");
    if (nsrc < 1 || nsrc > amsp::kMaxRanks) throw Error("rs_upcast_scale: 1..8 sources");
    ck(amsp::launch_rs_upcast_scale(reinterpret_cast<const uint16_t* const*>(srcs_bf16), nsrc,
                                    offset, dst, n, scale, static_cast<cudaStream_t>(stream)),
       "rs_upcast_scale");
  });
}

int amsp_k_ag_downcast(const float* src, uint64_t n, void* const* dsts_bf16, int ndst,
                       uint64_t dst_offset, void* stream) {
  return amsp::guarded([&] {
    if (!dsts_bf16 || (n && !src)) throw Error("ag_downcast: null argument");
    if (ndst < 1 || ndst > amsp::kMaxRanks) throw Error("ag_downcast: 1..8 destinations");
    ck(amsp::launch_ag_downcast(src, n, reinterpret_cast<uint16_t* const*>(dsts_bf16), ndst,
                                dst_offset, static_cast<cudaStream_t>(stream)),
       "ag_downcast");
  });
}

}  // extern "C"
