/* amsp_c.h — C-ABI of the B200-native AMSP model-state pipeline.
 *
 * Plain C: POD structs, plain pointers and sizes, opaque handles, no torch or
 * C++ types. Every call returns an int status (AMSP_OK=0, AMSP_EINVAL=1 bad
 * config, AMSP_EINFEASIBLE=2 nothing fits, AMSP_ECUDA=3 CUDA / peer error;
 * the 0/1/2 meanings mirror the reference CLI exit codes) and
 * amsp_last_error() returns a thread-local message. No C++ exception crosses
 * this boundary.
 *
 * Two halves:
 *  1. Planner (host only, no GPU needed). Each function is a drop-in for one
 *     reference entry point of the `shardplan` C++ API, cited per function.
 *     The full C++ API itself is include/amsp/plan.hpp (namespace shardplan).
 *  2. Engine + kernels (B200, sm_100a). The reference has NO data plane
 *     (SPEC.md:16); these entry points execute what its cost model and
 *     overlap simulator describe (SURVEY.md §3 call stack 5):
 *     gradient reduce (RS in the OS group + cross-replica sum) fused with
 *     the bf16->fp32 upcast and 1/W scale, sharded AdamW on the local OS
 *     shard, and the parameter gather fused with the fp32->bf16 downcast —
 *     one kernel over NVLink peer memory (cudaIpc-mapped buffers of every
 *     rank of the data-parallel group).
 *
 * Threading: planner calls are pure and thread-safe. One engine per GPU
 * (one process per GPU); engine calls are not reentrant.
 */
#ifndef AMSP_C_H_
#define AMSP_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMSP_OK 0
#define AMSP_EINVAL 1
#define AMSP_EINFEASIBLE 2
#define AMSP_ECUDA 3

#define AMSP_ABI_VERSION 2

int amsp_abi_version(void);
const char* amsp_last_error(void);

/* ------------------------------------------------------------ POD mirrors */

/* shardplan::DeviceMesh (reference domain.hpp:39-46) */
typedef struct { int per_node; int nodes; } amsp_mesh_t;

/* shardplan::ShardingPlan (domain.hpp:93-113) */
typedef struct {
  amsp_mesh_t p, g, os;
  int has_secondary;
  amsp_mesh_t secondary;
} amsp_plan_t;

/* shardplan::ClusterSpec + Topology (domain.hpp:51-67) */
typedef struct {
  int gpus_per_node, node_count;
  uint64_t gpu_memory_capacity;
  amsp_mesh_t dp_mesh;
  int leaf_count, nodes_per_leaf;
  double inter_leaf_penalty;
} amsp_cluster_t;

/* shardplan::ModelSpec (domain.hpp:72-88); module_params has
 * modules_per_layer entries and is only read during the call. */
typedef struct {
  uint64_t total_params;
  int layer_count, modules_per_layer;
  const uint64_t* module_params;
  int hidden, seq_len, micro_batch, micro_batch_count, vocab;
  int bytes_per_param, bytes_per_grad, bytes_per_os_per_param;
} amsp_model_t;

/* shardplan::CostConfig (cost_model.hpp:28-50); activation_mode 0 = None,
 * 1 = FullRecompute. amsp_cost_config_default() fills the reference
 * defaults. */
typedef struct {
  uint64_t bucket_size;
  int activation_mode;
  double activation_coeff_full, activation_coeff_recompute;
  int tmp_in_flight_buckets, tmp_include_gather_buffer, exact_residual_buckets;
  double flops_coeff_param, flops_coeff_attn;
} amsp_cost_config_t;

/* shardplan::TimeBreakdown / MemoryBreakdown (cost_model.hpp:52-68) */
typedef struct { double t_p, t_g, t_os_allreduce, t_os_broadcast, total; } amsp_time_t;
typedef struct {
  double d_params, d_grads, d_os, d_modelstate, d_activation, d_tmp, d_total;
} amsp_memory_t;

/* shardplan::PlanResult (planner.hpp:27-33) */
typedef struct {
  amsp_plan_t plan;
  amsp_time_t time;
  amsp_memory_t memory;
  int feasible;
  int rank;
} amsp_plan_result_t;

/* shardplan::SimConfig (overlap_sim.hpp:66-80). tier: 0 none, 1 ag_rs,
 * 2 ag_rs_ar, 3 ag_rs_ar_bc. time_source: 0 FLOPs, 1 table (the three
 * per-module tables then hold modules_per_layer entries each). */
typedef struct {
  int overlap_tier, recompute, comm_streams, compute_time_source;
  double peak_flops_per_gpu, compute_efficiency;
  const double* fwd_times;
  const double* bwd_grad_weight_times;
  const double* bwd_grad_input_times;
  double head_fwd_time, head_bwd_time;
} amsp_sim_config_t;

/* shardplan::BandwidthProfile, opaque. */
typedef struct amsp_profile amsp_profile_t;

void amsp_cost_config_default(amsp_cost_config_t* cfg);
void amsp_sim_config_default(amsp_sim_config_t* cfg);

/* ------------------------------------------------------------ planner */

/* synthetic_profile (comm_model.cpp:129-160) */
int amsp_profile_synthetic(double alpha_intra, double bw_intra,
                           double alpha_inter, double bw_inter,
                           const amsp_mesh_t* meshes, int n_meshes,
                           const uint64_t* sizes, int n_sizes,
                           amsp_profile_t** out);
/* profile_from_csv (comm_model.cpp:182-228) / profile_from_json (:251-287) /
 * load_profile (:289-297) */
int amsp_profile_from_csv(const char* csv_text, amsp_profile_t** out);
int amsp_profile_from_json(const char* json_text, amsp_profile_t** out);
int amsp_profile_load(const char* path, amsp_profile_t** out);
/* profile_to_canonical_json (comm_model.cpp:234-249). Writes up to cap bytes
 * (NUL-terminated when it fits); *needed = length without NUL. */
int amsp_profile_to_json(const amsp_profile_t* p, char* buf, size_t cap,
                         size_t* needed);
/* BandwidthProfile::collective_time (comm_model.cpp:121-127); kind 0 AG,
 * 1 RS, 2 AR, 3 BC. */
int amsp_collective_time(const amsp_profile_t* p, int kind, uint64_t size_bytes,
                         amsp_mesh_t mesh, double* seconds);
void amsp_profile_free(amsp_profile_t* p);

/* ring_time (comm_model.cpp:45-55) */
int amsp_ring_time(int kind, double size_bytes, int participants, double alpha,
                   double link_bandwidth, double* seconds);

/* validate_plan (domain.cpp:137-166). Violations are written as
 * "constraint:detail\n" lines into buf. */
int amsp_validate_plan(const amsp_plan_t* plan, const amsp_cluster_t* cluster,
                       int* n_violations, char* buf, size_t cap);
/* preset (domain.cpp:197-226); AMSP_EINFEASIBLE when it does not fit. */
int amsp_preset(const char* name, const amsp_cluster_t* cluster, amsp_plan_t* out);

/* memory_breakdown / total_comm_time / grad_bucket_count
 * (cost_model.cpp:142-171, :128-140, :57-65) */
int amsp_memory_breakdown(const amsp_model_t* model, const amsp_plan_t* plan,
                          const amsp_cost_config_t* cfg, amsp_memory_t* out);
int amsp_total_comm_time(const amsp_model_t* model, const amsp_cluster_t* cluster,
                         const amsp_plan_t* plan, const amsp_profile_t* profile,
                         const amsp_cost_config_t* cfg, amsp_time_t* out);
int amsp_grad_bucket_count(const amsp_model_t* model, const amsp_plan_t* plan,
                           const amsp_cost_config_t* cfg, uint64_t* out);

/* partition_tensors_greedy (cost_model.cpp:189-219) */
int amsp_partition_greedy(const uint64_t* sizes, int n, int shard_count,
                          int* assignment, uint64_t* shard_sizes);

/* enumerate_candidates (planner.cpp:110-129): up to cap plans; *n = total. */
int amsp_enumerate_candidates(const amsp_cluster_t* cluster, amsp_plan_t* plans,
                              int cap, int* n);
/* solve (planner.cpp:144-166). On AMSP_EINFEASIBLE *best holds the
 * minimal-memory candidate (NoFeasiblePlanError::closest). all/cap/n_all
 * optionally receive the ranked candidate list. */
int amsp_solve(const amsp_model_t* model, const amsp_cluster_t* cluster,
               const amsp_profile_t* profile, const amsp_cost_config_t* cfg,
               amsp_plan_result_t* best, uint64_t* evaluated, uint64_t* filtered,
               amsp_plan_result_t* all, int cap, int* n_all);

/* build_schedule + simulate_step + bubble_report + render_trace
 * (overlap_sim.cpp:442-577). Any output pointer may be NULL. */
int amsp_simulate(const amsp_model_t* model, const amsp_cluster_t* cluster,
                  const amsp_plan_t* plan, const amsp_profile_t* profile,
                  const amsp_cost_config_t* cfg, const amsp_sim_config_t* sim,
                  double* step_time, double* compute_idle, int* n_events,
                  char* trace, size_t trace_cap, size_t* trace_needed);

/* ------------------------------------------------------------ layout */

#define AMSP_LAYOUT_GREEDY 0     /* reference inter-tensor LPT index map */
#define AMSP_LAYOUT_CONTIGUOUS 1 /* even contiguous split, 8-element aligned */

/* One rank's optimizer-state segments over the flat parameter vector
 * (tensors concatenated in forward order): segment s covers flat elements
 * [flat[s], flat[s]+len[s]) stored at os[s] in the rank's fp32 shard. */
int amsp_layout_segments(const uint64_t* tensor_sizes, int n_tensors,
                         int shard_count, int shard, int layout,
                         uint64_t* flat, uint64_t* os, uint64_t* len, int cap,
                         int* n_segments, uint64_t* owned);

/* Parameter-sharded variant (s_p > 1, ZeRO-3 intra-tensor split): P
 * position p_pos holds slice p_pos of every tensor (tensors must be
 * multiples of s_p); its P shard is split over the k ranks of the OS group
 * sharing that P position. dst[s] is the segment's offset in the P shard. */
int amsp_pshard_layout(const uint64_t* tensor_sizes, int n_tensors, int sp, int p_pos,
                       int k, int os_pos, int layout, uint64_t* flat, uint64_t* os,
                       uint64_t* dst, uint64_t* len, int cap, int* n_segments,
                       uint64_t* owned);

/* B200 roofline of one engine step (engine/roofline.h):
 * algorithmic HBM / NVLink bytes of `rank` for `plan` on `dp`, with
 * `gathers` all-gather passes when s_p > 1, and the bound step time
 * max(hbm/hbm_bw, max(in, out)/nvlink_bw). rank < 0 = the slowest rank
 * (written to *slowest when non-NULL). No reference counterpart: the
 * reference costs communication only (cost_model.cpp:128-140). */
typedef struct {
  uint64_t owned, hbm_bytes, nvlink_in_bytes, nvlink_out_bytes;
  double t_hbm, t_nvlink, t_step;
} amsp_step_roofline_t;

int amsp_step_roofline(const uint64_t* tensor_sizes, int n_tensors, const amsp_plan_t* plan,
                       amsp_mesh_t dp, int rank, int layout, int gathers, double hbm_bw,
                       double nvlink_bw, int* slowest, amsp_step_roofline_t* out);

/* The engine's flat tensor list of a LLaMA-style model (embed, L x modules,
 * final norm, lm_head); *n = count, sizes[0..min(cap, n)) filled. */
int amsp_model_tensors(const amsp_model_t* model, uint64_t* sizes, int cap, int* n);

/* Roofline solver: the reference's candidates (enumerate_candidates,
 * planner.cpp:110-129), memory model and feasibility (evaluate_plan,
 * :131-141), restricted to plans the engine can run, ordered by the B200
 * step roofline of the slowest rank (2 gather passes when s_p > 1), then
 * T_comm, then the plan's lex key. Outputs as amsp_solve; code 2 when no
 * candidate qualifies (best = the leanest candidate). amsp_solve itself
 * stays the reference objective, bit-exact. */
int amsp_solve_roofline(const amsp_model_t* model, const amsp_cluster_t* cluster,
                        const amsp_profile_t* profile, const amsp_cost_config_t* cfg,
                        double hbm_bw, double nvlink_bw, int layout, amsp_plan_result_t* best,
                        amsp_step_roofline_t* best_step, amsp_plan_result_t* all,
                        amsp_step_roofline_t* all_steps, int cap, int* n_all);

/* Group of `rank` for component mesh `mesh` inside the DP mesh `dp`
 * (ranks numbered node-major: rank = node*dp.per_node + local). Returns the
 * block index, the rank's position in its block and the block's members in
 * position order. */
int amsp_mesh_group(amsp_mesh_t dp, amsp_mesh_t mesh, int rank, int* block,
                    int* position, int* members, int cap, int* n_members);

/* ------------------------------------------------------------ engine */

typedef struct amsp_engine amsp_engine_t;

typedef struct {
  const uint64_t* tensor_sizes; /* flat order; read during create only */
  int n_tensors;
  amsp_plan_t plan;
  amsp_mesh_t dp_mesh;          /* rank count = dp_mesh.per_node*dp_mesh.nodes */
  int rank;
  int device;                   /* CUDA ordinal */
  int layout;                   /* AMSP_LAYOUT_* */
  double lr, beta1, beta2, eps, weight_decay;
  uint64_t seed;
  int skip_gathers;             /* s_p > 1: 0 = amsp_engine_step runs the
                                   forward + backward parameter all-gathers
                                   itself; 1 = the caller schedules
                                   amsp_engine_gather (overlap scheduler) */
  int micro_batches;            /* M per step (0 = 1; at most 16). With M > 1
                                   and s_g > 1 the engine keeps the bf16 G
                                   shard accumulator of D_g = 2*Phi/s_g bytes
                                   (cost_model.cpp:151): micro-batches
                                   0..M-2 go through amsp_engine_accumulate
                                   (the T_g collectives, cost_model.cpp:
                                   119-126), the last one through
                                   amsp_engine_step. With s_g = 1 the
                                   gradient buffer accumulates in place. */
  uint64_t grad_ring_elems;     /* 0: the gradient buffer holds all Phi
                                   bf16 gradients (the pipeline API:
                                   synth_grads / accumulate / step /
                                   step_host). > 0 (needs s_g > 1): a ring of
                                   this many bf16 elements instead, written
                                   and consumed only by the overlap
                                   scheduler, which places every micro-
                                   batch's tensor gradients in it as backward
                                   produces them and frees them when every
                                   rank has reduced them, so gradient memory
                                   is D_g = 2*Phi/s_g (the accumulator) plus
                                   this transient ring (cost_model.cpp:151). */
} amsp_engine_config_t;

typedef struct {
  uint64_t total_params;        /* Phi */
  uint64_t owned;               /* elements of this rank's OS shard */
  int n_segments;
  int world, os_block, os_position, os_group_size, replica_count;
  int ntiles, grid, block;      /* fused-kernel launch geometry */
  void* grads;                  /* bf16 [Phi] */
  void* params;                 /* bf16 [Phi] */
  void* master;                 /* fp32 [owned] */
  void* exp_avg;                /* fp32 [owned] */
  void* exp_avg_sq;             /* fp32 [owned] */
  uint64_t device_bytes;        /* allocated by the engine */
  int sp;                       /* parameter shard factor s_p */
  int p_position;               /* position in the P group */
  uint64_t param_elems;         /* elements of `params` (Phi / s_p) */
  int n_units;                  /* all-gather units (s_p > 1) */
  uint64_t slot_elems;          /* gathered-unit slot capacity */
  int variant;                  /* fused-kernel variant in use (see amsp_engine_tune) */
  int micro_batches;            /* M */
  int grad_shards;              /* s_g */
  uint64_t acc_elems;           /* bf16 G-shard accumulator elements (0 when
                                   M = 1 or s_g = 1): Phi/s_p when s_g = s_p,
                                   else the OS shard (s_g = s_os) */
  int acc_sources;              /* ranks pulled per accumulation (|G block|) */
  int acc_holders;              /* accumulators summed by the last micro-batch */
  uint64_t grad_elems;          /* elements of the local gradient buffer */
  int secondary_shards;         /* ZeRO++ secondary mesh size s2 (1: none) */
  uint64_t secondary_elems;     /* this rank's secondary slice (Phi/s2) */
} amsp_engine_info_t;

#define AMSP_IPC_HANDLE_BYTES 64

int amsp_engine_create(const amsp_engine_config_t* cfg, amsp_engine_t** out);
int amsp_engine_info(const amsp_engine_t* e, amsp_engine_info_t* info);
/* Export this rank's peer-shared buffer (grads | params | flags). */
int amsp_engine_export_handle(amsp_engine_t* e, void* handle64);
/* s_p > 1: gather unit u = a run of consecutive tensors; its parameters are
 * all-gathered (NVLink pulls from the P group's P shards, the paper's per-
 * module AllGather, cost_model.cpp:46-49) into gathered slot `slot` (0/1)
 * as the full tensors concatenated in flat order. */
int amsp_engine_unit(const amsp_engine_t* e, int unit, int* first_tensor, int* n_tensors,
                     uint64_t* elems);
int amsp_engine_gather(amsp_engine_t* e, int unit, int slot, void* stream);
/* ZeRO++ (plan.has_secondary): the same all-gather from the secondary
 * group's secondary slices (the backward gather of the step). */
int amsp_engine_gather_secondary(amsp_engine_t* e, int unit, int slot, void* stream);
/* Map every other rank's buffer; handles = world * 64 bytes in rank order. */
int amsp_engine_import_handles(amsp_engine_t* e, const void* handles, int world);
/* Single-GPU emulation of a DP group (tests / smoke): link n engines created
 * in this process on the SAME device as ranks 0..n-1 of one group. Linked
 * engines skip the cross-GPU barriers, so the caller must run their steps
 * one after another on one stream (synth all grads, then step every rank). */
int amsp_engine_link_local(amsp_engine_t* const* engines, int n);
/* Like amsp_engine_link_local, but the linked engines keep the multi-GPU
 * synchronisation: every engine issues on its OWN default stream and runs
 * the real barrier_kernel flag protocol and the __threadfence_system release
 * of its parameter stores, exactly as with separate GPUs (one process, one
 * CUDA context: the ranks' kernels share the device, they are not
 * time-sliced processes). Calls may be interleaved rank by rank; the
 * barriers order them. */
int amsp_engine_link_local_sync(amsp_engine_t* const* engines, int n);
/* master = 0.02*u(seed, i), m = v = 0, params = bf16(master) (all ranks
 * derive the identical replicated initial parameters locally). */
int amsp_engine_init_state(amsp_engine_t* e, void* stream);
/* Synthetic bf16 gradients for this rank and step (oracle definition). */
int amsp_engine_synth_grads(amsp_engine_t* e, int step, void* stream);
/* Same for micro-batch mb of the step: written into the gradient buffer, or
 * with s_g = 1 and mb > 0 accumulated into it in place (bf16). */
int amsp_engine_synth_grads_mb(amsp_engine_t* e, int step, int mb, void* stream);
/* Micro-batch mb < M-1 of the step is complete in every rank's gradient
 * buffer: with s_g > 1, cross-GPU barrier, fold it into the G shard
 * accumulators (each holder pulls its accumulation block's bf16 gradients
 * over NVLink: the reduce-scatter / AllReduce + select & drop of
 * PAPER.md:320-326 as one pass), barrier (the buffer may be overwritten).
 * With s_g = 1 a no-op (the producer accumulates in place). */
int amsp_engine_accumulate(amsp_engine_t* e, int step, int mb, void* stream);
/* One AMSP optimizer step (1-based step index) with device-resident grads
 * (the last micro-batch when M > 1): cross-GPU barrier, fused reduce (of the
 * accumulators, then the raw gradients; scale 1/(W*M)) + AdamW + gather
 * kernel, cross-GPU barrier. */
int amsp_engine_step(amsp_engine_t* e, int step, void* stream);
/* Same step through host buffers: H2D of this rank's bf16 gradients
 * (total_params elements; pinned for async), the step, and D2H of the step
 * statistics (stats[0] = sum of squared reduced grads over the rank's shard).
 * Synchronizes the stream before returning. */
int amsp_engine_step_host(amsp_engine_t* e, int step, const void* host_grads,
                          float* host_stats, void* stream);
/* Device step statistics of the last step (synchronous). */
int amsp_engine_stats(amsp_engine_t* e, float* stats2);
/* Copy `count` elements at `offset` of a buffer to host (synchronous).
 * which: 0 grads(bf16) 1 params(bf16, the P shard) 2 master 3 exp_avg
 * 4 exp_avg_sq 5/6 gathered slot 0/1 (bf16) 7 G-shard accumulator (bf16). */
int amsp_engine_read(amsp_engine_t* e, int which, uint64_t offset, uint64_t count,
                     void* host_dst);
int amsp_engine_write(amsp_engine_t* e, int which, uint64_t offset, uint64_t count,
                      const void* host_src);
/* Fused-kernel tuning: variant 0 auto, 1 one vector in flight per thread,
 * 2 two vectors, 3 two vectors + >=3 CTAs/SM, 4 one vector + >=4 CTAs/SM,
 * 5 TMA bulk-copy pipeline (ring for 2 CTAs/SM), 6 TMA (ring for 1 CTA/SM),
 * 7 / 8 = 5 / 6 with bulk-store drains (no thread-issued global stores),
 * 9 / 10 / 12 = a 2- / 4- / 5-stage ring, 11 = 5 stages with bulk-store
 * drains -- 5..12 need 8-element-aligned segments;
 * grid 0 = SMs x resident CTAs (persistent). */
int amsp_engine_tune(amsp_engine_t* e, int variant, int grid);
/* All-gather implementation: grid > 0 = the SM (LDG/STG) kernel with that
 * many CTAs, 0 = the SM kernel with 4 CTAs per SM, -1 = copy engines (one
 * peer-to-local DMA per P-group member), -2 = the TMA bulk-copy kernel
 * (single-warp CTAs; needs 8-element-aligned P slices). */
int amsp_engine_tune_gather(amsp_engine_t* e, int grid);
/* Bracket every fused launch with CUDA events on the step's stream (enable
 * != 0), then read the summed kernel time of the launches since enabling
 * (synchronous; resets the count). */
int amsp_engine_time_kernel(amsp_engine_t* e, int enable);
int amsp_engine_kernel_ms(amsp_engine_t* e, double* total_ms, int* launches);
/* Same for the all-gather phase of each step (s_p > 1). */
int amsp_engine_gather_ms(amsp_engine_t* e, double* total_ms, int* steps);
/* Same for the micro-batch accumulation kernels (amsp_engine_accumulate). */
int amsp_engine_accum_ms(amsp_engine_t* e, double* total_ms, int* launches);
/* NVLink peer-read probe (bench): every rank pulls `bytes` from its peers'
 * gradient buffers into local scratch, after a cross-GPU barrier, `iters`
 * times; pattern 0 = ring (all from rank+1), 1 = all-to-all (an equal share
 * from every peer, 512-byte warp chunks interleaved -- the fused reduce's
 * pattern). *ms_per_iter = this rank's time per pull of `bytes`. */
int amsp_engine_nvlink_probe(amsp_engine_t* e, uint64_t bytes, int pattern, int iters,
                             double* ms_per_iter);
/* Number of kernels this engine launched so far. */
int amsp_engine_launch_count(const amsp_engine_t* e, uint64_t* n);
void amsp_engine_destroy(amsp_engine_t* e);

/* ------------------------------------------------------------ scheduler */
/* Overlap scheduler (north-star item 4): replays the reference's one-step
 * event graph (build_schedule, overlap_sim.cpp:442-457) on three CUDA
 * streams of the engine's GPU. Compute events run a compute stand-in for
 * their planned duration; AG / RS / AR-bucket events run the engine's NVLink
 * gather / barrier + pull-reduce; after the graph: barrier, AdamW + bf16
 * push to the OS-group owners, barrier. The engine's tensors must be the
 * LLaMA layout [embed, L x K modules, final norm, lm_head] of `model`. */
typedef struct amsp_sched amsp_sched_t;

typedef struct {
  amsp_model_t model;           /* micro_batch_count = the engine's M */
  amsp_cost_config_t cost;      /* bucket size U */
  amsp_sim_config_t sim;        /* tier, recompute, streams, compute times */
  int comm_ctas;                /* CTAs per communication kernel (0 = 128) */
  int compute_ctas;             /* CTAs of the compute stand-in (0 = SMs) */
  double time_scale;            /* multiplies compute durations (0 = 1) */
  int optimizer_overlap;        /* 0: AdamW + push after the step barrier
                                   (the paper's placement); 1: per module /
                                   bucket inside backward (see sched.cpp) */
  int compute_mode;             /* 0: timed stand-ins of the graph's
                                   durations; 1: cuBLAS bf16 GEMMs of each
                                   linear module's true shape (fwd / dgrad /
                                   wgrad into the real gradient buffer),
                                   reading the gathered weights */
  int tokens;                   /* GEMM rows T (0 = micro_batch * seq_len) */
  int gemm_sm_margin;           /* SMs withheld from GEMMs for the concurrent
                                   communication / optimizer kernels (cuBLAS
                                   SM-count target = SMs - margin) */
  int gather_mode;              /* all-gathers: 0 = SM kernel (NVLink pulls,
                                   tile-interleaved sources); 1 = copy
                                   engines (peer cudaMemcpyAsync, no SMs);
                                   2 = TMA bulk-copy kernel (single-warp
                                   CTAs, 8-element-aligned P slices) */
  int bc_mode;                  /* updated-parameter broadcast: 0 = auto:
                                   mirrored when the graph leads with the
                                   previous step's BroadcastShard events
                                   (tier ag_rs_ar_bc, s_p = 1, k > 1;
                                   overlap_sim.cpp:152-159) -- the optimizer
                                   writes only local params and the next
                                   step's BC events pull them by copy engine,
                                   gating the forward layer blocks;
                                   1 = push inside the optimizer kernels */
  int optimizer_variant;        /* kernel of the optimizer updates that run
                                   inside backward (optimizer_overlap = 1):
                                   0 = LDG fused kernel (small smem, co-resides
                                   with GEMM CTAs); 5 / 6 = the TMA bulk-copy
                                   pipeline (2 / 1 CTAs per SM; 8-element-aligned
                                   segments) on comm_ctas SMs, meant with
                                   gemm_sm_margin = comm_ctas */
  int reduce_mode;              /* gradient reduce inside the step (W > 1):
                                   0 = SM kernels pull peers' bf16 gradients
                                   over NVLink; 1 = copy engines stage every
                                   rank's gradients of the event's owned
                                   pieces into local HBM after the barrier,
                                   then the same kernels reduce locally (the
                                   NVLink traffic leaves the SMs to compute) */
  int grad_source;              /* gradients of the stand-in backward: 0 = the
                                   caller's (already in the gradient buffer;
                                   M must be 1); 1 = every grad-weight event
                                   writes its tensors' synthetic gradient of
                                   its micro-batch (the oracle definition),
                                   so gradients appear DURING the step and
                                   the per-bucket barriers order real data */
} amsp_sched_config_t;

typedef struct {
  int n_events, n_compute, n_gather, n_reduce, n_buckets, n_barriers, stream_count;
  double predicted_step_s;      /* simulate_step() of the same graph */
  double predicted_compute_s;   /* compute-stream busy time */
  int mirrored_bc;              /* 1: parameters of other OS owners arrive in
                                   the next step's BC events (call
                                   amsp_sched_flush after the last step) */
  uint64_t grad_ring_need;      /* gradient-ring engines: the smallest ring
                                   (bf16 elements) this schedule runs in */
} amsp_sched_info_t;

int amsp_sched_create(amsp_engine_t* e, const amsp_sched_config_t* cfg,
                      const amsp_profile_t* profile, amsp_sched_t** out);
int amsp_sched_info(const amsp_sched_t* s, amsp_sched_info_t* info);
/* Which graph event uses barrier `id` (diagnostics for a barrier timeout):
 * *event = the event index (-1: a step-level barrier), *role = 0 pre-reduce,
 * 1 second (optimizer) barrier, 2 release, 3 head accumulation, 4 head
 * release, 5 end-of-step A, 6 end-of-step B, 7 flush; *mb = its micro-batch.
 * Returns 1 (invalid) for an id no event uses. */
int amsp_sched_barrier_owner(const amsp_sched_t* s, int id, int* event, int* role, int* mb);
/* One step. mode 1 = the full step; 0 = compute only; 2 = compute + the
 * optimizer's local HBM work without any NVLink traffic (a timing proxy for
 * the exposed-communication baseline, not a valid update). stream = the
 * compute stream (NULL: engine's). */
int amsp_sched_step(amsp_sched_t* s, int step, void* stream, int mode);
/* Measured trace: with tracing on, every graph event of a step
 * is bracketed by CUDA events; amsp_sched_trace renders the last traced step
 * with the reference's render_trace (overlap_sim.cpp:560-577), so measured
 * and predicted (amsp_sched_predicted_trace) traces share one TEF schema
 * and event names. *step_ms = measured span of the graph. */
/* Mirrored broadcast only (info.mirrored_bc): pull every OS owner's updated
 * parameters now, so params are complete on every rank after the last step,
 * then a cross-GPU barrier. A no-op otherwise. Call on every rank. */
int amsp_sched_flush(amsp_sched_t* s, void* stream);
int amsp_sched_enable_trace(amsp_sched_t* s, int on);
int amsp_sched_trace(amsp_sched_t* s, char* buf, size_t cap, size_t* needed, double* step_ms);
int amsp_sched_predicted_trace(const amsp_sched_t* s, char* buf, size_t cap, size_t* needed);
void amsp_sched_destroy(amsp_sched_t* s);

/* ------------------------------------------------------------ kernels */
/* Raw launchers (device pointers + cudaStream_t passed as void*). */

/* dst[k] = grad(seed, step, rank, start+k) as bf16, k < n */
int amsp_k_synth_grad(void* dst_bf16, uint64_t start, uint64_t n, uint64_t seed,
                      int step, int rank, void* stream);
/* Compute stand-in: `ctas` CTAs each keep issuing FMAs for `ns` nanoseconds
 * (the overlap scheduler's timed compute; tests use it to delay a stream). */
int amsp_k_spin(int ctas, uint64_t ns, void* stream);
/* Plain fused AdamW on a contiguous shard: fp32 or bf16 grads (grad_is_bf16),
 * grad_scale applied, bf16 copy of the updated master written to param_out
 * (may be NULL). */
int amsp_k_adamw(const void* grad, int grad_is_bf16, float* master, float* m,
                 float* v, void* param_out_bf16, uint64_t n, int step,
                 double lr, double beta1, double beta2, double eps,
                 double weight_decay, double grad_scale, void* stream);
/* bf16 -> fp32 upcast with scale (the NCCL-path gradient epilogue). */
int amsp_k_upcast_scale(const void* src_bf16, float* dst, uint64_t n, float scale,
                        void* stream);

/* Reduce-scatter epilogue (north-star item 1) over plain pointers:
 * dst[k] = (sum_{r<nsrc} bf16 srcs[r][offset+k]) * scale in fixed rank order
 * (the fused kernel's rounding sequence). srcs may be cudaIpc peer pointers
 * (the RS pull) or local buffers; 1 <= nsrc <= 8. */
int amsp_k_rs_upcast_scale(const void* const* srcs_bf16, int nsrc, uint64_t offset,
                           float* dst, uint64_t n, float scale, void* stream);
/* All-gather epilogue (north-star item 3): bf16(src[k]) stored into
 * dsts[d][dst_offset + k] for every destination d < ndst (local or peer
 * parameter buffers); 1 <= ndst <= 8. */
int amsp_k_ag_downcast(const float* src, uint64_t n, void* const* dsts_bf16, int ndst,
                       uint64_t dst_offset, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AMSP_C_H_ */
