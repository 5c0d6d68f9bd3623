// Overlap scheduler: executes the reference's one-step event graph
// (shardplan::build_schedule, overlap_sim.cpp:122-457 — Fig 7(a)(b)(c) and
// the Table V tiers) on real CUDA streams of one B200, with the AMSP data
// plane doing the communication (north-star item 4).
//
//   stream 0 (caller's)  compute events -> compute stand-in kernels whose
//                        durations are the graph's (FLOPs / peak x eff, or
//                        a measured per-module table)
//   stream 1             AllGather (l, i)     -> NVLink gather of tensor (l,i)
//                        ReduceScatter (l, i) -> cross-GPU barrier + pull-
//                                                reduce of tensor (l,i)
//   stream 2             AllReduceBucket b    -> barrier + pull-reduce of
//                                                bucket b's owned elements
//                        BroadcastShard j     -> mirrored broadcast (below)
//                                                or a marker
//   after the graph      barrier -> update of whatever is left -> barrier
//
// Cross-stream dependencies are cudaEvents exactly as in Event::depends_on;
// events on one stream keep graph order. Gradient buckets are the graph's
// own cuts: the backward-ordered gradient byte stream (head first, then
// layers L-1..0, modules K-1..0) cut every s_p * U bytes (overlap_sim.cpp:
// 285-312), mapped onto the flat parameter vector.
//
// Optimizer placement (`optimizer_overlap`):
//   0 — the paper's barrier semantics (overlap_sim.cpp:166-174, PAPER.md:
//       299-312): reduces land in an fp32 shard during backward; AdamW +
//       bf16 push to the OS-group owners run once after the step's barrier.
//   1 — the optimizer moves into the backward pass: s_p > 1 runs the fused
//       reduce + AdamW + push per module right after its reduce-scatter
//       barrier (every rank has passed that module's gradient, so no rank
//       reads its parameters again this step); s_p = 1 runs AdamW + push per
//       bucket after a second barrier that certifies every rank finished the
//       bucket's grad-input (the last reader of those replicated params).
// Either way the arithmetic is bit-equal to the fused kernel and the oracle.
//
// Parameter broadcast (`bc_mode`):
//   mirrored (default when the graph leads with BroadcastShard events, i.e.
//       tier ag_rs_ar_bc with s_p = 1 and k = s_os/s_p > 1; overlap_sim.cpp:
//       152-159) — the optimizer kernels write the updated bf16 shard only
//       into this rank's own parameters; BroadcastShard j of the NEXT step
//       pulls, with copy-engine DMAs on the AR/BC stream, every parameter
//       the graph gates behind it (layer block j: layers with
//       ceil((l+1) n / L) - 1 = j, the head in the last block) from its OS
//       owner. Layer l's forward waits on its block exactly as in the graph,
//       so the broadcast overlaps the next forward instead of extending this
//       step's tail. After the last step, amsp_sched_flush pulls the rest.
//   push — the optimizer kernels store the bf16 shard into every OS-group
//       member directly (NVLink stores inside the update); BroadcastShard is
//       a marker.
#include <cmath>
#include <cstdlib>

#include "blas.h"
#include "compute.h"
#include "engine_impl.h"
#include "../convert.h"

namespace {

enum class Work { Compute, Gather, Reduce, ReduceAdam, Accumulate, Broadcast, Marker };

// One pull of the mirrored broadcast: params[dst, dst+len) from `owner`,
// part of layer `layer` (the head tensors: layer = L).
struct BcCopy {
  std::uint64_t dst = 0, len = 0;
  int owner = 0;
  int layer = 0;
};

// Real-compute mode: a compute event of a linear module (or the LM head) is
// a cuBLAS bf16 GEMM of its true shape over T tokens; a norm module's events
// are RMSNorm kernels (forward, input grad, weight grad into the gradient
// buffer). The attention core (QK^T, causal softmax, PV and their
// backward: 12*B*S^2*H FLOPs per layer, the reference's flops_coeff_attn,
// overlap_sim.cpp:97-110) runs inside the o-projection's forward (before
// its GEMM) and grad-input (after its GEMM) events, where the data flow of
// a LLaMA layer puts it.
enum class Gemm { None, Fwd, DGrad, WGrad, NormFwd, NormDGrad, NormWGrad };

struct EventWork {
  Work kind = Work::Marker;
  int stream = 0;
  int tensor = -1;
  Gemm gemm = Gemm::None;
  int g_in = 0, g_out = 0;
  // ZeRO++ (engine s2 > 1): the step's first all-gather of a tensor reads
  // the P shards and refreshes this rank's secondary slice; every later one
  // (backward, recompute, later micro-batches) reads the secondary group
  bool secondary = false, refresh = false;
  bool attention = false;  // attention core before (Fwd) / after (DGrad) the GEMM
  int barrier = -1;
  int seg_begin = 0, nseg = 0, ntiles = 0;
  unsigned long long ns = 0;
  bool record = false;
  // s_p = 1 with optimizer overlap: AdamW + push of this bucket after the
  // local grad-input event `after_event` and barrier `barrier2`.
  bool adam_after = false;
  int after_event = -1;
  int barrier2 = -1;
  // Single rank (no AllReduce buckets in the graph): fused update of the
  // bucket completed by this grad-input event, on the AR/BC stream.
  int post_begin = 0, post_nseg = 0, post_ntiles = 0;
  int bc = -1;  // Work::Broadcast: index into amsp_sched::bc_copies
  // Micro-batches (M > 1). mb = the event's micro-batch. A grad-weight event
  // may synthesize its tensors' gradients (grad_source = 1), accumulating in
  // place when s_g = 1, and first waits until every rank has pulled the
  // previous micro-batch's gradients of those tensors (release events of the
  // accumulations that covered them).
  int mb = 0;
  std::vector<int> synth_tensors;
  bool accum_in_place = false;
  std::vector<int> wait_release;
  // Work::Accumulate (non-last micro-batch, s_g > 1): barrier, fold the
  // pieces [seg_begin, +nseg) of the accumulation table into the G shard,
  // barrier `rel_barrier`, record this event's release event.
  int rel_barrier = -1;
  // s_g = s_p > 1: the head tensors have no ReduceScatter event in the graph
  // (domain.hpp:69-71), so the head grad-weight event of a non-last
  // micro-batch accumulates them on the AG/RS stream (index into
  // amsp_sched::head_acc, -1 = none).
  int head_acc = -1;
  // Tensors whose raw gradients this event's kernels read on some rank
  // (Accumulate / Reduce / ReduceAdam), for the gradient ring's lifetimes;
  // rel_barrier >= 0 on a Reduce / ReduceAdam: a release barrier + event
  // after the reduce (ring mode), like the accumulations'.
  std::vector<int> reads;
};

struct Table {
  int begin = 0, nseg = 0, ntiles = 0;
};

struct HeadAccum {
  Table t;
  int barrier = -1, rel_barrier = -1;
  int rel = -1;  // index of its release event in amsp_sched::rel_events
  int mb = 0;
  std::vector<int> reads;  // tensors whose gradients it pulls
};

constexpr int kFirstSchedBarrier = 16;  // ids 0..15 stay with the engine

}  // namespace

struct amsp_sched {
  amsp_engine* e = nullptr;
  shardplan::EventGraph graph;
  double predicted_step = 0.0, predicted_compute = 0.0;
  int comm_ctas = 128, compute_ctas = 148;
  double time_scale = 1.0;
  bool optimizer_overlap = true;
  int opt_variant = 0;  // kernel of the in-backward optimizer updates (cfg)
  std::vector<EventWork> work;
  int n_barriers = 0, end_a = 0, end_b = 0, n_buckets = 0, n_gather = 0, n_reduce = 0,
      n_compute = 0;
  Table resid, pending;  // end of step: fused update / AdamW-from-reduced update
  // Mirrored broadcast: per BroadcastShard event, the pulls it performs.
  bool mirror = false;
  std::vector<std::vector<BcCopy>> bc_copies;  // per BC event, in layer order
  std::vector<cudaEvent_t> layer_ev;          // per layer (+ head): pulls landed
  int flush_barrier = 0;
  int param_dsts(uint16_t** dsts) const {
    if (mirror) {
      dsts[0] = e->params_of(e->rank);
      return 1;
    }
    const int n = static_cast<int>(e->dst_members.size());
    for (int d = 0; d < n; ++d) dsts[d] = e->params_of(e->dst_members[d]);
    return n;
  }
  // BC event j: the pulls of its layer block, layer by layer, recording each
  // layer's event so that layer l's forward waits for its own parameters
  // only (a refinement of the graph's block gate: same data dependency).
  void broadcast(int j, cudaStream_t st) {
    uint16_t* mine = e->params_of(e->rank);
    const auto& cs = bc_copies[static_cast<std::size_t>(j)];
    for (std::size_t i = 0; i < cs.size(); ++i) {
      const BcCopy& c = cs[i];
      ck(cudaMemcpyAsync(mine + c.dst, e->params_of(c.owner) + c.dst, c.len * 2,
                         cudaMemcpyDeviceToDevice, st),
         "broadcast DMA");
      if (i + 1 == cs.size() || cs[i + 1].layer != c.layer)
        ck(cudaEventRecord(layer_ev[static_cast<std::size_t>(c.layer)], st), "event record");
    }
  }
  amsp::Seg* d_rsegs = nullptr;
  amsp::CopySeg* d_tcopy = nullptr;
  amsp::CopySeg* d_tcopy2 = nullptr;  // ZeRO++ secondary slices
  // Micro-batch accumulation tables (Seg::os = G-shard accumulator offset),
  // the release event of every Work::Accumulate event, and the head pieces.
  amsp::Seg* d_asegs = nullptr;
  std::vector<cudaEvent_t> rel_events;
  std::vector<HeadAccum> head_acc;
  std::vector<cudaEvent_t> head_done;  // head grad-weight finished (per head_acc)
  int grad_source = 0, micro = 1;

  void accumulate(const Table& t, bool first, cudaStream_t s) {
    if (t.ntiles == 0) return;
    amsp::AccumArgs a{};
    a.segs = d_asegs + t.begin;
    a.nseg = t.nseg;
    a.ntiles = t.ntiles;
    a.nsrc = static_cast<int>(e->acc_sources.size());
    for (int q = 0; q < a.nsrc; ++q) a.grads[q] = e->grads_of(e->acc_sources[q]);
    a.acc = e->acc_of(e->rank);
    a.first = first ? 1 : 0;
    ck(amsp::launch_accumulate(a, comm_ctas, s), "sched accumulate");
    ++e->launches;
  }

  // Backward stand-in's gradient output: micro-batch mb of tensor t.
  // Where tensor t's gradient of micro-batch mb lives in the gradient
  // buffer: its flat offset, or its slot in the gradient ring.
  std::vector<std::vector<std::uint64_t>> ring_off;  // [mb][t] (ring mode)
  std::uint64_t ring_need = 0;
  std::uint64_t grad_offset(int t, int mb) const {
    return e->ring ? ring_off[static_cast<std::size_t>(mb)][static_cast<std::size_t>(t)]
                   : e->pmap.tensor_offset[static_cast<std::size_t>(t)];
  }

  void synth(int t, int mb, bool in_place, cudaStream_t s) {
    const std::uint64_t a = e->pmap.tensor_offset[static_cast<std::size_t>(t)];
    ck(amsp::launch_synth_grad(e->grads_of(e->rank) + grad_offset(t, mb), a, e->tensor_sizes[t],
                               e->cfg.seed, cur_step, e->rank, s, mb, in_place),
       "synth grads");
    ++e->launches;
  }
  int cur_step = 1;
  // Copy-engine staged reduce (reduce_mode 1): after the barrier, every
  // rank's bf16 gradients of the event's owned pieces are DMA'd (peer ->
  // local, rotated start) into stage[r * stage_slot + ...]; the reduce /
  // fused kernel then reads only local HBM through d_ssegs, a copy of the
  // event's table whose `flat` is the staging offset. NVLink traffic moves
  // off the SMs, which stay with the GEMMs.
  bool reduce_dma = false;
  amsp::Seg* d_ssegs = nullptr;
  std::vector<amsp::Seg> h_rsegs, h_ssegs;
  uint16_t* stage = nullptr;
  std::uint64_t stage_slot = 0;

  void stage_in(const Table& t, cudaStream_t st) {
    for (int i = 0; i < e->world; ++i) {
      const int r = (e->rank + 1 + i) % e->world;
      uint16_t* dst = stage + static_cast<std::uint64_t>(r) * stage_slot;
      const uint16_t* src = e->grads_of(r);
      int j = t.begin;
      while (j < t.begin + t.nseg) {  // coalesce pieces contiguous in both spaces
        const std::uint64_t flat = h_rsegs[j].flat, off = h_ssegs[j].flat;
        std::uint64_t len = h_rsegs[j].len;
        ++j;
        while (j < t.begin + t.nseg && h_rsegs[j].flat == flat + len &&
               h_ssegs[j].flat == off + len)
          len += h_rsegs[j++].len;
        ck(cudaMemcpyAsync(dst + off, src + flat, len * 2, cudaMemcpyDeviceToDevice, st),
           "staged reduce DMA");
      }
    }
  }
  float* red = nullptr;
  // Real-compute mode buffers: activations / output-grads / outputs of
  // T x max-dim bf16, a 3-layer ring of gathered module weights (s_p > 1)
  // and a head-weight scratch (the head is never gathered by the graph).
  bool gemm_mode = false;
  bool gather_dma = false;  // all-gathers on the copy engines
  bool gather_tma = false;  // all-gathers by the bulk-copy (TMA) kernel
  int tokens = 0, layers_k = 1, gemm_sm_target = 0;
  uint16_t* act = nullptr;
  uint16_t* dout = nullptr;
  uint16_t* yout = nullptr;
  uint16_t* ring = nullptr;
  uint16_t* head_w = nullptr;
  std::uint64_t ring_slot = 0;
  // attention core: seq_len S, heads x head_dim, sequences per micro-batch;
  // probabilities P and their gradient dS, [heads, S, S] bf16 each
  int attn_s = 0, attn_heads = 0, attn_dim = 0, attn_seqs = 0, hidden = 0;
  uint16_t* probs = nullptr;
  uint16_t* dprobs = nullptr;
  float* norm_acc = nullptr;  // fp32 [H] scratch of the norm weight gradients

  void attention_fwd(cudaStream_t st) {
    amsp::Blas& blas = amsp::Blas::instance();
    const int S = attn_s, d = attn_dim, nh = attn_heads, H = hidden;
    const long long SS = static_cast<long long>(S) * S;
    const float scale = 1.0f / std::sqrt(static_cast<float>(d));
    for (int b = 0; b < attn_seqs; ++b) {
      const long long o = static_cast<long long>(b) * S * H;
      // scores_h = Q_h K_h^T  (Q = K = V = the activation buffer's head slices)
      blas.bgemm(st, false, true, S, S, d, act + o, H, d, act + o, H, d, probs, S, SS, nh);
      ck(amsp::launch_softmax_rows(probs, static_cast<long long>(nh) * S, S, S, scale, st),
         "attention softmax");
      // O_h = P_h V_h
      blas.bgemm(st, false, false, S, d, S, probs, S, SS, act + o, H, d, yout + o, H, d, nh);
      e->launches += 3;
    }
  }

  void attention_bwd(cudaStream_t st) {
    amsp::Blas& blas = amsp::Blas::instance();
    const int S = attn_s, d = attn_dim, nh = attn_heads, H = hidden;
    const long long SS = static_cast<long long>(S) * S;
    const float scale = 1.0f / std::sqrt(static_cast<float>(d));
    for (int b = 0; b < attn_seqs; ++b) {
      const long long o = static_cast<long long>(b) * S * H;
      // dP_h = dO_h V_h^T ; dS = softmax backward ; dV = P^T dO ; dQ = dS K ; dK = dS^T Q
      blas.bgemm(st, false, true, S, S, d, dout + o, H, d, act + o, H, d, dprobs, S, SS, nh);
      ck(amsp::launch_softmax_bwd_rows(probs, dprobs, static_cast<long long>(nh) * S, S, scale,
                                       st),
         "attention softmax backward");
      blas.bgemm(st, true, false, S, d, S, probs, S, SS, dout + o, H, d, yout + o, H, d, nh);
      blas.bgemm(st, false, false, S, d, S, dprobs, S, SS, act + o, H, d, yout + o, H, d, nh);
      blas.bgemm(st, true, false, S, d, S, dprobs, S, SS, act + o, H, d, yout + o, H, d, nh);
      e->launches += 5;
    }
  }

  uint16_t* gather_dst(int t) const {
    if (!gemm_mode) return e->slots[t & 1];
    const int l = (t - 1) / layers_k, i = (t - 1) % layers_k;
    return ring + static_cast<std::uint64_t>((l % 3) * layers_k + i) * ring_slot;
  }

  const uint16_t* weight_of(int t) const {
    if (t < 0) return head_w ? head_w : e->params_of(e->rank) + e->pmap.tensor_offset.back();
    if (e->sp > 1) return gather_dst(t);
    return e->params_of(e->rank) + e->pmap.tensor_offset[t];
  }

  void compute(const EventWork& w, cudaStream_t st) {
    if (w.gemm == Gemm::None) {
      ck(amsp::launch_spin(compute_ctas, w.ns, st), "compute stand-in");
      ++e->launches;
      return;
    }
    amsp::Blas& blas = amsp::Blas::instance();
    blas.set_sm_target(gemm_sm_target);
    const int t = w.tensor;  // -1: LM head
    const uint16_t* wt = weight_of(t);
    switch (w.gemm) {
      case Gemm::Fwd:
        if (w.attention) attention_fwd(st);
        blas.linear_fwd(st, act, wt, yout, tokens, w.g_in, w.g_out);
        break;
      case Gemm::DGrad:
        blas.linear_dgrad(st, dout, wt, yout, tokens, w.g_in, w.g_out);
        if (w.attention) attention_bwd(st);
        break;
      case Gemm::NormFwd:
        ck(amsp::launch_rmsnorm_fwd(act, wt, yout, tokens, hidden, st), "rmsnorm");
        break;
      case Gemm::NormDGrad:
        ck(amsp::launch_rmsnorm_dgrad(act, wt, dout, yout, tokens, hidden, st), "rmsnorm dgrad");
        break;
      case Gemm::NormWGrad:
        ck(amsp::launch_rmsnorm_wgrad(act, dout, norm_acc,
                                      e->grads_of(e->rank) + grad_offset(t, w.mb), tokens,
                                      hidden, w.accum_in_place, st),
           "rmsnorm wgrad");
        ++e->launches;
        break;
      case Gemm::WGrad: {
        const std::size_t ti = t < 0 ? e->tensor_sizes.size() - 1 : static_cast<std::size_t>(t);
        blas.linear_wgrad(st, dout, act,
                          e->grads_of(e->rank) + grad_offset(static_cast<int>(ti), w.mb), tokens,
                          w.g_in, w.g_out, w.accum_in_place);
        break;
      }
      case Gemm::None:
        break;
    }
    ++e->launches;
  }
  cudaStream_t comm[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> events;
  cudaEvent_t start_ev = nullptr, join_ev[2] = {nullptr, nullptr};
  uint32_t epoch = 0;
  amsp::AdamScalars scalars{};
  // Measured trace: timing events around every graph event of the last step.
  bool tracing = false;
  cudaEvent_t trace_origin = nullptr;
  std::vector<cudaEvent_t> t_begin, t_end;

  void enable_trace(bool on) {
    tracing = on;
    if (!on || !t_begin.empty()) return;
    ck(cudaEventCreate(&trace_origin), "event");
    t_begin.resize(graph.events.size());
    t_end.resize(graph.events.size());
    for (auto& ev : t_begin) ck(cudaEventCreate(&ev), "event");
    for (auto& ev : t_end) ck(cudaEventCreate(&ev), "event");
  }

  // The last traced step as a shardplan::Timeline, rendered by the same
  // render_trace as the simulator (identical TEF schema and names).
  std::string measured_trace(double* step_ms) {
    if (t_begin.empty()) throw Error("sched: tracing was never enabled");
    shardplan::Timeline tl;
    tl.events = graph.events;
    tl.streams.resize(graph.stream_count);
    for (std::size_t i = 0; i < graph.events.size(); ++i) {
      ck(cudaEventSynchronize(t_end[i]), "event sync");
      float a = 0.0f, b = 0.0f;
      ck(cudaEventElapsedTime(&a, trace_origin, t_begin[i]), "event elapsed");
      ck(cudaEventElapsedTime(&b, trace_origin, t_end[i]), "event elapsed");
      tl.streams[graph.events[i].stream].push_back(
          {static_cast<int>(i), a * 1e-3, std::max(a, b) * 1e-3});
    }
    tl.busy.assign(graph.stream_count, 0.0);
    for (int k = 0; k < graph.stream_count; ++k) {
      auto& v = tl.streams[k];
      std::stable_sort(v.begin(), v.end(), [](const shardplan::ScheduledEvent& x,
                                              const shardplan::ScheduledEvent& y) {
        return x.start < y.start;
      });
      for (const auto& se : v) {
        tl.busy[k] += se.end - se.start;
        tl.step_time = std::max(tl.step_time, se.end);
      }
    }
    tl.idle.resize(graph.stream_count);
    for (int k = 0; k < graph.stream_count; ++k) tl.idle[k] = tl.step_time - tl.busy[k];
    if (step_ms) *step_ms = tl.step_time * 1e3;
    return shardplan::render_trace(tl);
  }

  ~amsp_sched() {
    if (e) cudaSetDevice(e->cfg.device);
    cudaDeviceSynchronize();
    for (auto* v : {&events, &t_begin, &t_end})
      for (auto ev : *v)
        if (ev) cudaEventDestroy(ev);
    if (trace_origin) cudaEventDestroy(trace_origin);
    if (start_ev) cudaEventDestroy(start_ev);
    for (auto ev : join_ev)
      if (ev) cudaEventDestroy(ev);
    for (auto* v : {&layer_ev, &rel_events, &head_done})
      for (auto ev : *v)
        if (ev) cudaEventDestroy(ev);
    for (auto s : comm)
      if (s) cudaStreamDestroy(s);
    cudaFree(d_rsegs);
    cudaFree(d_tcopy);
    cudaFree(d_tcopy2);
    cudaFree(d_asegs);
    cudaFree(d_ssegs);
    cudaFree(stage);
    cudaFree(red);
    for (void* p : {static_cast<void*>(act), static_cast<void*>(dout), static_cast<void*>(yout),
                    static_cast<void*>(ring), static_cast<void*>(head_w),
                    static_cast<void*>(probs), static_cast<void*>(dprobs),
                    static_cast<void*>(norm_acc)})
      cudaFree(p);
    cudaGetLastError();  // teardown must not leave a sticky error for the next call
  }

  cudaStream_t stream_of(int s, cudaStream_t main) const {
    return s == 0 ? main : comm[s == 1 ? 0 : 1];
  }

  void barrier(int id, cudaStream_t s) {
    if (!e->synced()) return;
    ck(amsp::launch_barrier(e->d_peer_flags, e->world, e->rank, id, epoch, e->err, s),
       "sched barrier");
    ++e->launches;
  }

  void reduce(const Table& t, int grid, cudaStream_t s) {
    if (t.ntiles == 0) return;
    amsp::ReduceArgs a{};
    a.segs = (reduce_dma ? d_ssegs : d_rsegs) + t.begin;
    a.nseg = t.nseg;
    a.ntiles = t.ntiles;
    if (reduce_dma) stage_in(t, s);
    for (int r = 0; r < e->world; ++r)
      a.grads[r] = reduce_dma ? stage + static_cast<std::uint64_t>(r) * stage_slot
                              : e->grads_of(r);
    a.red = red;
    a.scale = static_cast<float>(e->grad_scale());
    if (e->staged) e->set_acc(a.acc, &a.nacc, &a.acc_by_dst);
    ck(amsp::launch_reduce(a, e->world, grid, s), "sched reduce");
    ++e->launches;
  }

  void adam_push(const Table& t, int grid, cudaStream_t s) {
    if (t.ntiles == 0) return;
    amsp::AdamPushArgs a{};
    a.segs = d_rsegs + t.begin;
    a.nseg = t.nseg;
    a.ntiles = t.ntiles;
    a.red = red;
    a.ndst = param_dsts(a.dsts);
    a.master = e->master;
    a.exp_avg = e->exp_avg;
    a.exp_avg_sq = e->exp_avg_sq;
    a.s = scalars;
    a.fence_peers = e->synced() ? 1 : 0;
    ck(amsp::launch_adam_push(a, grid, s), "adam push");
    ++e->launches;
  }

  void fused(const Table& t, int grid, cudaStream_t s, int variant = 0, bool staged = false) {
    if (t.ntiles == 0) return;
    amsp::FusedArgs a{};
    staged = staged && reduce_dma;
    a.segs = (staged ? d_ssegs : d_rsegs) + t.begin;
    a.nseg = t.nseg;
    a.ntiles = t.ntiles;
    if (staged) stage_in(t, s);
    for (int r = 0; r < e->world; ++r)
      a.grads[r] = staged ? stage + static_cast<std::uint64_t>(r) * stage_slot : e->grads_of(r);
    a.ndst = param_dsts(a.dsts);
    a.master = e->master;
    a.exp_avg = e->exp_avg;
    a.exp_avg_sq = e->exp_avg_sq;
    a.s = scalars;
    a.stats = nullptr;
    a.fence_peers = e->synced() ? 1 : 0;
    if (e->staged) e->set_acc(a.acc, &a.nacc, &a.acc_by_dst);
    ck(amsp::launch_fused_step(a, e->world, std::max(1, std::min(t.ntiles, grid)), variant, s),
       "sched fused");
    ++e->launches;
  }

  // The optimizer work of a table without communication (mode 2 baseline):
  // own gradients (W = 1 sum), own parameters only.
  void local_fused(const Table& t, int grid, cudaStream_t s, int variant = 0) {
    if (t.ntiles == 0) return;
    amsp::FusedArgs a{};
    a.segs = d_rsegs + t.begin;
    a.nseg = t.nseg;
    a.ntiles = t.ntiles;
    a.grads[0] = e->grads_of(e->rank);
    a.ndst = 1;
    a.dsts[0] = e->params_of(e->rank);
    a.master = e->master;
    a.exp_avg = e->exp_avg;
    a.exp_avg_sq = e->exp_avg_sq;
    a.s = scalars;
    ck(amsp::launch_fused_step(a, 1, std::max(1, std::min(t.ntiles, grid)), variant, s),
       "local optimizer");
    ++e->launches;
  }

  void gather_tensor(int t, cudaStream_t s, bool secondary = false, bool refresh = false) {
    const int n = secondary ? e->s2 : e->sp;
    const amsp::MeshGroup& grp = secondary ? e->sec_group : e->p_group;
    const amsp::PShardMap& map = secondary ? e->smap : e->pmap;
    auto src_of = [&](int q) {
      return secondary ? e->sec_of(grp.members[q]) : e->params_of(grp.members[q]);
    };
    if (gather_dma) {
      // Copy-engine all-gather: one peer-to-local DMA per group member
      // (rotated start, like the SM kernel) — no SMs taken from compute.
      const std::uint64_t len = map.slice_len[t], src = map.pshard_offset[t];
      uint16_t* dst = gather_dst(t);
      for (int j = 0; j < n; ++j) {
        const int q = (grp.position + 1 + j) % n;
        ck(cudaMemcpyAsync(dst + static_cast<std::uint64_t>(q) * len, src_of(q) + src, len * 2,
                           cudaMemcpyDeviceToDevice, s),
           "gather DMA");
      }
      if (refresh) e->refresh_secondary_tensor(t, dst, s);
      return;
    }
    amsp::GatherArgs g{};
    if (refresh && e->sec_fused) {  // the secondary slice stored by the gather itself
      g.sec = e->sec_of(e->rank);
      g.s2 = e->s2;
      g.pos2 = e->sec_group.position;
    }
    g.segs = (secondary ? d_tcopy2 : d_tcopy) + t;
    g.nseg = 1;
    const unsigned long long len = map.slice_len[t];
    g.ntiles = static_cast<int>((len + amsp::kTile - 1) / amsp::kTile) * n;
    g.sp = n;
    g.rot = (grp.position + 1) % n;
    for (int q = 0; q < n; ++q) g.src[q] = src_of(q);
    g.dst = gather_dst(t);
    g.grid = comm_ctas;
    ck(gather_tma ? amsp::launch_gather_tma(g, s) : amsp::launch_gather(g, s), "sched gather");
    ++e->launches;
    if (refresh && !e->sec_fused) e->refresh_secondary_tensor(t, gather_dst(t), s);
  }

  void run(int step, cudaStream_t main, int mode) {
    const bool with_comm = mode == 1, local_optimizer = mode == 2;
    if (step < 1) throw Error("sched: step index must be >= 1");
    e->require_peers();
    // Barrier ids >= kFirstSchedBarrier live in the engine's flag block and
    // are reused by every scheduler created on this engine: the epoch must
    // keep growing across schedulers, so it is the engine's counter.
    epoch = ++e->sched_epoch;
    cur_step = step;
    scalars = amsp::make_adam_scalars(e->cfg.lr, e->cfg.beta1, e->cfg.beta2, e->cfg.eps,
                                      e->cfg.weight_decay, step, e->grad_scale());
    ck(cudaEventRecord(start_ev, main), "event record");
    if (tracing) ck(cudaEventRecord(trace_origin, main), "event record");
    for (auto s : comm) ck(cudaStreamWaitEvent(s, start_ev, 0), "stream wait");
    const auto& evs = graph.events;
    for (std::size_t i = 0; i < evs.size(); ++i) {
      const EventWork& w = work[i];
      cudaStream_t st = stream_of(w.stream, main);
      for (int d : evs[i].depends_on) {
        if (work[d].stream == w.stream || !work[d].record) continue;
        if (with_comm && work[d].kind == Work::Broadcast &&
            evs[i].kind == shardplan::EventKind::FwdCompute) {
          // mirrored broadcast: this layer's own pulls (head: index L)
          const int l = evs[i].layer < 0 ? static_cast<int>(layer_ev.size()) - 1 : evs[i].layer;
          ck(cudaStreamWaitEvent(st, layer_ev[static_cast<std::size_t>(l)], 0), "stream wait");
        } else {
          ck(cudaStreamWaitEvent(st, events[d], 0), "stream wait");
        }
      }
      if (with_comm)
        for (int j : w.wait_release) ck(cudaStreamWaitEvent(st, rel_events[j], 0), "stream wait");
      if (tracing) ck(cudaEventRecord(t_begin[i], st), "event record");
      const Table t{w.seg_begin, w.nseg, w.ntiles};
      switch (w.kind) {
        case Work::Compute:
          compute(w, st);
          for (int tt : w.synth_tensors) synth(tt, w.mb, w.accum_in_place, st);
          break;
        case Work::Accumulate:
          if (with_comm) {
            barrier(w.barrier, st);  // micro-batch w.mb of these pieces is complete everywhere
            accumulate(t, w.mb == 0, st);
            barrier(w.rel_barrier, st);  // every holder has pulled them
            ck(cudaEventRecord(rel_events[i], st), "event record");
          }
          break;
        case Work::Gather:
          if (with_comm) {
            // ZeRO++: every rank's secondary slices exist before the first
            // gather from the secondary group
            if (w.barrier >= 0) barrier(w.barrier, st);
            gather_tensor(w.tensor, st, w.secondary, w.refresh);
          }
          break;
        case Work::Reduce:
          if (with_comm) {
            barrier(w.barrier, st);
            reduce(t, comm_ctas, st);
            if (w.rel_barrier >= 0) {  // gradient ring: every rank has pulled these
              barrier(w.rel_barrier, st);
              ck(cudaEventRecord(rel_events[i], st), "event record");
            }
            if (w.adam_after) {
              ck(cudaStreamWaitEvent(st, events[w.after_event], 0), "stream wait");
              barrier(w.barrier2, st);
              adam_push(t, comm_ctas, st);
            }
          } else if (local_optimizer && w.adam_after) {
            ck(cudaStreamWaitEvent(st, events[w.after_event], 0), "stream wait");
            local_fused(t, comm_ctas, st, opt_variant);
          }
          break;
        case Work::ReduceAdam:
          if (with_comm) {
            barrier(w.barrier, st);
            fused(t, comm_ctas, st, opt_variant, true);
            if (w.rel_barrier >= 0) {  // gradient ring: every rank has pulled these
              barrier(w.rel_barrier, st);
              ck(cudaEventRecord(rel_events[i], st), "event record");
            }
          } else if (local_optimizer) {
            local_fused(t, comm_ctas, st, opt_variant);
          }
          break;
        case Work::Broadcast:
          if (with_comm) broadcast(w.bc, st);
          break;
        case Work::Marker:
          break;
      }
      if (tracing) ck(cudaEventRecord(t_end[i], st), "event record");
      if (w.record) ck(cudaEventRecord(events[i], st), "event record");
      if (with_comm && w.head_acc >= 0) {
        // s_g = s_p: the head's micro-batch gradient into the P-shard
        // accumulator (no ReduceScatter event carries it)
        const HeadAccum& h = head_acc[static_cast<std::size_t>(w.head_acc)];
        cudaEvent_t done = head_done[static_cast<std::size_t>(w.head_acc)];
        ck(cudaEventRecord(done, st), "event record");
        ck(cudaStreamWaitEvent(comm[0], done, 0), "stream wait");
        barrier(h.barrier, comm[0]);
        accumulate(h.t, w.mb == 0, comm[0]);
        barrier(h.rel_barrier, comm[0]);
        ck(cudaEventRecord(rel_events[static_cast<std::size_t>(h.rel)], comm[0]), "event record");
      }
      if ((with_comm || local_optimizer) && w.post_ntiles > 0) {
        ck(cudaStreamWaitEvent(comm[1], events[i], 0), "stream wait");
        const Table pt{w.post_begin, w.post_nseg, w.post_ntiles};
        if (with_comm)
          fused(pt, comm_ctas, comm[1], opt_variant);
        else
          local_fused(pt, comm_ctas, comm[1], opt_variant);
      }
    }
    for (int k = 0; k < 2; ++k) {
      ck(cudaEventRecord(join_ev[k], comm[k]), "event record");
      ck(cudaStreamWaitEvent(main, join_ev[k], 0), "stream wait");
    }
    if (local_optimizer) {
      // Baseline "compute + optimizer, no communication": every optimizer
      // update at the SAME place as in the full step (in backward or after
      // it), but from this rank's own gradients into its own parameters:
      // the optimizer's HBM and SM work without any NVLink traffic or
      // barrier (a timing proxy; the values are not the step's). So the
      // exposed communication t(full) - t(this) compares like with like.
      local_fused(resid, e->sms * amsp::fused_blocks_per_sm(1, tail_variant()), main,
                  tail_variant());
      local_fused(pending, e->sms * 2, main);
      return;
    }
    if (!with_comm) return;
    // Barrier semantics (overlap_sim.cpp:166-174): every gradient is reduced
    // on every rank before the remaining owners update and push.
    // The LDG kernel: measured 156.7 ms vs 160.4 ms with the TMA pipeline
    // for the 7B W=1 GEMM step (profiles/r01_final_n1.json vs
    // r01_bench_n1_f3.json) over the per-tensor residual table.
    const int tv = tail_variant();
    const int full_grid = e->sms * tail_blocks_per_sm(tv);
    barrier(end_a, main);
    fused(resid, full_grid, main, tv);
    // one wave of resident CTAs (occupancy of the push kernel)
    adam_push(pending, e->sms * amsp::adam_push_blocks_per_sm(), main);
    barrier(end_b, main);
  }

  // Kernel of the end-of-step update over the residual table: the engine's
  // auto TMA variant when every residual piece is 8-element aligned and no
  // accumulators are summed (those are on the LDG kernels), else LDG. With
  // real compute at W=1 the TMA tail gives a 241.7 ms step vs 248.6 ms
  // (profiles/r02_tail_ab_7b_w1.jsonl). Tuning hook AMSP_TAIL_VARIANT.
  bool resid_aligned = false;
  int tail_variant() const {
    static const int forced = [] {
      const char* x = std::getenv("AMSP_TAIL_VARIANT");
      return x ? std::atoi(x) : -1;
    }();
    if (forced >= 0) return forced;
    if (!resid_aligned || e->variant < 5) return 0;
    if (e->staged && amsp::tma_acc_blocks_per_sm(e->world, e->variant) == 0) return 0;
    return e->variant;
  }
  int tail_blocks_per_sm(int v) const {
    return (v >= 5 && e->staged) ? amsp::tma_acc_blocks_per_sm(e->world, v)
                                 : amsp::fused_blocks_per_sm(e->world, v);
  }

  // Mirrored broadcast: pull every block now (after the last step), then a
  // barrier so no owner updates its shard while a peer still reads it.
  void flush(cudaStream_t main) {
    if (!mirror) return;
    e->require_peers();
    epoch = ++e->sched_epoch;
    for (std::size_t j = 0; j < bc_copies.size(); ++j) broadcast(static_cast<int>(j), main);
    barrier(flush_barrier, main);
  }
};

namespace {

using FlatRange = std::pair<std::uint64_t, std::uint64_t>;  // [begin, end)

// Owned pieces of the flat ranges: (flat, os, dst, len) with a fresh tile
// prefix, appended to `out`.
Table owned_pieces(const amsp::ShardLayout& L, const std::vector<FlatRange>& ranges,
                   std::vector<amsp::Seg>& out) {
  Table t;
  t.begin = static_cast<int>(out.size());
  for (const auto& [a, b] : ranges) {
    // segments are ascending in flat order (pshard_layout builds them so)
    auto it = std::upper_bound(L.segs.begin(), L.segs.end(), a,
                               [](std::uint64_t x, const amsp::Segment& s) { return x < s.flat; });
    if (it != L.segs.begin()) --it;
    for (; it != L.segs.end() && it->flat < b; ++it) {
      const std::uint64_t lo = std::max(a, it->flat), hi = std::min(b, it->flat + it->len);
      if (lo >= hi) continue;
      const std::uint64_t off = lo - it->flat;
      out.push_back({lo, it->os + off, it->dst + off, hi - lo, 0});
    }
  }
  long long tiles = 0;
  for (std::size_t i = static_cast<std::size_t>(t.begin); i < out.size(); ++i) {
    out[i].tile0 = static_cast<unsigned long long>(tiles);
    tiles += static_cast<long long>((out[i].len + amsp::kTile - 1) / amsp::kTile);
  }
  t.nseg = static_cast<int>(out.size()) - t.begin;
  t.ntiles = static_cast<int>(tiles);
  return t;
}

// Gradient ring (engine grad_ring_elems > 0; PAPER.md:316-326 / D_g =
// 2*Phi/s_g, cost_model.cpp:151). Every micro-batch's tensor gradients get a
// slot in the ring when their grad-weight event produces them, and the slot
// is reused once every rank has pulled it: the release barrier + event of
// the accumulation (non-last micro-batch) or of the reduce (last one, ring
// mode adds it) that read it. A producer whose slot overlaps older
// gradients waits on those release events; gradients only the end-of-step
// update reads (tensors without a reduce event, e.g. the head when s_p > 1)
// hold their slot for the whole step (the step's end barrier releases
// them). The placement is a deterministic simulation of the graph's issue
// order, identical on every rank, so every rank's ring has the same layout
// and peers address each other's slots directly. The tables' `flat` offsets
// (used only to address gradients) are remapped into the ring, split at
// tensor boundaries; slot starts keep flat's alignment mod 64 elements, so
// every kernel takes the same vector / scalar paths as without the ring.
namespace {

struct RingPlan {
  bool ok = true;
  std::vector<std::vector<std::uint64_t>> off;           // [mb][t]
  std::vector<std::vector<int>> waits;                    // per event: rel event ids
};

RingPlan simulate_ring(const amsp_sched* s, const std::vector<shardplan::Event>& evs,
                       const std::vector<int>& ev_mb, const std::vector<char>& covered,
                       std::uint64_t R) {
  const amsp_engine* e = s->e;
  const std::size_t n = e->tensor_sizes.size();
  const int Mb = s->micro;
  const int K = s->layers_k;
  RingPlan p;
  p.off.assign(static_cast<std::size_t>(Mb), std::vector<std::uint64_t>(n, ~0ull));
  p.waits.assign(evs.size(), {});
  // consumers still to come for every (mb, t)
  std::vector<std::vector<int>> pending(static_cast<std::size_t>(Mb), std::vector<int>(n, 0));
  for (std::size_t i = 0; i < evs.size(); ++i)
    for (int t : s->work[i].reads) ++pending[static_cast<std::size_t>(ev_mb[i])][t];
  for (const HeadAccum& h : s->head_acc)
    for (int t : h.reads) ++pending[static_cast<std::size_t>(h.mb)][t];
  for (std::size_t t = 0; t < n; ++t)
    if (!covered[t]) ++pending[static_cast<std::size_t>(Mb - 1)][t];  // end-of-step update
  struct Live {
    std::uint64_t a, b;
    int mb, t;
    std::vector<int> rel;
  };
  std::vector<Live> live;
  std::uint64_t cursor = 0;
  auto consume = [&](int mb, int t, int rel) {
    for (Live& L : live)
      if (L.mb == mb && L.t == t) {
        --pending[static_cast<std::size_t>(mb)][t];
        L.rel.push_back(rel);
        return;
      }
  };
  const std::vector<int> head = {static_cast<int>(n) - 1, static_cast<int>(n) - 2, 0};
  for (std::size_t i = 0; i < evs.size() && p.ok; ++i) {
    const EventWork& w = s->work[i];
    const int mb = ev_mb[i];
    if (evs[i].kind == shardplan::EventKind::BwdGradWeight) {
      const std::vector<int> ts =
          evs[i].layer < 0 ? head : std::vector<int>{1 + evs[i].layer * K + evs[i].module};
      for (int t : ts) {
        const std::uint64_t size = e->tensor_sizes[static_cast<std::size_t>(t)];
        const std::uint64_t phase = e->pmap.tensor_offset[static_cast<std::size_t>(t)] % 64;
        auto place = [phase](std::uint64_t from) {
          std::uint64_t st = from / 64 * 64 + phase;
          return st < from ? st + 64 : st;
        };
        // first fit from the cursor (wrapping once): skip slots still holding
        // gradients whose readers have not all been issued; slots whose
        // readers have been issued are reused behind their release events
        std::uint64_t a = place(cursor);
        bool wrapped = false;
        while (p.ok) {
          if (a + size > R) {
            if (wrapped) {
              p.ok = false;
              break;
            }
            wrapped = true;
            a = place(0);
            continue;
          }
          const Live* block = nullptr;
          for (const Live& L : live)
            if (L.a < a + size && a < L.b && pending[static_cast<std::size_t>(L.mb)][L.t] > 0 &&
                (!block || L.b > block->b))
              block = &L;
          if (!block) break;
          a = place(block->b);
        }
        if (!p.ok) break;
        for (std::size_t k = 0; k < live.size();) {
          const Live& L = live[k];
          if (L.a < a + size && a < L.b) {
            for (int r : L.rel) p.waits[i].push_back(r);
            live.erase(live.begin() + static_cast<long>(k));
          } else {
            ++k;
          }
        }
        live.push_back({a, a + size, mb, t, {}});
        p.off[static_cast<std::size_t>(mb)][static_cast<std::size_t>(t)] = a;
        cursor = a + size;
      }
      if (w.head_acc >= 0) {  // the head's accumulation runs right behind it
        const HeadAccum& h = s->head_acc[static_cast<std::size_t>(w.head_acc)];
        for (int t : h.reads) consume(h.mb, t, h.rel);
      }
    }
    if (w.kind == Work::Accumulate || w.kind == Work::Reduce || w.kind == Work::ReduceAdam)
      for (int t : w.reads) consume(mb, t, static_cast<int>(i));
  }
  for (auto& v : p.waits) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  return p;
}

// A table of `src` re-emitted into `dst` with every piece split at tensor
// boundaries and `flat` moved into micro-batch mb's ring slots.
Table remap_table(const amsp_sched* s, const Table& t, const std::vector<amsp::Seg>& src,
                  std::vector<amsp::Seg>& dst, int mb) {
  const amsp_engine* e = s->e;
  const auto& toff = e->pmap.tensor_offset;
  Table out;
  out.begin = static_cast<int>(dst.size());
  for (int j = t.begin; j < t.begin + t.nseg; ++j) {
    amsp::Seg sg = src[static_cast<std::size_t>(j)];
    while (sg.len > 0) {
      const std::size_t ti = static_cast<std::size_t>(
          std::upper_bound(toff.begin(), toff.begin() + static_cast<long>(e->tensor_sizes.size()),
                           sg.flat) - toff.begin() - 1);
      const std::uint64_t in_t = sg.flat - toff[ti];
      const std::uint64_t take = std::min<std::uint64_t>(sg.len, e->tensor_sizes[ti] - in_t);
      const std::uint64_t slot = s->ring_off[static_cast<std::size_t>(mb)][ti];
      if (slot == ~0ull) throw Error("sched: gradient ring has no slot for a reduced tensor");
      dst.push_back({slot + in_t, sg.os, sg.dst, take, 0});
      sg.flat += take;
      sg.os += take;
      sg.dst += take;
      sg.len -= take;
    }
  }
  long long tiles = 0;
  for (std::size_t i = static_cast<std::size_t>(out.begin); i < dst.size(); ++i) {
    dst[i].tile0 = static_cast<unsigned long long>(tiles);
    tiles += static_cast<long long>((dst[i].len + amsp::kTile - 1) / amsp::kTile);
  }
  out.nseg = static_cast<int>(dst.size()) - out.begin;
  out.ntiles = static_cast<int>(tiles);
  return out;
}

void plan_grad_ring(amsp_sched* s, const std::vector<shardplan::Event>& evs,
                    const std::vector<int>& ev_mb, const std::vector<char>& covered,
                    std::vector<amsp::Seg>& rsegs, std::vector<amsp::Seg>& asegs,
                    int& next_barrier) {
  amsp_engine* e = s->e;
  // smallest ring the schedule runs in (binary search over the simulation)
  std::uint64_t lo = *std::max_element(e->tensor_sizes.begin(), e->tensor_sizes.end());
  std::uint64_t hi = (e->phi + 64 * e->tensor_sizes.size()) * static_cast<std::uint64_t>(s->micro);
  if (!simulate_ring(s, evs, ev_mb, covered, hi).ok)
    throw Error("sched: the gradient ring cannot serve this schedule");
  while (lo + 64 < hi) {
    const std::uint64_t mid = (lo + hi) / 2;
    if (simulate_ring(s, evs, ev_mb, covered, mid).ok) hi = mid; else lo = mid;
  }
  s->ring_need = (hi + 63) / 64 * 64;
  if (e->grad_elems < s->ring_need)
    throw Error("sched: gradient ring of " + std::to_string(e->grad_elems) +
                " elements is too small for this schedule; it needs " +
                std::to_string(s->ring_need));
  RingPlan p = simulate_ring(s, evs, ev_mb, covered, e->grad_elems);
  if (!p.ok)  // placement is not monotone in the ring size: the exact size can fail
    throw Error("sched: gradient ring of " + std::to_string(e->grad_elems) +
                " elements cannot place this schedule; use " + std::to_string(s->ring_need));
  s->ring_off = std::move(p.off);
  const int last = s->micro - 1;
  std::vector<amsp::Seg> r2, a2;
  for (std::size_t i = 0; i < evs.size(); ++i) {
    EventWork& w = s->work[i];
    for (int j : p.waits[i]) w.wait_release.push_back(j);
    if (w.kind == Work::Reduce || w.kind == Work::ReduceAdam) {
      const Table t = remap_table(s, {w.seg_begin, w.nseg, w.ntiles}, rsegs, r2, last);
      w.seg_begin = t.begin;
      w.nseg = t.nseg;
      w.ntiles = t.ntiles;
      w.rel_barrier = next_barrier++;
    } else if (w.kind == Work::Accumulate) {
      const Table t = remap_table(s, {w.seg_begin, w.nseg, w.ntiles}, asegs, a2, w.mb);
      w.seg_begin = t.begin;
      w.nseg = t.nseg;
      w.ntiles = t.ntiles;
    }
    if (w.post_ntiles > 0) throw Error("sched: a gradient ring needs W > 1");
  }
  for (HeadAccum& h : s->head_acc) h.t = remap_table(s, h.t, asegs, a2, h.mb);
  s->resid = remap_table(s, s->resid, rsegs, r2, last);
  s->pending = remap_table(s, s->pending, rsegs, r2, last);
  rsegs = std::move(r2);
  asegs = std::move(a2);
}

}  // namespace

void build(amsp_sched* s, const amsp_sched_config_t* cfg, const amsp_profile_t* profile) {
  amsp_engine* e = s->e;
  using namespace amsp::conv;
  const shardplan::ModelSpec model = model_in(&cfg->model);
  model.check();
  const int L = model.layer_count, K = model.modules_per_layer;
  const int Mb = model.micro_batch_count;
  if (Mb != e->micro)
    throw Error("sched: the model's " + std::to_string(Mb) +
                " micro-batches differ from the engine's " + std::to_string(e->micro));
  s->micro = Mb;
  if (cfg->grad_source < 0 || cfg->grad_source > 1) throw Error("sched: unknown grad_source");
  s->grad_source = cfg->grad_source;
  if (Mb > 1 && cfg->compute_mode == 0 && s->grad_source == 0)
    throw Error("sched: M > 1 with stand-in compute needs grad_source = 1 (each grad-weight "
                "event produces its micro-batch gradient)");
  if (e->staged && cfg->optimizer_variant != 0)
    throw Error("sched: accumulated micro-batches reduce on the LDG kernels (optimizer_variant 0)");
  // Tensor list = [embed] + L x K modules + [final norm, lm_head].
  const std::size_t n = e->tensor_sizes.size();
  if (n != static_cast<std::size_t>(L) * K + 3)
    throw Error("sched: engine tensors must be embed + L*K modules + norm + head");
  for (int l = 0; l < L; ++l)
    for (int i = 0; i < K; ++i)
      if (e->tensor_sizes[1 + l * K + i] != model.module_params[i])
        throw Error("sched: engine tensor sizes do not match the model's layer template");
  if (e->phi != model.total_params)
    throw Error("sched: engine Phi differs from the model's total_params");
  auto tensor_of = [K](int l, int i) { return 1 + l * K + i; };
  auto range_of = [e](int t) {
    const std::uint64_t a = e->pmap.tensor_offset[t];
    return FlatRange{a, a + e->tensor_sizes[t]};
  };
  s->optimizer_overlap = cfg->optimizer_overlap != 0;
  if (cfg->optimizer_variant != 0 && (cfg->optimizer_variant < 5 || cfg->optimizer_variant > 12))
    throw Error("sched: optimizer_variant must be 0 (LDG) or 5..12 (TMA)");
  if (cfg->optimizer_variant != 0 && !e->segments_aligned())
    throw Error("sched: the TMA optimizer variant needs 8-element-aligned segments");
  s->opt_variant = cfg->optimizer_variant;

  shardplan::ClusterSpec cl;
  const DeviceMesh dp = to_mesh(e->cfg.dp_mesh);
  cl.gpus_per_node = dp.per_node;
  cl.node_count = dp.nodes;
  cl.gpu_memory_capacity = std::uint64_t{1} << 50;
  cl.dp_mesh = dp;
  cl.topology = {dp.nodes, 1, 1.0};
  const shardplan::ShardingPlan plan = plan_in(&e->cfg.plan);
  const shardplan::CostConfig cost = cost_in(&cfg->cost);
  const shardplan::SimConfig sim = sim_in(&cfg->sim, K);
  s->graph = shardplan::build_schedule(model, cl, plan, profile->p, cost, sim);
  const shardplan::Timeline tl = shardplan::simulate_step(s->graph);
  s->predicted_step = tl.step_time;
  s->predicted_compute = tl.busy.empty() ? 0.0 : tl.busy[0];

  // Gradient buckets as flat ranges (backward order: head = lm_head, final
  // norm, embed; then layers / modules descending), plus, per bucket, the
  // modules (tensors) it touches.
  std::vector<std::pair<int, FlatRange>> stream_ranges = {
      {static_cast<int>(n) - 1, range_of(static_cast<int>(n) - 1)},
      {static_cast<int>(n) - 2, range_of(static_cast<int>(n) - 2)},
      {0, range_of(0)}};
  for (int l = L - 1; l >= 0; --l)
    for (int i = K - 1; i >= 0; --i) stream_ranges.push_back({tensor_of(l, i), range_of(tensor_of(l, i))});
  const std::uint64_t cut =
      cost.bucket_size * static_cast<std::uint64_t>(plan.sp()) / model.bytes_per_grad;
  std::vector<std::vector<FlatRange>> buckets(1);
  std::vector<std::vector<int>> bucket_tensors(1);
  std::uint64_t filled = 0;
  for (auto [t, r] : stream_ranges) {
    auto [a, b] = r;
    while (a < b) {
      const std::uint64_t take = std::min(b - a, cut - filled);
      buckets.back().push_back({a, a + take});
      bucket_tensors.back().push_back(t);
      a += take;
      filled += take;
      if (filled == cut) {
        buckets.emplace_back();
        bucket_tensors.emplace_back();
        filled = 0;
      }
    }
  }
  if (buckets.back().empty()) {
    buckets.pop_back();
    bucket_tensors.pop_back();
  }

  const auto& evs = s->graph.events;
  // Micro-batch of every event: build_schedule emits forward then backward
  // per micro-batch (overlap_sim.cpp:161-164), and each forward pass has
  // exactly one FwdCompute of layer 0 / module 0.
  std::vector<int> ev_mb(evs.size(), 0);
  {
    int cur = -1;
    for (std::size_t i = 0; i < evs.size(); ++i) {
      if (evs[i].kind == shardplan::EventKind::FwdCompute && evs[i].layer == 0 &&
          evs[i].module == 0)
        ++cur;
      ev_mb[i] = std::max(cur, 0);
    }
    if (cur != Mb - 1) throw Error("sched: graph has " + std::to_string(cur + 1) +
                                   " forward passes for M = " + std::to_string(Mb));
  }
  auto last_mb = [&](std::size_t i) { return ev_mb[i] == Mb - 1; };
  // Last grad-input event of each tensor in the last micro-batch (head
  // tensors: the head's gi) -- the optimizer placement anchors.
  std::vector<int> gi_event(n, -1);
  for (std::size_t i = 0; i < evs.size(); ++i) {
    if (evs[i].kind != shardplan::EventKind::BwdGradInput || !last_mb(i)) continue;
    if (evs[i].layer < 0) {
      gi_event[0] = gi_event[n - 2] = gi_event[n - 1] = static_cast<int>(i);
    } else {
      gi_event[tensor_of(evs[i].layer, evs[i].module)] = static_cast<int>(i);
    }
  }

  s->gemm_mode = cfg->compute_mode == 1;
  s->gather_dma = cfg->gather_mode == 1;
  s->gather_tma = cfg->gather_mode == 2;
  if (cfg->gather_mode < 0 || cfg->gather_mode > 2) throw Error("sched: unknown gather_mode");
  if (s->gather_tma && e->sp > 1 && !e->copies_aligned())
    throw Error("sched: the TMA all-gather needs 8-element-aligned P slices");
  s->layers_k = K;
  // Mirrored broadcast: the graph leads with last step's BroadcastShard
  // events (tier ag_rs_ar_bc, k > 1) and parameters are not sharded.
  int n_bc = 0;
  for (const auto& ev : evs) n_bc += ev.kind == shardplan::EventKind::BroadcastShard;
  if (cfg->bc_mode < 0 || cfg->bc_mode > 1) throw Error("sched: unknown bc_mode");
  s->mirror = cfg->bc_mode == 0 && plan.sp() == 1 && n_bc > 0 &&
              evs.front().kind == shardplan::EventKind::BroadcastShard &&
              e->dst_members.size() > 1;
  if (s->mirror) {
    // Every OS-group member's shard layout (the same map the engine uses).
    const int k = static_cast<int>(e->dst_members.size());
    std::vector<amsp::ShardLayout> member(static_cast<std::size_t>(k));
    int me = -1;
    for (int q = 0; q < k; ++q) {
      member[q] = amsp::pshard_layout(e->tensor_sizes, 1, 0, k, q, e->cfg.layout);
      if (e->dst_members[q] == e->rank) me = q;
    }
    // Layer block of each tensor: the graph's shard_gate (overlap_sim.cpp:
    // 193-199); head tensors (embed, final norm, lm_head) in the last block.
    std::vector<int> block(n, n_bc - 1), layer(n, L);
    for (int l = 0; l < L; ++l) {
      const int j = std::max(0, ((l + 1) * n_bc + L - 1) / L - 1);
      for (int i = 0; i < K; ++i) {
        block[tensor_of(l, i)] = j;
        layer[tensor_of(l, i)] = l;
      }
    }
    s->bc_copies.assign(static_cast<std::size_t>(n_bc), {});
    for (std::size_t t = 0; t < n; ++t) {
      const auto [lo, hi] = range_of(static_cast<int>(t));
      for (int q = 0; q < k; ++q) {
        if (q == me) continue;
        for (const auto& sg : member[q].segs) {
          const std::uint64_t a = std::max(lo, sg.flat), b = std::min(hi, sg.flat + sg.len);
          if (a < b)
            s->bc_copies[block[t]].push_back(
                {sg.dst + (a - sg.flat), b - a, e->dst_members[q], layer[t]});
        }
      }
    }
    for (auto& cs : s->bc_copies)  // layer order inside each block (head last)
      std::stable_sort(cs.begin(), cs.end(),
                       [](const BcCopy& x, const BcCopy& y) { return x.layer < y.layer; });
    s->layer_ev.assign(static_cast<std::size_t>(L) + 1, nullptr);
  }
  std::uint64_t max_out = 0;
  std::vector<amsp::Seg> rsegs, asegs;
  // Accumulation index map (Seg::os = G-shard accumulator offset): the P
  // shard when s_g = s_p, the OS shard when s_g = s_os > s_p.
  amsp::ShardLayout acc_layout;
  if (e->staged) {
    if (e->acc_by_dst) {
      acc_layout = amsp::pshard_layout(e->tensor_sizes, e->sp, e->p_group.position, 1, 0,
                                       amsp::kLayoutContiguous);
      for (auto& sg : acc_layout.segs) sg.os = sg.dst;
    } else {
      acc_layout = e->layout;
    }
  }
  // release[mb][t]: the Accumulate events (rel_events indices) that pulled
  // tensor t's gradient of micro-batch mb.
  std::vector<std::vector<std::vector<int>>> release(
      static_cast<std::size_t>(Mb), std::vector<std::vector<int>>(n));
  const std::vector<int> head_tensors = {static_cast<int>(n) - 1, static_cast<int>(n) - 2, 0};
  std::vector<char> ag_seen(n, 0);  // ZeRO++: the step's first gather of the tensor
  bool first_secondary = true;
  std::vector<char> covered(n, 0);  // reduced by some event
  std::vector<char> updated(n, 0);  // optimizer already applied by some event
  int next_barrier = kFirstSchedBarrier;
  s->work.resize(evs.size());
  int ar_seen = 0;
  for (std::size_t i = 0; i < evs.size(); ++i) {
    const shardplan::Event& ev = evs[i];
    EventWork& w = s->work[i];
    w.stream = ev.stream;
    w.mb = ev_mb[i];
    const bool last = last_mb(i);
    if (ev.kind == shardplan::EventKind::BwdGradWeight) {
      const std::vector<int> ts =
          ev.layer < 0 ? head_tensors : std::vector<int>{tensor_of(ev.layer, ev.module)};
      if (!s->gemm_mode && s->grad_source == 1) w.synth_tensors = ts;
      w.accum_in_place = e->sg == 1 && w.mb > 0;
      if (w.mb > 0)
        for (int tt : ts)
          for (int j : release[static_cast<std::size_t>(w.mb - 1)][tt]) w.wait_release.push_back(j);
      if (!last && e->staged && e->acc_by_dst && ev.layer < 0) {
        std::vector<FlatRange> hr;
        for (int tt : ts) hr.push_back(range_of(tt));
        std::sort(hr.begin(), hr.end());
        HeadAccum h;
        h.t = owned_pieces(acc_layout, hr, asegs);
        h.barrier = next_barrier++;
        h.rel_barrier = next_barrier++;
        h.rel = static_cast<int>(evs.size() + s->head_acc.size());
        h.mb = w.mb;
        h.reads = ts;
        w.head_acc = static_cast<int>(s->head_acc.size());
        s->head_acc.push_back(h);
        for (int tt : ts) release[static_cast<std::size_t>(w.mb)][tt].push_back(h.rel);
      }
    }
    if (!last && (ev.kind == shardplan::EventKind::ReduceScatter ||
                  ev.kind == shardplan::EventKind::AllReduceBucket)) {
      // A non-last micro-batch: s_g = s_p folds each
      // module's reduce-scatter into the P-shard accumulator; s_g > s_p
      // folds each AllReduce bucket over ratio(g, p) + select & drop into
      // the OS-shard accumulator (overlap_sim.cpp:320-330). Both pull the
      // raw bf16 gradients of the rank's G block. Otherwise a marker.
      std::vector<FlatRange> ranges;
      std::vector<int> ts;
      if (ev.kind == shardplan::EventKind::ReduceScatter && e->staged && e->acc_by_dst) {
        const int tt = tensor_of(ev.layer, ev.module);
        ranges = {range_of(tt)};
        ts = {tt};
      } else if (ev.kind == shardplan::EventKind::AllReduceBucket) {
        if (!e->staged || e->acc_by_dst)
          throw Error("sched: AllReduce bucket in a non-last micro-batch without s_g > s_p");
        if (ev.module >= static_cast<int>(buckets.size()))
          throw Error("sched: bucket index beyond the gradient stream");
        ranges = buckets[ev.module];
        ts = bucket_tensors[ev.module];
      }
      if (ranges.empty()) {
        w.kind = Work::Marker;
        continue;
      }
      w.kind = Work::Accumulate;
      w.reads = ts;
      const Table at = owned_pieces(acc_layout, ranges, asegs);
      w.seg_begin = at.begin;
      w.nseg = at.nseg;
      w.ntiles = at.ntiles;
      w.barrier = next_barrier++;
      w.rel_barrier = next_barrier++;
      for (int tt : ts) release[static_cast<std::size_t>(w.mb)][tt].push_back(static_cast<int>(i));
      ++s->n_reduce;
      continue;
    }
    switch (ev.kind) {
      case shardplan::EventKind::FwdCompute:
      case shardplan::EventKind::BwdGradInput:
      case shardplan::EventKind::BwdGradWeight:
      case shardplan::EventKind::RecomputeFwd: {
        w.kind = Work::Compute;
        w.ns = static_cast<unsigned long long>(ev.duration * cfg->time_scale * 1e9);
        ++s->n_compute;
        if (!s->gemm_mode) break;
        const int t = ev.layer < 0 ? -1 : tensor_of(ev.layer, ev.module);
        const std::uint64_t size = e->tensor_sizes[t < 0 ? n - 1 : static_cast<std::size_t>(t)];
        const std::uint64_t H = static_cast<std::uint64_t>(model.hidden);
        if (size > H && size % H == 0) {  // linear module
          w.tensor = t;
          w.g_in = model.hidden;
          w.g_out = static_cast<int>(size / H);
          w.gemm = ev.kind == shardplan::EventKind::BwdGradInput    ? Gemm::DGrad
                   : ev.kind == shardplan::EventKind::BwdGradWeight ? Gemm::WGrad
                                                                    : Gemm::Fwd;
          max_out = std::max<std::uint64_t>(max_out, size / H);
          // LLaMA layer template (q,k,v,o,gate,up,down,attn_norm,mlp_norm):
          // the attention core sits between v and o
          w.attention = K == 9 && ev.module == 3 && w.gemm != Gemm::WGrad;
        } else if (size == H && H % 8 == 0 && t >= 0) {  // RMSNorm module
          w.tensor = t;
          w.gemm = ev.kind == shardplan::EventKind::BwdGradInput    ? Gemm::NormDGrad
                   : ev.kind == shardplan::EventKind::BwdGradWeight ? Gemm::NormWGrad
                                                                    : Gemm::NormFwd;
        }
        break;
      }
      case shardplan::EventKind::AllGather:
        w.kind = Work::Gather;
        w.tensor = tensor_of(ev.layer, ev.module);
        if (e->s2 > 1) {
          if (!ag_seen[static_cast<std::size_t>(w.tensor)]) {
            ag_seen[static_cast<std::size_t>(w.tensor)] = 1;
            w.refresh = true;
          } else {
            w.secondary = true;
            if (first_secondary) {
              w.barrier = next_barrier++;
              first_secondary = false;
            }
          }
        }
        ++s->n_gather;
        break;
      case shardplan::EventKind::ReduceScatter: {
        w.tensor = tensor_of(ev.layer, ev.module);
        w.reads = {w.tensor};
        covered[w.tensor] = 1;
        const Table t = owned_pieces(e->layout, {range_of(w.tensor)}, rsegs);
        w.seg_begin = t.begin;
        w.nseg = t.nseg;
        w.ntiles = t.ntiles;
        w.barrier = next_barrier++;
        if (s->optimizer_overlap) {
          w.kind = Work::ReduceAdam;
          updated[w.tensor] = 1;
        } else {
          w.kind = Work::Reduce;
        }
        ++s->n_reduce;
        break;
      }
      case shardplan::EventKind::AllReduceBucket: {
        ++ar_seen;
        if (plan.sp() > 1) {
          // The module reduce-scatters already summed over every DP rank.
          w.kind = Work::Marker;
          break;
        }
        if (ev.module >= static_cast<int>(buckets.size()))
          throw Error("sched: bucket index beyond the gradient stream");
        w.kind = Work::Reduce;
        w.reads = bucket_tensors[ev.module];
        const Table t = owned_pieces(e->layout, buckets[ev.module], rsegs);
        w.seg_begin = t.begin;
        w.nseg = t.nseg;
        w.ntiles = t.ntiles;
        w.barrier = next_barrier++;
        if (s->optimizer_overlap) {
          int last = -1;
          for (int tt : bucket_tensors[ev.module]) last = std::max(last, gi_event[tt]);
          if (last >= 0) {
            w.adam_after = true;
            w.after_event = last;
            w.barrier2 = next_barrier++;
            s->work[last].record = true;
          }
        }
        ++s->n_reduce;
        break;
      }
      case shardplan::EventKind::BroadcastShard:
        w.kind = s->mirror ? Work::Broadcast : Work::Marker;
        w.bc = ev.module;
        break;
    }
  }
  s->n_buckets = ar_seen;
  if (plan.sp() == 1 && ar_seen > 0) {
    if (ar_seen != static_cast<int>(buckets.size()))
      throw Error("sched: graph has " + std::to_string(ar_seen) + " buckets, executor cut " +
                  std::to_string(buckets.size()));
    std::fill(covered.begin(), covered.end(), 1);
    if (s->optimizer_overlap) {
      for (std::size_t b = 0; b < buckets.size(); ++b) {
        bool all_have_gi = true;
        for (int tt : bucket_tensors[b]) all_have_gi &= gi_event[tt] >= 0;
        if (!all_have_gi) throw Error("sched: bucket without grad-input events");
      }
      std::fill(updated.begin(), updated.end(), 1);
    }
  }
  // A single rank has nothing to reduce: with optimizer overlap its fused
  // update runs bucket by bucket behind the backward pass (the graph's own
  // bucket cuts), each after the grad-input that last reads those params.
  if (plan.sp() == 1 && ar_seen == 0 && s->optimizer_overlap && e->world == 1) {
    for (std::size_t b = 0; b < buckets.size(); ++b) {
      int last = -1;
      for (int tt : bucket_tensors[b]) last = std::max(last, gi_event[tt]);
      if (last < 0) continue;
      EventWork& w = s->work[last];
      if (w.post_ntiles > 0) {
        // Several buckets closed by one event: extend its table.
        const Table t = owned_pieces(e->layout, buckets[b], rsegs);
        if (t.begin != w.post_begin + w.post_nseg)
          throw Error("sched: non-contiguous post tables");
        for (int q = t.begin; q < t.begin + t.nseg; ++q)
          rsegs[q].tile0 += static_cast<unsigned long long>(w.post_ntiles);
        w.post_nseg += t.nseg;
        w.post_ntiles += t.ntiles;
      } else {
        const Table t = owned_pieces(e->layout, buckets[b], rsegs);
        w.post_begin = t.begin;
        w.post_nseg = t.nseg;
        w.post_ntiles = t.ntiles;
      }
      w.record = true;
      for (int tt : bucket_tensors[b]) covered[tt] = updated[tt] = 1;
    }
  }
  // After the graph: tensors nobody reduced get the fused update; reduced but
  // not yet updated ones get AdamW from the fp32 reduced gradients.
  std::vector<FlatRange> rest, pend;
  for (std::size_t t = 0; t < n; ++t) {
    if (!covered[t]) rest.push_back(range_of(static_cast<int>(t)));
    else if (!updated[t]) pend.push_back(range_of(static_cast<int>(t)));
  }
  s->resid = owned_pieces(e->layout, rest, rsegs);
  s->pending = owned_pieces(e->layout, pend, rsegs);
  s->resid_aligned = true;
  for (int j = s->resid.begin; j < s->resid.begin + s->resid.nseg; ++j) {
    const amsp::Seg& sg = rsegs[static_cast<std::size_t>(j)];
    if ((sg.flat | sg.os | sg.dst | sg.len) & 7u) s->resid_aligned = false;
  }
  if (e->ring) {
    if (!s->gemm_mode && s->grad_source == 0)
      throw Error("sched: a gradient ring is written by the step's own grad-weight events: use "
                  "compute='gemm' or grad_source = 1");
    plan_grad_ring(s, evs, ev_mb, covered, rsegs, asegs, next_barrier);
  }
  s->end_a = next_barrier++;
  s->end_b = next_barrier++;
  s->flush_barrier = next_barrier++;
  s->n_barriers = next_barrier - kFirstSchedBarrier;
  if (next_barrier > amsp::kBarrierIds) throw Error("sched: too many barriers per step");

  // An event is recorded when a later event on another stream waits on it.
  for (std::size_t i = 0; i < evs.size(); ++i)
    for (int d : evs[i].depends_on)
      if (s->work[d].stream != s->work[i].stream) s->work[d].record = true;

  if (cfg->reduce_mode < 0 || cfg->reduce_mode > 1) throw Error("sched: unknown reduce_mode");
  s->reduce_dma = cfg->reduce_mode == 1 && e->world > 1;
  if (s->reduce_dma) {
    s->h_rsegs = rsegs;
    s->h_ssegs = rsegs;
    std::uint64_t slot = 8;
    int stage_stream = -1;  // one staging buffer: its users must share a FIFO stream
    for (const EventWork& w : s->work) {
      if (w.kind != Work::Reduce && w.kind != Work::ReduceAdam) continue;
      if (stage_stream >= 0 && w.stream != stage_stream)
        throw Error("sched: staged reduces on two streams");
      stage_stream = w.stream;
      std::uint64_t off = 0;
      for (int j = w.seg_begin; j < w.seg_begin + w.nseg; ++j) {
        s->h_ssegs[j].flat = off;  // 8-element aligned staging offsets
        off += (rsegs[j].len + 7) / 8 * 8;
      }
      slot = std::max(slot, off);
    }
    s->stage_slot = slot;
  }

  // Device tables and buffers.
  e->use_device();
  if (s->reduce_dma) {
    ck(cudaMalloc(&s->stage, s->stage_slot * 2 * static_cast<std::uint64_t>(e->world)),
       "cudaMalloc reduce staging");
    ck(cudaMalloc(&s->d_ssegs, rsegs.size() * sizeof(amsp::Seg)), "cudaMalloc staged segs");
    ck(cudaMemcpy(s->d_ssegs, s->h_ssegs.data(), rsegs.size() * sizeof(amsp::Seg),
                  cudaMemcpyHostToDevice),
       "copy staged segs");
  }
  if (!rsegs.empty()) {
    ck(cudaMalloc(&s->d_rsegs, rsegs.size() * sizeof(amsp::Seg)), "cudaMalloc sched segs");
    ck(cudaMemcpy(s->d_rsegs, rsegs.data(), rsegs.size() * sizeof(amsp::Seg),
                  cudaMemcpyHostToDevice),
       "copy sched segs");
  }
  if (e->sp > 1) {
    std::vector<amsp::CopySeg> tc(n);
    for (std::size_t t = 0; t < n; ++t)
      tc[t] = {0, e->pmap.pshard_offset[t], e->pmap.slice_len[t], 0,
               e->s2 > 1 ? e->smap.pshard_offset[t] : 0};
    ck(cudaMalloc(&s->d_tcopy, n * sizeof(amsp::CopySeg)), "cudaMalloc tensor copies");
    ck(cudaMemcpy(s->d_tcopy, tc.data(), n * sizeof(amsp::CopySeg), cudaMemcpyHostToDevice),
       "copy tensor copies");
    if (e->s2 > 1) {
      for (std::size_t t = 0; t < n; ++t)
        tc[t] = {0, e->smap.pshard_offset[t], e->smap.slice_len[t], 0, 0};
      ck(cudaMalloc(&s->d_tcopy2, n * sizeof(amsp::CopySeg)), "cudaMalloc secondary copies");
      ck(cudaMemcpy(s->d_tcopy2, tc.data(), n * sizeof(amsp::CopySeg), cudaMemcpyHostToDevice),
         "copy secondary copies");
    }
  }
  if (!asegs.empty()) {
    ck(cudaMalloc(&s->d_asegs, asegs.size() * sizeof(amsp::Seg)), "cudaMalloc accumulation segs");
    ck(cudaMemcpy(s->d_asegs, asegs.data(), asegs.size() * sizeof(amsp::Seg),
                  cudaMemcpyHostToDevice),
       "copy accumulation segs");
  }
  s->rel_events.assign(evs.size() + s->head_acc.size(), nullptr);
  for (std::size_t i = 0; i < evs.size(); ++i)
    if (s->work[i].kind == Work::Accumulate || s->work[i].rel_barrier >= 0)
      ck(cudaEventCreateWithFlags(&s->rel_events[i], cudaEventDisableTiming), "event");
  for (const HeadAccum& h : s->head_acc) {
    ck(cudaEventCreateWithFlags(&s->rel_events[static_cast<std::size_t>(h.rel)],
                                cudaEventDisableTiming),
       "event");
    s->head_done.push_back(nullptr);
    ck(cudaEventCreateWithFlags(&s->head_done.back(), cudaEventDisableTiming), "event");
  }
  const bool needs_red = s->pending.ntiles > 0 || (plan.sp() == 1 && ar_seen > 0);
  if (needs_red)
    ck(cudaMalloc(&s->red, std::max<std::size_t>(e->layout.owned, 1) * sizeof(float)),
       "cudaMalloc reduced grads");
  s->events.resize(evs.size(), nullptr);
  for (std::size_t i = 0; i < evs.size(); ++i)
    if (s->work[i].record)
      ck(cudaEventCreateWithFlags(&s->events[i], cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&s->start_ev, cudaEventDisableTiming), "event");
  for (auto& ev : s->join_ev) ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
  for (auto& ev : s->layer_ev) ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
  // Communication streams get the highest priority so their CTAs are placed
  // first whenever SMs free up between compute CTAs.
  int lo_prio = 0, hi_prio = 0;
  ck(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio), "stream priorities");
  for (auto& st : s->comm)
    ck(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi_prio), "stream");
  if (s->gemm_mode && cfg->gemm_sm_margin > 0)
    s->gemm_sm_target = std::max(1, e->sms - cfg->gemm_sm_margin);
  if (s->gemm_mode) {
    amsp::Blas::instance();  // fail now, not mid-step, when cuBLAS is missing
    s->tokens = cfg->tokens > 0 ? cfg->tokens : model.micro_batch * model.seq_len;
    const std::uint64_t T = static_cast<std::uint64_t>(s->tokens);
    const std::uint64_t H = static_cast<std::uint64_t>(model.hidden);
    const std::uint64_t wide = std::max(max_out, H);
    auto alloc = [](uint16_t** p, std::uint64_t elems, const char* what) {
      ck(cudaMalloc(p, std::max<std::uint64_t>(elems, 8) * 2), what);
    };
    alloc(&s->act, T * H, "cudaMalloc activations");
    s->hidden = model.hidden;
    ck(cudaMalloc(&s->norm_acc, H * 4), "cudaMalloc norm scratch");
    ck(cudaMemset(s->norm_acc, 0, H * 4), "zero norm scratch");
    // Attention core: head_dim 128 (64 when H is not a multiple of 128),
    // T / S whole sequences per micro-batch.
    const int S = model.seq_len;
    const int d = model.hidden % 128 == 0 ? 128 : model.hidden % 64 == 0 ? 64 : 0;
    if (K == 9 && d > 0 && S > 0 && S % 8 == 0 && s->tokens % S == 0) {
      s->attn_s = S;
      s->attn_dim = d;
      s->attn_heads = model.hidden / d;
      s->attn_seqs = s->tokens / S;
      const std::uint64_t pe = static_cast<std::uint64_t>(s->attn_heads) * S * S;
      alloc(&s->probs, pe, "cudaMalloc attention probabilities");
      alloc(&s->dprobs, pe, "cudaMalloc attention probability grads");
      ck(amsp::launch_synth_grad(s->probs, 0, pe, 0x5EED, 4, 0, nullptr), "fill probs");
    } else {
      for (auto& w : s->work) w.attention = false;
    }
    alloc(&s->dout, T * wide, "cudaMalloc output grads");
    alloc(&s->yout, T * wide, "cudaMalloc outputs");
    // Small, finite synthetic activations (counter-based, like the grads).
    ck(amsp::launch_synth_grad(s->act, 0, T * H, 0x5EED, 1, 0, nullptr), "fill activations");
    ck(amsp::launch_synth_grad(s->dout, 0, T * wide, 0x5EED, 2, 0, nullptr), "fill out-grads");
    if (e->sp > 1) {
      std::uint64_t biggest = 0;
      for (int i = 0; i < K; ++i) biggest = std::max(biggest, model.module_params[i]);
      s->ring_slot = (biggest + 7) / 8 * 8;
      alloc(&s->ring, s->ring_slot * 3 * K, "cudaMalloc gathered-weight ring");
      alloc(&s->head_w, e->tensor_sizes[n - 1], "cudaMalloc head weight");
      ck(amsp::launch_synth_grad(s->head_w, 0, e->tensor_sizes[n - 1], 0x5EED, 3, 0, nullptr),
         "fill head weight");
    }
    ck(cudaDeviceSynchronize(), "gemm buffers");
  }
  if (s->opt_variant != 0)
    for (const auto& sg : rsegs)
      if ((sg.flat | sg.os | sg.dst | sg.len) & 7u)
        throw Error("sched: the TMA optimizer variant needs 8-element-aligned bucket pieces");
  s->comm_ctas = cfg->comm_ctas > 0 ? cfg->comm_ctas : 128;
  s->compute_ctas = cfg->compute_ctas > 0 ? cfg->compute_ctas : e->sms;
  s->time_scale = cfg->time_scale > 0 ? cfg->time_scale : 1.0;
}

}  // namespace

extern "C" {

int amsp_sched_create(amsp_engine_t* e, const amsp_sched_config_t* cfg,
                      const amsp_profile_t* profile, amsp_sched_t** out) {
  return amsp::guarded([&] {
    if (!e || !cfg || !profile || !out) throw Error("sched: null argument");
    auto s = std::make_unique<amsp_sched>();
    s->e = e;
    amsp_sched_config_t c = *cfg;
    if (c.time_scale <= 0) c.time_scale = 1.0;
    build(s.get(), &c, profile);
    *out = s.release();
  });
}

int amsp_sched_info(const amsp_sched_t* s, amsp_sched_info_t* info) {
  return amsp::guarded([&] {
    if (!s || !info) throw Error("sched: null argument");
    info->n_events = static_cast<int>(s->graph.events.size());
    info->n_compute = s->n_compute;
    info->n_gather = s->n_gather;
    info->n_reduce = s->n_reduce;
    info->n_buckets = s->n_buckets;
    info->n_barriers = s->n_barriers;
    info->stream_count = s->graph.stream_count;
    info->predicted_step_s = s->predicted_step;
    info->predicted_compute_s = s->predicted_compute;
    info->mirrored_bc = s->mirror ? 1 : 0;
    info->grad_ring_need = s->ring_need;
  });
}

int amsp_sched_barrier_owner(const amsp_sched_t* s, int id, int* event, int* role, int* mb) {
  return amsp::guarded([&] {
    if (!s || !event || !role || !mb) throw Error("sched: null argument");
    *event = -1;
    *mb = 0;
    const int step_level[3] = {s->end_a, s->end_b, s->flush_barrier};
    for (int k = 0; k < 3; ++k)
      if (id == step_level[k]) {
        *role = 5 + k;
        return;
      }
    for (std::size_t i = 0; i < s->work.size(); ++i) {
      const EventWork& w = s->work[i];
      const int ids[3] = {w.barrier, w.barrier2, w.rel_barrier};
      for (int k = 0; k < 3; ++k)
        if (ids[k] == id) {
          *event = static_cast<int>(i);
          *role = k;
          *mb = w.mb;
          return;
        }
      if (w.head_acc >= 0) {
        const HeadAccum& h = s->head_acc[static_cast<std::size_t>(w.head_acc)];
        if (h.barrier == id || h.rel_barrier == id) {
          *event = static_cast<int>(i);
          *role = h.barrier == id ? 3 : 4;
          *mb = h.mb;
          return;
        }
      }
    }
    throw Error("sched: no event uses barrier id " + std::to_string(id));
  });
}

int amsp_sched_step(amsp_sched_t* s, int step, void* stream, int mode) {
  return amsp::guarded([&] {
    if (!s) throw Error("sched: null argument");
    s->e->use_device();
    if (mode < 0 || mode > 2) throw Error("sched: mode must be 0, 1 or 2");
    s->run(step, s->e->pick(stream), mode);
  });
}

int amsp_sched_flush(amsp_sched_t* s, void* stream) {
  return amsp::guarded([&] {
    if (!s) throw Error("sched: null argument");
    s->e->use_device();
    s->flush(s->e->pick(stream));
  });
}

int amsp_sched_enable_trace(amsp_sched_t* s, int on) {
  return amsp::guarded([&] {
    if (!s) throw Error("sched: null argument");
    s->e->use_device();
    s->enable_trace(on != 0);
  });
}

int amsp_sched_trace(amsp_sched_t* s, char* buf, size_t cap, size_t* needed, double* step_ms) {
  return amsp::guarded([&] {
    if (!s) throw Error("sched: null argument");
    s->e->use_device();
    const std::string text = s->measured_trace(step_ms);
    if (needed) *needed = text.size();
    if (buf && cap) {
      const size_t n = std::min(cap - 1, text.size());
      std::memcpy(buf, text.data(), n);
      buf[n] = '\0';
    }
  });
}

int amsp_sched_predicted_trace(const amsp_sched_t* s, char* buf, size_t cap, size_t* needed) {
  return amsp::guarded([&] {
    if (!s) throw Error("sched: null argument");
    const std::string text = shardplan::render_trace(shardplan::simulate_step(s->graph));
    if (needed) *needed = text.size();
    if (buf && cap) {
      const size_t n = std::min(cap - 1, text.size());
      std::memcpy(buf, text.data(), n);
      buf[n] = '\0';
    }
  });
}

void amsp_sched_destroy(amsp_sched_t* s) { delete s; }

}  // extern "C"
