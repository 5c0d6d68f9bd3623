// Internal definition of the engine object shared by engine.cpp (C-ABI)
// and sched.cpp (overlap scheduler). Not part of the public API.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "amsp_c.h"
#include "kernels.h"
#include "layout.h"
#include "../status.h"

using shardplan::DeviceMesh;
using shardplan::Error;

namespace amsp_detail {

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw amsp::CudaFailure(std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}

constexpr std::size_t kAlign = 256;
constexpr std::size_t kFlagBytes =
    sizeof(uint32_t) * amsp::kBarrierIds * amsp::kMaxRanks;  // 256 KB
inline std::size_t align_up(std::size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

inline DeviceMesh to_mesh(amsp_mesh_t m) { return DeviceMesh{m.per_node, m.nodes}; }

// Device segment table with tile prefix sums.
template <class T>
int tile_prefix(std::vector<T>& segs) {
  long long tiles = 0;
  for (auto& s : segs) {
    s.tile0 = static_cast<unsigned long long>(tiles);
    tiles += static_cast<long long>((s.len + amsp::kTile - 1) / amsp::kTile);
  }
  if (tiles > 0x7fffffffLL) throw Error("engine: shard too large");
  return static_cast<int>(tiles);
}

// A run of consecutive tensors all-gathered by one launch.
struct GatherUnit {
  int first_tensor = 0, n_tensors = 0;
  std::uint64_t elems = 0;
  int seg_begin = 0, nseg = 0, ntiles = 0;
};

}  // namespace amsp_detail

using namespace amsp_detail;

struct amsp_engine {
  amsp_engine_config_t cfg{};
  std::vector<std::uint64_t> tensor_sizes;
  std::uint64_t phi = 0;
  int world = 1, rank = 0, sp = 1;
  amsp::ShardLayout layout;
  amsp::PShardMap pmap;
  amsp::MeshGroup os_group, p_group;
  std::vector<int> dst_members;  // OS-block ranks holding my P position
  int replicas = 1;

  // Micro-batches and gradient sharding. With M > 1 and
  // s_g > 1 ("staged") every rank holds a bf16 accumulator of its G shard:
  // the P shard (indexed by Seg::dst) when s_g = s_p, the OS shard (Seg::os)
  // when s_g = s_os > s_p. It sits at the end of the shared region (its size
  // may differ per rank; every other offset is identical on all ranks).
  int micro = 1, sg = 1;
  bool staged = false, acc_by_dst = false;
  // Gradient ring (cfg.grad_ring_elems > 0, s_g > 1): the gradient buffer is
  // a ring of grad_elems bf16 elements that only the overlap scheduler
  // addresses (sched.cpp, plan_grad_ring); otherwise grad_elems = Phi.
  std::uint64_t grad_elems = 0;
  bool ring = false;
  void require_full_grads(const char* what) const {
    if (ring)
      throw Error(std::string("engine: ") + what +
                  " needs the full gradient buffer; this engine keeps a gradient ring "
                  "(grad_ring_elems) that only the overlap scheduler writes");
  }
  std::size_t off_acc = 0;
  std::uint64_t acc_elems = 0;
  std::vector<int> acc_sources;  // my accumulation block, ascending rank
  std::vector<int> acc_holders;  // holder of my elements in every block, block order
  amsp::Seg* d_acc_segs = nullptr;
  int nacc_seg = 0, nacc_tiles = 0;

  // ZeRO++ secondary parameter shard (plan.secondary_params; engine.cpp
  // plan_secondary): s2 > 1 keeps Phi/s2 bf16 of every tensor's slice over
  // the secondary group, written from the forward all-gather, read by the
  // group's backward all-gathers.
  int s2 = 1;
  bool sec_fused = false;  // forward gathers store the secondary slice themselves
  amsp::MeshGroup sec_group;
  amsp::PShardMap smap;
  std::vector<GatherUnit> units2;  // the units' secondary copy tables
  std::vector<GatherUnit> units_push;  // the units' push tables (own slice only)

  // Shared region and its offsets (identical on every rank).
  char* shared = nullptr;
  std::size_t shared_bytes = 0, off_grads = 0, off_params = 0, off_flags = 0, off_sec = 0;
  std::size_t off_slots = 0, slot_bytes = 0;
  std::uint64_t param_elems = 0;
  void* peer_base[amsp::kMaxRanks] = {};
  bool imported = false;
  bool local_linked = false;  // single-GPU emulation of a group
  bool local_sync = false;    // ... with the real barriers / release fences
  // Cross-rank synchronisation is live (real group, or emulated with sync).
  bool synced() const { return world > 1 && (!local_linked || local_sync); }

  float* master = nullptr;
  float* exp_avg = nullptr;
  float* exp_avg_sq = nullptr;
  char* priv = nullptr;
  amsp::Seg* d_segs = nullptr;
  amsp::Seg* d_psegs = nullptr;
  amsp::CopySeg* d_copy = nullptr;
  uint16_t* slots[2] = {nullptr, nullptr};
  std::uint64_t slot_elems = 0;
  std::vector<GatherUnit> units;
  float* stats = nullptr;
  int* err = nullptr;
  uint32_t** d_peer_flags = nullptr;
  int nseg = 0, ntiles = 0, npseg = 0, nptiles = 0;
  int grid = 0, variant = 0, sms = 148, gather_grid = 0;
  // gather_grid: > 0 SM-kernel grid, 0 SM kernel with its default grid,
  // kGatherDma copy engines, kGatherTma the bulk-copy kernel.
  static constexpr int kGatherDma = -1, kGatherTma = -2, kGatherPush = -3;
  bool copies_aligned() const {
    for (std::size_t t = 0; t < pmap.slice_len.size(); ++t)
      if ((pmap.slice_len[t] | pmap.pshard_offset[t] | pmap.tensor_offset[t]) & 7u) return false;
    return true;
  }
  std::uint64_t device_bytes = 0;

  cudaStream_t own_stream = nullptr;
  // Linked (single-GPU emulated) engines share rank 0's stream so that one
  // rank's step is ordered after every rank's gradient production.
  cudaStream_t shared_default = nullptr;
  uint32_t epoch = 0;
  // Epoch of the scheduler barriers (ids >= 16), shared by every scheduler
  // of this engine so that a flag word never goes backwards (amsp_sched).
  uint32_t sched_epoch = 0;
  // Optional CUDA-event bracketing of every fused launch (bench roofline).
  bool time_kernel = false;
  using EventPairs = std::vector<std::pair<cudaEvent_t, cudaEvent_t>>;
  EventPairs kernel_events, gather_events, accum_events;
  std::size_t kernel_events_used = 0, gather_events_used = 0, accum_events_used = 0;
  std::uint64_t launches = 0;

  // When timing is on, records the start event of the next pair and returns
  // the end event to record after the timed work (else nullptr).
  cudaEvent_t record_begin(EventPairs& pairs, std::size_t& used, cudaStream_t s) {
    if (!time_kernel) return nullptr;
    if (used == pairs.size()) {
      cudaEvent_t x, y;
      ck(cudaEventCreate(&x), "event");
      ck(cudaEventCreate(&y), "event");
      pairs.emplace_back(x, y);
    }
    auto& ev = pairs[used++];
    ck(cudaEventRecord(ev.first, s), "event record");
    return ev.second;
  }

  static double sum_ms(EventPairs& pairs, std::size_t used) {
    double sum = 0.0;
    for (std::size_t i = 0; i < used; ++i) {
      ck(cudaEventSynchronize(pairs[i].second), "event sync");
      float ms = 0.0f;
      ck(cudaEventElapsedTime(&ms, pairs[i].first, pairs[i].second), "event elapsed");
      sum += ms;
    }
    return sum;
  }

  uint16_t* grads_of(int r) const {
    return reinterpret_cast<uint16_t*>(static_cast<char*>(peer_base[r]) + off_grads);
  }
  uint16_t* params_of(int r) const {
    return reinterpret_cast<uint16_t*>(static_cast<char*>(peer_base[r]) + off_params);
  }
  uint16_t* slot_of(int r, int k) const {
    return reinterpret_cast<uint16_t*>(static_cast<char*>(peer_base[r]) + off_slots +
                                       static_cast<std::size_t>(k & 1) * slot_bytes);
  }
  uint16_t* sec_of(int r) const {
    return reinterpret_cast<uint16_t*>(static_cast<char*>(peer_base[r]) + off_sec);
  }
  uint16_t* acc_of(int r) const {
    return reinterpret_cast<uint16_t*>(static_cast<char*>(peer_base[r]) + off_acc);
  }
  uint32_t* flags_of(int r) const {
    return reinterpret_cast<uint32_t*>(static_cast<char*>(peer_base[r]) + off_flags);
  }
  cudaStream_t pick(void* s) const {
    if (s) return static_cast<cudaStream_t>(s);
    return shared_default ? shared_default : own_stream;
  }
  void use_device() const { ck(cudaSetDevice(cfg.device), "cudaSetDevice"); }

  // Auto (v = 0): the TMA bulk-copy pipeline (variant 5) when every segment
  // is 8-element aligned. For one rank: 3-stage ring, 1 CTA per SM (29.9 ms =
  // 96.8% of measured copy bandwidth on LLaMA-7B, profiles/r01_tune_tma.jsonl).
  // For W > 1 the ring also carries the W-1 NVLink gradient pulls; 2 CTAs per
  // SM (7B ZeRO-1: 21.7 ms vs 23.3 ms for the LDG kernel at W = 2, 30.8 vs
  // 32.3 ms at W = 4; profiles/r01_tma_w_*.json). Unaligned segments fall back
  // to the LDG kernel: one vector in flight, <= 64 registers, 2 CTAs per SM
  // for one rank (profiles/r01_tune_7b.jsonl), the U = 2 kernel otherwise.
  bool segments_aligned() const {
    for (const auto& s : layout.segs)
      if ((s.flat | s.os | s.dst | s.len) & 7u) return false;
    return true;
  }

  void retune(int v, int forced_grid) {
    int g = 0;
    if (v == 0 && segments_aligned()) {
      // Variant 5 needs 2 CTAs per SM to beat the deep single-CTA ring; at
      // W = 8 its 2-stage ring (2 x 57 KB) no longer fits twice, so take 6.
      // Ring-depth / drain sweep on 7B ZeRO-1 (profiles/r01_s2_bulk_*.json,
      // r01_s2_stages*_*.json): W = 2 -> 5 stages with the bulk-store drain
      // (11): 19.25 ms vs 21.0 (7), 21.7 (5), 22.0 (5 stages, no drain);
      // W = 3..4 -> a 4-stage ring at 1 CTA/SM (10): 30.2-30.3 vs 30.3-30.8
      // ms (5); W = 1 -> 3 stages (5): 29.9 vs 30.8 (4 stages), 36.4 (2).
      variant = world == 2                  ? 11
                : (world == 3 || world == 4) ? 10
                : (world > 1 && amsp::fused_blocks_per_sm(world, 5) < 2) ? 6
                                                                          : 5;
      g = world == 1 ? sms : sms * amsp::fused_blocks_per_sm(world, variant);
    } else if (v == 0 && world == 1) {
      variant = 4;
      g = 2 * sms;
    } else {
      variant = v;
      g = sms * amsp::fused_blocks_per_sm(world, variant);
    }
    grid = forced_grid > 0 ? forced_grid : g;
    grid = std::max(1, std::min(ntiles, grid));
  }

  void publish_peer_flags() {
    uint32_t* h[amsp::kMaxRanks] = {};
    for (int r = 0; r < world; ++r) h[r] = flags_of(r);
    ck(cudaMemcpy(d_peer_flags, h, sizeof(h), cudaMemcpyHostToDevice),
       "copy peer flag table");
  }

  void barrier(cudaStream_t s) {
    if (!synced()) return;
    ++epoch;
    // ids 0/1 alternate (pre / post); the epoch keeps each id monotonic.
    ck(amsp::launch_barrier(d_peer_flags, world, rank, static_cast<int>(epoch & 1), epoch, err, s),
       "barrier launch");
    ++launches;
  }

  void check_err() {
    int h[5] = {};
    ck(cudaMemcpy(h, err, sizeof(h), cudaMemcpyDeviceToHost), "read error flag");
    if (h[0])
      throw amsp::CudaFailure(
          "cross-GPU barrier timed out (a peer did not arrive): rank " + std::to_string(rank) +
          " barrier id " + std::to_string(h[1]) + " (ids >= 16: scheduler) epoch " +
          std::to_string(h[2]) + ", peer " + std::to_string(h[3]) + " at epoch " +
          std::to_string(h[4]));
  }

  // Host-buffer step (s_p = 1), pipelined: the gradient upload is cut into
  // chunks of the flat index space on a copy stream, and the fused update of
  // chunk c runs as soon as chunk c has landed, so the PCIe copy hides the
  // update. With W > 1 a cross-GPU barrier per chunk proves every rank's
  // chunk c is resident before the owners pull it; a final barrier proves
  // every owner's parameter stores have landed.
  static constexpr std::uint64_t kHostChunk = std::uint64_t{1} << 28;  // elements (512 MB)
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> chunk_events;
  std::vector<int> chunk_begin, chunk_nseg, chunk_ntiles;
  amsp::Seg* d_chunk_segs = nullptr;

  void build_chunks() {
    std::vector<amsp::Seg> segs;
    for (std::uint64_t lo = 0; lo < phi; lo += kHostChunk) {
      const std::uint64_t hi = std::min(phi, lo + kHostChunk);
      chunk_begin.push_back(static_cast<int>(segs.size()));
      long long tiles = 0;
      for (const auto& s : layout.segs) {
        const std::uint64_t a = std::max(lo, s.flat), b = std::min(hi, s.flat + s.len);
        if (a >= b) continue;
        const std::uint64_t off = a - s.flat;
        segs.push_back({a, s.os + off, s.dst + off, b - a, static_cast<unsigned long long>(tiles)});
        tiles += static_cast<long long>((b - a + amsp::kTile - 1) / amsp::kTile);
      }
      chunk_nseg.push_back(static_cast<int>(segs.size()) - chunk_begin.back());
      chunk_ntiles.push_back(static_cast<int>(tiles));
    }
    ck(cudaMalloc(&d_chunk_segs, std::max<std::size_t>(segs.size(), 1) * sizeof(amsp::Seg)),
       "cudaMalloc chunk segs");
    ck(cudaMemcpy(d_chunk_segs, segs.data(), segs.size() * sizeof(amsp::Seg),
                  cudaMemcpyHostToDevice),
       "copy chunk segs");
    ck(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking), "copy stream");
    chunk_events.resize(chunk_begin.size());
    for (auto& ev : chunk_events)
      ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
  }

  void step_host_pipelined(int t, const void* host, cudaStream_t s) {
    if (sp != 1) throw Error("engine: the pipelined host step needs s_p = 1");
    require_peers();
    if (chunk_begin.empty()) build_chunks();
    const char* src = static_cast<const char*>(host);
    char* dst = reinterpret_cast<char*>(grads_of(rank));
    ck(cudaMemsetAsync(stats, 0, 2 * sizeof(float), s), "reset stats");
    // The copies must not overwrite gradients the previous work still reads
    // (for W > 1 the previous step ended with a barrier after every pull).
    ck(cudaEventRecord(chunk_events[0], s), "event record");
    ck(cudaStreamWaitEvent(copy_stream, chunk_events[0], 0), "stream wait");
    amsp::FusedArgs a{};
    for (int r = 0; r < world; ++r) a.grads[r] = grads_of(r);
    a.ndst = static_cast<int>(dst_members.size());
    for (int d = 0; d < a.ndst; ++d) a.dsts[d] = params_of(dst_members[d]);
    a.master = master;
    a.exp_avg = exp_avg;
    a.exp_avg_sq = exp_avg_sq;
    a.s = amsp::make_adam_scalars(cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.weight_decay, t,
                                  grad_scale());
    a.stats = stats;
    a.fence_peers = synced() ? 1 : 0;
    for (std::size_t c = 0; c < chunk_begin.size(); ++c) {
      const std::uint64_t lo = c * kHostChunk, n = std::min(kHostChunk, phi - lo);
      ck(cudaMemcpyAsync(dst + lo * 2, src + lo * 2, n * 2, cudaMemcpyHostToDevice, copy_stream),
         "H2D gradients");
      ck(cudaEventRecord(chunk_events[c], copy_stream), "event record");
      ck(cudaStreamWaitEvent(s, chunk_events[c], 0), "stream wait");
      barrier(s);  // chunk c of every rank is resident
      a.segs = d_chunk_segs + chunk_begin[c];
      a.nseg = chunk_nseg[c];
      a.ntiles = chunk_ntiles[c];
      if (a.ntiles > 0) {
        ck(amsp::launch_fused_step(a, world, std::max(1, std::min(a.ntiles, grid)), variant, s),
           "fused step launch");
        ++launches;
      }
    }
    barrier(s);  // every owner's parameter stores have landed
  }

  void require_peers() const {
    if (world > 1 && !imported)
      throw Error("engine: peers not imported (amsp_engine_import_handles)");
  }

  // AG of one gather unit into `dst` (default: slot `slot`; s_p > 1), from
  // the P shards of the P group, or with `secondary` from the secondary
  // shards of the secondary group (the ZeRO++ backward all-gather).
  void gather(int unit, int slot, cudaStream_t s, bool secondary = false,
              uint16_t* dst = nullptr, bool refresh = false) {
    if (sp == 1) throw Error("engine: gather needs parameter sharding (s_p > 1)");
    if (unit < 0 || unit >= static_cast<int>(units.size()))
      throw Error("engine: gather unit out of range");
    if (secondary && s2 == 1) throw Error("engine: no secondary parameter mesh");
    require_peers();
    const GatherUnit& u = secondary ? units2[static_cast<std::size_t>(unit)] : units[unit];
    const int n = secondary ? s2 : sp;
    const amsp::MeshGroup& grp = secondary ? sec_group : p_group;
    const amsp::PShardMap& map = secondary ? smap : pmap;
    if (!dst) dst = slots[slot & 1];
    auto src_of = [&](int q) {
      return secondary ? sec_of(grp.members[q]) : params_of(grp.members[q]);
    };
    if (gather_grid == kGatherDma || (refresh && !sec_fused)) {
      // Copy-engine all-gather: per tensor of the unit, one peer-to-local
      // DMA per group member (rotated start), no SMs involved.
      const std::uint64_t base = pmap.tensor_offset[u.first_tensor];
      for (int i = 0; i < u.n_tensors; ++i) {
        const std::size_t t = static_cast<std::size_t>(u.first_tensor + i);
        const std::uint64_t len = map.slice_len[t];
        for (int j = 0; j < n; ++j) {
          const int q = (grp.position + 1 + j) % n;
          ck(cudaMemcpyAsync(dst + (pmap.tensor_offset[t] - base) + q * len,
                             src_of(q) + map.pshard_offset[t], len * 2,
                             cudaMemcpyDeviceToDevice, s),
             "gather DMA");
        }
        if (refresh)
          refresh_secondary_tensor(static_cast<int>(t), dst + (pmap.tensor_offset[t] - base), s);
      }
      return;
    }
    amsp::GatherArgs g{};
    if (refresh) {
      g.sec = sec_of(rank);
      g.s2 = s2;
      g.pos2 = sec_group.position;
    }
    g.segs = d_copy + u.seg_begin;
    g.nseg = u.nseg;
    g.ntiles = u.ntiles;
    for (int q = 0; q < n; ++q) g.src[q] = src_of(q);
    g.dst = dst;
    g.grid = gather_grid > 0 ? gather_grid : 0;
    g.sp = n;
    g.rot = (grp.position + 1) % n;
    // (the push mode applies to the step's passes; a single gather pulls)
    const bool tma = gather_grid == kGatherTma || gather_grid == kGatherPush;
    ck(tma ? amsp::launch_gather_tma(g, s) : amsp::launch_gather(g, s), "gather launch");
    ++launches;
  }

  // Push all-gather of one unit (engine step only): this rank's P slice of
  // every tensor of the unit into slot `slot` of every P-group member.
  void push(int unit, int slot, cudaStream_t s) {
    const GatherUnit& u = units_push[static_cast<std::size_t>(unit)];
    amsp::PushArgs a{};
    a.segs = d_copy + u.seg_begin;
    a.nseg = u.nseg;
    a.ntiles = u.ntiles;
    a.sp = sp;
    a.q = p_group.position;
    a.src = params_of(rank);
    for (int j = 0; j < sp; ++j) a.dst[j] = slot_of(p_group.members[j], slot);
    a.fence_peers = synced() ? 1 : 0;
    ck(amsp::launch_push_tma(a, s), "push gather launch");
    ++launches;
  }

  // ZeRO++: keep this rank's secondary slice of tensor t from the gathered
  // tensor (a local copy; used when the gather cannot store it itself).
  void refresh_secondary_tensor(int t, const uint16_t* gathered, cudaStream_t s) {
    const std::uint64_t len = smap.slice_len[static_cast<std::size_t>(t)];
    ck(cudaMemcpyAsync(sec_of(rank) + smap.pshard_offset[static_cast<std::size_t>(t)],
                       gathered + static_cast<std::uint64_t>(sec_group.position) * len, len * 2,
                       cudaMemcpyDeviceToDevice, s),
       "secondary refresh");
  }

  // The step's gradient is the mean over W ranks x M micro-batches.
  double grad_scale() const { return 1.0 / (static_cast<double>(world) * micro); }

  template <class P>
  void set_acc(P* acc, int* nacc, int* by_dst) const {
    *nacc = static_cast<int>(acc_holders.size());
    for (int j = 0; j < *nacc; ++j) acc[j] = acc_of(acc_holders[j]);
    *by_dst = acc_by_dst ? 1 : 0;
  }

  void check_micro_batch(int mb) const {
    if (mb < 0 || mb >= micro)
      throw Error("engine: micro-batch " + std::to_string(mb) + " outside 0.." +
                  std::to_string(micro - 1));
  }

  // Micro-batch mb (< M-1) of every rank is in the gradient buffers: fold it
  // into the G-shard accumulators (s_g > 1; with s_g = 1 the producer has
  // accumulated in place and there is nothing to move).
  void accumulate(int mb, cudaStream_t s) {
    check_micro_batch(mb);
    if (mb == micro - 1) throw Error("engine: the last micro-batch goes through the step");
    require_peers();
    if (!staged) return;
    amsp::AccumArgs a{};
    a.segs = d_acc_segs;
    a.nseg = nacc_seg;
    a.ntiles = nacc_tiles;
    a.nsrc = static_cast<int>(acc_sources.size());
    for (int q = 0; q < a.nsrc; ++q) a.grads[q] = grads_of(acc_sources[q]);
    a.acc = acc_of(rank);
    a.first = mb == 0 ? 1 : 0;
    a.fence_peers = 0;  // local stores only; the trailing barrier orders them
    barrier(s);  // micro-batch mb is complete on every rank
    cudaEvent_t t_end =
        nacc_tiles > 0 ? record_begin(accum_events, accum_events_used, s) : nullptr;
    ck(amsp::launch_accumulate(a, sms * 4, s), "accumulate launch");
    if (t_end) ck(cudaEventRecord(t_end, s), "event record");
    if (nacc_tiles > 0) ++launches;
    barrier(s);  // every holder has pulled: the gradient buffers may be rewritten
  }

  void step(int t, cudaStream_t s) {
    if (t < 1) throw Error("engine: step index must be >= 1");
    require_peers();
    if (sp > 1 && !cfg.skip_gathers) {
      // Forward then backward parameter all-gathers (T_p's two AG terms,
      // cost_model.cpp:46-49); RS is fused into the optimizer kernel below.
      cudaEvent_t g_end = record_begin(gather_events, gather_events_used, s);
      const int n = static_cast<int>(units.size());
      if (gather_grid == kGatherPush && s2 == 1) {
        // push all-gather: every rank stores its own slice of each unit into
        // every P-group member's slot (NVLink stores); the slots are complete
        // at the barrier that follows the passes
        for (int u = 0; u < n; ++u) push(u, u, s);
        for (int u = n - 1; u >= 0; --u) push(u, u, s);
      } else {
        // (ZeRO++ pulls: the receiver keeps its secondary slice from its own
        // gathered tensor, a local store; pushing it into the members'
        // secondary buffers doubled the NVLink egress -- 97.4 vs 80.0 ms on
        // 13B at W = 4, profiles/r02_zeropp_push_vs_pull_13b.jsonl)
        for (int u = 0; u < n; ++u) gather(u, u, s, false, nullptr, s2 > 1);
        // ZeRO++: every rank's secondary slices are in place before the
        // backward all-gathers read them from the secondary group
        if (s2 > 1) barrier(s);
        for (int u = n - 1; u >= 0; --u) gather(u, u, s, s2 > 1);
      }
      if (g_end) ck(cudaEventRecord(g_end, s), "event record");
    }
    amsp::FusedArgs a{};
    a.segs = d_segs;
    a.nseg = nseg;
    a.ntiles = ntiles;
    for (int r = 0; r < world; ++r) a.grads[r] = grads_of(r);
    a.ndst = static_cast<int>(dst_members.size());
    for (int d = 0; d < a.ndst; ++d) a.dsts[d] = params_of(dst_members[d]);
    a.master = master;
    a.exp_avg = exp_avg;
    a.exp_avg_sq = exp_avg_sq;
    a.s = amsp::make_adam_scalars(cfg.lr, cfg.beta1, cfg.beta2, cfg.eps,
                                  cfg.weight_decay, t, grad_scale());
    a.stats = stats;
    a.fence_peers = synced() ? 1 : 0;
    int v = variant, g = grid;
    if (staged) {
      // the holders' accumulators first, then the raw last micro-batch
      set_acc(a.acc, &a.nacc, &a.acc_by_dst);
      const int acc_blocks = v >= 5 ? amsp::tma_acc_blocks_per_sm(world, v) : 0;
      if (acc_blocks > 0) {  // TMA ring with W + W/2 source slots per stage
        g = std::max(1, std::min(ntiles, sms * acc_blocks));
      } else if (v >= 5) {   // no accumulator instantiation: the LDG kernels
        v = world <= 4 ? 2 : 1;
        g = std::max(1, std::min(ntiles, sms * amsp::fused_blocks_per_sm(world, v)));
      }
    }
    ck(cudaMemsetAsync(stats, 0, 2 * sizeof(float), s), "reset stats");
    barrier(s);  // every rank's gradients are complete
    cudaEvent_t t_end =
        ntiles > 0 ? record_begin(kernel_events, kernel_events_used, s) : nullptr;
    ck(amsp::launch_fused_step(a, world, g, v, s), "fused step launch");
    if (t_end) ck(cudaEventRecord(t_end, s), "event record");
    if (ntiles > 0) ++launches;
    barrier(s);  // every owner's parameter stores have landed
  }
};

