// Host-side interface of the AMSP step kernels (kernels.cu), used by the
// engine (engine.cpp) and the raw C-ABI launchers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>


namespace amsp {

// Step-constant AdamW scalars, computed on the host in double and rounded
// once to float (same expression as amsp_o_adam_scalars()).
struct AdamScalars {
  float beta1, omb1, beta2, omb2;
  float step_size, inv_sqrt_bc2, eps, decay, grad_scale;
};

// One contiguous run of a rank's optimizer-state shard: flat elements
// [flat, flat+len) of the parameter vector, stored at os..os+len of the
// shard; tile0 = index of the segment's first kTile-element tile.
struct Seg {
  unsigned long long flat, os, dst, len, tile0;
};

// One tensor of an all-gather unit: every P-group member q holds its slice
// (len elements) at src of its P shard; slice q lands at dst + q*len of the
// gathered buffer. Tiles interleave the sources: tile v of the tensor copies
// chunk v / s_p from source (rot + v % s_p) % s_p, so at every instant a rank
// pulls evenly from all peers (no NVLink egress hot spot when ranks drift).
struct CopySeg {
  unsigned long long dst, src, len, tile0;
  unsigned long long sec;  // ZeRO++: offset of the tensor's slice in the secondary buffer
};

struct GatherArgs {
  const CopySeg* segs;  // this unit's tensors
  int nseg;
  int ntiles;
  int sp;               // P-group size
  int rot;              // source rotation (this rank's P position + 1)
  const uint16_t* src[8];  // P shards of the P-group members, position order
  uint16_t* dst;           // gathered unit buffer (local)
  int grid;                // CTAs (0 = 4 per SM)
  // ZeRO++ forward gather (sec != nullptr): every element of the tensor that
  // falls in this rank's secondary slice [pos2*L/s2, (pos2+1)*L/s2) is also
  // stored at sec + seg.sec + (index - pos2*L/s2) -- the secondary refresh
  // fused into the gather (no second read). L = len * sp; slices 8-aligned.
  uint16_t* sec;
  int s2, pos2;
};

// Push all-gather of one unit: this rank's slice q of every tensor (segs:
// dst = tensor offset in the unit, src = slice offset in the P shard, len =
// slice length, tile0 over ceil(len / kTile) tiles per tensor) is stored at
// dst[j] + seg.dst + q * len for every P-group member j (local or peer).
struct PushArgs {
  const CopySeg* segs;
  int nseg;
  int ntiles;
  int sp, q;
  const uint16_t* src;  // this rank's P shard (local HBM)
  uint16_t* dst[8];     // the members' slots, position order
  int fence_peers;
};

constexpr int kBlock = 256;
constexpr int kVecPerThread = 2;               // 8-element vectors per thread per tile
constexpr unsigned long long kTile = kBlock * 8ull * kVecPerThread;  // 4096
constexpr int kMaxRanks = 8;                   // NVSwitch domain of one HGX B200

// Arguments of the fused reduce + AdamW + gather kernel.
struct FusedArgs {
  const Seg* segs;
  int nseg;
  int ntiles;
  const uint16_t* grads[kMaxRanks];  // bf16 [Phi] of every DP rank, DP order
  uint16_t* dsts[kMaxRanks];         // bf16 [Phi] params of every OS-group rank
  int ndst;
  float* master;
  float* exp_avg;
  float* exp_avg_sq;
  AdamScalars s;
  float* stats;                      // += sum(g^2); may be null
  int fence_peers;                   // membar.sys before exit (peer stores)
  // Micro-batch accumulators (M > 1, s_g > 1): the bf16 G shards of the
  // accumulation-block holders of these elements, summed in this order
  // BEFORE the raw gradients; indexed by Seg::dst (s_g = s_p) or Seg::os.
  // LDG kernels only (nacc = 0 for the TMA variants).
  const uint16_t* acc[kMaxRanks];
  int nacc;
  int acc_by_dst;
};

AdamScalars make_adam_scalars(double lr, double beta1, double beta2, double eps,
                              double weight_decay, int step, double grad_scale);

// Blocks per SM the fused kernel sustains for `world` gradient sources and
// tuning `variant` (kernels.cu: 0 = auto).
int fused_blocks_per_sm(int world, int variant);
// CTAs per SM of the TMA variant's accumulator-source instantiation (M > 1,
// s_g > 1; W in {2, 4, 6, 8}, variants 5 / 10 / 11), 0 when there is none.
int tma_acc_blocks_per_sm(int world, int variant);

cudaError_t launch_fused_step(const FusedArgs& a, int world, int grid, int variant,
                              cudaStream_t stream);
// Barrier `id` (0 .. kBarrierIds-1): flag words [id*kMaxRanks, +world).
constexpr int kBarrierIds = 8192;
cudaError_t launch_barrier(uint32_t* const* peer_flags, int world, int rank, int id,
                           uint32_t epoch, int* err, cudaStream_t stream);

// Split form of the fused step, used by the overlap scheduler: the reduce
// runs per gradient bucket / module during backward into an fp32 shard
// buffer; AdamW + parameter push runs once after the step's barrier.
struct ReduceArgs {
  const Seg* segs;   // os = offset in the fp32 reduced-gradient shard
  int nseg;
  int ntiles;
  const uint16_t* grads[kMaxRanks];
  float* red;
  float scale;
  const uint16_t* acc[kMaxRanks];  // as FusedArgs::acc
  int nacc;
  int acc_by_dst;
};
// Micro-batch gradient accumulation (non-last micro-batch, s_g > 1; PAPER.md:
// 320-326): for every element of this rank's G shard, pull the bf16
// gradients of the nsrc ranks of its accumulation block (ascending rank) and
// fold them into the local bf16 accumulator: acc[os] = bf16((first ? 0 :
// acc[os]) + sum_q grads_q[flat]) -- the reduce-scatter / AllReduce + select
// & drop of the micro-batch in one pass. Seg::os = accumulator offset.
struct AccumArgs {
  const Seg* segs;
  int nseg;
  int ntiles;
  const uint16_t* grads[kMaxRanks];
  int nsrc;
  uint16_t* acc;
  int first;
  int fence_peers;
};
cudaError_t launch_accumulate(const AccumArgs& a, int grid, cudaStream_t stream);
// NVLink peer-read probe: pull vecs_per_src 16-byte vectors from each of
// nsrc (peer) buffers into a local buffer, interleaved across the sources in
// 512-byte warp chunks (rotated by `rot`) -- the all-to-all pull pattern of
// the fused step's gradient reduce, with nothing else in the way.
struct PullArgs {
  const uint4* src[kMaxRanks];
  int nsrc;
  int rot;
  uint4* dst;
  unsigned long long vecs_per_src;
};
cudaError_t launch_p2p_pull(const PullArgs& a, int grid, cudaStream_t stream);
struct AdamPushArgs {
  const Seg* segs;
  int nseg;
  int ntiles;
  const float* red;
  uint16_t* dsts[kMaxRanks];
  int ndst;
  float* master;
  float* exp_avg;
  float* exp_avg_sq;
  AdamScalars s;
  int fence_peers;
};
cudaError_t launch_reduce(const ReduceArgs& a, int world, int grid, cudaStream_t stream);
cudaError_t launch_adam_push(const AdamPushArgs& a, int grid, cudaStream_t stream);
int adam_push_blocks_per_sm();
// Compute stand-in: `ctas` CTAs, each busy for `ns` nanoseconds of FMA work.
cudaError_t launch_spin(int ctas, unsigned long long ns, cudaStream_t stream);
// params[dst+k] = bf16(master_init(flat+k)) over a P-shard segment table.
cudaError_t launch_init_params(const Seg* psegs, int nseg, int ntiles, uint16_t* params,
                               uint64_t seed, cudaStream_t stream);
cudaError_t launch_gather(const GatherArgs& a, cudaStream_t stream);
// Bulk-copy (TMA) variant of launch_gather: 32-thread CTAs, every CopySeg
// 8-element aligned (see kernels.cu gather_tma_kernel).
cudaError_t launch_gather_tma(const GatherArgs& a, cudaStream_t stream);
// Push all-gather (TMA bulk copies: local load, NVLink bulk stores).
cudaError_t launch_push_tma(const PushArgs& a, cudaStream_t stream);
cudaError_t launch_init_state(const Seg* segs, int nseg, int ntiles, float* master,
                              float* m, float* v, uint64_t seed, int grid,
                              cudaStream_t stream);
cudaError_t launch_synth_grad(uint16_t* dst, unsigned long long start,
                              unsigned long long n, uint64_t seed, int step,
                              int rank, cudaStream_t stream, int mb = 0,
                              bool accumulate = false);
cudaError_t launch_adamw_flat(const void* grad, bool bf16_grad, float* master,
                              float* m, float* v, uint16_t* param_out,
                              unsigned long long n, const AdamScalars& s,
                              cudaStream_t stream);
cudaError_t launch_rs_upcast_scale(const uint16_t* const* srcs, int nsrc,
                                   unsigned long long offset, float* dst,
                                   unsigned long long n, float scale, cudaStream_t stream);
cudaError_t launch_ag_downcast(const float* src, unsigned long long n, uint16_t* const* dsts,
                               int ndst, unsigned long long dst_offset, cudaStream_t stream);
cudaError_t launch_upcast_scale(const uint16_t* src, float* dst,
                                unsigned long long n, float scale,
                                cudaStream_t stream);

}  // namespace amsp
