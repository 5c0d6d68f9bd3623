// AMSP step kernels for B200 (sm_100a).
//
// The hot op is fused_step_kernel: for every element of this rank's
// optimizer-state shard it
//   1. pulls the bf16 gradient of every data-parallel rank over NVLink
//      (peer pointers mapped with cudaIpc), sums them in fp32 in a fixed
//      rank order and scales by 1/W  — the reduce-scatter inside the OS
//      group plus the cross-replica sum, with select & drop implicit
//      (cost_model.cpp:98-105 charges it as AR + drop);
//   2. applies AdamW to the fp32 master / m / v shard (HBM-bound);
//   3. downcasts the new master to bf16 and stores it into the parameter
//      buffer of every rank of the OS group — the all-gather / inter-tensor
//      broadcast of updated shards (cost_model.cpp:107-117), written
//      straight into each peer's gathered buffer.
// One launch therefore replaces AR(or RS) + upcast + Adam + downcast + AG.
// There is no tensor-core work (no contraction): the kernel is bounded by
// HBM and NVLink bandwidth and is written as a persistent grid of 256-thread
// CTAs streaming 128-bit vectors with several independent loads in flight.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace amsp {

AdamScalars make_adam_scalars(double lr, double beta1, double beta2, double eps,
                              double weight_decay, int step, double grad_scale) {
  const double bc1 = 1.0 - std::pow(beta1, static_cast<double>(step));
  const double bc2 = 1.0 - std::pow(beta2, static_cast<double>(step));
  AdamScalars s;
  s.beta1 = static_cast<float>(beta1);
  s.omb1 = static_cast<float>(1.0 - beta1);
  s.beta2 = static_cast<float>(beta2);
  s.omb2 = static_cast<float>(1.0 - beta2);
  s.step_size = static_cast<float>(lr / bc1);
  s.inv_sqrt_bc2 = static_cast<float>(1.0 / std::sqrt(bc2));
  s.eps = static_cast<float>(eps);
  s.decay = static_cast<float>(1.0 - lr * weight_decay);
  s.grad_scale = static_cast<float>(grad_scale);
  return s;
}

namespace {

// Segment owning `tile` (largest s with segs[s].tile0 <= tile).
__device__ __forceinline__ Seg find_seg(const Seg* segs, int nseg, int tile) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(&segs[mid].tile0) <= static_cast<unsigned long long>(tile))
      lo = mid;
    else
      hi = mid - 1;
  }
  Seg s;
  s.flat = __ldg(&segs[lo].flat);
  s.os = __ldg(&segs[lo].os);
  s.dst = __ldg(&segs[lo].dst);
  s.len = __ldg(&segs[lo].len);
  s.tile0 = __ldg(&segs[lo].tile0);
  return s;
}

// Segment lookup for persistent grid-stride loops: the table is staged in
// shared memory once per CTA (when it fits) and, since a CTA visits tiles in
// increasing order, the owning segment is found by advancing a cursor —
// no dependent global-memory search chain in front of every tile's loads.
template <class T, int CAP>
struct SegCursor {
  const T* table;
  int n, cur;
  bool staged;

  __device__ void init(T* smem, const T* global, int nseg) {
    n = nseg;
    cur = 0;
    staged = nseg <= CAP;
    if (staged) {
      const unsigned long long* src = reinterpret_cast<const unsigned long long*>(global);
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(smem);
      constexpr int kWords = sizeof(T) / 8;
      for (int i = threadIdx.x; i < nseg * kWords; i += blockDim.x) dst[i] = src[i];
      __syncthreads();
      table = smem;
    } else {
      table = global;
    }
  }

  __device__ const T& at(int tile) {
    const unsigned long long t = static_cast<unsigned long long>(tile);
    if (staged) {
      while (cur + 1 < n && table[cur + 1].tile0 <= t) ++cur;
    } else {
      int lo = cur, hi = n - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (table[mid].tile0 <= t) lo = mid; else hi = mid - 1;
      }
      cur = lo;
    }
    return table[cur];
  }
};

constexpr int kSegCap = 384;    // 15 KB of Seg in shared memory
constexpr int kCopyCap = 256;   // 10 KB of CopySeg

// Unscaled gradient of one element: the micro-batch accumulators (if any)
// in holder order, then the raw gradients in rank order (oracle recipe).
template <int W, class Args>
__device__ __forceinline__ float reduce_scalar(const Args& a, unsigned long long idx,
                                               unsigned long long acc_idx) {
  float g;
  int r0 = 0;
  if (a.nacc > 0) {
    g = bf16_at(a.acc[0][acc_idx]);
    for (int j = 1; j < a.nacc; ++j) g = __fadd_rn(g, bf16_at(a.acc[j][acc_idx]));
  } else {
    g = bf16_at(a.grads[0][idx]);
    r0 = 1;
  }
#pragma unroll
  for (int r = 0; r < W; ++r)
    if (r >= r0) g = __fadd_rn(g, bf16_at(a.grads[r][idx]));
  return g;
}

// Sum of the accumulators of 8 consecutive elements (vector path).
template <class Args>
__device__ __forceinline__ void acc_vec(const Args& a, unsigned long long acc_idx, float* out) {
  const uint4 w0 = ld_ro_v4(a.acc[0] + acc_idx);
  const uint32_t* u0 = reinterpret_cast<const uint32_t*>(&w0);
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    out[2 * w] = bf16_lo(u0[w]);
    out[2 * w + 1] = bf16_hi(u0[w]);
  }
  for (int j = 1; j < a.nacc; ++j) {
    const uint4 wj = ld_ro_v4(a.acc[j] + acc_idx);
    const uint32_t* uj = reinterpret_cast<const uint32_t*>(&wj);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      out[2 * w] = __fadd_rn(out[2 * w], bf16_lo(uj[w]));
      out[2 * w + 1] = __fadd_rn(out[2 * w + 1], bf16_hi(uj[w]));
    }
  }
}

// Element-wise path for ragged tails and unaligned segments.
template <int W>
__device__ void scalar_elems(const FusedArgs& a, const Seg& sg,
                             unsigned long long e, float& sq) {
  const unsigned long long end = e + 8 < sg.len ? e + 8 : sg.len;
  for (; e < end; ++e) {
    const unsigned long long f = sg.flat + e, o = sg.os + e;
    const float g = __fmul_rn(reduce_scalar<W>(a, f, (a.acc_by_dst ? sg.dst : sg.os) + e),
                              a.s.grad_scale);
    float p = a.master[o], m = a.exp_avg[o], v = a.exp_avg_sq[o];
    adamw(a.s, g, p, m, v);
    a.master[o] = p;
    a.exp_avg[o] = m;
    a.exp_avg_sq[o] = v;
    const uint16_t b = to_bf16(p);
    for (int d = 0; d < a.ndst; ++d) a.dsts[d][sg.dst + e] = b;
    sq += g * g;
  }
}

// U = 8-element vectors with all loads in flight before any math.
template <int W, int U, int MINB>
__global__ void __launch_bounds__(kBlock, MINB)
fused_step_kernel(const FusedArgs a) {
  __shared__ Seg s_segs[kSegCap];
  SegCursor<Seg, kSegCap> cursor;
  cursor.init(s_segs, a.segs, a.nseg);
  float sq = 0.0f;
  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const Seg sg = cursor.at(tile);
    const unsigned long long base =
        (static_cast<unsigned long long>(tile) - sg.tile0) * kTile;
    const bool aligned = ((sg.flat | sg.os | sg.dst) & 7ull) == 0;
#pragma unroll 1
    for (int it = 0; it < kVecPerThread; it += U) {
      unsigned long long e[U];
      bool full[U];
      uint4 graw[U][W];
      float4 p[U][2], m[U][2], v[U][2];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        e[u] = base + (static_cast<unsigned long long>(it + u) * kBlock + threadIdx.x) * 8ull;
        full[u] = aligned && e[u] + 8 <= sg.len;
        if (full[u]) {
          const unsigned long long f = sg.flat + e[u], o = sg.os + e[u];
#pragma unroll
          for (int r = 0; r < W; ++r) graw[u][r] = ld_ro_v4(a.grads[r] + f);
          p[u][0] = ld_state_v4(a.master + o);
          p[u][1] = ld_state_v4(a.master + o + 4);
          m[u][0] = ld_state_v4(a.exp_avg + o);
          m[u][1] = ld_state_v4(a.exp_avg + o + 4);
          v[u][0] = ld_state_v4(a.exp_avg_sq + o);
          v[u][1] = ld_state_v4(a.exp_avg_sq + o + 4);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (full[u]) {
          const unsigned long long f = sg.flat + e[u], o = sg.os + e[u];
          float* pf = reinterpret_cast<float*>(&p[u][0]);
          float* mf = reinterpret_cast<float*>(&m[u][0]);
          float* vf = reinterpret_cast<float*>(&v[u][0]);
          uint32_t packed[4];
          float accs[8];
          if (a.nacc > 0) acc_vec(a, (a.acc_by_dst ? sg.dst : sg.os) + e[u], accs);
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const uint32_t* g0 = reinterpret_cast<const uint32_t*>(&graw[u][0]);
            float glo = bf16_lo(g0[w]), ghi = bf16_hi(g0[w]);
            if (a.nacc > 0) {
              glo = __fadd_rn(accs[2 * w], glo);
              ghi = __fadd_rn(accs[2 * w + 1], ghi);
            }
#pragma unroll
            for (int r = 1; r < W; ++r) {
              const uint32_t* gr = reinterpret_cast<const uint32_t*>(&graw[u][r]);
              glo = __fadd_rn(glo, bf16_lo(gr[w]));
              ghi = __fadd_rn(ghi, bf16_hi(gr[w]));
            }
            glo = __fmul_rn(glo, a.s.grad_scale);
            ghi = __fmul_rn(ghi, a.s.grad_scale);
            sq += glo * glo + ghi * ghi;
            // Element order inside the vector: 2w, 2w+1 (p/m/v are float4 x2
            // laid out contiguously in registers).
            const int j = 2 * w;
            adamw(a.s, glo, pf[j], mf[j], vf[j]);
            adamw(a.s, ghi, pf[j + 1], mf[j + 1], vf[j + 1]);
            packed[w] = pack_bf16x2(pf[j], pf[j + 1]);
          }
          st_stream_v4(a.master + o, p[u][0]);
          st_stream_v4(a.master + o + 4, p[u][1]);
          st_stream_v4(a.exp_avg + o, m[u][0]);
          st_stream_v4(a.exp_avg + o + 4, m[u][1]);
          st_stream_v4(a.exp_avg_sq + o, v[u][0]);
          st_stream_v4(a.exp_avg_sq + o + 4, v[u][1]);
          const uint4 out = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          for (int d = 0; d < a.ndst; ++d) st_v4(a.dsts[d] + sg.dst + e[u], out);
        } else if (e[u] < sg.len) {
          scalar_elems<W>(a, sg, e[u], sq);
        }
      }
    }
  }
  // Peer parameter stores must be visible system-wide before the trailing
  // cross-GPU barrier releases the other ranks.
  if (a.fence_peers) __threadfence_system();
  if (a.stats != nullptr) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    __shared__ float part[kBlock / 32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.0f;
      for (int i = 0; i < kBlock / 32; ++i) t += part[i];
      atomicAdd(a.stats, t);
    }
  }
}

// Cross-GPU barrier over NVLink. Barrier `id` owns kMaxRanks flag words in
// every rank's flag array: thread r publishes this rank's epoch into rank
// r's word [id][rank] and waits until its own word [id][r] reaches the
// epoch. Distinct ids never interfere, so barriers issued on different
// streams may complete in any order. Bounded wait: after ~20 s it raises
// *err instead of hanging; once *err is set (by this or an earlier barrier
// of the rank) every later barrier gives up at once, so a lost peer costs
// one timeout, not one per barrier of the step.
__global__ void barrier_kernel(uint32_t* const* peer_flags, int world, int rank, int id,
                               uint32_t epoch, int* err) {
  const int t = threadIdx.x;
  __threadfence_system();
  if (t < world) {
    uint32_t* slot = peer_flags[t] + id * kMaxRanks + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(slot), "r"(epoch)
                 : "memory");
    const uint32_t* mine = peer_flags[rank] + id * kMaxRanks + t;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      uint32_t seen;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];"
                   : "=r"(seen)
                   : "l"(mine)
                   : "memory");
      if (static_cast<int32_t>(seen - epoch) >= 0) break;
      if (*reinterpret_cast<volatile int*>(err)) break;
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 20000000000ull) {
        // diagnostics for the host: which barrier, epoch, the late peer and
        // the epoch it had reached (the first timeout of the rank wins)
        if (atomicCAS(err, 0, 1) == 0) {
          err[1] = id;
          err[2] = static_cast<int>(epoch);
          err[3] = t;
          err[4] = static_cast<int>(seen);
        }
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

__global__ void init_params_kernel(const Seg* segs, int nseg, int ntiles,
                                   uint16_t* __restrict__ p, uint64_t seed) {
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const Seg sg = find_seg(segs, nseg, tile);
    const unsigned long long base =
        (static_cast<unsigned long long>(tile) - sg.tile0) * kTile;
    for (unsigned long long e = base + threadIdx.x; e < base + kTile && e < sg.len;
         e += blockDim.x)
      p[sg.dst + e] = to_bf16(master_init(seed, sg.flat + e));
  }
}

// All-gather of one unit (a run of tensors) from the P shards of the P group
// into a local gathered buffer: pure NVLink pulls, 128-bit when aligned.
__global__ void __launch_bounds__(256) gather_kernel(const GatherArgs a) {
  __shared__ CopySeg s_segs[kCopyCap];
  __shared__ const uint16_t* s_src[8];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) s_src[q] = a.src[q];  // constant indices: no local copy
  }
  SegCursor<CopySeg, kCopyCap> cursor;
  cursor.init(s_segs, a.segs, a.nseg);  // includes a __syncthreads when staged
  __syncthreads();
  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const CopySeg& cs = cursor.at(tile);
    const unsigned long long v = static_cast<unsigned long long>(tile) - cs.tile0;
    const unsigned long long chunk = v / a.sp;
    const int q = static_cast<int>((v % a.sp + a.rot) % a.sp);
    const unsigned long long len = cs.len, src = cs.src;
    const unsigned long long dst = cs.dst + static_cast<unsigned long long>(q) * len;
    const uint16_t* from = s_src[q];
    const unsigned long long base = chunk * kTile;
    if (((dst | src) & 7ull) == 0) {
      // All loads of the tile in flight before the first store (the asm
      // volatile accesses are never reordered by the compiler).
      uint4 v[kVecPerThread];
      unsigned long long e[kVecPerThread];
#pragma unroll
      for (int u = 0; u < kVecPerThread; ++u) {
        e[u] = base + (static_cast<unsigned long long>(u) * kBlock + threadIdx.x) * 8ull;
        if (e[u] + 8 <= len) v[u] = ld_ro_v4(from + src + e[u]);
      }
      // ZeRO++ fused secondary refresh: tensor-local index of this tile's
      // elements is q*len + e; my secondary slice is [lo2, lo2 + len2)
      const unsigned long long len2 = a.sec ? len * a.sp / a.s2 : 0;
      const unsigned long long lo2 = len2 * static_cast<unsigned long long>(a.pos2);
#pragma unroll
      for (int u = 0; u < kVecPerThread; ++u) {
        if (e[u] + 8 <= len) {
          st_v4(a.dst + dst + e[u], v[u]);
          const unsigned long long x = static_cast<unsigned long long>(q) * len + e[u];
          if (a.sec && x >= lo2 && x < lo2 + len2) st_v4(a.sec + cs.sec + (x - lo2), v[u]);
        } else {
          for (unsigned long long k = e[u]; k < len && k < e[u] + 8; ++k) {
            a.dst[dst + k] = from[src + k];
            const unsigned long long x = static_cast<unsigned long long>(q) * len + k;
            if (a.sec && x >= lo2 && x < lo2 + len2) a.sec[cs.sec + (x - lo2)] = from[src + k];
          }
        }
      }
    } else {
      const unsigned long long len2 = a.sec ? len * a.sp / a.s2 : 0;
      const unsigned long long lo2 = len2 * static_cast<unsigned long long>(a.pos2);
      for (unsigned long long e = base + threadIdx.x; e < base + kTile && e < len;
           e += blockDim.x) {
        a.dst[dst + e] = from[src + e];
        const unsigned long long x = static_cast<unsigned long long>(q) * len + e;
        if (a.sec && x >= lo2 && x < lo2 + len2) a.sec[cs.sec + (x - lo2)] = from[src + e];
      }
    }
  }
}

__global__ void init_state_kernel(const Seg* segs, int nseg, int ntiles,
                                  float* master, float* m, float* v, uint64_t seed) {
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const Seg sg = find_seg(segs, nseg, tile);
    const unsigned long long base =
        (static_cast<unsigned long long>(tile) - sg.tile0) * kTile;
    for (unsigned long long e = base + threadIdx.x;
         e < base + kTile && e < sg.len; e += blockDim.x) {
      master[sg.os + e] = master_init(seed, sg.flat + e);
      m[sg.os + e] = 0.0f;
      v[sg.os + e] = 0.0f;
    }
  }
}

// Synthetic gradient of micro-batch `mb` (the backward stand-in): written,
// or with `accumulate` folded into the bf16 buffer in place, dst = bf16(dst
// + g) -- the s_g = 1 gradient accumulation of the oracle recipe.
template <bool kAccumulate>
__global__ void synth_grad_kernel(uint16_t* __restrict__ dst, unsigned long long start,
                                  unsigned long long n, uint64_t seed, uint32_t step,
                                  uint32_t mb, uint32_t rank) {
  const unsigned long long stride = 8ull * gridDim.x * blockDim.x;
  for (unsigned long long i = 8ull * (blockIdx.x * blockDim.x + threadIdx.x); i < n;
       i += stride) {
    if (i + 8 <= n && ((reinterpret_cast<uintptr_t>(dst + i) & 15) == 0)) {
      float x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = grad_value(seed, step, mb, rank, start + i + k);
      if (kAccumulate) {
        // the micro-batch gradient is a bf16 value before it is accumulated
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = bf16_at(to_bf16(x[k]));
        const uint4 old = *reinterpret_cast<const uint4*>(dst + i);
        const uint32_t* o = reinterpret_cast<const uint32_t*>(&old);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          x[2 * k] = __fadd_rn(bf16_lo(o[k]), x[2 * k]);
          x[2 * k + 1] = __fadd_rn(bf16_hi(o[k]), x[2 * k + 1]);
        }
      }
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = pack_bf16x2(x[2 * k], x[2 * k + 1]);
      st_v4(dst + i, make_uint4(w[0], w[1], w[2], w[3]));
    } else {
      const unsigned long long end = i + 8 < n ? i + 8 : n;
      for (unsigned long long k = i; k < end; ++k) {
        const float g = grad_value(seed, step, mb, rank, start + k);
        dst[k] = to_bf16(kAccumulate ? __fadd_rn(bf16_at(dst[k]), bf16_at(to_bf16(g))) : g);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Raw C-ABI kernels (amsp_k_*) over plain contiguous buffers. Each thread
// owns kRawU 8-element groups per iteration and issues every 128-bit load of
// those groups before the first arithmetic op, so each SM keeps >= 8 KB of
// reads in flight (HBM3e needs ~40 KB/SM at 8 TB/s; with 8 CTAs of 256
// threads per SM that is 8*256*kRawU*bytes_per_group). The vector path
// needs every base pointer 16-byte aligned at the group boundary; a ragged
// tail (n % 8) and misaligned buffers take the scalar path, which performs
// the same rounded operations, so the result never depends on alignment.
constexpr int kRawU = 4;

__device__ __forceinline__ bool al16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

__device__ __forceinline__ void unpack8(const uint4& w, float* x) {
  const uint32_t* u = reinterpret_cast<const uint32_t*>(&w);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    x[2 * k] = bf16_lo(u[k]);
    x[2 * k + 1] = bf16_hi(u[k]);
  }
}

__device__ __forceinline__ uint4 pack8(const float* x) {
  return make_uint4(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]), pack_bf16x2(x[4], x[5]),
                    pack_bf16x2(x[6], x[7]));
}

// Grid-stride driver: fn_vec(group indices, valid mask) for full vector
// groups, fn_scalar(i) for the rest.
template <int U, class Vec, class Scalar>
__device__ __forceinline__ void raw_loop(unsigned long long n, bool vec_ok, Vec fn_vec,
                                         Scalar fn_scalar) {
  const unsigned long long groups = vec_ok ? n / 8 : 0;
  const unsigned long long tid = static_cast<unsigned long long>(blockIdx.x) * blockDim.x +
                                 threadIdx.x;
  const unsigned long long nthr = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long g0 = tid; g0 < groups; g0 += nthr * U) {
    unsigned long long g[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      g[u] = g0 + u * nthr;
      ok[u] = g[u] < groups;
    }
    fn_vec(g, ok);
  }
  for (unsigned long long i = groups * 8 + tid; i < n; i += nthr) fn_scalar(i);
}

// Plain AdamW over a contiguous shard (the raw amsp_k_adamw launcher):
// g = grad * scale (bf16 or fp32 grad), AdamW, optional bf16 param out.
template <bool kBf16Grad, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) adamw_flat_kernel(const void* __restrict__ grad,
                                                         float* master, float* m, float* v,
                                                         uint16_t* param_out,
                                                         unsigned long long n, AdamScalars s) {
  const bool vec_ok = al16(grad) && al16(master) && al16(m) && al16(v) &&
                      (param_out == nullptr || al16(param_out));
  raw_loop<U>(
      n, vec_ok,
      [=](const unsigned long long* g, const bool* ok) {
        uint4 gb[U];
        float4 gf[U][U], p[U][U], mm[U][U], vv[U][U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!ok[u]) continue;
          const unsigned long long i = g[u] * 8;
          if (kBf16Grad) {
            gb[u] = ld_ro_v4(static_cast<const uint16_t*>(grad) + i);
          } else {
            const float* gp = static_cast<const float*>(grad) + i;
            gf[u][0] = ld_state_v4(gp);
            gf[u][1] = ld_state_v4(gp + 4);
          }
          p[u][0] = ld_state_v4(master + i);
          p[u][1] = ld_state_v4(master + i + 4);
          mm[u][0] = ld_state_v4(m + i);
          mm[u][1] = ld_state_v4(m + i + 4);
          vv[u][0] = ld_state_v4(v + i);
          vv[u][1] = ld_state_v4(v + i + 4);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!ok[u]) continue;
          const unsigned long long i = g[u] * 8;
          float x[8];
          if (kBf16Grad) {
            unpack8(gb[u], x);
          } else {
            const float* f = reinterpret_cast<const float*>(&gf[u][0]);
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = f[k];
          }
          float* pf = reinterpret_cast<float*>(&p[u][0]);
          float* mf = reinterpret_cast<float*>(&mm[u][0]);
          float* vf = reinterpret_cast<float*>(&vv[u][0]);
#pragma unroll
          for (int k = 0; k < 8; ++k) adamw(s, __fmul_rn(x[k], s.grad_scale), pf[k], mf[k], vf[k]);
          st_stream_v4(master + i, p[u][0]);
          st_stream_v4(master + i + 4, p[u][1]);
          st_stream_v4(m + i, mm[u][0]);
          st_stream_v4(m + i + 4, mm[u][1]);
          st_stream_v4(v + i, vv[u][0]);
          st_stream_v4(v + i + 4, vv[u][1]);
          if (param_out) st_stream_u4(param_out + i, pack8(pf));
        }
      },
      [=](unsigned long long i) {
        float g = kBf16Grad ? bf16_at(static_cast<const uint16_t*>(grad)[i])
                            : static_cast<const float*>(grad)[i];
        g = __fmul_rn(g, s.grad_scale);
        float p = master[i], mm = m[i], vv = v[i];
        adamw(s, g, p, mm, vv);
        master[i] = p;
        m[i] = mm;
        v[i] = vv;
        if (param_out) param_out[i] = to_bf16(p);
      });
}

// Raw reduce-scatter epilogue over plain pointers (amsp_k_rs_upcast_scale,
// and amsp_k_upcast_scale with one source): dst[k] = (sum_r bf16
// srcs[r][offset + k]) * scale, fixed rank order, the same rounding sequence
// as the fused kernel. srcs may be peer pointers (NVLink reads).
struct RsArgs {
  const uint16_t* srcs[kMaxRanks];
  int nsrc;
  unsigned long long offset, n;
  float* dst;
  float scale;
};

template <int NS>
__global__ void __launch_bounds__(256, 2) rs_upcast_scale_kernel(const RsArgs a) {
  constexpr int kU = NS <= 2 ? 4 : 2;
  bool vec_ok = al16(a.dst);
#pragma unroll
  for (int r = 0; r < NS; ++r) vec_ok = vec_ok && al16(a.srcs[r] + a.offset);
  raw_loop<kU>(
      a.n, vec_ok,
      [=](const unsigned long long* g, const bool* ok) {
        uint4 w[kU][NS];
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
          for (int r = 0; r < NS; ++r)
            if (ok[u]) w[u][r] = ld_ro_v4(a.srcs[r] + a.offset + g[u] * 8);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (!ok[u]) continue;
          float x[8], y[8];
          unpack8(w[u][0], x);
#pragma unroll
          for (int r = 1; r < NS; ++r) {
            unpack8(w[u][r], y);
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = __fadd_rn(x[k], y[k]);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) x[k] = __fmul_rn(x[k], a.scale);
          float* d = a.dst + g[u] * 8;
          st_stream_v4(d, make_float4(x[0], x[1], x[2], x[3]));
          st_stream_v4(d + 4, make_float4(x[4], x[5], x[6], x[7]));
        }
      },
      [=](unsigned long long k) {
        float g = bf16_at(a.srcs[0][a.offset + k]);
#pragma unroll
        for (int r = 1; r < NS; ++r) g = __fadd_rn(g, bf16_at(a.srcs[r][a.offset + k]));
        a.dst[k] = __fmul_rn(g, a.scale);
      });
}

// Raw all-gather epilogue (amsp_k_ag_downcast): bf16(src[k]) stored into
// dsts[d][dst_offset + k] for every destination (local or peer pointers).
struct AgArgs {
  uint16_t* dsts[kMaxRanks];
  int ndst;
  unsigned long long dst_offset, n;
  const float* src;
};

template <int ND>
__global__ void __launch_bounds__(256) ag_downcast_kernel(const AgArgs a) {
  bool vec_ok = al16(a.src);
#pragma unroll
  for (int d = 0; d < ND; ++d) vec_ok = vec_ok && al16(a.dsts[d] + a.dst_offset);
  raw_loop<kRawU>(
      a.n, vec_ok,
      [=](const unsigned long long* g, const bool* ok) {
        float4 x[kRawU][2];
#pragma unroll
        for (int u = 0; u < kRawU; ++u) {
          if (!ok[u]) continue;
          x[u][0] = ld_ro_f4(a.src + g[u] * 8);
          x[u][1] = ld_ro_f4(a.src + g[u] * 8 + 4);
        }
#pragma unroll
        for (int u = 0; u < kRawU; ++u) {
          if (!ok[u]) continue;
          const uint4 b = pack8(reinterpret_cast<const float*>(&x[u][0]));
#pragma unroll
          for (int d = 0; d < ND; ++d) st_stream_u4(a.dsts[d] + a.dst_offset + g[u] * 8, b);
        }
      },
      [=](unsigned long long k) {
        const uint16_t b = to_bf16(a.src[k]);
#pragma unroll
        for (int d = 0; d < ND; ++d) a.dsts[d][a.dst_offset + k] = b;
      });
}

// Reduce half of the split step: red[os] = (sum_r grads_r[flat]) * scale,
// fixed rank order (bit-equal to the fused kernel's sum).
template <int W>
__global__ void __launch_bounds__(kBlock) reduce_kernel(const ReduceArgs a) {
  __shared__ Seg s_segs[kSegCap];
  SegCursor<Seg, kSegCap> cursor;
  cursor.init(s_segs, a.segs, a.nseg);
  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const Seg sg = cursor.at(tile);
    const unsigned long long base = (static_cast<unsigned long long>(tile) - sg.tile0) * kTile;
    const bool aligned = ((sg.flat | sg.os | (a.nacc ? sg.dst : 0ull)) & 7ull) == 0;
#pragma unroll 1
    for (int it = 0; it < kVecPerThread; ++it) {
      const unsigned long long e = base + (static_cast<unsigned long long>(it) * kBlock +
                                           threadIdx.x) * 8ull;
      if (e >= sg.len) continue;
      if (aligned && e + 8 <= sg.len) {
        uint4 g[W];
#pragma unroll
        for (int r = 0; r < W; ++r) g[r] = ld_ro_v4(a.grads[r] + sg.flat + e);
        float out[8], accs[8];
        if (a.nacc > 0) acc_vec(a, (a.acc_by_dst ? sg.dst : sg.os) + e, accs);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const uint32_t* g0 = reinterpret_cast<const uint32_t*>(&g[0]);
          float lo = bf16_lo(g0[w]), hi = bf16_hi(g0[w]);
          if (a.nacc > 0) {
            lo = __fadd_rn(accs[2 * w], lo);
            hi = __fadd_rn(accs[2 * w + 1], hi);
          }
#pragma unroll
          for (int r = 1; r < W; ++r) {
            const uint32_t* gr = reinterpret_cast<const uint32_t*>(&g[r]);
            lo = __fadd_rn(lo, bf16_lo(gr[w]));
            hi = __fadd_rn(hi, bf16_hi(gr[w]));
          }
          out[2 * w] = __fmul_rn(lo, a.scale);
          out[2 * w + 1] = __fmul_rn(hi, a.scale);
        }
        st_stream_v4(a.red + sg.os + e, make_float4(out[0], out[1], out[2], out[3]));
        st_stream_v4(a.red + sg.os + e + 4, make_float4(out[4], out[5], out[6], out[7]));
      } else {
        const unsigned long long end = e + 8 < sg.len ? e + 8 : sg.len;
        for (unsigned long long k = e; k < end; ++k)
          a.red[sg.os + k] = __fmul_rn(
              reduce_scalar<W>(a, sg.flat + k, (a.acc_by_dst ? sg.dst : sg.os) + k), a.scale);
      }
    }
  }
}

// AdamW + downcast + parameter push half of the split step.
__global__ void __launch_bounds__(kBlock) adam_push_kernel(const AdamPushArgs a) {
  __shared__ Seg s_segs[kSegCap];
  SegCursor<Seg, kSegCap> cursor;
  cursor.init(s_segs, a.segs, a.nseg);
  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const Seg sg = cursor.at(tile);
    const unsigned long long base = (static_cast<unsigned long long>(tile) - sg.tile0) * kTile;
    const bool aligned = ((sg.os | sg.dst) & 7ull) == 0;
    // all kVecPerThread vectors' loads in flight before any math (the HBM
    // latency, not the bandwidth, limited the one-vector-at-a-time loop)
    unsigned long long e[kVecPerThread];
    bool full[kVecPerThread];
    float4 g[kVecPerThread][2], p[kVecPerThread][2], m[kVecPerThread][2], v[kVecPerThread][2];
#pragma unroll
    for (int u = 0; u < kVecPerThread; ++u) {
      e[u] = base + (static_cast<unsigned long long>(u) * kBlock + threadIdx.x) * 8ull;
      full[u] = aligned && e[u] + 8 <= sg.len;
      if (full[u]) {
        const unsigned long long o = sg.os + e[u];
        g[u][0] = ld_state_v4(a.red + o);
        g[u][1] = ld_state_v4(a.red + o + 4);
        p[u][0] = ld_state_v4(a.master + o);
        p[u][1] = ld_state_v4(a.master + o + 4);
        m[u][0] = ld_state_v4(a.exp_avg + o);
        m[u][1] = ld_state_v4(a.exp_avg + o + 4);
        v[u][0] = ld_state_v4(a.exp_avg_sq + o);
        v[u][1] = ld_state_v4(a.exp_avg_sq + o + 4);
      }
    }
#pragma unroll
    for (int u = 0; u < kVecPerThread; ++u) {
      if (e[u] >= sg.len) continue;
      if (full[u]) {
        const unsigned long long o = sg.os + e[u];
        float* gf = reinterpret_cast<float*>(g[u]);
        float* pf = reinterpret_cast<float*>(p[u]);
        float* mf = reinterpret_cast<float*>(m[u]);
        float* vf = reinterpret_cast<float*>(v[u]);
        uint32_t packed[4];
#pragma unroll
        for (int j = 0; j < 8; ++j) adamw(a.s, gf[j], pf[j], mf[j], vf[j]);
#pragma unroll
        for (int w = 0; w < 4; ++w) packed[w] = pack_bf16x2(pf[2 * w], pf[2 * w + 1]);
        st_stream_v4(a.master + o, p[u][0]);
        st_stream_v4(a.master + o + 4, p[u][1]);
        st_stream_v4(a.exp_avg + o, m[u][0]);
        st_stream_v4(a.exp_avg + o + 4, m[u][1]);
        st_stream_v4(a.exp_avg_sq + o, v[u][0]);
        st_stream_v4(a.exp_avg_sq + o + 4, v[u][1]);
        const uint4 out = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        for (int d = 0; d < a.ndst; ++d) st_v4(a.dsts[d] + sg.dst + e[u], out);
      } else {
        const unsigned long long end = e[u] + 8 < sg.len ? e[u] + 8 : sg.len;
        for (unsigned long long k = e[u]; k < end; ++k) {
          float pp = a.master[sg.os + k], mm = a.exp_avg[sg.os + k], vv = a.exp_avg_sq[sg.os + k];
          adamw(a.s, a.red[sg.os + k], pp, mm, vv);
          a.master[sg.os + k] = pp;
          a.exp_avg[sg.os + k] = mm;
          a.exp_avg_sq[sg.os + k] = vv;
          const uint16_t b = to_bf16(pp);
          for (int d = 0; d < a.ndst; ++d) a.dsts[d][sg.dst + k] = b;
        }
      }
    }
  }
  if (a.fence_peers) __threadfence_system();
}

// Micro-batch accumulation into the local bf16 G shard (AccumArgs). NS =
// block size; both vectors of a thread's tile are loaded (NS x 2 loads in
// flight) before any math, like the fused kernel.
template <int NS, bool kFirst>
__global__ void __launch_bounds__(kBlock) accumulate_kernel(const AccumArgs a) {
  __shared__ Seg s_segs[kSegCap];
  SegCursor<Seg, kSegCap> cursor;
  cursor.init(s_segs, a.segs, a.nseg);
  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const Seg sg = cursor.at(tile);
    const unsigned long long base = (static_cast<unsigned long long>(tile) - sg.tile0) * kTile;
    const bool aligned = ((sg.flat | sg.os) & 7ull) == 0;
    unsigned long long e[kVecPerThread];
    uint4 g[kVecPerThread][NS], old[kVecPerThread];
#pragma unroll
    for (int u = 0; u < kVecPerThread; ++u) {
      e[u] = base + (static_cast<unsigned long long>(u) * kBlock + threadIdx.x) * 8ull;
      if (aligned && e[u] + 8 <= sg.len) {
#pragma unroll
        for (int q = 0; q < NS; ++q) g[u][q] = ld_ro_v4(a.grads[q] + sg.flat + e[u]);
        if (!kFirst) old[u] = *reinterpret_cast<const uint4*>(a.acc + sg.os + e[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kVecPerThread; ++u) {
      if (e[u] >= sg.len) continue;
      if (aligned && e[u] + 8 <= sg.len) {
        uint32_t packed[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const uint32_t* g0 = reinterpret_cast<const uint32_t*>(&g[u][0]);
          float lo = bf16_lo(g0[w]), hi = bf16_hi(g0[w]);
          if (!kFirst) {
            const uint32_t* o = reinterpret_cast<const uint32_t*>(&old[u]);
            lo = __fadd_rn(bf16_lo(o[w]), lo);
            hi = __fadd_rn(bf16_hi(o[w]), hi);
          }
#pragma unroll
          for (int q = 1; q < NS; ++q) {
            const uint32_t* gq = reinterpret_cast<const uint32_t*>(&g[u][q]);
            lo = __fadd_rn(lo, bf16_lo(gq[w]));
            hi = __fadd_rn(hi, bf16_hi(gq[w]));
          }
          packed[w] = pack_bf16x2(lo, hi);
        }
        st_v4(a.acc + sg.os + e[u], make_uint4(packed[0], packed[1], packed[2], packed[3]));
      } else {
        const unsigned long long end = e[u] + 8 < sg.len ? e[u] + 8 : sg.len;
        for (unsigned long long k = e[u]; k < end; ++k) {
          float s = bf16_at(a.grads[0][sg.flat + k]);
          if (!kFirst) s = __fadd_rn(bf16_at(a.acc[sg.os + k]), s);
#pragma unroll
          for (int q = 1; q < NS; ++q) s = __fadd_rn(s, bf16_at(a.grads[q][sg.flat + k]));
          a.acc[sg.os + k] = to_bf16(s);
        }
      }
    }
  }
  if (a.fence_peers) __threadfence_system();
}

__global__ void __launch_bounds__(256) p2p_pull_kernel(const PullArgs a) {
  const unsigned long long total = a.vecs_per_src * static_cast<unsigned long long>(a.nsrc);
  const unsigned long long stride = 2ull * gridDim.x * blockDim.x;
  for (unsigned long long v0 = (static_cast<unsigned long long>(blockIdx.x) * blockDim.x +
                                threadIdx.x);
       v0 < total; v0 += stride) {
    uint4 x[2];
    unsigned long long off[2];
    int q[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const unsigned long long v = v0 + u * (stride / 2);
      const unsigned long long chunk = v / 32;
      q[u] = static_cast<int>((chunk % a.nsrc + a.rot) % a.nsrc);
      off[u] = (chunk / a.nsrc) * 32 + v % 32;
      if (v < total) x[u] = ld_ro_v4(a.src[q[u]] + off[u]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const unsigned long long v = v0 + u * (stride / 2);
      if (v < total) st_v4(a.dst + v, x[u]);
    }
  }
}

// Compute stand-in for the overlap schedule: every CTA keeps its warps
// issuing dependent FMAs for `ns` nanoseconds (timed per CTA, so CTAs that
// wait for SM slots held by communication kernels finish later — the
// stand-in has a fixed amount of per-CTA work, like a GEMM tile loop).
__global__ void spin_kernel(unsigned long long ns, float* sink) {
  unsigned long long t0, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  float x = threadIdx.x * 1e-3f, y = 1.0f;
  do {
#pragma unroll
    for (int i = 0; i < 64; ++i) x = fmaf(x, 0.999f, y);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  } while (now - t0 < ns);
  if (x == 123.456f) sink[threadIdx.x] = x;  // keep the loop alive
}

// ---------------------------------------------------------------------------
// TMA-pipelined fused step (variants 5 / 6), any W.
//
// The last warp is a producer: one lane walks the CTA's tiles and, per tile,
// issues W + 3 bulk async copies (cp.async.bulk, the TMA engine's 1-D path):
// the bf16 gradients of every DP rank (local HBM for r = rank, NVLink peer
// memory otherwise) and the fp32 master / m / v of this rank's shard, into a
// kStages-deep shared-memory ring; completion is signalled through an
// mbarrier transaction count. Warps 0-7 consume: each thread sums its 8
// elements' gradients in fixed rank order from shared memory, applies AdamW
// and streams master / m / v locally and the bf16 params into every OS-group
// peer. Memory-level parallelism comes from the ring (kStages x stage bytes
// in flight per CTA) instead of registers, which is what limits the LDG
// version at 16 warps / SM (ncu: long-scoreboard stalls) -- and the NVLink
// pulls need the most bytes in flight of all (peer latency ~2x HBM).
// Ring depth: variant 5 sizes the ring for 2 CTAs / SM (<= 100 KB), variant
// 6 for 1 CTA / SM (<= 220 KB).
constexpr int kTmaConsumers = 256;
constexpr int kTmaTile = kTmaConsumers * 8;  // elements per stage (2048)
// Variants 7 / 8 add a bf16 output tile per stage: the consumers write the
// updated master / m / v back into the stage in place and the packed bf16
// params into it, and the producer drains the stage with bulk stores
// (cp.async.bulk shared -> global, local HBM and NVLink peers alike), so no
// thread issues a global store at all.
constexpr bool tma_bulk_out(int variant) {
  return variant == 7 || variant == 8 || variant == 11;
}
constexpr bool tma_two_ctas(int variant) {
  return variant == 5 || variant == 7 || variant == 9 || variant == 10;
}
// Fixed ring depths (0 = sized by the smem budget), capped to what fits.
constexpr int tma_fixed_stages(int variant) {
  return variant == 9 ? 2 : variant == 10 ? 4 : (variant == 11 || variant == 12) ? 5 : 0;
}
constexpr int tma_stage_bytes(int w, bool out = false) {
  return kTmaTile * (2 * w + 12 + (out ? 2 : 0));
}
// Variants 9 / 10 / 12: a fixed 2- / 4- / 5-stage ring; 11: 5 stages with
// the bulk-store drain (ring-depth sweep: at W = 1 three stages are best,
// 2 -> 36.4, 3 -> 29.9, 4 -> 30.8, 7 -> 32.8 ms; at W = 2 four beat three,
// profiles/r01_s2_stages_*.json).
constexpr int tma_stages(int w, int variant) {
  return tma_fixed_stages(variant) > 0
             ? (tma_fixed_stages(variant) * tma_stage_bytes(w, tma_bulk_out(variant)) <=
                        220 * 1024
                    ? tma_fixed_stages(variant)
                    : (220 * 1024 / tma_stage_bytes(w, tma_bulk_out(variant)) < 2
                           ? 2
                           : 220 * 1024 / tma_stage_bytes(w, tma_bulk_out(variant))))
         : (tma_two_ctas(variant) ? 100 * 1024 : 220 * 1024) /
                     tma_stage_bytes(w, tma_bulk_out(variant)) <
                 2
             ? 2
             : (tma_two_ctas(variant) ? 100 * 1024 : 220 * 1024) /
                   tma_stage_bytes(w, tma_bulk_out(variant));
}
constexpr int tma_smem(int w, int stages, bool out = false) {
  return stages * tma_stage_bytes(w, out) + 1024;
}

struct TmaStageMeta {
  unsigned long long os, dst, len;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_s2g_nocommit(void* gmem_dst, const void* smem_src,
                                                  uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_addr(smem_src)), "r"(bytes)
               : "memory");
}

// NA > 0: up to NA bf16 G-shard accumulators (the holders' of micro-batches
// 0..M-2, a.nacc <= NA of them) are pulled per stage beside the W raw
// gradients and summed first, in holder order, then the raw gradients in
// rank order: the LDG kernels' (and the oracle's) rounding sequence.
template <int W, int NA, int kStages, int kMinBlocks, bool kBulkOut>
__global__ void __launch_bounds__(kTmaConsumers + 32, kMinBlocks)
fused_step_tma_kernel(const FusedArgs a) {
  constexpr int G = W + NA;  // bf16 source slots per stage
  extern __shared__ __align__(128) unsigned char smem[];
  uint16_t* s_g = reinterpret_cast<uint16_t*>(smem);  // [kStages][G][kTmaTile]
  float* s_p = reinterpret_cast<float*>(smem + kStages * G * kTmaTile * 2);
  float* s_m = s_p + kStages * kTmaTile;
  float* s_v = s_m + kStages * kTmaTile;
  uint16_t* s_o = reinterpret_cast<uint16_t*>(s_v + kStages * kTmaTile);  // kBulkOut only
  uint64_t* full = reinterpret_cast<uint64_t*>(kBulkOut ? static_cast<void*>(s_o + kStages * kTmaTile)
                                                        : static_cast<void*>(s_o));
  uint64_t* empty = full + kStages;
  TmaStageMeta* meta = reinterpret_cast<TmaStageMeta*>(empty + kStages);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // Tiles of this CTA: blockIdx.x, +gridDim.x, ... over the segment table
  // re-cut into kTmaTile-element tiles (tile0 of a Seg counts kTile = 4096
  // tiles, so every kTile tile holds two TMA tiles).
  const int ntiles = a.ntiles * 2;
  if (warp == kTmaConsumers / 32) {  // producer warp
    if (lane == 0) {
      SegCursor<Seg, 1> cur;  // global-table binary search (one thread)
      cur.table = a.segs;
      cur.n = a.nseg;
      cur.cur = 0;
      cur.staged = false;
      // kBulkOut: drain stage s (its tile is finished by the consumers) with
      // bulk stores; always one bulk group per tile, possibly empty.
      auto store_back = [&](int s) {
        const TmaStageMeta md = meta[s];
        if (md.len) {
          bulk_s2g_nocommit(a.master + md.os, s_p + s * kTmaTile, md.len * 4);
          bulk_s2g_nocommit(a.exp_avg + md.os, s_m + s * kTmaTile, md.len * 4);
          bulk_s2g_nocommit(a.exp_avg_sq + md.os, s_v + s * kTmaTile, md.len * 4);
          for (int d = 0; d < a.ndst; ++d)
            bulk_s2g_nocommit(a.dsts[d] + md.dst, s_o + s * kTmaTile, md.len * 2);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      };
      int k = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int s = k % kStages;
        if (kBulkOut) {
          // Store tile k-S+1 (its stage is refilled next iteration), then make
          // sure the store of tile k-S, issued one iteration ago, has read
          // stage s before it is refilled: one tile of prefetch depth is
          // traded for never waiting on the store just issued.
          const int j = k - kStages + 1;
          if (j >= 0) {
            mbar_wait(&empty[j % kStages], (j / kStages) & 1);
            store_back(j % kStages);
          }
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        } else if (k >= kStages) {
          mbar_wait(&empty[s], ((k / kStages) - 1) & 1);
        }
        const Seg& sg = cur.at(t / 2);
        const unsigned long long base =
            (static_cast<unsigned long long>(t / 2) - sg.tile0) * kTile + (t & 1) * kTmaTile;
        unsigned long long len = 0;
        if (base < sg.len) len = sg.len - base < kTmaTile ? sg.len - base : kTmaTile;
        meta[s] = {sg.os + base, sg.dst + base, len};
        const int nacc = NA > 0 ? a.nacc : 0;
        mbar_expect_tx(&full[s], static_cast<uint32_t>(len * (2 * (W + nacc) + 12)));
        if (len) {
#pragma unroll
          for (int r = 0; r < W; ++r)
            bulk_g2s(s_g + (s * G + r) * kTmaTile, a.grads[r] + sg.flat + base, len * 2,
                     &full[s]);
          if (NA > 0) {
            const unsigned long long ai = (a.acc_by_dst ? sg.dst : sg.os) + base;
            for (int j = 0; j < nacc; ++j)
              bulk_g2s(s_g + (s * G + W + j) * kTmaTile, a.acc[j] + ai, len * 2, &full[s]);
          }
          bulk_g2s(s_p + s * kTmaTile, a.master + sg.os + base, len * 4, &full[s]);
          bulk_g2s(s_m + s * kTmaTile, a.exp_avg + sg.os + base, len * 4, &full[s]);
          bulk_g2s(s_v + s * kTmaTile, a.exp_avg_sq + sg.os + base, len * 4, &full[s]);
        }
      }
      if (kBulkOut) {
        for (int j = k - kStages + 1 > 0 ? k - kStages + 1 : 0; j < k; ++j) {
          mbar_wait(&empty[j % kStages], (j / kStages) & 1);
          store_back(j % kStages);
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        // Peer parameter stores visible system-wide before the trailing
        // cross-GPU barrier releases the other ranks.
        if (a.fence_peers) __threadfence_system();
      }
    }
    return;
  }

  float sq = 0.0f;
  int k = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % kStages;
    mbar_wait(&full[s], (k / kStages) & 1);
    const TmaStageMeta md = meta[s];
    const unsigned long long e = static_cast<unsigned long long>(threadIdx.x) * 8;
    if (e < md.len) {  // segment lengths are multiples of 8 on this path
      uint4 graw[W];
#pragma unroll
      for (int r = 0; r < W; ++r)
        graw[r] = *reinterpret_cast<const uint4*>(s_g + (s * G + r) * kTmaTile + e);
      float accs[8];
      if (NA > 0 && a.nacc > 0) {
        const uint4 w0 = *reinterpret_cast<const uint4*>(s_g + (s * G + W) * kTmaTile + e);
        const uint32_t* u0 = reinterpret_cast<const uint32_t*>(&w0);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          accs[2 * w] = bf16_lo(u0[w]);
          accs[2 * w + 1] = bf16_hi(u0[w]);
        }
        for (int j = 1; j < a.nacc; ++j) {
          const uint4 wj = *reinterpret_cast<const uint4*>(s_g + (s * G + W + j) * kTmaTile + e);
          const uint32_t* uj = reinterpret_cast<const uint32_t*>(&wj);
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            accs[2 * w] = __fadd_rn(accs[2 * w], bf16_lo(uj[w]));
            accs[2 * w + 1] = __fadd_rn(accs[2 * w + 1], bf16_hi(uj[w]));
          }
        }
      }
      float4 p[2], m[2], v[2];
      p[0] = *reinterpret_cast<const float4*>(s_p + s * kTmaTile + e);
      p[1] = *reinterpret_cast<const float4*>(s_p + s * kTmaTile + e + 4);
      m[0] = *reinterpret_cast<const float4*>(s_m + s * kTmaTile + e);
      m[1] = *reinterpret_cast<const float4*>(s_m + s * kTmaTile + e + 4);
      v[0] = *reinterpret_cast<const float4*>(s_v + s * kTmaTile + e);
      v[1] = *reinterpret_cast<const float4*>(s_v + s * kTmaTile + e + 4);
      float* pf = reinterpret_cast<float*>(p);
      float* mf = reinterpret_cast<float*>(m);
      float* vf = reinterpret_cast<float*>(v);
      uint32_t packed[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t* g0 = reinterpret_cast<const uint32_t*>(&graw[0]);
        float glo = bf16_lo(g0[w]), ghi = bf16_hi(g0[w]);
        if (NA > 0 && a.nacc > 0) {  // accumulators first, then the raw gradients
          glo = __fadd_rn(accs[2 * w], glo);
          ghi = __fadd_rn(accs[2 * w + 1], ghi);
        }
#pragma unroll
        for (int r = 1; r < W; ++r) {  // fixed rank order, as the LDG kernel
          const uint32_t* gr = reinterpret_cast<const uint32_t*>(&graw[r]);
          glo = __fadd_rn(glo, bf16_lo(gr[w]));
          ghi = __fadd_rn(ghi, bf16_hi(gr[w]));
        }
        glo = __fmul_rn(glo, a.s.grad_scale);
        ghi = __fmul_rn(ghi, a.s.grad_scale);
        sq += glo * glo + ghi * ghi;
        adamw(a.s, glo, pf[2 * w], mf[2 * w], vf[2 * w]);
        adamw(a.s, ghi, pf[2 * w + 1], mf[2 * w + 1], vf[2 * w + 1]);
        packed[w] = pack_bf16x2(pf[2 * w], pf[2 * w + 1]);
      }
      const uint4 out = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      if (kBulkOut) {  // in place; the producer's bulk stores drain the stage
        *reinterpret_cast<float4*>(s_p + s * kTmaTile + e) = p[0];
        *reinterpret_cast<float4*>(s_p + s * kTmaTile + e + 4) = p[1];
        *reinterpret_cast<float4*>(s_m + s * kTmaTile + e) = m[0];
        *reinterpret_cast<float4*>(s_m + s * kTmaTile + e + 4) = m[1];
        *reinterpret_cast<float4*>(s_v + s * kTmaTile + e) = v[0];
        *reinterpret_cast<float4*>(s_v + s * kTmaTile + e + 4) = v[1];
        *reinterpret_cast<uint4*>(s_o + s * kTmaTile + e) = out;
      } else {
        const unsigned long long o = md.os + e;
        st_stream_v4(a.master + o, p[0]);
        st_stream_v4(a.master + o + 4, p[1]);
        st_stream_v4(a.exp_avg + o, m[0]);
        st_stream_v4(a.exp_avg + o + 4, m[1]);
        st_stream_v4(a.exp_avg_sq + o, v[0]);
        st_stream_v4(a.exp_avg_sq + o + 4, v[1]);
        for (int d = 0; d < a.ndst; ++d) st_v4(a.dsts[d] + md.dst + e, out);
      }
    }
    // generic-proxy shared-memory writes -> visible to the bulk stores
    if (kBulkOut) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  // Peer parameter stores must be visible system-wide before the trailing
  // cross-GPU barrier releases the other ranks.
  if (!kBulkOut && a.fence_peers) __threadfence_system();
  if (a.stats != nullptr) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if (lane == 0) atomicAdd(a.stats, sq);
  }
}

// ---------------------------------------------------------------------------
// Push all-gather (engine step, s_p > 1): one thread per CTA; per tile one
// bulk load of this rank's own slice (local HBM) into a shared-memory stage,
// then one bulk store per P-group member, destinations rotated from q+1 so
// the ranks' stores spread over the peers, all in one bulk group. Peer
// stores ran at 703 GB/s against 667 for pulls (profiles/r01_p2p_4gpu.txt).
__global__ void __launch_bounds__(32) push_tma_kernel(const PushArgs a) {
  constexpr int kStages = 5;
  __shared__ __align__(128) uint16_t buf[kStages][kTile];
  __shared__ __align__(8) uint64_t full[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int n = a.ntiles > static_cast<int>(blockIdx.x)
                    ? (a.ntiles - 1 - static_cast<int>(blockIdx.x)) / gridDim.x + 1
                    : 0;
  SegCursor<CopySeg, 1> cur;
  cur.table = a.segs;
  cur.n = a.nseg;
  cur.cur = 0;
  cur.staged = false;
  unsigned long long dst_off[kStages];
  uint32_t bytes_of[kStages];
  auto load = [&](int i) {
    const int tile = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
    const CopySeg& cs = cur.at(tile);
    const unsigned long long off = (static_cast<unsigned long long>(tile) - cs.tile0) * kTile;
    const unsigned long long len = cs.len - off < kTile ? cs.len - off : kTile;
    const int s = i % kStages;
    dst_off[s] = cs.dst + static_cast<unsigned long long>(a.q) * cs.len + off;
    bytes_of[s] = static_cast<uint32_t>(len * 2);
    mbar_expect_tx(&full[s], bytes_of[s]);
    bulk_g2s(buf[s], a.src + cs.src + off, bytes_of[s], &full[s]);
  };
  for (int i = 0; i < n && i < kStages; ++i) load(i);
  for (int i = 0; i < n; ++i) {
    const int s = i % kStages;
    mbar_wait(&full[s], (i / kStages) & 1);
    for (int j = 0; j < a.sp; ++j) {
      const int d = (a.q + 1 + j) % a.sp;
      bulk_s2g_nocommit(a.dst[d] + dst_off[s], buf[s], bytes_of[s]);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    const int k = i - 1 + kStages;  // refill the stage tile i-1 used
    if (i >= 1 && k < n) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      load(k);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // peer stores visible system-wide before the barrier after the passes
  if (a.fence_peers) __threadfence_system();
}

// ---------------------------------------------------------------------------
// TMA all-gather of one unit (s_p > 1): one thread per CTA drives a ring of
// kGatherStages 8 KB shared-memory stages. Each tile is one bulk load
// (cp.async.bulk, peer P shard over NVLink -> shared memory, completion on an
// mbarrier) followed by one bulk store (shared -> the local gathered buffer,
// bulk async-group). Loads of the next kGatherStages - 1 tiles are in flight
// while a store drains, so the NVLink pulls keep ~32 KB in flight per CTA
// with no register staging, and the CTA is a single warp: it leaves the
// SM's warps, registers and most of its shared memory to the GEMMs it
// overlaps with. Tiles and source interleaving are those of gather_kernel.
// Every CopySeg must be 8-element aligned (16-byte bulk granularity).
constexpr int kGatherStages = 5;


__global__ void __launch_bounds__(32) gather_tma_kernel(const GatherArgs a) {
  __shared__ __align__(128) uint16_t buf[kGatherStages][kTile];
  __shared__ __align__(8) uint64_t full[kGatherStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kGatherStages; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

  const int n = a.ntiles > static_cast<int>(blockIdx.x)
                    ? (a.ntiles - 1 - static_cast<int>(blockIdx.x)) / gridDim.x + 1
                    : 0;
  SegCursor<CopySeg, 1> cur;  // global-table search from a forward cursor
  cur.table = a.segs;
  cur.n = a.nseg;
  cur.cur = 0;
  cur.staged = false;
  uint16_t* dst_of[kGatherStages];
  uint32_t bytes_of[kGatherStages];
  // ZeRO++ fused secondary refresh (a.sec): part of the tile inside this
  // rank's secondary slice, as (element offset in the tile, count, sec dst)
  uint32_t sec_from[kGatherStages], sec_n[kGatherStages];
  uint16_t* sec_dst[kGatherStages];
  auto load = [&](int i) {
    const int tile = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
    const CopySeg& cs = cur.at(tile);
    const unsigned long long v = static_cast<unsigned long long>(tile) - cs.tile0;
    const unsigned long long chunk = v / a.sp;
    const int q = static_cast<int>((v % a.sp + a.rot) % a.sp);
    const unsigned long long off = chunk * kTile;
    const unsigned long long len = cs.len - off < kTile ? cs.len - off : kTile;
    const int s = i % kGatherStages;
    dst_of[s] = a.dst + cs.dst + static_cast<unsigned long long>(q) * cs.len + off;
    bytes_of[s] = static_cast<uint32_t>(len * 2);
    sec_n[s] = 0;
    if (a.sec) {
      const unsigned long long len2 = cs.len * a.sp / a.s2;
      const unsigned long long lo2 = len2 * static_cast<unsigned long long>(a.pos2);
      const unsigned long long x0 = static_cast<unsigned long long>(q) * cs.len + off;
      const unsigned long long b0 = x0 > lo2 ? x0 : lo2;
      const unsigned long long b1 = x0 + len < lo2 + len2 ? x0 + len : lo2 + len2;
      if (b0 < b1) {
        sec_from[s] = static_cast<uint32_t>(b0 - x0);
        sec_n[s] = static_cast<uint32_t>(b1 - b0);
        sec_dst[s] = a.sec + cs.sec + (b0 - lo2);
      }
    }
    mbar_expect_tx(&full[s], bytes_of[s]);
    bulk_g2s(buf[s], a.src[q] + cs.src + off, bytes_of[s], &full[s]);
  };
  for (int i = 0; i < n && i < kGatherStages; ++i) load(i);
  for (int i = 0; i < n; ++i) {
    const int s = i % kGatherStages;
    mbar_wait(&full[s], (i / kGatherStages) & 1);
    bulk_s2g_nocommit(dst_of[s], buf[s], bytes_of[s]);
    if (sec_n[s]) bulk_s2g_nocommit(sec_dst[s], buf[s] + sec_from[s], sec_n[s] * 2);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");  // one group per tile
    const int j = i - 1 + kGatherStages;  // refill the stage tile i-1 used
    if (i >= 1 && j < n) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      load(j);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Per-device caches: the attribute and SM count belong to the device (and
// its context), not the process, so an engine on a second GPU in the same
// process must not reuse the first device's answer.
constexpr int kMaxDevices = 64;

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}

int sm_count() {
  static int cache[kMaxDevices] = {};
  const int dev = current_device();
  if (cache[dev] == 0) {
    int c = 148;
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = c;
  }
  return cache[dev];
}

using FusedFn = void (*)(const FusedArgs);

// Tuning variants of the fused kernel: U = vectors with loads in flight per
// thread, MINB = minimum resident CTAs per SM requested from ptxas.
//   0 auto (U=2 for W<=4, else U=1)  1 U=1  2 U=2  3 U=2,minB=3  4 U=1,minB=4
template <int W>
FusedFn pick_variant(int variant) {
  switch (variant) {
    case 1: return fused_step_kernel<W, 1, 1>;
    case 2: return fused_step_kernel<W, 2, 1>;
    case 3: return fused_step_kernel<W, 2, 3>;
    case 4: return fused_step_kernel<W, 1, 4>;
    default: return W <= 4 ? fused_step_kernel<W, 2, 1> : fused_step_kernel<W, 1, 1>;
  }
}

FusedFn select_fused(int world, int variant) {
  switch (world) {
    case 1: return pick_variant<1>(variant);
    case 2: return pick_variant<2>(variant);
    case 3: return pick_variant<3>(variant);
    case 4: return pick_variant<4>(variant);
    case 5: return pick_variant<5>(variant);
    case 6: return pick_variant<6>(variant);
    case 7: return pick_variant<7>(variant);
    case 8: return pick_variant<8>(variant);
    default: return nullptr;
  }
}

}  // namespace

// Variants 5 / 6: the TMA pipeline, ring sized for 2 / 1 CTAs per SM.
template <int W, int V, int NA = 0>
struct Tma {
  static constexpr bool kOut = tma_bulk_out(V);
  static constexpr int kStages = tma_stages(W + NA, V);
  static constexpr int kSmem = tma_smem(W + NA, kStages, kOut);
  static constexpr auto kFn =
      fused_step_tma_kernel<W, NA, kStages, tma_two_ctas(V) ? 2 : 1, kOut>;
  // The >48 KB dynamic shared-memory opt-in, once per device.
  static cudaError_t prepare() {
    static bool done[kMaxDevices] = {};
    const int dev = current_device();
    if (done[dev]) return cudaSuccess;
    const cudaError_t attr =
        cudaFuncSetAttribute(kFn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (attr == cudaSuccess) done[dev] = true;
    return attr;
  }
  static int blocks_per_sm() {
    int blocks = 0;
    if (prepare() == cudaSuccess)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kFn, kTmaConsumers + 32, kSmem);
    return blocks > 0 ? blocks : 1;
  }
  static cudaError_t launch(const FusedArgs& a, int grid, cudaStream_t stream) {
    const cudaError_t attr = prepare();
    if (attr != cudaSuccess) return attr;
    kFn<<<grid, kTmaConsumers + 32, kSmem, stream>>>(a);
    return cudaGetLastError();
  }
};

template <int V>
int tma_blocks_per_sm(int world) {
  switch (world) {
    case 1: return Tma<1, V>::blocks_per_sm();
    case 2: return Tma<2, V>::blocks_per_sm();
    case 3: return Tma<3, V>::blocks_per_sm();
    case 4: return Tma<4, V>::blocks_per_sm();
    case 5: return Tma<5, V>::blocks_per_sm();
    case 6: return Tma<6, V>::blocks_per_sm();
    case 7: return Tma<7, V>::blocks_per_sm();
    case 8: return Tma<8, V>::blocks_per_sm();
    default: return 1;
  }
}

// Accumulator sources (M > 1, s_g > 1): the per-W default variants only
// (5, 10, 11), with room for W/2 holders (s_g >= 2).
template <int V>
cudaError_t tma_launch_acc_v(const FusedArgs& a, int world, int grid, cudaStream_t stream) {
  if (a.nacc > (world > 1 ? world / 2 : 0)) return cudaErrorInvalidValue;
  switch (world) {
    case 2: return Tma<2, V, 1>::launch(a, grid, stream);
    case 4: return Tma<4, V, 2>::launch(a, grid, stream);
    case 6: return Tma<6, V, 3>::launch(a, grid, stream);
    case 8: return Tma<8, V, 4>::launch(a, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t tma_launch_acc(const FusedArgs& a, int world, int grid, int variant,
                           cudaStream_t stream) {
  if (variant == 5) return tma_launch_acc_v<5>(a, world, grid, stream);
  if (variant == 10) return tma_launch_acc_v<10>(a, world, grid, stream);
  if (variant == 11) return tma_launch_acc_v<11>(a, world, grid, stream);
  return cudaErrorInvalidValue;
}

// CTAs per SM of the accumulator-source instantiation (0 = none exists).
int tma_acc_blocks_per_sm(int world, int variant) {
  auto pick = [&](auto tag) -> int {
    constexpr int V = decltype(tag)::value;
    switch (world) {
      case 2: return Tma<2, V, 1>::blocks_per_sm();
      case 4: return Tma<4, V, 2>::blocks_per_sm();
      case 6: return Tma<6, V, 3>::blocks_per_sm();
      case 8: return Tma<8, V, 4>::blocks_per_sm();
      default: return 0;
    }
  };
  if (variant == 5) return pick(std::integral_constant<int, 5>{});
  if (variant == 10) return pick(std::integral_constant<int, 10>{});
  if (variant == 11) return pick(std::integral_constant<int, 11>{});
  return 0;
}

template <int V>
cudaError_t tma_launch(const FusedArgs& a, int world, int grid, cudaStream_t stream) {
  switch (world) {
    case 1: return Tma<1, V>::launch(a, grid, stream);
    case 2: return Tma<2, V>::launch(a, grid, stream);
    case 3: return Tma<3, V>::launch(a, grid, stream);
    case 4: return Tma<4, V>::launch(a, grid, stream);
    case 5: return Tma<5, V>::launch(a, grid, stream);
    case 6: return Tma<6, V>::launch(a, grid, stream);
    case 7: return Tma<7, V>::launch(a, grid, stream);
    case 8: return Tma<8, V>::launch(a, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

int fused_blocks_per_sm(int world, int variant) {
  if (variant == 5) return tma_blocks_per_sm<5>(world);
  if (variant == 6) return tma_blocks_per_sm<6>(world);
  if (variant == 7) return tma_blocks_per_sm<7>(world);
  if (variant == 8) return tma_blocks_per_sm<8>(world);
  if (variant == 9) return tma_blocks_per_sm<9>(world);
  if (variant == 10) return tma_blocks_per_sm<10>(world);
  if (variant == 11) return tma_blocks_per_sm<11>(world);
  if (variant == 12) return tma_blocks_per_sm<12>(world);
  FusedFn f = select_fused(world, variant);
  int blocks = 0;
  if (f) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, f, kBlock, 0);
  return blocks > 0 ? blocks : 1;
}

cudaError_t launch_fused_step(const FusedArgs& a, int world, int grid, int variant,
                              cudaStream_t stream) {
  if (a.ntiles == 0) return cudaSuccess;
  if (a.nacc > 0 && variant >= 5) return tma_launch_acc(a, world, grid, variant, stream);
  if (variant == 5) return tma_launch<5>(a, world, grid, stream);  // 8-aligned segments only
  if (variant == 6) return tma_launch<6>(a, world, grid, stream);
  if (variant == 7) return tma_launch<7>(a, world, grid, stream);
  if (variant == 8) return tma_launch<8>(a, world, grid, stream);
  if (variant == 9) return tma_launch<9>(a, world, grid, stream);
  if (variant == 10) return tma_launch<10>(a, world, grid, stream);
  if (variant == 11) return tma_launch<11>(a, world, grid, stream);
  if (variant == 12) return tma_launch<12>(a, world, grid, stream);
  FusedFn f = select_fused(world, variant);
  if (!f) return cudaErrorInvalidValue;
  f<<<grid, kBlock, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_barrier(uint32_t* const* peer_flags, int world, int rank, int id,
                           uint32_t epoch, int* err, cudaStream_t stream) {
  barrier_kernel<<<1, 32, 0, stream>>>(peer_flags, world, rank, id, epoch, err);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const ReduceArgs& a, int world, int grid, cudaStream_t stream) {
  if (a.ntiles == 0) return cudaSuccess;
  grid = std::max(1, std::min(a.ntiles, grid));
  switch (world) {
    case 1: reduce_kernel<1><<<grid, kBlock, 0, stream>>>(a); break;
    case 2: reduce_kernel<2><<<grid, kBlock, 0, stream>>>(a); break;
    case 3: reduce_kernel<3><<<grid, kBlock, 0, stream>>>(a); break;
    case 4: reduce_kernel<4><<<grid, kBlock, 0, stream>>>(a); break;
    case 5: reduce_kernel<5><<<grid, kBlock, 0, stream>>>(a); break;
    case 6: reduce_kernel<6><<<grid, kBlock, 0, stream>>>(a); break;
    case 7: reduce_kernel<7><<<grid, kBlock, 0, stream>>>(a); break;
    case 8: reduce_kernel<8><<<grid, kBlock, 0, stream>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int adam_push_blocks_per_sm() {
  int blocks = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, adam_push_kernel, kBlock, 0);
  return blocks > 0 ? blocks : 1;
}

cudaError_t launch_adam_push(const AdamPushArgs& a, int grid, cudaStream_t stream) {
  if (a.ntiles == 0) return cudaSuccess;
  adam_push_kernel<<<std::max(1, std::min(a.ntiles, grid)), kBlock, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_p2p_pull(const PullArgs& a, int grid, cudaStream_t stream) {
  if (a.nsrc < 1 || a.nsrc > kMaxRanks || a.vecs_per_src == 0) return cudaErrorInvalidValue;
  p2p_pull_kernel<<<grid > 0 ? grid : sm_count() * 4, 256, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_spin(int ctas, unsigned long long ns, cudaStream_t stream) {
  if (ns == 0 || ctas <= 0) return cudaSuccess;
  spin_kernel<<<ctas, 128, 0, stream>>>(ns, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_init_params(const Seg* psegs, int nseg, int ntiles, uint16_t* params,
                               uint64_t seed, cudaStream_t stream) {
  if (ntiles == 0) return cudaSuccess;
  init_params_kernel<<<std::min(ntiles, sm_count() * 8), 256, 0, stream>>>(psegs, nseg, ntiles,
                                                                           params, seed);
  return cudaGetLastError();
}

cudaError_t launch_gather(const GatherArgs& a, cudaStream_t stream) {
  if (a.ntiles == 0) return cudaSuccess;
  const int grid = a.grid > 0 ? a.grid : sm_count() * 4;
  gather_kernel<<<std::min(a.ntiles, grid), 256, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_push_tma(const PushArgs& a, cudaStream_t stream) {
  if (a.ntiles == 0) return cudaSuccess;
  if (a.sp < 1 || a.sp > kMaxRanks) return cudaErrorInvalidValue;
  // CTAs per SM (tuning hook AMSP_PUSH_CTAS; 2 / 4 / 5 give 57.4 / 57.7 / 58.0 ms
  // for 13B's passes at W = 4, profiles/r02_push_ctas_13b_w4.jsonl: saturated)
  static const int per_sm = [] {
    const char* x = std::getenv("AMSP_PUSH_CTAS");
    return x && std::atoi(x) > 0 ? std::atoi(x) : 4;
  }();
  push_tma_kernel<<<std::min(a.ntiles, sm_count() * per_sm), 32, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_gather_tma(const GatherArgs& a, cudaStream_t stream) {
  if (a.ntiles == 0) return cudaSuccess;
  const int grid = a.grid > 0 ? a.grid : sm_count() * 4;
  gather_tma_kernel<<<std::min(a.ntiles, grid), 32, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_init_state(const Seg* segs, int nseg, int ntiles, float* master,
                              float* m, float* v, uint64_t seed, int grid,
                              cudaStream_t stream) {
  if (ntiles == 0) return cudaSuccess;
  init_state_kernel<<<grid, 256, 0, stream>>>(segs, nseg, ntiles, master, m, v, seed);
  return cudaGetLastError();
}

cudaError_t launch_synth_grad(uint16_t* dst, unsigned long long start,
                              unsigned long long n, uint64_t seed, int step, int rank,
                              cudaStream_t stream, int mb, bool accumulate) {
  if (n == 0) return cudaSuccess;
  if (mb < 0 || mb > 15 || rank < 0 || rank > 15) return cudaErrorInvalidValue;
  const int grid = sm_count() * 8;
  const uint32_t t = static_cast<uint32_t>(step), m = static_cast<uint32_t>(mb),
                 r = static_cast<uint32_t>(rank);
  if (accumulate)
    synth_grad_kernel<true><<<grid, 256, 0, stream>>>(dst, start, n, seed, t, m, r);
  else
    synth_grad_kernel<false><<<grid, 256, 0, stream>>>(dst, start, n, seed, t, m, r);
  return cudaGetLastError();
}

template <int NS>
void accumulate_launch(const AccumArgs& a, int grid, cudaStream_t stream) {
  if (a.first)
    accumulate_kernel<NS, true><<<grid, kBlock, 0, stream>>>(a);
  else
    accumulate_kernel<NS, false><<<grid, kBlock, 0, stream>>>(a);
}

cudaError_t launch_accumulate(const AccumArgs& a, int grid, cudaStream_t stream) {
  if (a.ntiles == 0) return cudaSuccess;
  grid = std::max(1, std::min(a.ntiles, grid > 0 ? grid : sm_count() * 4));
  switch (a.nsrc) {
    case 1: accumulate_launch<1>(a, grid, stream); break;
    case 2: accumulate_launch<2>(a, grid, stream); break;
    case 3: accumulate_launch<3>(a, grid, stream); break;
    case 4: accumulate_launch<4>(a, grid, stream); break;
    case 5: accumulate_launch<5>(a, grid, stream); break;
    case 6: accumulate_launch<6>(a, grid, stream); break;
    case 7: accumulate_launch<7>(a, grid, stream); break;
    case 8: accumulate_launch<8>(a, grid, stream); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Persistent grid for the raw kernels: one wave of resident 256-thread CTAs
// (occupancy of the kernel `fn`), fewer when n is small.
template <class F>
int raw_grid(F* fn, unsigned long long n) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const unsigned long long per_cta = 256ull * 8 * kRawU;
  const unsigned long long need = (n + per_cta - 1) / per_cta;
  return static_cast<int>(
      std::max(1ull, std::min<unsigned long long>(need, 1ull * sm_count() * per_sm)));
}

template <bool B, int U, int MINB>
void adamw_flat_launch(const void* grad, float* master, float* m, float* v,
                       uint16_t* param_out, unsigned long long n, const AdamScalars& s,
                       cudaStream_t stream) {
  adamw_flat_kernel<B, U, MINB><<<raw_grid(adamw_flat_kernel<B, U, MINB>, n), 256, 0, stream>>>(
      grad, master, m, v, param_out, n, s);
}

// Default: 4 groups (32 elements) per thread at 1 CTA/SM, 94% of measured
// HBM on 2^28 elements vs 81% for 2 groups at 2 CTAs/SM and 1 group at 4
// (profiles/r02_bench_raw_adamw_variants.jsonl). Tuning hook
// (tools/bench_raw.py): AMSP_RAW_ADAMW = 1 -> <2 groups, 2 CTAs/SM>,
// 2 -> <1 group, 4 CTAs/SM>.
int raw_adamw_variant() {
  static const int v = [] {
    const char* e = std::getenv("AMSP_RAW_ADAMW");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

cudaError_t launch_adamw_flat(const void* grad, bool bf16_grad, float* master, float* m,
                              float* v, uint16_t* param_out, unsigned long long n,
                              const AdamScalars& s, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const int var = raw_adamw_variant();
  if (bf16_grad) {
    if (var == 1) adamw_flat_launch<true, 2, 2>(grad, master, m, v, param_out, n, s, stream);
    else if (var == 2) adamw_flat_launch<true, 1, 4>(grad, master, m, v, param_out, n, s, stream);
    else adamw_flat_launch<true, 4, 1>(grad, master, m, v, param_out, n, s, stream);
  } else {
    if (var == 1) adamw_flat_launch<false, 2, 2>(grad, master, m, v, param_out, n, s, stream);
    else if (var == 2) adamw_flat_launch<false, 1, 4>(grad, master, m, v, param_out, n, s, stream);
    else adamw_flat_launch<false, 4, 1>(grad, master, m, v, param_out, n, s, stream);
  }
  return cudaGetLastError();
}

cudaError_t launch_rs_upcast_scale(const uint16_t* const* srcs, int nsrc,
                                   unsigned long long offset, float* dst,
                                   unsigned long long n, float scale, cudaStream_t stream) {
  if (nsrc < 1 || nsrc > kMaxRanks) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  RsArgs a{};
  for (int r = 0; r < nsrc; ++r) a.srcs[r] = srcs[r];
  a.nsrc = nsrc;
  a.offset = offset;
  a.n = n;
  a.dst = dst;
  a.scale = scale;
  const int grid = raw_grid(rs_upcast_scale_kernel<8>, n);
  switch (nsrc) {
    case 1: rs_upcast_scale_kernel<1><<<grid, 256, 0, stream>>>(a); break;
    case 2: rs_upcast_scale_kernel<2><<<grid, 256, 0, stream>>>(a); break;
    case 3: rs_upcast_scale_kernel<3><<<grid, 256, 0, stream>>>(a); break;
    case 4: rs_upcast_scale_kernel<4><<<grid, 256, 0, stream>>>(a); break;
    case 5: rs_upcast_scale_kernel<5><<<grid, 256, 0, stream>>>(a); break;
    case 6: rs_upcast_scale_kernel<6><<<grid, 256, 0, stream>>>(a); break;
    case 7: rs_upcast_scale_kernel<7><<<grid, 256, 0, stream>>>(a); break;
    default: rs_upcast_scale_kernel<8><<<grid, 256, 0, stream>>>(a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_ag_downcast(const float* src, unsigned long long n, uint16_t* const* dsts,
                               int ndst, unsigned long long dst_offset, cudaStream_t stream) {
  if (ndst < 1 || ndst > kMaxRanks) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  AgArgs a{};
  for (int d = 0; d < ndst; ++d) a.dsts[d] = dsts[d];
  a.ndst = ndst;
  a.dst_offset = dst_offset;
  a.n = n;
  a.src = src;
  const int grid = raw_grid(ag_downcast_kernel<8>, n);
  switch (ndst) {
    case 1: ag_downcast_kernel<1><<<grid, 256, 0, stream>>>(a); break;
    case 2: ag_downcast_kernel<2><<<grid, 256, 0, stream>>>(a); break;
    case 3: ag_downcast_kernel<3><<<grid, 256, 0, stream>>>(a); break;
    case 4: ag_downcast_kernel<4><<<grid, 256, 0, stream>>>(a); break;
    case 5: ag_downcast_kernel<5><<<grid, 256, 0, stream>>>(a); break;
    case 6: ag_downcast_kernel<6><<<grid, 256, 0, stream>>>(a); break;
    case 7: ag_downcast_kernel<7><<<grid, 256, 0, stream>>>(a); break;
    default: ag_downcast_kernel<8><<<grid, 256, 0, stream>>>(a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_upcast_scale(const uint16_t* src, float* dst, unsigned long long n,
                                float scale, cudaStream_t stream) {
  return launch_rs_upcast_scale(&src, 1, 0, dst, n, scale, stream);
}

}  // namespace amsp
