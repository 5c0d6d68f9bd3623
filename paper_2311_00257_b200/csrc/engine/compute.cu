// Real-compute kernels of the overlap scheduler's compute='gemm' mode: the
// parts of a LLaMA layer that are not linear-module GEMMs (those run on
// cuBLAS, blas.cpp). They give the compute stream the shape and cost of a
// real step (6*Phi*B*S linear FLOPs + 12*L*B*S^2*H attention FLOPs, the
// reference's compute model, overlap_sim.cpp:97-110) so the measured
// exposed communication is against realistic compute. They are NOT part of
// the AMSP model-state path, and values only need to stay finite.
//
//   softmax_rows_kernel      causal row softmax of the attention scores
//   softmax_bwd_rows_kernel  dS = P * (dP - rowsum(P * dP))
//   rmsnorm_fwd_kernel       y = x * rsqrt(mean(x^2) + eps) * w
//   rmsnorm_dgrad_kernel     dx of the same
//   rmsnorm_wgrad_kernel     dw = sum_t dy * x_hat (fp32 column partials,
//                            then bf16 into the gradient buffer)
#include <cuda_runtime.h>

#include <algorithm>

#include "compute.h"
#include "kernels.cuh"

namespace amsp {
namespace {

constexpr int kWarps = 8;  // rows per CTA (one warp per row)

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// One warp per row of `cols` bf16 scores (cols % 8 == 0: each lane owns the
// 8-element chunks lane, lane+32, ...). Row r of a
// [rows_per_head, cols] block is query (r % rows_per_head); keys > query are
// masked (causal).
__global__ void __launch_bounds__(kWarps * 32) softmax_rows_kernel(uint16_t* p, long long rows,
                                                                   int cols, int q_rows,
                                                                   float scale) {
  const long long row = static_cast<long long>(blockIdx.x) * kWarps + threadIdx.x / 32;
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const int q = static_cast<int>(row % q_rows);
  uint16_t* x = p + row * cols;
  float mx = -INFINITY;
  for (int c = lane * 8; c < cols; c += 256) {
    const uint4 w = *reinterpret_cast<const uint4*>(x + c);
    const uint32_t* u = reinterpret_cast<const uint32_t*>(&w);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (c + 2 * k <= q) mx = fmaxf(mx, bf16_lo(u[k]) * scale);
      if (c + 2 * k + 1 <= q) mx = fmaxf(mx, bf16_hi(u[k]) * scale);
    }
  }
  mx = warp_max(mx);
  float sum = 0.0f;
  for (int c = lane * 8; c < cols; c += 256) {
    const uint4 w = *reinterpret_cast<const uint4*>(x + c);
    const uint32_t* u = reinterpret_cast<const uint32_t*>(&w);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (c + 2 * k <= q) sum += __expf(bf16_lo(u[k]) * scale - mx);
      if (c + 2 * k + 1 <= q) sum += __expf(bf16_hi(u[k]) * scale - mx);
    }
  }
  const float inv = 1.0f / warp_sum(sum);
  for (int c = lane * 8; c < cols; c += 256) {
    const uint4 w = *reinterpret_cast<const uint4*>(x + c);
    const uint32_t* u = reinterpret_cast<const uint32_t*>(&w);
    float y[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      y[2 * k] = c + 2 * k <= q ? __expf(bf16_lo(u[k]) * scale - mx) * inv : 0.0f;
      y[2 * k + 1] = c + 2 * k + 1 <= q ? __expf(bf16_hi(u[k]) * scale - mx) * inv : 0.0f;
    }
    *reinterpret_cast<uint4*>(x + c) =
        make_uint4(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]), pack_bf16x2(y[4], y[5]),
                   pack_bf16x2(y[6], y[7]));
  }
}

__global__ void __launch_bounds__(kWarps * 32) softmax_bwd_rows_kernel(const uint16_t* p,
                                                                       uint16_t* dp,
                                                                       long long rows, int cols,
                                                                       float scale) {
  const long long row = static_cast<long long>(blockIdx.x) * kWarps + threadIdx.x / 32;
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const uint16_t* pr = p + row * cols;
  uint16_t* dr = dp + row * cols;
  float dot = 0.0f;
  for (int c = lane * 8; c < cols; c += 256) {
    const uint4 a = *reinterpret_cast<const uint4*>(pr + c);
    const uint4 b = *reinterpret_cast<const uint4*>(dr + c);
    const uint32_t* ua = reinterpret_cast<const uint32_t*>(&a);
    const uint32_t* ub = reinterpret_cast<const uint32_t*>(&b);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      dot += bf16_lo(ua[k]) * bf16_lo(ub[k]) + bf16_hi(ua[k]) * bf16_hi(ub[k]);
  }
  dot = warp_sum(dot);
  for (int c = lane * 8; c < cols; c += 256) {
    const uint4 a = *reinterpret_cast<const uint4*>(pr + c);
    const uint4 b = *reinterpret_cast<const uint4*>(dr + c);
    const uint32_t* ua = reinterpret_cast<const uint32_t*>(&a);
    const uint32_t* ub = reinterpret_cast<const uint32_t*>(&b);
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      o[k] = pack_bf16x2(bf16_lo(ua[k]) * (bf16_lo(ub[k]) - dot) * scale,
                         bf16_hi(ua[k]) * (bf16_hi(ub[k]) - dot) * scale);
    *reinterpret_cast<uint4*>(dr + c) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// RMSNorm over rows of H (H % 8 == 0): one warp per token row.
__global__ void __launch_bounds__(kWarps * 32) rmsnorm_fwd_kernel(const uint16_t* x,
                                                                  const uint16_t* w, uint16_t* y,
                                                                  int T, int H, float eps) {
  const int row = blockIdx.x * kWarps + threadIdx.x / 32;
  if (row >= T) return;
  const int lane = threadIdx.x & 31;
  const uint16_t* xr = x + static_cast<long long>(row) * H;
  float ss = 0.0f;
  for (int c = lane * 8; c < H; c += 256) {
    float v[8];
    const uint4 a = *reinterpret_cast<const uint4*>(xr + c);
    const uint32_t* u = reinterpret_cast<const uint32_t*>(&a);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[2 * k] = bf16_lo(u[k]);
      v[2 * k + 1] = bf16_hi(u[k]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) ss += v[k] * v[k];
  }
  const float r = rsqrtf(warp_sum(ss) / H + eps);
  for (int c = lane * 8; c < H; c += 256) {
    const uint4 a = *reinterpret_cast<const uint4*>(xr + c);
    const uint4 b = *reinterpret_cast<const uint4*>(w + c);
    const uint32_t* ua = reinterpret_cast<const uint32_t*>(&a);
    const uint32_t* ub = reinterpret_cast<const uint32_t*>(&b);
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      o[k] = pack_bf16x2(bf16_lo(ua[k]) * r * bf16_lo(ub[k]), bf16_hi(ua[k]) * r * bf16_hi(ub[k]));
    *reinterpret_cast<uint4*>(y + static_cast<long long>(row) * H + c) =
        make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// dx = r * (w*dy - x_hat * mean(x_hat * w*dy)), x_hat = x * r.
__global__ void __launch_bounds__(kWarps * 32) rmsnorm_dgrad_kernel(const uint16_t* x,
                                                                    const uint16_t* w,
                                                                    const uint16_t* dy,
                                                                    uint16_t* dx, int T, int H,
                                                                    float eps) {
  const int row = blockIdx.x * kWarps + threadIdx.x / 32;
  if (row >= T) return;
  const int lane = threadIdx.x & 31;
  const long long base = static_cast<long long>(row) * H;
  float ss = 0.0f, dot = 0.0f;
  for (int c = lane * 8; c < H; c += 256) {
    const uint4 a = *reinterpret_cast<const uint4*>(x + base + c);
    const uint4 b = *reinterpret_cast<const uint4*>(w + c);
    const uint4 g = *reinterpret_cast<const uint4*>(dy + base + c);
    const uint32_t* ua = reinterpret_cast<const uint32_t*>(&a);
    const uint32_t* ub = reinterpret_cast<const uint32_t*>(&b);
    const uint32_t* ug = reinterpret_cast<const uint32_t*>(&g);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float x0 = bf16_lo(ua[k]), x1 = bf16_hi(ua[k]);
      ss += x0 * x0 + x1 * x1;
      dot += x0 * bf16_lo(ub[k]) * bf16_lo(ug[k]) + x1 * bf16_hi(ub[k]) * bf16_hi(ug[k]);
    }
  }
  ss = warp_sum(ss);
  dot = warp_sum(dot);
  const float r = rsqrtf(ss / H + eps);
  const float coef = dot * r * r / H;
  for (int c = lane * 8; c < H; c += 256) {
    const uint4 a = *reinterpret_cast<const uint4*>(x + base + c);
    const uint4 b = *reinterpret_cast<const uint4*>(w + c);
    const uint4 g = *reinterpret_cast<const uint4*>(dy + base + c);
    const uint32_t* ua = reinterpret_cast<const uint32_t*>(&a);
    const uint32_t* ub = reinterpret_cast<const uint32_t*>(&b);
    const uint32_t* ug = reinterpret_cast<const uint32_t*>(&g);
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      o[k] = pack_bf16x2(r * (bf16_lo(ub[k]) * bf16_lo(ug[k]) - bf16_lo(ua[k]) * coef),
                         r * (bf16_hi(ub[k]) * bf16_hi(ug[k]) - bf16_hi(ua[k]) * coef));
    *reinterpret_cast<uint4*>(dx + base + c) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// Column partial sums of dy * x_hat over a slab of rows per CTA (256
// threads, each owning 8 consecutive columns of a 2048-column panel),
// atomically added into fp32 acc[H].
constexpr int kNormSlab = 64;
__global__ void __launch_bounds__(256) rmsnorm_wgrad_kernel(const uint16_t* x,
                                                            const uint16_t* dy, float* acc,
                                                            int T, int H, float eps) {
  const int c = (blockIdx.y * 256 + threadIdx.x) * 8;
  const int r0 = blockIdx.x * kNormSlab;
  __shared__ float rstd[kNormSlab];
  // per-row rstd: warp w computes rows w, w+8, ...
  const int lane = threadIdx.x & 31, wid = threadIdx.x / 32;
  for (int rr = wid; rr < kNormSlab; rr += 8) {
    const int row = r0 + rr;
    float ss = 0.0f;
    if (row < T)
      for (int k = lane; k < H; k += 32) {
        const float v = bf16_at(x[static_cast<long long>(row) * H + k]);
        ss += v * v;
      }
    ss = warp_sum(ss);
    if (lane == 0) rstd[rr] = rsqrtf(ss / H + eps);
  }
  __syncthreads();
  if (c >= H) return;
  float s[8] = {};
  for (int rr = 0; rr < kNormSlab && r0 + rr < T; ++rr) {
    const long long o = static_cast<long long>(r0 + rr) * H + c;
    const uint4 a = *reinterpret_cast<const uint4*>(x + o);
    const uint4 g = *reinterpret_cast<const uint4*>(dy + o);
    const uint32_t* ua = reinterpret_cast<const uint32_t*>(&a);
    const uint32_t* ug = reinterpret_cast<const uint32_t*>(&g);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      s[2 * k] += bf16_lo(ua[k]) * rstd[rr] * bf16_lo(ug[k]);
      s[2 * k + 1] += bf16_hi(ua[k]) * rstd[rr] * bf16_hi(ug[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) atomicAdd(acc + c + k, s[k]);
}

__global__ void norm_grad_finish_kernel(float* acc, uint16_t* dw, int H, int accumulate) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < H; i += gridDim.x * blockDim.x) {
    const float g = accumulate ? __fadd_rn(bf16_at(dw[i]), acc[i]) : acc[i];
    dw[i] = to_bf16(g);
    acc[i] = 0.0f;  // ready for the next norm's partial sums
  }
}

}  // namespace

cudaError_t launch_softmax_rows(uint16_t* p, long long rows, int cols, int q_rows, float scale,
                                cudaStream_t s) {
  if (cols % 8 != 0 || rows <= 0) return cudaErrorInvalidValue;
  softmax_rows_kernel<<<static_cast<unsigned>((rows + kWarps - 1) / kWarps), kWarps * 32, 0,
                        s>>>(p, rows, cols, q_rows, scale);
  return cudaGetLastError();
}

cudaError_t launch_softmax_bwd_rows(const uint16_t* p, uint16_t* dp, long long rows, int cols,
                                    float scale, cudaStream_t s) {
  if (cols % 8 != 0 || rows <= 0) return cudaErrorInvalidValue;
  softmax_bwd_rows_kernel<<<static_cast<unsigned>((rows + kWarps - 1) / kWarps), kWarps * 32, 0,
                            s>>>(p, dp, rows, cols, scale);
  return cudaGetLastError();
}

cudaError_t launch_rmsnorm_fwd(const uint16_t* x, const uint16_t* w, uint16_t* y, int T, int H,
                               cudaStream_t s) {
  if (H % 8 != 0 || T <= 0) return cudaErrorInvalidValue;
  rmsnorm_fwd_kernel<<<(T + kWarps - 1) / kWarps, kWarps * 32, 0, s>>>(x, w, y, T, H, 1e-6f);
  return cudaGetLastError();
}

cudaError_t launch_rmsnorm_dgrad(const uint16_t* x, const uint16_t* w, const uint16_t* dy,
                                 uint16_t* dx, int T, int H, cudaStream_t s) {
  if (H % 8 != 0 || T <= 0) return cudaErrorInvalidValue;
  rmsnorm_dgrad_kernel<<<(T + kWarps - 1) / kWarps, kWarps * 32, 0, s>>>(x, w, dy, dx, T, H,
                                                                         1e-6f);
  return cudaGetLastError();
}

cudaError_t launch_rmsnorm_wgrad(const uint16_t* x, const uint16_t* dy, float* acc, uint16_t* dw,
                                 int T, int H, bool accumulate, cudaStream_t s) {
  if (H % 8 != 0 || T <= 0) return cudaErrorInvalidValue;
  const dim3 grid((T + kNormSlab - 1) / kNormSlab, (H + 2047) / 2048);
  rmsnorm_wgrad_kernel<<<grid, 256, 0, s>>>(x, dy, acc, T, H, 1e-6f);
  norm_grad_finish_kernel<<<(H + 255) / 256, 256, 0, s>>>(acc, dw, H, accumulate ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace amsp
