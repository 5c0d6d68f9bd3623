// Real-compute kernels of the overlap scheduler's compute='gemm' mode
// (compute.cu): attention softmax and RMSNorm, beside the cuBLAS GEMMs.
// Compute stand-ins with the real shapes and costs, not the AMSP path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace amsp {

// In-place causal softmax over `rows` rows of `cols` bf16 scores; row r is
// query r % q_rows (keys > query masked), logits scaled by `scale`.
cudaError_t launch_softmax_rows(uint16_t* p, long long rows, int cols, int q_rows, float scale,
                                cudaStream_t s);
// dp <- p * (dp - rowsum(p * dp)) * scale (softmax backward, in place).
cudaError_t launch_softmax_bwd_rows(const uint16_t* p, uint16_t* dp, long long rows, int cols,
                                    float scale, cudaStream_t s);
// RMSNorm over T rows of H: y = x * rsqrt(mean(x^2) + eps) * w.
cudaError_t launch_rmsnorm_fwd(const uint16_t* x, const uint16_t* w, uint16_t* y, int T, int H,
                               cudaStream_t s);
cudaError_t launch_rmsnorm_dgrad(const uint16_t* x, const uint16_t* w, const uint16_t* dy,
                                 uint16_t* dx, int T, int H, cudaStream_t s);
// dw[H] (bf16, += when accumulate) = sum_t dy * x_hat; acc = fp32[H] scratch,
// zero on entry and left zero.
cudaError_t launch_rmsnorm_wgrad(const uint16_t* x, const uint16_t* dy, float* acc, uint16_t* dw,
                                 int T, int H, bool accumulate, cudaStream_t s);

}  // namespace amsp
