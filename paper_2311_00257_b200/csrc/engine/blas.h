// Lazily loaded cuBLAS (bf16 GEMM for the overlap scheduler's real-compute
// mode). Loaded with dlopen on first use so libamsp.so itself has no link
// dependency on cuBLAS and still loads on a machine without it.
#pragma once

#include <cuda_runtime.h>

namespace amsp {

class Blas {
 public:
  // Throws shardplan::Error when cuBLAS cannot be loaded.
  static Blas& instance();

  // Row-major helpers over cublasGemmEx (bf16 in/out, fp32 accumulate).
  // y[T,out] = x[T,in] * w[out,in]^T
  void linear_fwd(cudaStream_t s, const void* x, const void* w, void* y, int T, int in, int out);
  // dx[T,in] = dy[T,out] * w[out,in]
  void linear_dgrad(cudaStream_t s, const void* dy, const void* w, void* dx, int T, int in,
                    int out);
  // dw[out,in] = dy[T,out]^T * x[T,in]  (+ dw when accumulate: gradient
  // accumulation over micro-batches in the bf16 gradient buffer)
  void linear_wgrad(cudaStream_t s, const void* dy, const void* x, void* dw, int T, int in,
                    int out, bool accumulate = false);
  // Limit the SMs GEMM kernels are sized for (0 = all): leaves SMs free for
  // concurrently running communication / optimizer kernels.
  void set_sm_target(int sms);

 private:
  Blas();
  void gemm(cudaStream_t s, bool ta, bool tb, int m, int n, int k, const void* a, int lda,
            const void* b, int ldb, void* c, int ldc, bool accumulate = false);
  void* lib_ = nullptr;
  void* handle_ = nullptr;
  int (*create_)(void**) = nullptr;
  int (*set_stream_)(void*, cudaStream_t) = nullptr;
  int (*set_sm_target_)(void*, int) = nullptr;
  int (*gemm_ex_)(void*, int, int, int, int, int, const void*, const void*, int, int,
                  const void*, int, int, const void*, void*, int, int, int, int) = nullptr;
};

}  // namespace amsp
