// Lazily loaded cuBLAS (bf16 GEMM for the overlap scheduler's real-compute
// mode). Loaded with dlopen on first use so libamsp.so itself has no link
// dependency on cuBLAS and still loads on a machine without it.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

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
  // Row-major strided-batched C_i = op(A_i) * op(B_i) (bf16, fp32 accumulate)
  // for i < batch, A_i = A + i*sA etc. (cublasGemmStridedBatchedEx).
  void bgemm(cudaStream_t s, bool ta, bool tb, int M, int N, int K, const void* A, int lda,
             long long sA, const void* B, int ldb, long long sB, void* C, int ldc, long long sC,
             int batch);
  // Limit the SMs GEMM kernels are sized for (0 = all): leaves SMs free for
  // concurrently running communication / optimizer kernels.
  void set_sm_target(int sms);

 private:
  Blas();
  // One cuBLAS handle per (device, stream), bound to that stream once: a
  // shared handle re-bound per call would reset (free) its workspace on every
  // stream switch, and cudaFree synchronises the device -- a deadlock when
  // another stream of the context holds a barrier kernel waiting on work this
  // host thread has yet to issue (emulated groups, tests/test_sync_*).
  void* handle_for(cudaStream_t s);
  void gemm(cudaStream_t s, bool ta, bool tb, int m, int n, int k, const void* a, int lda,
            const void* b, int ldb, void* c, int ldc, bool accumulate = false);
  void* lib_ = nullptr;
  void* handle_ = nullptr;  // probe handle (created when cuBLAS loads)
  std::mutex mu_;
  std::map<std::pair<int, cudaStream_t>, std::pair<void*, int>> handles_;  // -> (handle, sm target)
  int sm_target_ = 0;
  int (*create_)(void**) = nullptr;
  int (*set_stream_)(void*, cudaStream_t) = nullptr;
  int (*set_sm_target_)(void*, int) = nullptr;
  int (*gemm_ex_)(void*, int, int, int, int, int, const void*, const void*, int, int,
                  const void*, int, int, const void*, void*, int, int, int, int) = nullptr;
  int (*gemm_sb_)(void*, int, int, int, int, int, const void*, const void*, int, int, long long,
                  const void*, int, int, long long, const void*, void*, int, int, long long, int,
                  int, int) = nullptr;
};

}  // namespace amsp
