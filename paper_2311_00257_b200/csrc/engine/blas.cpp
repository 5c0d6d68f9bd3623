// dlopen'ed cuBLAS bf16 GEMM (see blas.h). The enum values used below are
// the stable cuBLAS ABI constants (cublas_api.h / library_types.h):
// CUBLAS_OP_N = 0, CUBLAS_OP_T = 1, CUDA_R_16BF = 14, CUDA_R_32F = 0,
// CUBLAS_COMPUTE_32F = 68, CUBLAS_GEMM_DEFAULT = -1.
#include "blas.h"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include "amsp/plan.hpp"

namespace amsp {

namespace {
constexpr int kOpN = 0, kOpT = 1, kBf16 = 14, kF32 = 0, kCompute32F = 68, kAlgoDefault = -1;
}

Blas& Blas::instance() {
  static Blas* b = nullptr;
  static std::once_flag once;
  std::call_once(once, [] { b = new Blas(); });
  if (!b->gemm_ex_) throw shardplan::Error("cuBLAS could not be loaded (libcublas.so.12)");
  return *b;
}

Blas::Blas() {
  for (const char* name : {"libcublas.so.12", "libcublas.so"}) {
    lib_ = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (lib_) break;
  }
  if (!lib_) return;
  create_ = reinterpret_cast<decltype(create_)>(dlsym(lib_, "cublasCreate_v2"));
  set_stream_ = reinterpret_cast<decltype(set_stream_)>(dlsym(lib_, "cublasSetStream_v2"));
  set_sm_target_ =
      reinterpret_cast<decltype(set_sm_target_)>(dlsym(lib_, "cublasSetSmCountTarget"));
  auto gemm = reinterpret_cast<decltype(gemm_ex_)>(dlsym(lib_, "cublasGemmEx"));
  gemm_sb_ = reinterpret_cast<decltype(gemm_sb_)>(dlsym(lib_, "cublasGemmStridedBatchedEx"));
  if (!create_ || !set_stream_ || !gemm) return;
  if (create_(&handle_) != 0) return;
  gemm_ex_ = gemm;
}

void* Blas::handle_for(cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) throw shardplan::Error("cudaGetDevice failed");
  std::lock_guard<std::mutex> lock(mu_);
  auto it = handles_.find({dev, s});
  if (it == handles_.end()) {
    void* h = nullptr;
    if (create_(&h) != 0) throw shardplan::Error("cublasCreate failed");
    if (set_stream_(h, s) != 0) throw shardplan::Error("cublasSetStream failed");
    it = handles_.emplace(std::make_pair(dev, s), std::make_pair(h, 0)).first;
  }
  if (it->second.second != sm_target_ && set_sm_target_) {
    if (set_sm_target_(it->second.first, sm_target_) != 0)
      throw shardplan::Error("cublasSetSmCountTarget failed");
    it->second.second = sm_target_;
  }
  return it->second.first;
}

void Blas::gemm(cudaStream_t s, bool ta, bool tb, int m, int n, int k, const void* a, int lda,
                const void* b, int ldb, void* c, int ldc, bool accumulate) {
  const float one = 1.0f, zero = 0.0f;
  const int st = gemm_ex_(handle_for(s), ta ? kOpT : kOpN, tb ? kOpT : kOpN, m, n, k, &one, a,
                          kBf16, lda, b, kBf16, ldb, accumulate ? &one : &zero, c, kBf16, ldc,
                          kCompute32F, kAlgoDefault);
  if (st != 0) throw shardplan::Error("cublasGemmEx failed with status " + std::to_string(st));
}

void Blas::bgemm(cudaStream_t s, bool ta, bool tb, int M, int N, int K, const void* A, int lda,
                 long long sA, const void* B, int ldb, long long sB, void* C, int ldc,
                 long long sC, int batch) {
  if (!gemm_sb_) throw shardplan::Error("cublasGemmStridedBatchedEx not found in cuBLAS");
  const float one = 1.0f, zero = 0.0f;
  // row-major C = op(A) op(B)  <=>  col-major C^T = op(B)^T op(A)^T
  const int st = gemm_sb_(handle_for(s), tb ? kOpT : kOpN, ta ? kOpT : kOpN, N, M, K, &one, B,
                          kBf16, ldb, sB, A, kBf16, lda, sA, &zero, C, kBf16, ldc, sC, batch,
                          kCompute32F, kAlgoDefault);
  if (st != 0)
    throw shardplan::Error("cublasGemmStridedBatchedEx failed with status " + std::to_string(st));
}

void Blas::set_sm_target(int sms) {
  // applied to each stream's handle at its next GEMM (older cuBLAS without
  // cublasSetSmCountTarget: ignored)
  std::lock_guard<std::mutex> lock(mu_);
  sm_target_ = sms;
}

// Column-major views: a row-major [r, c] matrix is a col-major [c, r] one.
void Blas::linear_fwd(cudaStream_t s, const void* x, const void* w, void* y, int T, int in,
                      int out) {
  // Yc[out,T] = Wc[in,out]^T * Xc[in,T]
  gemm(s, true, false, out, T, in, w, in, x, in, y, out);
}

void Blas::linear_dgrad(cudaStream_t s, const void* dy, const void* w, void* dx, int T, int in,
                        int out) {
  // dXc[in,T] = Wc[in,out] * dYc[out,T]
  gemm(s, false, false, in, T, out, w, in, dy, out, dx, in);
}

void Blas::linear_wgrad(cudaStream_t s, const void* dy, const void* x, void* dw, int T, int in,
                        int out, bool accumulate) {
  // dWc[in,out] = Xc[in,T] * dYc[out,T]^T
  gemm(s, false, true, in, out, T, x, in, dy, out, dw, in, accumulate);
}

}  // namespace amsp
