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
  if (!create_ || !set_stream_ || !gemm) return;
  if (create_(&handle_) != 0) return;
  gemm_ex_ = gemm;
}

void Blas::gemm(cudaStream_t s, bool ta, bool tb, int m, int n, int k, const void* a, int lda,
                const void* b, int ldb, void* c, int ldc, bool accumulate) {
  const float one = 1.0f, zero = 0.0f;
  if (set_stream_(handle_, s) != 0) throw shardplan::Error("cublasSetStream failed");
  const int st = gemm_ex_(handle_, ta ? kOpT : kOpN, tb ? kOpT : kOpN, m, n, k, &one, a, kBf16,
                          lda, b, kBf16, ldb, accumulate ? &one : &zero, c, kBf16, ldc,
                          kCompute32F, kAlgoDefault);
  if (st != 0) throw shardplan::Error("cublasGemmEx failed with status " + std::to_string(st));
}

void Blas::set_sm_target(int sms) {
  if (!set_sm_target_) return;  // older cuBLAS: ignore the hint
  if (set_sm_target_(handle_, sms) != 0) throw shardplan::Error("cublasSetSmCountTarget failed");
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
