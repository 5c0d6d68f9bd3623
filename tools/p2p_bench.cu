// NVLink peer-memory microbenchmark (tuning aid for the fused step kernel).
// One process drives every visible GPU with peer access enabled; kernels on
// different GPUs run concurrently and never wait on each other.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_bench tools/p2p_bench.cu
//   ./p2p_bench [bytes_per_gpu]
// Modes (GB/s per GPU, data bytes moved / time):
//   local     : HBM copy on each GPU
//   pull      : every GPU reads a peer's buffer into local memory
//   push      : every GPU writes its local buffer into a peer's memory
//   pull+push : every GPU pulls half and pushes half (two streams)
//   reduce2   : out[i] = a[i] + peer_b[i] (bf16 pairs, the fused kernel's read mix)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                    \
      std::exit(1);                                                             \
    }                                                                           \
  } while (0)

__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

__global__ void add_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b,
                           uint4* __restrict__ out, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint4 x = a[i], y = b[i];
    out[i] = make_uint4(x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w);
  }
}

// Gather-shaped pull: `parts` sources read back to back (one contiguous slice
// each), 2 x 16 B per thread per 8 KB tile, persistent grid-stride tiles.
struct Srcs {
  const uint4* p[8];
};
__global__ void gather_like(Srcs s, int parts, int rot, uint4* __restrict__ dst, size_t slice16) {
  const size_t tiles_per = (slice16 + 511) / 512;  // 512 x 16 B = 8 KB tiles
  const size_t ntiles = tiles_per * parts;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int j = static_cast<int>(t / tiles_per);
    const int q = (rot + j) % parts;
    const size_t base = (t % tiles_per) * 512;
    const uint4* src = s.p[q];
    size_t i0 = base + threadIdx.x, i1 = base + 256 + threadIdx.x;
    uint4 a, b;
    const bool ok0 = i0 < slice16, ok1 = i1 < slice16;
    if (ok0) a = src[i0];
    if (ok1) b = src[i1];
    if (ok0) dst[q * slice16 + i0] = a;
    if (ok1) dst[q * slice16 + i1] = b;
  }
}

int main(int argc, char** argv) {
  size_t bytes = argc > 1 ? strtoull(argv[1], nullptr, 10) : (size_t(1) << 31);
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  if (ng < 2) {
    std::printf("need >= 2 GPUs\n");
    return 0;
  }
  const size_t n = bytes / 16;
  std::vector<uint4*> a(ng), b(ng), c(ng);
  std::vector<cudaStream_t> s0(ng), s1(ng);
  std::vector<cudaEvent_t> e0(ng), e1(ng);
  int sms = 148;
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    for (int p = 0; p < ng; ++p)
      if (p != g) CK(cudaDeviceEnablePeerAccess(p, 0));
    CK(cudaMalloc(&a[g], bytes));
    CK(cudaMalloc(&b[g], bytes));
    CK(cudaMalloc(&c[g], bytes));
    CK(cudaMemset(a[g], 1, bytes));
    CK(cudaMemset(b[g], 2, bytes));
    CK(cudaStreamCreateWithFlags(&s0[g], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s1[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g));
  }
  auto run = [&](const char* name, int grid_mult, auto launch, double bytes_per_gpu) {
    for (int rep = 0; rep < 2; ++rep) {  // rep 0 = warm-up
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(e0[g], s0[g]));
        CK(cudaStreamWaitEvent(s1[g], e0[g], 0));
        launch(g, sms * grid_mult);
        cudaEvent_t j;
        CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
        CK(cudaEventRecord(j, s1[g]));
        CK(cudaStreamWaitEvent(s0[g], j, 0));
        CK(cudaEventRecord(e1[g], s0[g]));
      }
      double worst = 0;
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        worst = ms > worst ? ms : worst;
      }
      if (rep == 1)
        std::printf("%-28s grid=%4dx%d  %8.3f ms  %7.1f GB/s per GPU\n", name, sms, grid_mult,
                    worst, bytes_per_gpu / (worst * 1e-3) / 1e9);
    }
  };
  const int peers = ng;
  for (int gm : {2, 4, 8}) {
    run("local copy", gm, [&](int g, int grid) {
      copy_kernel<<<grid, 256, 0, s0[g]>>>(a[g], c[g], n);
    }, 2.0 * bytes);
    run("pull (read peer)", gm, [&](int g, int grid) {
      copy_kernel<<<grid, 256, 0, s0[g]>>>(a[(g + 1) % peers], c[g], n);
    }, 1.0 * bytes);
    run("push (write peer)", gm, [&](int g, int grid) {
      copy_kernel<<<grid, 256, 0, s0[g]>>>(a[g], c[(g + 1) % peers], n);
    }, 1.0 * bytes);
    run("pull+push (2 streams)", gm, [&](int g, int grid) {
      copy_kernel<<<grid / 2, 256, 0, s0[g]>>>(a[(g + 1) % peers], c[g], n / 2);
      copy_kernel<<<grid / 2, 256, 0, s1[g]>>>(b[g], c[(g + 1) % peers] + n / 2, n / 2);
    }, 1.0 * bytes);
    run("reduce2 (a + peer b)", gm, [&](int g, int grid) {
      add_kernel<<<grid, 256, 0, s0[g]>>>(a[g], b[(g + 1) % peers], c[g], n);
    }, 1.0 * bytes);
    // All-gather shaped: every GPU pulls one slice from each peer (rotated
    // start), slices of bytes/ng; data moved over NVLink = bytes*(ng-1)/ng.
    run("gather-like rotated", gm, [&](int g, int grid) {
      Srcs s{};
      for (int q = 0; q < ng; ++q) s.p[q] = a[q] + (size_t)q * (n / ng);
      gather_like<<<grid, 256, 0, s0[g]>>>(s, ng, g + 1, c[g], n / ng);
    }, 1.0 * bytes * (ng - 1) / ng);
    run("gather-like same order", gm, [&](int g, int grid) {
      Srcs s{};
      for (int q = 0; q < ng; ++q) s.p[q] = a[q] + (size_t)q * (n / ng);
      gather_like<<<grid, 256, 0, s0[g]>>>(s, ng, 0, c[g], n / ng);
    }, 1.0 * bytes * (ng - 1) / ng);
  }
  return 0;
}
