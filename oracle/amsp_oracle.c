/* amsp_oracle.c — CPU restatement of the AMSP model-state step.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the checker for the B200 data
 * plane: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it. The product path never calls it and has
 * no CPU fallback.
 *
 * PARITY UNPINNED (floating point). The reference (`shardplan`,
 * /root/reference/proj) is a planner + simulator and moves no data
 * (SPEC.md:16), so no reference code computes gradient reduction, Adam, or
 * casts. The arithmetic here is restated from the paper:
 *   - PAPER.md:272-279  per-module AG/RS on the s_p group;
 *   - PAPER.md:295-306  AllReduce over s_dp/s_p ranks, select & drop, then the
 *                       inter-tensor broadcast of updated shards (Fig 5b);
 *   - PAPER.md:320-324  s_g > s_p: keep own slice;
 *   - PAPER.md:341      2/2/12 bytes => bf16 P, bf16 G, fp32 master+m+v;
 * plus standard AdamW (decoupled weight decay, bias correction). The index
 * maps it consumes (greedy inter-tensor OS layout) ARE pinned: they come from
 * the reference's partition_tensors_greedy (cost_model.cpp:189-219), checked
 * against golden output of the compiled reference in tests/.
 *
 * Definitions shared with the GPU kernels (with the Adam
 * evaluation order fixed here so the GPU can be compared bit-for-bit):
 *   u(key)      = ((splitmix64(key) >> 40) - 2^23) * 2^-23        in [-1, 1)
 *   grad[r,t,i] = bf16_rne(2^-7 * u(seed ^ t<<48 ^ r<<40 ^ i))
 *   master0[i]  = fp32(0.02f * u(seed ^ 0xFFFF<<48 ^ i)),  m = v = 0
 *   g           = (((grad[0] + grad[1]) + ...) + grad[W-1]) * (1/W)   fp32
 *   m  = b1*m + (1-b1)*g
 *   v  = b2*v + ((1-b2)*g)*g
 *   d  = sqrt(v) * (1/sqrt(1-b2^t)) + eps
 *   p  = p * (1 - lr*wd)
 *   p  = p - (lr/(1-b1^t)) * (m / d)
 *   param = bf16_rne(p)
 * Every operation is a single IEEE-754 binary32 op (compiled with
 * -ffp-contract=off); the step scalars are computed in double and rounded
 * once to float by amsp_o_adam_scalars().
 *
 * Micro-batches and gradient sharding (the reference
 * charges them as T_g, cost_model.cpp:119-126, emits one AllReduceBucket per
 * bucket of every non-last micro-batch when s_g > s_p, overlap_sim.cpp:
 * 320-330, and stores D_g = b_g*Phi/s_g bytes, cost_model.cpp:151):
 *   grad[r,mu,t,i] = bf16_rne(2^-7 * u(seed ^ t<<48 ^ mu<<44 ^ r<<40 ^ i))
 *                    (mu = 0 is the single-micro-batch definition above)
 *   scale          = fp32(1 / (W*M))
 *   s_g = 1  ("in place"): every rank accumulates its own gradient in its
 *            full bf16 gradient buffer over all M micro-batches,
 *              acc_r = grad[r,0];  acc_r = bf16(acc_r + grad[r,mu]), mu >= 1
 *            and the step reduces   g = ((acc_0 + acc_1) + ...) * scale.
 *   s_g > 1  ("staged"): micro-batches 0..M-2 are reduced inside each
 *            accumulation block (the ranks of one G-mesh block; = the P-mesh
 *            block when s_g = s_p) into the block's bf16 G shard:
 *              mu = 0:  acc_b = bf16(grad[m0] + grad[m1] + ...)
 *              mu > 0:  acc_b = bf16(((acc_b + grad[m0]) + grad[m1]) + ...)
 *            (members m0 < m1 < ... of block b), and the step reduces the
 *            block accumulators in block order, then the raw last
 *            micro-batch of every rank in rank order:
 *              g = ((((acc_b0 + acc_b1) + ...) + grad[0,M-1]) + ... + grad[W-1,M-1]) * scale
 *   With M = 1 both reduce to the flat rank-order sum above.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#include "amsp_oracle.h"

#ifdef _OPENMP
#include <omp.h>
#endif

/* The CPU baseline uses every host thread regardless of OMP_NUM_THREADS
 * (torchrun exports 1); returns the thread count now in effect. */
int amsp_o_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

uint64_t amsp_o_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static float unit(uint64_t key) {
  int32_t q = (int32_t)(amsp_o_splitmix64(key) >> 40) - (1 << 23);
  return (float)q * (1.0f / 8388608.0f); /* exact */
}

uint16_t amsp_o_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return 0x7FC0;
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float amsp_o_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

uint16_t amsp_o_grad_bf16_mb(uint64_t seed, uint32_t step, uint32_t micro_batch,
                             uint32_t rank, uint64_t index) {
  uint64_t key = seed ^ ((uint64_t)step << 48) ^ ((uint64_t)micro_batch << 44) ^
                 ((uint64_t)rank << 40) ^ index;
  return amsp_o_f32_to_bf16(unit(key) * 0.0078125f);
}

uint16_t amsp_o_grad_bf16(uint64_t seed, uint32_t step, uint32_t rank,
                          uint64_t index) {
  return amsp_o_grad_bf16_mb(seed, step, 0, rank, index);
}

float amsp_o_master_init(uint64_t seed, uint64_t index) {
  return 0.02f * unit(seed ^ (0xFFFFull << 48) ^ index);
}

void amsp_o_adam_scalars(double lr, double beta1, double beta2, double eps,
                         double weight_decay, int step, int world,
                         amsp_o_scalars* s) {
  double bc1 = 1.0 - pow(beta1, (double)step);
  double bc2 = 1.0 - pow(beta2, (double)step);
  s->beta1 = (float)beta1;
  s->one_minus_beta1 = (float)(1.0 - beta1);
  s->beta2 = (float)beta2;
  s->one_minus_beta2 = (float)(1.0 - beta2);
  s->step_size = (float)(lr / bc1);
  s->inv_sqrt_bc2 = (float)(1.0 / sqrt(bc2));
  s->eps = (float)eps;
  s->decay = (float)(1.0 - lr * weight_decay);
  s->grad_scale = (float)(1.0 / (double)world);
}

void amsp_o_adam_elem(const amsp_o_scalars* s, float g, float* p, float* m,
                      float* v) {
  float mm = s->beta1 * *m + s->one_minus_beta1 * g;
  float vv = s->beta2 * *v + (s->one_minus_beta2 * g) * g;
  float d = sqrtf(vv) * s->inv_sqrt_bc2 + s->eps;
  float pp = *p * s->decay;
  pp = pp - s->step_size * (mm / d);
  *m = mm;
  *v = vv;
  *p = pp;
}

static float gf(uint64_t seed, int t, int mb, int r, uint64_t i) {
  return amsp_o_bf16_to_f32(amsp_o_grad_bf16_mb(seed, (uint32_t)t, (uint32_t)mb, (uint32_t)r, i));
}

static uint16_t accumulate(float acc, float g) { return amsp_o_f32_to_bf16(acc + g); }

/* Unscaled fp32 gradient of element i at step t under the accumulation
 * recipe `a` (NULL: one micro-batch, flat rank-order sum over `world`). */
float amsp_o_reduced_grad(uint64_t seed, int t, uint64_t i, int world, const amsp_o_accum* a) {
  const int M = a ? a->micro_batches : 1;
  if (M <= 1) {
    float g = gf(seed, t, 0, 0, i);
    for (int r = 1; r < world; ++r) g = g + gf(seed, t, 0, r, i);
    return g;
  }
  if (!a->staged) {
    float g = 0.0f;
    for (int r = 0; r < world; ++r) {
      uint16_t acc = amsp_o_grad_bf16_mb(seed, (uint32_t)t, 0, (uint32_t)r, i);
      for (int mb = 1; mb < M; ++mb)
        acc = accumulate(amsp_o_bf16_to_f32(acc), gf(seed, t, mb, r, i));
      g = r == 0 ? amsp_o_bf16_to_f32(acc) : g + amsp_o_bf16_to_f32(acc);
    }
    return g;
  }
  float g = 0.0f;
  for (int b = 0; b < a->nblocks; ++b) {
    uint16_t acc = 0;
    for (int mb = 0; mb + 1 < M; ++mb) {
      float s = 0.0f;
      int first = 1;
      for (int r = 0; r < world; ++r) {
        if (a->block_of[r] != b) continue;
        const float x = gf(seed, t, mb, r, i);
        if (first) s = mb == 0 ? x : amsp_o_bf16_to_f32(acc) + x;
        else s = s + x;
        first = 0;
      }
      acc = amsp_o_f32_to_bf16(s);
    }
    g = b == 0 ? amsp_o_bf16_to_f32(acc) : g + amsp_o_bf16_to_f32(acc);
  }
  for (int r = 0; r < world; ++r) g = g + gf(seed, t, M - 1, r, i);
  return g;
}

/* sc[t-1] = amsp_o_adam_scalars(..., t, world*M): hoisted out of the element
 * loop (two pow() per step dominated the per-element cost); same values. */
static void one_index(uint64_t i, uint64_t seed, int steps, int world,
                      const amsp_o_accum* a, const amsp_o_scalars* sc, float* mo,
                      float* mmo, float* vo, uint16_t* po) {
  float p = amsp_o_master_init(seed, i), m = 0.0f, v = 0.0f;
  for (int t = 1; t <= steps; ++t) {
    const amsp_o_scalars* s = &sc[t - 1];
    const float g = amsp_o_reduced_grad(seed, t, i, world, a) * s->grad_scale;
    amsp_o_adam_elem(s, g, &p, &m, &v);
  }
  if (mo) *mo = p;
  if (mmo) *mmo = m;
  if (vo) *vo = v;
  if (po) *po = amsp_o_f32_to_bf16(p);
}

static amsp_o_scalars* step_scalars(int steps, int world, const amsp_o_hyper* h) {
  amsp_o_scalars* sc = (amsp_o_scalars*)malloc(sizeof(amsp_o_scalars) * (size_t)(steps > 0 ? steps : 1));
  for (int t = 1; t <= steps; ++t)
    amsp_o_adam_scalars(h->lr, h->beta1, h->beta2, h->eps, h->weight_decay, t, world,
                        &sc[t - 1]);
  return sc;
}

static int divisor(int world, const amsp_o_accum* a) {
  return world * (a && a->micro_batches > 1 ? a->micro_batches : 1);
}

void amsp_o_trajectory_acc(const uint64_t* index, size_t n, uint64_t seed, int steps,
                           int world, const amsp_o_accum* a, const amsp_o_hyper* h,
                           float* master, float* m, float* v, uint16_t* param) {
  amsp_o_scalars* sc = step_scalars(steps, divisor(world, a), h);
#pragma omp parallel for schedule(static)
  for (size_t k = 0; k < n; ++k)
    one_index(index[k], seed, steps, world, a, sc, master ? master + k : NULL,
              m ? m + k : NULL, v ? v + k : NULL, param ? param + k : NULL);
  free(sc);
}

void amsp_o_trajectory_range_acc(uint64_t start, size_t n, uint64_t seed, int steps,
                                 int world, const amsp_o_accum* a, const amsp_o_hyper* h,
                                 float* master, float* m, float* v, uint16_t* param) {
  amsp_o_scalars* sc = step_scalars(steps, divisor(world, a), h);
#pragma omp parallel for schedule(static)
  for (size_t k = 0; k < n; ++k)
    one_index(start + k, seed, steps, world, a, sc, master ? master + k : NULL,
              m ? m + k : NULL, v ? v + k : NULL, param ? param + k : NULL);
  free(sc);
}

void amsp_o_trajectory(const uint64_t* index, size_t n, uint64_t seed,
                       int steps, int world, const amsp_o_hyper* h,
                       float* master, float* m, float* v, uint16_t* param) {
  amsp_o_trajectory_acc(index, n, seed, steps, world, NULL, h, master, m, v, param);
}

void amsp_o_trajectory_range(uint64_t start, size_t n, uint64_t seed,
                             int steps, int world, const amsp_o_hyper* h,
                             float* master, float* m, float* v,
                             uint16_t* param) {
  amsp_o_trajectory_range_acc(start, n, seed, steps, world, NULL, h, master, m, v, param);
}

void amsp_o_fill_grads_mb(uint16_t* dst, uint64_t start, size_t n, uint64_t seed,
                          uint32_t step, uint32_t micro_batch, uint32_t rank) {
#pragma omp parallel for schedule(static)
  for (size_t k = 0; k < n; ++k)
    dst[k] = amsp_o_grad_bf16_mb(seed, step, micro_batch, rank, start + k);
}

void amsp_o_fill_grads(uint16_t* dst, uint64_t start, size_t n, uint64_t seed,
                       uint32_t step, uint32_t rank) {
#pragma omp parallel for schedule(static)
  for (size_t k = 0; k < n; ++k)
    dst[k] = amsp_o_grad_bf16(seed, step, rank, start + k);
}

/* LPT greedy restated from the paper's Fig 5(b) and the reference's
 * partition_tensors_greedy (cost_model.cpp:189-219): largest first (ties by
 * index), each to the lightest shard (ties to the lower shard index).
 * O(n log n + n k); used to cross-check the engine's index map. */
static const uint64_t* g_sizes;
static int by_size_desc(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  if (g_sizes[x] != g_sizes[y]) return g_sizes[x] > g_sizes[y] ? -1 : 1;
  return x < y ? -1 : (x > y);
}

int amsp_o_partition_greedy(const uint64_t* sizes, int n, int k, int* order_buf,
                            int* assignment, uint64_t* shard_sizes) {
  if (k < 1) return 1;
  for (int i = 0; i < n; ++i) {
    if (sizes[i] == 0) return 1;
    order_buf[i] = i;
  }
  g_sizes = sizes;
  qsort(order_buf, (size_t)n, sizeof(int), by_size_desc);
  for (int s = 0; s < k; ++s) shard_sizes[s] = 0;
  for (int j = 0; j < n; ++j) {
    int best = 0;
    for (int s = 1; s < k; ++s)
      if (shard_sizes[s] < shard_sizes[best]) best = s;
    assignment[order_buf[j]] = best;
    shard_sizes[best] += sizes[order_buf[j]];
  }
  return 0;
}

/* One AMSP optimizer step over one rank's owned segments, on host memory:
 * fixed-order fp32 reduction of `world` bf16 gradient buffers, AdamW on the
 * rank's fp32 shard, bf16 downcast written into every destination parameter
 * buffer (the OS group's replicas). The CPU baseline of bench.py. */
void amsp_o_step(const uint16_t* const* grads, int world, const uint64_t* seg_flat,
                 const uint64_t* seg_os, const uint64_t* seg_len, int nseg,
                 float* master, float* m, float* v, uint16_t* const* params,
                 int ndst, const amsp_o_scalars* s) {
  for (int sg = 0; sg < nseg; ++sg) {
    const uint64_t f0 = seg_flat[sg], o0 = seg_os[sg];
    const int64_t len = (int64_t)seg_len[sg];
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < len; ++k) {
      float g = amsp_o_bf16_to_f32(grads[0][f0 + k]);
      for (int r = 1; r < world; ++r) g = g + amsp_o_bf16_to_f32(grads[r][f0 + k]);
      g = g * s->grad_scale;
      amsp_o_adam_elem(s, g, &master[o0 + k], &m[o0 + k], &v[o0 + k]);
      const uint16_t b = amsp_o_f32_to_bf16(master[o0 + k]);
      for (int d = 0; d < ndst; ++d) params[d][f0 + k] = b;
    }
  }
}
