/* amsp_oracle.h — CPU checker for the AMSP B200 data plane (test infra only;
 * see amsp_oracle.c for the definitions and the "parity unpinned" note). */
#ifndef AMSP_ORACLE_H_
#define AMSP_ORACLE_H_

#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  float beta1, one_minus_beta1, beta2, one_minus_beta2;
  float step_size, inv_sqrt_bc2, eps, decay, grad_scale;
} amsp_o_scalars;

typedef struct {
  double lr, beta1, beta2, eps, weight_decay;
} amsp_o_hyper;

/* Gradient-accumulation recipe (see amsp_oracle.c header). block_of[r]
 * numbers the accumulation blocks in order of their smallest rank. */
typedef struct {
  int micro_batches;  /* M >= 1 */
  int staged;         /* 0: s_g = 1 (in place); 1: s_g > 1 (block accumulators) */
  int nblocks;
  int block_of[16];
} amsp_o_accum;

int amsp_o_set_threads(int n);
uint64_t amsp_o_splitmix64(uint64_t x);
uint16_t amsp_o_f32_to_bf16(float f);
float amsp_o_bf16_to_f32(uint16_t h);
uint16_t amsp_o_grad_bf16(uint64_t seed, uint32_t step, uint32_t rank, uint64_t index);
uint16_t amsp_o_grad_bf16_mb(uint64_t seed, uint32_t step, uint32_t micro_batch,
                             uint32_t rank, uint64_t index);
float amsp_o_master_init(uint64_t seed, uint64_t index);
float amsp_o_reduced_grad(uint64_t seed, int t, uint64_t i, int world, const amsp_o_accum* a);
void amsp_o_trajectory_acc(const uint64_t* index, size_t n, uint64_t seed, int steps,
                           int world, const amsp_o_accum* a, const amsp_o_hyper* h,
                           float* master, float* m, float* v, uint16_t* param);
void amsp_o_trajectory_range_acc(uint64_t start, size_t n, uint64_t seed, int steps,
                                 int world, const amsp_o_accum* a, const amsp_o_hyper* h,
                                 float* master, float* m, float* v, uint16_t* param);
void amsp_o_fill_grads_mb(uint16_t* dst, uint64_t start, size_t n, uint64_t seed,
                          uint32_t step, uint32_t micro_batch, uint32_t rank);
void amsp_o_adam_scalars(double lr, double beta1, double beta2, double eps,
                         double weight_decay, int step, int world,
                         amsp_o_scalars* s);
void amsp_o_adam_elem(const amsp_o_scalars* s, float g, float* p, float* m, float* v);
void amsp_o_trajectory(const uint64_t* index, size_t n, uint64_t seed, int steps,
                       int world, const amsp_o_hyper* h, float* master, float* m,
                       float* v, uint16_t* param);
void amsp_o_trajectory_range(uint64_t start, size_t n, uint64_t seed, int steps,
                             int world, const amsp_o_hyper* h, float* master,
                             float* m, float* v, uint16_t* param);
void amsp_o_fill_grads(uint16_t* dst, uint64_t start, size_t n, uint64_t seed,
                       uint32_t step, uint32_t rank);
int amsp_o_partition_greedy(const uint64_t* sizes, int n, int k, int* order_buf,
                            int* assignment, uint64_t* shard_sizes);
void amsp_o_step(const uint16_t* const* grads, int world, const uint64_t* seg_flat,
                 const uint64_t* seg_os, const uint64_t* seg_len, int nseg,
                 float* master, float* m, float* v, uint16_t* const* params,
                 int ndst, const amsp_o_scalars* s);

#ifdef __cplusplus
}
#endif
#endif
