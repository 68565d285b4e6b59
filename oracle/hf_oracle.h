/* TEST INFRASTRUCTURE ONLY — CPU restatement of the hfuse hot path for parity checks and
 * the bounded CPU baseline. Never linked into the product (libhfuse.so).
 *
 * Pinned against the reference itself: tests/test_oracle.py checks every function below
 * against the reference interpreter (oracle/_ref/mkfuse_ref, built from
 * /root/reference/proj/src) via the committed fixtures in tests/golden/.
 */
#ifndef HF_ORACLE_H
#define HF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* memimage.cpp:10-61 */
uint64_t hfo_splitmix64(uint64_t* state);
uint64_t hfo_mix_seed(uint64_t file_seed, int has_override, uint64_t override_seed);
void hfo_fill_uniform(float* out, int64_t n, uint64_t seed, float lo, float hi);
void hfo_fill_range(int32_t* out, int64_t n, uint64_t seed, int32_t lo, int32_t hi);

/* memimage.cpp:198-242: FNV-1a 64 over (name, NUL, type, length, cells) per array,
 * arrays then scalars, each in name order (the caller iterates in sorted order). */
uint64_t hfo_fnv_init(void);
uint64_t hfo_fnv_array(uint64_t h, const char* name, int is_float, int64_t len, const void* cells);
uint64_t hfo_fnv_scalar(uint64_t h, const char* name, int is_float, uint32_t bits);

/* machine.cpp:236-283 with the pascal-like/b200 SMConfig fields passed explicitly. */
int hfo_occupancy(int regs, int64_t shmem, int threads, int64_t regs_per_sm, int64_t shmem_per_sm,
                  int max_threads_per_sm, int max_blocks_per_sm, int* limiting);
int hfo_register_bound(int regs1, int threads1, int regs2, int threads2, int64_t fused_shmem,
                       int64_t regs_per_sm, int64_t shmem_per_sm, int max_threads_per_sm);

/* The DL members (reference-form semantics, kernels/ref/*.mk). */
void hfo_bn_stats(const float* x, int N, int C, int HW, double* mean, double* var); /* fp64 */
void hfo_hist(const float* x, int64_t n, int32_t* bins64);                            /* exact */
void hfo_maxpool(const float* x, int NC, int H, int W, float* y, int32_t* idx);       /* exact */
void hfo_upsample(const float* x, int NC, int IH, int IW, float* y);                  /* exact */
void hfo_im2col(const float* x, int NC, int H, int W, float* col);                    /* exact */

int hfo_threads(void);

#ifdef __cplusplus
}
#endif
#endif
