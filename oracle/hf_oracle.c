/* TEST INFRASTRUCTURE ONLY — see hf_oracle.h. Compiled with -ffp-contract=off so every
 * float expression rounds exactly like the reference interpreter (x86-64 SSE, no FMA,
 * /root/reference/proj/src/exec.cpp:491-531). OpenMP splits independent output rows /
 * channels only; each value is computed by one thread in the reference order. */
#include "hf_oracle.h"

#include <math.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GOLDEN 0x9E3779B97F4A7C15ULL

static uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* memimage.cpp:10-16 */
uint64_t hfo_splitmix64(uint64_t* state) {
  *state += GOLDEN;
  return mix(*state);
}

/* memimage.cpp:20-24 */
uint64_t hfo_mix_seed(uint64_t file_seed, int has_override, uint64_t ov) {
  if (!has_override) return file_seed;
  uint64_t s = file_seed ^ (ov * GOLDEN);
  return hfo_splitmix64(&s);
}

/* memimage.cpp:26-29, 52-61; element i is the (i+1)-th splitmix64 output. */
void hfo_fill_uniform(float* out, int64_t n, uint64_t seed, float lo, float hi) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t bits = mix(seed + (uint64_t)(i + 1) * GOLDEN);
    float unit = (float)(bits >> 40) * (1.0f / 16777216.0f);
    out[i] = lo + unit * (hi - lo);
  }
}

/* memimage.cpp:39-50 */
void hfo_fill_range(int32_t* out, int64_t n, uint64_t seed, int32_t lo, int32_t hi) {
  uint64_t span = (uint64_t)((int64_t)hi - lo) + 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t bits = mix(seed + (uint64_t)(i + 1) * GOLDEN);
    out[i] = (int32_t)(lo + (int64_t)(bits % span));
  }
}

/* memimage.cpp:198-242 */
static uint64_t eat(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = (const unsigned char*)p;
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ULL;
  }
  return h;
}

static uint64_t eat_u32(uint64_t h, uint32_t v) {
  unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16),
                        (unsigned char)(v >> 24)};
  return eat(h, b, 4);
}

uint64_t hfo_fnv_init(void) { return 14695981039346656037ULL; }

uint64_t hfo_fnv_array(uint64_t h, const char* name, int is_float, int64_t len, const void* cells) {
  h = eat(h, name, strlen(name) + 1); /* name + NUL */
  h = eat_u32(h, is_float ? 1u : 0u);
  h = eat_u32(h, (uint32_t)len);
  /* little-endian cells == the u32 byte order of the reference */
  return eat(h, cells, (size_t)len * 4);
}

uint64_t hfo_fnv_scalar(uint64_t h, const char* name, int is_float, uint32_t bits) {
  h = eat(h, name, strlen(name) + 1);
  h = eat_u32(h, is_float ? 1u : 0u);
  return eat_u32(h, bits);
}

/* machine.cpp:236-267 */
int hfo_occupancy(int regs, int64_t shmem, int threads, int64_t regs_per_sm, int64_t shmem_per_sm,
                  int max_threads_per_sm, int max_blocks_per_sm, int* limiting) {
  int64_t q[4];
  q[0] = regs_per_sm / ((int64_t)regs * threads);
  q[1] = shmem == 0 ? INT64_MAX : shmem_per_sm / shmem;
  q[2] = max_threads_per_sm / threads;
  q[3] = max_blocks_per_sm;
  int64_t best = q[0];
  for (int i = 1; i < 4; ++i)
    if (q[i] < best) best = q[i];
  for (int i = 0; i < 4; ++i)
    if (q[i] == best) {
      if (limiting) *limiting = i;
      break;
    }
  return (int)best;
}

/* machine.cpp:269-283: b1, b2, b0, r0 by floor division */
int hfo_register_bound(int regs1, int threads1, int regs2, int threads2, int64_t fused_shmem,
                       int64_t regs_per_sm, int64_t shmem_per_sm, int max_threads_per_sm) {
  int64_t d0 = (int64_t)threads1 + threads2;
  int64_t b1 = regs_per_sm / ((int64_t)threads1 * regs1);
  int64_t b2 = regs_per_sm / ((int64_t)threads2 * regs2);
  int64_t bs = fused_shmem == 0 ? INT64_MAX : shmem_per_sm / fused_shmem;
  int64_t bt = max_threads_per_sm / d0;
  int64_t b0 = b1 < b2 ? b1 : b2;
  if (bs < b0) b0 = bs;
  if (bt < b0) b0 = bt;
  if (b0 <= 0) return -1;
  return (int)(regs_per_sm / (b0 * d0));
}

/* BatchNorm collect-statistics (kernels/ref/batchnorm.mk): mean and biased variance per
 * channel, computed in double (two-pass) as an independent high-precision oracle. */
void hfo_bn_stats(const float* x, int N, int C, int HW, double* mean, double* var) {
#pragma omp parallel for schedule(dynamic)
  for (int c = 0; c < C; ++c) {
    double s = 0.0;
    for (int b = 0; b < N; ++b) {
      const float* p = x + ((int64_t)b * C + c) * HW;
      for (int i = 0; i < HW; ++i) s += p[i];
    }
    double m = s / ((double)N * HW), q = 0.0;
    for (int b = 0; b < N; ++b) {
      const float* p = x + ((int64_t)b * C + c) * HW;
      for (int i = 0; i < HW; ++i) {
        double d = p[i] - m;
        q += d * d;
      }
    }
    mean[c] = m;
    var[c] = q / ((double)N * HW);
  }
}

/* Histogram (kernels/ref/histogram.mk): int((v - lo) * nbins / (hi - lo)) in float,
 * v == hi -> last bin, out-of-range values ignored; lo = -4, hi = 4, 64 bins. */
void hfo_hist(const float* x, int64_t n, int32_t* bins) {
  memset(bins, 0, 64 * sizeof(int32_t));
#pragma omp parallel
  {
    int32_t local[64] = {0};
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      float v = x[i];
      if (v >= -4.0f && v <= 4.0f) {
        int b = (int)((v - -4.0f) * 64.0f / (4.0f - -4.0f));
        if (b == 64) b = 63;
        local[b]++;
      }
    }
#pragma omp critical
    for (int b = 0; b < 64; ++b) bins[b] += local[b];
  }
}

/* MaxPool2d 3x3/s2/p1 with indices (kernels/ref/maxpool.mk, PyTorch scan + NaN rule). */
void hfo_maxpool(const float* x, int NC, int H, int W, float* y, int32_t* idx) {
  int OH = (H + 2 - 3) / 2 + 1, OW = (W + 2 - 3) / 2 + 1;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (int64_t)NC * OH; ++r) {
    int nc = (int)(r / OH), oh = (int)(r % OH);
    for (int ow = 0; ow < OW; ++ow) {
      int hs = oh * 2 - 1, ws = ow * 2 - 1;
      int he = hs + 3 < H ? hs + 3 : H, we = ws + 3 < W ? ws + 3 : W;
      if (hs < 0) hs = 0;
      if (ws < 0) ws = 0;
      float best = -INFINITY;
      int bi = hs * W + ws;
      for (int h = hs; h < he; ++h)
        for (int w = ws; w < we; ++w) {
          float v = x[((int64_t)nc * H + h) * W + w];
          if (v > best || v != v) {
            best = v;
            bi = h * W + w;
          }
        }
      y[r * OW + ow] = best;
      idx[r * OW + ow] = bi;
    }
  }
}

/* Upsample bilinear 2x, align_corners=False (kernels/ref/upsample.mk arithmetic). */
void hfo_upsample(const float* x, int NC, int IH, int IW, float* y) {
  int OH = 2 * IH, OW = 2 * IW;
  float rh = (float)IH / (float)OH, rw = (float)IW / (float)OW;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (int64_t)NC * OH; ++r) {
    int nc = (int)(r / OH), oh = (int)(r % OH);
    float h1r = rh * ((float)oh + 0.5f) - 0.5f;
    if (h1r < 0.0f) h1r = 0.0f;
    int h1 = (int)h1r;
    int h1p = h1 < IH - 1 ? 1 : 0;
    float h1l = h1r - (float)h1, h0l = 1.0f - h1l;
    const float* r0 = x + ((int64_t)nc * IH + h1) * IW;
    const float* r1 = x + ((int64_t)nc * IH + h1 + h1p) * IW;
    for (int ow = 0; ow < OW; ++ow) {
      float w1r = rw * ((float)ow + 0.5f) - 0.5f;
      if (w1r < 0.0f) w1r = 0.0f;
      int w1 = (int)w1r;
      int w1p = w1 < IW - 1 ? 1 : 0;
      float w1l = w1r - (float)w1, w0l = 1.0f - w1l;
      y[r * OW + ow] = h0l * (w0l * r0[w1] + w1l * r0[w1 + w1p]) + h1l * (w0l * r1[w1] + w1l * r1[w1 + w1p]);
    }
  }
}

/* Im2Col 3x3/p1/s1 (kernels/ref/im2col.mk). */
void hfo_im2col(const float* x, int NC, int H, int W, float* col) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (int64_t)NC * 9; ++r) {
    int nc = (int)(r / 9), k = (int)(r % 9);
    int kh = k / 3, kw = k % 3;
    for (int h = 0; h < H; ++h)
      for (int w = 0; w < W; ++w) {
        int ih = h + kh - 1, iw = w + kw - 1;
        float v = 0.0f;
        if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = x[((int64_t)nc * H + ih) * W + iw];
        col[(r * H + h) * W + w] = v;
      }
  }
}

int hfo_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
