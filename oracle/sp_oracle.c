/*
 * sp_oracle.c — CPU oracle for the averaging round. TEST INFRASTRUCTURE ONLY
 * (see sp_oracle.h for who may call it and what pins it).
 *
 * Compiled with -ffp-contract=off: every rounding below is the one written,
 * fmaf() is used exactly where the device uses __fmaf_rn.
 */
#include "sp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

uint64_t sp_oracle_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

void sp_oracle_fill_synthetic(float* out, int64_t n, uint64_t seed, int peer,
                              float scale, int64_t every, float mult) {
  const uint64_t key = seed ^ ((uint64_t)peer << 40);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t u = sp_oracle_splitmix64(key ^ (uint64_t)i) >> 40;
    float x = ((float)(int64_t)u - 8388608.0f) * (1.0f / 8388608.0f);
    x = x * scale;
    if (every > 0 && i % every == 0) x = x * mult;
    out[i] = x;
  }
}

void sp_oracle_part_offsets(int64_t n, int G, const double* fractions,
                            int64_t align, int64_t* offsets) {
  double cum = 0.0;
  offsets[0] = 0;
  for (int k = 1; k < G; ++k) {
    cum += fractions[k - 1];
    int64_t o = align * llround((double)n * cum / (double)align);
    if (o < offsets[k - 1]) o = offsets[k - 1];
    if (o > n) o = n;
    offsets[k] = o;
  }
  offsets[G] = n;
}

uint16_t sp_oracle_f2h(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t ax = x & 0x7fffffffu;
  if (ax >= 0x7f800000u) /* inf / nan */
    return (uint16_t)(sign | 0x7c00u | (ax > 0x7f800000u ? (0x200u | ((ax >> 13) & 0x3ffu)) : 0u));
  if (ax >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u); /* >= 65520 -> inf */
  if (ax < 0x38800000u) {                                    /* half subnormal */
    if (ax < 0x33000000u) return (uint16_t)sign;             /* < 2^-25 -> 0 */
    const uint32_t e = ax >> 23;
    const uint32_t mant = (ax & 0x7fffffu) | 0x800000u;
    const int shift = 126 - (int)e; /* 14..24 */
    uint32_t q = mant >> shift;
    const uint32_t rem = mant & ((1u << shift) - 1u), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (q & 1u))) ++q;
    return (uint16_t)(sign | q);
  }
  const uint32_t e = (ax >> 23) - 127u + 15u;
  const uint32_t mant = ax & 0x7fffffu;
  uint32_t q = (e << 10) | (mant >> 13);
  const uint32_t rem = mant & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (q & 1u))) ++q;
  return (uint16_t)(sign | q);
}

float sp_oracle_h2f(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1fu, mant = h & 0x3ffu;
  uint32_t x;
  if (e == 0) {
    if (mant == 0) {
      x = sign;
    } else { /* subnormal: mant * 2^-24, exact in fp32 */
      float f = (float)mant * (1.0f / 16777216.0f);
      memcpy(&x, &f, 4);
      x |= sign;
    }
  } else if (e == 31) {
    x = sign | 0x7f800000u | (mant << 13);
  } else {
    x = sign | ((e - 15u + 127u) << 23) | (mant << 13);
  }
  float f;
  memcpy(&f, &x, 4);
  return f;
}

void sp_oracle_pack_fp16(const float* x, uint16_t* out, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = sp_oracle_f2h(x[i]);
}

static inline int q8_code(float x, float inv) {
  float t = rintf(x * inv); /* x*inv rounded once, then RNE to integer */
  if (t > 127.0f) t = 127.0f;
  if (t < -127.0f) t = -127.0f;
  return (int)t;
}

static void quantize_block(const float* x, int64_t len, int8_t* codes, float* scale) {
  float amax = 0.0f;
  for (int64_t j = 0; j < len; ++j) {
    const float a = fabsf(x[j]);
    amax = a > amax ? a : amax;
  }
  const float inv = amax > 0.0f ? 127.0f / amax : 0.0f;
  for (int64_t j = 0; j < len; ++j) codes[j] = (int8_t)q8_code(x[j], inv);
  *scale = amax / 127.0f;
}

void sp_oracle_pack_q8(const float* x, int8_t* codes, float* scales, int64_t n, int block) {
  const int64_t nb = (n + block - 1) / block;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t s = b * block;
    const int64_t len = (n - s) < block ? (n - s) : block;
    quantize_block(x + s, len, codes + s, scales + b);
  }
}

void sp_oracle_weighted_average_f64(const double* const* values, const double* weights,
                                    int G, int64_t n, double* out) {
  double wsum = 0.0;
  for (int g = 0; g < G; ++g) wsum += weights ? weights[g] : 1.0;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += values[g][i] * (weights ? weights[g] : 1.0);
    out[i] = s / wsum;
  }
}

static inline float dequant(int wire, const void* buf, const float* scales, int block, int64_t i) {
  if (wire == SPO_FP32) return ((const float*)buf)[i];
  if (wire == SPO_FP16) return sp_oracle_h2f(((const uint16_t*)buf)[i]);
  return (float)((const int8_t*)buf)[i] * scales[i / block];
}

static void normalized_weights(const double* w, int G, float* wn, int* idx, int* np) {
  double s = 0.0;
  for (int g = 0; g < G; ++g) s += w[g];
  *np = 0;
  for (int g = 0; g < G; ++g) {
    if (w[g] == 0.0) continue;
    wn[*np] = (float)(w[g] / s);
    idx[*np] = g;
    ++*np;
  }
}

void sp_oracle_reduce(int wire, const void* const* wires, const float* const* scales,
                      const double* weights, int G, int64_t lo, int64_t hi, int block,
                      void* out_wire, float* out_scales) {
  float wn[64];
  int idx[64], np = 0;
  normalized_weights(weights, G, wn, idx, &np);
  if (wire != SPO_Q8) {
#pragma omp parallel for schedule(static)
    for (int64_t i = lo; i < hi; ++i) {
      /* first contributor by product (no +0 seed), then fmaf in peer order */
      float acc = wn[0] * dequant(wire, wires[idx[0]], NULL, block, i);
      for (int k = 1; k < np; ++k)
        acc = fmaf(wn[k], dequant(wire, wires[idx[k]], NULL, block, i), acc);
      if (wire == SPO_FP32)
        ((float*)out_wire)[i] = acc;
      else
        ((uint16_t*)out_wire)[i] = sp_oracle_f2h(acc);
    }
    return;
  }
  const int64_t b0 = lo / block, b1 = (hi + block - 1) / block;
  if (np == 1) { /* one contributor (weight 1): its codes and scales, unchanged */
    const int g = idx[0];
    memcpy((int8_t*)out_wire + lo, (const int8_t*)wires[g] + lo, (size_t)(hi - lo));
    for (int64_t b = b0; b < b1; ++b) out_scales[b] = scales[g][b];
    return;
  }
#pragma omp parallel
  {
    float* tmp = (float*)malloc(sizeof(float) * (size_t)block);
#pragma omp for schedule(static)
    for (int64_t b = b0; b < b1; ++b) {
      const int64_t s = b * block;
      const int64_t e = (s + block) < hi ? (s + block) : hi;
      for (int64_t i = s; i < e; ++i) {
        float acc = wn[0] * ((float)((const int8_t*)wires[idx[0]])[i] * scales[idx[0]][b]);
        for (int k = 1; k < np; ++k) {
          const int g = idx[k];
          const float x = (float)((const int8_t*)wires[g])[i] * scales[g][b];
          acc = fmaf(wn[k], x, acc);
        }
        tmp[i - s] = acc;
      }
      quantize_block(tmp, e - s, (int8_t*)out_wire + s, out_scales + b);
    }
    free(tmp);
  }
}

typedef struct {
  float b1, b2, omb1, omb2, eps, wd, ibc1, ibc2;
} lamb_k;

static inline float lamb_dir(const lamb_k* k, float p, float m, float v) {
  const float den = sqrtf(v * k->ibc2) + k->eps;
  return fmaf(k->wd, p, (m * k->ibc1) / den);
}

#define SPO_CHUNK 65536

void sp_oracle_lamb(int wire, const void* avg, const float* avg_scales, int block, float* p,
                    float* m, float* v, int64_t n, const int64_t* tsizes, int T,
                    const sp_oracle_lamb_hp* hp, int step, const float* trust_in,
                    float* trust_out) {
  lamb_k k;
  k.b1 = hp->beta1;
  k.b2 = hp->beta2;
  k.omb1 = 1.0f - hp->beta1;
  k.omb2 = 1.0f - hp->beta2;
  k.eps = hp->eps;
  k.wd = hp->weight_decay;
  if (hp->bias_correction) {
    k.ibc1 = (float)(1.0 / (1.0 - pow((double)hp->beta1, step)));
    k.ibc2 = (float)(1.0 / (1.0 - pow((double)hp->beta2, step)));
  } else {
    k.ibc1 = k.ibc2 = 1.0f;
  }
  (void)n;
  int64_t off = 0;
  for (int t = 0; t < T; ++t) {
    const int64_t s = off, e = off + tsizes[t];
    const int64_t nch = (tsizes[t] + SPO_CHUNK - 1) / SPO_CHUNK;
    double* part = (double*)calloc((size_t)(2 * nch), sizeof(double));
    /* pass 1: moments + fp64 norm partials per fixed chunk (deterministic
     * for any thread count) */
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nch; ++c) {
      const int64_t cs = s + c * SPO_CHUNK;
      const int64_t ce = (cs + SPO_CHUNK) < e ? (cs + SPO_CHUNK) : e;
      double pp = 0.0, uu = 0.0;
      for (int64_t i = cs; i < ce; ++i) {
        const float g = dequant(wire, avg, avg_scales, block, i);
        const float mi = fmaf(k.b1, m[i], k.omb1 * g);
        const float vi = fmaf(k.b2, v[i], k.omb2 * (g * g));
        m[i] = mi;
        v[i] = vi;
        const float u = lamb_dir(&k, p[i], mi, vi);
        pp += (double)p[i] * (double)p[i];
        uu += (double)u * (double)u;
      }
      part[2 * c] = pp;
      part[2 * c + 1] = uu;
    }
    double pp = 0.0, uu = 0.0;
    for (int64_t c = 0; c < nch; ++c) {
      pp += part[2 * c];
      uu += part[2 * c + 1];
    }
    free(part);
    const double r1 = sqrt(pp), r2 = sqrt(uu);
    float trust = (r1 > 0.0 && r2 > 0.0) ? (float)(r1 / r2) : 1.0f;
    if (trust_out) trust_out[t] = trust;
    if (trust_in) trust = trust_in[t];
    const float neg = -(hp->lr * trust);
    /* pass 2: update */
#pragma omp parallel for schedule(static)
    for (int64_t i = s; i < e; ++i) p[i] = fmaf(neg, lamb_dir(&k, p[i], m[i], v[i]), p[i]);
    off = e;
  }
}

int sp_oracle_round(int wire, int block, int G, int64_t n, const float* const* grads,
                    const double* weights, float* p, float* m, float* v,
                    const int64_t* tsizes, int T, const sp_oracle_lamb_hp* hp, int step,
                    int threads, float* trust_out) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  const int64_t nb = (n + block - 1) / block;
  const size_t wbytes = wire == SPO_FP32 ? 4 : wire == SPO_FP16 ? 2 : 1;
  void* wires[64] = {0};
  float* scales[64] = {0};
  for (int g = 0; g < G; ++g) {
    if (weights[g] == 0.0) continue;
    if (wire == SPO_FP32) {
      wires[g] = (void*)grads[g]; /* zero-copy, as on the device */
      continue;
    }
    wires[g] = malloc(wbytes * (size_t)n);
    if (wire == SPO_FP16) {
      sp_oracle_pack_fp16(grads[g], (uint16_t*)wires[g], n);
    } else {
      scales[g] = (float*)malloc(sizeof(float) * (size_t)nb);
      sp_oracle_pack_q8(grads[g], (int8_t*)wires[g], scales[g], n, block);
    }
  }
  void* avg = malloc(wbytes * (size_t)n);
  float* avg_scales = wire == SPO_Q8 ? (float*)malloc(sizeof(float) * (size_t)nb) : NULL;
  sp_oracle_reduce(wire, (const void* const*)wires, (const float* const*)scales, weights, G, 0,
                   n, block, avg, avg_scales);
  sp_oracle_lamb(wire, avg, avg_scales, block, p, m, v, n, tsizes, T, hp, step, NULL,
                 trust_out);
  for (int g = 0; g < G; ++g) {
    if (wire != SPO_FP32) free(wires[g]);
    free(scales[g]);
  }
  free(avg);
  free(avg_scales);
  return 0;
}

int sp_oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void sp_oracle_set_threads(int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
}

/* fp64 values (the reference run_plan's weighted mean) rounded to fp32, then
 * to the wire format: what a reference-side aggregator would put on the
 * wire. out is float[n] (fp32), uint16[n] (fp16) or int8[n] + scales. */
void sp_oracle_wire_from_f64(int wire, const double* x, void* out, float* scales, int64_t n,
                             int block) {
  if (wire == SPO_FP32) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) ((float*)out)[i] = (float)x[i];
    return;
  }
  if (wire == SPO_FP16) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) ((uint16_t*)out)[i] = sp_oracle_f2h((float)x[i]);
    return;
  }
  const int64_t nb = (n + block - 1) / block;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    float tmp[16384];
    const int64_t s = b * block;
    const int64_t len = (n - s) < block ? (n - s) : block;
    for (int64_t j = 0; j < len; ++j) tmp[j] = (float)x[s + j];
    quantize_block(tmp, len, (int8_t*)out + s, scales + b);
  }
}
