/* gen/asrgen.h — seeded, counter-based synthetic input generator (LAT / GAUSS families).
 *
 * TEST/BENCH INFRASTRUCTURE.  This module holds NONE of the method's arithmetic: no
 * score, threshold, schedule, softmax, entropy or ledger logic lives here.  It only
 * turns (seed, tensor id, sequence, layer, position, head, coordinate) into exact
 * bf16-representable values.  It is the one module that BOTH the oracle side
 * (tests, via the host library asrgen_host.c) and the CUDA side (bench / GPU tests,
 * via asrgen_dev.cu) may use; the two compile this same header, and everything up
 * to the final power-of-two scaling is integer arithmetic, so both produce
 * bit-identical values (checked by tests/test_gen_gpu.py).
 *
 * Spec (restated in DESIGN.md §"Input recipe"; shapes follow SURVEY.md §8(d)):
 *   mix(x)   = splitmix64 finalizer;  h(ctr) = mix(mix(seed) ^ ctr)
 *   ctr      = tensor<<56 | b<<44 | l<<37 | pos<<17 | head<<9 | idx
 *              (tensor 8b, b 12b, l 7b, pos 20b, head 8b, idx 9b)
 *   logits   : ctr = T_LOGIT<<56 | b<<44 | step<<20 | v   (step 24b, v 20b)
 *   gauss(h) = ((h&255)+(h>>8&255)+(h>>16&255)+(h>>24&255) - 510) / 128, rounded to bf16 (RNE)
 *   LAT Q    : q[0] = 7/16; q[1] = 7/16 on needle-query steps else 0; q[i>=2] = ((h%15)-7)/16
 *   LAT K    : k[0] = a_hot if hot(b,pos) else 0; k[1] = 128 if (b,pos) is the needle else 0;
 *              m = min(16, d-2) coordinates >= 2 chosen by rejection sampling on
 *              h(T_KSUP, b,l,pos,head, attempt) % (d-2), each set to +-1/16 (sign = bit 32)
 *              => ||k_cold||_1 <= 1, |q.k_cold| <= 7/16 for every (l, head)
 *   hot(b,pos)= h(T_HOT, b,0,pos,0,0) % 1000 < hot_permille
 *   V        : gauss(h(T_V, b,l,pos,head,i))            (both families)
 *   GAUSS Q/K: gauss(h(T_GQ|T_GK, ...))                 (attention-accuracy stress; no guard band)
 *   logits   : spike step  -> gauss(h)/16 for every v (near-uniform, H ~ ln V)
 *              other steps -> gauss(h), except v = peak(b,step) = h(T_PEAK,b,0,step,0,0) % V,
 *                             which is (peak_base16 + (step%8)*peak_step16)/16
 */
#ifndef ASRGEN_H
#define ASRGEN_H
#include <stdint.h>

#ifdef __CUDACC__
#define ASRGEN_HD __host__ __device__ __forceinline__
#else
#define ASRGEN_HD static inline
#include <string.h>
#endif

enum {
  ASRGEN_T_Q = 1, ASRGEN_T_KSUP = 2, ASRGEN_T_V = 3, ASRGEN_T_HOT = 4,
  ASRGEN_T_LOGIT = 5, ASRGEN_T_PEAK = 6, ASRGEN_T_GQ = 7, ASRGEN_T_GK = 8
};
enum { ASRGEN_LAT = 0, ASRGEN_GAUSS = 1 };

typedef struct {
  uint64_t seed;
  int32_t family;        /* ASRGEN_LAT | ASRGEN_GAUSS */
  int32_t L, Hq, Hkv, d; /* model shape */
  int32_t hot_permille;  /* LAT: fraction of hot tokens x1000 (0 = all-cold trace W0) */
  int32_t a_hot;         /* LAT: hot coordinate value k[0] (4 or 64) */
  int32_t needle_pos;    /* LAT: position of the needle token, -1 = none */
  int32_t needle_b;      /* sequence holding the needle, -1 = every sequence */
  int32_t query_first;   /* needle retrieval steps [query_first, query_first+query_count) */
  int32_t query_count;
  int32_t vocab;         /* logits row length */
  int32_t spike_first;   /* entropy spikes at steps spike_first + k*spike_period, k < spike_count */
  int32_t spike_period;
  int32_t spike_count;
  int32_t peak_base16;   /* baseline peak logit = (peak_base16 + (step%8)*peak_step16)/16 */
  int32_t peak_step16;
} asrgen_params;

ASRGEN_HD uint64_t asrgen_mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

ASRGEN_HD uint64_t asrgen_ctr(uint32_t t, uint32_t b, uint32_t l, uint32_t pos, uint32_t head,
                              uint32_t idx) {
  return ((uint64_t)t << 56) | ((uint64_t)b << 44) | ((uint64_t)l << 37) | ((uint64_t)pos << 17) |
         ((uint64_t)head << 9) | (uint64_t)idx;
}

ASRGEN_HD uint64_t asrgen_hash(const asrgen_params* p, uint64_t ctr) {
  return asrgen_mix(asrgen_mix(p->seed) ^ ctr);
}

ASRGEN_HD uint32_t asrgen_f2u(float f) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
#endif
}
ASRGEN_HD float asrgen_u2f(uint32_t u) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}

/* float -> bf16 bits, round to nearest even (inputs here are finite). */
ASRGEN_HD uint16_t asrgen_bf16_bits(float f) {
  uint32_t u = asrgen_f2u(f);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
ASRGEN_HD float asrgen_bf16_to_f(uint16_t b) { return asrgen_u2f(((uint32_t)b) << 16); }

/* Integer approximation of a normal (sum of 4 bytes), /128, rounded to bf16. */
ASRGEN_HD float asrgen_gauss(uint64_t h) {
  int32_t g = (int32_t)(h & 255u) + (int32_t)((h >> 8) & 255u) + (int32_t)((h >> 16) & 255u) +
              (int32_t)((h >> 24) & 255u) - 510;
  return asrgen_bf16_to_f(asrgen_bf16_bits((float)g * (1.0f / 128.0f)));
}

ASRGEN_HD int asrgen_is_hot(const asrgen_params* p, int b, int pos) {
  if (p->hot_permille <= 0) return 0;
  uint64_t h = asrgen_hash(p, asrgen_ctr(ASRGEN_T_HOT, (uint32_t)b, 0, (uint32_t)pos, 0, 0));
  return (int)(h % 1000u) < p->hot_permille;
}
ASRGEN_HD int asrgen_is_needle(const asrgen_params* p, int b, int pos) {
  return p->needle_pos >= 0 && pos == p->needle_pos && (p->needle_b < 0 || p->needle_b == b);
}
ASRGEN_HD int asrgen_is_query_step(const asrgen_params* p, int step) {
  return step >= p->query_first && step < p->query_first + p->query_count;
}
ASRGEN_HD int asrgen_is_spike_step(const asrgen_params* p, int step) {
  if (p->spike_count <= 0 || step < p->spike_first) return 0;
  int k = p->spike_period > 0 ? (step - p->spike_first) / p->spike_period : 0;
  if (k >= p->spike_count) return 0;
  return step == p->spike_first + k * (p->spike_period > 0 ? p->spike_period : 0);
}

/* Q element for sequence b at decode step `step`, layer l, query head h, coordinate i. */
ASRGEN_HD float asrgen_q(const asrgen_params* p, int b, int step, int l, int h, int i) {
  uint32_t t = p->family == ASRGEN_GAUSS ? ASRGEN_T_GQ : ASRGEN_T_Q;
  uint64_t x = asrgen_hash(p, asrgen_ctr(t, (uint32_t)b, (uint32_t)l, (uint32_t)step, (uint32_t)h,
                                         (uint32_t)i));
  if (p->family == ASRGEN_GAUSS) return asrgen_gauss(x);
  if (i == 0) return 7.0f / 16.0f;
  if (i == 1) return asrgen_is_query_step(p, step) ? 7.0f / 16.0f : 0.0f;
  return (float)((int32_t)(x % 15u) - 7) * (1.0f / 16.0f);
}

/* One K row (d values) for (b, l, pos, kv head). */
ASRGEN_HD void asrgen_k_row(const asrgen_params* p, int b, int l, int pos, int hk, float* out) {
  const int d = p->d;
  if (p->family == ASRGEN_GAUSS) {
    for (int i = 0; i < d; ++i)
      out[i] = asrgen_gauss(asrgen_hash(
          p, asrgen_ctr(ASRGEN_T_GK, (uint32_t)b, (uint32_t)l, (uint32_t)pos, (uint32_t)hk, (uint32_t)i)));
    return;
  }
  for (int i = 0; i < d; ++i) out[i] = 0.0f;
  if (d > 0 && asrgen_is_hot(p, b, pos)) out[0] = (float)p->a_hot;
  if (d > 1 && asrgen_is_needle(p, b, pos)) out[1] = 128.0f;
  if (d <= 2) return;
  const int span = d - 2;
  const int m = span < 16 ? span : 16;
  int chosen[16];
  int cnt = 0;
  for (int a = 0; a < 511 && cnt < m; ++a) {
    uint64_t x = asrgen_hash(
        p, asrgen_ctr(ASRGEN_T_KSUP, (uint32_t)b, (uint32_t)l, (uint32_t)pos, (uint32_t)hk, (uint32_t)a));
    int c = 2 + (int)(x % (uint64_t)span);
    int dup = 0;
    for (int t = 0; t < cnt; ++t) dup |= (chosen[t] == c);
    if (dup) continue;
    chosen[cnt++] = c;
    out[c] = ((x >> 32) & 1u) ? -1.0f / 16.0f : 1.0f / 16.0f;
  }
  /* deterministic completion (never reached for d >= 16 in practice) */
  for (int c = 2; c < d && cnt < m; ++c) {
    int dup = 0;
    for (int t = 0; t < cnt; ++t) dup |= (chosen[t] == c);
    if (!dup) { chosen[cnt++] = c; out[c] = 1.0f / 16.0f; }
  }
}

ASRGEN_HD float asrgen_v(const asrgen_params* p, int b, int l, int pos, int hk, int i) {
  return asrgen_gauss(asrgen_hash(
      p, asrgen_ctr(ASRGEN_T_V, (uint32_t)b, (uint32_t)l, (uint32_t)pos, (uint32_t)hk, (uint32_t)i)));
}

ASRGEN_HD int asrgen_peak_index(const asrgen_params* p, int b, int step) {
  uint64_t x = asrgen_hash(p, asrgen_ctr(ASRGEN_T_PEAK, (uint32_t)b, 0, (uint32_t)step, 0, 0));
  return (int)(x % (uint64_t)p->vocab);
}

/* Logit v of the row produced at decode step `step` for sequence b. */
ASRGEN_HD float asrgen_logit(const asrgen_params* p, int b, int step, int v) {
  uint64_t ctr = ((uint64_t)ASRGEN_T_LOGIT << 56) | ((uint64_t)(uint32_t)b << 44) |
                 ((uint64_t)(uint32_t)step << 20) | (uint64_t)(uint32_t)v;
  float g = asrgen_gauss(asrgen_hash(p, ctr));
  if (asrgen_is_spike_step(p, step)) return g * (1.0f / 16.0f);
  if (v == asrgen_peak_index(p, b, step))
    return (float)(p->peak_base16 + (step % 8) * p->peak_step16) * (1.0f / 16.0f);
  return g;
}

#endif /* ASRGEN_H */
