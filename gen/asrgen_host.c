/* gen/asrgen_host.c — host (CPU) build of the seeded input generator (see asrgen.h).
 * TEST/BENCH INFRASTRUCTURE: holds none of the method's arithmetic.
 * dtype: 0 = bf16 bits (uint16_t), 1 = float32.  Layouts are row-major as documented. */
#include <stdlib.h>
#include "asrgen.h"

static void put(void* out, long idx, int dtype, float v) {
  if (dtype == 0) ((uint16_t*)out)[idx] = asrgen_bf16_bits(v);
  else ((float*)out)[idx] = v;
}

/* K and V rows for sequence b, positions [pos0, pos0+npos): out [npos][L][Hkv][d]. */
void asrgen_host_kv(const asrgen_params* p, int b, int pos0, int npos, void* k_out, void* v_out,
                    int dtype) {
  const int L = p->L, Hk = p->Hkv, d = p->d;
  float* row = (float*)malloc(sizeof(float) * (size_t)d);
  for (int t = 0; t < npos; ++t)
    for (int l = 0; l < L; ++l)
      for (int h = 0; h < Hk; ++h) {
        long base = (((long)t * L + l) * Hk + h) * d;
        if (k_out) {
          asrgen_k_row(p, b, l, pos0 + t, h, row);
          for (int i = 0; i < d; ++i) put(k_out, base + i, dtype, row[i]);
        }
        if (v_out)
          for (int i = 0; i < d; ++i) put(v_out, base + i, dtype, asrgen_v(p, b, l, pos0 + t, h, i));
      }
  free(row);
}

/* Query for sequence b at decode step `step`: out [L][Hq][d]. */
void asrgen_host_q(const asrgen_params* p, int b, int step, void* out, int dtype) {
  const int L = p->L, Hq = p->Hq, d = p->d;
  for (int l = 0; l < L; ++l)
    for (int h = 0; h < Hq; ++h)
      for (int i = 0; i < d; ++i)
        put(out, ((long)l * Hq + h) * d + i, dtype, asrgen_q(p, b, step, l, h, i));
}

/* Logits row of sequence b at decode step `step`: out [vocab]. */
void asrgen_host_logits(const asrgen_params* p, int b, int step, void* out, int dtype) {
  for (int v = 0; v < p->vocab; ++v) put(out, v, dtype, asrgen_logit(p, b, step, v));
}

int asrgen_host_is_hot(const asrgen_params* p, int b, int pos) { return asrgen_is_hot(p, b, pos); }
int asrgen_host_is_needle(const asrgen_params* p, int b, int pos) { return asrgen_is_needle(p, b, pos); }
int asrgen_host_is_query_step(const asrgen_params* p, int step) { return asrgen_is_query_step(p, step); }
int asrgen_host_is_spike_step(const asrgen_params* p, int step) { return asrgen_is_spike_step(p, step); }
int asrgen_host_peak_index(const asrgen_params* p, int b, int step) { return asrgen_peak_index(p, b, step); }
uint64_t asrgen_host_mix(uint64_t x) { return asrgen_mix(x); }
