// gen/asrgen_dev.cu — device (sm_100a) build of the seeded input generator (see asrgen.h).
// TEST/BENCH INFRASTRUCTURE: holds none of the method's arithmetic.  Used by bench.py and the
// GPU tests to create inputs directly in HBM; bit-identical to asrgen_host.c.
// dtype: 0 = bf16 bits, 1 = float32.
#include <cuda_runtime.h>
#include "asrgen.h"

namespace {

__device__ __forceinline__ void put(void* out, long idx, int dtype, float v) {
  if (dtype == 0) reinterpret_cast<uint16_t*>(out)[idx] = asrgen_bf16_bits(v);
  else reinterpret_cast<float*>(out)[idx] = v;
}

// One thread per (b, t, l, kv head) row.  out [B][npos][L][Hkv][d] (row_stride_tokens = npos).
__global__ void kv_kernel(asrgen_params p, int B, const int* pos0_dev, int pos0, int npos,
                          void* k_out, void* v_out, int dtype) {
  const long rows = (long)B * npos * p.L * p.Hkv;
  const long r = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int h = (int)(r % p.Hkv);
  const int l = (int)((r / p.Hkv) % p.L);
  const int t = (int)((r / ((long)p.Hkv * p.L)) % npos);
  const int b = (int)(r / ((long)p.Hkv * p.L * npos));
  const int pos = (pos0_dev ? pos0_dev[b] : pos0) + t;
  const long base = r * p.d;
  float row[512];
  if (k_out) {
    asrgen_k_row(&p, b, l, pos, h, row);
    for (int i = 0; i < p.d; ++i) put(k_out, base + i, dtype, row[i]);
  }
  if (v_out)
    for (int i = 0; i < p.d; ++i) put(v_out, base + i, dtype, asrgen_v(&p, b, l, pos, h, i));
}

// One thread per element: out [B][L][Hq][d] for decode step `step`.
__global__ void q_kernel(asrgen_params p, int B, int step, void* out, int dtype) {
  const long n = (long)B * p.L * p.Hq * p.d;
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int i = (int)(e % p.d);
  const int h = (int)((e / p.d) % p.Hq);
  const int l = (int)((e / ((long)p.d * p.Hq)) % p.L);
  const int b = (int)(e / ((long)p.d * p.Hq * p.L));
  put(out, e, dtype, asrgen_q(&p, b, step, l, h, i));
}

// One thread per element: out [B][vocab] for decode step `step`.
__global__ void logits_kernel(asrgen_params p, int B, int step, void* out, int dtype) {
  const long n = (long)B * p.vocab;
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int v = (int)(e % p.vocab);
  const int b = (int)(e / p.vocab);
  put(out, e, dtype, asrgen_logit(&p, b, step, v));
}

inline unsigned nblk(long n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

extern "C" {

// K/V for B sequences, positions pos0(+pos0_dev[b]) .. +npos: out [B][npos][L][Hkv][d].
int asrgen_dev_kv(const asrgen_params* p, int B, const int* pos0_dev, int pos0, int npos, void* k_out,
                  void* v_out, int dtype, void* stream) {
  if (p->d > 512) return 1;
  long rows = (long)B * npos * p->L * p->Hkv;
  if (rows == 0) return 0;
  kv_kernel<<<nblk(rows, 128), 128, 0, (cudaStream_t)stream>>>(*p, B, pos0_dev, pos0, npos, k_out, v_out,
                                                              dtype);
  return (int)cudaGetLastError();
}

int asrgen_dev_q(const asrgen_params* p, int B, int step, void* out, int dtype, void* stream) {
  long n = (long)B * p->L * p->Hq * p->d;
  if (n == 0) return 0;
  q_kernel<<<nblk(n, 256), 256, 0, (cudaStream_t)stream>>>(*p, B, step, out, dtype);
  return (int)cudaGetLastError();
}

int asrgen_dev_logits(const asrgen_params* p, int B, int step, void* out, int dtype, void* stream) {
  long n = (long)B * p->vocab;
  if (n == 0) return 0;
  logits_kernel<<<nblk(n, 256), 256, 0, (cudaStream_t)stream>>>(*p, B, step, out, dtype);
  return (int)cudaGetLastError();
}

}  // extern "C"
