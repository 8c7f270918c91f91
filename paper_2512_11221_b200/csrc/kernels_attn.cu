// paper_2512_11221_b200/csrc/kernels_attn.cu — (a4) split-KV decode attention over the active
// index list A_i with the Eq. 2 relevance score fused into the QK^T pass, and (a4') the
// fixed-order combine of the split partials.
//
//   O_{l,h} = softmax(q_{l,h} K_{A,l,g(h)}^T / sqrt(d)) V_{A,l,g(h)}     Eq. 1, Alg. 1 line 1
//   part_{l}(a) = sum_h |q_{l,h} . k_{l,A[a],g(h)}|                      Eq. 2, Alg. 1 line 2
//
// This file holds the generic CUDA-core kernel (any head_dim in {16..256}, bf16 or fp32 KV):
// one CTA per work item (b, l, chunk of A_b), one warp per KV head, persistent grid-stride over
// the ragged work list (no host sync: the list is derived on the device from |A_b|).
// The bf16 / LLaMA-shape fast path lives in kernels_attn_mma.cu; the combine of the split
// partials runs in post_kernel (kernels_ledger.cu).
#include <cuda_bf16.h>
#include <math.h>

#include "asr_internal.h"

namespace asr {
namespace {

template <typename T>
struct Vec;  // EPL consecutive elements of T loaded as one vector
template <>
struct Vec<float> {
  template <int N>
  __device__ static void load(const float* p, float* out) {
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = p[i];
  }
};
template <>
struct Vec<__nv_bfloat16> {
  template <int N>
  __device__ static void load(const __nv_bfloat16* p, float* out) {
    if constexpr (N % 2 == 0) {
#pragma unroll
      for (int i = 0; i < N; i += 2) {
        __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(p + i);
        out[i] = __low2float(v);
        out[i + 1] = __high2float(v);
      }
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) out[i] = __bfloat162float(p[i]);
    }
  }
};

// Work-list prologue shared by every CTA: item_start[b] = sum_{b'<b} L * nch(b').
__device__ int build_items(const DevState& s, const int* alen, int* sh_start) {
  // B <= 4096 sequences: serial scan by thread 0 is fine (a few microseconds at most once per CTA)
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int b = 0; b < s.B; ++b) {
      sh_start[b] = acc;
      int chunk, nch;
      chunking(alen[b], s.max_splits, s.chunk_min, &chunk, &nch);
      acc += s.L * nch;
    }
    sh_start[s.B] = acc;
    if (blockIdx.x == 0)
      for (int b = 0; b <= s.B; ++b) s.item_start[b] = sh_start[b];
  }
  __syncthreads();
  return sh_start[s.B];
}

__device__ __forceinline__ int find_seq(const int* start, int B, int item) {
  int lo = 0, hi = B - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= item) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

constexpr int kMaxG = 8;  // query heads per KV head supported by the generic kernel

template <typename T, int D>
__global__ void attn_generic_kernel(DevState s, const T* __restrict__ q) {
  extern __shared__ int smem_i[];
  int* sh_start = smem_i;                                          // [B+1]
  float* sc = reinterpret_cast<float*>(smem_i + s.B + 1);          // [Hkv][32]
  constexpr int EPL = D >= 32 ? D / 32 : 1;
  constexpr int ACT = D >= 32 ? 32 : D;
  pdl_wait();
  pdl_trigger();
  Stamp stamp(s.tl, 1);
  const int p = *s.step & 1;   // A_i lists of this step
  const int* alen = s.act_len + p * s.B;
  const int total = build_items(s, alen, sh_start);
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = s.Hq / s.Hkv;
  const bool lane_on = lane < ACT;
  const float scale = 1.4426950408889634f / sqrtf((float)D);  // log2(e)/sqrt(d)
  const long row = (long)s.Hkv * D;                              // K (or V) elements per token-layer
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    const int b = find_seq(sh_start, s.B, item);
    const int A = alen[b];
    int chunk, nch;
    chunking(A, s.max_splits, s.chunk_min, &chunk, &nch);
    const int r = item - sh_start[b];
    const int l = r / nch, c = r % nch;
    const int a0 = c * chunk, a1 = min(A, a0 + chunk);
    const int* act = s.act_slot + act_off(s, p) + (long)b * s.max_ctx;   // device slots of A_i
    // q slice of the G heads of this warp's KV head
    float qr[kMaxG][EPL];
    float m[kMaxG], lsum[kMaxG], acc[kMaxG][EPL];
#pragma unroll
    for (int hh = 0; hh < kMaxG; ++hh) {
      m[hh] = -INFINITY;
      lsum[hh] = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; ++e) { acc[hh][e] = 0.f; qr[hh][e] = 0.f; }
      if (hh < G && lane_on)
        Vec<T>::template load<EPL>(q + (((long)b * s.L + l) * s.Hq + g * G + hh) * D + lane * EPL, qr[hh]);
    }
    for (int t0 = a0; t0 < a1; t0 += 32) {
      const int tn = min(32, a1 - t0);
      for (int tt = 0; tt < tn; ++tt) {
        const long slot = max(0, act[t0 + tt]);
        const T* kp = reinterpret_cast<const T*>(s.kv) + (slot * s.L + l) * 2 * row + (long)g * D;
        const T* vp = kp + row;
        float kr[EPL], vr[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) { kr[e] = 0.f; vr[e] = 0.f; }
        if (lane_on) {
          Vec<T>::template load<EPL>(kp + lane * EPL, kr);
          Vec<T>::template load<EPL>(vp + lane * EPL, vr);
        }
        float sabs = 0.f;
#pragma unroll
        for (int hh = 0; hh < kMaxG; ++hh) {
          if (hh >= G) break;
          float dot = 0.f;
#pragma unroll
          for (int e = 0; e < EPL; ++e) dot = fmaf(qr[hh][e], kr[e], dot);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
          sabs += fabsf(dot);
          const float x = dot * scale;
          const float mn = fmaxf(m[hh], x);
          const float corr = exp2f(m[hh] - mn);
          const float p = exp2f(x - mn);
          lsum[hh] = lsum[hh] * corr + p;
#pragma unroll
          for (int e = 0; e < EPL; ++e) acc[hh][e] = fmaf(p, vr[e], acc[hh][e] * corr);
          m[hh] = mn;
        }
        if (lane == 0) sc[g * 32 + tt] = sabs;
      }
      __syncthreads();
      if ((int)threadIdx.x < tn) {  // fixed-order sum over the KV heads -> one partial per token
        float t = 0.f;
        for (int gg = 0; gg < s.Hkv; ++gg) t += sc[gg * 32 + threadIdx.x];
        s.score_part[((long)b * s.L + l) * s.max_ctx + t0 + threadIdx.x] = t;
      }
      __syncthreads();
    }
#pragma unroll
    for (int hh = 0; hh < kMaxG; ++hh) {
      if (hh >= G) break;
      const long pi = (long)item * s.Hq + g * G + hh;
      if (lane == 0) {
        s.part_ml[pi * 2] = m[hh];
        s.part_ml[pi * 2 + 1] = lsum[hh];
      }
      if (lane_on)
#pragma unroll
        for (int e = 0; e < EPL; ++e) s.part_acc[pi * D + lane * EPL + e] = acc[hh][e];
    }
  }
  if (s.pool_mode) {   // the attention's end, against which the prefetch copies are timed
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&s.stall[1], gtimer());
  }
}

template <typename T>
const void* generic_func(int d) {
  switch (d) {
    case 16: return (const void*)attn_generic_kernel<T, 16>;
    case 32: return (const void*)attn_generic_kernel<T, 32>;
    case 64: return (const void*)attn_generic_kernel<T, 64>;
    case 128: return (const void*)attn_generic_kernel<T, 128>;
    default: return (const void*)attn_generic_kernel<T, 256>;
  }
}

}  // namespace

int attention_grid(const DevState& s, int num_sms) {
  if (attention_mma_supported(s)) return num_sms;  // persistent: one CTA per SM
  long max_items = (long)s.B * s.L * s.max_splits;
  long g = (long)num_sms * 4;
  return (int)(max_items < g ? max_items : g);
}

void node_attention(KNode& n, const DevState& s, const void* q, const void* k_new, const void* v_new, int grid,
                    const void* pre_logits, int logits_dtype, float* entropy_out, float* o) {
  n.s = s;
  n.set(0, q);
  if (attention_mma_supported(s)) {
    n.set(1, k_new);
    n.set(2, v_new);
    n.set(3, pre_logits);
    n.set(4, entropy_out);
    n.set(5, o);
    const void* f;
    int threads;
    unsigned smem;
    attention_mma_launch_shape(s, pre_logits && logits_dtype == 1, &f, &threads, &smem);
    n.finalize(f, dim3(grid), dim3(threads), smem);
    return;
  }
  const unsigned smem = (unsigned)(sizeof(int) * (s.B + 1) + sizeof(float) * 32 * s.Hkv);
  const void* f = s.dtype == 0 ? generic_func<__nv_bfloat16>(s.d) : generic_func<float>(s.d);
  n.finalize(f, dim3(grid), dim3(32 * s.Hkv), smem);
}

}  // namespace asr
