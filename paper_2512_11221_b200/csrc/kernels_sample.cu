// paper_2512_11221_b200/csrc/kernels_sample.cu — NEXT-1: the next-token draw that
// closes Alg. 1 ("Generate next token"): greedy, or temperature + top-k + top-p filtering and
// one categorical draw per row with the caller's uniform u.  Rules (R-sample) are those of
// oracle/sample.py:
//   greedy (T <= 0 or k == 1): the first maximal logit;
//   kept set: the k largest logits (ties to lower indices), then the shortest prefix of them in
//   (logit desc, index asc) order holding >= P of their probability mass;
//   draw: the smallest index j in the kept set with  sum_{i kept, i <= j} p_i  >  u * sum_{kept} p_i.
//
// One CTA (1024 threads) per row.  The boundaries are found by radix selection on an order-preserving
// 32-bit key of the logit (digits of 12, 12 and 8 bits, one pass over the row each, histograms of
// counts and of fixed-point probability mass in shared memory).  Masses are exp((x - max) / T) in
// fp32, summed as 2^-36 fixed point in 64-bit integers: every sum is exact and order-independent, so
// a draw is bitwise deterministic.
#include <cuda_bf16.h>
#include <stdint.h>

#include "asr_internal.h"

namespace asr {
namespace {

constexpr int kSampleThreads = 1024;
constexpr int kBins = 4096;
constexpr double kFix = 68719476736.0;   // 2^36

__device__ __forceinline__ float lg(const __nv_bfloat16* p, int j) { return __bfloat162float(p[j]); }
__device__ __forceinline__ float lg(const float* p, int j) { return p[j]; }

// order-preserving key of a float (-0 folded onto +0)
__device__ __forceinline__ uint32_t fkey(float x) {
  uint32_t b = __float_as_uint(x == 0.f ? 0.f : x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ unsigned long long wfix(float x, float m, float invT) {
  return (unsigned long long)((double)__expf((x - m) * invT) * kFix);
}

struct SampleShm {
  uint32_t cnt[kBins];
  unsigned long long mass[kBins];
  unsigned long long wsum[32];
  uint32_t wcnt[32];
  float fred[32];
  int ired[32];
  uint32_t digit;
  unsigned long long scan_total, tie_take;
  uint32_t above_cnt;
  int token;
};

// block-wide exclusive scan (thread order) of a 64-bit value; also returns the total
__device__ unsigned long long block_excl_scan(unsigned long long v, SampleShm& sh, unsigned long long* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sh.wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    const unsigned long long x = sh.wsum[lane];
    unsigned long long xi = x;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    sh.wsum[lane] = xi - x;
  }
  __syncthreads();
  const unsigned long long res = sh.wsum[w] + incl - v;
  if (threadIdx.x == kSampleThreads - 1) sh.scan_total = res + v;
  __syncthreads();
  *total = sh.scan_total;
  __syncthreads();
  return res;
}

// Find the digit d whose bin crosses `target` counting from the top bin down: above(d) < target <=
// above(d) + bin(d), where bin = counts (by_mass false) or masses.  Sets sh.digit, sh.above_cnt,
// sh.above_mass (the totals of the bins above d).  nbins <= kBins (a power of two >= 1024... or 256).
__device__ void find_digit(SampleShm& sh, int nbins, bool by_mass, unsigned long long target) {
  const int per = nbins / kSampleThreads > 0 ? nbins / kSampleThreads : 1;
  const int active = nbins / per;
  // thread t owns bins hi_t, hi_t - 1, ..., hi_t - per + 1 with hi_t = nbins - 1 - t * per
  const int hi = nbins - 1 - (int)threadIdx.x * per;
  unsigned long long sv = 0, sc = 0;
  if ((int)threadIdx.x < active)
    for (int k = 0; k < per; ++k) {
      sv += by_mass ? sh.mass[hi - k] : sh.cnt[hi - k];
      sc += sh.cnt[hi - k];
    }
  unsigned long long tot;
  const unsigned long long before = block_excl_scan(sv, sh, &tot);
  const unsigned long long before_c = block_excl_scan(sc, sh, &tot);
  const unsigned long long before_m = by_mass ? before : 0;   // mass above, when selecting by mass
  if ((int)threadIdx.x < active && before < target && target <= before + sv) {
    unsigned long long a = before, ac = before_c;
    for (int k = 0; k < per; ++k) {
      const unsigned long long v = by_mass ? sh.mass[hi - k] : sh.cnt[hi - k];
      if (a < target && target <= a + v) {
        sh.digit = (uint32_t)(hi - k);
        sh.above_cnt = (uint32_t)ac;
        sh.tie_take = a;   // the selected quantity above the digit (count or mass)
        break;
      }
      a += v;
      ac += sh.cnt[hi - k];
    }
  }
  (void)before_m;
  __syncthreads();
}

template <typename TL>
__global__ void __launch_bounds__(kSampleThreads) sample_kernel(const TL* __restrict__ logits, int V, float temperature,
                                                                int top_k, float top_p, const float* __restrict__ uniforms,
                                                                int32_t* __restrict__ token_out) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SampleShm& sh = *reinterpret_cast<SampleShm*>(smem_raw);
  const TL* x = logits + (long)blockIdx.x * V;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  // ---- max (and its first index, for greedy)
  float mx = -INFINITY;
  int mi = 0x7fffffff;
  for (int j = tid; j < V; j += kSampleThreads) {
    const float v = lg(x, j);
    if (v > mx) { mx = v; mi = j; }   // j grows per thread: the first maximum of the thread
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, mx, o);
    const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
    if (om > mx || (om == mx && oi < mi)) { mx = om; mi = oi; }
  }
  if (lane == 0) { sh.fred[w] = mx; sh.ired[w] = mi; }
  __syncthreads();
  if (w == 0) {
    mx = sh.fred[lane];
    mi = sh.ired[lane];
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, mx, o);
      const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
      if (om > mx || (om == mx && oi < mi)) { mx = om; mi = oi; }
    }
    if (lane == 0) { sh.fred[0] = mx; sh.ired[0] = mi; }
  }
  __syncthreads();
  const float m = sh.fred[0];
  if (!(temperature > 0.f) || top_k == 1 || V == 1) {
    if (tid == 0) token_out[blockIdx.x] = sh.ired[0];
    return;
  }
  const float invT = 1.0f / temperature;
  const bool use_k = top_k > 0 && top_k < V;
  const bool use_p = top_p > 0.f && top_p < 1.f;

  // ---- boundary of the kept set: key fk and how many of the tokens with key == fk (in index order)
  //      are kept (n_tie); the mass of everything above fk
  uint32_t fk = 0;               // all keys >= 0: keep everything
  unsigned long long n_tie = 0xffffffffffffffffull;
  unsigned long long above_fk_mass = 0;
  auto radix = [&](bool by_mass, unsigned long long target) {
    // 3 levels: digits [31:20], [19:8], [7:0]; returns via fk / counts / masses above
    uint32_t prefix = 0, pmask = 0;
    unsigned long long above_m = 0, above_c = 0;
    const int shifts[3] = {20, 8, 0}, bits[3] = {12, 12, 8};
    for (int lv = 0; lv < 3; ++lv) {
      const int nb = 1 << bits[lv];
      for (int k = tid; k < nb; k += kSampleThreads) { sh.cnt[k] = 0; sh.mass[k] = 0; }
      __syncthreads();
      for (int j = tid; j < V; j += kSampleThreads) {
        const float v = lg(x, j);
        const uint32_t key = fkey(v);
        if ((key & pmask) == prefix) {
          const uint32_t d = (key >> shifts[lv]) & (uint32_t)(nb - 1);
          atomicAdd(&sh.cnt[d], 1u);
          atomicAdd(&sh.mass[d], wfix(v, m, invT));
        }
      }
      __syncthreads();
      find_digit(sh, nb, by_mass, target - (by_mass ? above_m : above_c));
      const uint32_t d = sh.digit;
      const unsigned long long a_sel = sh.tie_take;   // selected quantity above d within this level
      // counts / masses of the bins above d (this level)
      unsigned long long am = 0, ac = 0;
      {
        unsigned long long tot;
        unsigned long long vm = 0, vc = 0;
        for (int k = tid; k < nb; k += kSampleThreads)
          if ((uint32_t)k > d) { vm += sh.mass[k]; vc += sh.cnt[k]; }
        block_excl_scan(vm, sh, &tot);
        am = tot;
        block_excl_scan(vc, sh, &tot);
        ac = tot;
      }
      (void)a_sel;
      above_m += am;
      above_c += ac;
      prefix |= d << shifts[lv];
      pmask |= (uint32_t)(nb - 1) << shifts[lv];
      __syncthreads();
    }
    // the boundary key, tokens strictly above it, and the mass strictly above it
    fk = prefix;
    return make_ulonglong2(above_c, above_m);
  };
  unsigned long long mass_kept_total = 0;
  if (use_k) {
    const ulonglong2 r = radix(false, (unsigned long long)top_k);
    const unsigned long long wk = 0;   // mass of one token at fk (recomputed below)
    (void)wk;
    n_tie = (unsigned long long)top_k - r.x;
    above_fk_mass = r.y;
    mass_kept_total = above_fk_mass + n_tie * wfix(__uint_as_float((fk & 0x80000000u) ? (fk & 0x7fffffffu) : ~fk), m, invT);
  } else {
    // total mass of the row
    unsigned long long v = 0, tot;
    for (int j = tid; j < V; j += kSampleThreads) v += wfix(lg(x, j), m, invT);
    block_excl_scan(v, sh, &tot);
    mass_kept_total = tot;
  }
  if (use_p) {
    // the shortest prefix (key desc, index asc) of the kept set with mass >= P * M: the boundary key
    // pk with mass(key > pk) < target <= mass(key >= pk); tokens at pk needed: ceil((target -
    // mass(key > pk)) / w(pk)) (all equal keys carry equal mass)
    const unsigned long long target = (unsigned long long)ceil((double)top_p * (double)mass_kept_total);
    const uint32_t fk_k = fk;
    const unsigned long long n_tie_k = n_tie;
    const ulonglong2 r = radix(true, target);
    const float xb = __uint_as_float((fk & 0x80000000u) ? (fk & 0x7fffffffu) : ~fk);
    const unsigned long long wb = wfix(xb, m, invT);
    const unsigned long long need = wb ? (target - r.y + wb - 1) / wb : 1;
    if (use_k && fk == fk_k) n_tie = need < n_tie_k ? need : n_tie_k;   // same boundary: the stricter
    else n_tie = need;
    above_fk_mass = r.y;
  }

  // ---- the draw: per-thread contiguous chunks, tie ranks and kept masses scanned across the block
  const int per = (V + kSampleThreads - 1) / kSampleThreads;
  const int j0 = min(V, tid * per), j1 = min(V, j0 + per);
  unsigned long long ties = 0;
  for (int j = j0; j < j1; ++j) ties += fkey(lg(x, j)) == fk;
  unsigned long long tot;
  const unsigned long long tie0 = block_excl_scan(ties, sh, &tot);
  unsigned long long km = 0, rank = tie0;
  for (int j = j0; j < j1; ++j) {
    const float v = lg(x, j);
    const uint32_t key = fkey(v);
    if (key > fk || (key == fk && rank++ < n_tie)) km += wfix(v, m, invT);
  }
  const unsigned long long km0 = block_excl_scan(km, sh, &tot);
  const unsigned long long target = (unsigned long long)((double)uniforms[blockIdx.x] * (double)tot);
  if (tid == 0) sh.token = -1;
  __syncthreads();
  if (km > 0 && km0 <= target && target < km0 + km) {
    unsigned long long acc = km0, r2 = tie0;
    for (int j = j0; j < j1; ++j) {
      const float v = lg(x, j);
      const uint32_t key = fkey(v);
      if (key > fk || (key == fk && r2++ < n_tie)) {
        acc += wfix(v, m, invT);
        if (acc > target) {
          sh.token = j;
          break;
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    int t = sh.token;
    if (t < 0) t = sh.ired[0];   // u * M rounded onto the very end: the kept set's maximum
    token_out[blockIdx.x] = t;
  }
}

}  // namespace

cudaError_t launch_sample(const void* logits, int logits_dtype, int batch, int vocab, float temperature, int top_k,
                          float top_p, const float* uniforms, int32_t* token_out, cudaStream_t st) {
  const unsigned smem = sizeof(SampleShm);
  const void* f = logits_dtype == 1 ? (const void*)sample_kernel<float> : (const void*)sample_kernel<__nv_bfloat16>;
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {const_cast<void**>(&logits), &vocab, &temperature, &top_k, &top_p, const_cast<float**>(&uniforms),
                  &token_out};
  return cudaLaunchKernel(f, dim3(batch), dim3(kSampleThreads), args, smem, st);
}

}  // namespace asr
