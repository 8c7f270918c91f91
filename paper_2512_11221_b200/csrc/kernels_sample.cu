// paper_2512_11221_b200/csrc/kernels_sample.cu — NEXT-1: the next-token draw that
// closes Alg. 1 ("Generate next token"): greedy, or temperature + top-k + top-p filtering and
// one categorical draw per row with the caller's uniform u.  Rules (R-sample) are those of
// oracle/sample.py:
//   greedy (T <= 0 or k == 1): the first maximal logit;
//   kept set: the k largest logits (ties to lower indices), then the shortest prefix of them in
//   (logit desc, index asc) order holding >= P of their probability mass;
//   draw: the smallest index j in the kept set with  sum_{i kept, i <= j} p_i  >  u * sum_{kept} p_i.
//
// One thread-block cluster of CS CTAs per row (16 for batches up to 4, 8 up to 7, else 4); CTA r owns
// the contiguous slice r of the row and, when it fits, keeps it in shared memory for all passes.  After
// a top-k boundary is found, each CTA compacts its elements at or above it (index order) into shared
// memory and every later pass reads only those.  Every
// quantity the decisions need (max, counts and masses above the split points of the boundary search,
// tie counts, kept masses) is reduced within each CTA and exchanged through distributed shared memory
// (DSMEM) after a cluster barrier; every CTA then takes the same decision in the same fixed order.
// The boundaries are found by an 8-ary search on an order-preserving 32-bit key of the logit (bf16
// keys have 16 significant bits: 6 passes; fp32: 11), counting for top-k and summing mass for top-p.  Masses are exp((x - max) / T) in fp32, summed
// as 2^-36 fixed point in 64-bit integers: every sum is exact and order-independent, so a draw is
// bitwise deterministic.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

#include "asr_internal.h"

namespace cg = cooperative_groups;

// -DASR_SAMPLE_PROF (diagnostic builds only): rank 0 / thread 0 of row 0 prints the phase times
#ifdef ASR_SAMPLE_PROF
#define SPROF(k) do { if (tid == 0 && rank == 0 && row == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); sp_t[k] = t_; } } while (0)
#else
#define SPROF(k) do { } while (0)
#endif

namespace asr {
namespace {

constexpr int kST = 512;             // threads per CTA
constexpr int kSW = kST / 32;        // warps per CTA
constexpr int kWays = 8;             // split points per search pass: kWays - 1
constexpr float kFix = 68719476736.0f;   // 2^36
constexpr int kCand = 1024;          // top-k candidates kept per CTA in shared memory (value + index)
constexpr int kFastK = 256;          // top-k fast path: k <= kFastK, at most kSlot(CS) candidates per CTA
constexpr int kCS16Slots = 2048;     // candidate slots of the fast path at rank 0 (kSlot = kCS16Slots / CS)
constexpr int kFastPB = 64;          // pure top-p fast path: candidates >= the 64-th largest thread maximum

__device__ __forceinline__ float lg(const __nv_bfloat16* p, int j) { return __bfloat162float(p[j]); }
__device__ __forceinline__ float lg(const float* p, int j) { return p[j]; }

// order-preserving key of a float (-0 folded onto +0)
__device__ __forceinline__ uint32_t fkey(float x) {
  uint32_t b = __float_as_uint(x == 0.f ? 0.f : x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unkey(uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k); }

__device__ __forceinline__ unsigned long long wfix(float x, float m, float invT) {
  return (unsigned long long)(__expf((x - m) * invT) * kFix);   // exact power-of-two scale
}

struct SampleShm {
  unsigned long long wq[kSW][2 * kWays];   // per-warp partials (reused by every reduction)
  unsigned long long out[2][2 * kWays];    // this CTA's totals by call parity, read by the cluster (DSMEM)
  unsigned long long res[2 * kWays];       // cluster totals of the last reduction
  float fout;
  int iout;
  float zout, sout;   // this CTA's entropy partials (Z, S) about the row max, read by the cluster's rank 0
  // top-k fast path
  uint32_t tkout;                    // this CTA's bound T_c, read by the cluster
  int cnt[16];                       // candidates of every CTA of the cluster (each CTA writes its own into all)
  unsigned long long cms[16], sms[16];   // pure top-p: every CTA's candidate mass and slice mass
  unsigned long long ck[kCS16Slots]; // rank 0: candidate keys (key << 32 | ~index), kSlot slots per CTA
  unsigned long long cd[kCand];      // rank 0: the candidates, dense, in index order
  unsigned long long kk2[kFastK];    // rank 0: the top-k keys, in index order
  unsigned long long kw[kFastK];     // rank 0: their masses
  unsigned long long wsum[kSW];      // per-warp partials
  unsigned long long bkey;           // rank 0: the top-p boundary key
  int tok;                           // rank 0: the drawn index
};

// Largest t with #{threads whose key >= t} >= k (k >= 1) over one key per thread of the CTA, built
// bit by bit from the top over the bits in `vary` (bits outside it are those of `fixed`): one
// __syncthreads_count per bit; every thread calls it.
__device__ __forceinline__ uint32_t block_kth_u32(uint32_t key, bool valid, int k, uint32_t vary, uint32_t fixed) {
  uint32_t t = fixed & ~vary;
  for (int bit = 31; bit >= 0; --bit) {
    if (!((vary >> bit) & 1u)) continue;
    const uint32_t c = t | (1u << bit);
    if (__syncthreads_count(valid && key >= c) >= k) t = c;
  }
  return t;
}

// Visit elements j = first, first + stride, ... < end: kU loads are issued before any is used (the
// loops are latency-bound otherwise: one L2 round trip per element), then f(value, j) runs on each.
constexpr int kU = 8;
template <typename TL, typename Fn>
__device__ __forceinline__ void visit(const TL* __restrict__ x, int first, int end, int stride, Fn&& f) {
  for (int j0 = first; j0 < end; j0 += kU * stride) {
    float v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int j = j0 + u * stride;
      v[u] = lg(x, j < end ? j : first);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int j = j0 + u * stride;
      if (j < end) f(v[u], j);
    }
  }
}

// The same over [s0, s1) split among the CTA's threads in runs of 8 consecutive elements (16-byte
// loads, two for fp32), two runs per thread in flight; needs s0 % 8 == 0 and a 16-byte aligned row,
// else it falls back to visit().  Each thread sees its elements in increasing index order.
template <typename TL, typename Fn>
__device__ __forceinline__ void visit8(const TL* __restrict__ x, int s0, int s1, bool aligned, Fn&& f) {
  if (!aligned) {
    visit(x, s0 + (int)threadIdx.x, s1, kST, f);
    return;
  }
  constexpr int kW = sizeof(TL) == 2 ? 1 : 2;   // 16-byte words per run of 8
  constexpr int kR = 2;                          // runs in flight per thread
  for (int b0 = s0 + (int)threadIdx.x * 8; b0 < s1; b0 += kR * kST * 8) {
    uint4 r[kR][kW];
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const int b = b0 + u * kST * 8;
      const uint4* src = reinterpret_cast<const uint4*>(x + (b + 8 <= s1 ? b : s0));
#pragma unroll
      for (int w = 0; w < kW; ++w) r[u][w] = src[w];   // global or the shared-memory copy of the slice
    }
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const int b = b0 + u * kST * 8;
      if (b >= s1) break;
      float v[8];
      if (b + 8 <= s1) {
        if constexpr (sizeof(TL) == 2) {
          const uint32_t q[4] = {r[u][0].x, r[u][0].y, r[u][0].z, r[u][0].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) { v[2 * e] = __uint_as_float(q[e] << 16); v[2 * e + 1] = __uint_as_float(q[e] & 0xffff0000u); }
        } else {
          const uint32_t q[8] = {r[u][0].x, r[u][0].y, r[u][0].z, r[u][0].w,
                                 r[u][kW - 1].x, r[u][kW - 1].y, r[u][kW - 1].z, r[u][kW - 1].w};
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(q[e]);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) f(v[e], b + e);
      } else {
        for (int e = 0; b + e < s1; ++e) f(lg(x, b + e), b + e);
      }
    }
  }
}

// What a pass reads: this CTA's slice of the row, or its compacted top-k candidates.  each(f) runs
// f(value, position) on every element (split among the CTA's threads); each_strided visits positions
// first, first + stride, ... < end; val / idx read one element and its vocabulary index.
template <typename TL>
struct SliceSrc {
  const TL* x;   // the row (global memory or the shared-memory copy, indexed by vocabulary index)
  int s0, n;
  bool aligned;
  template <typename Fn>
  __device__ __forceinline__ void each(Fn&& f) const { visit8(x, s0, s0 + n, aligned, f); }
  template <typename Fn>
  __device__ __forceinline__ void each_strided(int first, int end, int stride, Fn&& f) const {
    visit(x, s0 + first, s0 + end, stride, f);
  }
  __device__ __forceinline__ float val(int p) const { return lg(x, s0 + p); }
  __device__ __forceinline__ int idx(int p) const { return s0 + p; }
};
struct CandSrc {
  const float* v;   // shared memory, index order
  const int* ix;
  int n;
  template <typename Fn>
  __device__ __forceinline__ void each(Fn&& f) const {
    for (int p = threadIdx.x; p < n; p += kST) f(v[p], p);
  }
  template <typename Fn>
  __device__ __forceinline__ void each_strided(int first, int end, int stride, Fn&& f) const {
    for (int p = first; p < end; p += stride) f(v[p], p);
  }
  __device__ __forceinline__ float val(int p) const { return v[p]; }
  __device__ __forceinline__ int idx(int p) const { return ix[p]; }
};

template <typename F>
__device__ __forceinline__ F warp_sum(F v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum n (<= 2*kWays) per-thread integers over the cluster: warps, then the CTA's warps, then lane r of
// warp 0 reads CTA r's total through DSMEM (integer sums: exact in any order).  One cluster barrier:
// the CTA totals alternate between two slots by call parity `par`, so a slot is rewritten only after
// every CTA has passed the next call's barrier.  Every thread gets the totals in res[0..n).
template <int CS>
__device__ void cluster_sum(cg::cluster_group& cl, SampleShm& sh, const unsigned long long* v, int n,
                            unsigned long long* res, int& par) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 2 * kWays; ++k)
    if (k < n) {
      const unsigned long long s = warp_sum(v[k]);
      if (lane == 0) sh.wq[w][k] = s;
    }
  __syncthreads();
  if ((int)threadIdx.x < n) {
    unsigned long long t = 0;
    for (int q = 0; q < kSW; ++q) t += sh.wq[q][threadIdx.x];
    sh.out[par][threadIdx.x] = t;
  }
  cl.sync();
  if (w == 0) {
    // all n remote loads in flight before the first is used (one DSMEM round trip, not n)
    unsigned long long r[2 * kWays];
    const SampleShm* o = cl.map_shared_rank(&sh, lane < CS ? lane : 0);
#pragma unroll
    for (int k = 0; k < 2 * kWays; ++k) r[k] = (k < n && lane < CS) ? o->out[par][k] : 0ull;
#pragma unroll
    for (int k = 0; k < 2 * kWays; ++k)
      if (k < n) {
        const unsigned long long t = warp_sum(r[k]);
        if (lane == 0) sh.res[k] = t;
      }
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) res[k] = sh.res[k];
  par ^= 1;
}

// CS CTAs (one cluster) per row
// With entropy_out, the same read of the row also yields H = ln Z - S / Z of p = softmax(x / ent_temp)
// (Z = sum e^{(x-m)/T}, S = sum e^{(x-m)/T} (x-m)/T about the row max m; R-ent) for the step's recovery
// detector (asr_step with ASR_ENTROPY_GIVEN): fp32 per thread, CTA partials summed in warp / rank order.
template <typename TL, int CS>
__global__ void __launch_bounds__(kST, 2) sample_kernel(const TL* __restrict__ logits, int V, float temperature, int top_k,
                                                     float top_p, const float* __restrict__ uniforms,
                                                     int32_t* __restrict__ token_out, int cache, float ent_temp,
                                                     float* __restrict__ entropy_out) {
  __shared__ SampleShm sh;
  extern __shared__ __align__(16) uint8_t slice_smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int row = blockIdx.y;
  const TL* xg = logits + (long)row * V;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int S = ((V + CS - 1) / CS + 31) & ~31;   // slice of this CTA: [s0, s1)
  int par = 0;                                     // cluster_sum slot parity
#ifdef ASR_SAMPLE_PROF
  unsigned long long sp_t[12] = {};
#endif
  SPROF(0);
  const int s0 = min(V, rank * S), s1 = min(V, s0 + S);
  const bool galigned = (reinterpret_cast<uintptr_t>(xg) & 15) == 0;   // s0 is a multiple of 32
  // the slice is read by every pass: with `cache`, once from global into shared memory
  const TL* x = xg;
  if (cache) {
    TL* c = reinterpret_cast<TL*>(slice_smem);
    if (galigned) {
      const int n16 = (s1 - s0) * (int)sizeof(TL) / 16;
      const uint4* src = reinterpret_cast<const uint4*>(xg + s0);
      uint4* dst = reinterpret_cast<uint4*>(c);
      for (int k = tid; k < n16; k += kST) dst[k] = __ldg(src + k);
      for (int j = s0 + n16 * 16 / (int)sizeof(TL) + tid; j < s1; j += kST) c[j - s0] = xg[j];
    } else {
      for (int j = s0 + tid; j < s1; j += kST) c[j - s0] = xg[j];
    }
    __syncthreads();
    x = c - s0;   // x[j] for j in [s0, s1) now reads shared memory
  }
  const bool aligned = cache || galigned;
  SPROF(1);

  // ---- max and its first index (greedy)
  float mx = -INFINITY;
  int mi = 0x7fffffff;
  visit8(x, s0, s1, aligned, [&](float v, int j) {
    if (v > mx) { mx = v; mi = j; }
  });
  // top-k fast path (k <= kFastK): T_c = the CTA's k-th largest thread maximum — k of its elements are
  // >= T_c, so the row's k-th largest value g_k >= T* = max_c T_c and every top-k element is >= T*
  // (pure top-p — no top-k — takes the same path with the bound of the kFastPB largest thread maxima
  // when the candidates hold the nucleus: their mass reaches P of the row's, checked by every CTA)
  const bool fastk = temperature > 0.f && top_k > 1 && top_k <= kFastK && top_k < V;
  const bool fastp = temperature > 0.f && !(top_k > 0 && top_k < V) && top_k != 1 && top_p > 0.f && top_p < 1.f && V > 1;
  const bool fast = fastk || fastp;
  const int kb = fastk ? top_k : min(kFastPB, V);
  const uint32_t tkey = mx == -INFINITY ? 0u : fkey(mx);
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, mx, o);
    const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
    if (om > mx || (om == mx && oi < mi)) { mx = om; mi = oi; }
  }
  if (lane == 0) { sh.wq[w][0] = __float_as_uint(mx); sh.wq[w][1] = (unsigned)mi; }
  __syncthreads();
  SPROF(2);
  if (fast) {
    // T_c: the k-th largest thread-maximum key (bf16 keys: the low 16 bits are zero)
    const uint32_t tc = block_kth_u32(tkey, true, kb, sizeof(TL) == 2 ? 0xffff0000u : 0xffffffffu, 0u);
    if (tid == 0) sh.tkout = tc;
  }
  SPROF(3);
  if (tid == 0) {
    for (int q = 0; q < kSW; ++q) {
      const float om = __uint_as_float((uint32_t)sh.wq[q][0]);
      const int oi = (int)sh.wq[q][1];
      if (om > mx || (om == mx && oi < mi)) { mx = om; mi = oi; }
    }
    sh.fout = mx;
    sh.iout = mi;
  }
  cl.sync();
  // lane r of warp 0 reads CTA r's values (one DSMEM round trip), reduced by shuffles, then broadcast
  if (w == 0) {
    float om = -INFINITY;
    int oi = 0x7fffffff;
    uint32_t ot = 0;
    if (lane < CS) {
      const SampleShm* o = cl.map_shared_rank(&sh, lane);
      om = o->fout;
      oi = o->iout;
      ot = o->tkout;
    }
    for (int off = 16; off > 0; off >>= 1) {
      const float pm = __shfl_xor_sync(0xffffffffu, om, off);
      const int pi = __shfl_xor_sync(0xffffffffu, oi, off);
      const uint32_t pt = __shfl_xor_sync(0xffffffffu, ot, off);
      if (pm > om || (pm == om && pi < oi)) { om = pm; oi = pi; }
      ot = max(ot, pt);
    }
    if (lane == 0) { sh.wq[0][8] = __float_as_uint(om); sh.wq[0][9] = (unsigned)oi; sh.wq[0][10] = ot; }
  }
  __syncthreads();
  mx = __uint_as_float((uint32_t)sh.wq[0][8]);
  mi = (int)sh.wq[0][9];
  const uint32_t tstar = fast ? (uint32_t)sh.wq[0][10] : 0u;
  __syncthreads();   // sh.wq is reused below
  // (no second barrier: fout / tkout are never rewritten, and every path syncs the cluster again
  // before a CTA leaves)
  SPROF(4);
  const float m = mx;
  if (entropy_out) {   // the entropy of the row, from the same (cached) slice
    const float invTe = 1.0f / ent_temp;
    float z = 0.f, sx = 0.f;
    visit8(x, s0, s1, aligned, [&](float v, int) {
      const float d = (v - m) * invTe;
      const float e = __expf(d);
      z += e;
      sx += e > 0.f ? e * d : 0.f;
    });
    z = warp_sum(z);
    sx = warp_sum(sx);
    if (lane == 0) { sh.wq[w][0] = __float_as_uint(z); sh.wq[w][1] = __float_as_uint(sx); }
    __syncthreads();
    if (tid == 0) {
      float zc = 0.f, sc = 0.f;
      for (int q = 0; q < kSW; ++q) { zc += __uint_as_float((uint32_t)sh.wq[q][0]); sc += __uint_as_float((uint32_t)sh.wq[q][1]); }
      sh.zout = zc;
      sh.sout = sc;
    }
    cl.sync();
    if (rank == 0 && tid == 0) {
      float zt = 0.f, st = 0.f;
      for (int r = 0; r < CS; ++r) {
        const SampleShm* o = cl.map_shared_rank(&sh, r);
        zt += o->zout;
        st += o->sout;
      }
      entropy_out[row] = logf(zt) - st / zt;
    }
    __syncthreads();   // sh.wq is reused by the passes below
  }
  if (!(temperature > 0.f) || top_k == 1 || V == 1) {
    cl.sync();   // no CTA leaves while another reads its max (or, with entropy_out, its partials)
    if (rank == 0 && tid == 0) token_out[row] = mi;
    return;
  }
  const float invT = 1.0f / temperature;
  const bool use_k = top_k > 0 && top_k < V;
  const bool use_p = top_p > 0.f && top_p < 1.f;

  // ---- the kept set's boundary: key fk, and n_tie of the tokens with key == fk (in index order)
  uint32_t fk = 0;
  unsigned long long n_tie = ~0ull;
  const int kshift = sizeof(TL) == 2 ? 16 : 0;
  // largest key t in [lo, hi) with Q(key >= t) >= target, Q = count (by_mass false) or fixed-point mass
  // over the elements `src` holds; needs Q(>= lo) >= target > Q(>= hi); an 8-ary search (the key ranges
  // stay powers of two); returns Q(key > t)
  auto search = [&](const auto& src, bool by_mass, unsigned long long target, unsigned long long lo,
                    unsigned long long hi) -> unsigned long long {
    unsigned long long q_hi = 0;
    while (hi - lo > 1) {
      const unsigned long long step = (hi - lo + kWays - 1) / kWays;
      // split points as 32-bit keys (clamped: a point at or above hi holds nothing new)
      uint32_t tk[kWays - 1];
#pragma unroll
      for (int k = 0; k < kWays - 1; ++k) {
        const unsigned long long t = lo + (k + 1) * step;
        tk[k] = t >= (1ull << (32 - kshift)) ? 0xffffffffu : (uint32_t)t;
      }
      unsigned long long q[kWays];
      uint32_t qc[kWays];
#pragma unroll
      for (int k = 0; k < kWays - 1; ++k) { q[k] = 0; qc[k] = 0; }
      src.each([&](float v, int) {
        const uint32_t kk = fkey(v) >> kshift;
        if (kk < tk[0]) return;
        if (by_mass) {
          const unsigned long long wv = wfix(v, m, invT);
#pragma unroll
          for (int k = 0; k < kWays - 1; ++k)
            if (kk >= tk[k]) q[k] += wv;
        } else {
#pragma unroll
          for (int k = 0; k < kWays - 1; ++k) qc[k] += kk >= tk[k];
        }
      });
      if (!by_mass)
#pragma unroll
        for (int k = 0; k < kWays - 1; ++k) q[k] = qc[k];
      unsigned long long tot[kWays];
      cluster_sum<CS>(cl, sh, q, kWays - 1, tot, par);
      unsigned long long nlo = lo, nhi = hi, nq = q_hi;
      for (int k = kWays - 2; k >= 0; --k) {
        const unsigned long long t = lo + (k + 1) * step;
        if (t >= hi) continue;
        if (tot[k] >= target) { nlo = t; break; }
        nhi = t;
        nq = tot[k];
      }
      lo = nlo;
      hi = nhi;
      q_hi = nq;
    }
    fk = (uint32_t)(lo << kshift);
    return q_hi;
  };
  const unsigned long long key_hi = (unsigned long long)(fkey(m) >> kshift) + 1;   // Q(>= key_hi) = 0

  // the top-p boundary (if any), then the draw, over the elements `src` holds (all of this CTA's
  // elements with key >= fk, in index order)
  auto finish = [&](const auto& src, unsigned long long kept_mass) {
    if (use_p) {
      // the boundary key of the shortest mass prefix: mass(key > pk) < target <= mass(key >= pk); it
      // lies at or above the top-k boundary (mass(key >= fk) >= kept_mass >= target), and the tokens
      // at pk it needs are the fewest whose equal masses reach the target
      const unsigned long long target = (unsigned long long)ceil((double)top_p * (double)kept_mass);
      const uint32_t fk_k = fk;
      const unsigned long long n_tie_k = n_tie;
      const unsigned long long ma = search(src, true, target, fk >> kshift, use_k ? key_hi : (1ull << (32 - kshift)));
      const unsigned long long wb = wfix(unkey(fk), m, invT);
      const unsigned long long need = wb ? (target - ma + wb - 1) / wb : 1;
      n_tie = (use_k && fk == fk_k && n_tie_k < need) ? n_tie_k : need;
    }

    // ---- the draw: ties (key == fk) are ranked in index order; warp q owns the contiguous chunk q of
    //      this CTA's elements, read in coalesced groups of 32 lanes
    const int per = ((src.n + kSW - 1) / kSW + 31) & ~31;
    const int c0 = min(src.n, w * per), c1 = min(src.n, c0 + per);
    unsigned long long tw = 0;
    src.each_strided(c0 + lane, c1, 32, [&](float x1, int) { tw += fkey(x1) == fk; });
    tw = warp_sum(tw);
    if (lane == 0) sh.wq[w][0] = tw;
    __syncthreads();
    if (tid == 0) {
      unsigned long long t = 0;
      for (int q = 0; q < kSW; ++q) t += sh.wq[q][0];
      sh.out[par][0] = t;
    }
    cl.sync();
    unsigned long long tie_base = 0;   // ties before this warp's chunk
    for (int r = 0; r < rank; ++r) tie_base += cl.map_shared_rank(&sh, r)->out[par][0];
    for (int q = 0; q < w; ++q) tie_base += sh.wq[q][0];
    par ^= 1;
    __syncthreads();   // wq[.][0] read by every warp before it is reused
    auto group = [&](int p, float v, unsigned long long& rk) -> unsigned long long {   // this lane's kept mass
      const bool in = p < c1;
      const uint32_t key = in ? fkey(v) : 0u;
      const bool tie = in && key == fk;
      const unsigned tm = __ballot_sync(0xffffffffu, tie);
      const unsigned long long my = rk + __popc(tm & ((1u << lane) - 1u));
      rk += __popc(tm);
      return (in && (key > fk || (tie && my < n_tie))) ? wfix(v, m, invT) : 0ull;
    };
    // groups of 32 (one element per lane), kU groups' loads in flight per lane
    auto load_groups = [&](int g0, float* v) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int p = g0 + u * 32 + lane;
        v[u] = src.val(p < c1 ? p : c0);
      }
    };
    unsigned long long wk = 0, rk = tie_base;
    for (int g0 = c0; g0 < c1; g0 += kU * 32) {
      float v[kU];
      load_groups(g0, v);
#pragma unroll
      for (int u = 0; u < kU; ++u) wk += group(g0 + u * 32 + lane, v[u], rk);
    }
    wk = warp_sum(wk);
    if (lane == 0) sh.wq[w][1] = wk;
    __syncthreads();
    if (tid == 0) {
      unsigned long long t = 0;
      for (int q = 0; q < kSW; ++q) t += sh.wq[q][1];
      sh.out[par][1] = t;
    }
    cl.sync();
    unsigned long long before = 0, total = 0;
    for (int r = 0; r < CS; ++r) {
      const unsigned long long t = cl.map_shared_rank(&sh, r)->out[par][1];
      if (r < rank) before += t;
      total += t;
    }
    for (int q = 0; q < w; ++q) before += sh.wq[q][1];
    const unsigned long long target = (unsigned long long)((double)uniforms[row] * (double)total);
    if (wk > 0 && before <= target && target < before + wk) {   // warp-uniform: the warp holding the draw
      unsigned long long acc = before, r2 = tie_base;
      bool found = false;
      for (int g0 = c0; g0 < c1 && !found; g0 += kU * 32) {
        float v[kU];
        load_groups(g0, v);
        for (int u = 0; u < kU; ++u) {
          const int gp = g0 + u * 32;
          const unsigned long long wv = group(gp + lane, v[u], r2);
          unsigned long long incl = wv;   // inclusive scan over the group (lane order = index order)
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          const unsigned hit = __ballot_sync(0xffffffffu, wv > 0 && acc + incl > target);
          if (hit) {
            if (lane == __ffs(hit) - 1) token_out[row] = src.idx(gp + lane);
            found = true;
            break;
          }
          acc += __shfl_sync(0xffffffffu, incl, 31);
        }
      }
    }
  };

  float* cv = reinterpret_cast<float*>(slice_smem + (cache ? (S * (int)sizeof(TL) + 15) / 16 * 16 : 0));
  int* ci = reinterpret_cast<int*>(cv + kCand);
  if (fast) {
    // ---- top-k fast path: every CTA sends its elements >= T* (in index order) to kSlot slots of its
    //      own at rank 0 and its count to every CTA; after one cluster barrier all know whether every
    //      count fit (else all take the general path below); rank 0 then finishes alone
    const int kSlot = kCS16Slots / CS;
    const int per = ((s1 - s0 + kSW - 1) / kSW + 31) & ~31;
    const int c0 = s0 + min(s1 - s0, w * per), c1 = min(s1, c0 + per);
    const int cend = c0 + ((c1 - c0 + 31) & ~31);   // whole groups of 32: every lane reaches the ballots
    unsigned cnt = 0;
    unsigned long long cms = 0, sms = 0;   // pure top-p: masses of the candidates / of the whole slice
    if (fastp) {
      for (int j = c0 + lane; j < cend; j += 32) {
        const float v = lg(x, j < c1 ? j : c0);
        const bool in = j < c1 && fkey(v) >= tstar;
        cnt += __popc(__ballot_sync(0xffffffffu, in));
        const unsigned long long wv = j < c1 ? wfix(v, m, invT) : 0ull;
        sms += wv;
        if (in) cms += wv;
      }
    } else {
      for (int j = c0 + lane; j < cend; j += 32) {
        const bool in = j < c1 && fkey(lg(x, j < c1 ? j : c0)) >= tstar;
        cnt += __popc(__ballot_sync(0xffffffffu, in));
      }
    }
    if (fastp) {
      cms = warp_sum(cms);
      sms = warp_sum(sms);
      if (lane == 0) { sh.wq[w][11] = cms; sh.wq[w][12] = sms; }
    }
    if (lane == 0) sh.wq[w][2] = cnt;
    __syncthreads();
    unsigned wbase = 0, ccount = 0;
    for (int q = 0; q < kSW; ++q) {
      if (q < w) wbase += (unsigned)sh.wq[q][2];
      ccount += (unsigned)sh.wq[q][2];
    }
    if (tid < CS) {
      SampleShm* o = cl.map_shared_rank(&sh, tid);
      o->cnt[rank] = (int)ccount;
      if (fastp) {
        unsigned long long cc = 0, ss = 0;
        for (int q = 0; q < kSW; ++q) { cc += sh.wq[q][11]; ss += sh.wq[q][12]; }
        o->cms[rank] = cc;
        o->sms[rank] = ss;
      }
    }
    if (ccount <= (unsigned)kSlot) {
      unsigned long long* gk = cl.map_shared_rank(sh.ck, 0) + rank * kSlot;
      unsigned p0 = wbase;
      for (int j = c0 + lane; j < cend; j += 32) {
        const uint32_t kk = j < c1 ? fkey(lg(x, j < c1 ? j : c0)) : 0u;
        const bool in = j < c1 && kk >= tstar;
        const unsigned msk = __ballot_sync(0xffffffffu, in);
        if (in) gk[p0 + __popc(msk & ((1u << lane) - 1u))] = ((unsigned long long)kk << 32) | (0xffffffffu - (uint32_t)j);
        p0 += __popc(msk);
      }
    }
    cl.sync();   // counts and candidates have landed; no CTA reads another's memory after this
    SPROF(5);
    bool fit = true;
    int ntot = 0;
    for (int r = 0; r < CS; ++r) {
      fit = fit && sh.cnt[r] <= kSlot;
      ntot += sh.cnt[r];
    }
    fit = fit && ntot <= kCand;
    unsigned long long ptarget = 0;   // pure top-p: ceil(P * the row's mass), as the general path
    if (fastp) {
      unsigned long long ca = 0, mall = 0;
      for (int r = 0; r < CS; ++r) { ca += sh.cms[r]; mall += sh.sms[r]; }
      ptarget = (unsigned long long)ceil((double)top_p * (double)mall);
      fit = fit && ca >= ptarget;   // the candidates (a prefix of the sorted row) hold the nucleus
    }
    if (fit) {
      if (rank != 0) return;
      // rank 0: the candidates, dense and in index order (slot r holds CTA r's, CTAs in index order)
      for (int i = tid; i < CS * kSlot; i += kST) {
        const int r = i / kSlot, e = i - r * kSlot;
        if (e < sh.cnt[r]) {
          int off = 0;
          for (int q = 0; q < r; ++q) off += sh.cnt[q];
          sh.cd[off + e] = sh.ck[i];
        }
      }
      __syncthreads();
      // the k-th largest key (key desc, index asc: composite keys are unique); two candidates per thread
      const unsigned long long a0 = tid < ntot ? sh.cd[tid] : 0ull;
      const unsigned long long a1 = tid + kST < ntot ? sh.cd[tid + kST] : 0ull;
      if (fastp) {
        // ---- pure top-p over the candidates: the boundary key t = the largest key with mass(key >= t)
        //      >= ceil(P * M) (bit by bit over the key bits that vary), then the fewest ties at t in
        //      index order that reach it, then the draw — the general path's rules and arithmetic
        const bool v0 = tid < ntot, v1 = tid + kST < ntot;
        const uint32_t k0 = (uint32_t)(a0 >> 32), k1 = (uint32_t)(a1 >> 32);
        const unsigned long long w0 = v0 ? wfix(unkey(k0), m, invT) : 0ull, w1 = v1 ? wfix(unkey(k1), m, invT) : 0ull;
        auto bsum = [&](unsigned long long v) -> unsigned long long {
          v = warp_sum(v);
          if (lane == 0) sh.wsum[w] = v;
          __syncthreads();
          unsigned long long s2 = 0;
          for (int q = 0; q < kSW; ++q) s2 += sh.wsum[q];
          __syncthreads();
          return s2;
        };
        uint32_t vo = (v0 ? k0 : 0u) | (v1 ? k1 : 0u);
        uint32_t va = (v0 ? k0 : ~0u) & (v1 ? k1 : ~0u);
        for (int o = 16; o > 0; o >>= 1) {
          vo |= __shfl_xor_sync(0xffffffffu, vo, o);
          va &= __shfl_xor_sync(0xffffffffu, va, o);
        }
        if (lane == 0) { sh.wq[w][3] = vo; sh.wq[w][4] = va; }
        __syncthreads();
        vo = 0u;
        va = ~0u;
        for (int q = 0; q < kSW; ++q) { vo |= (uint32_t)sh.wq[q][3]; va &= (uint32_t)sh.wq[q][4]; }
        const uint32_t vary = vo ^ va;
        uint32_t tb = va & ~vary;
        for (int bit = 31; bit >= 0; --bit) {
          if (!((vary >> bit) & 1u)) continue;
          const uint32_t c = tb | (1u << bit);
          if (bsum((v0 && k0 >= c ? w0 : 0ull) + (v1 && k1 >= c ? w1 : 0ull)) >= ptarget) tb = c;
        }
        const unsigned long long ma = bsum((v0 && k0 > tb ? w0 : 0ull) + (v1 && k1 > tb ? w1 : 0ull));
        const unsigned long long wb = wfix(unkey(tb), m, invT);
        const unsigned long long need = wb ? (ptarget - ma + wb - 1) / wb : 1;
        // ties at tb in index order (every first-half candidate precedes the second half)
        const bool t0 = v0 && k0 == tb, t1 = v1 && k1 == tb;
        const unsigned lt = (1u << lane) - 1u;
        const unsigned mt0 = __ballot_sync(0xffffffffu, t0), mt1 = __ballot_sync(0xffffffffu, t1);
        if (lane == 0) { sh.wq[w][5] = __popc(mt0); sh.wq[w][6] = __popc(mt1); }
        __syncthreads();
        unsigned long long tb0 = 0, tb1 = 0;
        for (int q = 0; q < kSW; ++q) {
          if (q < w) { tb0 += sh.wq[q][5]; tb1 += sh.wq[q][6]; }
          tb1 += sh.wq[q][5];
        }
        const bool i0 = v0 && (k0 > tb || (t0 && tb0 + __popc(mt0 & lt) < need));
        const bool i1 = v1 && (k1 > tb || (t1 && tb1 + __popc(mt1 & lt) < need));
        // the draw: inclusive kept mass in index order (first half, then second), first > u * total
        const unsigned long long x0 = i0 ? w0 : 0ull, x1 = i1 ? w1 : 0ull;
        unsigned long long s0i = x0, s1i = x1;
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned long long y0 = __shfl_up_sync(0xffffffffu, s0i, o), y1 = __shfl_up_sync(0xffffffffu, s1i, o);
          if (lane >= o) { s0i += y0; s1i += y1; }
        }
        __syncthreads();   // wq[.][5..6] read by every thread
        if (lane == 31) { sh.wq[w][5] = s0i; sh.wq[w][6] = s1i; }
        if (tid == 0) sh.tok = 0x7fffffff;
        __syncthreads();
        unsigned long long off0 = 0, off1 = 0, tot0 = 0, tot1 = 0;
        for (int q = 0; q < kSW; ++q) {
          if (q < w) { off0 += sh.wq[q][5]; off1 += sh.wq[q][6]; }
          tot0 += sh.wq[q][5];
          tot1 += sh.wq[q][6];
        }
        const unsigned long long total = tot0 + tot1;
        const unsigned long long target = (unsigned long long)((double)uniforms[row] * (double)total);
        if (i0 && w0 > 0 && off0 + s0i > target) atomicMin(&sh.tok, (int)(0xffffffffu - (uint32_t)(a0 & 0xffffffffull)));
        if (i1 && w1 > 0 && tot0 + off1 + s1i > target) atomicMin(&sh.tok, (int)(0xffffffffu - (uint32_t)(a1 & 0xffffffffull)));
        __syncthreads();
        if (tid == 0) token_out[row] = sh.tok;
        return;
      }
      // the k-th largest value key kv over the candidates, bit by bit over the bits that vary (OR / AND
      // over the block; the others are fixed); then the top-k = keys above kv plus the first `need`
      // candidates at kv in index order (array order)
      const int K = top_k;
      const bool v0 = tid < ntot, v1 = tid + kST < ntot;
      const uint32_t k0 = (uint32_t)(a0 >> 32), k1 = (uint32_t)(a1 >> 32);
      uint32_t vo = (v0 ? k0 : 0u) | (v1 ? k1 : 0u);
      uint32_t va = (v0 ? k0 : ~0u) & (v1 ? k1 : ~0u);
      for (int o = 16; o > 0; o >>= 1) {
        vo |= __shfl_xor_sync(0xffffffffu, vo, o);
        va &= __shfl_xor_sync(0xffffffffu, va, o);
      }
      if (lane == 0) { sh.wq[w][3] = vo; sh.wq[w][4] = va; }
      __syncthreads();
      vo = 0u;
      va = ~0u;
      for (int q = 0; q < kSW; ++q) { vo |= (uint32_t)sh.wq[q][3]; va &= (uint32_t)sh.wq[q][4]; }
      const uint32_t vary = vo ^ va;
      uint32_t kv = va & ~vary;
      for (int bit = 31; bit >= 0; --bit) {
        if (!((vary >> bit) & 1u)) continue;
        const uint32_t c = kv | (1u << bit);
        int n = __syncthreads_count(v0 && k0 >= c);
        if (ntot > kST) n += __syncthreads_count(v1 && k1 >= c);   // (CTA-uniform)
        if (n >= K) kv = c;
      }
      SPROF(6);
      // ties at kv: their rank in index order (halves: every first-half candidate precedes the second)
      const bool t0 = v0 && k0 == kv, t1 = v1 && k1 == kv;
      const bool g0 = v0 && k0 > kv, g1 = v1 && k1 > kv;
      const unsigned lt = (1u << lane) - 1u;
      {
        const unsigned mt0 = __ballot_sync(0xffffffffu, t0), mt1 = __ballot_sync(0xffffffffu, t1);
        const unsigned mg0 = __ballot_sync(0xffffffffu, g0), mg1 = __ballot_sync(0xffffffffu, g1);
        if (lane == 0) {
          sh.wq[w][5] = __popc(mt0);
          sh.wq[w][6] = __popc(mt1);
          sh.wq[w][7] = __popc(mg0) + __popc(mg1);
        }
        __syncthreads();
        int tb0 = 0, tb1 = 0, ng = 0;
        for (int q = 0; q < kSW; ++q) {
          if (q < w) { tb0 += (int)sh.wq[q][5]; tb1 += (int)sh.wq[q][6]; }
          tb1 += (int)sh.wq[q][5];
          ng += (int)sh.wq[q][7];
        }
        const int need = K - ng;   // >= 1
        const bool i0 = g0 || (t0 && tb0 + __popc(mt0 & lt) < need);
        const bool i1 = g1 || (t1 && tb1 + __popc(mt1 & lt) < need);
        __syncthreads();   // wq[.][5..7] reused
        // the top-k into kk2, in index order
        const unsigned m0 = __ballot_sync(0xffffffffu, i0), m1 = __ballot_sync(0xffffffffu, i1);
        if (lane == 0) { sh.wq[w][5] = __popc(m0); sh.wq[w][6] = __popc(m1); }
        __syncthreads();
        int b0 = 0, b1 = 0;
        for (int q = 0; q < kSW; ++q) {
          if (q < w) { b0 += (int)sh.wq[q][5]; b1 += (int)sh.wq[q][6]; }
          b1 += (int)sh.wq[q][5];
        }
        if (i0) sh.kk2[b0 + __popc(m0 & lt)] = a0;
        if (i1) sh.kk2[b1 + __popc(m1 & lt)] = a1;
      }
      __syncthreads();
      SPROF(7);
      // per kept element e (one per thread): mass, and the mass ranked above it (key desc, index asc) —
      // exact fixed-point sums
      unsigned long long we = 0, above = 0;
      const unsigned long long ke = tid < K ? sh.kk2[tid] : 0ull;
      if (tid < K) {
        we = wfix(unkey((uint32_t)(ke >> 32)), m, invT);
        sh.kw[tid] = we;
      }
      __syncthreads();
      if (tid < K)
        for (int q = 0; q < K; ++q)
          if (sh.kk2[q] > ke) above += sh.kw[q];
      unsigned long long ws = warp_sum(we);
      if (lane == 0) sh.wsum[w] = ws;
      __syncthreads();
      unsigned long long kmass = 0;
      for (int q = 0; q < kSW; ++q) kmass += sh.wsum[q];
      // top-p: keep the elements ranked at or above the first whose running mass reaches
      // ceil(P * kept mass) (the general path's boundary: ties carry equal masses, ordered by index)
      unsigned long long cut = 0ull;   // keep keys >= cut
      if (use_p) {
        const unsigned long long target = (unsigned long long)ceil((double)top_p * (double)kmass);
        if (tid < K && above < target && above + we >= target) sh.bkey = ke;   // exactly one (masses > 0)
        __syncthreads();
        cut = sh.bkey;
      }
      // the kept mass and, in index order, the draw: the smallest kept index whose running mass exceeds
      // u * kept mass (zero masses are never drawn)
      const bool kept = tid < K && ke >= cut;
      unsigned long long kw = kept ? we : 0ull;
      unsigned long long upk = 0;
      if (kept)
        for (int q = 0; q <= tid; ++q)
          if (sh.kk2[q] >= cut) upk += sh.kw[q];
      ws = warp_sum(kw);
      if (lane == 0) sh.wq[w][7] = ws;
      if (tid == 0) sh.tok = 0x7fffffff;
      __syncthreads();
      unsigned long long total = 0;
      for (int q = 0; q < kSW; ++q) total += sh.wq[q][7];
      const unsigned long long target = (unsigned long long)((double)uniforms[row] * (double)total);
      if (kept && we > 0 && upk > target) atomicMin(&sh.tok, (int)(0xffffffffu - (uint32_t)(ke & 0xffffffffull)));
      __syncthreads();
      if (tid == 0) token_out[row] = sh.tok;
      SPROF(8);
#ifdef ASR_SAMPLE_PROF
      if (tid == 0 && row == 0)
        printf("sprof ntot %d | load %llu max %llu bound %llu xchg %llu gather %llu search %llu topk %llu finish %llu ns\n",
               ntot, sp_t[1] - sp_t[0], sp_t[2] - sp_t[1], sp_t[3] - sp_t[2], sp_t[4] - sp_t[3], sp_t[5] - sp_t[4],
               sp_t[6] - sp_t[5], sp_t[7] - sp_t[6], sp_t[8] - sp_t[7]);
#endif
      return;
    }
  }
  const SliceSrc<TL> slice{x, s0, s1 - s0, aligned};
  if (!use_k) {
    unsigned long long v = 0, tot;
    slice.each([&](float x1, int) { v += wfix(x1, m, invT); });
    cluster_sum<CS>(cl, sh, &v, 1, &tot, par);
    finish(slice, tot);
  } else {
    const unsigned long long ca = search(slice, false, (unsigned long long)top_k, 0, key_hi);
    n_tie = (unsigned long long)top_k - ca;
    // ---- compaction: this CTA's elements with key >= fk (top_k plus any further ties, so few) in
    //      index order into shared memory, when they fit; every later pass then reads only them.  The
    //      choice is per CTA: every later quantity is a sum over the elements with key >= fk.
    const int per = ((s1 - s0 + kSW - 1) / kSW + 31) & ~31;
    const int c0 = s0 + min(s1 - s0, w * per), c1 = min(s1, c0 + per);
    const int cend = c0 + ((c1 - c0 + 31) & ~31);   // whole groups of 32: every lane reaches the ballots
    unsigned cnt = 0;
    for (int j = c0 + lane; j < cend; j += 32) {
      const bool in = j < c1 && fkey(lg(x, j < c1 ? j : c0)) >= fk;
      cnt += __popc(__ballot_sync(0xffffffffu, in));
    }
    if (lane == 0) sh.wq[w][2] = cnt;
    __syncthreads();
    unsigned long long base = 0, ncand = 0;
    for (int q = 0; q < kSW; ++q) {
      if (q < w) base += sh.wq[q][2];
      ncand += sh.wq[q][2];
    }
    const bool compact = ncand <= (unsigned long long)kCand;   // CTA-uniform
    if (compact) {
      for (int j = c0 + lane; j < cend; j += 32) {
        const float v = lg(x, j < c1 ? j : c0);
        const bool in = j < c1 && fkey(v) >= fk;
        const unsigned msk = __ballot_sync(0xffffffffu, in);
        if (in) {
          const int p = (int)base + __popc(msk & ((1u << lane) - 1u));
          cv[p] = v;
          ci[p] = j;
        }
        base += __popc(msk);
      }
    }
    __syncthreads();
    if (compact) {
      const CandSrc cand{cv, ci, (int)ncand};
      unsigned long long v = 0, tot;
      cand.each([&](float x1, int) { if (fkey(x1) > fk) v += wfix(x1, m, invT); });
      cluster_sum<CS>(cl, sh, &v, 1, &tot, par);
      finish(cand, tot + n_tie * wfix(unkey(fk), m, invT));
    } else {
      unsigned long long v = 0, tot;
      slice.each([&](float x1, int) { if (fkey(x1) > fk) v += wfix(x1, m, invT); });
      cluster_sum<CS>(cl, sh, &v, 1, &tot, par);
      finish(slice, tot + n_tie * wfix(unkey(fk), m, invT));
    }
  }
  cl.sync();   // no CTA leaves while another may still read its shared memory
}

template <int CS>
cudaError_t launch_cs(const void* logits, int logits_dtype, int batch, int vocab, float temperature, int top_k,
                      float top_p, const float* uniforms, int32_t* token_out, float ent_temp, float* entropy_out,
                      cudaStream_t st) {
  const size_t esz = logits_dtype == 1 ? 4 : 2;
  const size_t slice = (size_t)(((vocab + CS - 1) / CS + 31) & ~31) * esz;
  int cache = slice <= 96 * 1024 ? 1 : 0;   // the slice in shared memory (two CTAs per SM still fit)
  const size_t smem = (cache ? (slice + 15) / 16 * 16 : 0) + (size_t)kCand * 8;   // + the top-k candidates
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, batch);
  cfg.blockDim = dim3(kST);
  cfg.dynamicSmemBytes = (unsigned)smem;
  cfg.stream = st;
  if (CS > 8) {   // non-portable cluster size
    cudaError_t e = logits_dtype == 1
                        ? cudaFuncSetAttribute(sample_kernel<float, CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)
                        : cudaFuncSetAttribute(sample_kernel<__nv_bfloat16, CS>,
                                               cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (logits_dtype == 1) {
    cudaError_t e = cudaFuncSetAttribute(sample_kernel<float, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024 + kCand * 8);
    if (e != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, sample_kernel<float, CS>, (const float*)logits, vocab, temperature, top_k, top_p,
                              uniforms, token_out, cache, ent_temp, entropy_out);
  }
  cudaError_t e = cudaFuncSetAttribute(sample_kernel<__nv_bfloat16, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       96 * 1024 + kCand * 8);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(&cfg, sample_kernel<__nv_bfloat16, CS>, (const __nv_bfloat16*)logits, vocab, temperature,
                            top_k, top_p, uniforms, token_out, cache, ent_temp, entropy_out);
}

}  // namespace

// A cluster of 16 CTAs per row for batches up to 4 (not greedy), 8 up to 7 (and for fp32 logits), 4
// otherwise; each CTA keeps its slice of the row in shared memory when it fits (all passes then read
// shared memory).
cudaError_t launch_sample(const void* logits, int logits_dtype, int batch, int vocab, float temperature, int top_k,
                          float top_p, const float* uniforms, int32_t* token_out, float ent_temp, float* entropy_out,
                          cudaStream_t st) {
  const bool greedy = !(temperature > 0.f) || top_k == 1;   // one pass: the larger cluster's launch costs more
  if (batch <= 4 && !greedy)   // few rows: 16-CTA clusters (non-portable size; one per GPC) halve every pass
    return launch_cs<16>(logits, logits_dtype, batch, vocab, temperature, top_k, top_p, uniforms, token_out, ent_temp,
                         entropy_out, st);
  if (batch >= 8 && logits_dtype != 1)
    return launch_cs<4>(logits, logits_dtype, batch, vocab, temperature, top_k, top_p, uniforms, token_out, ent_temp,
                        entropy_out, st);
  return launch_cs<8>(logits, logits_dtype, batch, vocab, temperature, top_k, top_p, uniforms, token_out, ent_temp,
                      entropy_out, st);
}

}  // namespace asr
