// paper_2512_11221_b200/csrc/kernels_attn_mma.cu — (a4)+(a1) fast path for bf16 KV, head_dim 128,
// 4 query heads per KV head (LLaMA-3-8B: 32 q / 8 KV heads): split-KV decode attention over the
// active index list A_i with the Eq. 2 score fused into the QK^T pass.
//
//   O_{l,h} = softmax(q_{l,h} K_{A,l,g(h)}^T / sqrt(d)) V_{A,l,g(h)}       Eq. 1, Alg. 1 line 1
//   part_l(a) = sum_h |q_{l,h} . k_{l,A[a],g(h)}|                           Eq. 2, Alg. 1 line 2
//
// Design (tools/microbench_gather.cu measured the gather mechanisms on B200):
// - persistent CTAs over the ragged work list (b, l, chunk of A_b), one CTA per SM;
// - warp specialisation: 1 producer warp gathers the 4 KiB K|V row pair of each of 16 active tokens
//   per stage with ONE `cp.async.bulk` (1-D TMA, SASS UBLKCP) per token into a 3-stage shared-memory
//   ring completed by mbarrier transaction bytes, and the 8 KiB q of each work item into a 2-slot
//   q ring; the rings run across work items (no pipeline drain between chunks); the active index
//   of the next tile is prefetched while the current tile waits for its stage; 4112-byte token rows
//   keep ldmatrix bank-conflict free;
// - 8 consumer warps, one per KV head: S^T = q K^T with `mma.sync.m16n8k16` bf16 -> fp32 (4 query
//   heads on M, tokens on N; exact on the lattice inputs), |S| summed over the 4 heads with quad
//   shuffles gives the Eq. 2 head sum, fp32 online softmax (exp2), then O += P V with P split into
//   bf16 hi + lo parts (two MMAs, ~2^-16 relative error instead of bf16's 2^-9);
// - the producer also finishes the score: after a stage is released it sums the 8 warps' head sums
//   per token in fixed order and writes one fp32 partial per (b, l, token) — the only extra HBM
//   traffic of the score (0.1 % of the KV bytes).
#include <cuda_bf16.h>
#include <stdint.h>

// phase A units inside the attention kernel run on one dedicated warp (the last of the CTA)
#define ASR_UNIT_THREADS() 32u
#define ASR_UNIT_TID() (threadIdx.x & 31u)
#define ASR_UNIT_SYNC() __syncwarp()
#include "step_units.cuh"

namespace asr {
namespace {

constexpr int kD = 128;
constexpr int kTM = 16;               // tokens per stage
constexpr int kMaxB = 1024;           // sequences per context on this path

// Geometry of the kernel for HK KV heads (= consumer warps) and up to kGMax query heads per KV head.
// Smaller HK means smaller token rows, so the ring gets more stages to keep ~200 KB in flight.
template <int HK>
struct Geo {
  static constexpr int kHK = HK;
  static constexpr int kGMax = HK == 8 ? 4 : 8;
  static constexpr int kStagesRing = HK == 8 ? 3 : (HK == 4 ? 6 : 12);
  static constexpr int kRowBytes = HK * kD * 2;       // one token-layer K (or V) row, all heads
  static constexpr int kTokBytes = 2 * kRowBytes;     // K row then V row (contiguous in the pool)
  static constexpr int kTokPad = kTokBytes + 16;      // ldmatrix conflict-free stride
  static constexpr int kStageBytes = kTM * kTokPad;
  static constexpr int kThreads = (HK + 2) * 32;   // HK consumers, 1 producer, 1 phase-A warp
  static constexpr int kQBytes = HK * kGMax * kD * 2; // q of one (b, l), all heads (upper bound)
  struct Smem {
    alignas(128) uint8_t kv[kStagesRing][kStageBytes];
    alignas(128) uint8_t q[2][kQBytes];    // q of the current / next work item
    float sc[kStagesRing][HK][kTM];       // per-warp head sums |S| of each token
    int start[kMaxB + 1];                 // work list: first item of each sequence
    int range[2];                         // this CTA's static tile range (rate-balanced split)
    int4 unitq[16][2];                    // work units announced by the producer: cursor, stop, unit
    alignas(8) uint64_t full[kStagesRing];
    alignas(8) uint64_t empty[kStagesRing];
    alignas(8) uint64_t qfull[2];
    alignas(8) uint64_t qempty[2];
  };
};

#define ASR_GEO(HK)                                        \
  using Smem = typename Geo<HK>::Smem;                     \
  constexpr int kHK = Geo<HK>::kHK;                        \
  constexpr int kStagesRing = Geo<HK>::kStagesRing;        \
  constexpr int kRowBytes = Geo<HK>::kRowBytes;            \
  constexpr int kTokBytes = Geo<HK>::kTokBytes;            \
  constexpr int kTokPad = Geo<HK>::kTokPad;                \
  constexpr int kStageBytes = Geo<HK>::kStageBytes;        \
  (void)kHK; (void)kStagesRing; (void)kRowBytes; (void)kTokBytes; (void)kTokPad; (void)kStageBytes

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// The same with an L2 cache policy (the KV stream is read once per step: evict_first keeps it from
// displacing the ledger, partials and q that the next kernels read).
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Near the end of its last tile each CTA prefetches into L2 its share (4 KiB chunks, round robin in
// sequence / array order) of the ledger rows the decide kernel reads next: residency, timer and count
// of positions [0, n) and the A_i list (otherwise each of the decide's dependent loads would go to
// DRAM).  Called by the whole producer warp: the per-sequence sizes are loaded 32 at a time by the
// lanes, lane 0 issues the prefetches.
__device__ void prefetch_ledger(const DevState& s, int p, const int* __restrict__ alen, int step, int lane) {
  constexpr int kChunk = 4096;
  int k = 0;   // running chunk index over all (sequence, array) rows
  for (int b0 = 0; b0 < s.B; b0 += 32) {
    const int bl = b0 + lane;
    const int n_l = bl < s.B ? s.prompt_len[bl] + step + 1 : 0;
    const int a_l = bl < s.B ? alen[bl] : 0;
    for (int q = 0; q < 32 && b0 + q < s.B; ++q) {
      const int n = __shfl_sync(0xffffffffu, n_l, q), A = __shfl_sync(0xffffffffu, a_l, q);
      if (lane != 0) continue;
      const int b = b0 + q;
      const long row = (long)b * s.max_ctx;
      const char* base[4] = {reinterpret_cast<const char*>(s.res + row), reinterpret_cast<const char*>(s.timer + row),
                             reinterpret_cast<const char*>(s.count + row),
                             reinterpret_cast<const char*>(s.act_pos + act_off(s, p) + row)};
      const int bytes[4] = {n, 4 * n, 4 * n, 4 * A};
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int len = (bytes[a] + 15) & ~15;
        for (int off = 0; off < len; off += kChunk, ++k)
          if (k % (int)gridDim.x == (int)blockIdx.x) prefetch_l2(base[a] + off, (uint32_t)min(kChunk, len - off));
      }
    }
  }
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D += A(16x16 bf16, row) * B(16x8 bf16, col), fp32 accumulate
__device__ __forceinline__ void mma_bf16(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct ItemInfo {
  int b, l, a0, n;  // sequence, layer, first compact index, tokens
};

// Position in the stream-K tile order (asr_internal.h): tile t = tile ti of item (b, l), whose
// sequence has A active tokens in `tiles` tiles.  `start` = per-sequence first tile (prefix sums).
struct Cursor {
  int t, b, l, ti, tiles, A;
  __device__ void seek(const DevState& s, const int* __restrict__ alen, const int* start, int tt) {
    t = tt;
    int lo = 0, hi = s.B - 1;   // last sequence whose first tile is <= t (skips empty sequences)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (start[mid] <= tt) lo = mid;
      else hi = mid - 1;
    }
    b = lo;
    A = __ldcg(alen + b);
    tiles = (A + kTM - 1) / kTM;
    const int r = tt - start[b];
    l = r / tiles;
    ti = r - l * tiles;
  }
  __device__ void next(const DevState& s, const int* __restrict__ alen) {   // one tile forward
    ++t;
    if (++ti < tiles) return;
    ti = 0;
    if (++l < s.L) return;
    l = 0;
    for (++b; b < s.B; ++b) {
      A = __ldcg(alen + b);
      tiles = (A + kTM - 1) / kTM;
      if (tiles) break;
    }
  }
  __device__ int cnt() const { return min(kTM, A - ti * kTM); }
};

// Barriers, once per launch before any phase touches the ring.
template <int HK>
__device__ void attention_prologue(typename Geo<HK>::Smem& sm) {
  ASR_GEO(HK);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStagesRing; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], kHK);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.qfull[i], 1);
      mbar_init(&sm.qempty[i], kHK);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

// Cut fractions of the rate-balanced split (asr_internal.h, sk_weighted) for step + 2 (same
// parity), from the rates the CTAs measured in step - 2 (complete: that kernel has finished), run by
// one warp beside the attention (the last CTA's phase-A warp), off the critical path: f_c = P_c / P_G,
// P the prefix sums of the rates normalised by their mean and clamped to [0.5, 2]; CTA c = 8 lane + i.
__device__ __noinline__ void sk_fractions(const DevState& s, int step) {
  const int lane = threadIdx.x & 31;
  const int Gg = gridDim.x;
  const float* wr = s.sk_w + sk_wbuf(step, false) * kSkBalMax;
  float* fw = s.sk_f + sk_wbuf(step, true) * kSkBalMax;
  float w[kSkBalPer];
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < kSkBalPer; ++i) {
    const int cc = lane * kSkBalPer + i;
    w[i] = cc < Gg ? __ldcg(wr + cc) : 0.f;
    tot += w[i];
  }
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if (!(tot > 0.f)) return;   // no rates yet: step + 2 keeps the uniform split
  const float inv_mean = (float)Gg / tot;
  float run = 0.f;
#pragma unroll
  for (int i = 0; i < kSkBalPer; ++i) {
    const int cc = lane * kSkBalPer + i;
    const float x = cc < Gg ? fminf(fmaxf(w[i] * inv_mean, 0.5f), 2.f) : 0.f;
    w[i] = run;   // exclusive prefix within the lane
    run += x;
  }
  float incl = run;
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  float excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0.f;
  const float inv_p = 1.f / __shfl_sync(0xffffffffu, incl, 31);
#pragma unroll
  for (int i = 0; i < kSkBalPer; ++i) {
    const int cc = lane * kSkBalPer + i;
    if (cc <= Gg) __stcg(fw + cc, cc == 0 ? 0.f : cc == Gg ? 1.f : (excl + w[i]) * inv_p);
  }
}

// Folds this CTA's streaming rate over its first pass (tiles per clock since c0) into the rate
// buffer the next step of the same parity reads (sk_weighted).
__device__ __forceinline__ void sk_rate_update(const DevState& s, int step, const int* range, long long c0) {
  const int tiles = range[1] - range[0];
  const long long dc = clock64() - c0;
  if (tiles <= 0 || dc <= 0) return;
  const float rate = (float)tiles * 1e6f / (float)dc;   // tiles per 10^6 clocks
  const float old = __ldcg(s.sk_w + sk_wbuf(step, false) * kSkBalMax + blockIdx.x);
  s.sk_w[sk_wbuf(step, true) * kSkBalMax + blockIdx.x] = old > 0.f ? old + s.sk_ewma * (rate - old) : rate;
}

// The attention + score phase of one step (needs A_i, |A_i|, q and the appended K/V in memory).
// With do_pre (batch 1, DevState::pre_in_attn) the CTA's extra warp runs its phase-A unit (entropy
// split or append; the last unit of the sequence also runs phase B) beside the attention warps.
template <int HK, typename TL, bool DYN>
__device__ __forceinline__ void attention_phase(const DevState& s, const __nv_bfloat16* __restrict__ q,
                                const __nv_bfloat16* __restrict__ k_new, const __nv_bfloat16* __restrict__ v_new,
                                typename Geo<HK>::Smem& sm, bool do_pre, const TL* pre_logits, float* entropy_out,
                                units::UnitShm& u, float* __restrict__ o) {
  ASR_GEO(HK);
  const int step = *s.step;
  const int p = step & 1;                    // A_i lists of this step
  const int* __restrict__ alen = s.act_len + p * s.B;
  const int* __restrict__ aslot = s.act_slot + act_off(s, p);
  const int G = s.Hq / s.Hkv;               // query heads per KV head (<= Geo<HK>::kGMax)
  const int qbytes = s.Hq * kD * 2;         // q of one (b, l)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    // rate-balanced split: this CTA's cut fractions (a step of this parity computed them); loaded
    // before the list lengths so the two latencies overlap
    const int c = blockIdx.x, Gg = gridDim.x;
    float f0 = 0.f, f1 = 0.f;
    if (!DYN && s.sk_bal) {
      const float* fr = s.sk_f + sk_wbuf(step, false) * kSkBalMax;
      f0 = __ldcg(fr + c);
      f1 = __ldcg(fr + c + 1);
    }
    int acc = 0;
    for (int b = 0; b < s.B; ++b) {
      sm.start[b] = acc;
      acc += s.L * ((__ldcg(alen + b) + kTM - 1) / kTM);
    }
    sm.start[s.B] = acc;
    if (blockIdx.x == 0)
      for (int b = 0; b <= s.B; ++b) s.item_start[b] = sm.start[b];
    if (!DYN && s.sk_bal) {
      // sk_weighted: T >= 8 G (G = grid); fractions NaN: none computed yet -> uniform cut
      int r0, r1;
      if (acc < 8 * Gg) {
        const int G = min(acc, Gg);
        r0 = c < G ? c * acc / G : 0;
        r1 = c < G ? (c + 1) * acc / G : 0;
      } else if (!(f0 >= 0.f) || !(f1 >= 0.f)) {
        r0 = (int)((long)c * acc / Gg);
        r1 = (int)((long)(c + 1) * acc / Gg);
      } else {
        r0 = c == 0 ? 0 : (int)((float)acc * f0);
        r1 = c + 1 == Gg ? acc : (int)((float)acc * f1);
      }
      sm.range[0] = r0;
      sm.range[1] = r1;
      s.sk_bound[c] = r0;   // the combine's piece lookup (step_units.cuh combine_warp)
    }
  }
  __syncthreads();
  // units of work (asr_internal.h): this CTA's static stream-K range, then dynamic chunks; the
  // producer announces each following unit in sm.unitq before the arrive of the current unit's last
  // tile (a CTA without a static range: before a first arrive on stage 0)
  // (DYN = false: the static stream-K split alone, compiled without the unit machinery — batch 1's
  // producer is register-bound and the chunk overheads outweigh the balance there: DESIGN.md §6.1)
  const SkPlan plan = sk_plan(sm.start[s.B], gridDim.x, DYN ? s.sk_dyn : 0, s.sk_chunk);   // gridDim.x == s.sk_grid
  int t_begin = 0, t_end = 0;
  if (!DYN && s.sk_bal) {
    t_begin = sm.range[0];
    t_end = sm.range[1];
  } else if ((int)blockIdx.x < plan.G) {
    t_begin = (int)((long)blockIdx.x * plan.Ts / plan.G);
    t_end = (int)((long)(blockIdx.x + 1) * plan.Ts / plan.G);
  }

  if (warp == kHK) {
    // ================================================================== producer warp
    ItemInfo pend[kStagesRing];      // occupant of each stage (for the score epilogue)
#pragma unroll
    for (int i = 0; i < kStagesRing; ++i) pend[i].n = 0;
    auto epilogue = [&](int stage, const ItemInfo& it) {
      // it.a0 is the tile's first compact index here, it.n its tokens
      if (lane < it.n) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < kHK; ++w) t += sm.sc[stage][w][lane];
        s.score_part[((long)it.b * s.L + it.l) * s.max_ctx + it.a0 + lane] = t;
      }
    };
    int g = 0;   // tiles issued (the drain below continues from it)
    if constexpr (DYN) {
      const char* kvb = reinterpret_cast<const char*>(s.kv);
      // dynamic chunks: the ticket is drawn a few tiles before the current unit ends (its latency hidden
      // behind them) and used when it does
      int ticket = -1;   // lane 0
      auto draw = [&]() {
        if constexpr (DYN)
          if (lane == 0 && ticket < 0) ticket = plan.nchunks > 0 ? atomicAdd(s.sk_ctr, 1) : plan.nchunks;
      };
      auto grab = [&](Cursor& c, int& stop, int& unit) -> bool {
        if constexpr (!DYN) return false;
        draw();
        const int k = __shfl_sync(0xffffffffu, ticket, 0);
        ticket = -1;
        if (k >= plan.nchunks) return false;
        const long t0 = plan.Ts + (long)k * plan.C;
        stop = (int)min(plan.T, t0 + plan.C);
        unit = plan.G + k;
        c.seek(s, alen, sm.start, (int)t0);
        return true;
      };
      auto announce = [&](int slot, bool have, const Cursor& c, int stop, int unit) {
        if (DYN && lane == 0) {
          sm.unitq[slot & 15][0] = have ? make_int4(c.t, c.b, c.l, c.ti) : make_int4(-1, 0, 0, 0);
          sm.unitq[slot & 15][1] = make_int4(c.tiles, c.A, stop, unit);
        }
      };
      Cursor cur;
      int t_stop = t_end, unit = blockIdx.x, u_local = 0;
      bool have = t_begin < t_end;
      if (have) {
        cur.seek(s, alen, sm.start, t_begin);
      } else if (DYN) {   // no static range: the first unit (or "none", with a bare arrive) for the consumers
        have = grab(cur, t_stop, unit);
        announce(0, have, cur, t_stop, unit);
        if (lane == 0 && !have) mbar_arrive(&sm.full[0]);
      }
      auto load_idx = [&](const Cursor& c) -> int {
        if (lane >= c.cnt()) return 0;
        // device slot; through L2: recovery may recompact A_i while the kernel runs (redo pass)
        return max(0, __ldcg(aslot + (long)c.b * s.max_ctx + c.ti * kTM + lane));
      };
      int j_cur = have ? load_idx(cur) : 0;
      int it_local = -1;
      bool unit_first = true;
      // L2 policy of the KV stream: evict_first (ASR_KV_EVICT_FIRST=0: evict_normal, for comparison)
      const uint64_t kv_policy = s.kv_evict_first ? policy_evict_first() : policy_evict_normal();
      while (have) {
        if (DYN && cur.t + 3 >= t_stop) draw();
        Cursor nxt = cur;
        nxt.next(s, alen);
        int n_stop = t_stop, n_unit = unit;
        bool n_have = true, n_first = false;
        if (nxt.t >= t_stop) {   // this is the unit's last tile: announce the next unit (or none)
          n_have = grab(nxt, n_stop, n_unit);
          n_first = true;
          if (DYN) announce(u_local + 1, n_have, nxt, n_stop, n_unit);
        }
        const int j_next = n_have ? load_idx(nxt) : 0;   // in flight while this tile waits for its stage
        if (unit_first || cur.ti == 0) {   // new piece: stage its q (Hq x 256 B) in the q ring
          ++it_local;
          const int qs = it_local & 1;
          mbar_wait(&sm.qempty[qs], ((uint32_t)(it_local >> 1) & 1u) ^ 1u);
          if (lane == 0) {
            mbar_expect_tx(&sm.qfull[qs], (uint32_t)qbytes);
            bulk_g2s(&sm.q[qs][0], q + ((long)cur.b * s.L + cur.l) * s.Hq * kD, (uint32_t)qbytes, &sm.qfull[qs]);
          }
        }
        const int stage = g % kStagesRing;
        const uint32_t ph = (uint32_t)(g / kStagesRing) & 1u;
        mbar_wait(&sm.empty[stage], ph ^ 1u);
        __syncwarp();
        epilogue(stage, pend[stage]);
        const int cnt = cur.cnt();
        ItemInfo tile{cur.b, cur.l, cur.ti * kTM, cnt};
  #pragma unroll
        for (int i = 0; i < kStagesRing; ++i)
          if (i == stage) pend[i] = tile;
        if (cnt < kTM) {
          // masked tail rows: their P is 0, but 0 * NaN would poison O, so their V slices get zeros
          // (generic-proxy stores, ordered before later bulk copies into the same rows by the fence)
          uint4* z = reinterpret_cast<uint4*>(&sm.kv[stage][0]);
          const int per_row = kRowBytes / 16;
          for (int t = cnt; t < kTM; ++t)
            for (int k = lane; k < per_row; k += 32) z[(t * kTokPad + kRowBytes) / 16 + k] = make_uint4(0, 0, 0, 0);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        if (lane == 0) mbar_expect_tx(&sm.full[stage], (uint32_t)cnt * kTokBytes);
        __syncwarp();
        if (lane < cnt) {
          if (cur.ti * kTM + lane == cur.A - 1) {
            // the token this step appends (always last in A_i): read from the caller's k_new / v_new, so
            // the attention does not wait for phase A's append
            const long r = ((long)cur.b * s.L + cur.l) * (kRowBytes / 2);
            bulk_g2s(&sm.kv[stage][lane * kTokPad], k_new + r, kRowBytes, &sm.full[stage]);
            bulk_g2s(&sm.kv[stage][lane * kTokPad + kRowBytes], v_new + r, kRowBytes, &sm.full[stage]);
          } else {
            const long slot = j_cur;
            bulk_g2s_hint(&sm.kv[stage][lane * kTokPad], kvb + (slot * s.L + cur.l) * (long)kTokBytes, kTokBytes,
                          &sm.full[stage], kv_policy);
          }
        }
        j_cur = j_next;
        cur = nxt;
        if (n_first) ++u_local;
        t_stop = n_stop;
        unit = n_unit;
        unit_first = n_first;
        have = n_have;
        ++g;
      }
      // no more chunks for this CTA: the last CTA to get here resets the chunk ticket for the next launch
      if (DYN && lane == 0 && plan.nchunks > 0 && atomicAdd(s.sk_ctr + 1, 1) == (int)gridDim.x - 1) {
        s.sk_ctr[0] = 0;
        s.sk_ctr[1] = 0;
      }
    } else {   // static stream-K range only (batch < 16): the round-1 producer, fewest registers
      const char* kvb = reinterpret_cast<const char*>(s.kv);
      Cursor cur;
      if (t_begin < t_end) cur.seek(s, alen, sm.start, t_begin);
      else cur.t = t_end;
      auto load_idx = [&](const Cursor& c) -> int {
        if (c.t >= t_end || lane >= c.cnt()) return 0;
        // device slot; through L2: recovery may recompact A_i while the kernel runs (redo pass)
        return max(0, __ldcg(aslot + (long)c.b * s.max_ctx + c.ti * kTM + lane));
      };
      int j_cur = load_idx(cur);
      int it_local = -1;
      // L2 policy of the KV stream: evict_first (ASR_KV_EVICT_FIRST=0: evict_normal, for comparison)
      const uint64_t kv_policy = s.kv_evict_first ? policy_evict_first() : policy_evict_normal();
      while (cur.t < t_end) {
        Cursor nxt = cur;
        nxt.next(s, alen);
        const int j_next = load_idx(nxt);   // in flight while this tile waits for its stage
        if (cur.t == t_begin || cur.ti == 0) {   // new piece: stage its q (Hq x 256 B) in the q ring
          ++it_local;
          const int qs = it_local & 1;
          mbar_wait(&sm.qempty[qs], ((uint32_t)(it_local >> 1) & 1u) ^ 1u);
          if (lane == 0) {
            mbar_expect_tx(&sm.qfull[qs], (uint32_t)qbytes);
            bulk_g2s(&sm.q[qs][0], q + ((long)cur.b * s.L + cur.l) * s.Hq * kD, (uint32_t)qbytes, &sm.qfull[qs]);
          }
        }
        const int stage = g % kStagesRing;
        const uint32_t ph = (uint32_t)(g / kStagesRing) & 1u;
        mbar_wait(&sm.empty[stage], ph ^ 1u);
        __syncwarp();
        epilogue(stage, pend[stage]);
        const int cnt = cur.cnt();
        ItemInfo tile{cur.b, cur.l, cur.ti * kTM, cnt};
  #pragma unroll
        for (int i = 0; i < kStagesRing; ++i)
          if (i == stage) pend[i] = tile;
        if (cnt < kTM) {
          // masked tail rows: their P is 0, but 0 * NaN would poison O, so their V slices get zeros
          // (generic-proxy stores, ordered before later bulk copies into the same rows by the fence)
          uint4* z = reinterpret_cast<uint4*>(&sm.kv[stage][0]);
          const int per_row = kRowBytes / 16;
          for (int t = cnt; t < kTM; ++t)
            for (int k = lane; k < per_row; k += 32) z[(t * kTokPad + kRowBytes) / 16 + k] = make_uint4(0, 0, 0, 0);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        if (lane == 0) mbar_expect_tx(&sm.full[stage], (uint32_t)cnt * kTokBytes);
        __syncwarp();
        if (lane < cnt) {
          if (cur.ti * kTM + lane == cur.A - 1) {
            // the token this step appends (always last in A_i): read from the caller's k_new / v_new, so
            // the attention does not wait for phase A's append
            const long r = ((long)cur.b * s.L + cur.l) * (kRowBytes / 2);
            bulk_g2s(&sm.kv[stage][lane * kTokPad], k_new + r, kRowBytes, &sm.full[stage]);
            bulk_g2s(&sm.kv[stage][lane * kTokPad + kRowBytes], v_new + r, kRowBytes, &sm.full[stage]);
          } else {
            const long slot = j_cur;
            bulk_g2s_hint(&sm.kv[stage][lane * kTokPad], kvb + (slot * s.L + cur.l) * (long)kTokBytes, kTokBytes,
                          &sm.full[stage], kv_policy);
          }
        }
        j_cur = j_next;
        cur = nxt;
        ++g;
      }
    }
    // large batches: phase D is not latency-bound; fused tail: the aux warp prefetched at the start
    // (the ledger rows phase D reads are prefetched into L2 by the aux warp, off the producer's exit)
    // drain: the last (up to) kStagesRing tiles still owe their score epilogue
    for (int k = 0; k < kStagesRing; ++k) {
      const int gg = g + k;  // waiting for the release of tile gg - kStagesRing
      const int stage = gg % kStagesRing;
      if (gg - kStagesRing < 0) continue;
      mbar_wait(&sm.empty[stage], ((uint32_t)(gg / kStagesRing) & 1u) ^ 1u);
      __syncwarp();
      epilogue(stage, pend[stage]);
    }
    return;   // the producer warp is done with this phase
  }
  if (warp == kHK + 1) {
    // ================================================================== phase-A warp (batch 1)
    if (do_pre && (int)blockIdx.x < units::phaseA_units(s, pre_logits != nullptr)) {
      if (s.tl && lane == 0) atomicMin(&s.tl[0], gtimer());
      units::phaseA_block<TL, __nv_bfloat16>(s, blockIdx.x, step, pre_logits, k_new, v_new, entropy_out, u);
      if (s.tl && lane == 0) atomicMax(&s.tl[1], gtimer());
    }
    // small batches: the ledger rows phase D (or the fused tail) reads, into L2 while the attention
    // streams (KV loads are evict_first, these stay) — not at the producer's exit, where it delayed
    // the CTA's end by ~2 us
    if (s.B <= 8) prefetch_ledger(s, step & 1, s.act_len + (step & 1) * s.B, step, lane);
    if (!DYN && s.sk_bal && s.sk_learn && blockIdx.x == gridDim.x - 1) sk_fractions(s, step);
    if (s.fuse_tail && !(s.tail_exp & 2)) {
      // instruction prefetch: a dry run (loads and arithmetic only, no stores, no waits) of the fused
      // tail's two functions while the attention streams, so their code is on chip when the tail runs
      // (it runs once per SM per step, right on the critical path); the arguments are opaque to the
      // compiler so both runs execute the one non-inlined copy
      const int D = sm.start[s.B] / s.L;
      const bool dry = opaque(0) != 0;
      uint32_t* no_scratch = reinterpret_cast<uint32_t*>((uintptr_t)opaque(0));
      if (D > 0)
        units::warp_settle_segment(s, 0, min((int)blockIdx.x, (sm.start[1] / s.L) - 1), step, no_scratch, opaque(0),
                                   dry);
      if (o) units::combine_warp_tail(s, (int)blockIdx.x % (s.B * s.L * s.Hq), o, dry);
    }
    return;
  }

  // ==================================================================== consumer warps (KV head = warp)
  const float scale = 1.4426950408889634f * 0.08838834764831845f;  // log2(e) / sqrt(128)
  const int r = lane >> 2, qd = lane & 3;   // fragment row / quad column
  const uint32_t kvbase = smem_u32(&sm.kv[0][0]);
  // ldmatrix lane addresses (bytes within a stage tile, this warp's head)
  const int mi = lane >> 3, ri = lane & 7;
  const uint32_t k_lane = (uint32_t)((ri + (mi >> 1) * 8) * kTokPad + warp * kD * 2 + (mi & 1) * 16);
  const uint32_t v_lane = (uint32_t)((ri + (mi & 1) * 8) * kTokPad + kRowBytes + warp * kD * 2 + (mi >> 1) * 16);
  int g = 0, it_local = -1;
  Cursor cur;
  int t_stop = t_end, unit = blockIdx.x;
  const bool has_static = t_begin < t_end;
  if (has_static) cur.seek(s, alen, sm.start, t_begin);
  else if (DYN) mbar_wait(&sm.full[0], 0u);   // unit 0 is announced before the first tile's (or a bare) arrive
  else cur.t = t_end;
  for (int u = 0; DYN || u == 0; ++u) {   // units; unit u + 1 is announced before the arrive of unit u's last tile
    if (DYN && (u > 0 || !has_static)) {
      const int4 u0 = sm.unitq[u & 15][0], u1 = sm.unitq[u & 15][1];
      if (u0.x < 0) break;
      cur.t = u0.x; cur.b = u0.y; cur.l = u0.z; cur.ti = u0.w;
      cur.tiles = u1.x; cur.A = u1.y; t_stop = u1.z; unit = u1.w;
    }
  while (cur.t < t_stop) {   // one piece (the part of one (b, l) item in this unit) per pass
    const long piece = (long)cur.b * s.L + cur.l + unit;
    const int pb = cur.b, pl = cur.l;
    const bool from_item_start = cur.ti == 0;
    bool to_item_end = false;
    // q fragments from the q ring (rows 0..3 = the 4 query heads of this KV head, rows 4..15 zero)
    ++it_local;
    const int qs = it_local & 1;
    mbar_wait(&sm.qfull[qs], (uint32_t)(it_local >> 1) & 1u);
    uint32_t qa[8][2];
    {
      const __nv_bfloat16* qh = reinterpret_cast<const __nv_bfloat16*>(&sm.q[qs][0]) + (warp * G + (r < G ? r : 0)) * kD;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t lo = *reinterpret_cast<const uint32_t*>(qh + ks * 16 + 2 * qd);
        uint32_t hi = *reinterpret_cast<const uint32_t*>(qh + ks * 16 + 8 + 2 * qd);
        qa[ks][0] = r < G ? lo : 0u;
        qa[ks][1] = r < G ? hi : 0u;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.qempty[qs]);
    float acc[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;
    for (bool more = true; more; ++g) {
      const int stage = g % kStagesRing;
      const uint32_t ph = (uint32_t)(g / kStagesRing) & 1u;
      const int cnt = cur.cnt();
      more = cur.ti + 1 < cur.tiles;   // the piece ends with its item's last tile or the range's end
      to_item_end = !more;
      cur.next(s, alen);
      more = more && cur.t < t_stop;
      mbar_wait(&sm.full[stage], ph);
      const uint32_t ks_addr = kvbase + stage * kStageBytes + k_lane;
      const uint32_t vs_addr = kvbase + stage * kStageBytes + v_lane;
      // ---- S^T[head][token] = q . k
      float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(ks_addr + ks * 32, b0, b1, b2, b3);
        mma_bf16(c0, qa[ks][0], 0u, qa[ks][1], 0u, b0, b1);
        mma_bf16(c1, qa[ks][0], 0u, qa[ks][1], 0u, b2, b3);
      }
      // tokens of this thread's columns: n0 = 2qd, n0+1 (tile 0), 8+2qd, 9+2qd (tile 1)
      const int n0 = 2 * qd;
      const bool v00 = n0 < cnt, v01 = n0 + 1 < cnt, v10 = n0 + 8 < cnt, v11 = n0 + 9 < cnt;
      // ---- Eq. 2 head sum: |S| over the G valid rows (rows >= G hold exact zeros: their q is zero)
      float s00 = fabsf(c0[0]), s01 = fabsf(c0[1]), s10 = fabsf(c1[0]), s11 = fabsf(c1[1]);
#pragma unroll
      for (int o = 4; o <= 16; o <<= 1) {
        s00 += __shfl_xor_sync(0xffffffffu, s00, o);
        s01 += __shfl_xor_sync(0xffffffffu, s01, o);
        s10 += __shfl_xor_sync(0xffffffffu, s10, o);
        s11 += __shfl_xor_sync(0xffffffffu, s11, o);
      }
      if (lane < 4) {
        float* scw = sm.sc[stage][warp];
        scw[n0] = s00;
        scw[n0 + 1] = s01;
        scw[n0 + 8] = s10;
        scw[n0 + 9] = s11;
      }
      // ---- online softmax (row = head r; rows >= 4 are padding and never written out)
      const float x00 = v00 ? c0[0] * scale : -INFINITY, x01 = v01 ? c0[1] * scale : -INFINITY;
      const float x10 = v10 ? c1[0] * scale : -INFINITY, x11 = v11 ? c1[1] * scale : -INFINITY;
      float mt = fmaxf(fmaxf(x00, x01), fmaxf(x10, x11));
      mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1));
      mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 2));
      const float m_new = fmaxf(m_run, mt);
      const float corr = exp2f(m_run - m_new);
      const float p00 = exp2f(x00 - m_new), p01 = exp2f(x01 - m_new);
      const float p10 = exp2f(x10 - m_new), p11 = exp2f(x11 - m_new);
      l_run = l_run * corr + (p00 + p01 + p10 + p11);
      m_run = m_new;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        acc[i][0] *= corr;
        acc[i][1] *= corr;
      }
      // P = hi + lo (bf16 each): bf16 P alone would break the 2e-3 bar
      const uint32_t ph0 = pack_bf16(p00, p01), ph1 = pack_bf16(p10, p11);
      const __nv_bfloat162 h0 = *reinterpret_cast<const __nv_bfloat162*>(&ph0);
      const __nv_bfloat162 h1 = *reinterpret_cast<const __nv_bfloat162*>(&ph1);
      const uint32_t pl0 = pack_bf16(p00 - __low2float(h0), p01 - __high2float(h0));
      const uint32_t pl1 = pack_bf16(p10 - __low2float(h1), p11 - __high2float(h1));
      // ---- O += P V
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vs_addr + dp * 32, b0, b1, b2, b3);
        mma_bf16(acc[2 * dp], ph0, 0u, ph1, 0u, b0, b1);
        mma_bf16(acc[2 * dp], pl0, 0u, pl1, 0u, b0, b1);
        mma_bf16(acc[2 * dp + 1], ph0, 0u, ph1, 0u, b2, b3);
        mma_bf16(acc[2 * dp + 1], pl0, 0u, pl1, 0u, b2, b3);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[stage]);
    }
    // ---- partial outputs of this item: rows 0..3 (lanes 0..15)
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    if (r < G && o && from_item_start && to_item_end) {
      // the whole item lies in one unit: O directly (the combine skips single-piece items)
      const float inv = 1.0f / l_run;
      float* dst = o + (((long)pb * s.L + pl) * s.Hq + warp * G + r) * kD + 2 * qd;
#pragma unroll
      for (int i = 0; i < 16; ++i) *reinterpret_cast<float2*>(dst + i * 8) = make_float2(acc[i][0] * inv, acc[i][1] * inv);
    } else if (r < G) {
      ASR_CHECK(s, piece >= 0 && piece < s.max_items);
      const long pi = piece * s.Hq + warp * G + r;
      if (qd == 0) {
        s.part_ml[pi * 2] = m_run;
        s.part_ml[pi * 2 + 1] = l_run;
      }
      float* dst = s.part_acc + pi * kD + 2 * qd;
#pragma unroll
      for (int i = 0; i < 16; ++i) *reinterpret_cast<float2*>(dst + i * 8) = make_float2(acc[i][0], acc[i][1]);
    }
  }
  }
}


// Barrier over the CTAs of the attention grid (one CTA per SM, all resident: persistent grid of
// num_SMs CTAs at one CTA per SM); used when recovery forces a second pass and before the fused
// tail.  bar is a monotonic 64-bit arrival counter (never reset): barrier instance k completes when
// it reaches (k+1) * gridDim.x.  Release on arrival, acquire on the wait (bar.sync makes them
// cumulative over the CTA's threads).
__device__ void grid_sync(unsigned* bar32, uint32_t* err) {
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(bar32);
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long G = gridDim.x;
    const unsigned long long old = atom_add_acqrel_u64(bar, 1ull);
    const unsigned long long target = old - old % G + G;
    if (ld_acquire_u64(bar) < target) {
      const unsigned long long t0 = gtimer();
      while (ld_acquire_u64(bar) < target) {
        __nanosleep(32);
        if (gtimer() - t0 > 2000000000ull) {   // 2 s: never on a healthy device; do not hang it
          atomicOr(err, kErrStall);
          break;
        }
      }
    }
  }
  __syncthreads();
}

// Fused tail of a step (DevState::fuse_tail): after a grid barrier (every partial and score of the
// step is in memory), the warps of the grid settle the step — Alg. 1 lines 3-15 + A_{i+1} per token
// tile (units::warp_decide_tile, placed by a decoupled look-back) and the fixed-order combine of the
// items split across CTAs (units::combine_warp) — then the last CTA out advances the step.  Replaces
// the phase-D kernel (its launch gap and one-block latency chains) at small batch.
template <int HK>
__device__ void fused_tail(const DevState& s, typename Geo<HK>::Smem& sm, int step, float* o) {
  if (s.tl && threadIdx.x == 0) atomicMax(&s.tl[kTlTail], gtimer());
  grid_sync(s.gbar, s.err);
  if (s.tl && threadIdx.x == 0) atomicMax(&s.tl[kTlTail + 1], gtimer());
  if (s.tl && threadIdx.x == 0) atomicMin(&s.tl[2 * 2], gtimer());
  const int nw = (int)(blockDim.x >> 5), warp = (int)(threadIdx.x >> 5);
  const int G = (int)gridDim.x, NW = G * nw;
  const int r = warp * G + (int)blockIdx.x;   // consecutive ranks sit on different CTAs
  const int D = sm.start[s.B] / s.L;         // token tiles of all sequences (start[] counts L per tile)
  for (int k = r; k < D; k += NW) {
    int lo = 0, hi = s.B - 1;                // last sequence whose first token tile is <= k
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (sm.start[mid] / s.L <= k) lo = mid;
      else hi = mid - 1;
    }
    // the KV ring is idle now: a slice of it per warp holds the segment's final residency words
    constexpr int kScap = (int)(sizeof(sm.kv) / 4) / (Geo<HK>::kThreads / 32);
    uint32_t* scratch = reinterpret_cast<uint32_t*>(&sm.kv[0][0]) + warp * kScap;
    units::warp_settle_segment(s, lo, k - sm.start[lo] / s.L, step, scratch, kScap, opaque(1) != 0);
  }
  if (s.tl && (threadIdx.x & 31) == 0) atomicMax(&s.tl[2 * kStages], gtimer());
  // combine tasks (one warp per (b, l, h)), first on the warps without a tile
  const int C = s.B * s.L * s.Hq;
  if (o && !(s.tail_exp & 1))   // (ASR_TAIL_EXP bit 0: no combine — timing diagnostics only)
    for (int k = ((r - D) % NW + NW) % NW; k < C; k += NW) units::combine_warp_tail(s, k, o, opaque(1) != 0);
  if (s.tl && (threadIdx.x & 31) == 0) atomicMax(&s.tl[2 * kStages + 2], gtimer());
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s.tl) atomicMax(&s.tl[2 * 2 + 1], gtimer());
    // every CTA read *s.step at its start; the next kernel sees all writes of this one
    if (atomicAdd(s.ticket, 1) == gridDim.x - 1) {   // the last CTA out: the step is done
      *s.ticket = 0;
      *s.redo = 0;
      *s.step = step + 1;
    }
  }
}

// The attention kernel over A_i as phase D of the previous step compacted it.  With pre_in_attn
// (batch 1) the CTAs' extra warps also run phase A and B of the step; since recovery (phase B) may
// recompact A_i while the attention runs, every CTA then waits for phase B (*pre_done) and, only if
// recovery fired (*redo, rare), all CTAs pass a grid barrier and redo the attention over the new A_i.
// With fuse_tail the kernel then settles the step itself (fused_tail).
template <int HK, typename TL, bool DYN>
__global__ void __launch_bounds__(Geo<HK>::kThreads, 1)
    attn_mma_kernel(const __grid_constant__ DevState s, const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_new,
                    const __nv_bfloat16* __restrict__ v_new, const TL* logits, float* entropy_out, float* o) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  auto& sm = *reinterpret_cast<typename Geo<HK>::Smem*>(smem_raw);
  __shared__ units::UnitShm u;
  __shared__ int redo;
  attention_prologue<HK>(sm);
  pdl_wait();      // upstream results (phase A when it runs as its own kernel)
  pdl_trigger();
  const bool do_pre = s.pre_in_attn;
  const int step = *s.step;
  const long long c0 = clock64();
  {
    Stamp stamp(s.tl, 1);
    attention_phase<HK, TL, DYN>(s, q, k_new, v_new, sm, do_pre, logits, entropy_out, u, o);
    if (s.tl && threadIdx.x == 0) atomicMin(&s.tl[2 * kStages + 7], gtimer());   // first CTA done
  }
  if (!DYN && s.sk_bal && s.sk_learn && !do_pre) {
    __syncthreads();
    if (threadIdx.x == 0) sk_rate_update(s, step, sm.range, c0);
  }
  if (do_pre) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (!DYN && s.sk_bal && s.sk_learn) sk_rate_update(s, step, sm.range, c0);
      if (s.tl) atomicMax(&s.tl[kTlTail + 8], gtimer());   // every warp of the CTA is past the attention
      const unsigned long long t0 = gtimer();
      bool ok = true;
      while (ld_acquire(s.pre_done) != step + 1) {   // acquire: phase B's ledger / A_i writes
        __nanosleep(64);
        if (gtimer() - t0 > 2000000000ull) {   // 2 s: never on a healthy device; do not hang it
          atomicOr(s.err, kErrStall);
          ok = false;
          break;
        }
      }
      redo = ok ? *reinterpret_cast<const volatile int*>(s.redo) : 0;
      if (s.tl) atomicMax(&s.tl[kTlTail + 9], gtimer());
    }
    __syncthreads();
    if (redo) {
      grid_sync(s.gbar, s.err);    // every CTA is past its first pass
      attention_prologue<HK>(sm);  // fresh ring barriers
      attention_phase<HK, TL, DYN>(s, q, k_new, v_new, sm, false, logits, entropy_out, u, o);
    }
  }
  if (s.pool_mode) {   // the attention's end, against which the prefetch copies are timed
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&s.stall[1], gtimer());
  }
  if (s.fuse_tail) fused_tail<HK>(s, sm, step, o);
}

}  // namespace

template <int HK>
int gmax() { return Geo<HK>::kGMax; }

bool attention_mma_supported(const DevState& s) {
  if (s.dtype != 0 || s.d != kD || s.B > kMaxB || s.Hq % s.Hkv) return false;
  const int G = s.Hq / s.Hkv;
  switch (s.Hkv) {
    case 8: return G <= gmax<8>();
    case 4: return G <= gmax<4>();
    case 2: return G <= gmax<2>();
    case 1: return G <= gmax<1>();
    default: return false;
  }
}

template <int HK, bool DYN>
cudaError_t prep_one() {
  cudaError_t e = cudaFuncSetAttribute(attn_mma_kernel<HK, __nv_bfloat16, DYN>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(typename Geo<HK>::Smem));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(attn_mma_kernel<HK, float, DYN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(typename Geo<HK>::Smem));
}

cudaError_t attention_mma_prepare() {
  cudaError_t e;
  if ((e = prep_one<8, false>()) != cudaSuccess || (e = prep_one<8, true>()) != cudaSuccess ||
      (e = prep_one<4, false>()) != cudaSuccess || (e = prep_one<2, false>()) != cudaSuccess ||
      (e = prep_one<1, false>()) != cudaSuccess)
    return e;
  return cudaSuccess;
}

template <int HK, bool DYN>
void shape_of(bool lf, const void** func, int* threads, unsigned* smem) {
  *func = lf ? (const void*)attn_mma_kernel<HK, float, DYN> : (const void*)attn_mma_kernel<HK, __nv_bfloat16, DYN>;
  *threads = Geo<HK>::kThreads;
  *smem = sizeof(typename Geo<HK>::Smem);
}

// The dynamic work split (DevState::sk_dyn > 0) exists for 8 KV heads only (the host clears sk_dyn
// otherwise).
void attention_mma_launch_shape(const DevState& s, bool logits_f32, const void** func, int* threads, unsigned* smem) {
  switch (s.Hkv) {
    case 8:
      if (s.sk_dyn > 0) shape_of<8, true>(logits_f32, func, threads, smem);
      else shape_of<8, false>(logits_f32, func, threads, smem);
      break;
    case 4: shape_of<4, false>(logits_f32, func, threads, smem); break;
    case 2: shape_of<2, false>(logits_f32, func, threads, smem); break;
    default: shape_of<1, false>(logits_f32, func, threads, smem); break;
  }
}

}  // namespace asr
