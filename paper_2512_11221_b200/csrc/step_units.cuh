// paper_2512_11221_b200/csrc/step_units.cuh — the ledger-side work units of one ASR-KF-EGR step.
// A unit runs on a team of ASR_UNIT_THREADS() threads (a multiple of 32, <= 1024; team rank
// ASR_UNIT_TID()) that synchronise with ASR_UNIT_SYNC(): the whole block in kernels_ledger.cu, one
// dedicated warp of the attention CTA in kernels_attn_mma.cu (where phase A of a batch-1 step runs
// inside the attention kernel, beside the producer and consumer warps).
//
//   phase A  warp_entropy_split   (a6) partial (m, Z, S) of one split of a logits row (one warp)
//            unit_append          (a0) the new token's K/V rows of (b, l) -> its slot
//            unit_finish          (a6) H = ln Z - S/Z, detector (R-det), ladder (R-ladder) and, when
//                                 a level fires (rare), the level (Sec 3.6) + recompaction of A_i;
//                                 run by the last phase-A unit of the sequence
//   phase C  attention            (a4)+(a1) — kernels_attn_mma.cu / kernels_attn.cu (A_i is known before
//                                 the step; at batch 1 phase A runs inside the tensor-core kernel)
//   phase D  unit_decide          (a2) Eq. 2 finish, threshold, Eq. 3, freeze, R0 tick (Alg. 1 3-15)
//            unit_prepare         (a0) ledger entry of the next appended position, (a3) A_{i+1} — run
//                                 by the last decide block of the sequence
//            combine_warp         (a4') fixed-order combine of the split-KV partials -> O
// Floating-point reductions are in a fixed order, so a step is bitwise deterministic.
#pragma once
#ifndef ASR_UNIT_THREADS
#define ASR_UNIT_THREADS() blockDim.x
#define ASR_UNIT_TID() threadIdx.x
#define ASR_UNIT_SYNC() __syncthreads()
#endif
#include <cuda_bf16.h>
#include <math.h>

#include "asr_internal.h"

namespace asr {
namespace units {
namespace {   // internal linkage: this header is compiled into several translation units

struct UnitShm {
  int sh[32], sh2[32], wsum[32];
  int ev[kEvBins];   // decide: Belady histogram of this block's resident frozen tokens (pressure mode)
  float wm[32], wz[32], ws[32];
  int level;
  int total;
  int last;
  int lo, hi;   // decide: this block's position range
  int pref;     // head-sharded mode: offset of this sequence in the packed per-token partial sums
};

// Head-sharded mode: offset of sequence b's entries in the packed per-token partial sums (the prefix
// over |A_b'| of the step's lists), computed by one thread.
__device__ __forceinline__ int packed_offset(const DevState& s, int b, int i) {
  int acc = 0;
  for (int x = 0; x < b; ++x) acc += s.act_len[(i & 1) * s.B + x];
  return acc;
}

__device__ __forceinline__ float tof(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float tof(float v) { return v; }

template <typename T>
__device__ __forceinline__ void load8(const T* p, float* x);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float* x) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[2 * i] = __uint_as_float(w[i] << 16);
    x[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float* x) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
}

// ---------------------------------------------------------------------------------- (a5) slot pool
// Pressure mode (pool_tokens > 0): device token slots come from a free stack.  Pops happen only in
// phase B (and asr_restore), pushes only in phase D, so the stack never sees both at once.
__device__ __forceinline__ int pool_pop(const DevState& s) {
  const int idx = atomicSub(s.free_top, 1) - 1;
  if (idx < 0) {
    atomicAdd(s.free_top, 1);
    atomicOr(s.err, kErrPoolEmpty);
    return -1;
  }
  ASR_CHECK(s, idx < s.kv_slots);
  const int slot = s.free_stack[idx];
  ASR_CHECK(s, slot >= 0 && slot < s.kv_slots);
  return slot;
}
__device__ __forceinline__ void pool_push(const DevState& s, int slot) {
  const int idx = atomicAdd(s.free_top, 1);
  ASR_CHECK(s, idx >= 0 && idx < s.kv_slots && slot >= 0 && slot < s.kv_slots);
  s.free_stack[idx] = slot;
}
// ---------------------------------------------------------------------------------- (a5) INT8 tier
// NEXT-4 wired into the host link: with mirror_bits = 8 the write-once host mirror holds every row
// (token, layer, K|V, KV head; d values) as R-quant INT8 codes + one fp32 scale (DESIGN.md §2,
// oracle/quant.py): scale = RN(amax / 127), code = clamp(rint(RN(x / scale)), +-127) (IEEE fp32
// divisions, half-to-even), x' = bf16_rn(code * scale).  A restore moves d + 4 bytes per row instead of
// 2d (1.94x fewer at d = 128) and writes the dequantised row into the device slot.
// One warp quantises one row (d a multiple of 32, <= 256): lane e holds values e*(d/32) ...
__device__ __forceinline__ void quant_row8_warp(const __nv_bfloat16* __restrict__ x, int d, int8_t* codes,
                                                float* scale_out) {
  const int lane = threadIdx.x & 31;
  const int per = d >> 5;   // values per lane (1 .. 8)
  float v[8];
  float amax = 0.f;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    v[e] = e < per ? __bfloat162float(x[lane * per + e]) : 0.f;
    amax = fmaxf(amax, fabsf(v[e]));
  }
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float scale = __fdiv_rn(amax, 127.f);
#pragma unroll
  for (int e = 0; e < 8; ++e)
    if (e < per) {
      int c = 0;
      if (scale != 0.f) c = max(-127, min(127, __float2int_rn(__fdiv_rn(v[e], scale))));
      codes[lane * per + e] = (int8_t)c;
    }
  if (lane == 0) *scale_out = scale;
}

// Block-cooperative copy of one token (all layers, K and V) from the pinned host mirror (mapped,
// read over the host link) into its device slot (INT8 tier: dequantised on the way).
__device__ void copy_token_h2d(const DevState& s, int b, int pos, int slot) {
  if (slot < 0) return;
  ASR_CHECK(s, slot < s.kv_slots && pos >= 0 && pos < s.cap);
  if (s.mirror_bits == 8) {
    const int R = s.L * 2 * s.Hkv;                 // rows of the token
    const long r0 = ((long)b * s.max_ctx + pos) * R;
    const int per_row = s.d / 16;                  // 16 codes per item
    const int items = R * per_row;
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<char*>(s.kv) + (long)slot * s.tok_bytes);
    for (int t0 = (int)ASR_UNIT_TID(); t0 < items; t0 += 4 * (int)ASR_UNIT_THREADS()) {
      uint4 cw[4];
      float sc[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {   // the items' codes and scales in flight over the host link
        const int t = min(t0 + k * (int)ASR_UNIT_THREADS(), items - 1);
        const int r = t / per_row, c = t % per_row;
        cw[k] = *reinterpret_cast<const uint4*>(s.host_codes + (r0 + r) * s.d + c * 16);
        sc[k] = s.host_scales[r0 + r];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int t = t0 + k * (int)ASR_UNIT_THREADS();
        if (t >= items) break;
        const int r = t / per_row, c = t % per_row;
        const uint32_t w[4] = {cw[k].x, cw[k].y, cw[k].z, cw[k].w};
        uint32_t o[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int c0 = (int)(int8_t)(w[q >> 1] >> (16 * (q & 1)));
          const int c1 = (int)(int8_t)(w[q >> 1] >> (16 * (q & 1) + 8));
          const __nv_bfloat162 h = __floats2bfloat162_rn((float)c0 * sc[k], (float)c1 * sc[k]);
          o[q] = *reinterpret_cast<const uint32_t*>(&h);
        }
        uint4* d4 = reinterpret_cast<uint4*>(dst + (long)r * s.d + c * 16);
        d4[0] = make_uint4(o[0], o[1], o[2], o[3]);
        d4[1] = make_uint4(o[4], o[5], o[6], o[7]);
      }
    }
    if (ASR_UNIT_TID() == 0) {
      atomicAdd(s.h2d, (unsigned long long)R * (s.d + 4));
      s.deq[(long)b * s.max_ctx + pos] = 1;
    }
    return;
  }
  const uint4* src = reinterpret_cast<const uint4*>(s.host_kv + ((long)b * s.max_ctx + pos) * s.tok_bytes);
  uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<char*>(s.kv) + (long)slot * s.tok_bytes);
  const int nv = (int)(s.tok_bytes / 16);
  for (int v0 = (int)ASR_UNIT_TID(); v0 < nv; v0 += 8 * (int)ASR_UNIT_THREADS()) {
    uint4 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int v = v0 + k * (int)ASR_UNIT_THREADS();
      if (v < nv) x[k] = src[v];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int v = v0 + k * (int)ASR_UNIT_THREADS();
      if (v < nv) dst[v] = x[k];
    }
  }
  if (ASR_UNIT_TID() == 0) atomicAdd(s.h2d, (unsigned long long)s.tok_bytes);
}

// ---------------------------------------------------------------------------------- (a6) entropy
// merge (m, Z, S) triples of the single-pass entropy (Z = sum e^{x-m}, S = sum e^{x-m}(x-m)),
// rescaled to M = max(m, om)
__device__ __forceinline__ void tri_merge(float& m, float& z, float& sx, float om, float oz, float os) {
  const float M = fmaxf(m, om);
  float nz = 0.f, ns = 0.f;
  if (z > 0.f) { const float f = __expf(m - M); nz += z * f; ns += f * (sx + z * (m - M)); }
  if (oz > 0.f) { const float f = __expf(om - M); nz += oz * f; ns += f * (os + oz * (om - M)); }
  m = M; z = nz; sx = ns;
}

// Partial (m, Z, S) of split `split` of row b's logits, computed by one warp (lane = lane index).
template <typename TL>
__device__ void warp_entropy_split(const DevState& s, const TL* __restrict__ logits, int b, int split, int lane) {
  const int V = s.vocab;
  const int seg = (((V + kEntSplits - 1) / kEntSplits) + 7) & ~7;   // multiple of 8 elements
  const int e0 = min(V, split * seg), e1 = min(V, e0 + seg);
  const TL* row = logits + (long)(b / s.ent_div) * V;   // per-layer ledgers: the sequence's row
  const bool vecok = (reinterpret_cast<uintptr_t>(row) & 31) == 0;
  const float invT = 1.0f / s.ent_temp;
  float m = -INFINITY, z = 0.f, sx = 0.f;
  auto accum = [&](float* x) {   // fold 8 logits into the running (m, Z, S)
    float mx = -INFINITY;
#pragma unroll
    for (int e = 0; e < 8; ++e) { x[e] *= invT; mx = fmaxf(mx, x[e]); }
    if (mx > m) {   // rescale the running sums to the new max
      if (z > 0.f) { const float f = __expf(m - mx); sx = f * (sx + z * (m - mx)); z *= f; }
      m = mx;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float d = x[e] - m;
      const float ex = __expf(d);
      z += ex;
      sx += ex > 0.f ? ex * d : 0.f;
    }
  };
  if (!vecok) {
    for (int v = e0 + lane * 8; v < e1; v += 32 * 8) {
      float x[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = (v + e < e1) ? tof(row[v + e]) : -INFINITY;
      accum(x);
    }
  } else {
    // all kIn 16-byte loads of a batch are issued before any is consumed (unconditional, clamped
    // addresses): a branch between them would make each wait for the previous one
    constexpr int kIn = 8;
    constexpr int kW = sizeof(TL) == 2 ? 1 : 2;   // 16-byte words per 8 logits
    for (int v0 = e0 + lane * 8; v0 < e1; v0 += kIn * 32 * 8) {
      uint4 raw[kIn][kW];
#pragma unroll
      for (int k = 0; k < kIn; ++k) {
        const int v = v0 + k * 32 * 8;
        const uint4* src = reinterpret_cast<const uint4*>(row + (v + 8 <= e1 ? v : e0));
#pragma unroll
        for (int w = 0; w < kW; ++w) raw[k][w] = __ldg(src + w);
      }
#pragma unroll 1
      for (int k = 0; k < kIn; ++k) {
        const int v = v0 + k * 32 * 8;
        if (v >= e1) break;
        float x[8];
        if (v + 8 <= e1) {
          if constexpr (sizeof(TL) == 2) {
            const uint32_t w4[4] = {raw[k][0].x, raw[k][0].y, raw[k][0].z, raw[k][0].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              x[2 * q] = __uint_as_float(w4[q] << 16);
              x[2 * q + 1] = __uint_as_float(w4[q] & 0xffff0000u);
            }
          } else {
            const uint32_t w8[8] = {raw[k][0].x, raw[k][0].y, raw[k][0].z, raw[k][0].w,
                                    raw[k][kW - 1].x, raw[k][kW - 1].y, raw[k][kW - 1].z, raw[k][kW - 1].w};
#pragma unroll
            for (int q = 0; q < 8; ++q) x[q] = __uint_as_float(w8[q]);
          }
        } else {   // the row's last, partial group of 8
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = (v + e < e1) ? tof(row[v + e]) : -INFINITY;
        }
        accum(x);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1)
    tri_merge(m, z, sx, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, z, o),
              __shfl_xor_sync(0xffffffffu, sx, o));
  if (lane == 0) {
    float* ep = s.ent_part + ((long)b * kEntSplits + split) * 3;
    ep[0] = m; ep[1] = z; ep[2] = sx;
  }
}

// ---------------------------------------------------------------------------------- (a3) compaction
// A_i = sorted Active positions into the parity-p lists.  A team compacts the positions [lo, hi) of
// a row (lo a multiple of 128) in 128-position groups: lane k of a warp reads the 4 residency bytes of
// positions 4k..4k+3 of a group (one coalesced 128-byte load per group); a warp scan of the per-lane
// counts gives every lane its output offset, so the writes of a group are contiguous too.
// Residency (and slots) are read through L2 (ld.global.cg): other blocks of the same kernel wrote
// them (decide slices, recovery), and this block's L1 may hold older lines.
__device__ __forceinline__ uint32_t active_bits4(const uint32_t* res4, int q, int lo, int n) {
  // bit k set iff position 4q + k in [lo, n) is Active (residency byte == 1); the load is
  // unconditional (clamped address) so a caller's batch of these issues all loads back to back
  const bool in = 4 * q < n && 4 * q + 4 > lo;
  const uint32_t e = __vcmpeq4(__ldcg(res4 + (in ? q : (lo >> 2))), 0x01010101u);   // 0xff per byte == 1
  if (!in) return 0u;
  uint32_t m = ((e >> 7) & 1u) | ((e >> 14) & 2u) | ((e >> 21) & 4u) | ((e >> 28) & 8u);
  const int left = n - 4 * q;
  if (left < 4) m &= (1u << left) - 1u;
  if (lo > 4 * q) m &= ~((1u << (lo - 4 * q)) - 1u);
  return m;
}

struct Compactor {
#ifndef ASR_KKEEP
#define ASR_KKEEP 1   // measured: 8 -> 1 saves ~2 us of the batch-1 phase D (code size), batch 64 unchanged
#endif
  static constexpr int kKeep = ASR_KKEEP;   // masks of a warp's first kKeep groups stay in registers
  const uint32_t* res4;
  int lo, hi, g0, g1, lo_al;
  uint32_t keep[kKeep];
  // count pass over [lo_, hi_): returns the team's total; u.wsum[w] = exclusive offset of warp w
  __device__ int count(const DevState& s, int b, int lo_, int hi_, UnitShm& u) {
    res4 = reinterpret_cast<const uint32_t*>(s.res + (long)b * s.max_ctx);   // rows are 64-byte aligned
    lo = lo_;
    hi = hi_;
    lo_al = lo & ~127;   // groups are 128-position aligned; positions below lo are masked
    const int tid = (int)ASR_UNIT_TID(), lane = tid & 31, w = tid >> 5, nw = (int)ASR_UNIT_THREADS() >> 5;
    const int ngrp = hi > lo ? (hi - lo_al + 127) >> 7 : 0;
    const int per = (ngrp + nw - 1) / nw;
    g0 = min(ngrp, w * per);
    g1 = min(ngrp, g0 + per);
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < kKeep; ++k) {
      keep[k] = g0 + k < g1 ? active_bits4(res4, (lo_al >> 2) + (g0 + k) * 32 + lane, lo, hi) : 0u;
      cnt += __popc(keep[k]);
    }
#pragma unroll 4
    for (int g = g0 + kKeep; g < g1; ++g) cnt += __popc(active_bits4(res4, (lo_al >> 2) + g * 32 + lane, lo, hi));
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) u.wsum[w] = cnt;
    ASR_UNIT_SYNC();
    if (w == 0) {
      const int x = lane < nw ? u.wsum[lane] : 0;
      int xi = x;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, xi, o);
        if (lane >= o) xi += y;
      }
      u.wsum[lane] = xi - x;  // exclusive warp offsets
      if (lane == 31) u.total = xi;
    }
    ASR_UNIT_SYNC();
    return u.total;
  }
  // write pass: the team's positions go to compact indices base, base + 1, ... of the parity-p lists
  __device__ void write(const DevState& s, int b, int p, int base_idx, const UnitShm& u) {
    const int tid = (int)ASR_UNIT_TID(), lane = tid & 31, w = tid >> 5;
    const long row = (long)b * s.max_ctx;
    int32_t* out = s.act_pos + act_off(s, p) + row;
    int32_t* out_slot = s.act_slot + act_off(s, p) + row;
    const int32_t* slot_of = s.slot_of + row;
    int off = base_idx + u.wsum[w];
    for (int g = g0; g < g1; ++g) {
      const int q = (lo_al >> 2) + g * 32 + lane;
      uint32_t m = 0u;
      if (g - g0 < kKeep) {
#pragma unroll
        for (int k = 0; k < kKeep; ++k)
          if (g - g0 == k) m = keep[k];
      } else {
        m = active_bits4(res4, q, lo, hi);
      }
      const int c = __popc(m);
      int incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int o = off + incl - c;
      while (m) {
        const int j = 4 * q + __ffs(m) - 1;
        ASR_CHECK(s, o >= 0 && o < s.max_ctx && j < s.max_ctx);
        out[o] = j;
        out_slot[o] = s.pool_mode ? __ldcg(slot_of + j) : (int)(row + j);
        ++o;
        m &= m - 1;
      }
      off += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
};

// A_i of [0, n) by one team.
__device__ void compact_positions(const DevState& s, int b, int n, int p, UnitShm& u) {
  Compactor c;
  const int total = c.count(s, b, 0, n, u);
  c.write(s, b, p, 0, u);
  if (ASR_UNIT_TID() == 0) {
    s.act_len[(p & 1) * s.B + b] = total;
    if (total == 0) atomicOr(s.err, kErrEmptyActive);
  }
  ASR_UNIT_SYNC();
}

// Ledger entry of position j = the token step i appends (Alg. 1 line 16 of the previous step:
// Active, c = 0, timer 0, its reserved slot in pressure mode).
__device__ __forceinline__ void ledger_entry_new(const DevState& s, int b, int j) {
  const long k = (long)b * s.max_ctx + j;
  s.res[k] = 1;
  s.timer[k] = 0;
  s.count[k] = 0;
  s.fstep[k] = -1;
  if (s.pool_mode) s.slot_of[k] = s.spare[b];   // the slot reserved by phase B
}

// At asr_create: the ledger entry of the position step 0 appends and A_0 (parity 0).
__device__ void unit_prepare(const DevState& s, int b, UnitShm& u) {
  const int n = s.prompt_len[b] + 1;  // tokens after step 0's append
  if (n > s.cap) return;
  if (ASR_UNIT_TID() == 0) ledger_entry_new(s, b, n - 1);
  ASR_UNIT_SYNC();
  compact_positions(s, b, n, 0, u);
}

template <typename TK>
__device__ void unit_append(const DevState& s, int b, int l, int i, const TK* __restrict__ k_new,
                            const TK* __restrict__ v_new) {
  const long pos = s.prompt_len[b] + i;
  const long slot = s.pool_mode ? (long)s.spare[b] : (long)b * s.max_ctx + pos;
  if (slot < 0) return;   // pool exhausted (latched by the pop)
  ASR_CHECK(s, slot < s.kv_slots && pos < s.cap);
  const int row = s.Hkv * s.d;  // elements of K (or V) per token-layer
  TK* dst = reinterpret_cast<TK*>(s.kv) + (slot * s.L + l) * 2 * row;
  // pressure mode: the write-once host mirror is written here too (mapped pinned memory), so a
  // token's bytes are off-GPU before it can ever be evicted (INT8 tier: quantised rows, below)
  TK* mir = s.pool_mode && s.mirror_bits == 0
                ? reinterpret_cast<TK*>(s.host_kv) + (((long)b * s.max_ctx + pos) * s.L + l) * 2 * row
                : nullptr;
  const TK* ks = k_new + ((long)b * s.L + l) * row;
  const TK* vs = v_new + ((long)b * s.L + l) * row;
  if constexpr (sizeof(TK) == 2) {
    if (s.pool_mode && s.mirror_bits == 8) {   // one warp per row: 2 * Hkv rows of d for this (b, l)
      const long r0 = (((long)b * s.max_ctx + pos) * s.L + l) * 2 * s.Hkv;
      const int nw = (int)ASR_UNIT_THREADS() >> 5, w = (int)ASR_UNIT_TID() >> 5;
      for (int r = w; r < 2 * s.Hkv; r += nw) {
        const TK* x = (r < s.Hkv ? ks : vs) + (long)(r % s.Hkv) * s.d;
        quant_row8_warp(reinterpret_cast<const __nv_bfloat16*>(x), s.d, s.host_codes + (r0 + r) * s.d,
                        s.host_scales + r0 + r);
      }
    }
  }
  const int vec = (int)(16 / sizeof(TK));
  if (row % vec == 0) {
    const int nv = row / vec;
    const int T = (int)ASR_UNIT_THREADS();
    for (int t0 = ASR_UNIT_TID(); t0 < 2 * nv; t0 += 8 * T) {   // 8 vectors in flight per thread
      uint4 x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int t = t0 + k * T;
        if (t < 2 * nv) x[k] = __ldg(reinterpret_cast<const uint4*>(t < nv ? ks : vs) + (t < nv ? t : t - nv));
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int t = t0 + k * T;
        if (t < 2 * nv) {
          reinterpret_cast<uint4*>(dst)[t] = x[k];
          if (mir) reinterpret_cast<uint4*>(mir)[t] = x[k];
        }
      }
    }
  } else {
    for (int t = ASR_UNIT_TID(); t < 2 * row; t += ASR_UNIT_THREADS()) {
      const TK x = t < row ? ks[t] : vs[t - row];
      dst[t] = x;
      if (mir) mir[t] = x;
    }
  }
}

// Layers [l0, l1) of sequence b's new token at once (full residency, no mirror write here, 16-byte
// rows): one flat loop over every 16-byte vector of those layers, 8 loads in flight per thread — a
// unit of several layers is then one or two memory round trips instead of one per layer (batch 64:
// 16 layers per unit; the per-layer loop left phase A's appends ending ~11 us after its entropy units).
template <typename TK>
__device__ void unit_append_layers(const DevState& s, int b, int l0, int l1, int i, const TK* __restrict__ k_new,
                                   const TK* __restrict__ v_new) {
  const long pos = s.prompt_len[b] + i;
  const long slot = (long)b * s.max_ctx + pos;
  ASR_CHECK(s, slot < s.kv_slots && pos < s.cap);
  const int row = s.Hkv * s.d;
  const int nv = row * (int)sizeof(TK) / 16;   // 16-byte vectors per K (or V) row of a layer
  const int per_l = 2 * nv;
  const int total = (l1 - l0) * per_l;
  const int T = (int)ASR_UNIT_THREADS();
  uint4* dst0 = reinterpret_cast<uint4*>(reinterpret_cast<TK*>(s.kv) + (slot * s.L + l0) * 2 * row);   // layers contiguous
  for (int t0 = ASR_UNIT_TID(); t0 < total; t0 += 8 * T) {
    uint4 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int t = t0 + k * T;
      if (t < total) {
        const int l = l0 + t / per_l, r = t % per_l;
        const TK* src = (r < nv ? k_new : v_new) + ((long)b * s.L + l) * row;
        x[k] = __ldg(reinterpret_cast<const uint4*>(src) + (r < nv ? r : r - nv));
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int t = t0 + k * T;
      if (t < total) dst0[t] = x[k];
    }
  }
}

// Recovery levels on one sequence's ledger over positions [0, n): returns this thread's
// restored count.  SR: frozen with d > 1; WR: frozen at step >= i - N; FR: every frozen token.
__device__ int apply_level(const DevState& s, int b, int n, int level, int i) {
  int restored = 0;
  uint8_t* res = s.res + (long)b * s.max_ctx;
  int32_t* timer = s.timer + (long)b * s.max_ctx;
  const int32_t* fstep = s.fstep + (long)b * s.max_ctx;
  for (int j = ASR_UNIT_TID(); j < n; j += ASR_UNIT_THREADS()) {
    if (res_active(res[j])) continue;
    bool go = level == 1 ? timer[j] > 1 : level == 2 ? fstep[j] >= i - s.wr_window : true;
    if (go) {
      res[j] = 1;
      timer[j] = 0;
      restored++;
      if (s.pool_mode && s.slot_of[(long)b * s.max_ctx + j] < 0) {   // evicted: copy back on demand
        s.slot_of[(long)b * s.max_ctx + j] = pool_pop(s);
        s.cp_list[(long)b * s.max_ctx + atomicAdd(&s.cp_count[b], 1)] = j;
      }
    }
  }
  if (level >= 3 && s.fr_clear_counts) {
    uint32_t* cnt = s.count + (long)b * s.max_ctx;
    for (int j = ASR_UNIT_TID(); j < n; j += ASR_UNIT_THREADS()) {
      cnt[j] = 0;
      if (s.hist_w > 0) {
        s.hmask[((long)b * s.max_ctx + j) * 2] = 0;
        s.hmask[((long)b * s.max_ctx + j) * 2 + 1] = 0;
      }
    }
  }
  return restored;
}

// Copy back (synchronously, whole block) every token apply_level listed for sequence b; returns
// the count.  Runs with no concurrent pushes (phase B / asr_restore).
__device__ int demand_copies(const DevState& s, int b) {
  ASR_UNIT_SYNC();
  const int nd = s.cp_count[b];
  for (int k = 0; k < nd; ++k) {
    const int j = s.cp_list[(long)b * s.max_ctx + k];
    copy_token_h2d(s, b, j, s.slot_of[(long)b * s.max_ctx + j]);
  }
  ASR_UNIT_SYNC();
  if (ASR_UNIT_TID() == 0) s.cp_count[b] = 0;
  ASR_UNIT_SYNC();
  return nd;
}

__device__ int block_sum_int(int v, UnitShm& u) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = ASR_UNIT_TID() >> 5, lane = ASR_UNIT_TID() & 31, nw = ASR_UNIT_THREADS() >> 5;
  ASR_UNIT_SYNC();
  if (lane == 0) u.sh[w] = v;
  ASR_UNIT_SYNC();
  int t = 0;
  for (int k = 0; k < nw; ++k) t += u.sh[k];
  ASR_UNIT_SYNC();
  return t;
}

// Phase B for sequence b: entropy of logits_prev (if given), detector, ladder, recovery.
__device__ void unit_finish(const DevState& s, int b, int i, bool has_logits, float* entropy_out, UnitShm& u) {
  const int lane = ASR_UNIT_TID() & 31, w = ASR_UNIT_TID() >> 5;
  if (ASR_UNIT_TID() == 0) {   // per-step counters (phase D of this step adds to them)
    if (s.pool_mode) {
      s.cp_count[b] = 0;                              // the previous step's copies are done
      s.pf_count[(i & 1) * s.B + b] = 0;              // this step's decide fills list i & 1
    }
    SeqStats& st = s.stats[b];
    st.evicted = 0;
    st.demand = st.pending_demand;
    st.pending_demand = 0;
    st.restored_pre = st.pending_restored;
    st.pending_restored = 0;
    st.restored_tick = 0;
    st.frozen_this_step = 0;
  }
  if (w == 0) {
    int level = 0;
    if (has_logits) {
      float H;
      if (s.ent_given) {   // the caller's H (asr_sample_entropy took it in its pass over the row)
        H = __ldcg(s.ent_given + b / s.ent_div);
      } else {
        // merge the kEntSplits partials in fp32 (lane k holds splits k and k + 32; fixed-order tree)
        const float* ep = s.ent_part + (long)b * kEntSplits * 3;   // written by other blocks: via L2
        float M = -INFINITY, Zl = 0.f, Sl = 0.f;
        float pv[kEntSplits / 32][3];   // all loads first, then the merges
#pragma unroll
        for (int k = 0; k < kEntSplits / 32; ++k)
#pragma unroll
          for (int c = 0; c < 3; ++c) pv[k][c] = __ldcg(ep + (k * 32 + lane) * 3 + c);
#pragma unroll
        for (int k = 0; k < kEntSplits / 32; ++k) tri_merge(M, Zl, Sl, pv[k][0], pv[k][1], pv[k][2]);
        for (int o = 16; o > 0; o >>= 1)
          tri_merge(M, Zl, Sl, __shfl_xor_sync(0xffffffffu, M, o), __shfl_xor_sync(0xffffffffu, Zl, o),
                    __shfl_xor_sync(0xffffffffu, Sl, o));
        H = logf(Zl) - Sl / Zl;
      }
      DetState& ds = s.det[b];
      double* hist = s.hist + (long)b * s.det_baseline;
      const int hl = ds.hist_len;
      // detector statistics over the previous <= det_baseline entropies (fp32 is ample: the decision
      // margin of R-det is >= 0.5 nats on the generator's rows and sigma_floor is 0.05)
      const float hv0 = lane < hl ? (float)hist[lane] : 0.f;
      const float hv1 = lane + 32 < hl ? (float)hist[lane + 32] : 0.f;
      float mu = hv0 + hv1;
      for (int t = lane + 64; t < hl; t += 32) mu += (float)hist[t];
      for (int o = 16; o > 0; o >>= 1) mu += __shfl_xor_sync(0xffffffffu, mu, o);
      mu = hl > 0 ? mu / hl : 0.f;
      float var = (lane < hl ? (hv0 - mu) * (hv0 - mu) : 0.f) + (lane + 32 < hl ? (hv1 - mu) * (hv1 - mu) : 0.f);
      for (int t = lane + 64; t < hl; t += 32) var += ((float)hist[t] - mu) * ((float)hist[t] - mu);
      for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
      if (lane == 0) {
        var = hl > 0 ? var / hl : 0.f;
        int trig = 0;
        if (s.det_enable && hl >= 2) {
          const float sd = fmaxf(sqrtf(var), s.det_sigma_floor);
          trig = H > mu + s.det_z * sd;   // detector: H > mean + z * max(sigma, floor)
        }
        if (hl < s.det_baseline) {
          hist[hl] = H;
          ds.hist_len = hl + 1;
        } else {
          hist[ds.hist_head] = H;
          ds.hist_head = (ds.hist_head + 1) % s.det_baseline;
        }
        if (trig) {
          const int dt = i - ds.last_action_step;
          if (!(ds.has_last && dt < s.det_cooldown)) {   // absorbed inside the cooldown
            level = (ds.has_last && dt < 2 * s.det_cooldown) ? (ds.level < 4 ? ds.level + 1 : 4) : 1;
            ds.level = level;
            ds.last_action_step = i;
            ds.has_last = 1;
          }
        }
        if (entropy_out && b % s.ent_div == 0) entropy_out[b / s.ent_div] = H;
        s.stats[b].entropy = H;
      }
    }
    if (lane == 0) u.level = level;
  }
  ASR_UNIT_SYNC();
  const int level = u.level;
  int restored = 0, demand = 0;
  if (level > 0) {   // rare: apply the level (copy evicted tokens back), then recompact A_i
    const int n = s.prompt_len[b] + i + 1;
    restored = block_sum_int(apply_level(s, b, n - 1, level, i), u);
    if (s.pool_mode) {
      const unsigned long long t0 = gtimer();
      demand = demand_copies(s, b);
      if (ASR_UNIT_TID() == 0 && demand) atomicAdd(&s.stall[0], gtimer() - t0);   // the step waits on these
    }
    compact_positions(s, b, n, i, u);
    if (ASR_UNIT_TID() == 0) *s.redo = 1;   // a speculative attention pass over the old A_i is void
  }
  int prefetched = 0;
  if (s.pool_mode) {
    // tokens whose timer reached 1 in the previous step's tick are restored by this step's tick
    // and attended next step: give them slots now; the copy kernel fills them during this step
    const int r = ((i + 1) & 1) * s.B + b;
    const int np = i > 0 ? s.pf_count[r] : 0;
    const int32_t* pl = s.pf_list + (long)r * s.max_ctx;
    int32_t* slot_of = s.slot_of + (long)b * s.max_ctx;
    for (int k = ASR_UNIT_TID(); k < np; k += ASR_UNIT_THREADS()) {
      const int j = pl[k];
      if (slot_of[j] >= 0) continue;   // already back (recovery demand copy)
      slot_of[j] = pool_pop(s);
      s.cp_list[(long)b * s.max_ctx + atomicAdd(&s.cp_count[b], 1)] = j;
    }
    ASR_UNIT_SYNC();
    prefetched = s.cp_count[b];
    if (ASR_UNIT_TID() == 0) s.spare[b] = pool_pop(s);   // slot of the token the next step appends
  }
  if (ASR_UNIT_TID() == 0) {
    SeqStats& st = s.stats[b];
    st.prefetched = prefetched;
    st.demand += demand;
    st.restored_rec = restored;
    st.recovery_action = level;
    st.rewalk_requested = level == 4;
    st.entropy_valid = has_logits ? 1 : 0;
    st.attended = s.act_len[(i & 1) * s.B + b];
  }
}

// ---------------------------------------------------------------------------------- (a2) decide
__device__ __forceinline__ uint32_t isqrt_u32(uint32_t c) {
  uint32_t r = (uint32_t)sqrtf((float)c);
  while ((uint64_t)r * r > c) --r;
  while ((uint64_t)(r + 1) * (r + 1) <= c) ++r;
  return r;
}

// Eq. 3: d = floor(sqrt(c) / k) (exact, worked values P:72).
__device__ __forceinline__ int duration(uint32_t c, float k, int kint) {
  if (kint > 0) return (int)(isqrt_u32(c) / (uint32_t)kint);
  const double kd = k;
  int m = (int)(sqrt((double)c) / kd);
  while (m > 0 && ((double)m * kd) * ((double)m * kd) > (double)c) --m;
  while (((double)(m + 1) * kd) * ((double)(m + 1) * kd) <= (double)c) ++m;
  return m;
}

// Eq. 2 numerator of attended index a: sum over layers in order l = 0..L-1 of the per-layer head sums
// (the loads of up to 32 layers are issued before the first add, so their latencies overlap).
__device__ __forceinline__ float layer_sum(const DevState& s, int b, int a) {
  // unconditional loads from clamped (always valid) addresses: straight-line code, no branch per load
  const float* sp = s.score_part + (long)b * s.L * s.max_ctx + a;
  float sum = 0.f;
  for (int l0 = 0; l0 < s.L; l0 += 32) {
    float v[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = __ldcg(sp + (long)min(l0 + q, s.L - 1) * s.max_ctx);
#pragma unroll
    for (int q = 0; q < 32; ++q) sum += l0 + q < s.L ? v[q] : 0.f;
  }
  return sum;
}

// Head-sharded mode: this shard's per-token sums (its heads, all layers) for a slice of A_b, packed
// at prefix_b + a (the all-reduce then moves 4 bytes per attended token: 4 * sum_b |A_b|); unit 0 of
// sequence 0 publishes the count for the host (mapped pinned memory).
__device__ void unit_score_sum(const DevState& s, int b, int x, int X, int i, UnitShm& u) {
  const int A = s.act_len[(i & 1) * s.B + b];
  if (ASR_UNIT_TID() == 0) {
    u.pref = packed_offset(s, b, i);
    if (b == 0 && x == 0 && s.tok_count) *(volatile int32_t*)s.tok_count = packed_offset(s, s.B, i);
  }
  ASR_UNIT_SYNC();
  const int per_a = (A + X - 1) / X;
  const int a_end = min(A, (x + 1) * per_a);
  for (int a = x * per_a + ASR_UNIT_TID(); a < a_end; a += ASR_UNIT_THREADS())
    s.tok_score[u.pref + a] = layer_sum(s, b, a);
}

// Alg. 1 lines 3-9 (+ the R0 tick of a token frozen now) for attended index a (position j) of
// sequence b at step i; returns through the counters.  Shared by the decide block (unit_decide) and
// the fused tail's tile decide (warp_decide_tile).
struct DecideCtx {
  long base;
  uint8_t tag_now;
  float heads, sqrt_d;
  int n, pf_row;
  int pref;   // head-sharded mode: offset of the sequence in the packed partial sums
};
__device__ __forceinline__ DecideCtx decide_ctx(const DevState& s, int b, int i) {
  DecideCtx c;
  c.base = (long)b * s.max_ctx;
  c.tag_now = res_tag(i);
  c.heads = (float)(s.L * s.score_heads);   // Eq. 2's H over all layers (R-layer)
  c.sqrt_d = sqrtf((float)s.d);
  c.n = s.prompt_len[b] + i + 1;
  c.pf_row = (i & 1) * s.B + b;            // prefetch list written by this step (pressure mode)
  c.pref = 0;
  return c;
}

// ev (pressure mode, Belady policy): shared histogram of the remaining timers of resident frozen
// tokens (the eviction candidates of this step, cut after phase D: asr.cpp / evict_kernel).
__device__ __forceinline__ void decide_token(const DevState& s, const DecideCtx& c, int b, int a, int j, int i,
                                             int& frozen_now, int& restored, int& evicted, int* ev = nullptr) {
  const long base = c.base;
  ASR_CHECK(s, j >= 0 && j < c.n && a >= 0 && a < s.max_ctx);
  float sj;
  if (s.ext_score) {
    sj = s.ext_score[(long)b * s.cap + j];   // policy replay: the caller's s_j, rows of max_context
  } else {
    const float sum = s.sharded ? s.tok_score[c.pref + a] : layer_sum(s, b, a);
    sj = sum / c.heads;               // mean over the L*Hq (layer, head) pairs (correctly rounded)
    if (s.score_scaled) sj = sj / c.sqrt_d;
  }
  s.score[base + a] = sj;
  if (!(j < c.n - s.window && j >= s.pinned && sj < s.tau)) return;
  uint32_t cc;                        // line 4: c_j <- c_j + 1 (lifetime, or within the window W)
  if (s.hist_w > 0) {
    // finite W: a 128-bit history of detections, bit t = step hstep - t; shift it to step
    // i, record this detection, keep the bits of (i - W, i] and count them
    unsigned long long* hm = s.hmask + (base + j) * 2;
    const int sh = i - s.hstep[base + j];
    unsigned long long lo = hm[0], hi = hm[1];
    if (sh >= 128) {
      lo = hi = 0;
    } else if (sh >= 64) {
      hi = lo << (sh - 64);
      lo = 0;
    } else if (sh > 0) {
      hi = (hi << sh) | (lo >> (64 - sh));
      lo <<= sh;
    }
    lo |= 1ull;
    if (s.hist_w < 64) {
      lo &= (1ull << s.hist_w) - 1ull;
      hi = 0;
    } else if (s.hist_w < 128) {
      hi &= (1ull << (s.hist_w - 64)) - 1ull;
    }
    hm[0] = lo;
    hm[1] = hi;
    s.hstep[base + j] = i;
    cc = (uint32_t)(__popcll(lo) + __popcll(hi));
    s.count[base + j] = cc;
  } else {
    cc = s.count[base + j] + 1;
    s.count[base + j] = cc;
  }
  const int dd = duration(cc, s.softness, s.softness_int);  // line 5
  if (dd <= 0) return;
  frozen_now++;                       // lines 6-7
  s.fstep[base + j] = i;
  const int t = s.tick_skip_new ? dd : dd - 1;   // R0: this step's tick applies too
  if (t <= 0) {
    s.timer[base + j] = 0;            // frozen and restored by the same tick (no absence)
    restored++;
    return;
  }
  s.timer[base + j] = t;
  s.res[base + j] = c.tag_now;
  if (s.pool_mode && t >= s.evict_min && s.slot_of[base + j] >= 0) {   // (a5) offload
    if (s.evict_policy == ASR_EVICT_AT_FREEZE) {
      pool_push(s, s.slot_of[base + j]);
      s.slot_of[base + j] = -1;
      evicted++;
      if (t == 1)   // back at the next step's tick (evict_min = 1): prefetch it
        s.pf_list[(long)c.pf_row * s.max_ctx + atomicAdd(&s.pf_count[c.pf_row], 1)] = j;
    } else if (ev) {
      atomicAdd(&ev[min(t, kEvBins - 1)], 1);   // a Belady candidate (returns in t + 1 steps)
    }
  }
}

// Alg. 1 lines 10-15 for position j, frozen before this step (residency r, timer tm at step start);
// tokens of A_i (r == 1, or this step's tag) are skipped.
__device__ __forceinline__ void tick_position(const DevState& s, const DecideCtx& c, int j, uint8_t r, int tm,
                                              int& restored, uint32_t& err, int* ev = nullptr) {
  if (r == 1 || r == c.tag_now) return;
  const long base = c.base;
  const int t = tm - 1;
  if (t <= 0) {
    s.res[base + j] = 1;
    s.timer[base + j] = 0;
    restored++;
    if (s.pool_mode && s.slot_of[base + j] < 0) err |= kErrNotResident;
  } else {
    s.timer[base + j] = t;
    if (r != 0) s.res[base + j] = 0;           // drop the previous step's tag
    if (j >= c.n - s.window) err |= kErrFrozenInWindow;
    if (s.pool_mode) {
      const int so = s.slot_of[base + j];
      if (t == 1 && so < 0)   // back next step: prefetch it
        s.pf_list[(long)c.pf_row * s.max_ctx + atomicAdd(&s.pf_count[c.pf_row], 1)] = j;
      else if (ev && so >= 0 && t >= s.evict_min)
        atomicAdd(&ev[min(t, kEvBins - 1)], 1);   // a Belady candidate
    }
  }
}

// Unit x of X for sequence b: a slice of the attended list (Alg. 1 lines 3-9 + the R0 tick of the
// tokens it freezes) and a slice of the positions (lines 10-15 for tokens frozen at earlier steps).
// The two index sets are disjoint (A_i = the tokens Active at the step start) and tokens frozen in
// this step carry the step-parity tag res_tag(i), so units need no ordering between them.
__device__ void unit_decide(const DevState& s, int b, int x, int X, int i, UnitShm& u) {
  DecideCtx dc = decide_ctx(s, b, i);
  if (s.sharded) {
    if (ASR_UNIT_TID() == 0) u.pref = packed_offset(s, b, i);
    ASR_UNIT_SYNC();
    dc.pref = u.pref;
  }
  const int n = dc.n;
  const long base = dc.base;
  const int A = s.act_len[(i & 1) * s.B + b];
  const int32_t* act_pos = s.act_pos + act_off(s, i) + base;
  const uint8_t* res = s.res + base;
  const int32_t* timer = s.timer + base;
  // prefetch the tick's ledger entries of this unit's position slice (independent of the freeze
  // loop: tokens of A_i read Active here and are skipped by the tick below)
#ifndef ASR_KPF
#define ASR_KPF 4
#endif
  constexpr int kPF = ASR_KPF;
  // this block: A-slice [a0, a_end) (x-th of X equal parts) and the positions [pos(a0), pos(a_end))
  // with pos(0) = 0, pos(A) = n — exactly its A-tokens and the frozen tokens between them, so the
  // block alone settles the final residency of its positions (unit_next_list compacts them)
  const int per_a = max(1, (A + X - 1) / X);
  const int a0 = min(A, x * per_a), a_end = min(A, (x + 1) * per_a);
  const int n0 = x == 0 ? 0 : a0 >= A ? n : act_pos[a0];
  const int n_end = a_end >= A ? n : act_pos[a_end];
  if (ASR_UNIT_TID() == 0) {
    u.lo = n0;
    u.hi = n_end;
  }
  uint8_t pr[kPF];
  int pt[kPF];
#pragma unroll
  for (int k = 0; k < kPF; ++k) {
    const int j = n0 + (int)ASR_UNIT_TID() + k * (int)ASR_UNIT_THREADS();
    pr[k] = j < n_end ? res[j] : (uint8_t)1;
    pt[k] = j < n_end ? timer[j] : 0;
  }
  int* ev = s.pool_mode && s.evict_policy == ASR_EVICT_BELADY ? u.ev : nullptr;
  if (ev) {
    for (int k = (int)ASR_UNIT_TID(); k < kEvBins; k += ASR_UNIT_THREADS()) ev[k] = 0;
    ASR_UNIT_SYNC();
  }
  int frozen_now = 0, restored = 0, evicted = 0;
  for (int a = a0 + ASR_UNIT_TID(); a < a_end; a += ASR_UNIT_THREADS())
    decide_token(s, dc, b, a, act_pos[a], i, frozen_now, restored, evicted, ev);
  // lines 10-15 for tokens frozen before this step
  uint32_t err = 0;
#pragma unroll
  for (int k = 0; k < kPF; ++k) {
    const int j = n0 + (int)ASR_UNIT_TID() + k * (int)ASR_UNIT_THREADS();
    if (j < n_end) tick_position(s, dc, j, pr[k], pt[k], restored, err, ev);
  }
  for (int j = n0 + (int)ASR_UNIT_TID() + kPF * (int)ASR_UNIT_THREADS(); j < n_end; j += ASR_UNIT_THREADS())
    tick_position(s, dc, j, res[j], timer[j], restored, err, ev);
  if (ev) {   // this block's candidates into the step's histogram (cut by the last decide block)
    ASR_UNIT_SYNC();
    for (int k = (int)ASR_UNIT_TID(); k < kEvBins; k += ASR_UNIT_THREADS())
      if (ev[k]) atomicAdd(&s.ev_hist[k], ev[k]);
  }
  if (err) atomicOr(s.err, err);
  int f = frozen_now, r = restored;
  for (int o = 16; o > 0; o >>= 1) {
    f += __shfl_xor_sync(0xffffffffu, f, o);
    r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  const int w = ASR_UNIT_TID() >> 5, lane = ASR_UNIT_TID() & 31;
  if (lane == 0) { u.sh[w] = f; u.sh2[w] = r; }
  ASR_UNIT_SYNC();
  if (ASR_UNIT_TID() == 0) {
    f = 0; r = 0;
    for (int k = 0; k < (int)(ASR_UNIT_THREADS() >> 5); ++k) { f += u.sh[k]; r += u.sh2[k]; }
    SeqStats& st = s.stats[b];
    if (f) atomicAdd(&st.frozen_this_step, f);
    if (r) atomicAdd(&st.restored_tick, r);
  }
  if (s.pool_mode) {
    for (int o = 16; o > 0; o >>= 1) evicted += __shfl_xor_sync(0xffffffffu, evicted, o);
    if (lane == 0 && evicted) atomicAdd(&s.stats[b].evicted, evicted);
  }
}

// ---------------------------------------------------------------------------------- fused tail
// One warp settles segment t of sequence b at step i (DevState::fuse_tail): the 16 attended tokens
// A_i[16t .. 16t+15] (Alg. 1 lines 3-9), the frozen positions between them and A_i[16t+16] (lines
// 10-15; the first segment starts at 0, the last runs through n, where it also writes the ledger
// entry of the position step i+1 appends), then its part of A_{i+1}: the segment's surviving
// positions are counted, published in seg_flag and placed by a decoupled look-back over the earlier
// segments (a warp waits only on smaller segments, whose warps never wait on larger ones: no
// deadlock, given every warp of the grid is resident).  Full residency only (slot = row + position).
//
// Written for latency: this code runs once per SM per step, right after the attention, so its
// instruction fetches (cold code, L2 or DRAM) are on the critical path — loops stay rolled and the
// function is small and not inlined, so one copy serves the dry run that pre-fetches it (wr = false:
// loads and arithmetic only, every store and wait predicated off) and the real run.  Data: three
// dependent rounds of loads (A_i entries; Eq. 2 partials, counts and the segment's residency /
// timers; the look-back); the final residency of every position is derived in registers (an Active
// position is the k-th token of the tile; its freeze decision comes from the deciding lane by
// ballot) and kept in a shared-memory scratch (fin) for the write pass.
__device__ __forceinline__ unsigned long long seg_word(int i, unsigned state, unsigned v) {
  return ((unsigned long long)((unsigned)(i + 1) & 0x3fffffffu) << 34) | ((unsigned long long)state << 32) | v;
}
// per-warp stamps of the fused tail: compiled in only with -DASR_TAIL_TRACE (diagnostic builds), since
// every instruction of this cold, once-per-step code is on the critical path
__device__ __forceinline__ void trace(const DevState& s, int slot, int k) {
#ifdef ASR_TAIL_TRACE
  if (s.tl && (threadIdx.x & 31) == 0)
    s.tl[kTimelineSlots + ((long)blockIdx.x * 32 + slot) * kTraceCols + k] = gtimer();
#endif
}
__device__ __noinline__ void warp_settle_segment(const DevState& s, int b, int t, int i, uint32_t* fin_scratch,
                                                 int scap, bool wr) {
  const int lane = threadIdx.x & 31;
  const int tslot = wr ? (int)(threadIdx.x >> 5) : 31;
  trace(s, tslot, 0);
  const long base = (long)b * s.max_ctx;
  const int p = i & 1;
  const uint8_t tag_now = res_tag(i);
  // ---- round 1: step geometry and the tile's A_i entries (lane 16: the next segment's first position)
  const int n = s.prompt_len[b] + i + 1;
  const int A = __ldcg(s.act_len + p * s.B + b);   // A_i may have been recompacted in this kernel
  const int a0 = t * 16;
  const int32_t* act_pos = s.act_pos + act_off(s, p) + base;
  const int j = lane <= 16 ? __ldcg(act_pos + min(a0 + lane, s.max_ctx - 1)) : 0;
  const int cnt = min(16, A - a0);
  const bool last = a0 + 16 >= A;
  const bool next = n + 1 <= s.cap;   // step i+1 can run
  const int lo = t == 0 ? 0 : __shfl_sync(0xffffffffu, j, 0);
  const int jn = __shfl_sync(0xffffffffu, j, 16);
  const int hi = last ? n : jn;
  const bool dec = lane < cnt;
  trace(s, tslot, 1);
  // ---- round 2: the deciding lanes' Eq. 2 partials and counts
  // (unconditional loads from clamped, always valid addresses: straight-line code, all in flight)
  float part[32];
  const int L = s.L;
  const float* sp = s.score_part + (long)b * L * s.max_ctx + min(a0 + lane, s.max_ctx - 1);
#pragma unroll
  for (int q = 0; q < 32; ++q) part[q] = __ldcg(sp + (long)min(q, L - 1) * s.max_ctx);
  const long jc = base + (dec ? j : 0);
  const uint32_t cnt_old = __ldcg(s.count + jc);
  unsigned long long hm_lo = 0, hm_hi = 0;
  int hst = 0;
  if (s.hist_w > 0) {
    hm_lo = __ldcg(s.hmask + jc * 2);
    hm_hi = __ldcg(s.hmask + jc * 2 + 1);
    hst = __ldcg(s.hstep + jc);
  }
  float sum = 0.f;
#pragma unroll
  for (int q = 0; q < 32; ++q) sum += q < L ? part[q] : 0.f;   // fixed order l = 0 .. L-1 (as layer_sum)
#pragma unroll 1
  for (int l = 32; l < s.L; ++l) sum += dec ? __ldcg(sp + (long)l * s.max_ctx) : 0.f;
  trace(s, tslot, 2);
  // ---- decide (lines 3-9) on the deciding lanes
  int frozen_now = 0, restored = 0;
  bool absent = false;               // frozen with a remaining absence (leaves A_{i+1})
  if (dec) {
    float sj = sum / (float)(s.L * s.score_heads);
    if (s.score_scaled) sj = sj / sqrtf((float)s.d);
    if (wr) s.score[base + a0 + lane] = sj;
    if (j < n - s.window && j >= s.pinned && sj < s.tau) {
      uint32_t c;
      if (s.hist_w > 0) {
        const int sh = i - hst;
        unsigned long long lo2 = hm_lo, hi2 = hm_hi;
        if (sh >= 128) {
          lo2 = hi2 = 0;
        } else if (sh >= 64) {
          hi2 = lo2 << (sh - 64);
          lo2 = 0;
        } else if (sh > 0) {
          hi2 = (hi2 << sh) | (lo2 >> (64 - sh));
          lo2 <<= sh;
        }
        lo2 |= 1ull;
        if (s.hist_w < 64) {
          lo2 &= (1ull << s.hist_w) - 1ull;
          hi2 = 0;
        } else if (s.hist_w < 128) {
          hi2 &= (1ull << (s.hist_w - 64)) - 1ull;
        }
        if (wr) {
          s.hmask[(base + j) * 2] = lo2;
          s.hmask[(base + j) * 2 + 1] = hi2;
          s.hstep[base + j] = i;
        }
        c = (uint32_t)(__popcll(lo2) + __popcll(hi2));
      } else {
        c = cnt_old + 1;
      }
      if (wr) s.count[base + j] = c;
      const int dd = duration(c, s.softness, s.softness_int);
      if (dd > 0) {
        frozen_now = 1;
        const int tt = s.tick_skip_new ? dd : dd - 1;   // R0: this step's tick applies too
        restored = tt <= 0;           // frozen and restored by the same tick (no absence)
        absent = tt > 0;
        if (wr) {
          s.fstep[base + j] = i;
          s.timer[base + j] = tt > 0 ? tt : 0;
          if (tt > 0) s.res[base + j] = tag_now;
        }
      }
    }
  }
  const unsigned absent_mask = __ballot_sync(0xffffffffu, absent);   // bit k: token a0 + k leaves
  trace(s, tslot, 3);
  // ---- tick (lines 10-15) of the positions frozen before this step; final residency per word of
  //      4 positions (bit e = position 4w + e survives), two words per lane per round of loads
  const uint32_t* res4 = reinterpret_cast<const uint32_t*>(s.res + base);
  const int4* tim4 = reinterpret_cast<const int4*>(s.timer + base);
  const int wlo = lo >> 2, whi = (hi + 3) >> 2;
  uint32_t err = 0;
  int rank = 0;          // Active positions of the segment seen so far (= tile index of the next one)
  int c_seg = 0;         // surviving positions of the segment (this lane's words)
#pragma unroll 1
  for (int m0 = 0; wlo + m0 < whi; m0 += 64) {
    uint32_t rw[2];
    int4 tw[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int w = min(wlo + m0 + 32 * h + lane, whi - 1);   // clamped: masked below by w < whi
      rw[h] = __ldcg(res4 + w);
      tw[h] = __ldcg(tim4 + w);
    }
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int w = wlo + m0 + 32 * h + lane;
      const uint32_t r4 = h ? rw[1] : rw[0];
      const int4 t4 = h ? tw[1] : tw[0];
      uint32_t act0 = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int q = 4 * w + e;
        const uint32_t r = (r4 >> (8 * e)) & 0xffu;
        // Active at the step start (the tag if a deciding lane's store was already visible)
        if (w < whi && q >= lo && q < hi && (r == 1u || r == tag_now)) act0 |= 1u << e;
      }
      const int ca = __popc(act0);
      int incl = ca;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int rk = rank + incl - ca;
      rank += __shfl_sync(0xffffffffu, incl, 31);
      uint32_t fin = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int q = 4 * w + e;
        const uint32_t r = (r4 >> (8 * e)) & 0xffu;
        const int tv = e == 0 ? t4.x : e == 1 ? t4.y : e == 2 ? t4.z : t4.w;
        if (w >= whi || q < lo || q >= hi) continue;
        if (act0 & (1u << e)) {
          if (rk >= 32 || !((absent_mask >> rk) & 1u)) fin |= 1u << e;
          ++rk;
        } else if (tv <= 1) {        // timer reaches 0: restored (Active in A_{i+1})
          fin |= 1u << e;
          restored++;
          if (wr) {
            s.res[base + q] = 1;
            s.timer[base + q] = 0;
          }
        } else {
          if (wr) {
            s.timer[base + q] = tv - 1;
            if (r != 0) s.res[base + q] = 0;        // drop the previous step's tag
          }
          if (q >= n - s.window) err |= kErrFrozenInWindow;
        }
      }
      c_seg += __popc(fin);
      const int widx = m0 + 32 * h + lane;
      if (widx < scap) fin_scratch[widx] = fin;
    }
  }
  trace(s, tslot, 4);
  int f = frozen_now, rr = restored;
  for (int o = 16; o > 0; o >>= 1) {
    f += __shfl_xor_sync(0xffffffffu, f, o);
    rr += __shfl_xor_sync(0xffffffffu, rr, o);
    c_seg += __shfl_xor_sync(0xffffffffu, c_seg, o);
  }
  if (wr) {
    if (err) atomicOr(s.err, err);
    if (lane == 0 && f) atomicAdd(&s.stats[b].frozen_this_step, f);
    if (lane == 0 && rr) atomicAdd(&s.stats[b].restored_tick, rr);
  }
  if (!next) return;   // no step i+1: A_{i+1} is never read
  if (wr && last && lane == 0) ledger_entry_new(s, b, n);
  const int c = c_seg + (last ? 1 : 0);   // + the position step i+1 appends
  // ---- publish (inclusive at once for the first segment), then look back over the earlier ones
  unsigned long long* flag = s.seg_flag + (long)b * s.max_tiles;
  const unsigned long long tag = (unsigned long long)((unsigned)(i + 1) & 0x3fffffffu) << 34;
  if (wr && lane == 0) atomicExch(&flag[t], seg_word(i, t == 0 ? 2u : 1u, (unsigned)c));
  trace(s, tslot, 5);
  int excl = 0;
#pragma unroll 1
  for (int k = t - 1; k >= 0; k -= 32) {
    const int idx = k - lane;
    unsigned long long v = 0;
    if (idx >= 0) {
      const volatile unsigned long long* fp = flag + idx;
      v = *fp;
      if (wr && (v & 0xfffffffc00000000ull) != tag) {
        const unsigned long long tm0 = gtimer();
        while ((v & 0xfffffffc00000000ull) != tag) {
          __nanosleep(20);
          v = *fp;
          if (gtimer() - tm0 > 2000000000ull) {   // 2 s: never on a healthy device; do not hang it
            atomicOr(s.err, kErrStall);
            break;
          }
        }
      }
    }
    const unsigned incl = __ballot_sync(0xffffffffu, idx >= 0 && ((v >> 32) & 3u) == 2u);
    // lanes up to (and including) the nearest inclusive predecessor contribute
    const int stop = incl ? __ffs(incl) - 1 : 31;
    int x = (lane <= stop && idx >= 0) ? (int)(v & 0xffffffffu) : 0;
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    excl += x;
    if (incl || !wr) break;
  }
  if (wr && lane == 0 && t > 0) atomicExch(&flag[t], seg_word(i, 2u, (unsigned)(excl + c)));
  trace(s, tslot, 6);
  // ---- write the segment's surviving positions (and device slots) to A_{i+1}[excl ...]
  int32_t* out = s.act_pos + act_off(s, p ^ 1) + base;
  int32_t* out_slot = s.act_slot + act_off(s, p ^ 1) + base;
  int off = excl;
  __syncwarp();
#pragma unroll 1
  for (int m0 = 0; wlo + m0 < whi; m0 += 32) {
    const int w = wlo + m0 + lane;
    uint32_t fin = 0;
    if (m0 + lane < scap) {
      fin = fin_scratch[m0 + lane];
    } else if (w < whi) {   // beyond the scratch: re-read the residency this warp just settled
      const uint32_t rw = __ldcg(res4 + w);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (((rw >> (8 * e)) & 0xffu) == 1u && 4 * w + e >= lo && 4 * w + e < hi) fin |= 1u << e;
    }
    const int cm = __popc(fin);
    int incl = cm;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int o = off + incl - cm;
    while (fin) {
      const int jj = 4 * w + __ffs(fin) - 1;
      if (wr) {
        out[o] = jj;
        out_slot[o] = (int)(base + jj);
      }
      ++o;
      fin &= fin - 1;
    }
    off += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (wr && last && lane == 0) {
    out[off] = n;
    out_slot[off] = (int)(base + n);
    s.act_len[(p ^ 1) * s.B + b] = off + 1;
  }
  trace(s, tslot, 7);
}

// (a4') combine for the fused tail, one warp per (b, l, h), head_dim 128, stream-K pieces: the same
// fixed-order merge as combine_warp in compact form (rolled over pieces, 8 piece loads in flight);
// wr = false: dry run (no store).
__device__ __noinline__ void combine_warp_tail(const DevState& s, int wid, float* __restrict__ o, bool wr) {
  const int lane = threadIdx.x & 31;
  const int tslot = wr ? 16 + (int)(threadIdx.x >> 5) : 31;
  trace(s, tslot, 0);
  const int h = wid % s.Hq;
  const int l = (wid / s.Hq) % s.L;
  const int b = wid / (s.Hq * s.L);
  const int is_b = __ldcg(s.item_start + b), is_b1 = __ldcg(s.item_start + b + 1);
  const long T = __ldcg(s.item_start + s.B);
  const int tiles = (is_b1 - is_b) / s.L;
  if (!tiles || T <= 0) return;
  const long S = is_b + (long)l * tiles;
  const SkPlan pl = sk_plan(T, s.sk_grid, s.sk_dyn, s.sk_chunk);
  const int cf = sk_unit_of(pl, S);
  int nch = sk_unit_of(pl, S + tiles - 1) - cf + 1;
  if (nch == 1) return;   // one CTA held the whole item and wrote O itself
  if (!wr) nch = min(nch, 8);
  const long it0 = (long)b * s.L + l + cf;
  ASR_CHECK(s, it0 >= 0 && it0 + nch <= s.max_items);
  float M = -INFINITY;
#pragma unroll 1
  for (int c = lane; c < nch; c += 32) M = fmaxf(M, __ldcg(s.part_ml + ((it0 + c) * s.Hq + h) * 2));
  for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
  float den = 0.f;
#pragma unroll 1
  for (int c0 = 0; c0 < nch; c0 += 32) {
    const long pl = (it0 + min(c0 + lane, nch - 1)) * s.Hq + h;   // clamped: weight 0 beyond nch
    const float m_l = __ldcg(s.part_ml + pl * 2), l_l = __ldcg(s.part_ml + pl * 2 + 1);
    const float wl = c0 + lane < nch ? exp2f(m_l - M) : 0.f;
    const float ll = c0 + lane < nch ? l_l : 0.f;
    const int cn = min(32, nch - c0);
#pragma unroll 1
    for (int cb = 0; cb < cn; cb += 8) {
      float4 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        v[q] = __ldcg(reinterpret_cast<const float4*>(s.part_acc + ((it0 + c0 + min(cb + q, cn - 1)) * s.Hq + h) * 128L) +
                      lane);
#pragma unroll
      for (int q = 0; q < 8; ++q) {   // chunk order: deterministic (w = 0 adds exact zeros past cn)
        const float w = cb + q < cn ? __shfl_sync(0xffffffffu, wl, (cb + q) & 31) : 0.f;
        const float lq = __shfl_sync(0xffffffffu, ll, (cb + q) & 31);
        if (cb + q < cn) den = fmaf(lq, w, den);
        num.x = fmaf(v[q].x, w, num.x);
        num.y = fmaf(v[q].y, w, num.y);
        num.z = fmaf(v[q].z, w, num.z);
        num.w = fmaf(v[q].w, w, num.w);
      }
    }
  }
  trace(s, tslot, 6);
  const float inv = 1.0f / den;
  if (wr)
    *reinterpret_cast<float4*>(o + (((long)b * s.L + l) * s.Hq + h) * 128L + lane * 4) =
        make_float4(num.x * inv, num.y * inv, num.z * inv, num.w * inv);
  trace(s, tslot, 7);
}

// After unit_decide of step i: A_{i+1} into parity (i+1) & 1.  Decide block x owns the positions
// [u.lo, u.hi) and has settled their final residency itself, so it compacts them without waiting for
// the other blocks; the block holding index A-1 also appends position n (the token step i+1 appends).
// Each block publishes its count in dagg[b][x] tagged with the step and adds up its predecessors'
// counts (look-back without a chain: lane k of warp 0 waits for block k) to place its part.  The
// host uses X > 1 only when every decide block is co-resident.
__device__ void unit_next_list(const DevState& s, int b, int x, int X, int i, UnitShm& u) {
  const int n = s.prompt_len[b] + i + 1;    // tokens held after step i
  const bool next = n + 1 <= s.cap;         // step i+1 can run
  const int tid = (int)ASR_UNIT_TID();
  const int A = s.act_len[(i & 1) * s.B + b];
  const int per_a = max(1, (A + X - 1) / X);
  const bool tail = x == max(0, A - 1) / per_a;   // holds index A-1 (the last position of A_i)
  const int lo = u.lo;
  int hi = u.hi;
  if (tail && next) {
    if (tid == 0) ledger_entry_new(s, b, n);
    hi = n + 1;
  }
  ASR_UNIT_SYNC();
  Compactor c;
  const int cnt = c.count(s, b, lo, hi, u);
  const unsigned long long tag = (unsigned long long)(unsigned)(i + 1) << 32;
  if (X > 1) {
    if (tid == 0) atomicExch(&s.dagg[(long)b * 32 + x], tag | (unsigned)cnt);
    if (tid < 32) {   // warp 0: lane k waits for block k < x
      int pre = 0;
      if (tid < x) {
        const volatile unsigned long long* a = s.dagg + (long)b * 32 + tid;
        unsigned long long v = *a;
        const unsigned long long t0 = gtimer();
        while ((v & 0xffffffff00000000ull) != tag) {
          __nanosleep(32);
          v = *a;
          if (gtimer() - t0 > 2000000000ull) {   // 2 s: never on a healthy device; do not hang it
            atomicOr(s.err, kErrStall);
            break;
          }
        }
        pre = (int)(v & 0xffffffffu);
      }
      for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
      if (tid == 0) u.level = pre;
    }
  } else if (tid == 0) {
    u.level = 0;
  }
  ASR_UNIT_SYNC();
  const int base = u.level;
  if (next) c.write(s, b, (i + 1) & 1, base, u);
  if (tid == 0 && tail && next) {
    s.act_len[((i + 1) & 1) * s.B + b] = base + cnt;
    if (base + cnt == 0) atomicOr(s.err, kErrEmptyActive);
  }
  ASR_UNIT_SYNC();
}

// ---------------------------------------------------------------------------------- (a5) Belady
// Pressure mode, Belady policy: after phase D of step i every resident frozen token with remaining
// timer t >= evict_min is in ev_hist (bin min(t, kEvBins-1)); it is next attended at step i + t + 1,
// known exactly (Eq. 3 fixes the absence at freeze time).  The slots the next step needs are its B
// appends, its prefetches (tokens returning then that were evicted) and pool_reserve for demand
// restores; if the free stack is short by `need`, the candidates returning LAST are evicted first
// (Belady's MIN with clairvoyant reuse times): every candidate above the cut bin T and `quota` of
// those in it.  Computed by the last decide block (one thread), applied by evict_kernel.
__device__ void belady_cut(const DevState& s, int i) {
  int pf = 0;
  for (int b = 0; b < s.B; ++b) pf += __ldcg(s.pf_count + (i & 1) * s.B + b);
  const int reserve = s.pool_reserve > 0 ? s.pool_reserve : s.B;
  const int need = s.B + pf + reserve - __ldcg(s.free_top);
  int T = kEvBins, quota = 0;
  if (need > 0) {
    int cum = 0;
    for (int k = kEvBins - 1; k >= s.evict_min && k >= 0; --k) {
      const int h = __ldcg(s.ev_hist + k);
      T = k;
      quota = min(h, need - cum);
      cum += h;
      if (cum >= need) break;
    }
  }
  s.ev_ctrl[0] = T;
  s.ev_ctrl[1] = quota;
  s.ev_ctrl[2] = 0;
  s.ev_ctrl[3] = need;
  for (int k = 0; k < kEvBins; ++k) s.ev_hist[k] = 0;
}

// Evict the cut (one thread per position, grid-stride over all sequences): a resident frozen token
// with bin > T, or in bin T while the quota lasts, gives its slot back (its bytes are in the host
// mirror since its append).  Pushes only: the next pops are in the next step's phase B.
__device__ void evict_positions(const DevState& s) {
  const int need = __ldcg(s.ev_ctrl + 3);
  if (need <= 0) return;
  const int T = __ldcg(s.ev_ctrl + 0), quota = __ldcg(s.ev_ctrl + 1);
  const int step = *s.step;   // phase D advanced it: positions held = prompt_len + step
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < (long)s.B * s.max_ctx; g += (long)gridDim.x * blockDim.x) {
    const int b = (int)(g / s.max_ctx), j = (int)(g % s.max_ctx);
    if (j >= s.prompt_len[b] + step) continue;
    const long k = (long)b * s.max_ctx + j;
    if (res_active(s.res[k])) continue;
    const int so = s.slot_of[k];
    const int t = s.timer[k];
    if (so < 0 || t < s.evict_min) continue;
    const int bin = min(t, kEvBins - 1);
    if (bin < T || (bin == T && atomicAdd(s.ev_ctrl + 2, 1) >= quota)) continue;
    pool_push(s, so);
    s.slot_of[k] = -1;
    atomicAdd(&s.stats[b].evicted, 1);
  }
}

// Pressure mode: copy the tokens phase B gave slots to (this step's prefetch list) from the host
// mirror, one token per block at a time; runs beside the attention kernel (graph branch).
__device__ void prefetch_copies(const DevState& s, int* start) {
  if (ASR_UNIT_TID() == 0) {
    int acc = 0;
    for (int b = 0; b < s.B; ++b) {
      start[b] = acc;
      acc += s.cp_count[b];
    }
    start[s.B] = acc;
  }
  ASR_UNIT_SYNC();
  const int total = start[s.B];
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    int lo = 0, hi = s.B - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (start[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    const int b = lo;
    const int j = s.cp_list[(long)b * s.max_ctx + (t - start[b])];
    copy_token_h2d(s, b, j, s.slot_of[(long)b * s.max_ctx + j]);
  }
}

// ---------------------------------------------------------------------------------- (a4') combine
// One warp per (b, l, h): lane c < nch reads split c's (m, l); each lane owns d/32 output elements;
// fixed split order -> deterministic.
__device__ void combine_warp(const DevState& s, int wid, float* __restrict__ o) {
  const int lane = ASR_UNIT_TID() & 31;
  const int h = wid % s.Hq;
  const int l = (wid / s.Hq) % s.L;
  const int b = wid / (s.Hq * s.L);
  int nch;
  long it0;
  // (read through L2: in the fused tail these were written by other CTAs of the same kernel)
  int bnd[kSkBalPer] = {};   // range starts of a rate-balanced split (loaded beside item_start; phase D
                             // runs after the attention kernel, so the non-coherent path is safe)
  if (s.sk_bal) {
#pragma unroll
    for (int i = 0; i < kSkBalPer; ++i) bnd[i] = i * 32 + lane < s.sk_grid ? __ldg(s.sk_bound + i * 32 + lane) : 0x7fffffff;
  }
  const int is_b = __ldcg(s.item_start + b), is_b1 = __ldcg(s.item_start + b + 1);
  const int per_seq = (is_b1 - is_b) / s.L;   // tiles (or chunks) per layer
  if (s.sk_grid) {   // stream-K pieces (asr_internal.h)
    const int tiles = per_seq;
    const long T = __ldcg(s.item_start + s.B), S = is_b + (long)l * tiles;
    const SkPlan pl = sk_plan(T, s.sk_grid, s.sk_dyn, s.sk_chunk);
    int cf, cl;
    if (sk_weighted(s.sk_bal, pl)) {   // unit of t: the number of range starts <= t, minus one
      cf = cl = -1;
#pragma unroll
      for (int i = 0; i < kSkBalPer; ++i) {
        cf += __popc(__ballot_sync(0xffffffffu, bnd[i] <= S));
        cl += __popc(__ballot_sync(0xffffffffu, bnd[i] <= S + tiles - 1));
      }
    } else {
      cf = tiles ? sk_unit_of(pl, S) : 0;
      cl = tiles ? sk_unit_of(pl, S + tiles - 1) : -1;
    }
    if (!tiles) cf = cl + 1;
    nch = cl - cf + 1;
    it0 = (long)b * s.L + l + cf;
    if (nch == 1) return;   // one CTA held the whole item and wrote O itself
  } else {
    nch = per_seq;
    it0 = is_b + (long)l * nch;
  }
  float M = -INFINITY;
  for (int c = lane; c < nch; c += 32) M = fmaxf(M, __ldcg(s.part_ml + ((it0 + c) * s.Hq + h) * 2));
  for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  const int epl = s.d >= 32 ? s.d / 32 : 1;   // elements per lane (d <= 256 -> <= 8)
  const bool on = lane * epl < s.d;
  float num[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float den = 0.f;
  for (int c0 = 0; c0 < nch; c0 += 32) {
    float wl = 0.f, ll = 0.f;
    if (c0 + lane < nch) {
      const long pi = (it0 + c0 + lane) * s.Hq + h;
      wl = exp2f(__ldcg(s.part_ml + pi * 2) - M);
      ll = __ldcg(s.part_ml + pi * 2 + 1);
    }
    const int cn = min(32, nch - c0);
    if (epl == 4) {
      for (int cb = 0; cb < cn; cb += 8) {   // 8 chunk vectors in flight, accumulated in chunk order
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (cb + q < cn)
            v[q] = __ldcg(reinterpret_cast<const float4*>(s.part_acc + ((it0 + c0 + cb + q) * s.Hq + h) * (long)s.d +
                                                          lane * 4));
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (cb + q >= cn) break;
          const float w = __shfl_sync(0xffffffffu, wl, cb + q);
          den = fmaf(__shfl_sync(0xffffffffu, ll, cb + q), w, den);
          num[0] = fmaf(v[q].x, w, num[0]); num[1] = fmaf(v[q].y, w, num[1]);
          num[2] = fmaf(v[q].z, w, num[2]); num[3] = fmaf(v[q].w, w, num[3]);
        }
      }
    } else {
      for (int c = 0; c < cn; ++c) {
        const float w = __shfl_sync(0xffffffffu, wl, c);
        den = fmaf(__shfl_sync(0xffffffffu, ll, c), w, den);
        if (on) {
          const float* src = s.part_acc + ((it0 + c0 + c) * s.Hq + h) * (long)s.d + lane * epl;
          for (int e = 0; e < epl; ++e) num[e] = fmaf(__ldcg(src + e), w, num[e]);
        }
      }
    }
  }
  if (on) {
    float* dst = o + (((long)b * s.L + l) * s.Hq + h) * s.d + lane * epl;
    const float inv = 1.0f / den;
    for (int e = 0; e < epl; ++e) dst[e] = num[e] * inv;
  }
}

// Work units of phase A: per sequence kEntSplits / ent_per_unit entropy units (with logits), then
// ceil(L / layers_per_unit) append units (the host picks the grouping so a large batch does not
// launch thousands of tiny blocks).
__host__ __device__ inline int ent_units_per_seq(const DevState& s) { return kEntSplits / s.ent_per_unit; }
__host__ __device__ inline int app_units_per_seq(const DevState& s) {
  return (s.L + s.layers_per_unit - 1) / s.layers_per_unit;
}
__host__ __device__ inline int phaseA_units(const DevState& s, bool has_logits) {
  return s.B * ((has_logits ? ent_units_per_seq(s) : 0) + app_units_per_seq(s));
}
// Sequence of phase-A unit `unit`, and how many units each sequence has.
__host__ __device__ inline int phaseA_seq(const DevState& s, bool has_logits, int unit) {
  const int ne = has_logits ? s.B * ent_units_per_seq(s) : 0;
  return unit < ne ? unit / ent_units_per_seq(s) : (unit - ne) / app_units_per_seq(s);
}
__host__ __device__ inline int phaseA_units_per_seq(const DevState& s, bool has_logits) {
  return (has_logits ? ent_units_per_seq(s) : 0) + app_units_per_seq(s);
}
template <typename TL, typename TK, bool kFlatAppend>
__device__ void run_phaseA_unit(const DevState& s, int unit, int i, const TL* logits, const TK* k_new,
                                const TK* v_new, UnitShm& u) {
  const int eu = ent_units_per_seq(s), au = app_units_per_seq(s);
  const int ne = logits ? s.B * eu : 0;
  if (unit < ne) {
    const int b = unit / eu, k = unit % eu;
    const int w = (int)ASR_UNIT_TID() >> 5, nw = (int)ASR_UNIT_THREADS() >> 5;
    for (int sp = k * s.ent_per_unit + w; sp < (k + 1) * s.ent_per_unit; sp += nw)   // one split per warp
      warp_entropy_split<TL>(s, logits, b, sp, (int)ASR_UNIT_TID() & 31);
  } else if (k_new) {   // (policy replay appends no K/V)
    const int a = unit - ne;
    const int b = a / au, k = a % au;
    const int l0 = k * s.layers_per_unit, l1 = min(s.L, (k + 1) * s.layers_per_unit);
    // (the flat loop only in the phase-A kernel: compiled into the attention kernel, whose phase-A
    // warp appends one layer per unit anyway, it slowed the batch-64 attention by 3 %: code layout)
    if (kFlatAppend && !s.pool_mode && (s.Hkv * s.d * (int)sizeof(TK)) % 16 == 0)
      unit_append_layers<TK>(s, b, l0, l1, i, k_new, v_new);
    else
      for (int l = l0; l < l1; ++l) unit_append<TK>(s, b, l, i, k_new, v_new);
  }
}

// Phase A unit `unit` of step i and, when it is the last unit of its sequence to finish (per-sequence
// ticket, threadfence pattern), phase B of that sequence (unit_finish) — no dependent launch between.
template <typename TL, typename TK, bool kFlatAppend = false>
__device__ void phaseA_block(const DevState& s, int unit, int i, const TL* logits, const TK* k_new, const TK* v_new,
                             float* entropy_out, UnitShm& u) {
  const bool has_logits = logits != nullptr;
  run_phaseA_unit<TL, TK, kFlatAppend>(s, unit, i, logits, k_new, v_new, u);
  if (s.tl && ASR_UNIT_TID() == 0)
    atomicMax(&s.tl[2 * kStages + 3 + ((has_logits && unit < s.B * ent_units_per_seq(s)) ? 0 : 1)], gtimer());
  const int b = phaseA_seq(s, has_logits, unit);
  ASR_UNIT_SYNC();
  if (ASR_UNIT_TID() == 0) {
    // release: this unit's results before the ticket; acquire: the last unit sees every unit's results
    u.last = atom_add_acqrel(&s.pre_ticket[b], 1) == phaseA_units_per_seq(s, has_logits) - 1;
    if (u.last) s.pre_ticket[b] = 0;
  }
  ASR_UNIT_SYNC();
  if (u.last) {
    if (s.tl && ASR_UNIT_TID() == 0) atomicMax(&s.tl[2 * kStages + 5], gtimer());
    unit_finish(s, b, i, has_logits || s.ent_given != nullptr, entropy_out, u);
    if (s.tl && ASR_UNIT_TID() == 0) atomicMax(&s.tl[2 * kStages + 6], gtimer());
    ASR_UNIT_SYNC();
    if (ASR_UNIT_TID() == 0)
      st_release(s.pre_done, i + 1);   // the attention kernel's CTAs wait for this when phase A runs inside it
  }
}

}  // namespace
}  // namespace units
}  // namespace asr
