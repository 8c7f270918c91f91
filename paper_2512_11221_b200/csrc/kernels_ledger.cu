// paper_2512_11221_b200/csrc/kernels_ledger.cu — the ledger side of one ASR-KF-EGR step (sm_100a):
//   pre_kernel      (a6) H(logits_prev) + spike detector + recovery ladder (Sec 3.6),
//                   (a0) append, recovery levels, (a3) compaction of A_i (Alg. 1)
//   post_kernel     (a4') fixed-order combine of the split-KV partials -> O, and
//                   (a2) Eq. 2 finish, threshold, Eq. 3 schedule, freeze, tick (Alg. 1 lines 3-15)
//   restore_kernel  explicit SR / WR / FR (asr_restore)
// All floating-point reductions are in a fixed order, so the step is bitwise deterministic; the
// integer counters use atomics (order-independent).
#include <cuda_bf16.h>
#include <math.h>

#include <cooperative_groups.h>

#include "asr_internal.h"

namespace cg = cooperative_groups;

namespace asr {
namespace {

// Block-wide sum of int (blockDim multiple of 32, <= 1024).  Result valid in every thread.
__device__ int block_sum_int(int v, int* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  int t = 0;
  for (int i = 0; i < nw; ++i) t += sh[i];
  __syncthreads();
  return t;
}

// ---------------------------------------------------------------------------------- (a6) entropy
// Per split of the row: m = max x/T, Z = sum e^{x/T - m}, S = sum e^{x/T - m} (x/T - m); the
// last block of a row (atomic ticket) merges the splits in split order:
//   H = ln Z - S / Z,  with (m, Z, S) rescaled to the global max,
// then runs the detector (R-det) and the ladder (R-ladder) in double precision.
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
__device__ __forceinline__ float tof(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float tof(float v) { return v; }

constexpr int kPreThreads = 512;

// Recovery levels on one sequence's ledger: returns the restored count of this thread.
__device__ int apply_level(const DevState& s, int b, int n, int level, int i) {
  int restored = 0;
  uint8_t* res = s.res + (long)b * s.max_ctx;
  int32_t* timer = s.timer + (long)b * s.max_ctx;
  const int32_t* fstep = s.fstep + (long)b * s.max_ctx;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    if (res_active(res[j])) continue;
    bool go = level == 1 ? timer[j] > 1 : level == 2 ? fstep[j] >= i - s.wr_window : true;
    if (go) {
      res[j] = 1;
      timer[j] = 0;
      restored++;
    }
  }
  if (level >= 3 && s.fr_clear_counts) {
    uint32_t* cnt = s.count + (long)b * s.max_ctx;
    for (int j = threadIdx.x; j < n; j += blockDim.x) cnt[j] = 0;
  }
  return restored;
}

// ------------------------------------------------------------------ pre_kernel
// (a6) entropy + detector + ladder + recovery, (a0) append and (a3) compaction in one launch.
// Sequence b is handled by one thread-block cluster of kCl CTAs (B200 clusters: the partial results
// meet in distributed shared memory behind hardware cluster barriers, no global atomics/fences):
//   every CTA r:  entropy partial (m, Z, S) of vocab slice r; active count of position slice r
//   barrier;      rank 0 merges the kCl entropy partials (fixed order), runs the detector and the
//                 ladder (R-det, R-ladder) and publishes the recovery level
//   barrier;      if a level fired (rare): every CTA applies it to its slice and recounts (+barrier)
//                 every CTA writes its slice of A_i at the offset of the lower ranks' counts
// Clusters >= B copy the new token's K/V rows, one (b, l) per CTA.
constexpr int kCl = 8;

struct PreShared {
  float em, ez, es;     // entropy partial of this CTA
  int cnt;              // Active positions in this CTA's slice
  int restored;         // restored by recovery in this CTA's slice
  int level;            // recovery level (rank 0 publishes)
  int wsum[32];
  float wm[32], wz[32], ws[32];
  double hist[kMaxDetBaseline];
};

__device__ __forceinline__ void tri_merge(float& m, float& z, float& sx, float om, float oz, float os) {
  // merge (m, Z, S) triples of the single-pass entropy: rescale both to M = max(m, om)
  const float M = fmaxf(m, om);
  float nz = 0.f, ns = 0.f;
  if (z > 0.f) { const float f = __expf(m - M); nz += z * f; ns += f * (sx + z * (m - M)); }
  if (oz > 0.f) { const float f = __expf(om - M); nz += oz * f; ns += f * (os + oz * (om - M)); }
  m = M; z = nz; sx = ns;
}

// Active positions of [p0, p1) (p0 multiple of 16): per-thread runs of 16-position vectors.
__device__ __forceinline__ int active_mask16(uint4 u, uint32_t* m) {  // 1 per byte iff residency == 1
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
  int c = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    m[k] = w[k] & 0x01010101u & ~((w[k] >> 1) & 0x01010101u);
    c += __popc(m[k]);
  }
  return c;
}

// Block count + exclusive scan of this CTA's slice: returns the thread's exclusive offset, writes the
// CTA total to ps.cnt.  Thread t owns vectors [v0, v1).
__device__ int slice_scan(const uint8_t* res, int v0, int v1, PreShared& ps, int* my_cnt) {
  int cnt = 0;
#pragma unroll 4
  for (int v = v0; v < v1; ++v) {
    uint32_t m[4];
    cnt += active_mask16(*reinterpret_cast<const uint4*>(res + v * 16), m);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) ps.wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = lane < (int)(blockDim.x >> 5) ? ps.wsum[lane] : 0;
    int xi = x;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    ps.wsum[lane] = xi - x;  // exclusive warp offsets
    if (lane == 31) ps.cnt = xi;
  }
  __syncthreads();
  *my_cnt = cnt;
  return ps.wsum[w] + incl - cnt;
}

template <typename TL, typename TK>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kPreThreads, 1)
    pre_kernel(DevState s, const TL* logits, float* entropy_out, const TK* k_new, const TK* v_new) {
  pdl_trigger();   // the attention kernel may start its (independent) prologue now
  Stamp stamp(s.tl, 0);
  const int i = *s.step;
  const int cid = blockIdx.x / kCl;
  if (cid >= s.B) {  // ---- append K/V rows of (b, l) (whole clusters take this branch)
    const int a = blockIdx.x - kCl * s.B;
    if (a >= s.B * s.L) return;
    const int b = a / s.L, l = a % s.L;
    const long pos = s.prompt_len[b] + i;
    const long slot = (long)b * s.max_ctx + pos;
    const int row = s.Hkv * s.d;  // elements of K (or V) per token-layer
    TK* dst = reinterpret_cast<TK*>(s.kv) + (slot * s.L + l) * 2 * row;
    const TK* ks = k_new + ((long)b * s.L + l) * row;
    const TK* vs = v_new + ((long)b * s.L + l) * row;
    const int vec = (int)(16 / sizeof(TK));
    if (row % vec == 0) {
      const int nv = row / vec;
      for (int t = threadIdx.x; t < 2 * nv; t += blockDim.x) {
        const uint4* src = reinterpret_cast<const uint4*>(t < nv ? ks : vs) + (t < nv ? t : t - nv);
        reinterpret_cast<uint4*>(dst)[t] = *src;
      }
    } else {
      for (int t = threadIdx.x; t < 2 * row; t += blockDim.x) dst[t] = t < row ? ks[t] : vs[t - row];
    }
    return;
  }
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  __shared__ PreShared ps;
  const int b = cid;
  const int n = s.prompt_len[b] + i + 1;  // total after the append
  const long base = (long)b * s.max_ctx;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  DetState& ds = s.det[b];
  // ---- rank 0 prefetches the detector history; the owner of position n-1 appends its ledger entry
  if (rank == 0 && logits)
    for (int t = threadIdx.x; t < ds.hist_len; t += blockDim.x) ps.hist[t] = s.hist[(long)b * s.det_baseline + t];
  const int nvec = (n + 15) >> 4;
  const int vr = (nvec + kCl - 1) / kCl;                    // vectors per rank
  const int rv0 = min(nvec, rank * vr), rv1 = min(nvec, rv0 + vr);
  if (threadIdx.x == 0 && (n - 1) >= rv0 * 16 && (n - 1) < rv1 * 16) {
    const long j = base + n - 1;   // the token produced by the previous step (Alg. 1 line 16)
    s.res[j] = 1;
    s.timer[j] = 0;
    s.count[j] = 0;
    s.fstep[j] = -1;
  }
  // ---- entropy partial of vocab slice `rank` (single pass, online (m, Z, S))
  if (logits) {
    const int V = s.vocab;
    const int vs = ((((V + kCl - 1) / kCl) + 7) & ~7);
    const int e0 = min(V, rank * vs), e1 = min(V, e0 + vs);
    const TL* row = logits + (long)b * V;
    const bool vecok = (reinterpret_cast<uintptr_t>(row) & 31) == 0;
    const float invT = 1.0f / s.ent_temp;
    float m = -INFINITY, z = 0.f, sx = 0.f;
    for (int v = e0 + (int)threadIdx.x * 8; v < e1; v += (int)blockDim.x * 8) {
      float x[8];
      if (vecok && v + 8 <= e1) {
        load8<TL>(row + v, x);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = (v + e < e1) ? tof(row[v + e]) : -INFINITY;
      }
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
    }
    for (int o = 16; o > 0; o >>= 1)
      tri_merge(m, z, sx, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, z, o),
                __shfl_xor_sync(0xffffffffu, sx, o));
    if (lane == 0) { ps.wm[w] = m; ps.wz[w] = z; ps.ws[w] = sx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      float M = -INFINITY, Z = 0.f, S = 0.f;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tri_merge(M, Z, S, ps.wm[k], ps.wz[k], ps.ws[k]);
      ps.em = M; ps.ez = Z; ps.es = S;
    }
  }
  // ---- count the Active positions of this rank's slice
  const uint8_t* res = s.res + base;
  const int per = (rv1 - rv0 + (int)blockDim.x - 1) / (int)blockDim.x;
  const int v0 = min(rv1, rv0 + (int)threadIdx.x * per), v1 = min(rv1, v0 + per);
  __syncthreads();   // the appended entry is visible to the counting threads of this CTA
  int my_cnt;
  int my_off = slice_scan(res, v0, v1, ps, &my_cnt);
  if (threadIdx.x == 0) ps.restored = 0;
  cl.sync();
  // ---- rank 0: H, detector, ladder
  if (rank == 0 && w == 0) {
    int level = 0;
    if (logits) {
      double M = -INFINITY, Z = 0.0, S = 0.0;
      if (lane == 0) {
        for (int r = 0; r < kCl; ++r) {   // fixed rank order
          const PreShared* o = cl.map_shared_rank(&ps, r);
          const double om = o->em, oz = o->ez, os = o->es;
          if (oz <= 0.0) continue;
          const double Mn = fmax(M, om);
          double nz = 0.0, ns = 0.0;
          if (Z > 0.0) { const double f = exp(M - Mn); nz += Z * f; ns += f * (S + Z * (M - Mn)); }
          const double f = exp(om - Mn);
          nz += oz * f;
          ns += f * (os + oz * (om - Mn));
          M = Mn; Z = nz; S = ns;
        }
      }
      const double H = __shfl_sync(0xffffffffu, log(Z) - S / Z, 0);
      const int hl = ds.hist_len;
      double mu = 0.0, var = 0.0;
      for (int t = lane; t < hl; t += 32) mu += ps.hist[t];
      for (int o = 16; o > 0; o >>= 1) mu += __shfl_xor_sync(0xffffffffu, mu, o);
      mu = hl > 0 ? mu / hl : 0.0;
      for (int t = lane; t < hl; t += 32) var += (ps.hist[t] - mu) * (ps.hist[t] - mu);
      for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
      if (lane == 0) {
        var = hl > 0 ? var / hl : 0.0;
        int trig = 0;
        if (s.det_enable && hl >= 2) {
          const double sd = fmax(sqrt(var), (double)s.det_sigma_floor);
          trig = H > mu + (double)s.det_z * sd;   // detector: H > mean + z * max(sigma, floor)
        }
        double* hist = s.hist + (long)b * s.det_baseline;
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
        if (entropy_out) entropy_out[b] = (float)H;
        s.stats[b].entropy = (float)H;
      }
    }
    if (lane == 0) ps.level = level;
  }
  cl.sync();
  const int level = cl.map_shared_rank(&ps, 0)->level;
  if (level > 0) {   // rare: recovery restores in every slice, then recount
    int r = 0;
    int32_t* timer = s.timer + base;
    const int32_t* fstep = s.fstep + base;
    uint8_t* resw = s.res + base;
    const int p0 = rv0 * 16, p1 = min(n - 1, rv1 * 16);
    for (int j = p0 + (int)threadIdx.x; j < p1; j += blockDim.x) {
      if (res_active(resw[j])) continue;
      const bool go = level == 1 ? timer[j] > 1 : level == 2 ? fstep[j] >= i - s.wr_window : true;
      if (go) { resw[j] = 1; timer[j] = 0; r++; }
    }
    if (level >= 3 && s.fr_clear_counts)
      for (int j = p0 + (int)threadIdx.x; j < p1; j += blockDim.x) s.count[base + j] = 0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    __syncthreads();
    if (lane == 0) atomicAdd(&ps.restored, r);
    __syncthreads();
    my_off = slice_scan(res, v0, v1, ps, &my_cnt);
    cl.sync();
  }
  // ---- write this slice of A_i at the offset of the lower ranks
  int off0 = 0, total = 0, restored = 0;
  for (int r = 0; r < kCl; ++r) {
    const PreShared* o = cl.map_shared_rank(&ps, r);
    const int c = o->cnt;
    if (r < rank) off0 += c;
    total += c;
    restored += o->restored;
  }
  int off = off0 + my_off;
  int32_t* out = s.act_pos + base;
  for (int v = v0; v < v1; ++v) {
    uint32_t m[4];
    active_mask16(*reinterpret_cast<const uint4*>(res + v * 16), m);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      while (m[k]) {
        const int bit = __ffs(m[k]) - 1;   // bit 8*q of byte q
        out[off++] = v * 16 + k * 4 + (bit >> 3);
        m[k] &= m[k] - 1;
      }
  }
  if (rank == 0 && threadIdx.x == 0) {
    s.act_len[b] = total;
    if (total == 0) atomicOr(s.err, kErrEmptyActive);
    SeqStats& st = s.stats[b];
    st.attended = total;
    st.restored_pre = st.pending_restored;
    st.pending_restored = 0;
    st.restored_tick = 0;
    st.frozen_this_step = 0;
    st.restored_rec = restored;
    st.recovery_action = level;
    st.rewalk_requested = level == 4;
    st.entropy_valid = logits ? 1 : 0;
    s.rec_action[b] = level;
  }
  cl.sync();   // keep every CTA's shared memory alive until the whole cluster has read it
}

// ------------------------------------------------------------------ (a2) decide + tick
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

// Grid (decide_blocks, B).  Block x of sequence b handles a slice of the attended list (Alg. 1
// lines 3-9 + the R0 tick of the tokens it freezes) and a slice of the positions (lines 10-15 for
// tokens frozen at earlier steps).  The two index sets are disjoint (A_i = the tokens Active at the
// step start), and tokens frozen in this step carry the step-parity tag res_tag(i), so the blocks
// need no ordering between them.
__device__ void decide_block(const DevState& s, int b, int x, int X, int nblocks_total) {
  __shared__ int sh[32];
  __shared__ int sh2[32];
  const int i = *s.step;
  const int n = s.prompt_len[b] + i + 1;
  const long base = (long)b * s.max_ctx;
  const int A = s.act_len[b];
  uint8_t* res = s.res + base;
  int32_t* timer = s.timer + base;
  uint32_t* cnt = s.count + base;
  int32_t* fstep = s.fstep + base;
  const float inv = 1.0f / (float)(s.L * s.Hq);
  const float inv_sqrt_d = rsqrtf((float)s.d);
  const uint8_t tag_now = res_tag(i);
  // ---- prefetch the tick's ledger entries of this block's position slice (independent of the
  //      freeze loop: tokens of A_i read Active here and are skipped by the tick below)
  constexpr int kPF = 4;
  const int per_n = (n + X - 1) / X;
  const int n0 = x * per_n, n_end = min(n, n0 + per_n);
  uint8_t pr[kPF];
  int pt[kPF];
#pragma unroll
  for (int k = 0; k < kPF; ++k) {
    const int j = n0 + (int)threadIdx.x + k * (int)blockDim.x;
    pr[k] = j < n_end ? res[j] : (uint8_t)1;
    pt[k] = j < n_end ? timer[j] : 0;
  }
  int frozen_now = 0, restored = 0;
  // ---- Alg. 1 lines 3-9 over this block's slice of A_i
  const int per_a = (A + X - 1) / X;
  const int a_end = min(A, (x + 1) * per_a);
  for (int a = x * per_a + threadIdx.x; a < a_end; a += blockDim.x) {
    const int j = s.act_pos[base + a];
    // sum over layers in order l = 0..L-1; loads issued 8 at a time so their latencies overlap
    const float* sp = s.score_part + (long)b * s.L * s.max_ctx + a;
    float sum = 0.f;
    int l = 0;
    for (; l + 8 <= s.L; l += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = sp[(long)(l + u) * s.max_ctx];
#pragma unroll
      for (int u = 0; u < 8; ++u) sum += v[u];
    }
    for (; l < s.L; ++l) sum += sp[(long)l * s.max_ctx];
    float sj = sum * inv;               // Eq. 2: mean over the L*Hq (layer, head) pairs
    if (s.score_scaled) sj *= inv_sqrt_d;
    s.score[base + a] = sj;
    if (j < n - s.window && j >= s.pinned && sj < s.tau) {
      const uint32_t c = cnt[j] + 1;    // line 4
      cnt[j] = c;
      const int dd = duration(c, s.softness, s.softness_int);  // line 5
      if (dd > 0) {                     // lines 6-7
        frozen_now++;
        fstep[j] = i;
        const int t = s.tick_skip_new ? dd : dd - 1;   // R0: this step's tick applies too
        if (t <= 0) {
          timer[j] = 0;                 // frozen and restored by the same tick (no absence)
          restored++;
        } else {
          timer[j] = t;
          res[j] = tag_now;
        }
      }
    }
  }
  // ---- lines 10-15 for tokens frozen before this step
  uint32_t err = 0;
#pragma unroll
  for (int k = 0; k < kPF; ++k) {
    const int j = n0 + (int)threadIdx.x + k * (int)blockDim.x;
    if (j >= n_end) continue;
    const uint8_t r = pr[k];
    if (r == 1 || r == tag_now) continue;
    const int t = pt[k] - 1;
    if (t <= 0) {
      res[j] = 1;
      timer[j] = 0;
      restored++;
    } else {
      timer[j] = t;
      if (r != 0) res[j] = 0;           // drop the previous step's tag
      if (j >= n - s.window) err |= kErrFrozenInWindow;
    }
  }
  for (int j = n0 + (int)threadIdx.x + kPF * (int)blockDim.x; j < n_end; j += blockDim.x) {   // n > kPF*threads*X
    const uint8_t r = res[j];
    if (r == 1 || r == tag_now) continue;
    const int t = timer[j] - 1;
    if (t <= 0) {
      res[j] = 1;
      timer[j] = 0;
      restored++;
    } else {
      timer[j] = t;
      if (r != 0) res[j] = 0;
      if (j >= n - s.window) err |= kErrFrozenInWindow;
    }
  }
  if (err) atomicOr(s.err, err);
  // block sums of the two counters in one pass
  int f = frozen_now, r = restored;
  for (int o = 16; o > 0; o >>= 1) {
    f += __shfl_xor_sync(0xffffffffu, f, o);
    r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sh[w] = f; sh2[w] = r; }
  __syncthreads();
  if (threadIdx.x == 0) {
    f = 0; r = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { f += sh[k]; r += sh2[k]; }
    SeqStats& st = s.stats[b];
    if (f) atomicAdd(&st.frozen_this_step, f);
    if (r) atomicAdd(&st.restored_tick, r);
    __threadfence();
    if (atomicAdd(s.ticket, 1) == nblocks_total - 1) {  // last decide block: advance the step
      *s.ticket = 0;
      *s.step = i + 1;
    }
  }
}

// Combine: one warp per (b, l, h); lane c < nch reads split c's (m, l); each lane owns d/32
// output elements.  Fixed split order -> deterministic.
__device__ void combine_warp(const DevState& s, int wid, float* __restrict__ o) {
  const int lane = threadIdx.x & 31;
  const int h = wid % s.Hq;
  const int l = (wid / s.Hq) % s.L;
  const int b = wid / (s.Hq * s.L);
  int chunk, nch;
  chunking(s.act_len[b], s.max_splits, s.chunk_min, &chunk, &nch);
  const long it0 = s.item_start[b] + (long)l * nch;
  float M = -INFINITY;
  for (int c = lane; c < nch; c += 32) M = fmaxf(M, s.part_ml[((it0 + c) * s.Hq + h) * 2]);
  for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  const int epl = s.d >= 32 ? s.d / 32 : 1;   // elements per lane (d <= 256 -> <= 8)
  const bool on = lane * epl < s.d;
  float num[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float den = 0.f;
  for (int c0 = 0; c0 < nch; c0 += 32) {
    float wl = 0.f, ll = 0.f;
    if (c0 + lane < nch) {
      const long pi = (it0 + c0 + lane) * s.Hq + h;
      wl = exp2f(s.part_ml[pi * 2] - M);
      ll = s.part_ml[pi * 2 + 1];
    }
    const int cn = min(32, nch - c0);
    if (epl == 4) {
      // 8 chunk vectors in flight at a time, accumulated in chunk order
      for (int cb = 0; cb < cn; cb += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (cb + u < cn)
            v[u] = *reinterpret_cast<const float4*>(s.part_acc + ((it0 + c0 + cb + u) * s.Hq + h) * (long)s.d +
                                                    lane * 4);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (cb + u >= cn) break;
          const float w = __shfl_sync(0xffffffffu, wl, cb + u);
          den = fmaf(__shfl_sync(0xffffffffu, ll, cb + u), w, den);
          num[0] = fmaf(v[u].x, w, num[0]); num[1] = fmaf(v[u].y, w, num[1]);
          num[2] = fmaf(v[u].z, w, num[2]); num[3] = fmaf(v[u].w, w, num[3]);
        }
      }
    } else {
      for (int c = 0; c < cn; ++c) {
        const float w = __shfl_sync(0xffffffffu, wl, c);
        den = fmaf(__shfl_sync(0xffffffffu, ll, c), w, den);
        if (on) {
          const float* src = s.part_acc + ((it0 + c0 + c) * s.Hq + h) * (long)s.d + lane * epl;
          for (int e = 0; e < epl; ++e) num[e] = fmaf(src[e], w, num[e]);
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

// Blocks [0, decide_blocks * B): decide + tick (block x of sequence b); the remaining blocks:
// combine, one warp per (b, l, h).
__global__ void __launch_bounds__(kDecideThreads) post_kernel(DevState s, float* __restrict__ o) {
  pdl_wait();      // every input comes from the attention kernel
  Stamp stamp(s.tl, 2);
  const int nd = s.decide_blocks * s.B;
  if ((int)blockIdx.x < nd) {
    decide_block(s, blockIdx.x / s.decide_blocks, blockIdx.x % s.decide_blocks, s.decide_blocks, nd);
    return;
  }
  const int wid = ((int)blockIdx.x - nd) * (kDecideThreads / 32) + (threadIdx.x >> 5);
  if (wid < s.B * s.L * s.Hq) combine_warp(s, wid, o);
}

// Explicit asr_restore at the boundary before step i (= *s.step); seq = -1 for all.
__global__ void __launch_bounds__(kLedgerThreads) restore_kernel(DevState s, int seq, int level) {
  __shared__ int sh[32];
  const int b = seq >= 0 ? seq : (int)blockIdx.x;
  const int i = *s.step;
  const int n = s.prompt_len[b] + i;  // tokens currently held
  int r = apply_level(s, b, n, level, i);
  r = block_sum_int(r, sh);
  if (threadIdx.x == 0) s.stats[b].pending_restored += r;
}

}  // namespace

void node_pre(KNode& n, const DevState& s, const void* logits, int logits_dtype, float* entropy_out,
              const void* k_new, const void* v_new) {
  n.s = s;
  n.set(0, logits);
  n.set(1, entropy_out);
  n.set(2, k_new);
  n.set(3, v_new);
  const bool lf = logits && logits_dtype == 1;
  const void* f;
  if (s.dtype == 0)
    f = lf ? (const void*)pre_kernel<float, __nv_bfloat16> : (const void*)pre_kernel<__nv_bfloat16, __nv_bfloat16>;
  else
    f = lf ? (const void*)pre_kernel<float, float> : (const void*)pre_kernel<__nv_bfloat16, float>;
  const int blocks = kCl * s.B + s.B * s.L;
  n.finalize(f, dim3((blocks + kCl - 1) / kCl * kCl), dim3(kPreThreads), 0);
}

void node_post(KNode& n, const DevState& s, float* o) {
  n.s = s;
  n.set(0, o);
  const int warps = s.B * s.L * s.Hq;
  const int wpb = kDecideThreads / 32;
  n.finalize((const void*)post_kernel, dim3(s.decide_blocks * s.B + (warps + wpb - 1) / wpb), dim3(kDecideThreads), 0);
}

void node_restore(KNode& n, const DevState& s, int seq, int level) {
  n.s = s;
  n.set(0, seq);
  n.set(1, level);
  n.finalize((const void*)restore_kernel, dim3(seq >= 0 ? 1 : s.B), dim3(kLedgerThreads), 0);
}

}  // namespace asr
