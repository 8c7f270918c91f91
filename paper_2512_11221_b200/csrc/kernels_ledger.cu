// paper_2512_11221_b200/csrc/kernels_ledger.cu — the ledger side of one ASR-KF-EGR step (sm_100a):
//   entropy_kernel     (a6) H(logits_prev), spike detector, recovery ladder   (Sec 3.6)
//   ledger_pre_kernel  (a0) append + (a6) recovery levels + (a3) compaction of A_i (Alg. 1)
//   decide_kernel      (a2) Eq. 2 finish, threshold, Eq. 3 schedule, freeze, tick (Alg. 1 lines 3-15)
//   restore_kernel     explicit SR / WR / FR (asr_restore)
// All reductions are in a fixed order, so the step is bitwise deterministic.
#include <cuda_bf16.h>
#include <math.h>

#include "asr_internal.h"

namespace asr {
namespace {

__device__ __forceinline__ float ldf(const void* p, long i, int dtype) {
  if (dtype == 0) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  return reinterpret_cast<const float*>(p)[i];
}

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
// Single pass per split: m = max x/T, Z = sum e^{x/T - m}, S = sum e^{x/T - m} (x/T - m);
// H = ln Z - S/Z.  The last block of a row (atomic ticket) merges the splits in split order,
// then runs the detector (R-det) and the ladder (R-ladder) in double precision.
__global__ void __launch_bounds__(256) entropy_kernel(DevState s, const void* logits, int ldt,
                                                      float* entropy_out) {
  const int split = blockIdx.x, b = blockIdx.y;
  const int V = s.vocab;
  const int seg = (V + kEntSplits - 1) / kEntSplits;
  const int v0 = split * seg, v1 = min(V, v0 + seg);
  const void* row = ldt == 0 ? (const void*)((const __nv_bfloat16*)logits + (long)b * V)
                             : (const void*)((const float*)logits + (long)b * V);
  const float invT = 1.0f / s.ent_temp;
  __shared__ float shm[32], shz[32], shs[32];
  __shared__ int last;
  // pass 1: max
  float m = -INFINITY;
  for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) m = fmaxf(m, ldf(row, v, ldt) * invT);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) shm[w] = m;
  __syncthreads();
  m = -INFINITY;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = fmaxf(m, shm[i]);
  // pass 2: Z and S relative to the block max
  float z = 0.f, sx = 0.f;
  for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
    float x = ldf(row, v, ldt) * invT - m;
    float e = expf(x);
    z += e;
    sx += e * x;
  }
  for (int o = 16; o > 0; o >>= 1) {
    z += __shfl_xor_sync(0xffffffffu, z, o);
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
  }
  if (lane == 0) { shz[w] = z; shs[w] = sx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    z = 0.f; sx = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { z += shz[i]; sx += shs[i]; }
    float* ep = s.ent_part + ((long)b * kEntSplits + split) * 3;
    ep[0] = m; ep[1] = z; ep[2] = sx;
    __threadfence();
    last = atomicAdd(&s.ent_ticket[b], 1) == kEntSplits - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  // merge splits in order (double)
  const volatile float* ep = s.ent_part + (long)b * kEntSplits * 3;
  double M = -INFINITY;
  for (int i = 0; i < kEntSplits; ++i)
    if (ep[i * 3 + 1] > 0.f) M = fmax(M, (double)ep[i * 3]);
  double Z = 0.0, S = 0.0;
  for (int i = 0; i < kEntSplits; ++i) {
    double zi = ep[i * 3 + 1];
    if (zi <= 0.0) continue;
    double dm = (double)ep[i * 3] - M, f = exp(dm);
    Z += zi * f;
    S += f * ((double)ep[i * 3 + 2] + zi * dm);
  }
  const double H = log(Z) - S / Z;
  s.ent_ticket[b] = 0;
  if (entropy_out) entropy_out[b] = (float)H;
  SeqStats& st = s.stats[b];
  st.entropy = (float)H;
  st.entropy_valid = 1;
  // detector: H > mean + z * max(sigma, floor) over the previous <= det_baseline values
  DetState& ds = s.det[b];
  double* hist = s.hist + (long)b * s.det_baseline;
  int trig = 0;
  if (s.det_enable && ds.hist_len >= 2) {
    double mu = 0.0;
    for (int t = 0; t < ds.hist_len; ++t) mu += hist[t];
    mu /= ds.hist_len;
    double var = 0.0;
    for (int t = 0; t < ds.hist_len; ++t) var += (hist[t] - mu) * (hist[t] - mu);
    var /= ds.hist_len;
    double sd = fmax(sqrt(var), (double)s.det_sigma_floor);
    trig = H > mu + (double)s.det_z * sd;
  }
  if (ds.hist_len < s.det_baseline) {
    hist[ds.hist_len++] = H;
  } else {
    hist[ds.hist_head] = H;
    ds.hist_head = (ds.hist_head + 1) % s.det_baseline;
  }
  int level = 0;
  if (trig) {
    const int i = *s.step;
    const int dt = i - ds.last_action_step;
    if (ds.has_last && dt < s.det_cooldown) {
      level = 0;  // absorbed
    } else {
      if (ds.has_last && dt < 2 * s.det_cooldown) level = ds.level < 4 ? ds.level + 1 : 4;
      else level = 1;
      ds.level = level;
      ds.last_action_step = i;
      ds.has_last = 1;
    }
  }
  s.rec_action[b] = level;
}

// Recovery levels on one sequence's ledger: returns the restored count of this thread.
__device__ int apply_level(const DevState& s, int b, int n, int level, int i) {
  int restored = 0;
  uint8_t* res = s.res + (long)b * s.max_ctx;
  int32_t* timer = s.timer + (long)b * s.max_ctx;
  const int32_t* fstep = s.fstep + (long)b * s.max_ctx;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    if (res[j] != 0) continue;
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

// ------------------------------------------------------------------ (a0) + recovery + (a3) compaction
// Blocks [0, B): the ledger of sequence b.  Blocks [B, B + B*L): append the new token's K/V rows
// of (b, l) into its slot of the pool.
template <typename T>
__global__ void __launch_bounds__(kLedgerThreads) ledger_pre_kernel(DevState s, const T* k_new,
                                                                    const T* v_new, int has_entropy) {
  const int i = *s.step;
  if ((int)blockIdx.x >= s.B) {  // ---- append K/V rows
    const int r = blockIdx.x - s.B;
    const int b = r / s.L, l = r % s.L;
    const long pos = s.prompt_len[b] + i;
    const long slot = (long)b * s.max_ctx + pos;
    const int row = s.Hkv * s.d;  // elements of K (or V) per token-layer
    T* dst = reinterpret_cast<T*>(s.kv) + (slot * s.L + l) * 2 * row;
    const T* ks = k_new + ((long)b * s.L + l) * row;
    const T* vs = v_new + ((long)b * s.L + l) * row;
    const int vec = (int)(16 / sizeof(T));
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
  // ---- ledger of sequence b
  __shared__ int sh[32];
  __shared__ int wsum[32];
  const int b = blockIdx.x;
  const int n = s.prompt_len[b] + i + 1;  // total after the append
  const long base = (long)b * s.max_ctx;
  SeqStats& st = s.stats[b];
  if (threadIdx.x == 0) {
    const int j = n - 1;  // the token produced by the previous step (Alg. 1 line 16)
    s.res[base + j] = 1;
    s.timer[base + j] = 0;
    s.count[base + j] = 0;
    s.fstep[base + j] = -1;
  }
  int level = has_entropy ? s.rec_action[b] : 0;
  int restored = 0;
  if (level > 0) restored = apply_level(s, b, n - 1, level, i);
  restored = block_sum_int(restored, sh);  // includes a __syncthreads
  if (threadIdx.x == 0) {
    st.restored_this_step = st.pending_restored + restored;
    st.pending_restored = 0;
    st.recovery_action = level;
    st.rewalk_requested = level == 4;
    if (!has_entropy) st.entropy_valid = 0;
    st.frozen_this_step = 0;
  }
  // compaction: each thread owns a contiguous segment of positions
  const int seg = (n + blockDim.x - 1) / blockDim.x;
  const int j0 = min(n, (int)threadIdx.x * seg), j1 = min(n, j0 + seg);
  const uint8_t* res = s.res + base;
  int cnt = 0;
  for (int j = j0; j < j1; ++j) cnt += res[j];
  // exclusive block scan of cnt
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
    int xi = x;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    wsum[lane] = xi - x;  // exclusive warp offsets
  }
  __syncthreads();
  int off = wsum[w] + incl - cnt;
  int32_t* out = s.act_pos + base;
  for (int j = j0; j < j1; ++j)
    if (res[j]) out[off++] = j;
  if (threadIdx.x == blockDim.x - 1) {
    s.act_len[b] = off;
    st.attended = off;
    if (off == 0) atomicOr(s.err, kErrEmptyActive);
  }
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

__global__ void __launch_bounds__(kLedgerThreads) decide_kernel(DevState s) {
  __shared__ int sh[32];
  const int b = blockIdx.x;
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
  // Alg. 1 lines 3-9 (each attended token is visited by exactly one thread)
  int frozen_now = 0;
  for (int a = threadIdx.x; a < A; a += blockDim.x) {
    const int j = s.act_pos[base + a];
    float sum = 0.f;
    for (int l = 0; l < s.L; ++l) sum += s.score_part[((long)b * s.L + l) * s.max_ctx + a];
    float sj = sum * inv;               // Eq. 2: mean over the L*Hq (layer, head) pairs
    if (s.score_scaled) sj *= inv_sqrt_d;
    s.score[base + a] = sj;
    if (j < n - s.window && j >= s.pinned && sj < s.tau) {
      const uint32_t c = cnt[j] + 1;    // line 4
      cnt[j] = c;
      const int dd = duration(c, s.softness, s.softness_int);  // line 5
      if (dd > 0) {                     // lines 6-7
        res[j] = 0;
        timer[j] = dd;
        fstep[j] = i;
        frozen_now++;
      }
    }
  }
  __syncthreads();
  // Alg. 1 lines 10-15: tick every frozen token (R0: including those frozen above)
  int restored = 0;
  uint32_t err = 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    if (res[j] != 0) continue;
    if (s.tick_skip_new && fstep[j] == i) continue;
    const int t = timer[j] - 1;
    if (t <= 0) {
      res[j] = 1;
      timer[j] = 0;
      restored++;
    } else {
      timer[j] = t;
      if (j >= n - s.window) err |= kErrFrozenInWindow;
    }
  }
  if (err) atomicOr(s.err, err);
  frozen_now = block_sum_int(frozen_now, sh);
  restored = block_sum_int(restored, sh);
  if (threadIdx.x == 0) {
    SeqStats& st = s.stats[b];
    st.frozen_this_step = frozen_now;
    st.restored_this_step += restored;
    st.active_post = A - frozen_now + restored;
    __threadfence();
    if (atomicAdd(s.ticket, 1) == (int)gridDim.x - 1) {  // last sequence: advance the step
      *s.ticket = 0;
      *s.step = i + 1;
    }
  }
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

cudaError_t launch_entropy(const DevState& s, const void* logits, int logits_dtype, float* entropy_out,
                           cudaStream_t st) {
  entropy_kernel<<<dim3(kEntSplits, s.B), 256, 0, st>>>(s, logits, logits_dtype, entropy_out);
  return cudaGetLastError();
}

cudaError_t launch_ledger_pre(const DevState& s, const void* k_new, const void* v_new, int has_entropy,
                              cudaStream_t st) {
  const int grid = s.B + s.B * s.L;
  if (s.dtype == 0)
    ledger_pre_kernel<__nv_bfloat16><<<grid, kLedgerThreads, 0, st>>>(
        s, (const __nv_bfloat16*)k_new, (const __nv_bfloat16*)v_new, has_entropy);
  else
    ledger_pre_kernel<float><<<grid, kLedgerThreads, 0, st>>>(s, (const float*)k_new, (const float*)v_new,
                                                              has_entropy);
  return cudaGetLastError();
}

cudaError_t launch_decide(const DevState& s, cudaStream_t st) {
  decide_kernel<<<s.B, kLedgerThreads, 0, st>>>(s);
  return cudaGetLastError();
}

cudaError_t launch_restore(const DevState& s, int seq, int level, cudaStream_t st) {
  restore_kernel<<<seq >= 0 ? 1 : s.B, kLedgerThreads, 0, st>>>(s, seq, level);
  return cudaGetLastError();
}

}  // namespace asr
