// paper_2512_11221_b200/csrc/asr_internal.h — device-side state shared by the kernels and the
// host orchestrator of libasr.so.  Not part of the public ABI (include/asr.h is).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "asr.h"

namespace asr {

constexpr int kStages = 3;          // pre (entropy+append+recovery), attention, post (combine+decide+next A)
// diagnostic timeline slots: [2k], [2k+1] = start / end of stage k; then phase D detail: end of the
// decide blocks, end of the next-step preparation (A_{i+1}), end of the combine; then phase A detail:
// end of the entropy units, end of the append units, start and end of phase B; the first attention
// CTA's end (with the stage end: the spread of the CTAs' ends); last: release of phase D (its first
// block past griddepcontrol.wait)
constexpr int kTimelineSlots = 2 * kStages + 9 + 11;
// fused-tail detail (max stamps): grid-barrier arrival, release, then per tile-decide warp: decide,
// tick, count, look-back, write; the first tile warp done (min); batch 1: the CTA past the
// attention (all warps), past its wait for phase B
constexpr int kTlTail = 2 * kStages + 9;
// per-warp trace of the fused tail (diagnostics, with the timeline): [CTA * 32 + slot][8] stamps,
// slot = warp (segment settle) or 16 + warp (combine)
constexpr int kTraceRows = 148 * 32, kTraceCols = 8;
__host__ __device__ constexpr bool tl_is_min(int k) {
  return (k < 2 * kStages && !(k & 1)) || k == 2 * kStages + 7 || k == 2 * kStages + 8 || k == kTlTail + 7;
}
constexpr int kEntSplits = 64;      // logits row splits for the entropy reduction

// Residency byte: 1 = Active; 0 = Frozen; 2 / 3 = Frozen during a step of even / odd index (tag used
// by the multi-block decide kernel to tell this step's freezes from older ones without ordering).
__host__ __device__ constexpr bool res_active(uint8_t x) { return x == 1; }
__host__ __device__ constexpr uint8_t res_tag(int step) { return (uint8_t)(2 + (step & 1)); }
constexpr int kMaxDetBaseline = 256;
constexpr int kEvBins = 64;         // Belady histogram bins of the remaining timer

// Per-sequence per-step statistics written by the kernels (read by asr_stats).
struct SeqStats {
  int32_t attended;           // |A_i|
  int32_t frozen_this_step;   // d > 0 in the freeze loop
  int32_t restored_tick;      // restored by the tick (incl. d = 1 freezes under R0)
  int32_t restored_pre;       // restored at the step boundary by explicit asr_restore calls
  int32_t restored_rec;       // restored at the step boundary by the entropy-triggered recovery
  int32_t pending_restored;   // explicit asr_restore since the last step
  int32_t recovery_action;
  int32_t rewalk_requested;
  int32_t entropy_valid;
  float entropy;
  int32_t evicted;            // pressure mode: slots released by this step's freezes
  int32_t prefetched;         // pressure mode: slots allocated for next-step restores (copied this step)
  int32_t demand;             // pressure mode: evicted tokens copied back on demand this step
  int32_t resident;           // pressure mode: tokens holding a slot (after the step)
  int32_t pending_demand;     // pressure mode: demand copies by asr_restore since the last step
  int32_t pad[1];
};

// Detector / ladder state per sequence (R-det, R-ladder).
struct DetState {
  int32_t hist_len, hist_head, level, last_action_step, has_last;
  int32_t pad[3];
};

// Error latch bits (asr_stats_t.device_error).
enum : uint32_t {
  kErrFrozenInWindow = 1u,   // a frozen token inside the protected window
  kErrEmptyActive = 2u,      // |A_i| == 0 (the current token is always active)
  kErrPoolEmpty = 8u,        // pressure mode: no free device slot (pool_tokens too small)
  kErrNotResident = 16u,     // pressure mode: an Active token without a device slot
  kErrStall = 32u,           // a wait inside the attention kernel timed out (phase B never finished)
  kErrCheck = 64u,           // a bounds check of the -DASR_CHECKS build failed (index out of its array)
};

// Bounds checks of the diagnostic build (tools/build.py with ASR_CHECKS=1, -DASR_CHECKS): an index
// outside its array latches kErrCheck (asr_stats reports ASR_E_INVARIANT) instead of corrupting
// memory.  compute-sanitizer is closed on this GPU pool; these checks and the oracle comparisons of
// tools/sanitize.py stand in for it.  Compiled out otherwise.
#ifdef ASR_CHECKS
#define ASR_CHECK(st, cond)                           \
  do {                                                \
    if (!(cond)) atomicOr((st).err, asr::kErrCheck);  \
  } while (0)
#else
#define ASR_CHECK(st, cond) \
  do {                      \
  } while (0)
#endif

// Everything a kernel may need; passed by value (all pointers are device pointers).
struct DevState {
  int B, L, Hq, Hkv, d, max_ctx;
  int cap;                    // max_context (tokens a sequence may hold)
  int dtype;                  // 0 bf16, 1 f32
  int window, pinned, tick_skip_new, score_scaled;
  float tau, softness;
  int softness_int;           // k if k is a positive integer, else 0
  int vocab;
  float ent_temp;
  int det_enable, det_baseline, det_cooldown, wr_window, fr_clear_counts;
  float det_z, det_sigma_floor;
  int max_splits, chunk_min;
  int decide_blocks;          // blocks per sequence of the decide kernel
  int sk_grid;                // > 0: stream-K split of the tensor-core attention over sk_grid CTAs (sk_* below)
  int sk_dyn, sk_chunk;       // 1/sk_dyn of the tiles go out as dynamic chunks of sk_chunk tiles (0: none)
  int32_t* sk_ctr;            // [2] next dynamic chunk, CTAs done with chunks (the last one resets both)
  int sk_bal;                 // 1: rate-balanced static split (sk_weighted below; sk_dyn == 0 only)
  int sk_learn;               // 1: the launch measures its rates / computes later cuts (steps; 0: asr_time_attention)
  float sk_ewma;              // weight of a new rate measurement in the per-CTA rate average (0.5)
  float* sk_w;                // [4][kSkBalMax] per-CTA streaming rates (EWMA), by step parity, double-buffered
  float* sk_f;                // [4][kSkBalMax] cut fractions f_0..f_G (NaN: not computed yet), same buffering
  int* sk_bound;              // [kSkBalMax] this step's static range starts (+ Ts), written by CTA 0
  int pre_in_attn;            // 1: phase A (+B) runs inside the tensor-core attention kernel (batch 1)
  int hist_w;                 // W of Eq. 3's count: 0 = lifetime count, 1..128 = detections in (i-W, i]
  const float* ext_score;     // policy replay (NEXT-2): s_j given per position [B][max_ctx]; NULL = Eq. 2
  const float* ent_given;     // [B] H(logits_prev) computed by the caller (asr_sample_entropy); NULL = from logits
  int ent_div;                // sequences per logits row: 1, or n_layers with per-layer ledgers (NEXT-3)
  unsigned long long* hmask;  // [B][max_ctx][2] finite W: bit t = detection at step hstep - t
  int32_t* hstep;             // [B][max_ctx]    finite W: step of bit 0 (never: a large negative)
  int combine_in_decide;      // 1: the combine runs as extra blocks of the phase-D kernel (small batch)
  int kv_evict_first;         // 1: the attention's KV bulk copies carry an L2 evict_first policy
  int ent_per_unit;           // entropy splits per phase-A unit (divides kEntSplits)
  int layers_per_unit;        // layers per phase-A append unit
  // pressure mode (pool_tokens > 0)
  int pool_mode;              // 0 full residency (slot = b*max_ctx + pos), 1 slot pool
  int evict_min;              // never evict tokens returning in fewer steps (at-freeze policy: evict at >=)
  int evict_policy;           // 0 Belady under pressure (histogram in phase D + evict kernel), 1 at freeze
  int pool_reserve;           // free slots kept beyond the next step's appends + prefetches
  int32_t* ev_hist;           // [kEvBins] resident frozen tokens per remaining timer (min(t, kEvBins-1))
  int32_t* ev_ctrl;           // [4] Belady cut of this step: timer threshold T, quota at T, used, need
  unsigned long long* stall;  // [3] h2d stall ns (cumulative), attention end, prefetch-copy end (stamps)
  long tok_bytes;             // bytes of one token (all layers, K and V)
  long kv_slots;              // device token slots of the KV pool (bounds checks)
  long max_items;             // split-KV partial slots (bounds checks)
  int32_t* slot_of;           // [B][max_ctx] device slot of each position, -1 = evicted (pool mode)
  int32_t* spare;             // [B] slot reserved for the next appended token (pool mode)
  int32_t* free_stack;        // [pool] free slots
  int32_t* free_top;          // [1] number of free slots
  char* host_kv;              // device-mapped pointer of the pinned host mirror (pool mode)
  int mirror_bits;            // 0: bf16 mirror; 8: R-quant INT8 tier (codes + one fp32 scale per row)
  int8_t* host_codes;         // INT8 tier: mapped [B][max_ctx][L][2][Hkv][d] codes
  float* host_scales;         // INT8 tier: mapped [B][max_ctx][L][2][Hkv] scales
  uint8_t* deq;               // INT8 tier: [B][max_ctx] 1 = the device slot holds the dequantised row values
  int32_t* pf_list;           // [2][B][max_ctx] positions to prefetch (timer reached 1), by step parity
  int32_t* pf_count;          // [2][B]
  int32_t* cp_list;           // [B][max_ctx] positions whose slot the copy kernel fills this step
  int32_t* cp_count;          // [B]
  unsigned long long* h2d;    // [1] bytes copied host -> device by the kernels (prefetch + demand)
  // head-sharded mode
  int sharded;                // 1: decide reads tok_score (summed across shards) instead of score_part
  int score_heads;            // H of Eq. 2 (all shards)
  float* tok_score;           // packed [sum_b |A_b|]: entry prefix_b + a = the per-token score sum of
                              // attended index a of sequence b over this shard's heads, all layers
  int32_t* tok_count;         // mapped pinned host int: sum_b |A_b| of the step (the all-reduce count)

  void* kv;                   // pool [B*max_ctx][L][2][Hkv][d]
  uint8_t* res;               // [B][max_ctx] 1 Active / 0 Frozen
  int32_t* timer;             // [B][max_ctx]
  uint32_t* count;            // [B][max_ctx]
  int32_t* fstep;             // [B][max_ctx]
  int32_t* prompt_len;        // [B]
  int32_t* step;              // [1] index of the next (or current) step
  // A_i by step parity p = i & 1 (act_* below): phase D of step i compacts A_{i+1} into parity p^1
  // while step i's kernels still read parity p; recovery and asr_restore recompact parity p in place
  int32_t* act_pos;           // [2][B][max_ctx]
  int32_t* act_slot;          // [2][B][max_ctx] device slot of each attended position
  int32_t* act_len;           // [2][B]
  int32_t* item_start;        // [B+1] attention work list: first item / tile of each sequence
  float* score_part;          // [B][L][max_ctx] per-layer Eq. 2 head sums per attended index
  float* score;               // [B][max_ctx]   s_j per attended index (last step)
  float* part_ml;             // [max_items][Hq][2] (m in log2 domain, l)
  float* part_acc;            // [max_items][Hq][d]
  float* ent_part;            // [B][kEntSplits][3]
  double* hist;               // [B][det_baseline]
  DetState* det;              // [B]
  SeqStats* stats;            // [B]
  uint32_t* err;              // [1]
  int32_t* ticket;            // [1]
  int32_t* pre_ticket;        // [B] last phase-A unit of a sequence runs its phase B (unit_finish)
  unsigned long long* dagg;   // [B][32] per decide block: (step + 1) << 32 | its count of A_{i+1}
  int32_t* redo;              // [1] recovery changed some A_i after the attention started (pre_in_attn)
  int32_t* pre_done;          // [1] = step + 1 once phase B of the step is done
  unsigned* gbar;             // [2] grid barrier of the attention kernel (redo pass, fused tail)
  // fused tail (fuse_tail = 1): the attention kernel itself combines O, decides + ticks and compacts
  // A_{i+1} after a grid barrier (one kernel per step; no phase-D launch).  A_{i+1} is compacted per
  // segment: segment t of sequence b = the positions from A_i[16t] up to A_i[16t+16] (the first from
  // 0, the last through the appended position), placed by a decoupled look-back over seg_flag.
  int fuse_tail;
  int tail_exp;               // diagnostics (ASR_TAIL_EXP): bit 0 no combine, bit 1 dry decide pass first
  int max_tiles;              // ceil(max_ctx / 16): seg_flag row length
  unsigned long long* seg_flag;   // [B][max_tiles] (step+1) << 34 | state << 32 | value
  unsigned long long* tl;     // [kTimelineSlots] diagnostic timeline (globaltimer ns), NULL = off
};

// Offset of the parity-p copy of the act_* lists.
__host__ __device__ inline long act_off(const DevState& s, int p) { return (long)(p & 1) * s.B * s.max_ctx; }

#ifdef __CUDACC__
// Programmatic dependent launch (PDL): a kernel may let its dependent start early, and a dependent
// waits for its programmatic upstream before touching the upstream's outputs.  Both are no-ops
// without a programmatic edge (direct launches, profiled graphs).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// A value the compiler cannot see through (keeps a non-inlined function from being cloned and
// specialised for a constant argument, so a dry run executes the very code of the real run).
__device__ __forceinline__ int opaque(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// Release / acquire synchronisation at GPU scope (cheaper than __threadfence(), which is a
// sequentially consistent fence: MEMBAR.SC.GPU + an L1 invalidation on sm_100).
__device__ __forceinline__ int atom_add_acqrel(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long atom_add_acqrel_u64(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.acq_rel.gpu.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Diagnostic timeline: thread 0 of every block stamps %globaltimer at entry (atomicMin) and exit
// (atomicMax) into tl[2*stage], tl[2*stage+1].  Only when DevState::tl is set (ASR_TIMELINE=1).
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct Stamp {
  unsigned long long* tl;
  int stage;
  __device__ Stamp(unsigned long long* t, int k) : tl(t), stage(k) {
    if (tl && threadIdx.x == 0) atomicMin(&tl[2 * stage], gtimer());
  }
  __device__ ~Stamp() {
    if (tl && threadIdx.x == 0) atomicMax(&tl[2 * stage + 1], gtimer());
  }
};
#endif  // __CUDACC__

__host__ __device__ inline void chunking(int A, int max_splits, int chunk_min, int* chunk, int* nch) {
  int c = (A + max_splits - 1) / max_splits;
  c = (c + 15) & ~15;   // whole 16-token tiles: a partial tile shrinks the bytes in flight of its stage
  if (c < chunk_min) c = chunk_min;
  *chunk = c;
  *nch = (A + c - 1) / c;
}

// Work split of the tensor-core attention (DevState::sk_grid = grid > 0).  The L * ceil(A_b / 16)
// 16-token tiles of all (b, l) items, in (b, l, tile) order, T in total, are handed out as *units*:
// the first Ts tiles are cut into G = min(grid, Ts) contiguous static ranges [floor(cTs/G),
// floor((c+1)Ts/G)), one per CTA (units 0..G-1) — stream-K; the last T/sk_dyn tiles (nchunks chunks
// of C tiles) are taken dynamically (units G + k, chunk k drawn from an atomic ticket) by the CTAs
// that finish their range first: SMs stream at different rates (the last CTA of a purely static
// split ended 25-35 % after the first; profiles/README.md).  The part of item i = b*L + l that unit u
// covers writes its softmax partial to slot i + u (unique and consecutive per item: units grow along
// the tile order), so item i's partials are slots i + sk_unit_of(S_i) .. i + sk_unit_of(S_i +
// tiles_b - 1), S_i = item_start[b] + l * tiles_b; an item inside one unit is written to O directly.
// Slots: at most B*L + G + nchunks <= B*L + grid * (1 + kSkMaxChunksPerCta).
constexpr int kSkTile = 16;
constexpr int kSkMaxChunksPerCta = 8;
__host__ __device__ inline int sk_span(long T, int grid) { return T < grid ? (int)T : grid; }
__host__ __device__ inline int sk_cta_of(long t, long T, int G) { return (int)(((t + 1) * (long)G - 1) / T); }
struct SkPlan {
  long T, Ts;      // tiles, static tiles
  int G, C;        // static ranges, tiles per chunk
  int nchunks;
};
__host__ __device__ inline SkPlan sk_plan(long T, int grid, int dyn_div, int chunk) {
  SkPlan p;
  p.T = T;
  const long td = dyn_div > 0 ? T / dyn_div : 0;   // tiles handed out dynamically
  long c = chunk > 0 ? chunk : 1;
  const long cmin = (td + (long)kSkMaxChunksPerCta * grid - 1) / ((long)kSkMaxChunksPerCta * grid);
  if (c < cmin) c = cmin;                          // bounded slot count
  p.C = (int)c;
  p.nchunks = (int)(td / p.C);
  p.Ts = T - (long)p.nchunks * p.C;
  p.G = sk_span(p.Ts, grid);
  return p;
}
__host__ __device__ inline int sk_unit_of(const SkPlan& p, long t) {
  return t < p.Ts ? sk_cta_of(t, p.Ts, p.G) : p.G + (int)((t - p.Ts) / p.C);
}
// Rate-balanced static split (DevState::sk_bal, static split only): SMs stream at different but
// stable rates (profiles/README.md: per-CTA durations correlate 0.99 between the halves of a run,
// with a step-parity component), so the static ranges are cut in proportion to each CTA's measured
// rate: range c = [floor(T f_c), floor(T f_{c+1})), f_c = P_c / P_G, P the prefix sums of the rates
// normalised by their mean and clamped to [0.5, 2] — with T >= 8G every range holds >= 2 tiles and
// the slot scheme above is unchanged.  Each CTA measures its rate (tiles per clock) over its first
// pass and folds it (EWMA 1/2) into the other buffer of its step parity; one warp computes the
// fractions for step i + 2 from the rates of step i - 2 beside step i's attention (so no launch
// reads what it writes, and nothing of it sits on the critical path); each CTA then needs f_c and
// f_{c+1} only, and stores its range start in sk_bound for the combine.  Only the order of the
// partial sums in the softmax combine depends on the split (O within fp32 rounding; scores and
// decisions do not).
constexpr int kSkBalMax = 256;      // grid <= 255 (the + 1 boundary fits)
constexpr int kSkBalPer = kSkBalMax / 32;
__host__ __device__ inline bool sk_weighted(int sk_bal, const SkPlan& p) {
  return sk_bal && p.nchunks == 0 && p.Ts >= 8L * p.G;
}
__host__ __device__ inline int sk_wbuf(int step, bool write) {
  return (step & 1) * 2 + (((step >> 1) & 1) ^ (write ? 1 : 0));
}

// One kernel launch described as data, so the same description serves a direct launch
// (cudaLaunchKernel) and a CUDA-graph kernel node (cudaGraphAddKernelNode /
// cudaGraphExecKernelNodeSetParams when a caller pointer changes).
struct KNode {
  cudaKernelNodeParams p{};
  DevState s{};
  uint64_t extra[6] = {0, 0, 0, 0, 0, 0};   // pointer / int arguments after DevState (8-byte slots)
  void* argv[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  // step-graph dependencies (indices into the step's node list): full edges and at most one
  // programmatic (PDL) edge; a node with none is a root of the graph
  int dep_full[2] = {-1, -1};
  int dep_prog = -1;
  void finalize(const void* func, dim3 grid, dim3 block, unsigned smem) {
    argv[0] = &s;
    for (int k = 0; k < 6; ++k) argv[k + 1] = &extra[k];
    p.func = const_cast<void*>(func);
    p.gridDim = grid;
    p.blockDim = block;
    p.sharedMemBytes = smem;
    p.kernelParams = argv;
    p.extra = nullptr;
  }
  template <typename P>
  void set(int k, P v) {
    extra[k] = 0;
    static_assert(sizeof(P) <= 8, "arg too large");
    memcpy(&extra[k], &v, sizeof(P));
  }
  cudaError_t launch(cudaStream_t st) const {
    return cudaLaunchKernel(p.func, p.gridDim, p.blockDim, const_cast<void**>(argv), p.sharedMemBytes, st);
  }
};

// NCCL entry points, resolved with dlopen at first use (nccl_dl.cpp); head-sharded mode only.
struct NcclApi {
  bool ok = false;
  int (*get_unique_id)(void* out128) = nullptr;
  int (*comm_init_rank)(void** comm, int nranks, const void* id128, int rank) = nullptr;
  int (*all_reduce)(const void* send, void* recv, size_t count, int dtype, int op, void* comm,
                    cudaStream_t st) = nullptr;
  int (*comm_destroy)(void* comm) = nullptr;
  const char* (*get_error)(int rc) = nullptr;
  const char* err(int rc) const { return get_error ? get_error(rc) : "nccl error"; }
};
NcclApi& nccl_api();

// Node builders (kernels_*.cu).
void node_phaseA(KNode& n, const DevState& s, const void* logits, int logits_dtype, const void* k_new,
                 const void* v_new, float* entropy_out);
void node_attention(KNode& n, const DevState& s, const void* q, const void* k_new, const void* v_new, int grid,
                    const void* pre_logits, int logits_dtype, float* entropy_out, float* o);
void node_phaseD(KNode& n, const DevState& s, float* o);
void node_combine(KNode& n, const DevState& s, float* o);
void node_prepare(KNode& n, const DevState& s);            // A_0 at asr_create
void node_restore(KNode& n, const DevState& s, int seq, int level);
void node_copy(KNode& n, const DevState& s, int grid);   // pressure mode: prefetch copies
void node_evict(KNode& n, const DevState& s, int grid);  // pressure mode: Belady eviction after phase D
void node_scoresum(KNode& n, const DevState& s);          // head-sharded mode: layer sums -> tok_score
int attention_grid(const DevState& s, int num_sms);
cudaError_t launch_sample(const void* logits, int logits_dtype, int batch, int vocab, float temperature, int top_k,
                          float top_p, const float* uniforms, int32_t* token_out, float ent_temp, float* entropy_out,
                          cudaStream_t st);   // NEXT-1 (+ the row's entropy in the same pass)
cudaError_t launch_kv_quantize(const void* kv, long rows, int n, int bits, int8_t* codes, float* scales,
                               cudaStream_t st);   // NEXT-4
cudaError_t launch_kv_dequantize(const int8_t* codes, const float* scales, long rows, int n, int bits, void* kv,
                                 cudaStream_t st);  // NEXT-4
bool attention_mma_supported(const DevState& s);   // bf16, d=128, 1/2/4/8 KV heads, <= 4 (8) q heads per KV head
cudaError_t attention_mma_prepare();               // opt-in to > 48 KiB dynamic shared memory
void attention_mma_launch_shape(const DevState& s, bool logits_f32, const void** func, int* threads, unsigned* smem);

}  // namespace asr
