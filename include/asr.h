/* include/asr.h — C ABI of the B200-native ASR-KF-EGR per-decode-step KV-management hot path.
 *
 * Method: "Adaptive Soft Rolling KV Freeze with Entropy-Guided Recovery", arXiv 2512.11221.
 * P:n below is line n of the paper text (/root/reference/PAPER.md, section legend in SURVEY.md);
 * readings of ambiguous passages are listed in DESIGN.md §"Readings" (R-tick, R-W, R-win, ...).
 *
 * One context (asr_ctx) owns B sequences.  Each asr_step runs Alg. 1 lines 1-15 for
 * every sequence and every layer on the GPU, with no host synchronisation:
 *   (a0) append the previous step's token K/V (Alg. 1 line 16 of the previous step)
 *   (a6) entropy of logits_prev + spike detector + recovery ladder SR->WR->FR->RR (Sec 3.6)
 *   (a3) compact the active index list A_i (Alg. 1 "Active KV cache A")
 *   (a4) decode attention softmax(q K_A^T / sqrt(d)) V_A over A_i only (Eq. 1; line 1)
 *   (a1) relevance s_j = (1/H) sum_h |q^(h) . k_j^(h)| fused into (a4) (Eq. 2; line 2)
 *   (a2) threshold s_j < tau outside the window, c_j += 1, d_j = floor(sqrt(c_j)/k), freeze if d_j > 0,
 *        then tick every frozen timer and restore at d_j <= 0 (Eq. 3; lines 3-15 P:89-101)
 *   (a5) frozen KV lives in a write-once pinned host mirror (Sec 3.3); see asr_config.
 * All calls return asr_status.  Thread-compatible: one thread at a time per context.
 * Errors: argument / configuration errors are detected synchronously and change nothing;
 * device-side invariant violations latch a flag that surfaces as ASR_E_INVARIANT from the next
 * asr_step / asr_stats.  asr_last_error() gives a one-line, thread-local message.
 */
#ifndef ASR_H
#define ASR_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct asr_ctx asr_ctx;

typedef enum {
  ASR_OK = 0,
  ASR_E_INVALID = 1,   /* bad argument or configuration (nothing was changed) */
  ASR_E_INVARIANT = 2, /* device-detected ledger invariant violation (latched) */
  ASR_E_CUDA = 3,      /* CUDA runtime error */
  ASR_E_OOM = 4,       /* device or pinned-host allocation failed */
  ASR_E_CAPACITY = 5,  /* a sequence would exceed max_context */
  ASR_E_NCCL = 6,      /* NCCL error (head-sharded mode), or libnccl.so.2 not loadable */
  ASR_E_STATE = 7      /* call order (e.g. use after destroy) */
} asr_status;

typedef enum { ASR_KV_BF16 = 0, ASR_KV_F32 = 1 } asr_dtype;
/* asr_step_io.logits_dtype = ASR_ENTROPY_GIVEN: logits_prev points to fp32 H[batch], the entropy of the
 * previous step's logits rows already taken by asr_sample_entropy (one read of each row yields both the
 * next token and H); the step skips its own pass over the rows. */
enum { ASR_ENTROPY_GIVEN = 2 };
typedef enum { ASR_TICK_LITERAL = 0 /* R0: Alg. 1 order, default */, ASR_TICK_SKIP_NEW = 1 /* R1 */ } asr_tick;
typedef enum { ASR_SCORE_RAW = 0 /* Eq. 2 literal, default */, ASR_SCORE_SCALED = 1 /* x 1/sqrt(d) */ } asr_score_mode;
typedef enum { ASR_SR = 1, ASR_WR = 2, ASR_FR = 3 } asr_level; /* P:80; RR = FR + rewalk flag */
typedef enum { ASR_MEM_DEVICE = 0, ASR_MEM_HOST = 1 } asr_memory;

typedef struct {
  /* model shape: Hq % Hkv == 0; query head h reads KV head h / (Hq/Hkv) (GQA, R-gqa);
   * head_dim in {16, 32, 64, 128, 256} */
  int32_t n_layers, n_q_heads, n_kv_heads, head_dim;
  int32_t batch;          /* B sequences in this context */
  int32_t max_context;    /* tokens per sequence (capacity) */
  int32_t kv_dtype;       /* asr_dtype of q, k, v (and of the pool) */
  int32_t window;         /* K >= 1: positions >= n-K are never frozen (R-win) */
  float tau;              /* threshold, strict s_j < tau */
  float softness;         /* k > 0 of Eq. 3 */
  int32_t history_window; /* W of Eq. 3's count c_j: 0 = lifetime (R-W, default, Table-pinned);
                             1..128 = detections within the last W steps (a per-token bitmask) */
  int32_t pinned_prefix;  /* positions < pinned_prefix are never frozen (R-sink, default 0) */
  int32_t score_mode;     /* asr_score_mode */
  int32_t tick_order;     /* asr_tick */
  int32_t vocab;          /* logits row length for the entropy stage (0 = entropy off) */
  float entropy_temperature;                  /* T_ent (R-ent), default 1 */
  int32_t det_enable;     /* spike detector on (R-det) */
  int32_t det_baseline;   /* previous entropies in the detector window (<= 256), default 64 */
  int32_t det_cooldown;   /* ladder cooldown (R-ladder), default 16 */
  int32_t wr_window;      /* N of WR "last N steps", default = window */
  float det_z;            /* z threshold, default 3 */
  float det_sigma_floor;  /* sigma floor in nats, default 0.05 */
  int32_t fr_clear_counts;/* FR also clears detection counts (SPEC reading), default 0 */
  int32_t host_mirror;    /* 1 = keep the write-once pinned host copy of every token's KV */
  int32_t profile_stages; /* 1 = record CUDA events around every stage (asr_stage_times) */
  int32_t device;         /* CUDA device ordinal */
  int32_t evict_min_absence; /* pressure mode: tokens returning in fewer than this many steps are never
                                evicted (default 2; a token back next step would be copied right back) */
  int32_t pool_reserve;   /* pressure mode: device slots kept free beyond the next step's appends and
                           * prefetches, for demand restores (recovery / asr_restore); 0 = batch */
  int64_t pool_tokens;    /* 0: full residency (every token keeps its device slot; freezing only flips
                           * its residency bit).  > 0: pressure mode (Sec 3.3, "moves the token's
                           * KV pair from GPU to CPU"): the device holds pool_tokens token slots; frozen
                           * tokens are evicted to the pinned host mirror and prefetched back one step
                           * before their timer expires; entropy-triggered / explicit restores of
                           * evicted tokens are copied back on demand.  Needs host_mirror = 1. */
  int32_t score_heads;    /* head-sharded mode: H of Eq. 2's 1/H over ALL shards (the context holds only
                           * n_q_heads of them); 0 = n_q_heads (unsharded).  The per-token partial sums
                           * must then be summed across shards between asr_step_attend and
                           * asr_step_decide (asr_attach_nccl does it inside asr_step). */
  int32_t evict_policy;   /* pressure mode (Sec 3.3): ASR_EVICT_BELADY (default): frozen tokens
                           * keep their device slots until the pool runs short; then, after each step,
                           * the resident frozen tokens returning LAST (largest remaining timer: the
                           * return step is known at freeze time, Eq. 3) are evicted until the free
                           * slots cover the next step's appends + prefetches + pool_reserve.
                           * ASR_EVICT_AT_FREEZE: every token frozen for >= evict_min_absence steps
                           * is evicted when it freezes (round-1 policy, kept for comparison). */
  int32_t mirror_bits;    /* pressure mode, bf16 KV, head_dim a multiple of 32: 0 = the host mirror holds
                           * bf16 rows; 8 = the quantised frozen tier (NEXT-4, R-quant): every row
                           * (token, layer, K|V, KV head) stored as INT8 codes + one fp32 scale, written
                           * at append, dequantised into the device slot on prefetch / demand restore
                           * (1.94x fewer host-link bytes at d = 128; lossy by R-quant's bound) */
  int32_t per_layer_ledgers; /* NEXT-3 ("per-token granularity" made per (token, layer)): 0 = one
                           * ledger per sequence, s_j the mean over all layers' heads (R-layer, default);
                           * 1 = one ledger per (sequence, layer): layer l freezes token j on its own
                           * score s_j^(l) = (1/Hq) sum_h |q_l,h . k_l,j,h| and attends its own active
                           * list.  The context then holds batch * n_layers virtual sequences of one
                           * layer each: every per-sequence call (asr_stats, asr_restore, asr_read_kv,
                           * asr_step_policy's score rows) indexes seq = b * n_layers + l; the step's
                           * q / k_new / v_new / o keep their [batch][n_layers] shapes; logits_prev /
                           * entropy stay [batch] (ASR_ENTROPY_GIVEN avoids n_layers passes per row). */
} asr_config;
typedef enum { ASR_EVICT_BELADY = 0, ASR_EVICT_AT_FREEZE = 1 } asr_evict_policy;

/* Fills *cfg with the paper's defaults (K=32, tau=0.5, k=2: P:112) and LLaMA-3-8B shape. */
void asr_config_defaults(asr_config* cfg);

/* Per-step buffers, owned by the CALLER.
 * memory = ASR_MEM_DEVICE: device pointers, valid until the caller's stream passes the step; o and
 *   entropy are complete at that point.
 * memory = ASR_MEM_HOST: host pointers (pinned for asynchrony).  The library copies the inputs into
 *   one of two device staging sets on its own copy stream as soon as the step is issued (overlapping
 *   the previous step's kernels) and copies o / entropy back on a second copy stream while the next
 *   step computes.  Inputs may be reused once the caller's stream passes the step; outputs are
 *   complete after asr_flush() has been ordered on a stream and that stream passes it, or after
 *   asr_stats() / asr_destroy().  Bytes are counted in asr_stats_t.bytes_h2d / bytes_d2h. */
typedef struct {
  const void* q;           /* [B][L][Hq][d]  kv_dtype: the current query Q_i (Eq. 1-2) */
  const void* k_new;       /* [B][L][Hkv][d] kv_dtype: K of the token appended this step */
  const void* v_new;       /* [B][L][Hkv][d] kv_dtype */
  const void* logits_prev; /* [B][vocab] or NULL: the previous step's output logits (Sec 3.6); or fp32 [B]
                            * entropies with ASR_ENTROPY_GIVEN */
  int32_t logits_dtype;    /* ASR_KV_BF16, ASR_KV_F32 or ASR_ENTROPY_GIVEN */
  int32_t memory;          /* asr_memory of every pointer in this struct */
  float* o;                /* out [B][L][Hq][d] fp32 attention output over A_i */
  float* entropy;          /* out [B] fp32 H(logits_prev), or NULL */
} asr_step_io;

typedef struct {
  int64_t step;               /* index i of the last completed step (-1 before the first) */
  int64_t total;              /* n = tokens held after that step */
  int64_t attended;           /* |A_i| attended in that step */
  int64_t active;             /* Active after the tick (Table 1/3 "Active KV" convention) */
  int64_t frozen;             /* total - active */
  int64_t frozen_this_step;   /* tokens given d>0 (incl. d=1 ones the same tick restores, R0) */
  int64_t restored_this_step; /* tick restores + recovery + explicit asr_restore since last step */
  double compression;         /* 1 - active/total (Tables 1/3) */
  float entropy;              /* H(logits_prev) in nats */
  int32_t entropy_valid;
  int32_t recovery_action;    /* 0 none, 1 SR, 2 WR, 3 FR, 4 RR */
  int32_t rewalk_requested;   /* RR: the caller should regenerate (needs the model; out of scope) */
  int64_t bytes_h2d, bytes_d2h; /* host-link bytes moved by the library for this context so far */
  uint32_t device_error;      /* latched invariant flags (0 = none): 1 a frozen token inside the
                               * protected window, 2 an empty active set, 8 pressure mode found no free
                               * device slot, 16 an active token without a device slot, 32 a wait inside
                               * the batch-1 attention kernel timed out */
  int64_t resident;           /* tokens of this sequence holding a device slot (pressure mode; else total) */
  int64_t evicted_this_step;  /* device slots released by this step's freezes (pressure mode) */
  int64_t prefetched_this_step; /* tokens copied host -> device ahead of their timer expiry */
  int64_t demand_restored_this_step; /* evicted tokens copied back on demand (recovery / asr_restore) */
  int64_t h2d_stall_ns;       /* context-wide, cumulative: device time the steps waited on the host link
                               * (demand copies before compaction + prefetch copies outlasting the
                               * attention kernel), %globaltimer on the device (pressure mode) */
  int64_t free_slots;         /* pressure mode: free device slots after the last step (else 0) */
  int64_t allreduce_bytes;    /* head-sharded mode, context-wide, cumulative: bytes of per-token partial
                               * sums all-reduced by asr_step (4 per attended token of the batch) */
} asr_stats_t;

/* Host buffers for a full ledger snapshot of one sequence (any pointer may be NULL). */
typedef struct {
  uint8_t* residency;     /* [capacity] 1 Active, 0 Frozen (positions < total) */
  int32_t* timer;         /* [capacity] d_j */
  uint32_t* count;        /* [capacity] c_j */
  int32_t* freeze_step;   /* [capacity] step of the last freeze, -1 never */
  int32_t* active_list;   /* [capacity] A_i of the last step (sorted positions) */
  int32_t* active_len;    /* [1] |A_i| */
  float* scores;          /* [capacity] s_j per attended index of the last step */
  int32_t capacity;       /* length of the arrays above (>= total) */
  uint8_t* dequantized;   /* [capacity] INT8 tier (mirror_bits = 8): 1 = the token's device slot holds its
                           * dequantised rows (it was copied back from the quantised mirror) */
} asr_ledger_view;

/* Create a context: allocates the device KV pool [B][max_context][L][2][Hkv][d], the ledger and
 * workspaces (and the pinned mirror if host_mirror), then prefills prompt_len[b] tokens of each
 * sequence as Active with c = d = 0 (no decisions at prefill, R-prefill).
 *   prompt_k, prompt_v: [B][prompt_stride][L][Hkv][d] kv_dtype in `memory` (NULL if all lengths 0)
 *   prompt_len: host [B], 0 <= prompt_len[b] <= prompt_stride, prompt_len[b] < max_context
 * Returns after the prompt copies complete.  *out is NULL on failure. */
asr_status asr_create(const asr_config* cfg, const void* prompt_k, const void* prompt_v,
                      const int32_t* prompt_len, int32_t prompt_stride, int32_t memory,
                      void* cuda_stream, asr_ctx** out);

/* One generation step for every sequence (asynchronous on cuda_stream, no host sync).
 * ASR_E_CAPACITY if any sequence is full (nothing is changed). */
asr_status asr_step(asr_ctx* ctx, const asr_step_io* io, void* cuda_stream);

/* The two halves of asr_step, for head-sharded contexts (score_heads > n_q_heads):
 * asr_step_attend runs append, entropy/recovery, compaction, attention + score and leaves this
 * shard's per-token partial score sums (over its heads and all layers) in a device buffer;
 * asr_step_decide runs combine + decide + tick reading the (summed) buffer.  Every shard must see the
 * same inputs except q / k_new / v_new, which hold its own heads; their ledgers stay identical. */
asr_status asr_step_attend(asr_ctx* ctx, const asr_step_io* io, void* cuda_stream);
asr_status asr_step_decide(asr_ctx* ctx, void* cuda_stream);
/* Device buffer of the last asr_step_attend's per-token partial score sums, packed: sequence b's
 * attended index a at (sum over b' < b of |A_b'|) + a, count = sum over b of |A_b| fp32 values; sum
 * it element-wise across shards (e.g. an NCCL all-reduce) before asr_step_decide.  Synchronises the
 * context's stream (the count is produced on the device). */
asr_status asr_score_partials(asr_ctx* ctx, float** dev_ptr, int64_t* count);
/* Head-sharded mode over NCCL (NVLink/NVSwitch): rank 0 creates an id (128 bytes), every rank
 * passes it to asr_attach_nccl (collective; one GPU per rank); from then on asr_step runs attend,
 * an in-place ncclAllReduce (sum) of the packed per-token partial sums (4 bytes per attended token;
 * the host reads the count from mapped memory after the attention, one host wait per step) on the
 * step's stream, and decide.  Needs libnccl.so.2 in the process (loaded with dlopen); NCCL failures
 * return ASR_E_NCCL. */
asr_status asr_nccl_unique_id(void* out, int32_t n);
asr_status asr_attach_nccl(asr_ctx* ctx, const void* unique_id, int32_t nranks, int32_t rank);

/* Explicit recovery at the boundary before the next step: SR restores frozen tokens with
 * d > 1, WR those frozen in the last wr_window steps, FR all.  seq = -1 applies to all. */
asr_status asr_restore(asr_ctx* ctx, int32_t seq, int32_t level, void* cuda_stream);

/* Statistics of the last step for one sequence; optional ledger snapshot.  Synchronises the
 * context's stream.  ASR_E_INVARIANT if a device invariant was violated. */
asr_status asr_stats(asr_ctx* ctx, int32_t seq, asr_stats_t* out, asr_ledger_view* detail);

/* Read the stored K/V of one token (all layers, [L][Hkv][d] each, kv_dtype) into host buffers,
 * from the device pool (from_mirror = 0) or the pinned host mirror (1).  Synchronises. */
asr_status asr_read_kv(asr_ctx* ctx, int32_t seq, int32_t pos, int32_t from_mirror, void* k_out,
                       void* v_out);

/* Accumulated device time since the last call (needs profiling on: profile_stages or
 * asr_set_profile): ms[0] entropy + detector + ladder + append + recovery + compaction, ms[1]
 * attention + fused score, ms[2] combine + decide + tick, ms[3] whole steps (CUDA events around the
 * step's kernels).  At batch 1 phase A/B run inside the attention kernel, so ms[0] is ~0 there.
 * *launches = kernel launches of the library in that period.  n >= 4.  Synchronises. */
asr_status asr_stage_times(asr_ctx* ctx, double* ms, int32_t n, int64_t* launches);

/* Make cuda_stream wait (without blocking the host) until the host-memory outputs of every step
 * issued so far have landed (ASR_MEM_HOST).  No-op otherwise. */
asr_status asr_flush(asr_ctx* ctx, void* cuda_stream);

/* Measurement: enqueue `reps` back-to-back launches of the attention kernel ((a4) + (a1)) over the
 * A_i the next asr_step will attend, without phase A/B and without the decide, on cuda_stream (no
 * host sync).  Inputs (q, the appended token) and O come from internal scratch; the score and split
 * partials it writes are recomputed by the next step, so the context's state is unchanged.  Bracket
 * it with CUDA events to time the kernel alone (bench.py's roofline).  reps >= 1. */
asr_status asr_time_attention(asr_ctx* ctx, int32_t reps, void* cuda_stream);

/* Switch stage profiling (the events asr_stage_times reads) on or off for the following steps.
 * While it is on, stages are separated by event nodes, so the kernels of one step do not overlap
 * (no programmatic dependent launch); off is the production configuration. */
asr_status asr_set_profile(asr_ctx* ctx, int32_t on);

/* Diagnostic: device timeline of the last step (needs ASR_TIMELINE=1 in the environment at
 * asr_create): us[2k], us[2k+1] = first-block start and last-block end of stage k (pre, attention,
 * post) in microseconds relative to the pre stage's start (%globaltimer); with n >= 15 also us[6..14] =
 * end of the decide blocks, of the next step's A_{i+1} compaction and of the combine; end of the
 * entropy units, of the append units, start and end of phase B; the first attention CTA's end; the
 * time the post stage passed its wait for the attention; with the fused tail (one kernel per step)
 * eight more: grid-barrier arrival (last CTA) and release, the ends of the tile warps' decide,
 * tick, count, look-back and write, and the first tile warp done.  n >= 6.
 * Synchronises. */
asr_status asr_timeline(asr_ctx* ctx, double* us, int32_t n);

/* NEXT-2: one policy-replay step — Alg. 1 lines 3-15 and the step-
 * boundary recovery (§3.6) with the per-token scores given instead of computed: scores is a
 * device array [batch][max_context] fp32 holding s_j of every position (only the step's attended
 * positions are read; compared with tau as in Eq. 2's decision); logits_prev (device, optional) feeds
 * the entropy detector as in asr_step.  No attention runs and no K/V is appended (the positions this
 * call appends have no K/V: use a context for replay only).  Not with a slot pool.  Asynchronous;
 * asr_stats reports the step as for asr_step.  Many (tau, K, k, W) settings can be swept at once by
 * replaying one score trace through several contexts. */
asr_status asr_step_policy(asr_ctx* ctx, const float* scores, const void* logits_prev, int32_t logits_dtype,
                           float* entropy, void* cuda_stream);

/* NEXT-1 (Alg. 1 "Generate next token"): one draw per row of
 * logits[batch][vocab] (device; logits_dtype ASR_KV_BF16 or ASR_KV_F32) — greedy if temperature <= 0
 * or top_k == 1; otherwise p = softmax(x / temperature), keep the top_k largest logits (top_k <= 0:
 * all; ties to lower indices), then the shortest prefix of those (logit desc, index asc) holding
 * >= top_p of their mass (top_p >= 1: all), and return the smallest vocab index j of the kept set whose
 * cumulative kept mass (in vocab order) exceeds uniforms[b] * the kept mass; uniforms[batch] in [0, 1)
 * (device, the caller's random numbers); token_out[batch] (device, int32).  Stateless (no context),
 * asynchronous on cuda_stream, bitwise deterministic.  Rules and pins: oracle/sample.py.
 * Errors: ASR_E_INVALID for a NULL pointer, an unknown dtype, batch outside 1..65535, vocab outside
 * 1..2^24-1, or a non-finite temperature / top_p; launch failures as ASR_E_CUDA. */
asr_status asr_sample(const void* logits, int32_t logits_dtype, int32_t batch, int32_t vocab, float temperature,
                      int32_t top_k, float top_p, const float* uniforms, int32_t* token_out, void* cuda_stream);

/* NEXT-1 fused with the entropy stage (a6): the draw of asr_sample and, from the same read of each row
 * (the row slice is kept in shared memory), entropy_out[b] = H(softmax(logits[b] / entropy_temperature))
 * in nats (R-ent; Sec 3.6) — the value the next asr_step's detector needs, passed there with
 * logits_dtype = ASR_ENTROPY_GIVEN instead of the logits rows.  entropy_out: device fp32 [batch].
 * Errors as asr_sample, plus ASR_E_INVALID for a NULL entropy_out or entropy_temperature <= 0. */
asr_status asr_sample_entropy(const void* logits, int32_t logits_dtype, int32_t batch, int32_t vocab,
                              float temperature, int32_t top_k, float top_p, const float* uniforms, int32_t* token_out,
                              float entropy_temperature, float* entropy_out, void* cuda_stream);

/* NEXT-4 (§Future Work, "hybrid compression combining ASR-KF-EGR with
 * quantization methods"): the frozen tier stored quantised so a restore moves fewer bytes over the host
 * link (row a5).  The paper fixes no scheme; the reading R-quant (oracle/quant.py):
 *   a row = one head vector (token, layer, K|V, KV head) of row_elems = head_dim bf16 values, i.e. the
 *   frozen tier [token][L][2][Hkv][d] is rows = tokens * L * 2 * Hkv rows of d;
 *   qmax = 2^(bits-1) - 1 (127 or 7); scale = max|x| / qmax (IEEE fp32 division, round to nearest);
 *   code = clamp(rint(x / scale), -qmax, qmax) (x / scale an IEEE fp32 division, rint half-to-even),
 *   all codes 0 when scale = 0;  dequantised x' = bf16_rn(fp32(code) * scale).
 * asr_kv_quantize: kv [rows][row_elems] bf16 (device, 16-byte aligned) -> codes (device) [rows][row_elems]
 *   int8 for bits = 8, or [rows][row_elems / 2] bytes for bits = 4 (16-byte aligned either way;
 *   element 2i in the low nibble, 2i+1 in the high nibble, 4-bit two's complement), and scales[rows]
 *   fp32 (device).
 * asr_kv_dequantize: the inverse map, codes + scales -> kv [rows][row_elems] bf16 (device).
 * row_elems in {8, 16, 32, 64, 128, 256}; bits in {8, 4}; rows in [0, 2^40] (0: no-op).  Stateless,
 * asynchronous on cuda_stream, bitwise deterministic.  Buffers are the caller's (ranges must not
 * overlap).  Rows holding non-finite values get unspecified codes (the KV cache is finite).
 * Errors: ASR_E_INVALID for a NULL or misaligned pointer or an argument out of range (nothing is
 * launched); launch failures as ASR_E_CUDA. */
asr_status asr_kv_quantize(const void* kv, int64_t rows, int32_t row_elems, int32_t bits, void* codes, float* scales,
                           void* cuda_stream);
asr_status asr_kv_dequantize(const void* codes, const float* scales, int64_t rows, int32_t row_elems, int32_t bits,
                             void* kv, void* cuda_stream);

/* Synchronise and free everything the context owns. */
asr_status asr_destroy(asr_ctx* ctx);

const char* asr_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ASR_H */
