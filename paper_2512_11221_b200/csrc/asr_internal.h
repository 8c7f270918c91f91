// paper_2512_11221_b200/csrc/asr_internal.h — device-side state shared by the kernels and the
// host orchestrator of libasr.so.  Not part of the public ABI (include/asr.h is).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace asr {

constexpr int kStages = 5;          // entropy, ledger_pre, attention, combine, decide
constexpr int kEntSplits = 32;      // logits row splits for the entropy reduction
constexpr int kLedgerThreads = 1024;
constexpr int kMaxDetBaseline = 256;

// Per-sequence per-step statistics written by the kernels (read by asr_stats).
struct SeqStats {
  int32_t attended;
  int32_t active_post;
  int32_t frozen_this_step;
  int32_t restored_this_step;
  int32_t pending_restored;   // explicit asr_restore since the last step
  int32_t recovery_action;
  int32_t rewalk_requested;
  int32_t entropy_valid;
  float entropy;
  int32_t pad[3];
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
  kErrTimer = 4u,            // Active token with timer != 0 or Frozen with timer < 1
};

// Everything a kernel may need; passed by value (all pointers are device pointers).
struct DevState {
  int B, L, Hq, Hkv, d, max_ctx;
  int dtype;                  // 0 bf16, 1 f32
  int window, pinned, tick_skip_new, score_scaled;
  float tau, softness;
  int softness_int;           // k if k is a positive integer, else 0
  int vocab;
  float ent_temp;
  int det_enable, det_baseline, det_cooldown, wr_window, fr_clear_counts;
  float det_z, det_sigma_floor;
  int max_splits, chunk_min;

  void* kv;                   // pool [B*max_ctx][L][2][Hkv][d]
  uint8_t* res;               // [B][max_ctx] 1 Active / 0 Frozen
  int32_t* timer;             // [B][max_ctx]
  uint32_t* count;            // [B][max_ctx]
  int32_t* fstep;             // [B][max_ctx]
  int32_t* prompt_len;        // [B]
  int32_t* step;              // [1] index of the next (or current) step
  int32_t* act_pos;           // [B][max_ctx]
  int32_t* act_len;           // [B]
  int32_t* item_start;        // [B+1]
  float* score_part;          // [B][L][max_ctx] per-layer Eq. 2 head sums per attended index
  float* score;               // [B][max_ctx]   s_j per attended index (last step)
  float* part_ml;             // [max_items][Hq][2] (m in log2 domain, l)
  float* part_acc;            // [max_items][Hq][d]
  float* ent_part;            // [B][kEntSplits][3]
  int32_t* ent_ticket;        // [B]
  double* hist;               // [B][det_baseline]
  DetState* det;              // [B]
  int32_t* rec_action;        // [B]
  SeqStats* stats;            // [B]
  uint32_t* err;              // [1]
  int32_t* ticket;            // [1]
};

__host__ __device__ inline void chunking(int A, int max_splits, int chunk_min, int* chunk, int* nch) {
  int c = (A + max_splits - 1) / max_splits;
  c = (c + 15) & ~15;
  if (c < chunk_min) c = chunk_min;
  *chunk = c;
  *nch = (A + c - 1) / c;
}

// Kernel launchers (kernels_*.cu).  Return cudaGetLastError().
cudaError_t launch_entropy(const DevState& s, const void* logits, int logits_dtype, float* entropy_out,
                           cudaStream_t st);
cudaError_t launch_ledger_pre(const DevState& s, const void* k_new, const void* v_new, int has_entropy,
                              cudaStream_t st);
cudaError_t launch_attention(const DevState& s, const void* q, int grid, cudaStream_t st);
cudaError_t launch_combine(const DevState& s, float* o, cudaStream_t st);
cudaError_t launch_decide(const DevState& s, cudaStream_t st);
cudaError_t launch_restore(const DevState& s, int seq, int level, cudaStream_t st);
int attention_grid(const DevState& s, int num_sms);
bool attention_mma_supported(const DevState& s);   // bf16, d=128, 8 KV heads, 4 q heads per KV head
cudaError_t launch_attention_mma(const DevState& s, const void* q, int grid, cudaStream_t st);

}  // namespace asr
