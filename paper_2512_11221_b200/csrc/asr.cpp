// paper_2512_11221_b200/csrc/asr.cpp — host side of libasr.so: the C ABI of include/asr.h.
// Owns the device KV pool, ledger, workspaces, the write-once pinned host mirror and the
// side stream that fills it; launches one step as a fixed sequence of kernels on the caller's
// stream with no host synchronisation.
#include "asr.h"

#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <array>
#include <memory>
#include <string>
#include <vector>

#include "asr_internal.h"

using asr::DevState;

namespace {

thread_local std::string g_err;

asr_status fail(asr_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(e_ == cudaErrorMemoryAllocation ? ASR_E_OOM : ASR_E_CUDA,                \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                     \
  } while (0)

}  // namespace

struct asr_ctx {
  asr_config cfg{};
  DevState s{};
  int num_sms = 0;
  int attn_grid = 0;
  size_t kv_elem = 2;
  size_t tok_bytes = 0;          // one token, all layers, K and V
  std::vector<int32_t> prompt_len;
  bool uniform_prompt = true;
  int user_batch = 0;            // batch of the caller's logits / entropy rows (batch / n_layers with per-layer ledgers)
  int64_t step = 0;              // host mirror of the device step counter
  void* host_mirror = nullptr;   // pinned [B][max_ctx][L][2][Hkv][d]
  int8_t* host_codes = nullptr;  // INT8 tier (mirror_bits = 8): pinned mapped codes and scales
  float* host_scales = nullptr;
  size_t mirror_tok_bytes = 0;   // host-mirror bytes of one token
  int32_t* tok_count_host = nullptr;   // mapped pinned: the packed all-reduce count of the last attend
  cudaEvent_t ev_attend = nullptr;
  int64_t allreduce_bytes = 0;
  cudaStream_t side = nullptr;   // mirror copies
  cudaEvent_t ev_append = nullptr, ev_mirror = nullptr;
  cudaStream_t last_stream = nullptr;
  // ASR_MEM_HOST: double-buffered device staging; inputs arrive on io_in while the previous step
  // computes, outputs leave on io_out while the next step computes
  struct Staging {
    void* q = nullptr;
    void* k = nullptr;
    void* v = nullptr;
    void* logits = nullptr;
    size_t logits_bytes = 0;
    float* o = nullptr;
    float* ent = nullptr;
    cudaEvent_t in_done = nullptr, graph_done = nullptr, out_done = nullptr;
    bool used = false;
  };
  Staging stg[2];
  cudaStream_t io_in = nullptr, io_out = nullptr;
  cudaEvent_t last_out = nullptr;
  int64_t bytes_h2d = 0, bytes_d2h = 0;
  int64_t launches = 0;
  // CUDA graph of one step, per variant (with / without the entropy stage)
  struct StepGraph {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t x = nullptr;
    bool profiled = false;
    std::vector<cudaGraphNode_t> knodes;
    std::vector<asr::KNode> last;
    std::vector<cudaGraphNode_t> evnodes;
  };
  StepGraph graphs[36];  // [entropy given][has_logits][device io | host io set 0 | 1][full | attend | decide]
  bool attend_pending = false;
  std::unique_ptr<struct StepArgsBox> pending;
  asr::NcclApi nccl;
  void* nccl_comm = nullptr;
  bool use_graph = true;
  bool use_pdl = true;
  bool timeline_on = false;     // ASR_TIMELINE=1
  void *scratch_q = nullptr, *scratch_k = nullptr, *scratch_v = nullptr;   // asr_time_attention
  float* scratch_o = nullptr;
  unsigned long long* tl_buf = nullptr;
  // stage profiling
  std::vector<std::array<cudaEvent_t, asr::kStages + 1>> prof_pending;
  std::vector<std::array<cudaEvent_t, asr::kStages + 1>> prof_free;
  std::vector<void*> allocs;

  ~asr_ctx();
  void release() {
    if (nccl_comm && nccl.comm_destroy) nccl.comm_destroy(nccl_comm);
    nccl_comm = nullptr;
    for (auto& g : graphs) {
      if (g.x) cudaGraphExecDestroy(g.x);
      if (g.g) cudaGraphDestroy(g.g);
    }
    for (void* p : allocs) cudaFree(p);
    if (host_mirror) cudaFreeHost(host_mirror);
    if (host_codes) cudaFreeHost(host_codes);
    if (host_scales) cudaFreeHost(host_scales);
    if (tok_count_host) cudaFreeHost(tok_count_host);
    if (ev_attend) cudaEventDestroy(ev_attend);
    if (side) cudaStreamDestroy(side);
    if (io_in) cudaStreamDestroy(io_in);
    if (io_out) cudaStreamDestroy(io_out);
    for (auto& x : stg)
      for (cudaEvent_t e : {x.in_done, x.graph_done, x.out_done})
        if (e) cudaEventDestroy(e);
    if (ev_append) cudaEventDestroy(ev_append);
    if (ev_mirror) cudaEventDestroy(ev_mirror);
    for (auto& a : prof_pending)
      for (auto e : a) cudaEventDestroy(e);
    for (auto& a : prof_free)
      for (auto e : a) cudaEventDestroy(e);
  }

  // Device memory.  Arrays up to kArenaMax bytes are carved (256-byte aligned) out of one arena, so
  // the ledger, lists, detector state and counters that each step's latency chains touch share a
  // few large pages instead of one allocation (and TLB entry) each; bigger arrays (KV pool,
  // partials) get their own allocation.
  static constexpr size_t kArena = 32u << 20, kArenaMax = 4u << 20;
  char* arena = nullptr;
  size_t arena_used = 0;
  template <typename P>
  cudaError_t alloc(P** p, size_t bytes) {
    bytes = bytes ? (bytes + 255) & ~(size_t)255 : 256;
    static const bool no_arena = [] { const char* e = getenv("ASR_NO_ARENA"); return e && e[0] == '1'; }();
    if (bytes <= kArenaMax && !no_arena) {
      if (!arena) {
        cudaError_t e = cudaMalloc(&arena, kArena);
        if (e != cudaSuccess) return e;
        allocs.push_back(arena);
      }
      if (arena_used + bytes <= kArena) {
        *p = reinterpret_cast<P*>(arena + arena_used);
        arena_used += bytes;
        return cudaSuccess;
      }
    }
    void* v = nullptr;
    cudaError_t e = cudaMalloc(&v, bytes);
    if (e == cudaSuccess) {
      allocs.push_back(v);
      *p = reinterpret_cast<P*>(v);
    }
    return e;
  }
};

struct StepArgsBox;   // defined below (holds a StepArgs between asr_step_attend and asr_step_decide)

extern "C" {

const char* asr_last_error(void) { return g_err.c_str(); }

void asr_config_defaults(asr_config* c) {
  memset(c, 0, sizeof(*c));
  c->n_layers = 32;
  c->n_q_heads = 32;
  c->n_kv_heads = 8;
  c->head_dim = 128;
  c->batch = 1;
  c->max_context = 8192;
  c->kv_dtype = ASR_KV_BF16;
  c->window = 32;
  c->tau = 0.5f;
  c->softness = 2.0f;
  c->history_window = 0;
  c->pinned_prefix = 0;
  c->score_mode = ASR_SCORE_RAW;
  c->tick_order = ASR_TICK_LITERAL;
  c->vocab = 128256;
  c->entropy_temperature = 1.0f;
  c->det_enable = 1;
  c->det_baseline = 64;
  c->det_cooldown = 16;
  c->wr_window = 32;
  c->det_z = 3.0f;
  c->det_sigma_floor = 0.05f;
  c->fr_clear_counts = 0;
  c->host_mirror = 1;
  c->profile_stages = 0;
  c->device = 0;
  c->evict_min_absence = 2;
  c->pool_reserve = 0;
  c->pool_tokens = 0;
  c->score_heads = 0;
  c->evict_policy = ASR_EVICT_BELADY;
  c->mirror_bits = 0;
  c->per_layer_ledgers = 0;
}

static asr_status validate(const asr_config* c) {
  if (!c) return fail(ASR_E_INVALID, "config is NULL");
  if (c->n_layers < 1 || c->n_layers > 128) return fail(ASR_E_INVALID, "n_layers out of range [1,128]");
  if (c->n_kv_heads < 1 || c->n_kv_heads > 32) return fail(ASR_E_INVALID, "n_kv_heads out of range [1,32]");
  if (c->n_q_heads < 1 || c->n_q_heads % c->n_kv_heads)
    return fail(ASR_E_INVALID, "n_q_heads must be a positive multiple of n_kv_heads");
  if (c->n_q_heads / c->n_kv_heads > 8) return fail(ASR_E_INVALID, "at most 8 query heads per KV head");
  int d = c->head_dim;
  if (d != 16 && d != 32 && d != 64 && d != 128 && d != 256)
    return fail(ASR_E_INVALID, "head_dim must be one of 16, 32, 64, 128, 256");
  if (c->batch < 1 || c->batch > 4096) return fail(ASR_E_INVALID, "batch out of range [1,4096]");
  if (c->max_context < 2 || c->max_context > (1 << 20)) return fail(ASR_E_INVALID, "max_context out of range");
  if (c->kv_dtype != ASR_KV_BF16 && c->kv_dtype != ASR_KV_F32) return fail(ASR_E_INVALID, "kv_dtype");
  if (c->window < 1) return fail(ASR_E_INVALID, "window (K) must be >= 1");
  if (!(c->softness > 0.f) || !isfinite(c->softness)) return fail(ASR_E_INVALID, "softness k must be > 0");
  if (!isfinite(c->tau)) return fail(ASR_E_INVALID, "tau must be finite");
  if (c->history_window < 0 || c->history_window > 128)
    return fail(ASR_E_INVALID, "history_window: W = 0 (infinite, R-W) or 1..128");
  if (c->pinned_prefix < 0) return fail(ASR_E_INVALID, "pinned_prefix < 0");
  if (c->score_mode != ASR_SCORE_RAW && c->score_mode != ASR_SCORE_SCALED) return fail(ASR_E_INVALID, "score_mode");
  if (c->tick_order != ASR_TICK_LITERAL && c->tick_order != ASR_TICK_SKIP_NEW) return fail(ASR_E_INVALID, "tick_order");
  if (c->vocab < 0 || c->vocab >= (1 << 24)) return fail(ASR_E_INVALID, "vocab out of range");
  if (c->vocab > 0 && !(c->entropy_temperature > 0.f)) return fail(ASR_E_INVALID, "entropy_temperature must be > 0");
  if (c->det_baseline < 1 || c->det_baseline > asr::kMaxDetBaseline)
    return fail(ASR_E_INVALID, "det_baseline out of range [1,256]");
  if (c->det_cooldown < 0 || c->wr_window < 0) return fail(ASR_E_INVALID, "det_cooldown / wr_window < 0");
  if (c->pool_tokens < 0) return fail(ASR_E_INVALID, "pool_tokens < 0");
  if (c->pool_tokens > 0 && !c->host_mirror) return fail(ASR_E_INVALID, "pool_tokens > 0 needs host_mirror = 1");
  if (c->pool_tokens > ((int64_t)1 << 31) - 1) return fail(ASR_E_INVALID, "pool_tokens too large");
  if (c->evict_policy != ASR_EVICT_BELADY && c->evict_policy != ASR_EVICT_AT_FREEZE)
    return fail(ASR_E_INVALID, "evict_policy");
  if (c->pool_reserve < 0) return fail(ASR_E_INVALID, "pool_reserve < 0");
  if (c->mirror_bits != 0 && c->mirror_bits != 8) return fail(ASR_E_INVALID, "mirror_bits must be 0 or 8");
  if (c->mirror_bits == 8 && (c->pool_tokens <= 0 || c->kv_dtype != ASR_KV_BF16 || c->head_dim % 32))
    return fail(ASR_E_INVALID, "mirror_bits = 8 needs pressure mode (pool_tokens > 0), bf16 KV and head_dim >= 32");
  if (c->score_heads != 0 && c->score_heads < c->n_q_heads)
    return fail(ASR_E_INVALID, "score_heads must be 0 or >= n_q_heads (the heads of all shards)");
  return ASR_OK;
}

static asr_status create_impl(const asr_config* cfg, const void* prompt_k, const void* prompt_v,
                              const int32_t* prompt_len, int32_t prompt_stride, int32_t memory, void* cuda_stream,
                              asr_ctx** out, int ent_div);

// NEXT-3 per-layer ledgers: the context is built over batch * n_layers virtual sequences of one layer
// each (ledger, lists, pool slots of a token-layer); the prompt is rearranged from [B][stride][L]
// [Hkv][d] to [B*L][stride][1][Hkv][d] on the device first.  Everything else is the per-sequence
// engine unchanged; ent_div = L maps a virtual sequence to its logits row / entropy slot.
asr_status asr_create(const asr_config* cfg, const void* prompt_k, const void* prompt_v,
                      const int32_t* prompt_len, int32_t prompt_stride, int32_t memory, void* cuda_stream,
                      asr_ctx** out) {
  if (!cfg || !cfg->per_layer_ledgers) return create_impl(cfg, prompt_k, prompt_v, prompt_len, prompt_stride, memory,
                                                          cuda_stream, out, 1);
  if (!out) return fail(ASR_E_INVALID, "out is NULL");
  *out = nullptr;
  if (cfg->per_layer_ledgers != 1) return fail(ASR_E_INVALID, "per_layer_ledgers must be 0 or 1");
  asr_status v = validate(cfg);
  if (v) return v;
  if (!prompt_len) return fail(ASR_E_INVALID, "prompt_len is NULL");
  const int B = cfg->batch, L = cfg->n_layers;
  if ((int64_t)B * L > 4096) return fail(ASR_E_INVALID, "per-layer ledgers: batch * n_layers must be <= 4096");
  asr_config vc = *cfg;
  vc.batch = B * L;
  vc.n_layers = 1;
  vc.per_layer_ledgers = 0;
  if (vc.pool_tokens > 0) vc.pool_tokens *= L;   // token-layer slots
  std::vector<int32_t> vlen((size_t)B * L);
  int32_t pmax = 0;
  for (int b = 0; b < B; ++b) {
    if (prompt_len[b] < 0 || prompt_len[b] > prompt_stride)
      return fail(ASR_E_INVALID, "prompt_len[b] must be in [0, prompt_stride]");
    for (int l = 0; l < L; ++l) vlen[(size_t)b * L + l] = prompt_len[b];
    pmax = prompt_len[b] > pmax ? prompt_len[b] : pmax;
  }
  if (pmax == 0 || !prompt_k || !prompt_v)
    return create_impl(&vc, nullptr, nullptr, vlen.data(), 0, ASR_MEM_DEVICE, cuda_stream, out, L);
  CUDA_TRY(cudaSetDevice(cfg->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const size_t row = (size_t)cfg->n_kv_heads * cfg->head_dim * (cfg->kv_dtype == ASR_KV_BF16 ? 2 : 4);
  const size_t bytes = (size_t)B * L * pmax * row;
  void *vk = nullptr, *vv = nullptr;
  CUDA_TRY(cudaMalloc(&vk, bytes));
  cudaError_t e = cudaMalloc(&vv, bytes);
  if (e != cudaSuccess) {
    cudaFree(vk);
    return fail(ASR_E_OOM, "per-layer ledgers: prompt staging");
  }
  const cudaMemcpyKind kind = memory == ASR_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  for (int b = 0; b < B && e == cudaSuccess; ++b)
    for (int l = 0; l < L && e == cudaSuccess; ++l) {
      if (!prompt_len[b]) continue;
      const size_t src = ((size_t)b * prompt_stride * L + l) * row, dst = ((size_t)b * L + l) * pmax * row;
      e = cudaMemcpy2DAsync((char*)vk + dst, row, (const char*)prompt_k + src, L * row, row, prompt_len[b], kind, st);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync((char*)vv + dst, row, (const char*)prompt_v + src, L * row, row, prompt_len[b], kind, st);
    }
  asr_status r = e == cudaSuccess ? create_impl(&vc, vk, vv, vlen.data(), pmax, ASR_MEM_DEVICE, cuda_stream, out, L)
                                  : fail(ASR_E_CUDA, std::string("per-layer prompt copy: ") + cudaGetErrorString(e));
  cudaStreamSynchronize(st);
  cudaFree(vk);
  cudaFree(vv);
  return r;
}

static asr_status create_impl(const asr_config* cfg, const void* prompt_k, const void* prompt_v,
                              const int32_t* prompt_len, int32_t prompt_stride, int32_t memory, void* cuda_stream,
                              asr_ctx** out, int ent_div) {
  if (!out) return fail(ASR_E_INVALID, "out is NULL");
  *out = nullptr;
  asr_status v = validate(cfg);
  if (v) return v;
  if (!prompt_len) return fail(ASR_E_INVALID, "prompt_len is NULL");
  if (memory != ASR_MEM_DEVICE && memory != ASR_MEM_HOST) return fail(ASR_E_INVALID, "memory");
  int32_t pmax = 0;
  for (int b = 0; b < cfg->batch; ++b) {
    if (prompt_len[b] < 0 || prompt_len[b] > prompt_stride || prompt_len[b] >= cfg->max_context)
      return fail(ASR_E_INVALID, "prompt_len[b] must be in [0, min(prompt_stride, max_context-1)]");
    pmax = prompt_len[b] > pmax ? prompt_len[b] : pmax;
  }
  if (pmax > 0 && (!prompt_k || !prompt_v)) return fail(ASR_E_INVALID, "prompt_k / prompt_v is NULL");
  int64_t prompt_total = 0;
  for (int b = 0; b < cfg->batch; ++b) prompt_total += prompt_len[b];
  if (cfg->pool_tokens > 0 && cfg->pool_tokens < prompt_total + 2 * (int64_t)cfg->batch)
    return fail(ASR_E_INVALID, "pool_tokens must hold every prompt token plus two slots per sequence");
  CUDA_TRY(cudaSetDevice(cfg->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;

  asr_ctx* c = new asr_ctx();
  c->cfg = *cfg;
  c->prompt_len.assign(prompt_len, prompt_len + cfg->batch);
  for (int b = 1; b < cfg->batch; ++b) c->uniform_prompt &= prompt_len[b] == prompt_len[0];
  asr_status rc = [&]() -> asr_status {
    DevState& s = c->s;
    s.B = cfg->batch;
    s.L = cfg->n_layers;
    s.ent_div = ent_div;
    c->user_batch = cfg->batch / ent_div;
    s.Hq = cfg->n_q_heads;
    s.Hkv = cfg->n_kv_heads;
    s.d = cfg->head_dim;
    s.max_ctx = (cfg->max_context + 63) & ~63;   // row stride of every per-sequence array (aligned)
    s.cap = cfg->max_context;
    s.dtype = cfg->kv_dtype;
    s.window = cfg->window;
    s.pinned = cfg->pinned_prefix;
    s.tick_skip_new = cfg->tick_order == ASR_TICK_SKIP_NEW;
    s.score_scaled = cfg->score_mode == ASR_SCORE_SCALED;
    s.tau = cfg->tau;
    s.softness = cfg->softness;
    s.softness_int = (floorf(cfg->softness) == cfg->softness && cfg->softness <= 65535.f) ? (int)cfg->softness : 0;
    s.vocab = cfg->vocab;
    s.ent_temp = cfg->entropy_temperature;
    s.det_enable = cfg->det_enable;
    s.det_baseline = cfg->det_baseline;
    s.det_cooldown = cfg->det_cooldown;
    s.wr_window = cfg->wr_window;
    s.fr_clear_counts = cfg->fr_clear_counts;
    s.det_z = cfg->det_z;
    s.det_sigma_floor = cfg->det_sigma_floor;
    CUDA_TRY(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, cfg->device));
    // split-KV policy: enough work items to fill the SMs; fp32 KV keeps chunks <= 256 tokens
    // split-KV policy: enough work items to fill the SMs (a balanced split into 37-token chunks at
    // batch 1 measured slower: partial tiles shrink the bytes in flight; profiles/README.md)
    s.chunk_min = 64;
    long want = (8L * c->num_sms + (long)s.B * s.L - 1) / ((long)s.B * s.L);
    if (s.dtype == ASR_KV_F32) {
      long acc = (s.max_ctx + 255) / 256;
      want = want > acc ? want : acc;
    }
    long cap = (s.max_ctx + s.chunk_min - 1) / s.chunk_min;
    s.max_splits = (int)(want < 1 ? 1 : want > cap ? cap : want);
    if (s.max_splits > 64 && s.dtype == ASR_KV_BF16) s.max_splits = 64;
    {
      // decide blocks per sequence: ~256 positions each, at most 32 (round 2: 256 / 512 / 1024 -> 49.8 / 49.9 / 50.5 us
      // per 8K batch-1 step); X > 1 only if all B*X blocks are co-resident
      // (one per SM), since a block waits for its predecessors' counts to place its part of A_{i+1}
      const char* dbe = getenv("ASR_DECIDE_POSITIONS");   // positions per decide block (tuning)
      const int per_block = dbe ? atoi(dbe) : 256;
      int db = (s.max_ctx + per_block - 1) / (per_block > 0 ? per_block : 2048);
      db = db < 1 ? 1 : db > 32 ? 32 : db;
      if ((long)s.B * db > c->num_sms) db = 1;
      s.decide_blocks = db;
    }

    c->kv_elem = s.dtype == ASR_KV_BF16 ? 2 : 4;
    c->tok_bytes = (size_t)s.L * 2 * s.Hkv * s.d * c->kv_elem;
    s.tok_bytes = (long)c->tok_bytes;
    const size_t BT = (size_t)s.B * s.max_ctx;
    s.pool_mode = cfg->pool_tokens > 0 ? 1 : 0;
    s.evict_min = cfg->evict_min_absence > 0 ? cfg->evict_min_absence : 2;
    s.evict_policy = cfg->evict_policy;
    s.pool_reserve = cfg->pool_reserve;
    const size_t slots = s.pool_mode ? (size_t)cfg->pool_tokens : BT;
    CUDA_TRY(c->alloc(&s.kv, slots * c->tok_bytes));
    s.kv_slots = (long)slots;
    CUDA_TRY(c->alloc(&s.act_slot, 2 * BT * 4));
    s.score_heads = cfg->score_heads > 0 ? cfg->score_heads : s.Hq;
    s.sharded = s.score_heads != s.Hq ? 1 : 0;
    CUDA_TRY(c->alloc(&s.tok_score, BT * 4));
    CUDA_TRY(cudaMemsetAsync(s.tok_score, 0, BT * 4, st));
    {   // the packed all-reduce count, read by the host after the attention (head-sharded mode)
      cudaError_t e = cudaHostAlloc((void**)&c->tok_count_host, 64, cudaHostAllocMapped | cudaHostAllocPortable);
      if (e != cudaSuccess) return fail(ASR_E_OOM, "pinned host allocation failed");
      *c->tok_count_host = 0;
      CUDA_TRY(cudaHostGetDevicePointer((void**)&s.tok_count, c->tok_count_host, 0));
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_attend, cudaEventDisableTiming));
    }
    std::vector<size_t> slot0(s.B, 0);   // first slot of each sequence's prompt
    for (int b = 0; b < s.B; ++b) slot0[b] = s.pool_mode ? (b ? slot0[b - 1] + prompt_len[b - 1] : 0) : (size_t)b * s.max_ctx;
    if (s.pool_mode) {
      const int64_t used = prompt_total;
      CUDA_TRY(c->alloc(&s.slot_of, BT * 4));
      CUDA_TRY(c->alloc(&s.spare, (size_t)s.B * 4));
      CUDA_TRY(c->alloc(&s.free_stack, slots * 4));
      CUDA_TRY(c->alloc(&s.free_top, 4));
      CUDA_TRY(c->alloc(&s.pf_list, 2 * BT * 4));
      CUDA_TRY(c->alloc(&s.pf_count, 2 * (size_t)s.B * 4));
      CUDA_TRY(c->alloc(&s.cp_list, BT * 4));
      CUDA_TRY(c->alloc(&s.cp_count, (size_t)s.B * 4));
      CUDA_TRY(c->alloc(&s.h2d, 8));
      CUDA_TRY(c->alloc(&s.ev_hist, asr::kEvBins * 4));
      CUDA_TRY(c->alloc(&s.ev_ctrl, 16));
      CUDA_TRY(c->alloc(&s.stall, 24));
      CUDA_TRY(cudaMemset(s.ev_hist, 0, asr::kEvBins * 4));
      CUDA_TRY(cudaMemset(s.ev_ctrl, 0, 16));
      CUDA_TRY(cudaMemset(s.stall, 0, 24));
      std::vector<int32_t> so(BT, -1), sp(s.B), fs;
      for (int b = 0; b < s.B; ++b)
        for (int p = 0; p < prompt_len[b]; ++p) so[(size_t)b * s.max_ctx + p] = (int32_t)(slot0[b] + p);
      for (int b = 0; b < s.B; ++b) sp[b] = (int32_t)(used + b);
      for (int64_t k = (int64_t)slots - 1; k >= used + s.B; --k) fs.push_back((int32_t)k);
      const int32_t top = (int32_t)fs.size();
      CUDA_TRY(cudaMemcpy(s.slot_of, so.data(), BT * 4, cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(s.spare, sp.data(), (size_t)s.B * 4, cudaMemcpyHostToDevice));
      if (top) CUDA_TRY(cudaMemcpy(s.free_stack, fs.data(), (size_t)top * 4, cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(s.free_top, &top, 4, cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemset(s.pf_count, 0, 2 * (size_t)s.B * 4));
      CUDA_TRY(cudaMemset(s.cp_count, 0, (size_t)s.B * 4));
      CUDA_TRY(cudaMemset(s.h2d, 0, 8));
    }
    CUDA_TRY(c->alloc(&s.res, BT));
    CUDA_TRY(c->alloc(&s.timer, BT * 4));
    CUDA_TRY(c->alloc(&s.count, BT * 4));
    CUDA_TRY(c->alloc(&s.fstep, BT * 4));
    s.hist_w = cfg->history_window;
    if (s.hist_w > 0) {   // finite W: per-token detection history (NEXT-3)
      CUDA_TRY(c->alloc(&s.hmask, BT * 16));
      CUDA_TRY(c->alloc(&s.hstep, BT * 4));
      CUDA_TRY(cudaMemsetAsync(s.hmask, 0, BT * 16, st));
      CUDA_TRY(cudaMemsetAsync(s.hstep, 0xc0, BT * 4, st));   // 0xc0c0c0c0: never detected
    }
    CUDA_TRY(c->alloc(&s.prompt_len, (size_t)s.B * 4));
    CUDA_TRY(c->alloc(&s.step, 4));
    CUDA_TRY(c->alloc(&s.act_pos, 2 * BT * 4));
    CUDA_TRY(c->alloc(&s.act_len, 2 * (size_t)s.B * 4));
    CUDA_TRY(c->alloc(&s.dagg, (size_t)s.B * 32 * 8));
    CUDA_TRY(c->alloc(&s.redo, 4));
    CUDA_TRY(c->alloc(&s.pre_done, 4));
    CUDA_TRY(c->alloc(&s.gbar, 8));
    CUDA_TRY(c->alloc(&s.item_start, (size_t)(s.B + 1) * 4));
    CUDA_TRY(c->alloc(&s.score_part, BT * s.L * 4));
    CUDA_TRY(c->alloc(&s.score, BT * 4));
    size_t max_items = (size_t)s.B * s.L * s.max_splits;
    const size_t sk_slots = (size_t)s.B * s.L + (size_t)c->num_sms * (1 + asr::kSkMaxChunksPerCta);   // units
    if (max_items < sk_slots) max_items = sk_slots;
    CUDA_TRY(c->alloc(&s.sk_ctr, 8));
    CUDA_TRY(cudaMemsetAsync(s.sk_ctr, 0, 8, st));
    s.max_items = (long)max_items;
    CUDA_TRY(c->alloc(&s.part_ml, max_items * s.Hq * 2 * 4));
    CUDA_TRY(c->alloc(&s.part_acc, max_items * s.Hq * s.d * 4));
    CUDA_TRY(c->alloc(&s.ent_part, (size_t)s.B * asr::kEntSplits * 3 * 4));
      CUDA_TRY(c->alloc(&s.hist, (size_t)s.B * s.det_baseline * 8));
    CUDA_TRY(c->alloc(&s.det, (size_t)s.B * sizeof(asr::DetState)));
      CUDA_TRY(c->alloc(&s.stats, (size_t)s.B * sizeof(asr::SeqStats)));
    CUDA_TRY(c->alloc(&s.err, 4));
    CUDA_TRY(c->alloc(&s.ticket, 4));
    CUDA_TRY(c->alloc(&s.pre_ticket, (size_t)s.B * 4));
    // ledger init: prompt tokens Active, c = d = 0 (R-prefill); everything else zero
    CUDA_TRY(cudaMemsetAsync(s.res, 0, BT, st));
    CUDA_TRY(cudaMemsetAsync(s.timer, 0, BT * 4, st));
    CUDA_TRY(cudaMemsetAsync(s.count, 0, BT * 4, st));
    CUDA_TRY(cudaMemsetAsync(s.fstep, 0xff, BT * 4, st));
    CUDA_TRY(cudaMemsetAsync(s.step, 0, 4, st));
      CUDA_TRY(cudaMemsetAsync(s.det, 0, (size_t)s.B * sizeof(asr::DetState), st));
      CUDA_TRY(cudaMemsetAsync(s.stats, 0, (size_t)s.B * sizeof(asr::SeqStats), st));
    CUDA_TRY(cudaMemsetAsync(s.err, 0, 4, st));
    CUDA_TRY(cudaMemsetAsync(s.ticket, 0, 4, st));
    CUDA_TRY(cudaMemsetAsync(s.pre_ticket, 0, (size_t)s.B * 4, st));
    CUDA_TRY(cudaMemsetAsync(s.dagg, 0, (size_t)s.B * 32 * 8, st));
    CUDA_TRY(cudaMemsetAsync(s.redo, 0, 4, st));
    CUDA_TRY(cudaMemsetAsync(s.pre_done, 0, 4, st));
    CUDA_TRY(cudaMemsetAsync(s.gbar, 0, 8, st));
    CUDA_TRY(cudaMemsetAsync(s.act_len, 0, 2 * (size_t)s.B * 4, st));
    CUDA_TRY(cudaMemcpyAsync(s.prompt_len, prompt_len, (size_t)s.B * 4, cudaMemcpyHostToDevice, st));
    for (int b = 0; b < s.B; ++b)
      if (prompt_len[b] > 0) CUDA_TRY(cudaMemsetAsync(s.res + (size_t)b * s.max_ctx, 1, prompt_len[b], st));
    s.mirror_bits = cfg->mirror_bits;
    if (cfg->host_mirror && s.mirror_bits == 8) {   // the INT8 frozen tier: codes + scales, mapped
      const size_t R = (size_t)s.L * 2 * s.Hkv;
      cudaError_t e = cudaHostAlloc(&c->host_codes, BT * R * s.d, cudaHostAllocPortable | cudaHostAllocMapped);
      if (e == cudaSuccess)
        e = cudaHostAlloc(&c->host_scales, BT * R * 4, cudaHostAllocPortable | cudaHostAllocMapped);
      if (e != cudaSuccess) return fail(ASR_E_OOM, "pinned host mirror allocation failed");
      CUDA_TRY(cudaHostGetDevicePointer((void**)&s.host_codes, c->host_codes, 0));
      CUDA_TRY(cudaHostGetDevicePointer((void**)&s.host_scales, c->host_scales, 0));
      CUDA_TRY(c->alloc(&s.deq, BT));
      CUDA_TRY(cudaMemsetAsync(s.deq, 0, BT, st));
      c->mirror_tok_bytes = R * (s.d + 4);
    } else if (cfg->host_mirror) {
      cudaError_t e = cudaHostAlloc(&c->host_mirror, BT * c->tok_bytes,
                                    cudaHostAllocPortable | (s.pool_mode ? cudaHostAllocMapped : 0));
      if (e != cudaSuccess) return fail(ASR_E_OOM, "pinned host mirror allocation failed");
      if (s.pool_mode) CUDA_TRY(cudaHostGetDevicePointer((void**)&s.host_kv, c->host_mirror, 0));
      c->mirror_tok_bytes = c->tok_bytes;
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_append, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_mirror, cudaEventDisableTiming));
    // prompt KV: [B][stride][L][Hkv][d] K and V -> slots [L][2][Hkv][d]
    const size_t row = (size_t)s.Hkv * s.d * c->kv_elem;  // K (or V) bytes per token-layer
    const cudaMemcpyKind kind = memory == ASR_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    for (int b = 0; b < s.B; ++b) {
      if (prompt_len[b] == 0) continue;
      const size_t rows = (size_t)prompt_len[b] * s.L;
      const size_t src_off = (size_t)b * prompt_stride * s.L * row;
      char* dst = (char*)s.kv + slot0[b] * c->tok_bytes;
      CUDA_TRY(cudaMemcpy2DAsync(dst, 2 * row, (const char*)prompt_k + src_off, row, row, rows, kind, st));
      CUDA_TRY(cudaMemcpy2DAsync(dst + row, 2 * row, (const char*)prompt_v + src_off, row, row, rows, kind, st));
      if (c->host_mirror) {
        char* hdst = (char*)c->host_mirror + (size_t)b * s.max_ctx * c->tok_bytes;
        CUDA_TRY(cudaMemcpyAsync(hdst, dst, (size_t)prompt_len[b] * c->tok_bytes, cudaMemcpyDeviceToHost, st));
        c->bytes_d2h += (int64_t)prompt_len[b] * c->tok_bytes;
      } else if (c->host_codes) {   // the prompt's rows quantised straight into the mapped INT8 tier
        const size_t R = (size_t)s.L * 2 * s.Hkv;
        CUDA_TRY(asr::launch_kv_quantize(dst, (long)(prompt_len[b] * R), s.d, 8,
                                         s.host_codes + (size_t)b * s.max_ctx * R * s.d,
                                         s.host_scales + (size_t)b * s.max_ctx * R, st));
        c->bytes_d2h += (int64_t)prompt_len[b] * c->mirror_tok_bytes;
      }
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    // batch 1 on the tensor-core path: phase A (+B) inside the attention kernel, on an extra warp of
    // CTAs 0..95, one unit each (not with the slot pool, whose prefetch copies must follow phase B)
    {
      const char* pa = getenv("ASR_PRE_KERNEL");
      const bool force_kernel = pa && pa[0] == '1';
      s.pre_in_attn = asr::attention_mma_supported(s) && !s.pool_mode && !force_kernel &&
                      asr::kEntSplits * s.B + s.L * s.B <= c->num_sms;
      // phase-A unit grouping: one unit per warp-sized piece inside the attention kernel; otherwise
      // one entropy split per warp (8 per 256-thread unit) and appends grouped to ~one unit per SM
      auto pow2ceil = [](long v) { int p = 1; while (p < v) p <<= 1; return p; };
      const char* epu = getenv("ASR_ENT_PER_UNIT");   // tuning: entropy splits per phase-A unit (divides 64)
      s.ent_per_unit = s.pre_in_attn ? 1 : epu ? atoi(epu) : 8;
      if (asr::kEntSplits % s.ent_per_unit) s.ent_per_unit = 8;
      const int l = s.pre_in_attn ? 1 : pow2ceil(((long)s.L * s.B + c->num_sms - 1) / c->num_sms);
      s.layers_per_unit = l > s.L ? s.L : l;
      // small batch: the combine rides in the phase-D kernel (one launch fewer on the critical path)
      s.combine_in_decide = (long)s.B * s.L * s.Hq <= 64L * c->num_sms;
    }
    c->attn_grid = asr::attention_grid(s, c->num_sms);
    // fused tail (opt-in, ASR_FUSE_TAIL=1): the attention kernel settles the step itself (decide + tick
    // + A_{i+1} + combine after a grid barrier) — tensor-core path, full residency, unsharded.  Off by
    // default: measured 56.1 vs 53.2 us per batch-1 8K step
    {
      const char* ft = getenv("ASR_FUSE_TAIL");
      s.max_tiles = (s.max_ctx + 15) / 16;
      s.fuse_tail = asr::attention_mma_supported(s) && !s.pool_mode && !s.sharded && ft && ft[0] == '1';
      const char* te = getenv("ASR_TAIL_EXP");
      s.tail_exp = te ? atoi(te) : 0;
      CUDA_TRY(c->alloc(&s.seg_flag, (size_t)s.B * s.max_tiles * 8));
      CUDA_TRY(cudaMemsetAsync(s.seg_flag, 0, (size_t)s.B * s.max_tiles * 8, st));
    }
    if (asr::attention_mma_supported(s)) CUDA_TRY(asr::attention_mma_prepare());
    const char* ng = getenv("ASR_NO_GRAPH");
    c->use_graph = !(ng && ng[0] == '1');
    // device timeline: [2*kStages] stamps + [kStages] accumulated phase ns + [1] step count
    const size_t tl_words = asr::kTimelineSlots + (size_t)asr::kTraceRows * asr::kTraceCols;
    CUDA_TRY(c->alloc(&c->tl_buf, sizeof(unsigned long long) * tl_words));
    CUDA_TRY(cudaMemsetAsync(c->tl_buf, 0, sizeof(unsigned long long) * tl_words, st));
    const char* tlenv = getenv("ASR_TIMELINE");
    c->timeline_on = tlenv && tlenv[0] == '1';
    s.tl = nullptr;
    s.sk_grid = asr::attention_mma_supported(s) ? c->attn_grid : 0;
    // A_0 of every sequence (the ledger entry of the first appended position + compaction)
    {
      asr::KNode pn;
      asr::node_prepare(pn, s);
      CUDA_TRY(pn.launch(st));
      CUDA_TRY(cudaStreamSynchronize(st));
    }
    {   // dynamic tail of the attention's work split (asr_internal.h): 1/sk_dyn of the tiles in chunks
      const char* sd = getenv("ASR_SK_DYN");
      const char* sc = getenv("ASR_SK_CHUNK");
      // measured (profiles/r2): batch 64 at 8K 1890 -> 1810 us per step; batch 1 loses 1-5 us (chunk
      // overheads and the producer's registers), so batch < 16 keeps the static split
      s.sk_dyn = sd ? atoi(sd) : (s.B >= 16 ? 8 : 0);
      s.sk_chunk = sc ? atoi(sc) : 2;
      if (s.Hkv != 8) s.sk_dyn = 0;   // the dynamic variant is compiled for 8 KV heads only
      // rate-balanced static split (asr_internal.h, sk_weighted), batch 1 by default (ASR_SK_BALANCE=1:
      // any static-split batch, 0: off).  Measured (profiles/r2/balance_ab.txt): batch 1 8K 51.1 ->
      // 49.5 us, 32K 79.3 -> 77.2 us; batch 4 / 8 / 64 the attention alone gains 2-5 % but the step
      // loses 3-55 us — there the rates move with the cut (the first-to-last CTA spread grew from
      // 226 to 384 us at batch 64), so the feedback chases its own effect
      const char* sb = getenv("ASR_SK_BALANCE");
      const bool bal = sb ? sb[0] == '1' : s.B == 1;
      s.sk_bal = bal && s.sk_grid > 0 && s.sk_grid < asr::kSkBalMax && s.sk_dyn == 0 && !s.fuse_tail;
      s.sk_learn = 1;
      const char* se = getenv("ASR_SK_EWMA");
      s.sk_ewma = se ? (float)atof(se) : 0.5f;
      if (!(s.sk_ewma > 0.f && s.sk_ewma <= 1.f)) s.sk_ewma = 0.5f;
      CUDA_TRY(c->alloc(&s.sk_w, sizeof(float) * 4 * asr::kSkBalMax));
      CUDA_TRY(cudaMemsetAsync(s.sk_w, 0, sizeof(float) * 4 * asr::kSkBalMax, st));
      CUDA_TRY(c->alloc(&s.sk_f, sizeof(float) * 4 * asr::kSkBalMax));
      CUDA_TRY(cudaMemsetAsync(s.sk_f, 0xff, sizeof(float) * 4 * asr::kSkBalMax, st));   // NaN: not computed yet
      CUDA_TRY(c->alloc(&s.sk_bound, sizeof(int) * asr::kSkBalMax));
      CUDA_TRY(cudaMemsetAsync(s.sk_bound, 0, sizeof(int) * asr::kSkBalMax, st));
    }
    const char* ke = getenv("ASR_KV_EVICT_FIRST");
    s.kv_evict_first = !(ke && ke[0] == '0');
    const char* np = getenv("ASR_NO_PDL");
    c->use_pdl = !(np && np[0] == '1');
    c->last_stream = st;
    return ASR_OK;
  }();
  if (rc) {
    delete c;
    return rc;
  }
  *out = c;
  return ASR_OK;
}

static asr_status ensure_staging(asr_ctx* c, asr_ctx::Staging& S, bool logits, int logits_dtype) {
  const DevState& s = c->s;
  if (!S.q) {
    CUDA_TRY(c->alloc(&S.q, (size_t)s.B * s.L * s.Hq * s.d * c->kv_elem));
    CUDA_TRY(c->alloc(&S.k, (size_t)s.B * s.L * s.Hkv * s.d * c->kv_elem));
    CUDA_TRY(c->alloc(&S.v, (size_t)s.B * s.L * s.Hkv * s.d * c->kv_elem));
    CUDA_TRY(c->alloc(&S.o, (size_t)s.B * s.L * s.Hq * s.d * 4));
    CUDA_TRY(c->alloc(&S.ent, (size_t)c->user_batch * 4));
    CUDA_TRY(cudaEventCreateWithFlags(&S.in_done, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&S.graph_done, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&S.out_done, cudaEventDisableTiming));
  }
  if (!c->io_in) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c->io_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->io_out, cudaStreamNonBlocking));
  }
  if (logits) {
    size_t need = (size_t)c->user_batch * (logits_dtype == ASR_ENTROPY_GIVEN ? 1 : s.vocab) *
                  (logits_dtype == ASR_KV_BF16 ? 2 : 4);
    if (need > S.logits_bytes) {
      CUDA_TRY(c->alloc(&S.logits, need));
      S.logits_bytes = need;
    }
  }
  return ASR_OK;
}

static cudaError_t prof_mark(asr_ctx* c, std::array<cudaEvent_t, asr::kStages + 1>* ev, int k, cudaStream_t st) {
  if (!ev) return cudaSuccess;
  return cudaEventRecord((*ev)[k], st);
}

// ---------------------------------------------------------------------------------------- one step
// A step is prepared (inputs staged, profiling events), launched in one or two parts (the full step,
// or attend + decide around the head-sharded all-reduce), then finished (mirror, outputs, counters).
enum Part { kPartFull = 0, kPartAttend = 1, kPartDecide = 2 };

struct StepArgs {
  bool has_logits = false, host_io = false, ent_given = false;
  int logits_dtype = 0;
  const void *q = nullptr, *kn = nullptr, *vn = nullptr, *lg = nullptr;
  float *o = nullptr, *ent = nullptr;           // device outputs (staging in host-io mode)
  float *o_user = nullptr, *ent_user = nullptr;  // caller's outputs
  std::array<cudaEvent_t, asr::kStages + 1>* ev = nullptr;
  bool ev_done[asr::kStages + 1] = {false, false, false, false};
  DevState sd{};
};

struct StepArgsBox {
  StepArgs a;
};
asr_ctx::~asr_ctx() { release(); }

static asr_status step_prepare(asr_ctx* c, const asr_step_io* io, cudaStream_t st, StepArgs& a) {
  if (!io || !io->q || !io->k_new || !io->v_new || !io->o) return fail(ASR_E_INVALID, "io has NULL q/k_new/v_new/o");
  if (io->memory != ASR_MEM_DEVICE && io->memory != ASR_MEM_HOST) return fail(ASR_E_INVALID, "io->memory");
  const DevState& s = c->s;
  a.ent_given = io->logits_prev != nullptr && io->logits_dtype == ASR_ENTROPY_GIVEN;
  a.has_logits = io->logits_prev != nullptr && s.vocab > 0 && !a.ent_given;
  a.logits_dtype = io->logits_dtype;
  if (a.has_logits && io->logits_dtype != ASR_KV_BF16 && io->logits_dtype != ASR_KV_F32)
    return fail(ASR_E_INVALID, "logits_dtype");
  for (int b = 0; b < s.B; ++b)
    if (c->prompt_len[b] + c->step + 1 > c->cfg.max_context)
      return fail(ASR_E_CAPACITY, "sequence " + std::to_string(b) + " is at max_context");
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  a.q = io->q;
  a.kn = io->k_new;
  a.vn = io->v_new;
  a.lg = io->logits_prev;
  a.o = a.o_user = io->o;
  a.ent = a.ent_user = io->entropy;
  a.host_io = io->memory == ASR_MEM_HOST;
  asr_ctx::Staging& S = c->stg[c->step & 1];
  if (a.host_io) {
    asr_status r = ensure_staging(c, S, a.has_logits || a.ent_given, a.ent_given ? ASR_ENTROPY_GIVEN : io->logits_dtype);
    if (r) return r;
    // inputs: copied on io_in as soon as the step is issued (overlapping the previous step's kernels),
    // once the graph that last read this staging set is done
    if (S.used) CUDA_TRY(cudaStreamWaitEvent(c->io_in, S.graph_done, 0));
    const size_t qb = (size_t)s.B * s.L * s.Hq * s.d * c->kv_elem;
    const size_t kb = (size_t)s.B * s.L * s.Hkv * s.d * c->kv_elem;
    CUDA_TRY(cudaMemcpyAsync(S.q, a.q, qb, cudaMemcpyHostToDevice, c->io_in));
    CUDA_TRY(cudaMemcpyAsync(S.k, a.kn, kb, cudaMemcpyHostToDevice, c->io_in));
    CUDA_TRY(cudaMemcpyAsync(S.v, a.vn, kb, cudaMemcpyHostToDevice, c->io_in));
    c->bytes_h2d += (int64_t)(qb + 2 * kb);
    if (a.has_logits || a.ent_given) {
      const size_t lb = a.ent_given ? (size_t)c->user_batch * 4
                                    : (size_t)c->user_batch * s.vocab * (io->logits_dtype == ASR_KV_BF16 ? 2 : 4);
      CUDA_TRY(cudaMemcpyAsync(S.logits, a.lg, lb, cudaMemcpyHostToDevice, c->io_in));
      c->bytes_h2d += (int64_t)lb;
      a.lg = S.logits;
    }
    CUDA_TRY(cudaEventRecord(S.in_done, c->io_in));
    CUDA_TRY(cudaStreamWaitEvent(st, S.in_done, 0));
    // the outputs this staging set held two steps ago must have left before the kernels overwrite them
    if (S.used) CUDA_TRY(cudaStreamWaitEvent(st, S.out_done, 0));
    a.q = S.q;
    a.kn = S.k;
    a.vn = S.v;
    a.o = S.o;
    a.ent = a.ent ? S.ent : nullptr;
  }
  if (c->cfg.profile_stages) {
    if (c->prof_free.empty()) {
      std::array<cudaEvent_t, asr::kStages + 1> e;
      for (auto& x : e) CUDA_TRY(cudaEventCreate(&x));
      c->prof_free.push_back(e);
    }
    c->prof_pending.push_back(c->prof_free.back());
    c->prof_free.pop_back();
    a.ev = &c->prof_pending.back();
  }
  a.sd = s;   // the step's view: timeline stamps when profiling the fused kernel or on request
  if (a.ent_given) a.sd.ent_given = static_cast<const float*>(a.lg);   // H per sequence, no logits pass
  if (c->timeline_on) a.sd.tl = c->tl_buf;
  if (a.sd.tl) {   // timeline of this step: start stamps = +inf, end stamps = 0 (+ phase D detail)
    unsigned long long init[asr::kTimelineSlots];
    for (int k = 0; k < asr::kTimelineSlots; ++k)
      init[k] = asr::tl_is_min(k) ? ~0ull : 0ull;
    CUDA_TRY(cudaMemcpyAsync(a.sd.tl, init, sizeof(init), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(a.sd.tl + asr::kTimelineSlots, 0,
                             sizeof(unsigned long long) * asr::kTraceRows * asr::kTraceCols, st));
  }
  return ASR_OK;
}

// The step's kernels and their dependencies (A_i was compacted by the previous step's phase D).
//  batch 1, tensor-core path (DevState::pre_in_attn):
//     attention (phase A + B on an extra warp of CTAs 0..95; a second pass inside the kernel only if
//     recovery recompacted A_i) --> { combine, [scoresum -->] phase D }
//  otherwise:
//     phase A (+B) --PDL--> attention --> { combine, [scoresum -->] phase D }, and in pressure mode the
//     prefetch copy kernel as a branch after phase A (nothing waits on it within the step).
//  (--> = full edge: a dependent launched early beside the attention waits for whole SMs and then ran
//  its latency chain slower than a fresh launch.)
// A profiled step (event nodes between the stages) runs the same kernels as a chain.
static asr_status step_launch(asr_ctx* c, StepArgs& a, int part, cudaStream_t st) {
  const DevState& s = c->s;
  const DevState& sd = a.sd;
  const bool prof = a.ev != nullptr;
  asr::KNode kn_list[8];
  int stage_of[8];   // 0 ledger pre, 1 attention, 2 decide/combine (profiling events)
  int nk = 0;
  const void* lgp = a.has_logits ? a.lg : nullptr;
  float* entp = (a.has_logits || a.ent_given) ? a.ent : nullptr;
  int kT = -1;
  if (part != kPartDecide) {
    if (s.pre_in_attn) {
      asr::node_attention(kn_list[nk], sd, a.q, a.kn, a.vn, c->attn_grid, lgp, a.logits_dtype, entp, a.o);
      stage_of[nk++] = 1;
    } else {
      const int kA = nk;
      asr::node_phaseA(kn_list[nk], sd, lgp, a.logits_dtype, a.kn, a.vn, entp);
      stage_of[nk++] = 0;
      if (s.pool_mode) {
        asr::node_copy(kn_list[nk], sd, 32);
        kn_list[nk].dep_full[0] = kA;
        stage_of[nk++] = 1;
      }
      asr::node_attention(kn_list[nk], sd, a.q, a.kn, a.vn, c->attn_grid, nullptr, 0, nullptr, a.o);
      kn_list[nk].dep_prog = kA;
      stage_of[nk++] = 1;
    }
    kT = nk - 1;
    if (s.sharded) {
      asr::node_scoresum(kn_list[nk], sd);
      kn_list[nk].dep_prog = kT;
      stage_of[nk++] = 2;
    }
  }
  if (part != kPartAttend && !s.fuse_tail) {   // decide (after scoresum in head-shard mode) — on the critical path
    asr::node_phaseD(kn_list[nk], sd, a.o);
    if (part == kPartFull) kn_list[nk].dep_full[0] = nk - 1;
    stage_of[nk++] = 2;
    if (s.pool_mode && s.evict_policy == ASR_EVICT_BELADY) {   // the Belady cut phase D computed
      asr::node_evict(kn_list[nk], sd, c->num_sms);
      kn_list[nk].dep_full[0] = nk - 1;
      stage_of[nk++] = 2;
    }
  }
  if (part != kPartDecide && !s.combine_in_decide && !s.fuse_tail) {
    // combine: a branch after the attention (full edges: kernels launched early beside the
    // attention wait for whole SMs and measured slower)
    asr::node_combine(kn_list[nk], sd, a.o);
    kn_list[nk].dep_full[0] = kT;
    stage_of[nk++] = 2;
  }
  const bool last_part = part != kPartAttend;
  auto record = [&](int k) -> cudaError_t {   // event k once per step
    if (!prof || a.ev_done[k]) return cudaSuccess;
    a.ev_done[k] = true;
    return cudaEventRecord((*a.ev)[k], st);
  };
  if (!c->use_graph) {   // direct launches in list order (a chain on the stream)
    for (int k = 0; k < nk; ++k) {
      for (int e = 0; e <= stage_of[k]; ++e) CUDA_TRY(record(e));
      CUDA_TRY(kn_list[k].launch(st));
    }
    if (last_part)
      for (int e = 0; e <= asr::kStages; ++e) CUDA_TRY(record(e));
  } else {
    const int variant = (a.has_logits ? 9 : 0) + (a.ent_given ? 18 : 0) + (a.host_io ? 3 * (1 + (int)(c->step & 1)) : 0) +
                        part;
    asr_ctx::StepGraph& G = c->graphs[variant];
    if (G.x && G.profiled != prof) {
      cudaGraphExecDestroy(G.x);
      cudaGraphDestroy(G.g);
      G = asr_ctx::StepGraph();
    }
    // the events this part records (stage boundaries it crosses)
    std::vector<int> evs;
    if (prof) {
      bool done[asr::kStages + 1];
      for (int e = 0; e <= asr::kStages; ++e) done[e] = a.ev_done[e];
      for (int k = 0; k < nk; ++k)
        for (int e = 0; e <= stage_of[k]; ++e)
          if (!done[e]) { evs.push_back(e); done[e] = true; }
      if (last_part)
        for (int e = 0; e <= asr::kStages; ++e)
          if (!done[e]) { evs.push_back(e); done[e] = true; }
    }
    if (!G.x) {
      CUDA_TRY(cudaGraphCreate(&G.g, 0));
      G.profiled = prof;
      std::vector<cudaGraphNode_t> node(nk, nullptr);
      cudaGraphNode_t prev = nullptr;   // profiled chain
      size_t ei = 0;
      auto add_events_upto = [&](int stage) -> asr_status {   // event nodes for boundaries <= stage
        while (ei < evs.size() && evs[ei] <= stage) {
          cudaGraphNode_t e;
          CUDA_TRY(cudaGraphAddEventRecordNode(&e, G.g, prev ? &prev : nullptr, prev ? 1 : 0, (*a.ev)[evs[ei]]));
          G.evnodes.push_back(e);
          prev = e;
          ++ei;
        }
        return ASR_OK;
      };
      for (int k = 0; k < nk; ++k) {
        if (prof) {   // serial chain with event nodes at the stage boundaries, no PDL
          asr_status r = add_events_upto(stage_of[k]);
          if (r) return r;
          CUDA_TRY(cudaGraphAddKernelNode(&node[k], G.g, prev ? &prev : nullptr, prev ? 1 : 0, &kn_list[k].p));
          prev = node[k];
        } else {
          CUDA_TRY(cudaGraphAddKernelNode(&node[k], G.g, nullptr, 0, &kn_list[k].p));
        }
        G.knodes.push_back(node[k]);
        G.last.push_back(kn_list[k]);
      }
      for (int k = 0; k < nk && !prof; ++k) {   // edges (a dependency may be listed after its dependent)
        for (int f : kn_list[k].dep_full)
          if (f >= 0) CUDA_TRY(cudaGraphAddDependencies(G.g, &node[f], &node[k], 1));
        const int pg = kn_list[k].dep_prog;
        if (pg < 0) continue;
        if (!c->use_pdl) {
          CUDA_TRY(cudaGraphAddDependencies(G.g, &node[pg], &node[k], 1));
          continue;
        }
        // programmatic edge: the kernel may launch once its upstream triggered (griddepcontrol.
        // launch_dependents); it calls griddepcontrol.wait before reading the upstream's results
        cudaGraphEdgeData ed{};
        ed.from_port = cudaGraphKernelNodePortProgrammatic;
        ed.to_port = 0;
        ed.type = cudaGraphDependencyTypeProgrammatic;
        CUDA_TRY(cudaGraphAddDependencies_v2(G.g, &node[pg], &node[k], &ed, 1));
      }
      if (prof) {
        asr_status r = add_events_upto(asr::kStages);
        if (r) return r;
      }
      CUDA_TRY(cudaGraphInstantiate(&G.x, G.g, 0));
    } else {
      for (int k = 0; k < nk; ++k) {
        if (memcmp(G.last[k].extra, kn_list[k].extra, sizeof(kn_list[k].extra)) != 0 ||
            memcmp(&G.last[k].s, &kn_list[k].s, sizeof(DevState)) != 0) {   // a pointer of the step changed
          CUDA_TRY(cudaGraphExecKernelNodeSetParams(G.x, G.knodes[k], &kn_list[k].p));
          memcpy(G.last[k].extra, kn_list[k].extra, sizeof(kn_list[k].extra));
          G.last[k].s = kn_list[k].s;
        }
      }
      for (size_t e = 0; e < evs.size(); ++e)
        CUDA_TRY(cudaGraphExecEventRecordNodeSetEvent(G.x, G.evnodes[e], (*a.ev)[evs[e]]));
    }
    for (int e : evs) a.ev_done[e] = true;
    CUDA_TRY(cudaGraphLaunch(G.x, st));
  }
  c->launches += nk;
  return ASR_OK;
}

static asr_status step_finish(asr_ctx* c, StepArgs& a, cudaStream_t st) {
  const DevState& s = c->s;
  // (a5) write-once host mirror of the appended token (side stream, overlapped with compute)
  if ((c->host_mirror || c->host_codes) && s.pool_mode) {
    c->bytes_d2h += (int64_t)s.B * c->mirror_tok_bytes;   // written by the append units (mapped mirror)
  } else if (c->host_mirror) {
    CUDA_TRY(cudaEventRecord(c->ev_append, st));
    CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_append, 0));
    const size_t pitch = (size_t)s.max_ctx * c->tok_bytes;
    if (c->uniform_prompt) {
      const size_t off = (size_t)(c->prompt_len[0] + c->step) * c->tok_bytes;
      CUDA_TRY(cudaMemcpy2DAsync((char*)c->host_mirror + off, pitch, (const char*)s.kv + off, pitch,
                                 c->tok_bytes, s.B, cudaMemcpyDeviceToHost, c->side));
    } else {
      for (int b = 0; b < s.B; ++b) {
        const size_t off = (size_t)b * pitch + (size_t)(c->prompt_len[b] + c->step) * c->tok_bytes;
        CUDA_TRY(cudaMemcpyAsync((char*)c->host_mirror + off, (const char*)s.kv + off, c->tok_bytes,
                                 cudaMemcpyDeviceToHost, c->side));
      }
    }
    c->bytes_d2h += (int64_t)s.B * c->tok_bytes;
  }
  if (a.host_io) {   // outputs leave on io_out while the next step computes (asr_flush / asr_stats)
    asr_ctx::Staging& S = c->stg[c->step & 1];
    CUDA_TRY(cudaEventRecord(S.graph_done, st));
    CUDA_TRY(cudaStreamWaitEvent(c->io_out, S.graph_done, 0));
    const size_t ob = (size_t)s.B * s.L * s.Hq * s.d * 4;
    CUDA_TRY(cudaMemcpyAsync(a.o_user, a.o, ob, cudaMemcpyDeviceToHost, c->io_out));
    c->bytes_d2h += (int64_t)ob;
    if (a.ent_user && (a.has_logits || a.ent_given)) {
      CUDA_TRY(cudaMemcpyAsync(a.ent_user, a.ent, (size_t)c->user_batch * 4, cudaMemcpyDeviceToHost, c->io_out));
      c->bytes_d2h += (int64_t)c->user_batch * 4;
    }
    CUDA_TRY(cudaEventRecord(S.out_done, c->io_out));
    c->last_out = S.out_done;
    S.used = true;
  }
  c->step++;
  c->last_stream = st;
  return ASR_OK;
}

asr_status asr_step(asr_ctx* c, const asr_step_io* io, void* cuda_stream) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  if (c->attend_pending) return fail(ASR_E_STATE, "asr_step_attend without asr_step_decide");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (c->s.sharded && !c->nccl_comm)
    return fail(ASR_E_STATE, "head-sharded context: use asr_step_attend / asr_step_decide or asr_attach_nccl");
  StepArgs a;
  asr_status r = step_prepare(c, io, st, a);
  if (r) return r;
  if (c->s.sharded) {
    r = step_launch(c, a, kPartAttend, st);
    if (r) return r;
    // sum the shards' per-token partial scores in place (NCCL over NVLink / NVSwitch): exactly the
    // sum_b |A_b| packed entries, whose count the attention part produced on the device
    CUDA_TRY(cudaEventRecord(c->ev_attend, st));
    CUDA_TRY(cudaEventSynchronize(c->ev_attend));
    const size_t count = (size_t)*(volatile int32_t*)c->tok_count_host;
    const int rc = c->nccl.all_reduce(c->s.tok_score, c->s.tok_score, count, 7 /*ncclFloat32*/, 0 /*ncclSum*/,
                                      c->nccl_comm, st);
    if (rc != 0) return fail(ASR_E_NCCL, std::string("ncclAllReduce: ") + c->nccl.err(rc));
    c->allreduce_bytes += (int64_t)count * 4;
    r = step_launch(c, a, kPartDecide, st);
  } else {
    r = step_launch(c, a, kPartFull, st);
  }
  if (r) return r;
  return step_finish(c, a, st);
}

asr_status asr_step_attend(asr_ctx* c, const asr_step_io* io, void* cuda_stream) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  if (c->attend_pending) return fail(ASR_E_STATE, "asr_step_attend twice without asr_step_decide");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  c->pending = std::make_unique<StepArgsBox>();
  asr_status r = step_prepare(c, io, st, c->pending->a);
  if (r) return r;
  r = step_launch(c, c->pending->a, kPartAttend, st);
  if (r) return r;
  c->attend_pending = true;
  c->last_stream = st;
  return ASR_OK;
}

asr_status asr_step_decide(asr_ctx* c, void* cuda_stream) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  if (!c->attend_pending) return fail(ASR_E_STATE, "asr_step_decide without asr_step_attend");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  asr_status r = step_launch(c, c->pending->a, kPartDecide, st);
  if (r) return r;
  c->attend_pending = false;
  r = step_finish(c, c->pending->a, st);
  c->pending.reset();
  return r;
}

asr_status asr_score_partials(asr_ctx* c, float** dev_ptr, int64_t* count) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  if (!dev_ptr || !count) return fail(ASR_E_INVALID, "NULL output");
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  CUDA_TRY(cudaStreamSynchronize(c->last_stream));
  *dev_ptr = c->s.tok_score;
  *count = (int64_t)*(volatile int32_t*)c->tok_count_host;
  return ASR_OK;
}

asr_status asr_nccl_unique_id(void* out, int32_t n) {
  if (!out || n < 128) return fail(ASR_E_INVALID, "out must hold 128 bytes");
  asr::NcclApi& api = asr::nccl_api();
  if (!api.ok) return fail(ASR_E_NCCL, "libnccl.so.2 not loadable");
  const int rc = api.get_unique_id(out);
  if (rc != 0) return fail(ASR_E_NCCL, std::string("ncclGetUniqueId: ") + api.err(rc));
  return ASR_OK;
}

asr_status asr_attach_nccl(asr_ctx* c, const void* unique_id, int32_t nranks, int32_t rank) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  if (!unique_id || nranks < 1 || rank < 0 || rank >= nranks) return fail(ASR_E_INVALID, "bad NCCL rank arguments");
  asr::NcclApi& api = asr::nccl_api();
  if (!api.ok) return fail(ASR_E_NCCL, "libnccl.so.2 not loadable");
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  void* comm = nullptr;
  const int rc = api.comm_init_rank(&comm, nranks, unique_id, rank);
  if (rc != 0) return fail(ASR_E_NCCL, std::string("ncclCommInitRank: ") + api.err(rc));
  c->nccl = api;
  c->nccl_comm = comm;
  // from now on every step runs attend -> all-reduce -> decide; cached graphs captured the
  // unsharded kernel arguments
  c->s.sharded = 1;
  c->s.fuse_tail = 0;   // the all-reduce sits between the attention and the decide
  for (auto& g : c->graphs) {
    if (g.x) cudaGraphExecDestroy(g.x);
    if (g.g) cudaGraphDestroy(g.g);
    g = asr_ctx::StepGraph();
  }
  return ASR_OK;
}

asr_status asr_restore(asr_ctx* c, int32_t seq, int32_t level, void* cuda_stream) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  if (seq < -1 || seq >= c->s.B) return fail(ASR_E_INVALID, "seq out of range");
  if (level != ASR_SR && level != ASR_WR && level != ASR_FR) return fail(ASR_E_INVALID, "level must be SR, WR or FR");
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  asr::KNode n;
  asr::node_restore(n, c->s, seq, level);
  CUDA_TRY(n.launch((cudaStream_t)cuda_stream));
  c->launches++;
  c->last_stream = (cudaStream_t)cuda_stream;
  return ASR_OK;
}

asr_status asr_stats(asr_ctx* c, int32_t seq, asr_stats_t* out, asr_ledger_view* detail) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  if (seq < 0 || seq >= c->s.B) return fail(ASR_E_INVALID, "seq out of range");
  if (!out) return fail(ASR_E_INVALID, "out is NULL");
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  CUDA_TRY(cudaStreamSynchronize(c->last_stream));
  CUDA_TRY(cudaStreamSynchronize(c->side));
  if (c->io_out) CUDA_TRY(cudaStreamSynchronize(c->io_out));
  const DevState& s = c->s;
  asr::SeqStats st;
  uint32_t err = 0;
  CUDA_TRY(cudaMemcpy(&st, s.stats + seq, sizeof(st), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(&err, s.err, 4, cudaMemcpyDeviceToHost));
  memset(out, 0, sizeof(*out));
  const int64_t n = c->prompt_len[seq] + c->step;
  out->step = c->step - 1;
  out->total = n;
  out->attended = st.attended;
  out->active = c->step > 0 ? (int64_t)st.attended - st.frozen_this_step + st.restored_tick : n;
  out->frozen = n - out->active;
  out->frozen_this_step = st.frozen_this_step;
  out->restored_this_step = (int64_t)st.restored_pre + st.restored_rec + st.restored_tick;
  out->compression = n > 0 ? 1.0 - (double)out->active / (double)n : 0.0;
  out->entropy = st.entropy;
  out->entropy_valid = st.entropy_valid;
  out->recovery_action = st.recovery_action;
  out->rewalk_requested = st.rewalk_requested;
  out->bytes_h2d = c->bytes_h2d;
  out->bytes_d2h = c->bytes_d2h;
  out->allreduce_bytes = c->allreduce_bytes;
  out->device_error = err;
  out->resident = n;
  if (s.pool_mode) {
    unsigned long long h2d = 0;
    CUDA_TRY(cudaMemcpy(&h2d, s.h2d, 8, cudaMemcpyDeviceToHost));
    out->bytes_h2d += (int64_t)h2d;
    std::vector<int32_t> so(n);
    if (n) CUDA_TRY(cudaMemcpy(so.data(), s.slot_of + (size_t)seq * s.max_ctx, n * 4, cudaMemcpyDeviceToHost));
    int64_t r = 0;
    for (int64_t j = 0; j < n; ++j) r += so[j] >= 0;
    out->resident = r;
    out->evicted_this_step = st.evicted;
    out->prefetched_this_step = st.prefetched;
    out->demand_restored_this_step = st.demand;
    unsigned long long stl[3] = {0, 0, 0};
    int32_t free_top = 0;
    CUDA_TRY(cudaMemcpy(stl, s.stall, 24, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(&free_top, s.free_top, 4, cudaMemcpyDeviceToHost));
    out->h2d_stall_ns = (int64_t)stl[0] + ((stl[1] && stl[2] > stl[1]) ? (int64_t)(stl[2] - stl[1]) : 0);
    out->free_slots = free_top;
  }
  if (detail) {
    if (detail->capacity < n) return fail(ASR_E_INVALID, "detail->capacity < total");
    const size_t base = (size_t)seq * s.max_ctx;
    if (detail->residency) {
      CUDA_TRY(cudaMemcpy(detail->residency, s.res + base, n, cudaMemcpyDeviceToHost));
      for (int64_t j = 0; j < n; ++j) detail->residency[j] = asr::res_active(detail->residency[j]) ? 1 : 0;
    }
    if (detail->timer) CUDA_TRY(cudaMemcpy(detail->timer, s.timer + base, n * 4, cudaMemcpyDeviceToHost));
    if (detail->count && s.hist_w > 0) {
      // detections within the window that ends at the last completed step
      std::vector<unsigned long long> hm(2 * (size_t)n);
      std::vector<int32_t> hs(n);
      if (n) {
        CUDA_TRY(cudaMemcpy(hm.data(), s.hmask + 2 * base, 16 * (size_t)n, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(hs.data(), s.hstep + base, 4 * (size_t)n, cudaMemcpyDeviceToHost));
      }
      const int64_t last = c->step - 1;
      for (int64_t j = 0; j < n; ++j) {
        int c2 = 0;
        for (int t = 0; t < 128; ++t) {
          const bool bit = (hm[2 * j + (t >> 6)] >> (t & 63)) & 1ull;
          if (bit && (int64_t)hs[j] - t > last - s.hist_w) ++c2;
        }
        detail->count[j] = (uint32_t)c2;
      }
    } else if (detail->count) {
      CUDA_TRY(cudaMemcpy(detail->count, s.count + base, n * 4, cudaMemcpyDeviceToHost));
    }
    if (detail->freeze_step) CUDA_TRY(cudaMemcpy(detail->freeze_step, s.fstep + base, n * 4, cudaMemcpyDeviceToHost));
    int32_t A = 0;
    const int p = (int)((c->step - 1) & 1);   // parity of the last step's A_i
    CUDA_TRY(cudaMemcpy(&A, s.act_len + (size_t)p * s.B + seq, 4, cudaMemcpyDeviceToHost));
    if (c->step == 0) A = 0;
    if (detail->active_len) *detail->active_len = A;
    if (detail->active_list && A)
      CUDA_TRY(cudaMemcpy(detail->active_list, s.act_pos + asr::act_off(s, p) + base, (size_t)A * 4,
                          cudaMemcpyDeviceToHost));
    if (detail->scores && A) CUDA_TRY(cudaMemcpy(detail->scores, s.score + base, (size_t)A * 4, cudaMemcpyDeviceToHost));
    if (detail->dequantized) {
      if (s.deq) CUDA_TRY(cudaMemcpy(detail->dequantized, s.deq + base, n, cudaMemcpyDeviceToHost));
      else memset(detail->dequantized, 0, n);
    }
  }
  if (err) return fail(ASR_E_INVARIANT, "device invariant violation, flags=" + std::to_string(err));
  return ASR_OK;
}

asr_status asr_read_kv(asr_ctx* c, int32_t seq, int32_t pos, int32_t from_mirror, void* k_out, void* v_out) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  const DevState& s = c->s;
  if (seq < 0 || seq >= s.B) return fail(ASR_E_INVALID, "seq out of range");
  if (pos < 0 || pos >= c->prompt_len[seq] + c->step) return fail(ASR_E_INVALID, "pos not stored");
  if (from_mirror && !c->host_mirror && !c->host_codes) return fail(ASR_E_INVALID, "no host mirror");
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  CUDA_TRY(cudaStreamSynchronize(c->last_stream));
  CUDA_TRY(cudaStreamSynchronize(c->side));
  std::vector<char> tok(c->tok_bytes);
  const size_t off = ((size_t)seq * s.max_ctx + pos) * c->tok_bytes;
  if (from_mirror && c->host_codes) {   // INT8 tier: the dequantised rows, bf16_rn(code * scale)
    const size_t R = (size_t)s.L * 2 * s.Hkv, r0 = ((size_t)seq * s.max_ctx + pos) * R;
    uint16_t* o = reinterpret_cast<uint16_t*>(tok.data());
    for (size_t r = 0; r < R; ++r)
      for (int e = 0; e < s.d; ++e) {
        const float x = (float)c->host_codes[(r0 + r) * s.d + e] * c->host_scales[r0 + r];
        uint32_t u;
        memcpy(&u, &x, 4);
        o[r * s.d + e] = (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);   // round to nearest even
      }
  } else if (from_mirror) {
    memcpy(tok.data(), (const char*)c->host_mirror + off, c->tok_bytes);
  } else {
    size_t doff = off;
    if (s.pool_mode) {
      int32_t slot = -1;
      CUDA_TRY(cudaMemcpy(&slot, s.slot_of + (size_t)seq * s.max_ctx + pos, 4, cudaMemcpyDeviceToHost));
      if (slot < 0) return fail(ASR_E_INVALID, "token is not resident on the device (evicted)");
      doff = (size_t)slot * c->tok_bytes;
    }
    CUDA_TRY(cudaMemcpy(tok.data(), (const char*)s.kv + doff, c->tok_bytes, cudaMemcpyDeviceToHost));
  }
  const size_t row = (size_t)s.Hkv * s.d * c->kv_elem;
  for (int l = 0; l < s.L; ++l) {
    if (k_out) memcpy((char*)k_out + l * row, tok.data() + (2 * l) * row, row);
    if (v_out) memcpy((char*)v_out + l * row, tok.data() + (2 * l + 1) * row, row);
  }
  return ASR_OK;
}

asr_status asr_stage_times(asr_ctx* c, double* ms, int32_t n, int64_t* launches) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  if (!ms || n < asr::kStages + 1) return fail(ASR_E_INVALID, "ms must hold 4 values");
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  CUDA_TRY(cudaStreamSynchronize(c->last_stream));
  for (int k = 0; k < n; ++k) ms[k] = 0.0;
  for (auto& a : c->prof_pending) {
    for (int k = 0; k < asr::kStages; ++k) {
      float t = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&t, a[k], a[k + 1]));
      ms[k] += t;
    }
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, a[0], a[asr::kStages]));
    ms[asr::kStages] += t;
    c->prof_free.push_back(a);
  }
  c->prof_pending.clear();
  if (launches) *launches = c->launches;
  c->launches = 0;
  return ASR_OK;
}

asr_status asr_timeline(asr_ctx* c, double* us, int32_t n) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  if (!c->timeline_on) return fail(ASR_E_STATE, "timeline off (set ASR_TIMELINE=1 before asr_create)");
  if (!us || n < 2 * asr::kStages) return fail(ASR_E_INVALID, "us must hold 6 values");
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  CUDA_TRY(cudaStreamSynchronize(c->last_stream));
  const int total = asr::kTimelineSlots + asr::kTraceRows * asr::kTraceCols;
  std::vector<unsigned long long> t(total);
  CUDA_TRY(cudaMemcpy(t.data(), c->tl_buf, sizeof(unsigned long long) * total, cudaMemcpyDeviceToHost));
  const int m = n < total ? n : total;
  for (int k = 0; k < m; ++k)
    us[k] = (k >= asr::kTimelineSlots && t[k] == 0) ? -1.0 : ((double)t[k] - (double)t[0]) * 1e-3;
  return ASR_OK;
}

asr_status asr_time_attention(asr_ctx* c, int32_t reps, void* cuda_stream) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  if (reps < 1) return fail(ASR_E_INVALID, "reps must be >= 1");
  if (c->attend_pending) return fail(ASR_E_STATE, "between asr_step_attend and asr_step_decide");
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  const DevState& s = c->s;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (!c->scratch_o) {
    const size_t qb = (size_t)s.B * s.L * s.Hq * s.d * c->kv_elem, kb = (size_t)s.B * s.L * s.Hkv * s.d * c->kv_elem;
    CUDA_TRY(c->alloc(&c->scratch_q, qb));
    CUDA_TRY(c->alloc(&c->scratch_k, kb));
    CUDA_TRY(c->alloc(&c->scratch_v, kb));
    CUDA_TRY(c->alloc(&c->scratch_o, (size_t)s.B * s.L * s.Hq * s.d * 4));
    CUDA_TRY(cudaMemsetAsync(c->scratch_q, 0, qb, st));
    CUDA_TRY(cudaMemsetAsync(c->scratch_k, 0, kb, st));
    CUDA_TRY(cudaMemsetAsync(c->scratch_v, 0, kb, st));
  }
  DevState sd = s;
  sd.pre_in_attn = 0;   // the attention alone
  sd.fuse_tail = 0;
  sd.tl = nullptr;
  sd.sk_learn = 0;      // uses the step's cut, leaves the rate / cut state as it was
  asr::KNode n;
  asr::node_attention(n, sd, c->scratch_q, c->scratch_k, c->scratch_v, c->attn_grid, nullptr, 0, nullptr,
                      c->scratch_o);
  for (int r = 0; r < reps; ++r) CUDA_TRY(n.launch(st));
  c->last_stream = st;
  return ASR_OK;
}

asr_status asr_step_policy(asr_ctx* c, const float* scores, const void* logits_prev, int32_t logits_dtype,
                           float* entropy, void* cuda_stream) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  if (!scores) return fail(ASR_E_INVALID, "asr_step_policy: scores is NULL");
  if (c->attend_pending) return fail(ASR_E_STATE, "between asr_step_attend and asr_step_decide");
  const DevState& s = c->s;
  if (s.pool_mode) return fail(ASR_E_STATE, "asr_step_policy: not with a slot pool (pool_tokens > 0)");
  const bool has_logits = logits_prev != nullptr && s.vocab > 0;
  if (has_logits && logits_dtype != ASR_KV_BF16 && logits_dtype != ASR_KV_F32)
    return fail(ASR_E_INVALID, "logits_dtype");
  for (int b = 0; b < s.B; ++b)
    if (c->prompt_len[b] + c->step + 1 > c->cfg.max_context)
      return fail(ASR_E_CAPACITY, "sequence " + std::to_string(b) + " is at max_context");
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  DevState sd = s;
  sd.ext_score = scores;
  sd.pre_in_attn = 0;
  sd.tl = nullptr;
  asr::KNode na, nd;
  asr::node_phaseA(na, sd, has_logits ? logits_prev : nullptr, logits_dtype, nullptr, nullptr,
                   has_logits ? entropy : nullptr);
  asr::node_phaseD(nd, sd, nullptr);
  CUDA_TRY(na.launch(st));
  CUDA_TRY(nd.launch(st));
  c->launches += 2;
  c->step++;
  c->last_stream = st;
  return ASR_OK;
}

asr_status asr_sample(const void* logits, int32_t logits_dtype, int32_t batch, int32_t vocab, float temperature,
                      int32_t top_k, float top_p, const float* uniforms, int32_t* token_out, void* cuda_stream) {
  if (!logits || !uniforms || !token_out) return fail(ASR_E_INVALID, "asr_sample: NULL pointer");
  if (logits_dtype != ASR_KV_BF16 && logits_dtype != ASR_KV_F32) return fail(ASR_E_INVALID, "asr_sample: logits_dtype");
  if (batch < 1 || batch > 65535 || vocab < 1 || vocab >= (1 << 24))   // grid.y = batch
    return fail(ASR_E_INVALID, "asr_sample: batch / vocab out of range");
  if (!isfinite(temperature) || !isfinite(top_p)) return fail(ASR_E_INVALID, "asr_sample: temperature / top_p");
  CUDA_TRY(asr::launch_sample(logits, logits_dtype, batch, vocab, temperature, top_k, top_p, uniforms, token_out,
                              1.f, nullptr, (cudaStream_t)cuda_stream));
  return ASR_OK;
}

asr_status asr_sample_entropy(const void* logits, int32_t logits_dtype, int32_t batch, int32_t vocab,
                              float temperature, int32_t top_k, float top_p, const float* uniforms, int32_t* token_out,
                              float entropy_temperature, float* entropy_out, void* cuda_stream) {
  if (!entropy_out) return fail(ASR_E_INVALID, "asr_sample_entropy: entropy_out is NULL");
  if (!(entropy_temperature > 0.f) || !isfinite(entropy_temperature))
    return fail(ASR_E_INVALID, "asr_sample_entropy: entropy_temperature must be > 0");
  if (!logits || !uniforms || !token_out) return fail(ASR_E_INVALID, "asr_sample_entropy: NULL pointer");
  if (logits_dtype != ASR_KV_BF16 && logits_dtype != ASR_KV_F32)
    return fail(ASR_E_INVALID, "asr_sample_entropy: logits_dtype");
  if (batch < 1 || batch > 65535 || vocab < 1 || vocab >= (1 << 24))
    return fail(ASR_E_INVALID, "asr_sample_entropy: batch / vocab out of range");
  if (!isfinite(temperature) || !isfinite(top_p)) return fail(ASR_E_INVALID, "asr_sample_entropy: temperature / top_p");
  CUDA_TRY(asr::launch_sample(logits, logits_dtype, batch, vocab, temperature, top_k, top_p, uniforms, token_out,
                              entropy_temperature, entropy_out, (cudaStream_t)cuda_stream));
  return ASR_OK;
}

static bool aligned(const void* p, uintptr_t a) { return ((uintptr_t)p & (a - 1)) == 0; }

static asr_status kvq_check(const char* fn, const void* kv, int64_t rows, int32_t n, int32_t bits, const void* codes,
                            const void* scales) {
  const std::string f(fn);
  if (!kv || !codes || !scales) return fail(ASR_E_INVALID, f + ": NULL pointer");
  if (rows < 0 || rows > ((int64_t)1 << 40)) return fail(ASR_E_INVALID, f + ": rows out of range [0, 2^40]");
  if (n != 8 && n != 16 && n != 32 && n != 64 && n != 128 && n != 256)
    return fail(ASR_E_INVALID, f + ": row_elems must be one of 8, 16, 32, 64, 128, 256");
  if (bits != 8 && bits != 4) return fail(ASR_E_INVALID, f + ": bits must be 8 or 4");
  if (!aligned(kv, 16) || !aligned(codes, 16) || !aligned(scales, 4))
    return fail(ASR_E_INVALID, f + ": misaligned pointer (kv and codes 16 B, scales 4 B)");
  return ASR_OK;
}

asr_status asr_kv_quantize(const void* kv, int64_t rows, int32_t row_elems, int32_t bits, void* codes, float* scales,
                           void* cuda_stream) {
  const asr_status st = kvq_check("asr_kv_quantize", kv, rows, row_elems, bits, codes, scales);
  if (st != ASR_OK) return st;
  CUDA_TRY(asr::launch_kv_quantize(kv, (long)rows, row_elems, bits, (int8_t*)codes, scales, (cudaStream_t)cuda_stream));
  return ASR_OK;
}

asr_status asr_kv_dequantize(const void* codes, const float* scales, int64_t rows, int32_t row_elems, int32_t bits,
                             void* kv, void* cuda_stream) {
  const asr_status st = kvq_check("asr_kv_dequantize", kv, rows, row_elems, bits, codes, scales);
  if (st != ASR_OK) return st;
  CUDA_TRY(asr::launch_kv_dequantize((const int8_t*)codes, scales, (long)rows, row_elems, bits, kv,
                                     (cudaStream_t)cuda_stream));
  return ASR_OK;
}

asr_status asr_set_profile(asr_ctx* c, int32_t on) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  c->cfg.profile_stages = on ? 1 : 0;
  return ASR_OK;
}

asr_status asr_flush(asr_ctx* c, void* cuda_stream) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  if (c->last_out) CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)cuda_stream, c->last_out, 0));
  return ASR_OK;
}

asr_status asr_destroy(asr_ctx* c) {
  if (!c) return fail(ASR_E_STATE, "context is NULL");
  cudaSetDevice(c->cfg.device);
  cudaStreamSynchronize(c->last_stream);
  cudaStreamSynchronize(c->side);
  if (c->io_in) cudaStreamSynchronize(c->io_in);
  if (c->io_out) cudaStreamSynchronize(c->io_out);
  delete c;
  return ASR_OK;
}

}  // extern "C"
