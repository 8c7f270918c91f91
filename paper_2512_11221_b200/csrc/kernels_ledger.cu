// paper_2512_11221_b200/csrc/kernels_ledger.cu — the generic multi-kernel schedule of the ledger
// units (step_units.cuh), used for every shape the persistent step kernel does not cover (fp32 KV,
// head_dim != 128, other GQA groupings):
//   phaseA_kernel   (a6) entropy splits, (a0) append, (a3) speculative compaction — one unit per block
//   phaseB_kernel   (a6) H, detector, ladder, recovery levels (+ recompaction)    — one block per sequence
//   [attention]     kernels_attn.cu
//   phaseD_kernel   (a2) decide + tick and (a4') combine; the last decide block advances the step
//   restore_kernel  explicit SR / WR / FR (asr_restore)
#include "step_units.cuh"

namespace asr {
namespace {

constexpr int kUnitThreads = 512;

template <typename TL, typename TK>
__global__ void __launch_bounds__(kUnitThreads) phaseA_kernel(DevState s, const TL* logits, const TK* k_new,
                                                              const TK* v_new) {
  pdl_trigger();
  Stamp stamp(s.tl, 0);
  __shared__ units::UnitShm u;
  units::run_phaseA_unit<TL, TK>(s, blockIdx.x, *s.step, logits, k_new, v_new, u);
}

__global__ void __launch_bounds__(kUnitThreads) phaseB_kernel(DevState s, int has_logits, float* entropy_out) {
  pdl_wait();
  pdl_trigger();
  Stamp stamp(s.tl, 0);
  __shared__ units::UnitShm u;
  units::unit_finish(s, blockIdx.x, *s.step, has_logits != 0, entropy_out, u);
}

// Blocks [0, decide_blocks * B): decide + tick (unit x of sequence b); the remaining blocks: combine,
// one warp per (b, l, h).  The last decide block (atomic ticket) advances the step counter.
__global__ void __launch_bounds__(kUnitThreads) phaseD_kernel(DevState s, float* __restrict__ o) {
  pdl_wait();      // every input comes from the attention kernel
  Stamp stamp(s.tl, 2);
  __shared__ units::UnitShm u;
  const int nd = s.decide_blocks * s.B;
  if ((int)blockIdx.x < nd) {
    const int i = *s.step;
    units::unit_decide(s, blockIdx.x / s.decide_blocks, blockIdx.x % s.decide_blocks, s.decide_blocks, i, u);
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(s.ticket, 1) == nd - 1) {
        *s.ticket = 0;
        *s.step = i + 1;
      }
    }
    return;
  }
  const int wid = ((int)blockIdx.x - nd) * (kUnitThreads / 32) + (threadIdx.x >> 5);
  if (wid < s.B * s.L * s.Hq) units::combine_warp(s, wid, o);
}

// Head-sharded mode: per-token partial score sums of this shard (grid decide_blocks x B).
__global__ void __launch_bounds__(kUnitThreads) scoresum_kernel(DevState s) {
  pdl_wait();
  units::unit_score_sum(s, blockIdx.x / s.decide_blocks, blockIdx.x % s.decide_blocks, s.decide_blocks);
}

// Explicit asr_restore at the boundary before step i (= *s.step); seq = -1 for all.  In pressure
// mode the evicted tokens it restores are copied back before it returns.
__global__ void __launch_bounds__(1024) restore_kernel(DevState s, int seq, int level) {
  __shared__ units::UnitShm u;
  const int b = seq >= 0 ? seq : (int)blockIdx.x;
  const int i = *s.step;
  const int n = s.prompt_len[b] + i;  // tokens currently held
  if (s.pool_mode && threadIdx.x == 0) s.cp_count[b] = 0;
  __syncthreads();
  const int r = units::block_sum_int(units::apply_level(s, b, n, level, i), u);
  const int d = s.pool_mode ? units::demand_copies(s, b) : 0;
  if (threadIdx.x == 0) {
    s.stats[b].pending_restored += r;
    s.stats[b].pending_demand += d;
  }
}

// Pressure mode: fill the slots phase B allocated for next-step restores (graph branch beside the
// attention kernel; reads the pinned host mirror over the host link).
constexpr int kCopyThreads = 256;
__global__ void __launch_bounds__(kCopyThreads) copy_kernel(DevState s) {
  __shared__ int start[4097];
  units::prefetch_copies(s, start);
}

}  // namespace

void node_phaseA(KNode& n, const DevState& s, const void* logits, int logits_dtype, const void* k_new,
                 const void* v_new) {
  n.s = s;
  n.set(0, logits);
  n.set(1, k_new);
  n.set(2, v_new);
  const bool lf = logits && logits_dtype == 1;
  const void* f;
  if (s.dtype == 0)
    f = lf ? (const void*)phaseA_kernel<float, __nv_bfloat16> : (const void*)phaseA_kernel<__nv_bfloat16, __nv_bfloat16>;
  else
    f = lf ? (const void*)phaseA_kernel<float, float> : (const void*)phaseA_kernel<__nv_bfloat16, float>;
  n.finalize(f, dim3(units::phaseA_units(s, logits != nullptr)), dim3(kUnitThreads), 0);
}

void node_phaseB(KNode& n, const DevState& s, int has_logits, float* entropy_out) {
  n.s = s;
  n.set(0, has_logits);
  n.set(1, entropy_out);
  n.finalize((const void*)phaseB_kernel, dim3(s.B), dim3(kUnitThreads), 0);
}

void node_phaseD(KNode& n, const DevState& s, float* o) {
  n.s = s;
  n.set(0, o);
  const int warps = s.B * s.L * s.Hq;
  const int wpb = kUnitThreads / 32;
  n.finalize((const void*)phaseD_kernel, dim3(s.decide_blocks * s.B + (warps + wpb - 1) / wpb), dim3(kUnitThreads), 0);
}

void node_scoresum(KNode& n, const DevState& s) {
  n.s = s;
  n.finalize((const void*)scoresum_kernel, dim3(s.decide_blocks * s.B), dim3(kUnitThreads), 0);
}

void node_copy(KNode& n, const DevState& s, int grid) {
  n.s = s;
  n.finalize((const void*)copy_kernel, dim3(grid), dim3(kCopyThreads), 0);
}

void node_restore(KNode& n, const DevState& s, int seq, int level) {
  n.s = s;
  n.set(0, seq);
  n.set(1, level);
  n.finalize((const void*)restore_kernel, dim3(seq >= 0 ? 1 : s.B), dim3(1024), 0);
}

}  // namespace asr
