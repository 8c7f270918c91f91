// paper_2512_11221_b200/csrc/kernels_ledger.cu — the ledger kernels of a step (units in step_units.cuh):
//   phaseA_kernel   (a6) entropy splits, (a0) append; the last unit of each sequence runs its phase B
//                   (entropy, detector, ladder, recovery + recompaction)
//   [attention]     kernels_attn_mma.cu / kernels_attn.cu
//   phaseD_kernel   (a2) decide + tick, A_{i+1} (last decide block of a sequence) and (a4') combine;
//                   the last decide block overall advances the step
//   prepare_kernel  A_0 at asr_create;  restore_kernel  explicit SR / WR / FR (asr_restore)
#include "step_units.cuh"

namespace asr {
namespace {

constexpr int kUnitThreads = 512;
#ifndef ASR_PHASED_THREADS
#define ASR_PHASED_THREADS 512
#endif
#ifndef ASR_PHASED_MINB
#define ASR_PHASED_MINB 1
#endif
constexpr int kPhaseDThreads = ASR_PHASED_THREADS;   // phase-D block size (128 / 256 measured slower: profiles/r2/phaseD_block_ab.txt)
constexpr int kPhaseAThreads = 256;   // 16K registers: a phase-A block fits beside an attention CTA

// One phase-A unit per block (+ phase B of its sequence if it finishes last).
template <typename TL, typename TK>
__global__ void __launch_bounds__(kPhaseAThreads) phaseA_kernel(DevState s, const TL* logits, const TK* k_new,
                                                                const TK* v_new, float* entropy_out) {
  pdl_trigger();
  Stamp stamp(s.tl, 0);
  __shared__ units::UnitShm u;
  if (s.pool_mode && blockIdx.x == 0 && threadIdx.x == 0) {
    // the previous step's prefetch copies that outlasted its attention kernel: a host-link stall
    const unsigned long long ae = s.stall[1], ce = s.stall[2];
    if (ae && ce > ae) s.stall[0] += ce - ae;
    s.stall[1] = s.stall[2] = 0;
  }
  units::phaseA_block<TL, TK, true>(s, blockIdx.x, *s.step, logits, k_new, v_new, entropy_out, u);
}

// decide_blocks blocks per sequence: decide + tick (unit x of sequence b), then together A_{i+1} into
// the other parity (unit_next_list); the last decide block overall advances the step counter and
// clears the redo flag.  With combine_in_decide (small batch) further blocks combine O (one warp
// per (b, l, h)), saving the separate combine launch.
__global__ void __launch_bounds__(kPhaseDThreads, ASR_PHASED_MINB) phaseD_kernel(DevState s, float* __restrict__ o) {
  Stamp stamp(s.tl, 2);
  pdl_wait();      // every input comes from the attention kernel(s) and phase A
  if (s.tl && threadIdx.x == 0) atomicMin(&s.tl[2 * kStages + 8], gtimer());
  __shared__ units::UnitShm u;
  const int nd = s.decide_blocks * s.B;
  if ((int)blockIdx.x >= nd) {   // combine_in_decide: blocks after the decide blocks combine O
    if (!o) return;                // policy replay: no attention, nothing to combine
    const int wid = ((int)blockIdx.x - nd) * (kPhaseDThreads / 32) + (threadIdx.x >> 5);
    if (wid < s.B * s.L * s.Hq) units::combine_warp(s, wid, o);
    if (s.tl) {
      __syncthreads();
      if (threadIdx.x == 0) atomicMax(&s.tl[2 * kStages + 2], gtimer());
    }
    return;
  }
  {
    const int i = *s.step;
    const int b = blockIdx.x / s.decide_blocks;
    units::unit_decide(s, b, blockIdx.x % s.decide_blocks, s.decide_blocks, i, u);
    __syncthreads();
    if (s.tl && threadIdx.x == 0) atomicMax(&s.tl[2 * kStages], gtimer());
    units::unit_next_list(s, b, blockIdx.x % s.decide_blocks, s.decide_blocks, i, u);
    if (s.tl && threadIdx.x == 0) atomicMax(&s.tl[2 * kStages + 1], gtimer());
    if (threadIdx.x == 0) {
      // every block read *s.step at its start; the next kernel sees all writes of this one.  Release /
      // acquire: the last block sees every block's Belady histogram (pressure mode)
      if (atom_add_acqrel(s.ticket, 1) == nd - 1) {   // the last decide block of the step
        if (s.pool_mode && s.evict_policy == ASR_EVICT_BELADY) units::belady_cut(s, i);
        *s.ticket = 0;
        *s.redo = 0;
        *s.step = i + 1;
      }
    }
  }
}

// (a4') combine of the split-KV partials -> O, one warp per (b, l, h); a graph branch beside phase D.
constexpr int kCombineThreads = 256;
__global__ void __launch_bounds__(kCombineThreads) combine_kernel(DevState s, float* __restrict__ o) {
  pdl_wait();
  const int wid = (int)blockIdx.x * (kCombineThreads / 32) + (threadIdx.x >> 5);
  if (wid < s.B * s.L * s.Hq) units::combine_warp(s, wid, o);
  if (s.tl) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&s.tl[2 * kStages + 2], gtimer());
  }
}

// A_0 of every sequence (asr_create): one block per sequence.
__global__ void __launch_bounds__(kUnitThreads) prepare_kernel(DevState s) {
  __shared__ units::UnitShm u;
  units::unit_prepare(s, blockIdx.x, u);
}

// Head-sharded mode: per-token partial score sums of this shard (grid decide_blocks x B).
__global__ void __launch_bounds__(kUnitThreads) scoresum_kernel(DevState s) {
  pdl_wait();
  __shared__ units::UnitShm u;
  units::unit_score_sum(s, blockIdx.x / s.decide_blocks, blockIdx.x % s.decide_blocks, s.decide_blocks, *s.step, u);
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
  const unsigned long long t0 = gtimer();
  const int d = s.pool_mode ? units::demand_copies(s, b) : 0;
  if (d && threadIdx.x == 0) atomicAdd(&s.stall[0], gtimer() - t0);
  if (threadIdx.x == 0) {
    s.stats[b].pending_restored += r;
    s.stats[b].pending_demand += d;
  }
  if (n + 1 <= s.cap) units::compact_positions(s, b, n + 1, i, u);   // A_i with the restored tokens
}

// Pressure mode: fill the slots phase B allocated for next-step restores (graph branch beside the
// attention kernel; reads the pinned host mirror over the host link).
constexpr int kCopyThreads = 256;
__global__ void __launch_bounds__(kCopyThreads) copy_kernel(DevState s) {
  __shared__ int start[4097];
  units::prefetch_copies(s, start);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&s.stall[2], gtimer());   // vs the attention's end: stall if later
}

// Pressure mode, Belady policy: evict the cut phase D computed (after phase D, in the step graph).
constexpr int kEvictThreads = 256;
__global__ void __launch_bounds__(kEvictThreads) evict_kernel(DevState s) { units::evict_positions(s); }

}  // namespace

void node_phaseA(KNode& n, const DevState& s, const void* logits, int logits_dtype, const void* k_new,
                 const void* v_new, float* entropy_out) {
  n.s = s;
  n.set(0, logits);
  n.set(1, k_new);
  n.set(2, v_new);
  n.set(3, entropy_out);
  const bool lf = logits && logits_dtype == 1;
  const void* f;
  if (s.dtype == 0)
    f = lf ? (const void*)phaseA_kernel<float, __nv_bfloat16> : (const void*)phaseA_kernel<__nv_bfloat16, __nv_bfloat16>;
  else
    f = lf ? (const void*)phaseA_kernel<float, float> : (const void*)phaseA_kernel<__nv_bfloat16, float>;
  n.finalize(f, dim3(units::phaseA_units(s, logits != nullptr)), dim3(kPhaseAThreads), 0);
}

void node_phaseD(KNode& n, const DevState& s, float* o) {
  n.s = s;
  n.set(0, o);
  const int warps = s.B * s.L * s.Hq;
  const int wpb = kPhaseDThreads / 32;
  const int nc = s.combine_in_decide ? (warps + wpb - 1) / wpb : 0;
  n.finalize((const void*)phaseD_kernel, dim3(s.decide_blocks * s.B + nc), dim3(kPhaseDThreads), 0);
}

void node_combine(KNode& n, const DevState& s, float* o) {
  n.s = s;
  n.set(0, o);
  const int warps = s.B * s.L * s.Hq;
  const int wpb = kCombineThreads / 32;
  n.finalize((const void*)combine_kernel, dim3((warps + wpb - 1) / wpb), dim3(kCombineThreads), 0);
}

void node_prepare(KNode& n, const DevState& s) {
  n.s = s;
  n.finalize((const void*)prepare_kernel, dim3(s.B), dim3(kUnitThreads), 0);
}

void node_scoresum(KNode& n, const DevState& s) {
  n.s = s;
  n.finalize((const void*)scoresum_kernel, dim3(s.decide_blocks * s.B), dim3(kUnitThreads), 0);
}

void node_copy(KNode& n, const DevState& s, int grid) {
  n.s = s;
  n.finalize((const void*)copy_kernel, dim3(grid), dim3(kCopyThreads), 0);
}

void node_evict(KNode& n, const DevState& s, int grid) {
  n.s = s;
  n.finalize((const void*)evict_kernel, dim3(grid), dim3(kEvictThreads), 0);
}

void node_restore(KNode& n, const DevState& s, int seq, int level) {
  n.s = s;
  n.set(0, seq);
  n.set(1, level);
  n.finalize((const void*)restore_kernel, dim3(seq >= 0 ? 1 : s.B), dim3(1024), 0);
}

}  // namespace asr
