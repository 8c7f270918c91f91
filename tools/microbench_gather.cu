// tools/microbench_gather.cu — measurement tool (not part of the product): achievable read bandwidth
// of the attention kernel's access pattern — 4 KiB K|V rows of (token, layer) gathered through a
// sorted active index list — for several load mechanisms, against a streaming read of the same bytes.
// 4 sequences x 8192 slots x 32 layers x 4 KiB = 4 GiB pool; active set ~1792 tokens per sequence.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbg tools/microbench_gather.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

// LDG: each warp reads whole 4 KiB rows, U rows in flight per warp
template <int U>
__global__ void gather_ldg(const uint4* __restrict__ base, const int* __restrict__ rows, int nrows,
                           unsigned long long* sink) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int r0 = warp * U; r0 < nrows; r0 += nw * U) {
    uint4 v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = min(r0 + u, nrows - 1);
      const uint4* p = base + (long)rows[r] * 256;
#pragma unroll
      for (int k = 0; k < 8; ++k) v[u][k] = __ldcg(p + k * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) { acc.x ^= v[u][k].x; acc.y ^= v[u][k].y; acc.z ^= v[u][k].z; acc.w ^= v[u][k].w; }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) atomicAdd(sink, 1ull);
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// cp.async.bulk (1-D TMA): one producer lane per CTA issues ROWS rows per stage (4 KiB each) into a
// NST-stage ring; the other warps "consume" (touch one word) and release the stage.
template <int ROWS, int NST>
__global__ void gather_bulk(const uint8_t* __restrict__ base, const int* __restrict__ rows, int nrows,
                            unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwc = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[i])), "r"(nwc));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int ntiles = (nrows + ROWS - 1) / ROWS;
  if (warp == nwc) {
    int g = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++g) {
      const int st = g % NST;
      const uint32_t ph = (g / NST) & 1;
      asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(
                       su32(&empty[st])), "r"(ph ^ 1) : "memory");
      const int cnt = min(ROWS, nrows - t * ROWS);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(cnt * 4096)
                     : "memory");
      __syncwarp();
      for (int k = lane; k < cnt; k += 32) {
        const uint8_t* src = base + (long)rows[t * ROWS + k] * 4096;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                         su32(sm + ((long)st * ROWS + k) * 4096)), "l"(src), "r"(su32(&full[st])) : "memory");
      }
    }
    return;
  }
  uint32_t acc = 0;
  int g = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++g) {
    const int st = g % NST;
    const uint32_t ph = (g / NST) & 1;
    asm volatile("{.reg .pred P; W2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W2;}" ::"r"(
                     su32(&full[st])), "r"(ph) : "memory");
    acc ^= *reinterpret_cast<const uint32_t*>(sm + ((long)st * ROWS + (warp % ROWS)) * 4096 + lane * 4);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])) : "memory");
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  const int B = 4, slots = 8192, L = 32;
  const size_t bytes = (size_t)B * slots * L * 4096;  // 4 GiB
  uint8_t* buf;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  std::vector<int> act;
  for (int t = 0; t < slots; ++t)
    if (t >= slots - 512 || t % 6 == 0) act.push_back(t);
  std::vector<int> rows_tm, rows_lm, rows_seq;
  for (int b = 0; b < B; ++b)
    for (int l = 0; l < L; ++l)
      for (int t : act) {
        rows_tm.push_back((b * slots + t) * L + l);          // token-major pool, item order
        rows_lm.push_back((l * B + b) * slots + t);          // layer-major pool
      }
  for (size_t k = 0; k < rows_tm.size(); ++k) rows_seq.push_back((int)k);
  const double mb = rows_tm.size() * 4096.0 / 1e6;
  printf("rows %zu, %.1f MB per pass\n", rows_tm.size(), mb);
  int* drows;
  CK(cudaMalloc(&drows, sizeof(int) * rows_tm.size()));
  uint8_t* l2flush;
  CK(cudaMalloc(&l2flush, 256 << 20));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, const std::vector<int>& rows, auto launch) {
    CK(cudaMemcpy(drows, rows.data(), sizeof(int) * rows.size(), cudaMemcpyHostToDevice));
    float best = 1e9;
    for (int it = 0; it < 8; ++it) {
      CK(cudaMemset(l2flush, it, 256 << 20));
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    printf("%-52s %8.1f us  %7.1f GB/s\n", name, best * 1e3, mb * 1e6 / (best * 1e-3) / 1e9);
  };
  const int n = (int)rows_tm.size();
  const uint4* b4 = reinterpret_cast<const uint4*>(buf);
  timeit("LDG U=1  streaming", rows_seq, [&] { gather_ldg<1><<<148 * 8, 256>>>(b4, drows, n, sink); });
  timeit("LDG U=2  streaming", rows_seq, [&] { gather_ldg<2><<<148 * 4, 256>>>(b4, drows, n, sink); });
  timeit("LDG U=1  token-major gather", rows_tm, [&] { gather_ldg<1><<<148 * 8, 256>>>(b4, drows, n, sink); });
  timeit("LDG U=2  token-major gather", rows_tm, [&] { gather_ldg<2><<<148 * 4, 256>>>(b4, drows, n, sink); });
  timeit("LDG U=2  layer-major gather", rows_lm, [&] { gather_ldg<2><<<148 * 4, 256>>>(b4, drows, n, sink); });
  auto bulk = [&](auto kern, int rows_per_stage, int nst, const std::vector<int>& rows, const char* name) {
    const int smem = rows_per_stage * nst * 4096;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    timeit(name, rows, [&] { kern<<<148, 32 * 9, smem>>>(buf, drows, n, sink); });
  };
  bulk(gather_bulk<16, 3>, 16, 3, rows_seq, "BULK 16 rows x 3 stages streaming");
  bulk(gather_bulk<16, 3>, 16, 3, rows_tm, "BULK 16 rows x 3 stages token-major gather");
  bulk(gather_bulk<8, 6>, 8, 6, rows_tm, "BULK 8 rows x 6 stages token-major gather");
  bulk(gather_bulk<4, 12>, 4, 12, rows_tm, "BULK 4 rows x 12 stages token-major gather");
  bulk(gather_bulk<2, 24>, 2, 24, rows_tm, "BULK 2 rows x 24 stages token-major gather");
  return 0;
}
