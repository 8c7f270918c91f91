// tools/microbench_compact.cu — measurement tool (not part of the product): latency of one block
// compacting a residency row (step_units.cuh compact_positions) at batch 1, 8K context, and of its
// pieces, with %globaltimer stamps, to find what dominates phase D's next-step preparation.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2512_11221_b200/csrc
//        -o tools/mbc tools/microbench_compact.cu
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include "step_units.cuh"

using namespace asr;

__global__ void k_compact(DevState s, int n, unsigned long long* t, int reps) {
  __shared__ units::UnitShm u;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    unsigned long long t0 = gtimer();
    units::compact_positions(s, 0, n, 1, u);
    unsigned long long t1 = gtimer();
    if (threadIdx.x == 0) t[r] = t1 - t0;
  }
}

// stamps inside a copy of compact_positions: t[0] load pass, t[1] after block scan, t[2] write pass
__global__ void k_parts(DevState s, int n, unsigned long long* t) {
  __shared__ units::UnitShm u;
  __syncthreads();
  const unsigned long long t0 = gtimer();
  const long base = 0;
  const uint32_t* res4 = reinterpret_cast<const uint32_t*>(s.res + base);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  const int ngrp = (n + 127) >> 7;
  const int per = (ngrp + nw - 1) / nw;
  const int g0 = min(ngrp, w * per), g1 = min(ngrp, g0 + per);
  uint32_t keep[8];
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    keep[k] = g0 + k < g1 ? units::active_bits4(res4, (g0 + k) * 32 + lane, 0, n) : 0u;
    cnt += __popc(keep[k]);
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) u.wsum[w] = cnt;
  const unsigned long long t1 = gtimer();
  __syncthreads();
  if (w == 0) {
    const int x = lane < nw ? u.wsum[lane] : 0;
    int xi = x;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    u.wsum[lane] = xi - x;
    if (lane == 31) u.total = xi;
  }
  __syncthreads();
  const unsigned long long t2 = gtimer();
  int off = u.wsum[w];
  int32_t* out = s.act_pos;
  for (int g = g0; g < g1; ++g) {
    const int q = g * 32 + lane;
    uint32_t m = 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (g - g0 == k) m = keep[k];
    const int c = __popc(m);
    int incl = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int o = off + incl - c;
    while (m) {
      const int j = 4 * q + __ffs(m) - 1;
      out[o] = j;
      ++o;
      m &= m - 1;
    }
    off += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncthreads();
  const unsigned long long t3 = gtimer();
  if (tid == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; }
}

__global__ void k_empty(unsigned long long* t) {
  unsigned long long t0 = gtimer();
  __syncthreads();
  if (threadIdx.x == 0) t[0] = gtimer() - t0;
}

int main() {
  const int n = 8200, max_ctx = 8256;
  DevState s{};
  s.B = 1;
  s.max_ctx = max_ctx;
  std::vector<uint8_t> res(max_ctx, 0);
  srand(1);
  for (int j = 0; j < n; ++j) res[j] = (j >= n - 512 || rand() % 8 == 0) ? 1 : (rand() % 3 == 0 ? 2 : 0);
  cudaMalloc(&s.res, max_ctx);
  cudaMemcpy(s.res, res.data(), max_ctx, cudaMemcpyHostToDevice);
  cudaMalloc(&s.act_pos, 2 * max_ctx * 4);
  cudaMalloc(&s.act_slot, 2 * max_ctx * 4);
  cudaMalloc(&s.act_len, 8);
  cudaMalloc(&s.err, 4);
  unsigned long long* t;
  cudaMalloc(&t, 64 * 8);
  for (int threads : {128, 256, 512, 1024}) {
    k_compact<<<1, threads>>>(s, n, t, 16);
    cudaDeviceSynchronize();
    unsigned long long h[16];
    cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %4d: compact ns first %llu, then", threads, h[0]);
    for (int r = 1; r < 16; r += 3) printf(" %llu", h[r]);
    printf("\n");
  }
  for (int threads : {256, 512, 1024}) {
    for (int r = 0; r < 3; ++r) k_parts<<<1, threads>>>(s, n, t);
    cudaDeviceSynchronize();
    unsigned long long h[3];
    cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %4d: load+reduce %llu ns, block scan %llu ns, write pass %llu ns\n", threads, h[0], h[1], h[2]);
  }
  k_empty<<<1, 512>>>(t);
  cudaDeviceSynchronize();
  unsigned long long h0;
  cudaMemcpy(&h0, t, 8, cudaMemcpyDeviceToHost);
  printf("globaltimer + syncthreads: %llu ns\n", h0);
  int len = 0;
  cudaMemcpy(&len, s.act_len + 1, 4, cudaMemcpyDeviceToHost);
  int cnt = 0;
  for (int j = 0; j < n; ++j) cnt += res[j] == 1;
  printf("act_len %d expected %d  (%s)\n", len, cnt, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
