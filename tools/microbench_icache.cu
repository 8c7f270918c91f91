// tools/microbench_icache.cu — measurement tool (not part of the product): cost of executing cold,
// straight-line code once (instruction fetch from L2 / DRAM) vs warm, on one warp per SM, to size
// the latency-bound tails of the step kernels.  Straight-line bodies of N independent integer ops.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbi tools/microbench_icache.cu
#include <cuda_runtime.h>
#include <stdio.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int N>
__global__ void body(unsigned* out, unsigned seed, unsigned long long* tsum) {
  unsigned a = seed + threadIdx.x, b = seed * 3u, c = seed ^ 0x9e3779b9u, d = seed + 7u;
  const unsigned long long t0 = gt();
#pragma unroll
  for (int k = 0; k < N; ++k) {   // 4 independent chains: ~N * 4 instructions of straight-line code
    a = a * 0x01000193u + k;
    b = (b ^ (k * 0x85ebca6bu)) + a;
    c = c * 5u + (b >> 3);
    d = d + (c ^ 0xc2b2ae35u);
  }
  const unsigned long long t1 = gt();
  if ((threadIdx.x & 31) == 0) atomicAdd(tsum, t1 - t0);
  if (a + b + c + d == 0x12345u) out[0] = a;
}

__global__ void flushl2(int4* f, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    f[i] = make_int4(1, 2, 3, 4);
}

template <int N>
void run(unsigned* out, unsigned long long* ts, int4* f, size_t fn) {
  unsigned long long h;
  for (int rep = 0; rep < 3; ++rep) {
    flushl2<<<1024, 256>>>(f, fn);
    cudaMemset(ts, 0, 8);
    body<N><<<148, 32>>>(out, rep, ts);   // cold after the flush (code in DRAM)
    cudaMemcpy(&h, ts, 8, cudaMemcpyDeviceToHost);
    const double cold = h / 148.0;
    cudaMemset(ts, 0, 8);
    body<N><<<148, 32>>>(out, rep + 1, ts);   // again: code in L2 (and maybe the SM's I-caches)
    cudaMemcpy(&h, ts, 8, cudaMemcpyDeviceToHost);
    const double warm = h / 148.0;
    printf("N=%5d (~%6d instr, %6.1f KB): after L2 flush %8.0f ns (%.2f ns/instr), re-run %8.0f ns (%.2f ns/instr)\n", N,
           4 * N, 4 * N * 16 / 1024.0, cold, cold / (4 * N), warm, warm / (4 * N));
  }
}

int main() {
  unsigned* out;
  unsigned long long* ts;
  int4* f;
  const size_t fn = (512ul << 20) / 16;
  cudaMalloc(&out, 64);
  cudaMalloc(&ts, 8);
  cudaMalloc(&f, fn * 16);
  run<64>(out, ts, f, fn);
  run<256>(out, ts, f, fn);
  run<1024>(out, ts, f, fn);
  run<2048>(out, ts, f, fn);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
