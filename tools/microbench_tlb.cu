// tools/microbench_tlb.cu — measurement tool (not part of the product): does streaming a large KV
// pool (the attention's gather: 4 KiB at a 128 KiB token stride, every layer) make the ledger
// kernels' later dependent loads slow through TLB misses?  Dependent-load latency (one thread, ld.cg)
// over a small array after gathering pools of 0 .. 16 GiB, hops within one 2 MiB page vs across pages.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbt tools/microbench_tlb.cu
#include <cuda_runtime.h>
#include <stdio.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void chase(const int* p, int start, int n, unsigned long long* out) {
  int j = start;
  unsigned long long t0 = gt();
  for (int k = 0; k < n; ++k) j = __ldcg(p + j);
  unsigned long long t1 = gt();
  out[0] = (t1 - t0) / n;
  out[1] = j;
}

// every CTA reads 4 KiB pieces (one per warp iteration) at token stride 128 KiB, all 32 "layers"
__global__ void gather(const char* pool, size_t tokens, unsigned long long* sink) {
  unsigned long long acc = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t nw = (size_t)gridDim.x * (blockDim.x >> 5);
  for (size_t t = blockIdx.x * (size_t)(blockDim.x >> 5) + warp; t < tokens * 32; t += nw) {
    const size_t tok = t % tokens, l = t / tokens;
    const int4* src = reinterpret_cast<const int4*>(pool + tok * 131072 + l * 4096);
    for (int k = lane; k < 256; k += 32) {
      int4 v = __ldcs(src + k);
      acc += v.x;
    }
  }
  if (acc == 42) sink[0] = acc;
}

int main() {
  const size_t A = 32u << 20;
  int* arena;
  cudaMalloc(&arena, A);
  const int N = (int)(A / 4);
  int* h = new int[N];
  unsigned long long* o;
  cudaMalloc(&o, 64);
  unsigned long long r[2];
  const size_t maxpool = 16ul << 30;
  char* pool = nullptr;
  if (cudaMalloc(&pool, maxpool) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(pool, 1, maxpool);
  for (int mode = 0; mode < 2; ++mode) {
    // mode 0: hops of 4 KiB inside the first 1 MiB (same page); mode 1: hops of 2 MiB + 4 KiB (new page each)
    const int hop = mode == 0 ? 1024 : (2 << 20) / 4 + 1024;
    const int span = mode == 0 ? (1 << 20) / 4 : N;
    for (int i = 0; i < N; ++i) h[i] = 0;
    for (int i = 0, k = 0; k < 16; ++k) { int nx = (i + hop) % span; h[i] = nx; i = nx; }
    cudaMemcpy(arena, h, A, cudaMemcpyHostToDevice);
    for (size_t gb : {0ul, 1ul, 4ul, 16ul}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (gb) gather<<<148, 512>>>(pool, (gb << 30) / 131072, o + 4);
        // evict the chase lines from L2: stream 256 MiB through a separate region of the pool
        gather<<<148, 512>>>(pool + (maxpool - (1ul << 30)), 2048, o + 4);
        chase<<<1, 1>>>(arena, 0, 16, o);
        cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
        unsigned long long cold = r[0];
        chase<<<1, 1>>>(arena, 0, 16, o);
        cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
        printf("%s hops, after gathering %2zu GiB pool: cold %4llu ns, warm %4llu ns per dependent load\n",
               mode == 0 ? "in-page   " : "cross-page", gb, cold, r[0]);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
