// tools/microbench_latency.cu — measurement tool (not part of the product): latency of dependent
// global loads on B200 — DRAM (after a 512 MiB flush), L2 hits, ld.global.cg — and of the
// threadfence + atomicAdd ticket, to calibrate the ledger kernels' latency chains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbl tools/microbench_latency.cu
#include <cuda_runtime.h>
#include <stdio.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// chase: p[i] holds the index of the next element (stride apart); 16 dependent loads
__global__ void chase(const int* p, int start, int n, unsigned long long* out, int cg) {
  int j = start;
  unsigned long long t0 = gt();
  for (int k = 0; k < n; ++k) j = cg ? __ldcg(p + j) : p[j];
  unsigned long long t1 = gt();
  out[0] = (t1 - t0) / n;
  out[1] = j;
}

__global__ void ticket(int* c, unsigned long long* out) {
  unsigned long long t0 = gt();
  for (int k = 0; k < 16; ++k) {
    __threadfence();
    atomicAdd(c, 1);
  }
  unsigned long long t1 = gt();
  out[0] = (t1 - t0) / 16;
}

__global__ void touch(char* f, size_t n) {
  for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16; i < n; i += (size_t)gridDim.x * blockDim.x * 16)
    *reinterpret_cast<int4*>(f + i) = make_int4(1, 2, 3, 4);
}

int main() {
  const int N = 1 << 24;   // 64 MiB of ints
  int* p;
  cudaMalloc(&p, N * 4L);
  int* h = new int[N];
  const int stride = 1 << 16;   // 256 KiB apart: a new page-ish line every hop
  for (int i = 0; i < N; ++i) h[i] = (i + stride) % N;
  cudaMemcpy(p, h, N * 4L, cudaMemcpyHostToDevice);
  char* f;
  const size_t F = 512ul << 20;
  cudaMalloc(&f, F);
  unsigned long long* o;
  cudaMalloc(&o, 64);
  unsigned long long r[2];
  for (int cg = 0; cg < 2; ++cg) {
    touch<<<1024, 256>>>(f, F);
    chase<<<1, 1>>>(p, 0, 16, o, cg);
    cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
    printf("cg=%d after flush: %llu ns per dependent load\n", cg, r[0]);
    chase<<<1, 1>>>(p, 0, 16, o, cg);
    cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
    printf("cg=%d warm (same lines): %llu ns per dependent load\n", cg, r[0]);
  }
  // small stride (same 2 MiB region), after flush
  for (int i = 0; i < N; ++i) h[i] = (i + 64) % N;
  cudaMemcpy(p, h, N * 4L, cudaMemcpyHostToDevice);
  touch<<<1024, 256>>>(f, F);
  chase<<<1, 1>>>(p, 0, 16, o, 0);
  cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
  printf("after flush, 256 B hops: %llu ns per dependent load\n", r[0]);
  int* c;
  cudaMalloc(&c, 4);
  cudaMemset(c, 0, 4);
  ticket<<<1, 1>>>(c, o);
  cudaMemcpy(r, o, 8, cudaMemcpyDeviceToHost);
  printf("threadfence + atomicAdd: %llu ns\n", r[0]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
