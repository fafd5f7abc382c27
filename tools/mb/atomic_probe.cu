// Same-address global atomics from many warps: cost of one RED per warp on a
// shared counter vs a per-CTA shared-memory reduction with one RED per CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomic_probe atomic_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_warp_red(unsigned long long* c, int iters, int two) {
  for (int i = 0; i < iters; ++i) {
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(c, 1ull);
      if (two) atomicAdd(c + 1, 1ull);
    }
  }
}

__global__ void k_cta_red(unsigned long long* c, int iters, int two) {
  __shared__ unsigned long long s[2];
  if (threadIdx.x < 2) s[threadIdx.x] = 0;
  __syncthreads();
  for (int i = 0; i < iters; ++i) {
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&s[0], 1ull);
      if (two) atomicAdd(&s[1], 1ull);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(c, s[0]);
    if (two) atomicAdd(c + 1, s[1]);
  }
}

__global__ void k_none(unsigned long long* c, int iters, int two) {
  if (c == nullptr) c[0] = iters + two;
}

int main() {
  unsigned long long* c;
  cudaMalloc(&c, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 740, threads = 256;
  for (int iters : {1, 6, 12}) {
    for (int two : {0, 1}) {
      for (int kind = 0; kind < 3; ++kind) {
        float best = 1e9f;
        for (int rep = 0; rep < 20; ++rep) {
          cudaMemset(c, 0, 64);
          cudaEventRecord(a);
          if (kind == 0) k_warp_red<<<blocks, threads>>>(c, iters, two);
          else if (kind == 1) k_cta_red<<<blocks, threads>>>(c, iters, two);
          else k_none<<<blocks, threads>>>(c, iters, two);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        unsigned long long h[2];
        cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
        printf("{\"iters\": %d, \"two\": %d, \"kind\": \"%s\", \"us\": %.2f, \"count0\": %llu}\n", iters, two,
               kind == 0 ? "warp_red" : kind == 1 ? "cta_red" : "empty", best * 1e3, h[0]);
      }
    }
  }
  return 0;
}
