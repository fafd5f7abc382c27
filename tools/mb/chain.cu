#include <cstdio>
#include <cstdint>
__global__ void k_chain(const uint32_t* masks, int nchunk, float t0, float t1, float* out, long long* cyc, int mode) {
  float a = 0.f;
  long long c0 = clock64();
  if (mode == 0) {
    for (int k = 0; k < nchunk; ++k) {
      uint32_t m = masks[k];
#pragma unroll
      for (int i = 0; i < 16; ++i) a = __fadd_rn(a, ((m >> i) & 1u) ? t1 : t0);
    }
  } else if (mode == 1) {  // pure chain, no selects
#pragma unroll 16
    for (int k = 0; k < nchunk * 16; ++k) a = __fadd_rn(a, t1);
  } else if (mode == 3) {  // software pipeline: selects of chunk k+1 while adding chunk k
    float v[16], w[16];
    uint32_t m = masks[0];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = ((m >> i) & 1u) ? t1 : t0;
    for (int k = 0; k < nchunk; ++k) {
      const uint32_t mn = k + 1 < nchunk ? masks[k + 1] : 0u;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        a = __fadd_rn(a, v[i]);
        w[i] = ((mn >> i) & 1u) ? t1 : t0;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = w[i];
    }
  } else {  // selects precomputed into registers per chunk, adds separately
    for (int k = 0; k < nchunk; ++k) {
      uint32_t m = masks[k];
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = ((m >> i) & 1u) ? t1 : t0;
#pragma unroll
      for (int i = 0; i < 16; ++i) a = __fadd_rn(a, v[i]);
    }
  }
  long long c1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
int main() {
  int n = 574;
  uint32_t* m; float* o; long long* c;
  cudaMalloc(&m, n * 4); cudaMalloc(&o, 128 * 4); cudaMalloc(&c, 8);
  cudaMemset(m, 0x5a, n * 4);
  for (int mode = 0; mode < 4; ++mode) {
    for (int threads : {16, 32}) {
      k_chain<<<1, threads>>>(m, n, 0.1f, 0.2f, o, c, mode);
      k_chain<<<1, threads>>>(m, n, 0.1f, 0.2f, o, c, mode);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("mode %d threads %d: %lld cycles, %.2f per add\n", mode, threads, h, (double)h / (n * 16));
    }
  }
  return 0;
}
