// Microbenchmark: dependent FADD chain fed from shared memory (consumer of
// the long stub kernel), alone and with producer warps + phase barriers.
#include <cstdio>
#include <cstdint>
constexpr int G = 16, PH = 32;
__global__ void k(const uint32_t* masks, int nchunk, float t0, float t1, float* out, long long* cyc, int mode) {
  extern __shared__ float vals[];  // [2][PH][16][G]
  __shared__ float st0[G], st1[G];
  if (threadIdx.x < G) { st0[threadIdx.x] = t0 + threadIdx.x; st1[threadIdx.x] = t1 + threadIdx.x; }
  __syncthreads();
  float a = 0.f;
  long long c0 = clock64();
  if (mode == 0) {  // consumer alone from a static smem buffer (no producers)
    for (int e = threadIdx.x; e < 2 * PH * 16 * G; e += blockDim.x) vals[e] = (e & 1) ? t1 : t0;
    __syncthreads();
    c0 = clock64();
    if (threadIdx.x < G) {
      for (int k = 0; k < nchunk; ++k) {
        const float* vp = vals + (k % (2 * PH)) * 16 * G + threadIdx.x;
        float x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = vp[i * G];
#pragma unroll
        for (int i = 0; i < 16; ++i) a = __fadd_rn(a, x[i]);
      }
    }
  } else {  // phases: warps 1..3 produce, warp 0 lanes < G consume, barrier per phase
    const int nph = (nchunk + PH - 1) / PH;
    for (int p = 0; p <= nph; ++p) {
      if (threadIdx.x >= 32 && p < nph) {
        float* dst = vals + (p & 1) * PH * 16 * G;
        for (int e = threadIdx.x - 32; e < PH * 16; e += blockDim.x - 32) {
          const float* src = ((masks[p * PH + (e >> 4)] >> (e & 15)) & 1u) ? st1 : st0;
#pragma unroll
          for (int d = 0; d < G; d += 4) *reinterpret_cast<float4*>(dst + e * G + d) = *reinterpret_cast<const float4*>(src + d);
        }
      }
      if (p > 0 && threadIdx.x < G) {
        const float* base = vals + ((p - 1) & 1) * PH * 16 * G + threadIdx.x;
        for (int kk = 0; kk < PH; ++kk) {
          const float* vp = base + kk * 16 * G;
          float x[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) x[i] = vp[i * G];
#pragma unroll
          for (int i = 0; i < 16; ++i) a = __fadd_rn(a, x[i]);
        }
      }
      __syncthreads();
    }
  }
  long long c1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
int main() {
  int n = 576;
  uint32_t* m; float* o; long long* c;
  cudaMalloc(&m, n * 4); cudaMalloc(&o, 1024 * 4); cudaMalloc(&c, 8);
  cudaMemset(m, 0x5a, n * 4);
  int smem = 2 * PH * 16 * G * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    for (int threads : {32, 128, 256}) {
      k<<<1, threads, smem>>>(m, n, 0.1f, 0.2f, o, c, mode);
      k<<<1, threads, smem>>>(m, n, 0.1f, 0.2f, o, c, mode);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("mode %d threads %d: %lld cycles, %.2f per add (%s)\n", mode, threads, h, (double)h / (n * 16),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
