// DLRM feature interaction (DLRM mode, next to the EmbeddingBag kernels):
// per sample, z = [x; e_0 .. e_{T-1}] (n = T+1 vectors of D), and the top
// MLP's input row is [x | z_i . z_j for i > j in row-major lower-triangle
// order (torch.tril_indices(n, n, -1)) | zero padding to out_stride].
// One fused kernel replaces cat + bmm + triangle gather + cat (and their
// backward: bmm x2 + index_add + slicing): a warp per sample stages z in
// shared memory, all dots in fp32, bf16 or fp32 I/O.
//
// Backward: with G the symmetric pair-gradient matrix (zero diagonal),
// dz = G z; dx = dout[:, :D] + dz_0, demb_t = dz_{t+1}.
#include "internal.cuh"

#include <cuda_bf16.h>

namespace bp {

constexpr int kIxWarps = 8;

__device__ __forceinline__ float ld_any(const void* p, long long i, int bf16) {
  return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]) : reinterpret_cast<const float*>(p)[i];
}

__device__ __forceinline__ void st_any(void* p, long long i, float v, int bf16) {
  if (bf16) reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else reinterpret_cast<float*>(p)[i] = v;
}

// smem per warp: z[n][D+1]; per block: pair table (i, j) of the lower triangle
__global__ void __launch_bounds__(kIxWarps * 32) k_interact_fwd(const void* __restrict__ x, int x_bf16,
                                                                const float* __restrict__ emb, long long B, int T,
                                                                int D, void* __restrict__ out, int out_bf16,
                                                                int out_stride) {
  extern __shared__ float ix_smem[];
  const int n = T + 1, P = n * (n - 1) / 2, ld = D + 1;
  uint8_t* pi = reinterpret_cast<uint8_t*>(ix_smem + kIxWarps * n * ld);
  uint8_t* pj = pi + P;
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    int i = 1;
    while ((i + 1) * i / 2 <= k) ++i;
    pi[k] = (uint8_t)i;
    pj[k] = (uint8_t)(k - i * (i - 1) / 2);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* z = ix_smem + warp * n * ld;
  for (long long b = (long long)blockIdx.x * kIxWarps + warp; b < B; b += (long long)gridDim.x * kIxWarps) {
    for (int e = lane; e < n * D; e += 32) {
      const int i = e / D, d = e - i * D;
      z[i * ld + d] = i == 0 ? ld_any(x, b * D + d, x_bf16) : emb[(b * T + (i - 1)) * D + d];
    }
    __syncwarp();
    const long long o = b * out_stride;
    for (int d = lane; d < D; d += 32) st_any(out, o + d, z[d], out_bf16);
    for (int k = lane; k < P; k += 32) {
      const float* zi = z + pi[k] * ld;
      const float* zj = z + pj[k] * ld;
      float acc = 0.f;
      for (int d = 0; d < D; ++d) acc = fmaf(zi[d], zj[d], acc);
      st_any(out, o + D + k, acc, out_bf16);
    }
    for (int c = D + P + lane; c < out_stride; c += 32) st_any(out, o + c, 0.f, out_bf16);
    __syncwarp();
  }
}

// smem per warp: z[n][D+1], G[n][n+1]
__global__ void __launch_bounds__(kIxWarps * 32) k_interact_bwd(const void* __restrict__ x, int x_bf16,
                                                                const float* __restrict__ emb,
                                                                const void* __restrict__ gout, int g_bf16,
                                                                long long B, int T, int D, int out_stride,
                                                                void* __restrict__ gx, float* __restrict__ gemb) {
  extern __shared__ float ix_smem[];
  const int n = T + 1, ld = D + 1, lg = n + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* z = ix_smem + warp * (n * ld + n * lg);
  float* G = z + n * ld;
  for (long long b = (long long)blockIdx.x * kIxWarps + warp; b < B; b += (long long)gridDim.x * kIxWarps) {
    for (int e = lane; e < n * D; e += 32) {
      const int i = e / D, d = e - i * D;
      z[i * ld + d] = i == 0 ? ld_any(x, b * D + d, x_bf16) : emb[(b * T + (i - 1)) * D + d];
    }
    const long long o = b * out_stride;
    for (int e = lane; e < n * n; e += 32) {
      const int i = e / n, j = e - i * n;
      float g = 0.f;
      if (i > j) g = ld_any(gout, o + D + i * (i - 1) / 2 + j, g_bf16);
      else if (j > i) g = ld_any(gout, o + D + j * (j - 1) / 2 + i, g_bf16);
      G[i * lg + j] = g;
    }
    __syncwarp();
    for (int e = lane; e < n * D; e += 32) {
      const int i = e / D, d = e - i * D;
      float acc = 0.f;
      for (int j = 0; j < n; ++j) acc = fmaf(G[i * lg + j], z[j * ld + d], acc);
      if (i == 0) st_any(gx, b * D + d, acc + ld_any(gout, o + d, g_bf16), x_bf16);
      else gemb[(b * T + (i - 1)) * D + d] = acc;
    }
    __syncwarp();
  }
}

static size_t fwd_smem(int T, int D) {
  const int n = T + 1;
  return sizeof(float) * kIxWarps * n * (D + 1) + 2 * (size_t)(n * (n - 1) / 2) + 16;
}

static size_t bwd_smem(int T, int D) {
  const int n = T + 1;
  return sizeof(float) * kIxWarps * (n * (D + 1) + n * (n + 1));
}

static int check_shape(long long B, int T, int D, int out_stride) {
  if (B < 0 || T < 1 || T > 127 || D < 1 || D > 256) return BP_ERR_INVALID;
  const int n = T + 1;
  if (out_stride < D + n * (n - 1) / 2) return BP_ERR_INVALID;
  if (bwd_smem(T, D) > (200u << 10)) return BP_ERR_INVALID;
  return BP_OK;
}

}  // namespace bp

extern "C" int bp_dlrm_interact_forward(const void* d_x, int32_t x_bf16, const float* d_emb, int64_t B, int32_t T,
                                        int32_t D, void* d_out, int32_t out_bf16, int32_t out_stride,
                                        bp_stream_t stream) {
  using namespace bp;
  const int rc = check_shape(B, T, D, out_stride);
  if (rc != BP_OK) return rc;
  if (B == 0) return BP_OK;
  const size_t smem = fwd_smem(T, D);
  BP_CUDA_TRY(cudaFuncSetAttribute(k_interact_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long long blocks = std::min<long long>((B + kIxWarps - 1) / kIxWarps, (long long)kNumSMs * 16);
  k_interact_fwd<<<(unsigned)blocks, kIxWarps * 32, smem, (cudaStream_t)stream>>>(d_x, x_bf16, d_emb, B, T, D, d_out,
                                                                                  out_bf16, out_stride);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_dlrm_interact_backward(const void* d_x, int32_t x_bf16, const float* d_emb, const void* d_gout,
                                         int32_t g_bf16, int64_t B, int32_t T, int32_t D, int32_t out_stride,
                                         void* d_gx, float* d_gemb, bp_stream_t stream) {
  using namespace bp;
  const int rc = check_shape(B, T, D, out_stride);
  if (rc != BP_OK) return rc;
  if (B == 0) return BP_OK;
  const size_t smem = bwd_smem(T, D);
  BP_CUDA_TRY(cudaFuncSetAttribute(k_interact_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long long blocks = std::min<long long>((B + kIxWarps - 1) / kIxWarps, (long long)kNumSMs * 16);
  k_interact_bwd<<<(unsigned)blocks, kIxWarps * 32, smem, (cudaStream_t)stream>>>(
      d_x, x_bf16, d_emb, d_gout, g_bf16, B, T, D, out_stride, d_gx, d_gemb);
  BP_LAUNCH_CHECK();
  return BP_OK;
}
