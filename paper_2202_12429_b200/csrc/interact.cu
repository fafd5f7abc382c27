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
                                                                void* __restrict__ gx, float* __restrict__ gemb,
                                                                const uint32_t* __restrict__ gemb_rows) {
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
      else gemb[(gemb_rows ? (long long)gemb_rows[b * T + (i - 1)] : b * T + (i - 1)) * D + d] = acc;
    }
    __syncwarp();
  }
}

// Fast path (n = T+1 <= 32, D in {4, 8, 16, 32}), a warp per sample.
//   forward: lane i owns z_i in registers and walks j < i over shared-memory
//   rows read as float4 broadcasts (every lane reads the same z_j: no bank
//   conflicts); the output row is staged in shared memory and written
//   coalesced.  (A balanced variant -- lanes taking pairs round-robin,
//   both rows from shared memory -- measured slower, 37 vs 30 us: twice the
//   shared-memory traffic and no broadcasts.)
//   backward: the next sample's inputs are loaded into registers while the
//   current one is computed (each warp walks ~4 samples); G (symmetric pair
//   gradients, odd row stride, pairs k -> (i, j) from a per-block table) and
//   z staged, lane i computes dz_i = sum_j G_ij z_j (z_j float4 broadcasts).
constexpr int kIxBlocksPerSM = 4;
// k_interact_bwd_reg: resident CTAs per SM (launch bounds and grid).  D = 16
// takes 91 registers: 2 CTAs; a 3-CTA cap (80 registers) spilled and measured
// slower (46 vs 43 us at the Criteo-Kaggle shape, tools/ix_bench.py)
constexpr int ix_bwd_bps(int D) { return D >= 32 ? 1 : 2; }

// pair k = (i, j), i > j: both G offsets, i*LG + j (low half) and j*LG + i
// (high half), so the scatter needs no index arithmetic
__device__ __forceinline__ void build_pairs(uint32_t* pij, int P, int LG) {
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    int i = 1;
    while ((i + 1) * i / 2 <= k) ++i;
    const int j = k - i * (i - 1) / 2;
    pij[k] = (uint32_t)(i * LG + j) | ((uint32_t)(j * LG + i) << 16);
  }
}

// raw 32-bit image of element i (bf16 bits zero-extended, or the fp32 bits):
// the prefetch keeps loads unconsumed until the next sample is computed (a
// conversion at load time stalled the warp on the load right away)
__device__ __forceinline__ uint32_t ld_raw(const void* p, long long i, int bf16) {
  return bf16 ? (uint32_t)reinterpret_cast<const uint16_t*>(p)[i] : reinterpret_cast<const uint32_t*>(p)[i];
}

__device__ __forceinline__ float raw_f(uint32_t r, int bf16) { return __uint_as_float(bf16 ? r << 16 : r); }

template <int D>
__global__ void __launch_bounds__(kIxWarps * 32) k_interact_fwd_reg(const void* __restrict__ x, int x_bf16,
                                                                    const float* __restrict__ emb, long long B,
                                                                    int T, void* __restrict__ out, int out_bf16,
                                                                    int out_stride) {
  extern __shared__ float ix_smem[];
  const int n = T + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* z = ix_smem + warp * (32 * D + ((out_stride + 3) & ~3));  // [n][D] then the staged output row
  float* o = z + 32 * D;
  for (long long b = (long long)blockIdx.x * kIxWarps + warp; b < B; b += (long long)gridDim.x * kIxWarps) {
    for (int e = lane; e < n * D; e += 32)
      z[e] = e < D ? ld_any(x, b * D + e, x_bf16) : emb[b * T * D + (e - D)];
    __syncwarp();
    if (lane < n) {
      float zi[D];
#pragma unroll
      for (int d = 0; d < D; d += 4) {
        const float4 v = *reinterpret_cast<const float4*>(z + lane * D + d);
        zi[d] = v.x; zi[d + 1] = v.y; zi[d + 2] = v.z; zi[d + 3] = v.w;
      }
      if (lane == 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) o[d] = zi[d];
      }
      float* orow = o + D + lane * (lane - 1) / 2;
      for (int j = 0; j < lane; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int d = 0; d < D; d += 4) {
          const float4 v = *reinterpret_cast<const float4*>(z + j * D + d);
          acc = fmaf(zi[d], v.x, acc);
          acc = fmaf(zi[d + 1], v.y, acc);
          acc = fmaf(zi[d + 2], v.z, acc);
          acc = fmaf(zi[d + 3], v.w, acc);
        }
        orow[j] = acc;
      }
    }
    const int P = n * (n - 1) / 2;
    for (int c = D + P + lane; c < out_stride; c += 32) o[c] = 0.f;
    __syncwarp();
    const long long ob = b * out_stride;
    if (out_bf16 && (out_stride & 1) == 0) {
      __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(out) + ob;
      for (int c = 2 * lane; c < out_stride; c += 64) {
        if (c + 1 < out_stride) {
          *reinterpret_cast<__nv_bfloat162*>(op + c) = __floats2bfloat162_rn(o[c], o[c + 1]);
        } else {
          op[c] = __float2bfloat16_rn(o[c]);
        }
      }
    } else {
      for (int c = lane; c < out_stride; c += 32) st_any(out, ob + c, o[c], out_bf16);
    }
    __syncwarp();
  }
}

template <int D>
__global__ void __launch_bounds__(kIxWarps * 32, ix_bwd_bps(D)) k_interact_bwd_reg(const void* __restrict__ x, int x_bf16,
                                                                    const float* __restrict__ emb,
                                                                    const void* __restrict__ gout, int g_bf16,
                                                                    long long B, int T, int out_stride,
                                                                    void* __restrict__ gx, float* __restrict__ gemb,
                                                                    const uint32_t* __restrict__ gemb_rows) {
  extern __shared__ float ix_smem[];
  constexpr int LG = 33;  // G row stride (odd)
  constexpr int GR = 16;  // pairs per lane (P <= 496)
  const int n = T + 1, P = n * (n - 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* z = ix_smem + warp * (32 * D + 32 * LG);
  float* G = z + 32 * D;
  uint32_t* pij = reinterpret_cast<uint32_t*>(ix_smem + kIxWarps * (32 * D + 32 * LG));
  build_pairs(pij, P, LG);
  __syncthreads();
  const uint32_t* emb_u = reinterpret_cast<const uint32_t*>(emb);
  uint32_t zr[D], gr[GR], go = 0u;
  long long dr = 0;
  const long long stride = (long long)gridDim.x * kIxWarps;
  long long b = (long long)blockIdx.x * kIxWarps + warp;
  auto load = [&](long long bb) {
    const long long ob = bb * out_stride;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      const int e = lane + 32 * r;
      zr[r] = e < n * D ? (e < D ? ld_raw(x, bb * D + e, x_bf16) : emb_u[bb * T * D + (e - D)]) : 0u;
    }
#pragma unroll
    for (int r = 0; r < GR; ++r) {
      const int k = lane + 32 * r;
      gr[r] = k < P ? ld_raw(gout, ob + D + k, g_bf16) : 0u;
    }
    go = lane < D ? ld_raw(gout, ob + lane, g_bf16) : 0u;  // gx = gout[:, :D] + dz_0
    const long long p = bb * T + (lane - 1);                  // this lane's embedding-gradient row
    dr = (gemb_rows && lane >= 1 && lane < n) ? (long long)gemb_rows[p] : p;
  };
  if (b < B) load(b);
  for (; b < B; b += stride) {
#pragma unroll
    for (int r = 0; r < D; ++r) {
      const int e = lane + 32 * r;
      if (e < n * D) z[e] = raw_f(zr[r], e < D ? x_bf16 : 0);
    }
    if (lane < n) G[lane * LG + lane] = 0.f;
#pragma unroll
    for (int r = 0; r < GR; ++r) {
      const int k = lane + 32 * r;
      if (k < P) {
        const uint32_t e = pij[k];
        const float gv = raw_f(gr[r], g_bf16);
        G[e & 0xFFFFu] = gv;
        G[e >> 16] = gv;
      }
    }
    const float go_cur = raw_f(go, g_bf16);
    const long long drow = dr;
    __syncwarp();
    if (b + stride < B) load(b + stride);  // next sample in flight during this one's math
    float acc[D];
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d] = 0.f;
    if (lane < n) {
      for (int j = 0; j < n; ++j) {
        const float g = G[lane * LG + j];
#pragma unroll
        for (int d = 0; d < D; d += 4) {
          const float4 v = *reinterpret_cast<const float4*>(z + j * D + d);
          acc[d] = fmaf(g, v.x, acc[d]);
          acc[d + 1] = fmaf(g, v.y, acc[d + 1]);
          acc[d + 2] = fmaf(g, v.z, acc[d + 2]);
          acc[d + 3] = fmaf(g, v.w, acc[d + 3]);
        }
      }
    }
    // gx row: lane 0 holds dz_0; gout[:, :D] sits in lanes 0..D-1
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const float gd = __shfl_sync(0xffffffffu, go_cur, d);
      if (lane == 0) st_any(gx, b * D + d, acc[d] + gd, x_bf16);
    }
    if (lane >= 1 && lane < n) {
      float4* dst = reinterpret_cast<float4*>(gemb + drow * D);
#pragma unroll
      for (int d = 0; d < D; d += 4) dst[d / 4] = make_float4(acc[d], acc[d + 1], acc[d + 2], acc[d + 3]);
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
  const long long nblk = std::min<long long>((B + kIxWarps - 1) / kIxWarps, (long long)kNumSMs * 16);
  if (T + 1 <= 32 && (D == 4 || D == 8 || D == 16 || D == 32)) {
    const size_t sm = sizeof(float) * kIxWarps * (32 * D + ((out_stride + 3) & ~3));
#define BP_IX_FWD(DD)                                                                                              \
  {                                                                                                                \
    BP_CUDA_TRY(cudaFuncSetAttribute(k_interact_fwd_reg<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    k_interact_fwd_reg<DD><<<(unsigned)nblk, kIxWarps * 32, sm, (cudaStream_t)stream>>>(d_x, x_bf16, d_emb, B, T,    \
                                                                                        d_out, out_bf16, out_stride); \
  }
    switch (D) {
      case 4: BP_IX_FWD(4); break;
      case 8: BP_IX_FWD(8); break;
      case 16: BP_IX_FWD(16); break;
      default: BP_IX_FWD(32); break;
    }
#undef BP_IX_FWD
    BP_LAUNCH_CHECK();
    return BP_OK;
  }
  const size_t smem = fwd_smem(T, D);
  BP_CUDA_TRY(cudaFuncSetAttribute(k_interact_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long long blocks = std::min<long long>((B + kIxWarps - 1) / kIxWarps, (long long)kNumSMs * 16);
  k_interact_fwd<<<(unsigned)blocks, kIxWarps * 32, smem, (cudaStream_t)stream>>>(d_x, x_bf16, d_emb, B, T, D, d_out,
                                                                                  out_bf16, out_stride);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_dlrm_interact_backward_rows(const void* d_x, int32_t x_bf16, const float* d_emb,
                                              const void* d_gout, int32_t g_bf16, int64_t B, int32_t T, int32_t D,
                                              int32_t out_stride, void* d_gx, float* d_gemb,
                                              const uint32_t* d_gemb_rows, bp_stream_t stream);

extern "C" int bp_dlrm_interact_backward(const void* d_x, int32_t x_bf16, const float* d_emb, const void* d_gout,
                                         int32_t g_bf16, int64_t B, int32_t T, int32_t D, int32_t out_stride,
                                         void* d_gx, float* d_gemb, bp_stream_t stream) {
  return bp_dlrm_interact_backward_rows(d_x, x_bf16, d_emb, d_gout, g_bf16, B, T, D, out_stride, d_gx, d_gemb,
                                        nullptr, stream);
}

// d_gemb_rows (optional): embedding-gradient row of (b, t) = d_gemb_rows[b*T + t]
// instead of b*T + t -- the EmbeddingBag's key-sorted order (bp_prep_occ_rank),
// so bp_embbag_backward_sorted streams it.
extern "C" int bp_dlrm_interact_backward_rows(const void* d_x, int32_t x_bf16, const float* d_emb,
                                              const void* d_gout, int32_t g_bf16, int64_t B, int32_t T, int32_t D,
                                              int32_t out_stride, void* d_gx, float* d_gemb,
                                              const uint32_t* d_gemb_rows, bp_stream_t stream) {
  using namespace bp;
  const int rc = check_shape(B, T, D, out_stride);
  if (rc != BP_OK) return rc;
  if (B == 0) return BP_OK;
  const long long nblk = std::min<long long>((B + kIxWarps - 1) / kIxWarps, (long long)kNumSMs * ix_bwd_bps(D));
  if (T + 1 <= 32 && (D == 4 || D == 8 || D == 16 || D == 32)) {
    const size_t sm = sizeof(float) * kIxWarps * (32 * D + 32 * 33) + sizeof(uint32_t) * 512;
#define BP_IX_BWD(DD)                                                                                              \
  {                                                                                                                \
    BP_CUDA_TRY(cudaFuncSetAttribute(k_interact_bwd_reg<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    BP_CUDA_TRY(cudaFuncSetAttribute(k_interact_bwd_reg<DD>, cudaFuncAttributePreferredSharedMemoryCarveout,         \
                                     cudaSharedmemCarveoutMaxShared));                                                 \
    k_interact_bwd_reg<DD><<<(unsigned)nblk, kIxWarps * 32, sm, (cudaStream_t)stream>>>(                          \
        d_x, x_bf16, d_emb, d_gout, g_bf16, B, T, out_stride, d_gx, d_gemb, d_gemb_rows);                                         \
  }
    switch (D) {
      case 4: BP_IX_BWD(4); break;
      case 8: BP_IX_BWD(8); break;
      case 16: BP_IX_BWD(16); break;
      default: BP_IX_BWD(32); break;
    }
#undef BP_IX_BWD
    BP_LAUNCH_CHECK();
    return BP_OK;
  }
  const size_t smem = bwd_smem(T, D);
  BP_CUDA_TRY(cudaFuncSetAttribute(k_interact_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long long blocks = std::min<long long>((B + kIxWarps - 1) / kIxWarps, (long long)kNumSMs * 16);
  k_interact_bwd<<<(unsigned)blocks, kIxWarps * 32, smem, (cudaStream_t)stream>>>(
      d_x, x_bf16, d_emb, d_gout, g_bf16, B, T, D, out_stride, d_gx, d_gemb, d_gemb_rows);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

// Mixed-precision SGD of the dense MLPs in one launch (DLRM mode, bf16
// compute copy): for every tensor k, master_k -= lr * float(grad_k) (fp32),
// then lowp_k = bf16(master_k) -- replaces ~2 x (#tensors) eager kernels per
// step.  The tensor table travels by value in the kernel parameters, so the
// launch is CUDA-graph capturable.
namespace bp {

struct SgdTable {
  int n;
  float lr;
  float* master[BP_SGD_MAX_TENSORS];
  __nv_bfloat16* lowp[BP_SGD_MAX_TENSORS];
  const __nv_bfloat16* grad[BP_SGD_MAX_TENSORS];
  long long end[BP_SGD_MAX_TENSORS];  // inclusive prefix sums of the sizes
};

__global__ void __launch_bounds__(256) k_master_sgd(const SgdTable t) {
  const long long total = t.end[t.n - 1];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int k = 0;
    while (i >= t.end[k]) ++k;
    const long long j = i - (k ? t.end[k - 1] : 0);
    const float m = __fsub_rn(t.master[k][j], __fmul_rn(t.lr, __bfloat162float(t.grad[k][j])));
    t.master[k][j] = m;
    t.lowp[k][j] = __float2bfloat16_rn(m);
  }
}

}  // namespace bp

extern "C" int bp_dlrm_master_sgd(const bp_sgd_tensors* tensors, float lr, bp_stream_t stream) {
  using namespace bp;
  if (!tensors || tensors->n < 1 || tensors->n > BP_SGD_MAX_TENSORS) return BP_ERR_INVALID;
  SgdTable t;
  t.n = tensors->n;
  t.lr = lr;
  long long acc = 0;
  for (int k = 0; k < t.n; ++k) {
    if (tensors->numel[k] < 0) return BP_ERR_INVALID;
    t.master[k] = tensors->master[k];
    t.lowp[k] = reinterpret_cast<__nv_bfloat16*>(tensors->lowp[k]);
    t.grad[k] = reinterpret_cast<const __nv_bfloat16*>(tensors->grad[k]);
    acc += tensors->numel[k];
    t.end[k] = acc;
  }
  if (acc == 0) return BP_OK;
  k_master_sgd<<<grid_for(acc, 256, kNumSMs * 8), 256, 0, (cudaStream_t)stream>>>(t);
  BP_LAUNCH_CHECK();
  return BP_OK;
}
