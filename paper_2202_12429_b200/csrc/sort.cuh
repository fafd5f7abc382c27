// Device-wide primitives used by the batch prep, planner and cache:
//  * exclusive scan of u32 flags/counts (reduce -> scan partials -> downsweep)
//  * stable LSD radix sort of (key, u32 value) pairs, 9-bit digits, with
//    warp-level __match_any_sync ranking so Zipf-hot keys (thousands of equal
//    digits per tile) cost one shared-memory update per warp round instead of
//    one atomic per element.
//
// Element counts may live in device memory (``d_n``): kernels are launched
// for the host-known upper bound and read the true count on the device, so
// producers and consumers chain on a stream without a host round trip.
#pragma once

#include "common.cuh"

namespace bp {

constexpr int kScanThreads = 256;
constexpr int kScanIpt = 16;
constexpr int kScanTile = kScanThreads * kScanIpt;  // 4096

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortIpt = 16;
constexpr int kSortTile = kSortThreads * kSortIpt;  // 4096 elements per CTA
constexpr int kSortWarpTile = 32 * kSortIpt;         // 512 elements per warp
constexpr int kSortMaxBits = 9;
constexpr int kSortMaxRadix = 1 << kSortMaxBits;

__device__ __forceinline__ long long load_count(long long n, const long long* d_n) {
  return d_n ? (*d_n < n ? *d_n : n) : n;
}

// Inclusive block scan for 256 threads; returns inclusive value, writes block total.
__device__ __forceinline__ uint32_t block_inclusive_scan_256(uint32_t v, uint32_t* sh_warp, uint32_t* total) {
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (unsigned)o) v += t;
  }
  if (lane == 31) sh_warp[warp] = v;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (kScanThreads / 32) ? sh_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= (unsigned)o) w += t;
    }
    if (lane < (kScanThreads / 32)) sh_warp[lane] = w;
  }
  __syncthreads();
  const uint32_t add = warp ? sh_warp[warp - 1] : 0;
  *total = sh_warp[kScanThreads / 32 - 1];
  __syncthreads();
  return v + add;
}

static __global__ void k_scan_reduce(const uint32_t* __restrict__ in, long long n, const long long* d_n,
                              uint32_t* __restrict__ partials) {
  n = load_count(n, d_n);
  const long long base = (long long)blockIdx.x * kScanTile;
  uint32_t s = 0;
#pragma unroll 4
  for (int r = 0; r < kScanIpt; ++r) {
    const long long i = base + r * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  s = warp_sum(s);
  __shared__ uint32_t sh[kScanThreads / 32];
  if (lane_id() == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += sh[w];
    partials[blockIdx.x] = t;
  }
}

// Single CTA: exclusive scan of ``tiles`` partials in place; writes the grand
// total to *total (u32) and optionally *total64.
static __global__ void k_scan_partials(uint32_t* partials, int tiles, uint32_t* total, long long* total64) {
  __shared__ uint32_t sh[kScanThreads / 32];
  uint32_t carry = 0;
  for (int base = 0; base < tiles; base += kScanThreads) {
    const int i = base + threadIdx.x;
    const uint32_t v = i < tiles ? partials[i] : 0;
    uint32_t tot;
    const uint32_t inc = block_inclusive_scan_256(v, sh, &tot);
    if (i < tiles) partials[i] = carry + inc - v;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    if (total) *total = carry;
    if (total64) *total64 = (long long)carry;
  }
}

static __global__ void k_scan_down(const uint32_t* __restrict__ in, long long n, const long long* d_n,
                            const uint32_t* __restrict__ partials, uint32_t* __restrict__ out) {
  n = load_count(n, d_n);
  __shared__ uint32_t sh[kScanThreads / 32];
  const long long base = (long long)blockIdx.x * kScanTile;
  if (base >= n) return;  // whole CTA exits together
  uint32_t carry = partials[blockIdx.x];
  for (int r = 0; r < kScanIpt; ++r) {
    const long long i = base + r * kScanThreads + threadIdx.x;
    const uint32_t v = i < n ? in[i] : 0;
    uint32_t tot;
    const uint32_t inc = block_inclusive_scan_256(v, sh, &tot);
    if (i < n) out[i] = carry + inc - v;
    carry += tot;
  }
}

struct ScanTemp {
  uint32_t* partials;  // >= tiles_for(n_max)
};

inline int scan_tiles(long long n) { return (int)((n + kScanTile - 1) / kScanTile); }

// Exclusive scan; *d_total (u32) and *d_total64 receive the sum.  in and out may alias.
inline cudaError_t exclusive_scan(const uint32_t* in, uint32_t* out, long long n_max, const long long* d_n,
                                  uint32_t* partials, uint32_t* d_total, long long* d_total64,
                                  cudaStream_t s) {
  const int tiles = scan_tiles(n_max > 0 ? n_max : 1);
  k_scan_reduce<<<tiles, kScanThreads, 0, s>>>(in, n_max, d_n, partials);
  k_scan_partials<<<1, kScanThreads, 0, s>>>(partials, tiles, d_total, d_total64);
  k_scan_down<<<tiles, kScanThreads, 0, s>>>(in, n_max, d_n, partials, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- radix sort

template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_radix_upsweep(const K* __restrict__ keys, long long n,
                                                                const long long* d_n, int shift, int bits,
                                                                uint32_t* __restrict__ hist, int tiles) {
  n = load_count(n, d_n);
  __shared__ uint32_t cnt[kSortMaxRadix];
  const int radix = 1 << bits;
  for (int i = threadIdx.x; i < radix; i += kSortThreads) cnt[i] = 0;
  __syncthreads();
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const long long base = (long long)blockIdx.x * kSortTile + warp * kSortWarpTile;
  const K mask = (K)(radix - 1);
  for (int r = 0; r < kSortIpt; ++r) {
    const long long i = base + r * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = valid ? (uint32_t)((keys[i] >> shift) & mask) : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (valid && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&cnt[d], (uint32_t)__popc(peers));
  }
  __syncthreads();
  for (int d = threadIdx.x; d < radix; d += kSortThreads) hist[(long long)d * tiles + blockIdx.x] = cnt[d];
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_radix_downsweep(const K* __restrict__ keys_in,
                                                                  const uint32_t* __restrict__ vals_in,
                                                                  K* __restrict__ keys_out,
                                                                  uint32_t* __restrict__ vals_out, long long n,
                                                                  const long long* d_n, int shift, int bits,
                                                                  const uint32_t* __restrict__ hist, int tiles) {
  n = load_count(n, d_n);
  __shared__ uint32_t wcnt[kSortWarps][kSortMaxRadix];
  const int radix = 1 << bits;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  for (int i = lane; i < radix; i += 32) wcnt[warp][i] = 0;
  __syncwarp();
  const long long base = (long long)blockIdx.x * kSortTile + warp * kSortWarpTile;
  const K mask = (K)(radix - 1);
  K k[kSortIpt];
  uint32_t v[kSortIpt];
  uint32_t rank[kSortIpt];
#pragma unroll
  for (int r = 0; r < kSortIpt; ++r) {
    const long long i = base + r * 32 + lane;
    const bool valid = i < n;
    k[r] = valid ? keys_in[i] : (K)0;
    v[r] = valid ? vals_in[i] : 0u;
    const uint32_t d = valid ? (uint32_t)((k[r] >> shift) & mask) : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned below = peers & ((1u << lane) - 1u);
    const uint32_t prev = valid ? wcnt[warp][d] : 0u;
    rank[r] = prev + (uint32_t)__popc(below);
    __syncwarp();
    if (valid && below == 0) wcnt[warp][d] = prev + (uint32_t)__popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = threadIdx.x; d < radix; d += kSortThreads) {
    uint32_t run = hist[(long long)d * tiles + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortIpt; ++r) {
    const long long i = base + r * 32 + lane;
    if (i < n) {
      const uint32_t d = (uint32_t)((k[r] >> shift) & mask);
      const uint32_t dst = wcnt[warp][d] + rank[r];
      keys_out[dst] = k[r];
      vals_out[dst] = v[r];
    }
  }
}

inline int sort_tiles(long long n) { return (int)((n + kSortTile - 1) / kSortTile); }
inline size_t sort_hist_words(long long n) { return (size_t)kSortMaxRadix * (size_t)(sort_tiles(n > 0 ? n : 1)); }

// Stable sort of (key, value) pairs on bits [begin_bit, end_bit).  Ping-pongs
// between the a/b buffers; returns in *which the buffer holding the result
// (0 = a, 1 = b).  ``hist`` must hold sort_hist_words(n_max) u32 and
// ``partials`` scan_tiles(sort_hist_words(n_max)) + 1 u32.  The digit-major
// histogram [radix][tiles] is scanned by the multi-CTA exclusive scan.
template <typename K>
cudaError_t radix_sort_pairs(K* keys_a, uint32_t* vals_a, K* keys_b, uint32_t* vals_b, long long n_max,
                             const long long* d_n, int begin_bit, int end_bit, uint32_t* hist, uint32_t* partials,
                             int* which, cudaStream_t s) {
  *which = 0;
  if (n_max <= 0 || end_bit <= begin_bit) return cudaSuccess;
  const int tiles = sort_tiles(n_max);
  K* kin = keys_a;
  uint32_t* vin = vals_a;
  K* kout = keys_b;
  uint32_t* vout = vals_b;
  for (int shift = begin_bit; shift < end_bit; shift += kSortMaxBits) {
    const int bits = (end_bit - shift) < kSortMaxBits ? (end_bit - shift) : kSortMaxBits;
    const long long len = (long long)(1 << bits) * tiles;
    k_radix_upsweep<K><<<tiles, kSortThreads, 0, s>>>(kin, n_max, d_n, shift, bits, hist, tiles);
    cudaError_t e = exclusive_scan(hist, hist, len, nullptr, partials, nullptr, nullptr, s);
    if (e != cudaSuccess) return e;
    k_radix_downsweep<K><<<tiles, kSortThreads, 0, s>>>(kin, vin, kout, vout, n_max, d_n, shift, bits, hist,
                                                         tiles);
    K* tk = kin;
    kin = kout;
    kout = tk;
    uint32_t* tv = vin;
    vin = vout;
    vout = tv;
    *which ^= 1;
  }
  return cudaGetLastError();
}

inline size_t sort_partials_words(long long n) { return (size_t)scan_tiles((long long)sort_hist_words(n)) + 1; }

inline int bit_width_u64(unsigned long long x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

}  // namespace bp
