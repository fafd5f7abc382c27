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
constexpr int kScanIpt = 4;
constexpr int kScanTile = kScanThreads * kScanIpt;  // 1024

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

// Single-pass exclusive scan with decoupled look-back.  Each CTA scans a
// 4096-element tile (16 consecutive elements per thread, vector loads),
// publishes its aggregate, then thread 0 walks back over predecessor tiles
// until it meets an inclusive prefix.  Tile status words pack
// (epoch:30 | flag:2 | value:32), so the state array never needs clearing:
// entries from earlier calls carry another epoch and read as "not ready".
constexpr unsigned long long kFlagAgg = 1ull, kFlagPrefix = 2ull;

__device__ __forceinline__ unsigned long long scan_pack(uint32_t epoch, unsigned long long flag, uint32_t v) {
  return ((unsigned long long)(epoch & 0x3FFFFFFFu) << 34) | (flag << 32) | v;
}

static __global__ void __launch_bounds__(kScanThreads) k_scan_onepass(const uint32_t* in, uint32_t* out, long long n,
                                                                      const long long* d_n,
                                                                      unsigned long long* state, uint32_t epoch,
                                                                      uint32_t* total, long long* total64) {
  n = load_count(n, d_n);
  const long long tile = blockIdx.x;
  const long long base = tile * kScanTile;
  if (base >= n && tile > 0) return;
  __shared__ uint32_t sh_warp[kScanThreads / 32];
  __shared__ uint32_t sh_prefix;
  const long long i0 = base + (long long)threadIdx.x * kScanIpt;
  uint32_t v[kScanIpt];
  if (i0 + kScanIpt <= n && ((reinterpret_cast<uintptr_t>(in + i0) & 15) == 0)) {
    const uint4* p = reinterpret_cast<const uint4*>(in + i0);
#pragma unroll
    for (int q = 0; q < kScanIpt / 4; ++q) {
      const uint4 w = p[q];
      v[4 * q] = w.x;
      v[4 * q + 1] = w.y;
      v[4 * q + 2] = w.z;
      v[4 * q + 3] = w.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kScanIpt; ++q) v[q] = i0 + q < n ? in[i0 + q] : 0u;
  }
  uint32_t run = 0;
#pragma unroll
  for (int q = 0; q < kScanIpt; ++q) {
    const uint32_t x = v[q];
    v[q] = run;  // exclusive within the thread
    run += x;
  }
  uint32_t block_total;
  const uint32_t thread_excl = block_inclusive_scan_256(run, sh_warp, &block_total) - run;
  if (threadIdx.x < 32) {
    // Warp-parallel look-back: lane l inspects tile (j - l); the nearest
    // tile holding an inclusive prefix ends the walk, and the aggregates of
    // the tiles in front of it are summed in one warp reduction.
    volatile unsigned long long* st = state;
    const unsigned lane = threadIdx.x;
    const uint32_t ep = epoch & 0x3FFFFFFFu;
    uint32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) st[0] = scan_pack(epoch, kFlagPrefix, block_total);
    } else {
      if (lane == 0) st[tile] = scan_pack(epoch, kFlagAgg, block_total);
      for (long long j = tile - 1;; j -= 32) {
        const long long idx = j - (long long)lane;
        unsigned long long w = 0;
        if (idx >= 0) {
          do {
            w = st[idx];
          } while ((uint32_t)(w >> 34) != ep || ((w >> 32) & 3ull) == 0);
        }
        const unsigned pm = __ballot_sync(0xffffffffu, idx >= 0 && ((w >> 32) & 3ull) == kFlagPrefix);
        const unsigned stop = pm ? (unsigned)(__ffs(pm) - 1) : 31u;
        uint32_t v = (idx >= 0 && lane <= stop) ? (uint32_t)w : 0u;
        prefix += warp_sum(v);
        if (pm || j - 32 < 0) break;
      }
      if (lane == 0) st[tile] = scan_pack(epoch, kFlagPrefix, prefix + block_total);
    }
    if (lane == 0) {
      sh_prefix = prefix;
      if (base + kScanTile >= n) {
        if (total) *total = prefix + block_total;
        if (total64) *total64 = (long long)(prefix + block_total);
      }
    }
  }
  __syncthreads();
  const uint32_t add = sh_prefix + thread_excl;
  if (i0 + kScanIpt <= n && ((reinterpret_cast<uintptr_t>(out + i0) & 15) == 0)) {
    uint4* p = reinterpret_cast<uint4*>(out + i0);
#pragma unroll
    for (int q = 0; q < kScanIpt / 4; ++q)
      p[q] = make_uint4(v[4 * q] + add, v[4 * q + 1] + add, v[4 * q + 2] + add, v[4 * q + 3] + add);
  } else {
#pragma unroll
    for (int q = 0; q < kScanIpt; ++q)
      if (i0 + q < n) out[i0 + q] = v[q] + add;
  }
}

// Decoupled look-back for one tile, run by ONE full warp: publishes the
// tile's aggregate, walks back over its predecessors (lane l inspects tile
// j - l) until an inclusive prefix, publishes its own inclusive prefix and
// returns the exclusive prefix on every lane.  Same epoch-tagged status
// words as k_scan_onepass (the state needs no clearing between calls that
// use distinct epochs, only once after allocation).
// Status words sit kLookbackStride words apart (one 128-byte line each): the
// pollers of a tile then never queue on a line shared with other tiles.
constexpr int kLookbackStride = 16;

__device__ __forceinline__ uint32_t warp_lookback(unsigned long long* state, long long tile, uint32_t epoch,
                                                  uint32_t agg) {
  struct Strided {
    volatile unsigned long long* p;
    __device__ volatile unsigned long long& operator[](long long i) const { return p[i * kLookbackStride]; }
  } st{state};
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t ep = epoch & 0x3FFFFFFFu;
  if (tile == 0) {
    if (lane == 0) st[0] = scan_pack(epoch, kFlagPrefix, agg);
    return 0;
  }
  if (lane == 0) st[tile] = scan_pack(epoch, kFlagAgg, agg);
  uint32_t prefix = 0;
  for (long long j = tile - 1;; j -= 32) {
    const long long idx = j - (long long)lane;
    unsigned long long w = 0;
    if (idx >= 0) {
      do {
        w = st[idx];
      } while ((uint32_t)(w >> 34) != ep || ((w >> 32) & 3ull) == 0);
    }
    const unsigned pm = __ballot_sync(0xffffffffu, idx >= 0 && ((w >> 32) & 3ull) == kFlagPrefix);
    const unsigned stop = pm ? (unsigned)(__ffs(pm) - 1) : 31u;
    const uint32_t v = (idx >= 0 && lane <= stop) ? (uint32_t)w : 0u;
    prefix += warp_sum(v);
    if (pm || j - 32 < 0) break;
  }
  if (lane == 0) st[tile] = scan_pack(epoch, kFlagPrefix, prefix + agg);
  return prefix;
}

inline int scan_tiles(long long n) { return (int)((n + kScanTile - 1) / kScanTile); }
// u32 words of tile state an exclusive_scan over n elements needs.
inline long long scan_state_words(long long n) { return 2ll * (scan_tiles(n > 0 ? n : 1) + 1); }

inline uint32_t next_scan_epoch() {
  static unsigned int counter = 0;
  return __atomic_add_fetch(&counter, 1u, __ATOMIC_RELAXED);
}

// Exclusive scan; *d_total (u32) and *d_total64 receive the sum.  in and out
// may alias.  ``state`` needs scan_state_words(n_max) u32 (8-byte aligned).
inline cudaError_t exclusive_scan(const uint32_t* in, uint32_t* out, long long n_max, const long long* d_n,
                                  uint32_t* state, uint32_t* d_total, long long* d_total64, cudaStream_t s) {
  const int tiles = scan_tiles(n_max > 0 ? n_max : 1);
  unsigned long long* st = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(state) + 7) & ~uintptr_t(7));
  // Epoch tags already separate calls; clearing the (tiny) state as well
  // rules out a recycled pool buffer whose garbage happens to match an epoch.
  cudaError_t e = cudaMemsetAsync(st, 0, sizeof(unsigned long long) * tiles, s);
  if (e != cudaSuccess) return e;
  k_scan_onepass<<<tiles, kScanThreads, 0, s>>>(in, out, n_max, d_n, st, next_scan_epoch(), d_total, d_total64);
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

inline size_t sort_partials_words(long long n) { return (size_t)scan_state_words((long long)sort_hist_words(n)); }

inline int bit_width_u64(unsigned long long x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

}  // namespace bp
