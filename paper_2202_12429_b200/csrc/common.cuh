// Shared device helpers for the BagPipe embedding-access path (sm_100a).
//
// Hash primitives are bit-exact restatements of reference hashing.py:24-79
// (FNV-1a 64 over little-endian u64 words, splitmix64, top-53-bit unit) and
// the store's functional initialisation of reference store.py:29-42, which
// computes in float64 and rounds once to float32.  All float arithmetic that
// must match numpy uses explicit round-to-nearest intrinsics so nvcc cannot
// contract a multiply-add into an FMA.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/bagpipe_b200.h"

namespace bp {

constexpr uint64_t kFnvOffset = 0xCBF29CE484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001B3ull;
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;
constexpr int kKeyTableShift = 44;
constexpr uint64_t kRowMask = (1ull << kKeyTableShift) - 1;
constexpr int kNumSMs = 148;

__host__ __device__ __forceinline__ uint64_t fnv_u64(uint64_t h, uint64_t v) {
#pragma unroll
  for (int s = 0; s < 64; s += 8) h = (h ^ ((v >> s) & 0xFFull)) * kFnvPrime;
  return h;
}

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + kGamma;
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}

// Component j of key (t, r): float32(-0.05 + 0.1 * unit(splitmix(seed ^ fnv(t, r, j)))),
// the product and sum in float64 exactly as numpy evaluates them.
__device__ __forceinline__ float init_component(uint64_t seed, uint64_t h_tr, uint64_t j) {
  const uint64_t m = splitmix64(seed ^ fnv_u64(h_tr, j));
  const double unit = (double)(m >> 11) * 0x1.0p-53;
  return __double2float_rn(__dadd_rn(-0.05, __dmul_rn(0.1, unit)));
}

__device__ __forceinline__ uint32_t table_of(uint64_t key) { return (uint32_t)(key >> kKeyTableShift); }
__device__ __forceinline__ uint64_t row_of(uint64_t key) { return key & kRowMask; }

// Device-side error record shared by every object of one context.  The first
// error in (iteration, index) order wins, mirroring the reference raising at
// the first failing key of the first failing call.
// Layout mirrors bp_error_t in include/bagpipe_b200.h.
struct ErrorRecord {
  int code;  // 0 = no error
  int lock;
  long long iteration;
  long long index;
  unsigned long long key;
};

// Error path only: a short critical section keeps (code, iteration, index,
// key) consistent; the fast pre-check avoids the lock once an earlier error
// is recorded.
static __device__ __noinline__ void raise_error(ErrorRecord* err, int code, long long iteration, long long index,
                                         uint64_t key) {
  if (err == nullptr) return;
  volatile ErrorRecord* v = err;
  if (v->code != 0 && (v->iteration < iteration || (v->iteration == iteration && v->index <= index))) return;
  while (atomicCAS(&err->lock, 0, 1) != 0) {
  }
  __threadfence();
  if (v->code == 0 || iteration < v->iteration || (iteration == v->iteration && index < v->index)) {
    v->iteration = iteration;
    v->index = index;
    v->key = key;
    v->code = code;
  }
  __threadfence();
  atomicExch(&err->lock, 0);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// CTA-aggregated atomicAdd: every thread of the CTA must call it (it holds
// two barriers); one global atomic per CTA.  Same-address atomics serialise
// in the L2's atomic unit (~0.65 ns each on B200: tools/mb/atomic_probe.cu),
// so one per warp of a 1,664-CTA grid alone costs ~9 us.
__device__ __forceinline__ void cta_add(unsigned long long* ctr, unsigned long long v) {
  __shared__ unsigned long long s_acc;
  if (threadIdx.x == 0) s_acc = 0;
  __syncthreads();
  v = warp_sum(v);
  if (lane_id() == 0 && v) atomicAdd(&s_acc, v);
  __syncthreads();
  if (threadIdx.x == 0 && s_acc) atomicAdd(ctr, s_acc);
}

// Warp-aggregated atomicAdd of a predicate count.
__device__ __forceinline__ void warp_count_add(unsigned long long* ctr, bool pred) {
  const unsigned mask = __ballot_sync(0xffffffffu, pred);
  if (lane_id() == 0 && mask) atomicAdd(ctr, (unsigned long long)__popc(mask));
}

inline int grid_for(long long n, int threads, int max_blocks = kNumSMs * 16) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

}  // namespace bp

#define BP_CUDA_TRY(expr)                                                     \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      bp_set_last_error(cudaGetErrorString(_e), __FILE__, __LINE__);          \
      return _e == cudaErrorMemoryAllocation ? BP_ERR_OOM : BP_ERR_CUDA;      \
    }                                                                         \
  } while (0)

#define BP_LAUNCH_CHECK() BP_CUDA_TRY(cudaGetLastError())

void bp_set_last_error(const char* msg, const char* file, int line);
