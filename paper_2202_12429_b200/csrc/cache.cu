// Trainer TTL cache in HBM: reference cache.py:31-286.
//
// Layout (structure of arrays, capacity C slots):
//   slot_of[id]   int32   dense id -> slot (-1 absent); ids are schema ids g
//                         (a direct-mapped "hash map": 4 B per table row,
//                         135 MB at Criteo-Kaggle scale, no probing) or
//                         registry ids for schema-less caches
//   values[C][D]  float32 row arena (64 B rows at D=16, 16-byte aligned)
//   key/id/ttl/dirty/used per slot
//   free[C]       LIFO of free slots; evictions push their slots in
//                 descending order so the lowest freed slot is reused first
//                 (reference cache.py:209-210).
// Eviction scans the ttl/used arrays (C x 9 B) and compacts with a scan, so it
// is exact for any plan, including fault-injected ones.
#include "internal.cuh"

namespace bp {

struct CacheCounters {
  long long occupancy, free_top, insertions, evictions, peak_occupancy, abort;
  unsigned int ticket;  // k_insert: blocks finished (the last one commits the counters)
  unsigned int evict_ticket;  // k_evict_planned: blocks finished
  unsigned long long evict_dirty;  // k_evict_planned: dirty rows so far (reset by the last block)
};

}  // namespace bp

struct bp_cache {
  bp_ctx* ctx;
  const bp_schema* sc;
  long long capacity;
  int dim;
  bp::Registry reg;
  long long id_cap;
  int32_t* d_slot_of;
  uint64_t* d_slot_key;
  uint32_t* d_slot_id;
  long long* d_ttl;
  uint8_t* d_dirty;
  uint8_t* d_used;
  float* d_values;
  uint32_t* d_free;
  bp::CacheCounters* d_ctr;
  bp::CacheCounters* h_ctr;
  uint32_t* d_flag;
  uint32_t* d_pos;
  uint32_t* d_partials;
  long long ids_cap;
  uint32_t* d_ids_tmp;
  int32_t* d_slot_tmp;
};

namespace bp {

__global__ void k_fill_i32(int32_t* p, long long n, int32_t v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_free_init(uint32_t* free_list, long long cap) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cap; i += (long long)gridDim.x * blockDim.x)
    free_list[i] = (uint32_t)(cap - 1 - i);  // pops (from the top) yield 0, 1, 2, ...
}

// One launch: every block checks the capacity against the counters as they
// were at launch (nothing changes them until the last block), inserts its
// share, and the last block to finish commits free_top / occupancy /
// insertions / peak -- all blocks have read the counters by then.
__global__ void k_insert(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ ids,
                         const float* __restrict__ rows, const int64_t* __restrict__ ttls, long long n,
                         const long long* d_n, int dim, CacheCounters* __restrict__ ctr, long long capacity,
                         int32_t* __restrict__ slot_of, uint64_t* __restrict__ slot_key,
                         uint32_t* __restrict__ slot_id, long long* __restrict__ ttl, uint8_t* __restrict__ dirty,
                         uint8_t* __restrict__ used, float* __restrict__ values, const uint32_t* __restrict__ free_list,
                         ErrorRecord* err, long long iteration, long long sub, long long* n_out) {
  // d_n - sub rows (the engine skips a dropped first key this way), written
  // back to n_out for the step counters
  if (d_n) {
    const long long m = *d_n - sub;
    n = m < 0 ? 0 : (m < n ? m : n);
  }
  if (n_out && blockIdx.x == 0 && threadIdx.x == 0) *n_out = n;
  const long long occ = ctr->occupancy, top = ctr->free_top;
  const bool abort = occ + n > capacity;
  if (abort) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_error(err, BP_ERR_CACHE_CAPACITY, iteration, 0, 0);
  } else {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
      const uint32_t id = ids[i];
      if (id == kNoId || slot_of[id] >= 0) {
        raise_error(err, BP_ERR_CACHE_ORDERING, iteration, i, keys[i]);
        continue;
      }
      const uint32_t slot = free_list[top - 1 - i];
      slot_of[id] = (int32_t)slot;
      slot_key[slot] = keys[i];
      slot_id[slot] = id;
      ttl[slot] = ttls[i];
      dirty[slot] = 0;
      used[slot] = 1;
      if ((dim & 3) == 0) {
        const float4* src = reinterpret_cast<const float4*>(rows + i * dim);
        float4* dst = reinterpret_cast<float4*>(values + (long long)slot * dim);
        for (int d = 0; d < (dim >> 2); ++d) dst[d] = src[d];
      } else {
        for (int d = 0; d < dim; ++d) values[(long long)slot * dim + d] = rows[i * dim + d];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctr->ticket, 1u) == gridDim.x - 1) {
      ctr->abort = abort ? 1 : 0;
      if (!abort) {
        ctr->free_top = top - n;
        ctr->occupancy = occ + n;
        ctr->insertions += n;
        if (occ + n > ctr->peak_occupancy) ctr->peak_occupancy = occ + n;
      }
      ctr->ticket = 0;
    }
  }
}

__global__ void k_set_ttl(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ ids,
                          const int64_t* __restrict__ ttls, long long n, const long long* d_n,
                          const int32_t* __restrict__ slot_of, long long* __restrict__ ttl, ErrorRecord* err,
                          long long iteration) {
  n = load_count(n, d_n);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t id = ids[i];
    const int32_t slot = id == kNoId ? -1 : slot_of[id];
    if (slot < 0) raise_error(err, BP_ERR_CACHE_ORDERING, iteration, i, keys[i]);
    else ttl[slot] = ttls[i];
  }
}

__global__ void k_resolve(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ ids, long long n,
                          const long long* d_n, const int32_t* __restrict__ slot_of, int32_t* __restrict__ out,
                          ErrorRecord* err, long long iteration) {
  n = load_count(n, d_n);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t id = ids[i];
    const int32_t slot = id == kNoId ? -1 : slot_of[id];
    if (slot < 0) raise_error(err, BP_ERR_CACHE_MISS, iteration, i, keys[i]);
    out[i] = slot;
  }
}

// Engine fused step of reference engine.py:525-543 for one batch, over its
// key-sorted uniques s: TTL update (apply_ttl_updates) then slot resolution
// (resolve_slots).  Error precedence follows the reference call order: an
// absent key in the TTL list is CacheOrderingError (phase 0) even if a miss
// (phase 1) would come first in key order; indices report first-occurrence
// positions (the order both reference loops walk).
__global__ void k_apply_resolve(const uint32_t* __restrict__ ids_s, const uint64_t* __restrict__ keys_s,
                                const uint32_t* __restrict__ perm_s2k, const int64_t* __restrict__ ttl_k,
                                const long long* d_U, uint64_t skip_key, int has_skip,
                                const int32_t* __restrict__ slot_of, long long* __restrict__ ttl,
                                int32_t* __restrict__ slots_s, ErrorRecord* err, long long iteration) {
  const long long U = *d_U;
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < U; s += (long long)gridDim.x * blockDim.x) {
    const uint32_t id = ids_s[s];
    const uint64_t key = keys_s[s];
    const long long k = perm_s2k[s];
    const int32_t slot = id == kNoId ? -1 : slot_of[id];
    const bool skipped = has_skip && key == skip_key;
    if (slot < 0) {
      raise_error(err, skipped ? BP_ERR_CACHE_MISS : BP_ERR_CACHE_ORDERING, iteration,
                  skipped ? (k | (1ll << 40)) : k, key);
    } else if (!skipped) {
      ttl[slot] = ttl_k[k];
    }
    slots_s[s] = slot;
  }
}

// k_apply_resolve of this batch and the next batch's id stamp (k_mark_ids)
// in one launch: independent work on the same stream, one launch gap less
// on the engine's compute stream.
__global__ void k_apply_resolve_mark(const uint32_t* __restrict__ ids_s, const uint64_t* __restrict__ keys_s,
                                     const uint32_t* __restrict__ perm_s2k, const int64_t* __restrict__ ttl_k,
                                     const long long* d_U, uint64_t skip_key, int has_skip,
                                     const int32_t* __restrict__ slot_of, long long* __restrict__ ttl,
                                     int32_t* __restrict__ slots_s, ErrorRecord* err, long long iteration,
                                     const uint32_t* __restrict__ next_ids, const long long* d_next_U,
                                     int64_t* __restrict__ mark, long long tag, int64_t* zero2) {
  if (zero2 && blockIdx.x == 0 && threadIdx.x < 2) zero2[threadIdx.x] = 0;  // the step's stats (no memset)
  const long long U = *d_U, NU = *d_next_U;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < U; s += stride) {
    const uint32_t id = ids_s[s];
    const uint64_t key = keys_s[s];
    const long long k = perm_s2k[s];
    const int32_t slot = id == kNoId ? -1 : slot_of[id];
    const bool skipped = has_skip && key == skip_key;
    if (slot < 0) {
      raise_error(err, skipped ? BP_ERR_CACHE_MISS : BP_ERR_CACHE_ORDERING, iteration,
                  skipped ? (k | (1ll << 40)) : k, key);
    } else if (!skipped) {
      ttl[slot] = ttl_k[k];
    }
    slots_s[s] = slot;
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < NU; i += stride) mark[next_ids[i]] = tag;
}

int apply_resolve_mark(bp_cache* c, bp_prep* P, const int64_t* d_ttl_k, uint64_t skip_key, int32_t has_skip,
                       int32_t* d_slots_s, bp_prep* N, int64_t* d_mark, int64_t tag, int64_t* d_zero2,
                       cudaStream_t s) {
  if (!c->sc || !P->schema_mode || !N->schema_mode) return BP_ERR_INVALID;
  if (P->n_occ == 0 || N->n_occ == 0) {  // the separate launches handle the empty cases
    int rc = bp_cache_apply_resolve(c, P, d_ttl_k, skip_key, has_skip, d_slots_s, s);
    return rc ? rc : mark_ids_zero(N, d_mark, tag, d_zero2, s);
  }
  const long long n = P->n_occ > N->n_occ ? P->n_occ : N->n_occ;
  k_apply_resolve_mark<<<grid_for(n, 256), 256, 0, s>>>(
      P->d_uniq_id_s, P->d_uniq_key_s, P->d_perm_s2k, d_ttl_k, P->d_num_unique, skip_key, has_skip, c->d_slot_of,
      c->d_ttl, d_slots_s, c->ctx ? c->ctx->d_err : nullptr, P->iteration, N->d_uniq_id_s, N->d_num_unique, d_mark,
      tag, d_zero2);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

__global__ void k_gather(const float* __restrict__ values, const int32_t* __restrict__ slots, long long n,
                         const long long* d_n, int dim, float* __restrict__ out) {
  n = load_count(n, d_n);
  const long long total = n * dim;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / dim;
    const int32_t slot = slots[r];
    out[i] = slot >= 0 ? values[(long long)slot * dim + (i - r * dim)] : 0.f;
  }
}

__global__ void k_update(float* __restrict__ values, uint8_t* __restrict__ dirty, const int32_t* __restrict__ slots,
                         const float* __restrict__ rows, const uint8_t* __restrict__ mask, long long n,
                         const long long* d_n, int dim) {
  n = load_count(n, d_n);
  const long long total = n * dim;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / dim;
    const int d = (int)(i - r * dim);
    const int32_t slot = slots[r];
    if (slot < 0) continue;
    values[(long long)slot * dim + d] = rows[i];
    if (d == 0 && mask && mask[r]) dirty[slot] = 1;
  }
}

__global__ void k_evict_flag(const uint8_t* __restrict__ used, const long long* __restrict__ ttl, long long cap,
                             long long completed, int drain, uint32_t* __restrict__ flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cap; i += (long long)gridDim.x * blockDim.x)
    flag[i] = used[i] && (drain || ttl[i] <= completed) ? 1u : 0u;
}

__global__ void k_evict_out(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, long long cap,
                            const long long* __restrict__ d_count, long long out_cap, int dim,
                            const uint64_t* __restrict__ slot_key, const uint32_t* __restrict__ slot_id,
                            const float* __restrict__ values, uint8_t* __restrict__ dirty, uint8_t* __restrict__ used,
                            int32_t* __restrict__ slot_of, const CacheCounters* __restrict__ ctr,
                            uint32_t* __restrict__ free_list, uint64_t* __restrict__ out_keys,
                            uint32_t* __restrict__ out_ids, float* __restrict__ out_rows,
                            uint8_t* __restrict__ out_dirty, unsigned long long* __restrict__ n_dirty,
                            ErrorRecord* err, long long iteration) {
  const long long cnt = *d_count;
  if (cnt > out_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_error(err, BP_ERR_ENGINE, iteration, cnt, 0);
    return;
  }
  const long long top = ctr->free_top;
  unsigned long long nd = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cap; i += (long long)gridDim.x * blockDim.x) {
    if (!flag[i]) continue;
    const long long p = pos[i];
    const uint8_t dty = dirty[i];
    nd += dty;
    if (out_keys) out_keys[p] = slot_key[i];
    if (out_ids) out_ids[p] = slot_id[i];
    if (out_dirty) out_dirty[p] = dty;
    if (out_rows) {
      if ((dim & 3) == 0) {
        const float4* src = reinterpret_cast<const float4*>(values + i * dim);
        float4* dst = reinterpret_cast<float4*>(out_rows + p * dim);
        for (int d = 0; d < (dim >> 2); ++d) dst[d] = src[d];
      } else {
        for (int d = 0; d < dim; ++d) out_rows[p * dim + d] = values[i * dim + d];
      }
    }
    slot_of[slot_id[i]] = -1;
    used[i] = 0;
    dirty[i] = 0;
    free_list[top + (cnt - 1 - p)] = (uint32_t)i;
  }
  cta_add(n_dirty, nd);
}

__global__ void k_evict_planned(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ ids,
                                const long long* __restrict__ d_n, long long n_max, int dim,
                                const float* __restrict__ values, uint8_t* __restrict__ dirty,
                                uint8_t* __restrict__ used, int32_t* __restrict__ slot_of,
                                CacheCounters* __restrict__ ctr, uint32_t* __restrict__ free_list,
                                uint64_t* __restrict__ out_keys, uint32_t* __restrict__ out_ids,
                                float* __restrict__ out_rows, uint8_t* __restrict__ out_dirty,
                                long long* __restrict__ out_count, ErrorRecord* err, long long iteration,
                                const int64_t* __restrict__ d_expect, StepRecord rec) {
  const long long n = load_count(n_max, d_n);
  const long long top = ctr->free_top;
  unsigned long long nd = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t id = ids[i];
    const int32_t slot = slot_of[id];
    if (slot < 0) {
      raise_error(err, BP_ERR_ENGINE, iteration, (1ll << 41) | i, keys[i]);
      continue;
    }
    const uint8_t dty = dirty[slot];
    nd += dty;
    if (out_keys) out_keys[i] = keys[i];
    out_ids[i] = id;
    out_dirty[i] = dty;
    if ((dim & 3) == 0) {
      const float4* src = reinterpret_cast<const float4*>(values + (long long)slot * dim);
      float4* dst = reinterpret_cast<float4*>(out_rows + i * dim);
      for (int d = 0; d < (dim >> 2); ++d) dst[d] = src[d];
    } else {
      for (int d = 0; d < dim; ++d) out_rows[i * dim + d] = values[(long long)slot * dim + d];
    }
    slot_of[id] = -1;
    used[slot] = 0;
    dirty[slot] = 0;
    free_list[top + i] = (uint32_t)slot;
  }
  // the last block to finish commits the counters (no separate end kernel,
  // no memset of the output counts) and, for the engine, the step record
  __shared__ unsigned long long sh_nd;
  if (threadIdx.x == 0) sh_nd = 0;
  __syncthreads();
  nd = warp_sum(nd);
  if (lane_id() == 0 && nd) atomicAdd(&sh_nd, nd);
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (sh_nd) atomicAdd(&ctr->evict_dirty, sh_nd);
  __threadfence();
  if (atomicAdd(&ctr->evict_ticket, 1u) != gridDim.x - 1) return;
  __threadfence();
  const unsigned long long n_dirty = atomicExch(&ctr->evict_dirty, 0ull);
  ctr->evict_ticket = 0;
  ctr->free_top += n;
  ctr->occupancy -= n;
  ctr->evictions += n;
  out_count[0] = n;
  out_count[1] = (long long)n_dirty;
  if (d_expect && ctr->occupancy != *d_expect) raise_error(err, BP_ERR_ENGINE, iteration, 1ll << 41, 0);
  if (rec.out) write_step_record(rec, n, (long long)n_dirty, err);
}

__global__ void k_evict_end(CacheCounters* ctr, const long long* d_count, long long out_cap) {
  const long long cnt = *d_count;
  if (cnt > out_cap) return;
  ctr->free_top += cnt;
  ctr->occupancy -= cnt;
  ctr->evictions += cnt;
}

__global__ void k_checksum(const uint8_t* __restrict__ used, const uint64_t* __restrict__ slot_key,
                           const long long* __restrict__ ttl, const uint8_t* __restrict__ dirty,
                           const float* __restrict__ values, long long cap, int dim, unsigned long long* out) {
  unsigned long long acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cap; i += (long long)gridDim.x * blockDim.x) {
    if (!used[i]) continue;
    const uint64_t key = slot_key[i];
    // (table << 44) ^ row: equal to the packed key because rows < 2^44.
    uint64_t w = splitmix64(key);
    w = splitmix64(w ^ (uint64_t)ttl[i]);
    w = splitmix64(w ^ ((uint64_t)dirty[i] << 63));
    for (int d = 0; d < dim; ++d) w = splitmix64(w ^ (uint64_t)__float_as_uint(values[i * dim + d]));
    acc ^= w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane_id() == 0 && acc) atomicXor(out, acc);
}

// Schema ids for API keys; out-of-schema keys map to kNoId (-> absent).
__global__ void k_schema_ids_soft(const int64_t* base, const int64_t* rows, int num_tables, const uint64_t* keys,
                                  long long n, const long long* d_n, uint32_t* ids) {
  n = load_count(n, d_n);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    ids[i] = schema_id(base, rows, num_tables, keys[i]);
}

static int cache_grow_ids(bp_cache* c, long long new_cap, cudaStream_t s) {
  int32_t* n;
  BP_CUDA_TRY(pool_alloc(&n, new_cap, s));
  k_fill_i32<<<grid_for(new_cap, 256), 256, 0, s>>>(n, new_cap, -1);
  if (c->id_cap) {
    BP_CUDA_TRY(cudaMemcpyAsync(n, c->d_slot_of, c->id_cap * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    cudaFreeAsync(c->d_slot_of, s);
  }
  c->d_slot_of = n;
  c->id_cap = new_cap;
  return BP_OK;
}

static int cache_tmp(bp_cache* c, long long n, cudaStream_t s) {
  if (c->ids_cap >= n) return BP_OK;
  if (c->ids_cap) {
    cudaFreeAsync(c->d_ids_tmp, s);
    cudaFreeAsync(c->d_slot_tmp, s);
  }
  long long cap = 1024;
  while (cap < n) cap <<= 1;
  c->ids_cap = cap;
  BP_CUDA_TRY(pool_alloc(&c->d_ids_tmp, cap, s));
  BP_CUDA_TRY(pool_alloc(&c->d_slot_tmp, cap, s));
  return BP_OK;
}

// ids for caller keys: given ids, schema ids, or registry ids.
static int cache_ids(bp_cache* c, const uint64_t* keys, const uint32_t* ids, long long n, const long long* d_n,
                     int insert, const uint32_t** out, cudaStream_t s) {
  if (ids) {
    *out = ids;
    return BP_OK;
  }
  int rc = cache_tmp(c, n, s);
  if (rc) return rc;
  if (c->sc) {
    k_schema_ids_soft<<<grid_for(n, 256), 256, 0, s>>>(c->sc->d_table_base, c->sc->d_rows, c->sc->num_tables, keys,
                                                       n, d_n, c->d_ids_tmp);
    BP_LAUNCH_CHECK();
  } else {
    if (insert) {
      int grown = 0;
      rc = registry_reserve(&c->reg, n, s, &grown);
      if (rc) return rc;
      if (grown) {
        rc = cache_grow_ids(c, c->reg.id_capacity, s);
        if (rc) return rc;
      }
    }
    rc = registry_map(&c->reg, keys, n, d_n, c->d_ids_tmp, insert, s);
    if (rc) return rc;
  }
  *out = c->d_ids_tmp;
  return BP_OK;
}

}  // namespace bp

extern "C" int bp_cache_create(bp_ctx* ctx, const bp_schema* sc, int64_t capacity, int32_t dim, bp_cache** out) {
  using namespace bp;
  if (capacity < 1 || dim < 1 || capacity >= (int64_t)kNoId) return BP_ERR_CONFIG;
  cudaStream_t s = 0;
  bp_cache* c = new bp_cache();
  c->ctx = ctx;
  c->sc = sc;
  c->capacity = capacity;
  c->dim = dim;
  const long long C = capacity;
  BP_CUDA_TRY(cudaMalloc(&c->d_slot_key, C * sizeof(uint64_t)));
  BP_CUDA_TRY(cudaMalloc(&c->d_slot_id, C * sizeof(uint32_t)));
  BP_CUDA_TRY(cudaMalloc(&c->d_ttl, C * sizeof(long long)));
  BP_CUDA_TRY(cudaMalloc(&c->d_dirty, C));
  BP_CUDA_TRY(cudaMalloc(&c->d_used, C));
  BP_CUDA_TRY(cudaMalloc(&c->d_values, C * dim * sizeof(float)));
  BP_CUDA_TRY(cudaMalloc(&c->d_free, C * sizeof(uint32_t)));
  BP_CUDA_TRY(cudaMalloc(&c->d_flag, C * sizeof(uint32_t)));
  BP_CUDA_TRY(cudaMalloc(&c->d_pos, C * sizeof(uint32_t)));
  BP_CUDA_TRY(cudaMalloc(&c->d_partials, scan_state_words(C) * sizeof(uint32_t)));
  BP_CUDA_TRY(cudaMalloc(&c->d_ctr, sizeof(CacheCounters)));
  BP_CUDA_TRY(cudaMallocHost(&c->h_ctr, sizeof(CacheCounters)));
  BP_CUDA_TRY(cudaMemset(c->d_dirty, 0, C));
  BP_CUDA_TRY(cudaMemset(c->d_used, 0, C));
  BP_CUDA_TRY(cudaMemset(c->d_values, 0, C * dim * sizeof(float)));
  BP_CUDA_TRY(cudaMemset(c->d_ttl, 0, C * sizeof(long long)));
  CacheCounters init{};
  init.free_top = C;
  BP_CUDA_TRY(cudaMemcpy(c->d_ctr, &init, sizeof(init), cudaMemcpyHostToDevice));
  k_free_init<<<grid_for(C, 256), 256, 0, s>>>(c->d_free, C);
  int rc;
  if (sc) {
    rc = cache_grow_ids(c, sc->total_rows, s);
  } else {
    rc = registry_init(&c->reg, 1024, s);
    if (rc == BP_OK) rc = cache_grow_ids(c, c->reg.id_capacity, s);
  }
  if (rc) return rc;
  BP_CUDA_TRY(cudaStreamSynchronize(s));
  *out = c;
  return BP_OK;
}

extern "C" int bp_cache_destroy(bp_cache* c) {
  if (!c) return BP_OK;
  cudaDeviceSynchronize();
  cudaStream_t s = 0;
  cudaFree(c->d_slot_key);
  cudaFree(c->d_slot_id);
  cudaFree(c->d_ttl);
  cudaFree(c->d_dirty);
  cudaFree(c->d_used);
  cudaFree(c->d_values);
  cudaFree(c->d_free);
  cudaFree(c->d_flag);
  cudaFree(c->d_pos);
  cudaFree(c->d_partials);
  cudaFree(c->d_ctr);
  cudaFreeHost(c->h_ctr);
  if (c->d_slot_of) cudaFreeAsync(c->d_slot_of, s);
  if (c->ids_cap) {
    cudaFreeAsync(c->d_ids_tmp, s);
    cudaFreeAsync(c->d_slot_tmp, s);
  }
  if (!c->sc) bp::registry_free(&c->reg, s);
  cudaStreamSynchronize(s);
  delete c;
  return BP_OK;
}

extern "C" int bp_cache_get_stats(bp_cache* c, bp_stream_t stream, bp_cache_stats* out) {
  cudaStream_t s = (cudaStream_t)stream;
  BP_CUDA_TRY(cudaMemcpyAsync(c->h_ctr, c->d_ctr, sizeof(bp::CacheCounters), cudaMemcpyDeviceToHost, s));
  long long reg = 0;
  if (!c->sc) BP_CUDA_TRY(cudaMemcpyAsync(&reg, c->reg.d_count, sizeof(long long), cudaMemcpyDeviceToHost, s));
  BP_CUDA_TRY(cudaStreamSynchronize(s));
  out->occupancy = c->h_ctr->occupancy;
  out->insertions = c->h_ctr->insertions;
  out->evictions = c->h_ctr->evictions;
  out->peak_occupancy = c->h_ctr->peak_occupancy;
  out->capacity = c->capacity;
  out->registry_size = reg;
  return BP_OK;
}

namespace bp {
// bp_cache_insert of (*d_n - sub) rows that also stores that count in n_out
// (the engine's plan-slot insert: no separate count kernel).
int cache_insert_sub(bp_cache* c, const uint64_t* d_keys, const uint32_t* d_ids, const float* d_rows,
                     const int64_t* d_ttls, int64_t n, const int64_t* d_n, int64_t sub, int64_t* n_out,
                     int64_t iteration, cudaStream_t s);
}  // namespace bp

extern "C" int bp_cache_insert(bp_cache* c, const uint64_t* d_keys, const uint32_t* d_ids, const float* d_rows,
                               const int64_t* d_ttls, int64_t n, const int64_t* d_n, int64_t iteration,
                               bp_stream_t stream) {
  return bp::cache_insert_sub(c, d_keys, d_ids, d_rows, d_ttls, n, d_n, 0, nullptr, iteration, (cudaStream_t)stream);
}

int bp::cache_insert_sub(bp_cache* c, const uint64_t* d_keys, const uint32_t* d_ids, const float* d_rows,
                         const int64_t* d_ttls, int64_t n, const int64_t* d_n, int64_t sub, int64_t* n_out_,
                         int64_t iteration, cudaStream_t s) {
  using namespace bp;
  long long* n_out = (long long*)n_out_;
  if (n <= 0) {
    if (n_out) BP_CUDA_TRY(cudaMemsetAsync(n_out, 0, sizeof(long long), s));
    return BP_OK;
  }
  const uint32_t* ids;
  int rc = cache_ids(c, d_keys, d_ids, n, (const long long*)d_n, 1, &ids, s);
  if (rc) return rc;
  ErrorRecord* err = c->ctx ? c->ctx->d_err : nullptr;
  k_insert<<<grid_for(n, 256), 256, 0, s>>>(d_keys, ids, d_rows, d_ttls, n, (const long long*)d_n, c->dim, c->d_ctr,
                                            c->capacity, c->d_slot_of, c->d_slot_key, c->d_slot_id, c->d_ttl,
                                            c->d_dirty, c->d_used, c->d_values, c->d_free, err, iteration, sub,
                                            n_out);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_cache_set_ttl(bp_cache* c, const uint64_t* d_keys, const uint32_t* d_ids, const int64_t* d_ttls,
                                int64_t n, const int64_t* d_n, int64_t iteration, bp_stream_t stream) {
  using namespace bp;
  if (n <= 0) return BP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t* ids;
  int rc = cache_ids(c, d_keys, d_ids, n, (const long long*)d_n, 0, &ids, s);
  if (rc) return rc;
  k_set_ttl<<<grid_for(n, 256), 256, 0, s>>>(d_keys, ids, d_ttls, n, (const long long*)d_n, c->d_slot_of, c->d_ttl,
                                             c->ctx ? c->ctx->d_err : nullptr, iteration);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_cache_resolve(bp_cache* c, const uint64_t* d_keys, const uint32_t* d_ids, int64_t n,
                                const int64_t* d_n, int64_t iteration, int32_t* d_slots, bp_stream_t stream) {
  using namespace bp;
  if (n <= 0) return BP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t* ids;
  int rc = cache_ids(c, d_keys, d_ids, n, (const long long*)d_n, 0, &ids, s);
  if (rc) return rc;
  k_resolve<<<grid_for(n, 256), 256, 0, s>>>(d_keys, ids, n, (const long long*)d_n, c->d_slot_of, d_slots,
                                             c->ctx ? c->ctx->d_err : nullptr, iteration);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_cache_apply_resolve(bp_cache* c, bp_prep* P, const int64_t* d_ttl_k, uint64_t skip_key,
                                      int32_t has_skip, int32_t* d_slots_s, bp_stream_t stream) {
  using namespace bp;
  if (P->n_occ == 0) return BP_OK;
  if (!c->sc || !P->schema_mode) return BP_ERR_INVALID;
  k_apply_resolve<<<grid_for(P->n_occ, 256), 256, 0, (cudaStream_t)stream>>>(
      P->d_uniq_id_s, P->d_uniq_key_s, P->d_perm_s2k, d_ttl_k, P->d_num_unique, skip_key, has_skip, c->d_slot_of,
      c->d_ttl, d_slots_s, c->ctx ? c->ctx->d_err : nullptr, P->iteration);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_cache_gather(bp_cache* c, const int32_t* d_slots, int64_t n, const int64_t* d_n, float* d_out,
                               bp_stream_t stream) {
  using namespace bp;
  if (n <= 0) return BP_OK;
  k_gather<<<grid_for(n * c->dim, 256), 256, 0, (cudaStream_t)stream>>>(c->d_values, d_slots, n,
                                                                        (const long long*)d_n, c->dim, d_out);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_cache_update(bp_cache* c, const int32_t* d_slots, const float* d_rows, const uint8_t* d_dirty,
                               int64_t n, const int64_t* d_n, bp_stream_t stream) {
  using namespace bp;
  if (n <= 0) return BP_OK;
  k_update<<<grid_for(n * c->dim, 256), 256, 0, (cudaStream_t)stream>>>(c->d_values, c->d_dirty, d_slots, d_rows,
                                                                        d_dirty, n, (const long long*)d_n, c->dim);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_cache_evict(bp_cache* c, int64_t completed, int32_t drain, const bp_evict_buffers* o,
                              int64_t out_capacity, bp_stream_t stream) {
  using namespace bp;
  cudaStream_t s = (cudaStream_t)stream;
  const long long C = c->capacity;
  BP_CUDA_TRY(cudaMemsetAsync(o->d_count, 0, 2 * sizeof(int64_t), s));
  k_evict_flag<<<grid_for(C, 256), 256, 0, s>>>(c->d_used, c->d_ttl, C, completed, drain, c->d_flag);
  BP_CUDA_TRY(exclusive_scan(c->d_flag, c->d_pos, C, nullptr, c->d_partials, nullptr, (long long*)o->d_count, s));
  k_evict_out<<<grid_for(C, 256), 256, 0, s>>>(c->d_flag, c->d_pos, C, (const long long*)o->d_count, out_capacity,
                                               c->dim, c->d_slot_key, c->d_slot_id, c->d_values, c->d_dirty,
                                               c->d_used, c->d_slot_of, c->d_ctr, c->d_free, o->d_keys, o->d_ids,
                                               o->d_rows, o->d_dirty, (unsigned long long*)&o->d_count[1],
                                               c->ctx ? c->ctx->d_err : nullptr, completed);
  k_evict_end<<<1, 1, 0, s>>>(c->d_ctr, (const long long*)o->d_count, out_capacity);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

int bp::cache_evict_planned_rec(bp_cache* c, const uint64_t* d_keys, const uint32_t* d_ids, const int64_t* d_n,
                                int64_t n_max, const int64_t* d_expect, int64_t iteration, const bp_evict_buffers* o,
                                const StepRecord& rec, cudaStream_t s) {
  using namespace bp;
  ErrorRecord* err = c->ctx ? c->ctx->d_err : nullptr;
  k_evict_planned<<<grid_for(n_max, 256, kNumSMs * 4), 256, 0, s>>>(
      d_keys, d_ids, (const long long*)d_n, n_max, c->dim, c->d_values, c->d_dirty, c->d_used, c->d_slot_of, c->d_ctr,
      c->d_free, o->d_keys, o->d_ids, o->d_rows, o->d_dirty, (long long*)o->d_count, err, iteration, d_expect, rec);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_cache_evict_planned(bp_cache* c, const uint64_t* d_keys, const uint32_t* d_ids, const int64_t* d_n,
                                      int64_t n_max, const int64_t* d_expect, int64_t iteration,
                                      const bp_evict_buffers* o, bp_stream_t stream) {
  return bp::cache_evict_planned_rec(c, d_keys, d_ids, d_n, n_max, d_expect, iteration, o, bp::StepRecord{},
                                     (cudaStream_t)stream);
}

extern "C" int bp_cache_checksum(bp_cache* c, uint64_t* d_out, bp_stream_t stream) {
  using namespace bp;
  cudaStream_t s = (cudaStream_t)stream;
  BP_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(uint64_t), s));
  k_checksum<<<grid_for(c->capacity, 256), 256, 0, s>>>(c->d_used, c->d_slot_key, c->d_ttl, c->d_dirty, c->d_values,
                                                        c->capacity, c->dim, (unsigned long long*)d_out);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_cache_get_view(const bp_cache* c, bp_cache_view* v) {
  v->capacity = c->capacity;
  v->dim = c->dim;
  v->pad = 0;
  v->d_values = c->d_values;
  v->d_ttl = (int64_t*)c->d_ttl;
  v->d_dirty = c->d_dirty;
  v->d_used = c->d_used;
  v->d_slot_key = c->d_slot_key;
  return BP_OK;
}
