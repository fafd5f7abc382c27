// Context, schema, key registry and generic utilities of the C ABI.
#include <cstring>
#include <mutex>
#include <string>

#include "internal.cuh"

static thread_local std::string g_last_error;

void bp_set_last_error(const char* msg, const char* file, int line) {
  g_last_error = std::string(msg) + " (" + file + ":" + std::to_string(line) + ")";
}

extern "C" const char* bp_version(void) { return "bagpipe_b200 0.1.0 sm_100a"; }

// Struct sizes of the ABI, so bindings can reject a stale header/library pair.
extern "C" int64_t bp_abi_sizeof(int32_t which) {
  switch (which) {
    case 0: return (int64_t)sizeof(bp_error_t);
    case 1: return (int64_t)sizeof(bp_prep_view);
    case 2: return (int64_t)sizeof(bp_plan_buffers);
    case 3: return (int64_t)sizeof(bp_planner_stats);
    case 4: return (int64_t)sizeof(bp_cache_stats);
    case 5: return (int64_t)sizeof(bp_evict_buffers);
    case 6: return (int64_t)sizeof(bp_cache_view);
    case 7: return (int64_t)sizeof(bp_engine_config);
    case 8: return (int64_t)sizeof(bp_step_result);
    case 9: return (int64_t)sizeof(bp_engine_parts_t);
    case 10: return (int64_t)sizeof(bp_planner_dump_t);
    case 11: return (int64_t)sizeof(bp_peer_xchg);
    case 12: return (int64_t)sizeof(bp_sgd_tensors);
    default: return -1;
  }
}
extern "C" const char* bp_last_error_message(void) { return g_last_error.c_str(); }

static void raise_pool_threshold() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
    uint64_t threshold = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  });
}

extern "C" int bp_ctx_create(bp_ctx** out) {
  raise_pool_threshold();
  bp_ctx* c = new bp_ctx();
  BP_CUDA_TRY(cudaMalloc(&c->d_err, sizeof(bp::ErrorRecord)));
  BP_CUDA_TRY(cudaMemset(c->d_err, 0, sizeof(bp::ErrorRecord)));
  BP_CUDA_TRY(cudaMallocHost(&c->h_err, sizeof(bp::ErrorRecord)));
  std::memset(c->h_err, 0, sizeof(bp::ErrorRecord));
  *out = c;
  return BP_OK;
}

extern "C" int bp_ctx_destroy(bp_ctx* c) {
  if (!c) return BP_OK;
  cudaFree(c->d_err);
  cudaFreeHost(c->h_err);
  delete c;
  return BP_OK;
}

extern "C" int bp_ctx_check(bp_ctx* c, bp_stream_t stream, bp_error_t* h_out) {
  cudaStream_t s = (cudaStream_t)stream;
  BP_CUDA_TRY(cudaMemcpyAsync(c->h_err, c->d_err, sizeof(bp::ErrorRecord), cudaMemcpyDeviceToHost, s));
  BP_CUDA_TRY(cudaStreamSynchronize(s));
  static_assert(sizeof(bp::ErrorRecord) == sizeof(bp_error_t), "error record layout");
  std::memcpy(h_out, c->h_err, sizeof(bp_error_t));
  if (c->h_err->code != 0) {
    BP_CUDA_TRY(cudaMemsetAsync(c->d_err, 0, sizeof(bp::ErrorRecord), s));
    BP_CUDA_TRY(cudaStreamSynchronize(s));
  }
  return h_out->code;
}

extern "C" int bp_schema_create(int32_t num_tables, const int64_t* h_rows, int32_t emb_dim, bp_schema** out) {
  if (num_tables < 1 || emb_dim < 1) return BP_ERR_INVALID;
  bp_schema* sc = new bp_schema();
  sc->num_tables = num_tables;
  sc->emb_dim = emb_dim;
  sc->h_table_base = new int64_t[num_tables + 1];
  sc->h_table_base[0] = 0;
  for (int t = 0; t < num_tables; ++t) {
    if (h_rows[t] < 1) return BP_ERR_INVALID;
    sc->h_table_base[t + 1] = sc->h_table_base[t] + h_rows[t];
  }
  sc->total_rows = sc->h_table_base[num_tables];
  if (sc->total_rows >= (int64_t)bp::kNoId) return BP_ERR_INVALID;  // dense ids are u32
  sc->id_bits = bp::bit_width_u64((unsigned long long)(sc->total_rows - 1));
  if (sc->id_bits < 1) sc->id_bits = 1;
  BP_CUDA_TRY(cudaMalloc(&sc->d_table_base, sizeof(int64_t) * (num_tables + 1)));
  BP_CUDA_TRY(cudaMalloc(&sc->d_rows, sizeof(int64_t) * num_tables));
  BP_CUDA_TRY(cudaMemcpy(sc->d_table_base, sc->h_table_base, sizeof(int64_t) * (num_tables + 1),
                         cudaMemcpyHostToDevice));
  BP_CUDA_TRY(cudaMemcpy(sc->d_rows, h_rows, sizeof(int64_t) * num_tables, cudaMemcpyHostToDevice));
  *out = sc;
  return BP_OK;
}

extern "C" int bp_schema_destroy(bp_schema* sc) {
  if (!sc) return BP_OK;
  cudaFree(sc->d_table_base);
  cudaFree(sc->d_rows);
  delete[] sc->h_table_base;
  delete sc;
  return BP_OK;
}

extern "C" int64_t bp_schema_total_rows(const bp_schema* sc) { return sc->total_rows; }

__global__ void k_schema_ids(const int64_t* base, const int64_t* rows, int num_tables, const uint64_t* keys,
                             long long n, uint32_t* ids, bp::ErrorRecord* err) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t id = bp::schema_id(base, rows, num_tables, keys[i]);
    if (id == bp::kNoId) bp::raise_error(err, BP_ERR_STORE_KEY, -1, i, keys[i]);
    ids[i] = id;
  }
}

extern "C" int bp_schema_ids(bp_ctx* ctx, const bp_schema* sc, const uint64_t* d_keys, int64_t n, uint32_t* d_ids,
                             bp_stream_t stream) {
  if (n <= 0) return BP_OK;
  k_schema_ids<<<bp::grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(sc->d_table_base, sc->d_rows,
                                                                        sc->num_tables, d_keys, n, d_ids,
                                                                        ctx ? ctx->d_err : nullptr);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

// ------------------------------------------------------------------ registry

namespace bp {

__global__ void k_fill_u64(uint64_t* p, long long n, uint64_t v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_registry_claim(uint64_t* keys, long long slots, const uint64_t* in, long long n,
                                 const long long* d_n, uint32_t* claim, long long* slot_of_input) {
  n = load_count(n, d_n);
  const uint64_t mask = (uint64_t)slots - 1;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint64_t key = in[i];
    uint64_t h = registry_hash(key) & mask;
    uint32_t won = 0;
    for (;;) {
      const uint64_t prev = atomicCAS((unsigned long long*)&keys[h], (unsigned long long)kEmptyKey,
                                      (unsigned long long)key);
      if (prev == kEmptyKey) {
        won = 1;
        break;
      }
      if (prev == key) break;
      h = (h + 1) & mask;
    }
    claim[i] = won;
    slot_of_input[i] = (long long)h;
  }
}

__global__ void k_registry_assign(uint32_t* ids, const uint32_t* claim, const uint32_t* scan, long long n,
                                  const long long* d_n, const long long* slot_of_input, long long* d_count,
                                  const uint32_t* d_total) {
  n = load_count(n, d_n);
  const long long base = *d_count;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (claim[i]) ids[slot_of_input[i]] = (uint32_t)(base + scan[i]);
}

__global__ void k_registry_bump(long long* d_count, const uint32_t* d_total) { *d_count += *d_total; }

__global__ void k_registry_lookup(const uint64_t* keys, const uint32_t* ids, long long slots, const uint64_t* in,
                                  long long n, const long long* d_n, uint32_t* out) {
  n = load_count(n, d_n);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = registry_find(keys, ids, slots, in[i]);
}

__global__ void k_registry_rehash(const uint64_t* okeys, const uint32_t* oids, long long oslots, uint64_t* nkeys,
                                  uint32_t* nids, long long nslots) {
  const uint64_t mask = (uint64_t)nslots - 1;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < oslots; i += (long long)gridDim.x * blockDim.x) {
    const uint64_t key = okeys[i];
    if (key == kEmptyKey) continue;
    uint64_t h = registry_hash(key) & mask;
    while (atomicCAS((unsigned long long*)&nkeys[h], (unsigned long long)kEmptyKey, (unsigned long long)key) !=
           kEmptyKey)
      h = (h + 1) & mask;
    nids[h] = oids[i];
  }
}

static long long pow2_at_least(long long x) {
  long long p = 1;
  while (p < x) p <<= 1;
  return p;
}

int registry_init(Registry* r, long long id_capacity, cudaStream_t s) {
  r->id_capacity = pow2_at_least(id_capacity < 64 ? 64 : id_capacity);
  r->slots = r->id_capacity * 2;
  BP_CUDA_TRY(pool_alloc(&r->d_keys, r->slots, s));
  BP_CUDA_TRY(pool_alloc(&r->d_ids, r->slots, s));
  BP_CUDA_TRY(pool_alloc(&r->d_count, 1, s));
  k_fill_u64<<<grid_for(r->slots, 256), 256, 0, s>>>(r->d_keys, r->slots, kEmptyKey);
  BP_CUDA_TRY(cudaMemsetAsync(r->d_count, 0, sizeof(long long), s));
  r->count_upper = 0;
  return BP_OK;
}

void registry_free(Registry* r, cudaStream_t s) {
  if (r->d_keys) cudaFreeAsync(r->d_keys, s);
  if (r->d_ids) cudaFreeAsync(r->d_ids, s);
  if (r->d_count) cudaFreeAsync(r->d_count, s);
  if (r->d_claim) cudaFreeAsync(r->d_claim, s);
  if (r->d_claim_scan) cudaFreeAsync(r->d_claim_scan, s);
  if (r->d_partials) cudaFreeAsync(r->d_partials, s);
  *r = Registry();
}

int registry_reserve(Registry* r, long long n, cudaStream_t s, int* grown) {
  *grown = 0;
  if (r->count_upper + n <= r->id_capacity) {
    r->count_upper += n;
    return BP_OK;
  }
  long long count = 0;
  BP_CUDA_TRY(cudaMemcpyAsync(&count, r->d_count, sizeof(long long), cudaMemcpyDeviceToHost, s));
  BP_CUDA_TRY(cudaStreamSynchronize(s));
  if (count + n > r->id_capacity) {
    const long long ncap = pow2_at_least(2 * (count + n));
    const long long nslots = ncap * 2;
    uint64_t* nkeys;
    uint32_t* nids;
    BP_CUDA_TRY(pool_alloc(&nkeys, nslots, s));
    BP_CUDA_TRY(pool_alloc(&nids, nslots, s));
    k_fill_u64<<<grid_for(nslots, 256), 256, 0, s>>>(nkeys, nslots, kEmptyKey);
    k_registry_rehash<<<grid_for(r->slots, 256), 256, 0, s>>>(r->d_keys, r->d_ids, r->slots, nkeys, nids, nslots);
    BP_LAUNCH_CHECK();
    cudaFreeAsync(r->d_keys, s);
    cudaFreeAsync(r->d_ids, s);
    r->d_keys = nkeys;
    r->d_ids = nids;
    r->slots = nslots;
    r->id_capacity = ncap;
    *grown = 1;
  }
  r->count_upper = count + n;
  return BP_OK;
}

int registry_map(Registry* r, const uint64_t* d_keys, long long n, const long long* d_n, uint32_t* d_ids,
                 int insert, cudaStream_t s) {
  if (n <= 0) return BP_OK;
  if (insert) {
    if (r->claim_cap < n) {
      if (r->d_claim) cudaFreeAsync(r->d_claim, s);
      if (r->d_claim_scan) cudaFreeAsync(r->d_claim_scan, s);
      if (r->d_partials) cudaFreeAsync(r->d_partials, s);
      r->claim_cap = pow2_at_least(n);
      BP_CUDA_TRY(pool_alloc(&r->d_claim, r->claim_cap, s));
      BP_CUDA_TRY(pool_alloc(&r->d_claim_scan, r->claim_cap + 1, s));
      BP_CUDA_TRY(pool_alloc(&r->d_partials, scan_state_words(r->claim_cap), s));
    }
    long long* slot_of_input;
    BP_CUDA_TRY(pool_alloc(&slot_of_input, n, s));
    k_registry_claim<<<grid_for(n, 256), 256, 0, s>>>(r->d_keys, r->slots, d_keys, n, d_n, r->d_claim,
                                                      slot_of_input);
    uint32_t* d_total = r->d_claim_scan + r->claim_cap;
    BP_CUDA_TRY(exclusive_scan(r->d_claim, r->d_claim_scan, n, d_n, r->d_partials, d_total, nullptr, s));
    k_registry_assign<<<grid_for(n, 256), 256, 0, s>>>(r->d_ids, r->d_claim, r->d_claim_scan, n, d_n,
                                                       slot_of_input, r->d_count, d_total);
    k_registry_bump<<<1, 1, 0, s>>>(r->d_count, d_total);
    cudaFreeAsync(slot_of_input, s);
    BP_LAUNCH_CHECK();
  }
  k_registry_lookup<<<grid_for(n, 256), 256, 0, s>>>(r->d_keys, r->d_ids, r->slots, d_keys, n, d_n, d_ids);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

// -------------------------------------------------------------- utilities

__global__ void k_iota_u32(uint32_t* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = (uint32_t)i;
}

__global__ void k_xor_rows(const float* rows, long long n, int dim, unsigned long long* out) {
  unsigned long long acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    uint64_t w = splitmix64((uint64_t)i);
    for (int d = 0; d < dim; ++d) w = splitmix64(w ^ (uint64_t)__float_as_uint(rows[i * dim + d]));
    acc ^= w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane_id() == 0 && acc) atomicXor(out, acc);
}

}  // namespace bp

extern "C" int bp_sort_keys_u64(uint64_t* d_keys, uint32_t* d_vals, int64_t n, int32_t key_bits, bp_stream_t stream) {
  if (n <= 1) return BP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t* kb;
  uint32_t* vb;
  uint32_t *hist, *partials;
  BP_CUDA_TRY(bp::pool_alloc(&kb, n, s));
  BP_CUDA_TRY(bp::pool_alloc(&vb, n, s));
  BP_CUDA_TRY(bp::pool_alloc(&hist, bp::sort_hist_words(n), s));
  BP_CUDA_TRY(bp::pool_alloc(&partials, bp::sort_partials_words(n), s));
  int which = 0;
  BP_CUDA_TRY(bp::radix_sort_pairs<uint64_t>(d_keys, d_vals, kb, vb, n, nullptr, 0, key_bits, hist, partials, &which,
                                             s));
  if (which) {
    BP_CUDA_TRY(cudaMemcpyAsync(d_keys, kb, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    BP_CUDA_TRY(cudaMemcpyAsync(d_vals, vb, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  }
  cudaFreeAsync(kb, s);
  cudaFreeAsync(vb, s);
  cudaFreeAsync(hist, s);
  cudaFreeAsync(partials, s);
  return BP_OK;
}

extern "C" int bp_xor_checksum_rows(const float* d_rows, int64_t n, int32_t dim, uint64_t* d_out, bp_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  BP_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(uint64_t), s));
  if (n <= 0) return BP_OK;
  bp::k_xor_rows<<<bp::grid_for(n, 256), 256, 0, s>>>(d_rows, n, dim, (unsigned long long*)d_out);
  BP_LAUNCH_CHECK();
  return BP_OK;
}
