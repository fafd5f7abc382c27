// Internal object layouts shared by the translation units of libbagpipe_b200.
#pragma once

#include "sort.cuh"

struct bp_ctx {
  bp::ErrorRecord* d_err;
  bp::ErrorRecord* h_err;  // pinned
};

struct bp_schema {
  int32_t num_tables;
  int32_t emb_dim;
  int64_t total_rows;
  int32_t id_bits;         // bit width of total_rows - 1 (sort key width)
  int64_t* d_table_base;   // [num_tables + 1]
  int64_t* d_rows;         // [num_tables]
  int64_t* h_table_base;
};

namespace bp {

constexpr uint32_t kNoId = 0xFFFFFFFFu;
// Segments at least this long (occurrences of one key in one batch) take the
// shared-memory path of the trainer kernel (trainer.cu).
constexpr uint32_t kLongSeg = 512;
// ...and those this long are scheduled first (longest-processing-time order).
constexpr uint32_t kVeryLongSeg = 4096;
constexpr uint64_t kEmptyKey = ~0ull;

// Memory from the device's stream-ordered pool (release threshold raised at
// context creation so steady-state iterations never hit cudaMalloc).
template <typename T>
inline cudaError_t pool_alloc(T** p, size_t count, cudaStream_t s) {
  return cudaMallocAsync((void**)p, (count ? count : 1) * sizeof(T), s);
}

// GPU hash map packed key -> dense id for schema-less objects (the planner
// and cache API accept keys of any table/row without a schema).  Insert-only,
// linear probing; ids are assigned densely in call order via a scan over the
// CAS winners, so every per-key array of the owner can be indexed by id.
struct Registry {
  uint64_t* d_keys = nullptr;  // [slots]
  uint32_t* d_ids = nullptr;   // [slots]
  long long* d_count = nullptr;
  uint32_t* d_claim = nullptr;  // scratch [claim_cap]
  uint32_t* d_claim_scan = nullptr;
  uint32_t* d_partials = nullptr;
  long long claim_cap = 0;
  long long slots = 0;
  long long id_capacity = 0;
  long long count_upper = 0;
};

int registry_init(Registry* r, long long id_capacity, cudaStream_t s);
void registry_free(Registry* r, cudaStream_t s);
// Makes room for n more ids; returns 1 in *grown when id_capacity changed.
int registry_reserve(Registry* r, long long n, cudaStream_t s, int* grown);
// ids for unique keys; insert=1 registers unknown keys, insert=0 yields kNoId.
int registry_map(Registry* r, const uint64_t* d_keys, long long n, const long long* d_n, uint32_t* d_ids,
                 int insert, cudaStream_t s);

__device__ __forceinline__ uint64_t registry_hash(uint64_t key) { return splitmix64(key); }

__device__ __forceinline__ uint32_t registry_find(const uint64_t* keys, const uint32_t* ids, long long slots,
                                                  uint64_t key) {
  const uint64_t mask = (uint64_t)slots - 1;
  uint64_t h = registry_hash(key) & mask;
  for (long long probe = 0; probe < slots; ++probe) {
    const uint64_t k = keys[h];
    if (k == key) return ids[h];
    if (k == kEmptyKey) return kNoId;
    h = (h + 1) & mask;
  }
  return kNoId;
}

// The engine's per-step counter record in mapped pinned memory (engine.cu
// layout: unique, inserted, critical, dirty keys, evicted, evicted dirty,
// drained, drained dirty, then the error record), written by the last block
// of the step's eviction kernel; out == nullptr: none.
struct StepRecord {
  const unsigned long long* num_unique = nullptr;
  const long long* n_ins = nullptr;
  const unsigned long long* stats = nullptr;
  uint64_t* out = nullptr;
};

__device__ __forceinline__ void write_step_record(const StepRecord& r, long long evicted, long long evicted_dirty,
                                                  const ErrorRecord* err) {
  r.out[0] = *r.num_unique;
  r.out[1] = (uint64_t)*r.n_ins;
  r.out[2] = r.stats[0];
  r.out[3] = r.stats[1];
  r.out[4] = (uint64_t)evicted;
  r.out[5] = (uint64_t)evicted_dirty;
  r.out[6] = 0;
  r.out[7] = 0;
  constexpr int kErrWords = sizeof(ErrorRecord) / sizeof(uint64_t);
  const volatile uint64_t* ew = reinterpret_cast<const volatile uint64_t*>(err);
  for (int k = 0; k < kErrWords; ++k) r.out[8 + k] = ew ? ew[k] : 0;
  __threadfence_system();
}

int cache_evict_planned_rec(bp_cache* c, const uint64_t* d_keys, const uint32_t* d_ids, const int64_t* d_n,
                            int64_t n_max, const int64_t* d_expect, int64_t iteration, const bp_evict_buffers* o,
                            const StepRecord& rec, cudaStream_t s);
int cache_insert_sub(bp_cache* c, const uint64_t* d_keys, const uint32_t* d_ids, const float* d_rows,
                     const int64_t* d_ttls, int64_t n, const int64_t* d_n, int64_t sub, int64_t* n_out,
                     int64_t iteration, cudaStream_t s);
int mark_ids_zero(bp_prep* P, int64_t* d_mark, int64_t tag, int64_t* d_zero2, cudaStream_t s);
int apply_resolve_mark(bp_cache* c, bp_prep* P, const int64_t* d_ttl_k, uint64_t skip_key, int32_t has_skip,
                       int32_t* d_slots_s, bp_prep* N, int64_t* d_mark, int64_t tag, int64_t* d_zero2,
                       cudaStream_t s);

// Green-context SM partition (green.cu): a stream of the hot (hot != 0) or
// the rest partition, or nullptr when partitioning is off.
int green_stream(int hot, int priority, cudaStream_t* out);
bool green_link_mode();
void green_auto(int dim);
// The stub trainer's hot-key chains go to this stream when set (trainer.cu).
void set_long_stream(cudaStream_t s);
int store_log_append_fenced(bp_store* st, const uint32_t* d_ids, const float* d_rows, const uint8_t* d_dirty,
                            int64_t m, cudaStream_t s, cudaEvent_t before_commit);

// Dense id of a packed key in schema mode; kNoId if out of schema.
__device__ __forceinline__ uint32_t schema_id(const int64_t* base, const int64_t* rows, int num_tables,
                                              uint64_t key) {
  const uint32_t t = table_of(key);
  const uint64_t r = row_of(key);
  if (t >= (uint32_t)num_tables || r >= (uint64_t)rows[t]) return kNoId;
  return (uint32_t)(base[t] + (long long)r);
}

}  // namespace bp

struct bp_prep {
  bp_ctx* ctx;
  long long n_occ;
  long long iteration;
  int num_ranks;
  int flags;
  int schema_mode;
  long long* d_num_unique;
  uint64_t* d_uniq_key_s;
  uint32_t* d_uniq_id_s;
  uint64_t* d_uniq_key_k;
  uint32_t* d_perm_s2k;
  uint32_t* d_perm_k2s;
  uint32_t* d_seg_start;
  uint32_t* d_occ_pos;
  uint8_t* d_occ_label;
  uint32_t* d_occ_k;
  uint32_t* d_occ_s;       // occurrence -> key-sorted unique index (BP_PREP_OCC_SORTED)
  uint32_t* d_seg_of;      // sorted position -> key-sorted unique index (BP_PREP_OCC_SORTED)
  uint32_t* d_occ_rank;    // occurrence -> sorted position (BP_PREP_OCC_SORTED)
  long long* d_rank_bounds;
  uint32_t* d_long;        // segments with >= kLongSeg occurrences: very long ones from the
                           // front, the others from the back (capacity long_cap)
  long long* d_num_long;   // [2]: very long, long
  long long long_cap;
  long long h_num_unique;  // -1 until read back
  cudaStream_t stream;
  // one stream-ordered allocation holds every buffer above and the build
  // temporaries below (one cudaMallocAsync / cudaFreeAsync per batch)
  void* d_arena;
  void *t_ka, *t_kb;
  uint32_t *t_va, *t_vb, *t_hist, *t_head, *t_segx, *t_first_flag, *t_first_rank, *t_partials;
  // cluster columnar path: per-example first-occurrence masks and look-back
  // words, zeroed with d_num_long by one memset of zero_bytes
  uint32_t* t_ex_mask;
  unsigned long long *t_col_state, *t_tile_state;
  size_t zero_bytes;
};
