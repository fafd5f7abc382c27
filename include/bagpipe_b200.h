/*
 * bagpipe_b200.h -- C ABI of the B200-native BagPipe embedding-access path.
 *
 * The reference (embcache 0.1.0, a pure Python/numpy package) has no FFI:
 * its "plugin API" is the Python module API.  Each entry point below replaces
 * the numpy/dict body of one reference function; the Python package
 * paper_2202_12429_b200 keeps the reference's names and binds these symbols
 * with ctypes (see INTEGRATION.md for the binding a maintainer would add to
 * the reference itself).
 *
 * Conventions
 *   - Every function returns a status: BP_OK or one BP_ERR_* code.  Codes map
 *     1:1 to the reference exception classes (reference errors.py:6-77).
 *     Nothing throws across the ABI.
 *   - Pointers named d_* are device pointers (cudaMalloc / torch CUDA
 *     tensors); h_* are host pointers.  Streams are cudaStream_t passed as
 *     void*.  All work is asynchronous on the given stream unless the comment
 *     says "synchronises".
 *   - Counts that a previous kernel produced may be passed as a device
 *     pointer (d_n, int64); the matching host ``n`` is then an upper bound.
 *     Pass d_n = NULL to use ``n`` as the exact count.
 *   - Device-side contract violations (cache miss, duplicate insert, ...) are
 *     recorded in the context's bp_error_t (first error in (iteration, index)
 *     order wins) and surfaced by bp_ctx_check, which synchronises.
 *   - Keys are packed u64: (table_id << 44) | row_id (reference engine.py:117-121).
 */
#ifndef BAGPIPE_B200_H
#define BAGPIPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BP_OK 0
#define BP_ERR_CONFIG 1         /* ConfigurationError   */
#define BP_ERR_CACHE_MISS 2     /* CacheMissError(key, iteration) */
#define BP_ERR_CACHE_CAPACITY 3 /* CacheCapacityError   */
#define BP_ERR_CACHE_ORDERING 4 /* CacheOrderingError   */
#define BP_ERR_STORE_KEY 5      /* StoreKeyError        */
#define BP_ERR_STORE 6          /* StoreError           */
#define BP_ERR_ENGINE 7         /* EngineError          */
#define BP_ERR_CUDA 100         /* CUDA runtime failure */
#define BP_ERR_OOM 101          /* allocation failure   */
#define BP_ERR_INVALID 102      /* bad argument at the ABI (ConfigurationError) */

typedef void* bp_stream_t; /* cudaStream_t */

typedef struct bp_error_t {
  int32_t code; /* BP_ERR_* or 0 */
  int32_t lock;
  int64_t iteration;
  int64_t index; /* position of the offending key in the call's key order */
  uint64_t key;  /* packed key */
} bp_error_t;

typedef struct bp_ctx bp_ctx;
typedef struct bp_schema bp_schema;
typedef struct bp_prep bp_prep;
typedef struct bp_planner bp_planner;
typedef struct bp_cache bp_cache;
typedef struct bp_store bp_store;

/* ---------------------------------------------------------------- context */
const char* bp_version(void);
/* sizeof of ABI structs (0 bp_error_t, 1 bp_prep_view, 2 bp_plan_buffers,
 * 3 bp_planner_stats, 4 bp_cache_stats, 5 bp_evict_buffers, 6 bp_cache_view,
 * 7 bp_engine_config, 8 bp_step_result, 9 bp_engine_parts_t,
 * 10 bp_planner_dump_t); -1 for an unknown id. */
int64_t bp_abi_sizeof(int32_t which);
const char* bp_last_error_message(void);
int bp_ctx_create(bp_ctx** out);
int bp_ctx_destroy(bp_ctx* ctx);
/* Synchronises the stream, copies the error record out and clears it. */
int bp_ctx_check(bp_ctx* ctx, bp_stream_t stream, bp_error_t* h_out);

/* ----------------------------------------------------------------- schema
 * Schema = table cardinalities; dense id g = table_base[t] + row is monotone
 * in (table, row) and indexes every per-row array (store rows, cache slot map,
 * planner tracker).  Replaces reference traces.py:42-71 (Schema). */
int bp_schema_create(int32_t num_tables, const int64_t* h_rows_per_table, int32_t emb_dim, bp_schema** out);
int bp_schema_destroy(bp_schema* schema);
int64_t bp_schema_total_rows(const bp_schema* schema);

/* ------------------------------------------------------------ batch prep
 * Replaces Batch.unique_keys (reference traces.py:91-103) and _prep_batch
 * (reference engine.py:142-182): dedupe in first-occurrence order, key-sorted
 * unique order, per-key occurrence lists in occurrence order (the order of
 * np.add.at), per-occurrence labels and trainer-rank bounds.
 * schema may be NULL (registry mode: keys of any table/row; ids are then
 * assigned by the consumer objects).  d_keys/d_labels: n_occ entries, device.
 * h_rank_bounds: num_ranks+1 occurrence positions (rank r owns
 * [b[r], b[r+1])).  flags: BP_PREP_OCC_INDEX also materialises the
 * occurrence -> unique (first-occurrence index) map.  row_bits/table_bits
 * (registry mode only): bit widths of the largest row / table id, so the
 * sort runs only over live key bits. */
#define BP_PREP_OCC_INDEX 1
#define BP_PREP_OCC_SORTED 2 /* occurrence -> key-sorted unique index (EmbeddingBag gather) */
int bp_prep_create(bp_ctx* ctx, const bp_schema* schema, const uint64_t* d_keys, const uint8_t* d_labels,
                   int64_t n_occ, const int64_t* h_rank_bounds, int32_t num_ranks, int64_t iteration,
                   int32_t flags, int32_t row_bits, int32_t table_bits, bp_stream_t stream, bp_prep** out);
int bp_prep_destroy(bp_prep* prep);
/* Columnar batch (schema mode): keys laid out [n_ex][n_cols], every example
 * holding one key of table d_tables[c] (device, strictly increasing) in
 * column c -- the Criteo layout.  A key then occurs in one column only, so
 * the prep sorts each column in one CTA's shared memory (n_ex <= 16384;
 * larger batches take the generic path).  Output identical to bp_prep_create. */
int bp_prep_create_columnar(bp_ctx* ctx, const bp_schema* schema, const uint64_t* d_keys, const uint8_t* d_labels,
                            int64_t n_ex, int32_t n_cols, const int32_t* d_tables, const int64_t* h_rank_bounds,
                            int32_t num_ranks, int64_t iteration, int32_t flags, bp_stream_t stream, bp_prep** out);

typedef struct bp_prep_view {
  int64_t n_occ;
  int64_t iteration;
  int32_t num_ranks;
  int32_t pad;
  const int64_t* d_num_unique;   /* device scalar U */
  const uint64_t* d_uniq_key_s;  /* [U] unique keys, key-sorted        */
  const uint32_t* d_uniq_id_s;   /* [U] dense ids g (schema mode)      */
  const uint64_t* d_uniq_key_k;  /* [U] unique keys, first-occurrence order */
  const uint32_t* d_perm_s2k;    /* [U] sorted index -> first-occurrence index */
  const uint32_t* d_perm_k2s;    /* [U] first-occurrence index -> sorted index */
  const uint32_t* d_seg_start;   /* [U+1] CSR offsets (sorted order) into d_occ_pos */
  const uint32_t* d_occ_pos;     /* [n_occ] occurrence positions grouped by key, ascending */
  const uint8_t* d_occ_label;    /* [n_occ] label of d_occ_pos[j] */
  const uint32_t* d_occ_k;       /* [n_occ] occurrence -> first-occurrence unique index (flag) */
  const int64_t* d_rank_bounds;  /* [num_ranks+1] */
} bp_prep_view;
int bp_prep_get_view(const bp_prep* prep, bp_prep_view* out);
/* Synchronises; host copy of U. */
int bp_prep_num_unique(bp_prep* prep, bp_stream_t stream, int64_t* h_out);

/* ---------------------------------------------------------------- planner
 * Oracle Cacher state (reference lookahead.py:38-123).  The window queue and
 * lookahead/halving decisions stay on the host (they are scalar); per-key
 * state (latest_tracker, in_cache mirror) is device-resident.
 * schema NULL => registry mode (GPU hash map key -> dense id). */
int bp_planner_create(bp_ctx* ctx, const bp_schema* schema, int64_t capacity, bp_planner** out);
int bp_planner_destroy(bp_planner* planner);
/* emit_next_plan refill step for one appended batch: tracker[e] = iteration
 * for every unique key (reference lookahead.py:75-82). */
int bp_planner_refill(bp_planner* planner, bp_prep* prep, bp_stream_t stream);

typedef struct bp_plan_buffers {
  /* caller-allocated device buffers with room for U entries each */
  uint64_t* d_prefetch_keys;  /* sorted by key */
  uint32_t* d_prefetch_ids;   /* dense ids of the above (schema mode) */
  int64_t* d_prefetch_ttls;   /* ttl of each prefetched key */
  int64_t* d_ttl_k;           /* ttl per unique key, first-occurrence order */
  uint64_t* d_evict_keys;     /* planner's evict set {e : ttl == iteration}, sorted */
  uint32_t* d_evict_ids;      /* dense ids of the above (may be NULL) */
  int64_t* d_counts;          /* [5]: n_prefetch, n_evict, projected, resident_before, resident_after */
} bp_plan_buffers;

typedef struct bp_planner_stats {
  int64_t tracked;          /* len(latest_tracker) == projected occupancy */
  int64_t in_cache;         /* len(in_cache) */
  int64_t insertions;
  int64_t removals;
  int64_t peak_occupancy;
  int64_t peak_projected;
  int64_t last_projected;   /* projected occupancy recorded by the last pop */
  int64_t last_prefetch;
  int64_t last_evict;
  int64_t registry_size;
} bp_planner_stats;

/* Pop step of emit_next_plan for the front batch (reference lookahead.py:84-110):
 * records projected occupancy, assigns TTLs, prefetch/mirror, erases keys whose
 * last windowed use is this batch.  Writes the plan into *bufs. */
int bp_planner_pop(bp_planner* planner, bp_prep* prep, const bp_plan_buffers* bufs, bp_stream_t stream);
/* Enumerate keys with planner state (tracked and/or mirrored), arbitrary
 * order: flags bit0 = in latest_tracker, bit1 = in the in_cache mirror.
 * *d_count receives the total (entries beyond cap are dropped). */
typedef struct bp_planner_dump_t {
  uint64_t* d_keys;
  int64_t* d_last;
  uint8_t* d_flags;
  int64_t* d_count;
} bp_planner_dump_t;
int bp_planner_dump(bp_planner* planner, const bp_planner_dump_t* out, int64_t cap, bp_stream_t stream);
/* Synchronises. */
int bp_planner_get_stats(bp_planner* planner, bp_stream_t stream, bp_planner_stats* h_out);

/* ------------------------------------------------------------------ cache
 * Trainer TTL cache in HBM (reference cache.py:31-286): dense id -> slot map,
 * row arena [capacity, dim] f32, ttl/dirty/used per slot, LIFO free list
 * (lowest freed slot reused first, like reference cache.py:209-210). */
int bp_cache_create(bp_ctx* ctx, const bp_schema* schema, int64_t capacity, int32_t dim, bp_cache** out);
int bp_cache_destroy(bp_cache* cache);

typedef struct bp_cache_stats {
  int64_t occupancy;
  int64_t insertions;
  int64_t evictions;
  int64_t peak_occupancy;
  int64_t capacity;
  int64_t registry_size;
} bp_cache_stats;
int bp_cache_get_stats(bp_cache* cache, bp_stream_t stream, bp_cache_stats* h_out); /* synchronises */

/* apply_prefetch (reference cache.py:99-136): insert clean rows with TTLs.
 * d_ids may be NULL (ids derived from keys).  Duplicate -> CACHE_ORDERING.
 * Capacity is checked on the device too (CACHE_CAPACITY). */
int bp_cache_insert(bp_cache* cache, const uint64_t* d_keys, const uint32_t* d_ids, const float* d_rows,
                    const int64_t* d_ttls, int64_t n, const int64_t* d_n, int64_t iteration, bp_stream_t stream);
/* apply_ttl_updates (reference cache.py:138-149); absent key -> CACHE_ORDERING. */
int bp_cache_set_ttl(bp_cache* cache, const uint64_t* d_keys, const uint32_t* d_ids, const int64_t* d_ttls,
                     int64_t n, const int64_t* d_n, int64_t iteration, bp_stream_t stream);
/* resolve_slots (reference cache.py:151-164); miss -> CACHE_MISS(key, iteration),
 * first missing key in the given order.  Missing entries get slot -1. */
int bp_cache_resolve(bp_cache* cache, const uint64_t* d_keys, const uint32_t* d_ids, int64_t n,
                     const int64_t* d_n, int64_t iteration, int32_t* d_slots, bp_stream_t stream);
/* values_at (copy) and update_rows (reference cache.py:166-184). d_dirty may be NULL. */
int bp_cache_gather(bp_cache* cache, const int32_t* d_slots, int64_t n, const int64_t* d_n, float* d_out,
                    bp_stream_t stream);
int bp_cache_update(bp_cache* cache, const int32_t* d_slots, const float* d_rows, const uint8_t* d_dirty,
                    int64_t n, const int64_t* d_n, bp_stream_t stream);
/* evict_expired_arrays / drain_arrays (reference cache.py:214-242): every used
 * slot with ttl <= completed (drain: all).  Output in slot order; sorting by
 * key is bp_sort_keys.  Outputs need room for ``capacity`` entries. */
typedef struct bp_evict_buffers {
  uint64_t* d_keys;
  uint32_t* d_ids;
  float* d_rows;
  uint8_t* d_dirty;
  int64_t* d_count;  /* [2]: evicted, evicted dirty */
} bp_evict_buffers;
int bp_cache_evict(bp_cache* cache, int64_t completed, int32_t drain, const bp_evict_buffers* out,
                   int64_t out_capacity, bp_stream_t stream);
/* Engine step of reference engine.py:525-543 over a schema-mode prep: TTL
 * updates for every batch key (except skip_key when has_skip, the
 * drop_prefetch fault) then slot resolution into d_slots_s (key-sorted
 * order).  Absent TTL key -> CACHE_ORDERING; absent skipped key ->
 * CACHE_MISS (index | 1<<40 marks the resolve phase). */
int bp_cache_apply_resolve(bp_cache* cache, bp_prep* prep, const int64_t* d_ttl_k, uint64_t skip_key,
                           int32_t has_skip, int32_t* d_slots_s, bp_stream_t stream);
/* Eviction of a planned, key-sorted evict set (engine fast path): releases
 * exactly d_ids[0..*d_n) (ENGINE error if one is not resident) into *out in
 * that order, then checks the cache occupancy against *d_expect (the
 * planner mirror's size after the batch): any divergence from the
 * ttl <= iteration scan semantics of bp_cache_evict is an ENGINE error. */
int bp_cache_evict_planned(bp_cache* cache, const uint64_t* d_keys, const uint32_t* d_ids, const int64_t* d_n,
                           int64_t n_max, const int64_t* d_expect, int64_t iteration, const bp_evict_buffers* out,
                           bp_stream_t stream);
/* content_checksum (reference cache.py:249-272) into a device u64. */
int bp_cache_checksum(bp_cache* cache, uint64_t* d_out, bp_stream_t stream);
/* Raw views for inspection (device pointers). */
typedef struct bp_cache_view {
  int64_t capacity;
  int32_t dim;
  int32_t pad;
  float* d_values;
  int64_t* d_ttl;
  uint8_t* d_dirty;
  uint8_t* d_used;
  uint64_t* d_slot_key;
} bp_cache_view;
int bp_cache_get_view(const bp_cache* cache, bp_cache_view* out);

/* ------------------------------------------------------------------ store
 * Embedding Server (reference store.py:65-201): the full table lives in
 * pinned host memory, row-major in (table, row, component) order -- the
 * digest order of reference store.py:179-185.  Initial values are computed on
 * the GPU (reference store.py:29-42) and streamed to the host table. */
int bp_store_create(bp_ctx* ctx, const bp_schema* schema, uint64_t seed, bp_stream_t stream, bp_store** out);
/* As bp_store_create; components >= init_dims of every row start at 0
 * (optimizer state stored beside the weights). */
int bp_store_create_ex(bp_ctx* ctx, const bp_schema* schema, uint64_t seed, int32_t init_dims, bp_stream_t stream,
                       bp_store** out);
int bp_store_destroy(bp_store* store);
float* bp_store_host_table(bp_store* store);
uint8_t* bp_store_written_bitmap(bp_store* store); /* device, 1 bit per row */
/* fetch (reference store.py:106-129): zero-copy gather of rows g from the
 * pinned table over the host link into d_out[n, dim]. */
int bp_store_fetch(bp_store* store, const uint32_t* d_ids, int64_t n, const int64_t* d_n, float* d_out,
                   bp_stream_t stream);
/* fetch as store.py:106-129 states it: written rows (device bitmap) gathered
 * over the host link, never-written rows computed on the GPU from their
 * packed keys d_keys[i] (functional init, store.py:29-42) -- no PCIe read. */
int bp_store_fetch_lazy(bp_store* store, const uint32_t* d_ids, const uint64_t* d_keys, int64_t n,
                        const int64_t* d_n, float* d_out, bp_stream_t stream);
/* Write-back log (log-structured host store): bp_store_log_append copies a
 * chunk of rows into a pinned log by one copy-engine DMA and commits its
 * dirty rows (d_dirty NULL: all) as the newest copies of their ids; fetches
 * read a row from the log or the table, whichever is newest.  Compaction
 * (when the log is full, or explicitly before host-side reads of the table)
 * folds the newest log entries into the table.  Stream-ordered. */
int bp_store_enable_log(bp_store* store, int64_t log_rows, bp_stream_t stream);
int bp_store_log_append(bp_store* store, const uint32_t* d_ids, const float* d_rows, const uint8_t* d_dirty,
                        int64_t m, bp_stream_t stream);
int bp_store_compact(bp_store* store, bp_stream_t stream);
int64_t bp_store_log_rows(bp_store* store); /* capacity, 0 = no log */
/* lazy-fetch counters since creation: [0] rows read over the host link,
 * [1] rows computed on the GPU.  Synchronises the device. */
int bp_store_link_counters(bp_store* store, int64_t* h_out2);
/* write_back (reference store.py:131-155): zero-copy scatter into the
 * pinned table; ids must be unique within one call. */
int bp_store_write(bp_store* store, const uint32_t* d_ids, const float* d_rows, int64_t n,
                   const int64_t* d_n, bp_stream_t stream);
/* write_back of only the masked (dirty) rows of an eviction chunk. */
int bp_store_write_masked(bp_store* store, const uint32_t* d_ids, const float* d_rows, const uint8_t* d_mask,
                          int64_t n, const int64_t* d_n, bp_stream_t stream);
/* initial_values (reference store.py:29-42) for arbitrary packed keys. */
int bp_init_values(uint64_t seed, int32_t dim, const uint64_t* d_keys, int64_t n, float* d_out,
                   bp_stream_t stream);
/* dense ids for packed keys (schema mode); out-of-schema -> STORE_KEY. */
int bp_schema_ids(bp_ctx* ctx, const bp_schema* schema, const uint64_t* d_keys, int64_t n, uint32_t* d_ids,
                  bp_stream_t stream);

/* ---------------------------------------------------------------- trainer
 * Fused stub backward + rank-ordered combine + SGD (reference trainer.py:37-53,
 * 92-105, 140-146; engine.py:545-579).  For every unique key (sorted order s)
 * the kernel walks the key's occurrences in occurrence order: per rank
 * G_r = ((0 + g_1) + g_2) + ... with g = c_value*v + c_label*(label - 0.5),
 * then combined = ((0 + G_r0) + G_r1) + ... in ascending rank, exactly the
 * association of np.add.at.  mode BP_STUB_SGD updates rows in place
 * (v - lr*combined) and sets dirty where combined != 0; mode BP_STUB_GRAD
 * writes combined to d_grad_out[s] instead.
 * d_rows: row arena; d_row_index: row of sorted unique s (NULL = s itself).
 * d_next_mark/next_tag: optional dense per-id array in which bp_mark_ids
 * stamped the next batch's ids with next_tag: keys found there are counted
 * as critical (reference engine.py:560-569) into d_stats[0]; keys whose
 * combined gradient is non-zero are counted into d_stats[1].  Labels must
 * be < 128 (bit 7 of the prep's label bytes flags trainer-rank starts). */
#define BP_STUB_SGD 0
#define BP_STUB_GRAD 1
int bp_stub_step(bp_ctx* ctx, bp_prep* prep, float* d_rows, const int32_t* d_row_index, uint8_t* d_dirty,
                 int32_t dim, float c_value, float c_label, float lr, int32_t mode, float* d_grad_out,
                 const int64_t* d_next_mark, int64_t next_tag, int64_t* d_stats, bp_stream_t stream);
/* bp_stub_step runs its long-segment kernel on a side stream of the calling
 * thread, concurrently with the short-segment kernel (1, default) or both on
 * `stream` in sequence (0). */
/* Tuning: CTAs per SM of the short-segment stub trainer kernel (1..6,
 * default 5: one slot per SM stays free for the long-segment kernel). */
int bp_set_stub_short_ctas(int32_t per_sm);
/* Tuning: preferred shared-memory carveout (%) of the short-segment kernel
 * (default 100; -1 = driver default).  Set before the first bp_stub_step. */
int bp_set_stub_carveout(int32_t percent);
/* Tuning: threads per long-segment (hot-key chain) CTA, 64..1024 (default 1024). */
int bp_set_stub_long_threads(int32_t threads);
/* Dynamic shared memory of a hot-key chain CTA (its SM's room for short-kernel
 * CTAs): bytes, default 120 KB. */
int bp_set_stub_long_smem(int32_t bytes);
/* Tuning: green-context SM partition of engines created afterwards: its
 * small part of `sms` SMs (rounded up by the driver to its split
 * granularity, 8 on B200; bp_green_info reports the result) runs the
 * host-link streams (bp_set_green_link 1, the default) or the stub trainer's
 * hot-key chains (0), every other engine stream the rest.  0 = off; -1
 * (default) = 8 SMs per 32 row components, at most 16. */
int bp_set_green_sms(int32_t sms);
/* {hot-partition SMs, rest SMs} of the partition in use ({0, 0} when off). */
int bp_green_info(int32_t* out2);
/* With a green partition (bp_set_green_sms): 1 = its small part runs the
 * engine's host-link streams instead of the hot-key chains. */
int bp_set_green_link(int32_t on);
/* Trainer stub stream layout: 0 = one stream; 1 = hot-key chains on a side
 * stream; 2 (default) = chains first on the caller's stream, short kernel on
 * the side stream. */
int bp_set_stub_fork(int32_t mode);
/* Engine write-back (link mode 0, log): 1 (default) = row DMA on its own
 * stream, overlapping the prefetch reads; 0 = on the link stream. */
int bp_set_split_writeback(int32_t on);
/* mark[id] = tag for every unique key of a schema-mode prep. */
int bp_mark_ids(bp_prep* prep, int64_t* d_mark, int64_t tag, bp_stream_t stream);
/* np.add.at(out, idx, vals) row-wise in input order, over a registry-mode
 * prep built from keys = idx (combine_core, reference trainer.py:92-105).
 * d_out rows absent from idx are left untouched. */
int bp_add_at_rows(bp_prep* prep, const float* d_vals, int32_t dim, float* d_out, bp_stream_t stream);
/* row index (low 44 bits) of each key-sorted unique key, as int32. */
int bp_prep_key_rows(bp_prep* prep, int32_t* d_out, bp_stream_t stream);
/* sgd_step (reference trainer.py:140-146): out = v - lr*g, single precision. */
int bp_sgd(const float* d_values, const float* d_grads, float lr, int64_t count, float* d_out, bp_stream_t stream);

/* ----------------------------------------------------------------- engine
 * Native runtime of the pipelined iteration (reference engine.py:487-649):
 * owns the store, cache, planner, two streams (compute, host link) and every
 * per-iteration buffer (plan / staging / chunk rings), so one iteration is a
 * handful of calls and no allocation.  The host keeps the scalar control
 * flow (window, gate, flush cadence, simulated clock) and drives:
 *   add_batch -> refill/pop -> fetch -> train -> flush -> release_batch. */
typedef struct bp_engine bp_engine;
typedef struct bp_engine_config {
  int64_t capacity;   /* cache entries */
  int64_t max_occ;    /* largest batch (occurrences) */
  uint64_t seed;      /* store seed */
  int32_t dim;
  int32_t num_ranks;  /* data-parallel trainers T (combine order) */
  float c_value, c_label, lr;
  int32_t record_keys; /* keep evicted keys for event logs */
  int32_t plan_slots, chunk_slots, prep_slots;
  int32_t timing;      /* record per-stage CUDA events (bp_engine_stage_times) */
  int32_t init_dims;   /* store: components >= init_dims start at 0 (0 = all initialised) */
  int32_t prep_flags;  /* BP_PREP_* for every batch prep (BP_PREP_OCC_SORTED in DLRM mode) */
} bp_engine_config;
typedef struct bp_step_result {
  int64_t unique, inserted, critical, dirty_keys, evicted, evicted_dirty, drained, drained_dirty;
  bp_error_t err;
} bp_step_result;
typedef struct bp_engine_parts_t {
  bp_store* store;
  bp_cache* cache;
  bp_planner* planner;
  bp_stream_t compute_stream;
  bp_stream_t link_stream;
} bp_engine_parts_t;
int bp_engine_create(bp_ctx* ctx, const bp_schema* schema, const bp_engine_config* cfg, bp_engine** out);
int bp_engine_destroy(bp_engine* engine);
int bp_engine_parts(bp_engine* engine, bp_engine_parts_t* out);
/* keys/labels: host pointers (keys_on_host=1: copied into a pinned ring by
 * the engine's upload worker thread, asynchronously -- they must stay valid
 * until bp_engine_release_batch of that position) or device pointers that
 * stay valid until the prep kernels ran. */
int bp_engine_add_batch(bp_engine* engine, int64_t pos, int64_t iteration, const uint64_t* keys,
                        const uint8_t* labels, int64_t n_occ, const int64_t* h_rank_bounds, int32_t num_ranks,
                        int32_t keys_on_host);
int bp_engine_add_batch_columnar(bp_engine* engine, int64_t pos, int64_t iteration, const uint64_t* keys,
                                 const uint8_t* labels, int64_t n_ex, int32_t n_cols, const int32_t* h_tables,
                                 const int64_t* h_rank_bounds, int32_t num_ranks, int32_t keys_on_host);
/* Compact columnar batch entering the window (reference Batch.rows /
 * Batch.labels of a Criteo-layout batch, traces.py): the row ids of the
 * tables h_tables[n_cols] as planes of u32, u16 and u8 columns (h_widths[c]
 * = 4, 2 or 1; planes [n_ex][n_w] in that order in one buffer) and one label
 * per example; expanded to packed keys + occurrence labels on the prep
 * stream.  on_host: planes and ex_labels are pinned host memory (DMA'd),
 * else device memory.  n_cols <= 64. */
int bp_engine_add_batch_packed(bp_engine* e, int64_t pos, int64_t iteration, const void* planes,
                               const uint8_t* ex_labels, int64_t n_ex, int32_t n_cols, const int32_t* h_tables,
                               const int8_t* h_widths, const int64_t* h_rank_bounds, int32_t num_ranks,
                               int32_t on_host);
int bp_engine_prep(bp_engine* engine, int64_t pos, bp_prep** out);
int bp_engine_release_batch(bp_engine* engine, int64_t pos);
int bp_engine_refill(bp_engine* engine, int64_t pos);
int bp_engine_pop(bp_engine* engine, int64_t pos, int32_t* slot_out);
int bp_engine_plan_counts(bp_engine* engine, int32_t slot, int64_t* h_out4); /* waits for that pop */
int bp_engine_plan_ready(bp_engine* engine, int32_t slot, int32_t* out);      /* non-blocking query */
int bp_engine_plan_view(bp_engine* engine, int32_t slot, bp_plan_buffers* out, float** d_staging);
int bp_engine_fetch(bp_engine* engine, int32_t slot);
/* Host-link mode: 0 = zero-copy row kernels, 1 = copy engines + `threads`
 * host threads gathering/scattering rows in pinned staging (0: auto),
 * 2 = zero-copy prefetch, copy-engine write-back + host scatter. */
int bp_engine_set_link_mode(bp_engine* engine, int32_t mode, int32_t threads);
/* Link gate (DLRM mode): each prefetch waits for the latest EmbeddingBag
 * forward enqueued before it, so its host-link reads overlap the dense step
 * rather than the embedding kernels (deadlock-free: everything waiting on a
 * fetch is enqueued after it). */
int bp_engine_set_link_gate(bp_engine* engine, int32_t on);
/* Enable the store's write-back log (mode 0 flushes append to it by DMA). */
int bp_engine_set_write_log(bp_engine* engine, int64_t log_rows);
/* Host worker-pool row gather (op 0) / scatter (op 1) rate probe (tools). */
int bp_host_rows_bench(float* table, int32_t dim, const uint32_t* ids, int64_t n, int32_t threads, int32_t op,
                       double* seconds);
int bp_engine_flush(bp_engine* engine, const int32_t* h_chunk_slots, int32_t n);
int bp_engine_train(bp_engine* engine, int64_t pos, int32_t plan_slot, int64_t next_pos, uint64_t skip_key,
                    int32_t has_skip, int32_t chunk_slot, int32_t drain_slot, bp_step_result* out);
/* The same iteration split in two: _begin enqueues it (no host wait), _end
 * waits for it and fills ``out``; the host can emit plans in between. */
int bp_engine_train_begin(bp_engine* engine, int64_t pos, int32_t plan_slot, int64_t next_pos, uint64_t skip_key,
                          int32_t has_skip, int32_t chunk_slot, int32_t drain_slot);
int bp_engine_train_end(bp_engine* engine, bp_step_result* out);
/* DLRM mode iteration, split around the (PyTorch) dense model:
 * forward = apply plan + lookup + next-batch stamp + EmbeddingBag forward of
 * the batch's single-key bags into d_pooled[n_occ][model_dim] (async on the
 * compute stream); backward = EmbeddingBag backward + optimizer in place +
 * eviction (+ drain), counters, one synchronisation (like bp_engine_train). */
int bp_engine_dlrm_forward(bp_engine* engine, int64_t pos, int32_t plan_slot, int64_t next_pos, uint64_t skip_key,
                           int32_t has_skip, int32_t model_dim, float* d_pooled);
int bp_engine_dlrm_backward(bp_engine* engine, int64_t pos, int32_t plan_slot, const float* d_grad,
                            int32_t model_dim, int32_t opt, float lr, float eps, int32_t chunk_slot,
                            int32_t drain_slot, bp_step_result* out);
/* Sorted-gradient backward (no reference counterpart; DLRM mode): the dense
 * model stores the pooled-row gradient of occurrence p at row d_rows[p] (from
 * bp_engine_dlrm_grad_rows: the key-sorted position, bp_prep_occ_rank), and
 * the EmbeddingBag backward streams it (bp_embbag_backward_sorted). */
int bp_engine_dlrm_grad_rows(bp_engine* engine, int64_t pos, uint32_t* d_rows);
int bp_engine_dlrm_backward_sorted(bp_engine* engine, int64_t pos, int32_t plan_slot, const float* d_grad_sorted,
                                   int32_t model_dim, int32_t opt, float lr, float eps, int32_t chunk_slot,
                                   int32_t drain_slot, bp_step_result* out);
/* Asynchronous form of the DLRM backward (either gradient order): enqueues
 * only; bp_engine_train_end waits for the iteration and reads its counters. */
int bp_engine_dlrm_backward_begin(bp_engine* engine, int64_t pos, int32_t plan_slot, const float* d_grad,
                                  int32_t grad_sorted, int32_t model_dim, int32_t opt, float lr, float eps,
                                  int32_t chunk_slot, int32_t drain_slot);
int bp_engine_chunk_keys(bp_engine* engine, int32_t chunk_slot, uint64_t* h_out, int64_t n);
int bp_engine_chunk_view(bp_engine* engine, int32_t chunk_slot, bp_evict_buffers* out);
int bp_engine_sync(bp_engine* engine);
/* Make `stream` wait for all work issued so far on the engine's streams
 * (compute, plan, host-link) without blocking the host. */
int bp_engine_join(bp_engine* engine, bp_stream_t stream);
/* Per-stage event timing on/off (bp_engine_stage_times). */
int bp_engine_set_timing(bp_engine* engine, int32_t on);
/* Benchmarks: every iteration first writes `bytes` (> L2) of d_buf on the
 * compute stream; exclusive != 0 fences the plan and host-link streams
 * around the write.  d_buf = NULL disables. */
int bp_engine_set_l2_flush(bp_engine* engine, void* d_buf, int64_t bytes, int32_t exclusive);
/* Per-stage device time since the last call, 8 stages: prep, planner, fetch
 * (link), apply (insert+TTL+lookup+mark), trainer (stub trainer or DLRM
 * EmbeddingBag forward), evict, flush (link), trainer_bwd (DLRM EmbeddingBag
 * backward + optimizer).  Synchronises the device. */
int bp_engine_stage_times(bp_engine* engine, double* h_ms8, int64_t* h_counts8);

/* ------------------------------------------------------- EmbeddingBag (DLRM)
 * North-star piece 4 (no reference counterpart: parity vs a PyTorch fp32 CPU
 * model within tolerance).  Rows are read from a row arena (the cache) with
 * row_stride >= dim; optimizer state (Adagrad) sits at [dim, 2*dim).
 * forward: d_bag_offsets NULL => one occurrence per bag (bag = occurrence
 * position, Criteo layout): pooled row p = cached row of occurrence p;
 * otherwise bags [off[b], off[b+1]) of occurrences are summed (mode 1: mean).
 * Both read the occurrence -> unique map d_occ_s (BP_PREP_OCC_SORTED prep,
 * or bp_prep_occ_sorted_index).
 * backward: per unique key g = sum of its occurrences' bag gradients
 * (x d_bag_scale[bag] if given), then SGD or Adagrad in place; dirty marks
 * rows with g != 0; d_stats[1] += number of such keys. */
#define BP_OPT_SGD 0
#define BP_OPT_ADAGRAD 1
int bp_embbag_forward(bp_prep* prep, const float* d_values, int32_t row_stride, const int32_t* d_slots_s,
                      int32_t dim, const int64_t* d_bag_offsets, int64_t n_bags, int32_t mode,
                      const uint32_t* d_occ_s, float* d_out, bp_stream_t stream);
int bp_embbag_backward(bp_prep* prep, const float* d_grad, const int64_t* d_occ_bag, const float* d_bag_scale,
                       float* d_values, int32_t row_stride, const int32_t* d_slots_s, uint8_t* d_dirty, int32_t dim,
                       int32_t opt, float lr, float eps, int64_t* d_stats, bp_stream_t stream);
int bp_prep_occ_sorted_index(bp_prep* prep, uint32_t* d_occ_s, bp_stream_t stream);
/* d_out[p] = key-sorted position of occurrence p (BP_PREP_OCC_SORTED prep). */
int bp_prep_occ_rank(bp_prep* prep, uint32_t* d_out, bp_stream_t stream);
/* backward over gradient rows already in key-sorted order (row j = gradient
 * of sorted occurrence j): dim in {4, 8, 16, 32}; same update as
 * bp_embbag_backward, summation order fixed by the data. */
int bp_embbag_backward_sorted(bp_prep* prep, const float* d_grad_sorted, float* d_values, int32_t row_stride,
                              const int32_t* d_slots_s, uint8_t* d_dirty, int32_t dim, int32_t opt, float lr,
                              float eps, int64_t* d_stats, bp_stream_t stream);
/* The same with a caller-owned scratch of bp_embbag_bwd_scratch_bytes(n_occ,
 * dim) bytes, zeroed once (kept zero between calls): no per-call allocation. */
int64_t bp_embbag_bwd_scratch_bytes(int64_t n_occ, int32_t dim);
int bp_embbag_backward_sorted_scratch(bp_prep* prep, const float* d_grad_sorted, float* d_values, int32_t row_stride,
                                      const int32_t* d_slots_s, uint8_t* d_dirty, int32_t dim, int32_t opt, float lr,
                                      float eps, int64_t* d_stats, void* d_scratch, int64_t scratch_bytes,
                                      bp_stream_t stream);

/* ---------------------------------------------------------- peer exchange */
/* DLRM hybrid parallelism over NVLink peer memory (csrc/peer.cu).  Rank
 * `rank` of `world` owns the embedding columns d_col_tables[0..n_cols)
 * (global table ids) of a global batch of world * bl examples, occurrences
 * example-major ([B][n_cols]).  Example owner q holds, for its bl examples,
 * a [bl][t_global][dim] f32 row buffer that every rank addresses through
 * d_peer_rows[q] (CUDA IPC); d_peer_flags[q] is q's flag array ([world]
 * u32), d_flags this rank's own.  The forward stores pooled rows into the
 * example owners' buffers, the backward loads gradient rows from them. */
#define BP_IPC_HANDLE_BYTES 64
typedef struct bp_peer_xchg {
  int32_t world;
  int32_t rank;
  int64_t bl;
  int32_t t_global;
  int32_t n_cols;
  const int32_t* d_col_tables;
  float* const* d_peer_rows;
  uint32_t* const* d_peer_flags;
  uint32_t* d_flags;
} bp_peer_xchg;
int bp_ipc_alloc(int64_t bytes, void** d_ptr, uint8_t* handle); /* zeroed cudaMalloc + IPC handle */
int bp_ipc_open(const uint8_t* handle, void** d_ptr);
int bp_ipc_close(void* d_ptr);
int bp_ipc_free(void* d_ptr);
/* All ranks: store `epoch` into every peer's flags (after a system fence),
 * wait until every rank's flag here reached it (bounded: ENGINE error in the
 * context instead of a hang). */
int bp_peer_barrier(bp_ctx* ctx, const bp_peer_xchg* x, uint32_t epoch, bp_stream_t stream);
/* EmbeddingBag forward of single-key bags straight into the example owners'
 * row buffers (d_peer_rows of `rows`). */
/* The peer backward through the key-sorted path: the rank's gradient rows
 * pulled over NVLink into key-sorted order in d_sorted (n_occ * dim floats),
 * then the staged sorted backward (d_scratch: bp_embbag_bwd_scratch_bytes,
 * zeroed once). */
int bp_embbag_backward_peer_sorted(bp_prep* prep, const bp_peer_xchg* grads, float scale, float* d_values,
                                   int32_t row_stride, const int32_t* d_slots_s, uint8_t* d_dirty, int32_t dim,
                                   int32_t opt, float lr, float eps, int64_t* d_stats, float* d_sorted,
                                   void* d_scratch, int64_t scratch_bytes, bp_stream_t stream);
/* Engine peer backward: 1 (default) = the key-sorted path above, 0 = the
 * reduce-by-key gather straight from the peers' buffers. */
int bp_set_peer_sorted(int32_t on);
int bp_embbag_forward_peer(bp_prep* prep, const float* d_values, int32_t row_stride, const int32_t* d_slots_s,
                           int32_t dim, const bp_peer_xchg* rows, bp_stream_t stream);
/* EmbeddingBag backward + optimizer reading each occurrence's gradient row
 * from the example owner's buffer (d_peer_rows of `grads`) times `scale`. */
int bp_embbag_backward_peer(bp_prep* prep, const bp_peer_xchg* grads, float scale, float* d_values,
                            int32_t row_stride, const int32_t* d_slots_s, uint8_t* d_dirty, int32_t dim, int32_t opt,
                            float lr, float eps, int64_t* d_stats, bp_stream_t stream);
/* Engine DLRM iteration with the peer exchange: forward = apply + lookup +
 * bp_embbag_forward_peer into `rows`; backward = bp_embbag_backward_peer from
 * `grads` (x scale) + eviction + counters (synchronises like
 * bp_engine_dlrm_backward).  The caller runs the barriers. */
int bp_engine_dlrm_forward_peer(bp_engine* engine, int64_t pos, int32_t plan_slot, int64_t next_pos,
                                uint64_t skip_key, int32_t has_skip, int32_t model_dim, const bp_peer_xchg* rows);
int bp_engine_dlrm_backward_peer(bp_engine* engine, int64_t pos, int32_t plan_slot, const bp_peer_xchg* grads,
                                 float scale, int32_t model_dim, int32_t opt, float lr, float eps,
                                 int32_t chunk_slot, int32_t drain_slot, bp_step_result* out);
/* Asynchronous form: enqueue only; bp_engine_train_end reads the counters. */
int bp_engine_dlrm_backward_peer_begin(bp_engine* engine, int64_t pos, int32_t plan_slot, const bp_peer_xchg* grads,
                                       float scale, int32_t model_dim, int32_t opt, float lr, float eps,
                                       int32_t chunk_slot, int32_t drain_slot);

/* DLRM feature interaction (dense-model side of DLRM mode; the reference has
 * no model).  z = [x; emb_0..emb_{T-1}] per sample (T+1 vectors of D);
 * out row = [x | z_i . z_j, i > j, torch.tril_indices(T+1, T+1, -1) order |
 * zeros up to out_stride].  x / out / gout / gx are bf16 when the flag is
 * set, else f32; emb and gemb are f32; fp32 arithmetic.  backward:
 * gx = gout[:, :D] + (G z)_0, gemb_t = (G z)_{t+1}, G the symmetric pair
 * gradient.  T <= 127, D <= 256. */
int bp_dlrm_interact_forward(const void* d_x, int32_t x_bf16, const float* d_emb, int64_t B, int32_t T, int32_t D,
                             void* d_out, int32_t out_bf16, int32_t out_stride, bp_stream_t stream);
int bp_dlrm_interact_backward(const void* d_x, int32_t x_bf16, const float* d_emb, const void* d_gout, int32_t g_bf16,
                              int64_t B, int32_t T, int32_t D, int32_t out_stride, void* d_gx, float* d_gemb,
                              bp_stream_t stream);
/* As bp_dlrm_interact_backward, with gemb row of (b, t) = d_gemb_rows[b*T + t]
 * (NULL: b*T + t), e.g. the EmbeddingBag's key-sorted order. */
int bp_dlrm_interact_backward_rows(const void* d_x, int32_t x_bf16, const float* d_emb, const void* d_gout,
                                   int32_t g_bf16, int64_t B, int32_t T, int32_t D, int32_t out_stride, void* d_gx,
                                   float* d_gemb, const uint32_t* d_gemb_rows, bp_stream_t stream);
/* Mixed-precision SGD of the dense model in one launch: for each tensor k,
 * master[k] -= lr * grad[k] (bf16 gradient, fp32 master), then lowp[k] =
 * bf16(master[k]).  The table is read at launch (CUDA-graph capturable). */
#define BP_SGD_MAX_TENSORS 32
typedef struct bp_sgd_tensors {
  int32_t n;
  int32_t pad;
  float* master[BP_SGD_MAX_TENSORS];
  void* lowp[BP_SGD_MAX_TENSORS];       /* bf16 */
  const void* grad[BP_SGD_MAX_TENSORS]; /* bf16 */
  int64_t numel[BP_SGD_MAX_TENSORS];
} bp_sgd_tensors;
int bp_dlrm_master_sgd(const bp_sgd_tensors* tensors, float lr, bp_stream_t stream);

/* --------------------------------------------------------- trace ingest */
/* EMTRC1 records -> device batch columns (replaces the per-record decode of
 * reference traces.py:231-296, iter_trace / read_trace).  d_records holds n
 * packed records "<B{num_dense}f{num_tables}Q" (the bytes after the
 * header); outputs: d_keys[n*T] packed (t << 44 | row) in occurrence order,
 * d_occ_labels[n*T] (the label of each occurrence), d_labels[n] and
 * d_dense[n*D] (either may be NULL). */
int bp_trace_decode(const uint8_t* d_records, int64_t n, int32_t num_dense, int32_t num_tables, uint64_t* d_keys,
                    uint8_t* d_occ_labels, uint8_t* d_labels, float* d_dense, bp_stream_t stream);

/* ------------------------------------------------------------ utilities */
/* Debug: per-CTA phase clock64() stamps of the long-segment trainer kernel
 * into d_buf[148][8] (NULL disables; tools/kernel_bench.py --trace). */
int bp_debug_long_trace(void* d_buf);
/* Debug: launch shape of bp_embbag_backward_sorted (-1 = default = 9, the
 * register-resident reduce + update; 0 = the staged one-kernel form; 1-8 the
 * other measured shapes, tools/kernel_bench.py). */
int bp_debug_bwd_variant(int32_t variant);
/* Debug: EmbeddingBag single-key forward shape (0 occurrence-order gather, 1 key-sorted scatter). */
int bp_debug_fwd_variant(int32_t variant);
/* Debug: columnar batch prep on thread-block clusters (1, default) or the
 * per-column single-CTA sort (0); outputs are identical. */
int bp_debug_prep_cluster(int32_t on);
/* Tuning: smallest items per thread of the cluster prep (4, 8 default, 16). */
int bp_debug_prep_shape(int32_t ipt_min);
/* Debug: %globaltimer phase stamps of one kernel into d_buf (NULL disables):
 * which 0 = the cluster prep [column][16 CTAs][16], 1 = the fused planner pop
 * [tile][8] (tools/planner_bench.py --trace). */
int bp_debug_phase_trace(int32_t which, void* d_buf);
int bp_debug_pop_trace(void* d_buf);
/* Debug: bit 0 turns the store's fetch kernels, bit 1 its write kernels into
 * no-ops (results become wrong; only for measuring the host link's share). */
int bp_debug_skip_link(int32_t skip);
/* Debug: {gather ns, calls, rows, scatter ns, calls, rows, upload-copy ns,
 * calls, bytes} of the host worker jobs since the previous call. */
int bp_debug_link_cb_stats(int64_t* out9);
/* Launch shape of the host-link (zero-copy fetch / write-back) kernels:
 * blocks (default 32), threads per block (256) and unused dynamic shared
 * memory per block (default 0; ~200 KB makes a link block own its SM). */
int bp_set_link_blocks(int32_t blocks);
int bp_set_link_config(int32_t blocks, int32_t threads, int32_t smem_bytes);
/* Blocks of the write-back scatter kernel (0: the link kernels' block count). */
int bp_set_write_blocks(int32_t blocks);
/* Sort packed keys ascending with a u32 payload (stable); n host-known. */
int bp_sort_keys_u64(uint64_t* d_keys, uint32_t* d_vals, int64_t n, int32_t key_bits, bp_stream_t stream);
/* Order-independent digest helpers for parity tests. */
int bp_xor_checksum_rows(const float* d_rows, int64_t n, int32_t dim, uint64_t* d_out, bp_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* BAGPIPE_B200_H */
