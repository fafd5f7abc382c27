// Oracle Cacher (Algorithm 1) on the device: reference lookahead.py:38-123.
//
// Host side keeps the scalar part (window queue length, lookahead L and its
// pressure halving).  The per-key state of LookaheadState -- latest_tracker
// (key -> last windowed iteration) and the in_cache mirror -- lives in dense
// arrays indexed by the key's dense id (schema id g, or a registry id), so
// refill and pop are conflict-free parallel passes over one batch's unique
// keys: within a batch every key is unique, so no two threads touch the
// same id.
//
//   refill(batch j):  tracker[e] = j for e in U_j                (lookahead.py:75-82)
//   pop(batch i):     projected = |tracker|  (recorded before popping)
//                     ttl(e) = tracker[e]; prefetch iff e not mirrored;
//                     erase e from tracker+mirror iff ttl == i     (lookahead.py:84-110)
//                     -- one launch, k_pop_fused
// Prefetch and evict lists are compactions over the batch's KEY-SORTED
// uniques, so plan.prefetch comes out sorted without a sort; ttl_updates are
// scattered to first-occurrence order through the prep permutation.
#include "internal.cuh"

namespace bp {

constexpr uint8_t kTracked = 1;
constexpr uint8_t kMirrored = 2;

struct PlannerCounters {
  long long tracked, in_cache, insertions, removals, peak_occupancy, peak_projected, last_projected, last_prefetch,
      last_evict, registry_size;
  long long resident_before;
};

}  // namespace bp

struct bp_planner {
  bp_ctx* ctx;
  const bp_schema* sc;
  long long capacity;
  bp::Registry reg;
  long long id_cap;
  long long* d_last;
  uint8_t* d_flags;
  bp::PlannerCounters* d_ctr;
  bp::PlannerCounters* h_ctr;  // pinned
  // scratch sized for the largest batch seen
  long long scratch_cap;
  uint32_t* d_ids;
  unsigned long long* d_pop_state;  // [2][pop_state_tiles] look-back words of k_pop_fused
  long long pop_state_tiles;
  cudaStream_t home;
};

namespace bp {

__global__ void k_refill(const uint32_t* __restrict__ ids, const long long* d_U, long long iteration,
                         long long* __restrict__ last, uint8_t* __restrict__ flags, PlannerCounters* ctr) {
  const long long U = *d_U;
  unsigned long long added = 0;
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < U; s += (long long)gridDim.x * blockDim.x) {
    const uint32_t id = ids[s];
    const uint8_t f = flags[id];
    if (!(f & kTracked)) {
      flags[id] = f | kTracked;
      ++added;
    }
    last[id] = iteration;  // appended iterations increase: plain store == tracker[e] = j
  }
  cta_add((unsigned long long*)&ctr->tracked, added);
}

// The whole pop of one batch in ONE launch (reference lookahead.py:84-110):
// per key-sorted unique s the TTL, prefetch and evict decisions, then the two
// compactions by a block scan of the (prefetch, evict) flag pair plus one
// decoupled look-back per list (prefetch comes out key-sorted, evict too).
// The CTA owning the last tile reads the totals from its inclusive prefixes
// and does the scalar bookkeeping (projected occupancy before the pop,
// counters after it) -- no memset, no one-thread kernels, no flag arrays.
constexpr int kPopThreads = 256;
constexpr int kPopIpt = 4;
constexpr int kPopTile = kPopThreads * kPopIpt;
__device__ unsigned long long* g_pop_trace = nullptr;  // debug: [tile][8] %globaltimer stamps

__device__ __forceinline__ unsigned long long pop_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kPopThreads) k_pop_fused(
    const uint32_t* __restrict__ ids, const uint32_t* __restrict__ perm_s2k, const long long* d_U,
    long long iteration, long long* __restrict__ last, uint8_t* __restrict__ flags, int64_t* __restrict__ ttl_k,
    const uint64_t* __restrict__ keys_s, uint64_t* __restrict__ pf_keys, uint32_t* __restrict__ pf_ids,
    int64_t* __restrict__ pf_ttls, uint64_t* __restrict__ ev_keys, uint32_t* __restrict__ ev_ids,
    unsigned long long* st_pf, unsigned long long* st_ev, uint32_t epoch, PlannerCounters* ctr, int64_t* counts) {
  __shared__ uint32_t sh_warp[kPopThreads / 32];
  __shared__ uint32_t sh_pfx[2];
  const long long U = *d_U;
  const long long tile = blockIdx.x;
  const long long base = tile * kPopTile;
  const long long n_tiles = U > 0 ? (U + kPopTile - 1) / kPopTile : 1;
  if (tile >= n_tiles) return;
  unsigned long long* tr = g_pop_trace ? g_pop_trace + tile * 8 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = pop_timer();
  uint32_t pf_bits = 0, ev_bits = 0;
  long long ttl[kPopIpt];
  uint32_t id[kPopIpt], k2[kPopIpt];
  uint8_t f[kPopIpt];
  // two dependent rounds of loads, each with every item in flight: the
  // stores into flags below would otherwise order each item's loads after
  // the previous item's store
#pragma unroll
  for (int q = 0; q < kPopIpt; ++q) {
    const long long s = base + (long long)threadIdx.x * kPopIpt + q;
    id[q] = s < U ? __ldg(ids + s) : 0u;
    k2[q] = s < U ? __ldg(perm_s2k + s) : 0u;
  }
#pragma unroll
  for (int q = 0; q < kPopIpt; ++q) {
    const long long s = base + (long long)threadIdx.x * kPopIpt + q;
    ttl[q] = s < U ? last[id[q]] : 0;
    f[q] = s < U ? flags[id[q]] : (uint8_t)0;
  }
#pragma unroll
  for (int q = 0; q < kPopIpt; ++q) {
    const long long s = base + (long long)threadIdx.x * kPopIpt + q;
    if (s < U) {
      ttl_k[k2[q]] = ttl[q];
      const bool pf = !(f[q] & kMirrored);
      const bool ev = ttl[q] == iteration;
      flags[id[q]] = ev ? (uint8_t)0 : (uint8_t)(f[q] | kMirrored);
      pf_bits |= (uint32_t)pf << q;
      ev_bits |= (uint32_t)ev << q;
    }
  }
  if (tr && threadIdx.x == 0) tr[1] = pop_timer();
  // (prefetch count, evict count) of this thread packed as 16 | 16 bits
  const uint32_t mine = (uint32_t)__popc(pf_bits) | ((uint32_t)__popc(ev_bits) << 16);
  uint32_t tile_total;
  const uint32_t excl = block_inclusive_scan_256(mine, sh_warp, &tile_total) - mine;
  const uint32_t warp = threadIdx.x >> 5;
  if (tr && threadIdx.x == 0) tr[2] = pop_timer();
  if (warp < 2) {
    const uint32_t agg = warp == 0 ? (tile_total & 0xFFFFu) : (tile_total >> 16);
    const uint32_t pfx = warp_lookback(warp == 0 ? st_pf : st_ev, tile, epoch, agg);
    if ((threadIdx.x & 31u) == 0) sh_pfx[warp] = pfx;
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[3] = pop_timer();
  uint32_t pos_pf = sh_pfx[0] + (excl & 0xFFFFu);
  uint32_t pos_ev = sh_pfx[1] + (excl >> 16);
#pragma unroll
  for (int q = 0; q < kPopIpt; ++q) {
    const long long s = base + (long long)threadIdx.x * kPopIpt + q;
    if ((pf_bits >> q) & 1u) {
      pf_keys[pos_pf] = keys_s[s];
      pf_ids[pos_pf] = id[q];
      pf_ttls[pos_pf] = ttl[q];
      ++pos_pf;
    }
    if ((ev_bits >> q) & 1u) {
      if (ev_keys) ev_keys[pos_ev] = keys_s[s];
      if (ev_ids) ev_ids[pos_ev] = id[q];
      ++pos_ev;
    }
  }
  if (tr && threadIdx.x == 0) tr[4] = pop_timer();
  if (tile == n_tiles - 1 && threadIdx.x == 0) {
    const long long npf = (long long)sh_pfx[0] + (tile_total & 0xFFFFu);
    const long long nev = (long long)sh_pfx[1] + (tile_total >> 16);
    // pop_begin: the projected occupancy is len(tracker) before popping
    ctr->last_projected = ctr->tracked;
    if (ctr->tracked > ctr->peak_projected) ctr->peak_projected = ctr->tracked;
    counts[2] = ctr->tracked;
    counts[3] = ctr->in_cache;
    const long long occ = ctr->in_cache + npf;
    if (occ > ctr->peak_occupancy) ctr->peak_occupancy = occ;
    ctr->insertions += npf;
    ctr->removals += nev;
    ctr->tracked -= nev;
    ctr->in_cache += npf - nev;
    ctr->last_prefetch = npf;
    ctr->last_evict = nev;
    counts[0] = npf;
    counts[1] = nev;
    counts[4] = ctr->in_cache;  // mirror size after this batch
  }
}

static int planner_scratch(bp_planner* p, long long n, cudaStream_t s) {
  if (p->scratch_cap >= n) return BP_OK;
  if (p->scratch_cap) cudaFreeAsync(p->d_ids, s);
  long long cap = 1024;
  while (cap < n) cap <<= 1;
  p->scratch_cap = cap;
  BP_CUDA_TRY(pool_alloc(&p->d_ids, cap, s));
  return BP_OK;
}

static int planner_grow(bp_planner* p, long long new_cap, cudaStream_t s) {
  long long* nl;
  uint8_t* nf;
  BP_CUDA_TRY(pool_alloc(&nl, new_cap, s));
  BP_CUDA_TRY(pool_alloc(&nf, new_cap, s));
  BP_CUDA_TRY(cudaMemsetAsync(nf, 0, new_cap, s));
  if (p->id_cap) {
    BP_CUDA_TRY(cudaMemcpyAsync(nl, p->d_last, p->id_cap * sizeof(long long), cudaMemcpyDeviceToDevice, s));
    BP_CUDA_TRY(cudaMemcpyAsync(nf, p->d_flags, p->id_cap, cudaMemcpyDeviceToDevice, s));
    cudaFreeAsync(p->d_last, s);
    cudaFreeAsync(p->d_flags, s);
  }
  p->d_last = nl;
  p->d_flags = nf;
  p->id_cap = new_cap;
  return BP_OK;
}

// Dense ids of the prep's sorted unique keys for this planner.
static int planner_ids(bp_planner* p, bp_prep* P, int insert, const uint32_t** ids, cudaStream_t s) {
  if (p->sc) {
    *ids = P->d_uniq_id_s;
    return BP_OK;
  }
  int rc = planner_scratch(p, P->n_occ, s);
  if (rc) return rc;
  if (insert) {
    int grown = 0;
    rc = registry_reserve(&p->reg, P->n_occ, s, &grown);
    if (rc) return rc;
    if (grown) {
      rc = planner_grow(p, p->reg.id_capacity, s);
      if (rc) return rc;
    }
  }
  rc = registry_map(&p->reg, P->d_uniq_key_s, P->n_occ, P->d_num_unique, p->d_ids, insert, s);
  if (rc) return rc;
  *ids = p->d_ids;
  return BP_OK;
}

}  // namespace bp

extern "C" int bp_planner_create(bp_ctx* ctx, const bp_schema* sc, int64_t capacity, bp_planner** out) {
  using namespace bp;
  if (capacity < 1) return BP_ERR_CONFIG;
  cudaStream_t s = 0;
  bp_planner* p = new bp_planner();
  p->ctx = ctx;
  p->sc = sc;
  p->capacity = capacity;
  p->home = s;
  BP_CUDA_TRY(cudaMalloc(&p->d_ctr, sizeof(PlannerCounters)));
  BP_CUDA_TRY(cudaMemset(p->d_ctr, 0, sizeof(PlannerCounters)));
  BP_CUDA_TRY(cudaMallocHost(&p->h_ctr, sizeof(PlannerCounters)));
  int rc;
  if (sc) {
    rc = planner_grow(p, sc->total_rows, s);
  } else {
    rc = registry_init(&p->reg, 1024, s);
    if (rc == BP_OK) rc = planner_grow(p, p->reg.id_capacity, s);
  }
  if (rc) return rc;
  BP_CUDA_TRY(cudaStreamSynchronize(s));
  *out = p;
  return BP_OK;
}

extern "C" int bp_planner_destroy(bp_planner* p) {
  if (!p) return BP_OK;
  cudaDeviceSynchronize();
  cudaStream_t s = 0;
  if (p->d_last) cudaFreeAsync(p->d_last, s);
  if (p->d_flags) cudaFreeAsync(p->d_flags, s);
  if (p->scratch_cap) cudaFreeAsync(p->d_ids, s);
  if (!p->sc) bp::registry_free(&p->reg, s);
  if (p->d_pop_state) cudaFreeAsync(p->d_pop_state, s);
  cudaFree(p->d_ctr);
  cudaFreeHost(p->h_ctr);
  cudaStreamSynchronize(s);
  delete p;
  return BP_OK;
}

extern "C" int bp_planner_refill(bp_planner* p, bp_prep* P, bp_stream_t stream) {
  using namespace bp;
  if (P->n_occ == 0) return BP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t* ids;
  int rc = planner_ids(p, P, 1, &ids, s);
  if (rc) return rc;
  k_refill<<<grid_for(P->n_occ, 256), 256, 0, s>>>(ids, P->d_num_unique, P->iteration, p->d_last, p->d_flags,
                                                   p->d_ctr);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_planner_pop(bp_planner* p, bp_prep* P, const bp_plan_buffers* b, bp_stream_t stream) {
  using namespace bp;
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t* ids = nullptr;
  if (P->n_occ > 0) {
    int rc = planner_ids(p, P, 0, &ids, s);
    if (rc) return rc;
  }
  // look-back words of the two compactions: persistent, zeroed once, epoch-tagged
  const long long nn = P->n_occ > 0 ? P->n_occ : 1;
  const long long tiles = (nn + kPopTile - 1) / kPopTile;
  if (p->pop_state_tiles < tiles) {
    if (p->d_pop_state) cudaFreeAsync(p->d_pop_state, s);
    long long cap = 64;
    while (cap < tiles) cap <<= 1;
    BP_CUDA_TRY(pool_alloc(&p->d_pop_state, 2 * cap * kLookbackStride, s));
    BP_CUDA_TRY(cudaMemsetAsync(p->d_pop_state, 0, 2 * cap * kLookbackStride * sizeof(unsigned long long), s));
    p->pop_state_tiles = cap;
  }
  k_pop_fused<<<(int)tiles, kPopThreads, 0, s>>>(ids, P->d_perm_s2k, P->d_num_unique, P->iteration, p->d_last,
                                                 p->d_flags, b->d_ttl_k, P->d_uniq_key_s, b->d_prefetch_keys,
                                                 b->d_prefetch_ids, b->d_prefetch_ttls, b->d_evict_keys,
                                                 b->d_evict_ids, p->d_pop_state,
                                                 p->d_pop_state + p->pop_state_tiles * kLookbackStride,
                                                 next_scan_epoch(), p->d_ctr,
                                                 b->d_counts);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_debug_pop_trace(void* d_buf) {
  BP_CUDA_TRY(cudaMemcpyToSymbol(bp::g_pop_trace, &d_buf, sizeof(void*)));
  return BP_OK;
}

extern "C" int bp_planner_get_stats(bp_planner* p, bp_stream_t stream, bp_planner_stats* out) {
  using namespace bp;
  cudaStream_t s = (cudaStream_t)stream;
  BP_CUDA_TRY(cudaMemcpyAsync(p->h_ctr, p->d_ctr, sizeof(PlannerCounters), cudaMemcpyDeviceToHost, s));
  long long reg = 0;
  if (!p->sc) BP_CUDA_TRY(cudaMemcpyAsync(&reg, p->reg.d_count, sizeof(long long), cudaMemcpyDeviceToHost, s));
  BP_CUDA_TRY(cudaStreamSynchronize(s));
  const PlannerCounters& c = *p->h_ctr;
  out->tracked = c.tracked;
  out->in_cache = c.in_cache;
  out->insertions = c.insertions;
  out->removals = c.removals;
  out->peak_occupancy = c.peak_occupancy;
  out->peak_projected = c.peak_projected;
  out->last_projected = c.last_projected;
  out->last_prefetch = c.last_prefetch;
  out->last_evict = c.last_evict;
  out->registry_size = reg;
  return BP_OK;
}

// --------------------------------------------------------------- inspection
// Enumerates every id with planner state (tracked and/or mirrored): key, last
// windowed iteration, flags.  Order is arbitrary; used by the API to expose
// LookaheadState.in_cache / latest_tracker and by tests.

namespace bp {

__device__ __forceinline__ uint64_t schema_key_of(const int64_t* base, int num_tables, uint32_t id) {
  int lo = 0, hi = num_tables;  // largest t with base[t] <= id
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (base[mid] <= (long long)id) lo = mid;
    else hi = mid;
  }
  return ((uint64_t)lo << kKeyTableShift) | (uint64_t)((long long)id - base[lo]);
}

__global__ void k_dump_schema(const uint8_t* flags, const long long* last, long long n, const int64_t* base,
                              int num_tables, uint64_t* out_keys, int64_t* out_last, uint8_t* out_flags,
                              long long cap, unsigned long long* count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint8_t f = flags[i];
    if (!f) continue;
    const unsigned long long p = atomicAdd(count, 1ull);
    if ((long long)p >= cap) continue;
    out_keys[p] = schema_key_of(base, num_tables, (uint32_t)i);
    out_last[p] = last[i];
    out_flags[p] = f;
  }
}

__global__ void k_dump_registry(const uint64_t* rkeys, const uint32_t* rids, long long slots, const uint8_t* flags,
                                const long long* last, uint64_t* out_keys, int64_t* out_last, uint8_t* out_flags,
                                long long cap, unsigned long long* count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < slots; i += (long long)gridDim.x * blockDim.x) {
    const uint64_t key = rkeys[i];
    if (key == kEmptyKey) continue;
    const uint32_t id = rids[i];
    const uint8_t f = flags[id];
    if (!f) continue;
    const unsigned long long p = atomicAdd(count, 1ull);
    if ((long long)p >= cap) continue;
    out_keys[p] = key;
    out_last[p] = last[id];
    out_flags[p] = f;
  }
}

}  // namespace bp

extern "C" int bp_planner_dump(bp_planner* p, const bp_planner_dump_t* o, int64_t cap, bp_stream_t stream) {
  using namespace bp;
  cudaStream_t s = (cudaStream_t)stream;
  BP_CUDA_TRY(cudaMemsetAsync(o->d_count, 0, sizeof(int64_t), s));
  if (p->sc) {
    k_dump_schema<<<grid_for(p->id_cap, 256), 256, 0, s>>>(p->d_flags, p->d_last, p->id_cap, p->sc->d_table_base,
                                                           p->sc->num_tables, o->d_keys, o->d_last, o->d_flags, cap,
                                                           (unsigned long long*)o->d_count);
  } else {
    k_dump_registry<<<grid_for(p->reg.slots, 256), 256, 0, s>>>(p->reg.d_keys, p->reg.d_ids, p->reg.slots,
                                                                p->d_flags, p->d_last, o->d_keys, o->d_last,
                                                                o->d_flags, cap, (unsigned long long*)o->d_count);
  }
  BP_LAUNCH_CHECK();
  return BP_OK;
}
