// Embedding Server: the full table in pinned host memory, served over the
// host link by zero-copy kernels (reference store.py:65-201).
//
// Layout: one row-major float32 matrix [total_rows, dim] in (table, row,
// component) order -- byte-for-byte the stream the reference digests
// (store.py:179-185) -- so the digest is a single blake2b pass over host
// memory and no per-shard dictionaries exist.  Hash sharding (store.py:80-104)
// never changes values (reference tests/test_store.py:42-45); it is kept as
// metadata only (num_shards is echoed in reports).
//
// Initial values are the functional init of store.py:29-42 evaluated on the
// GPU and written straight into the mapped host table, so creating a 2.2 GB
// Criteo-Kaggle store costs one PCIe pass instead of 113 s of numpy.
#include "internal.cuh"

struct bp_store {
  bp_ctx* ctx;
  const bp_schema* sc;
  uint64_t seed;
  int dim;
  float* h_table;       // pinned, mapped
  float* d_table;       // device alias of h_table (UVA)
  uint32_t* d_written;  // bitmap, 1 bit per row
  int init_dims;        // components < init_dims carry the functional init, the rest start at 0
  unsigned long long* d_link_rows;  // [2] lazy fetches: rows read over the host link, rows computed
  // write-back log (bp_store_enable_log): rows appended by copy-engine DMA,
  // newest location of every written-back row in d_loc (-1: the table)
  long long log_rows = 0;  // capacity (0: no log)
  long long log_pos = 0;   // rows appended since the last compaction
  float* h_log = nullptr;  // pinned, mapped [log_rows][dim]
  float* d_log = nullptr;  // device alias
  int32_t* d_loc = nullptr;       // [total_rows]
  uint32_t* d_log_ids = nullptr;  // [log_rows] row id of each log entry
};

namespace bp {

// One thread per (row, 4-component chunk); dims not divisible by 4 use a
// scalar tail.  FNV over (t, r) is shared by all components of a row.
__global__ void k_store_init(float* __restrict__ out, long long row0, long long nrows, uint32_t table,
                             uint64_t seed, int dim, int init_dims) {
  const int chunks = (dim + 3) >> 2;
  const long long total = nrows * chunks;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / chunks;
    const int c = (int)(i - r * chunks);
    const uint64_t h_tr = fnv_u64(fnv_u64(kFnvOffset, table), (uint64_t)r);
    float v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = c * 4 + q;
      v[q] = j < init_dims ? init_component(seed, h_tr, (uint64_t)j) : 0.f;
    }
    float* dst = out + (row0 + r) * dim + c * 4;
    if ((dim & 3) == 0) {
      *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
      for (int q = 0; q < 4 && c * 4 + q < dim; ++q) dst[q] = v[q];
    }
  }
}

__global__ void k_init_values(uint64_t seed, int dim, const uint64_t* __restrict__ keys, long long n,
                              float* __restrict__ out) {
  const long long total = n * dim;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long k = i / dim;
    const int j = (int)(i - k * dim);
    const uint64_t key = keys[k];
    const uint64_t h_tr = fnv_u64(fnv_u64(kFnvOffset, (uint64_t)table_of(key)), row_of(key));
    out[i] = init_component(seed, h_tr, (uint64_t)j);
  }
}

// Row gather from the mapped host table: 16-byte lanes, (dim/4) lanes per row
// so each row is one contiguous PCIe read; every thread issues kIlp
// independent loads before its stores to keep enough host-link reads in
// flight (random 64 B rows are latency-bound on PCIe).
constexpr int kIlp = 4;

// Blocks of the host-link kernels.  Each block keeps 256 x kIlp 16-byte host
// reads in flight; a few dozen blocks saturate PCIe, and fewer blocks leave
// more SMs whose L1/LSU queues are not clogged by microsecond-latency host
// accesses (co-resident compute kernels stall behind them).
static int g_link_blocks = 32;
// Debug only (tools/profile_step.py --skip-link): store fetch/write kernels
// become no-ops, to measure what the host-link traffic costs the step.
static int g_skip_link = 0;
// Threads per link block and dynamic shared memory requested (unused; > 0
// makes a link block own its SM so no compute CTA shares it with the PCIe
// traffic -- measured no better on the bench step, so off by default).
static int g_link_threads = 256;
static int g_link_smem = 0;
// Blocks of the write-back scatter kernel (0: g_link_blocks).  Posted PCIe
// writes never stall their thread, so the scatter's rate -- and how far it
// floods the memory system's queues ahead of co-running kernels -- is set by
// how many threads issue them.
static int g_write_blocks = 0;


// Newest copy of row g: its write-back log entry, else the table.
__device__ __forceinline__ const float4* row_src(const float4* table, const float4* log, const int32_t* loc, uint32_t g,
                                                 int q) {
  const int32_t p = loc ? loc[g] : -1;
  return p >= 0 ? log + (long long)p * q : table + (long long)g * q;
}

__global__ void k_store_fetch_v4(const float4* __restrict__ table, const uint32_t* __restrict__ ids, long long n,
                                 const long long* d_n, int q, float4* __restrict__ out,
                                 const float4* __restrict__ log, const int32_t* __restrict__ loc) {
  n = load_count(n, d_n);
  const long long total = n * q;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total; i0 += stride * kIlp) {
    float4 v[kIlp];
#pragma unroll
    for (int r = 0; r < kIlp; ++r) {
      const long long i = i0 + r * stride;
      if (i < total) {
        const long long row = i / q;
        // evict-first: host rows are used once, keep them from displacing
        // the L2-resident cache arena
        v[r] = __ldcs((log ? row_src(table, log, loc, ids[row], q) : table + (long long)ids[row] * q) +
                      (i - row * q));
      }
    }
#pragma unroll
    for (int r = 0; r < kIlp; ++r) {
      const long long i = i0 + r * stride;
      if (i < total) out[i] = v[r];
    }
  }
}

// Lazy fetch (reference store.py:106-129: "written value if present, else
// the functional init"): rows never written back are computed on the GPU from
// their key (no host-link read); only written rows are gathered over PCIe.
// At Criteo-Kaggle most prefetches are first touches, so this removes most
// of the zero-copy reads -- and their stall on co-running kernels.
__global__ void k_store_fetch_lazy_v4(const float4* __restrict__ table, const uint32_t* __restrict__ written,
                                      const uint32_t* __restrict__ ids, const uint64_t* __restrict__ keys,
                                      long long n, const long long* d_n, int q, uint64_t seed, int init_dims,
                                      float4* __restrict__ out, unsigned long long* __restrict__ link_rows,
                                      const float4* __restrict__ log, const int32_t* __restrict__ loc) {
  n = load_count(n, d_n);
  unsigned n_host = 0, n_init = 0;
  const long long total = n * q;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total; i0 += stride * kIlp) {
    float4 v[kIlp];
    bool host[kIlp];
#pragma unroll
    for (int r = 0; r < kIlp; ++r) {
      const long long i = i0 + r * stride;
      host[r] = false;
      if (i < total) {
        const long long row = i / q;
        const uint32_t g = ids[row];
        host[r] = (written[g >> 5] >> (g & 31)) & 1u;
        if (host[r]) v[r] = __ldcs(row_src(table, log, loc, g, q) + (i - row * q));
        if (i - row * q == 0) (host[r] ? n_host : n_init) += 1;
      }
    }
#pragma unroll
    for (int r = 0; r < kIlp; ++r) {
      const long long i = i0 + r * stride;
      if (i < total && !host[r]) {
        const long long row = i / q;
        const int c = (int)(i - row * q);
        const uint64_t key = keys[row];
        const uint64_t h_tr = fnv_u64(fnv_u64(kFnvOffset, (uint64_t)table_of(key)), row_of(key));
        float w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int j = c * 4 + k;
          w[k] = j < init_dims ? init_component(seed, h_tr, (uint64_t)j) : 0.f;
        }
        v[r] = make_float4(w[0], w[1], w[2], w[3]);
      }
    }
#pragma unroll
    for (int r = 0; r < kIlp; ++r) {
      const long long i = i0 + r * stride;
      if (i < total) out[i] = v[r];
    }
  }
  if (link_rows) {
    for (int off = 16; off > 0; off >>= 1) {
      n_host += __shfl_down_sync(0xffffffffu, n_host, off);
      n_init += __shfl_down_sync(0xffffffffu, n_init, off);
    }
    if ((threadIdx.x & 31) == 0) {
      if (n_host) atomicAdd(link_rows, (unsigned long long)n_host);
      if (n_init) atomicAdd(link_rows + 1, (unsigned long long)n_init);
    }
  }
}

__global__ void k_store_fetch_scalar(const float* __restrict__ table, const uint32_t* __restrict__ ids, long long n,
                                     const long long* d_n, int dim, float* __restrict__ out) {
  n = load_count(n, d_n);
  const long long total = n * dim;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / dim;
    out[i] = table[(long long)ids[r] * dim + (i - r * dim)];
  }
}

// Scatter rows into the host table; ``mask`` (optional) skips clean rows, the
// write-back of only dirty evictions (reference engine.py:403-413).  Reads of
// the (device) source rows are batched kIlp deep before the posted PCIe writes.
__global__ void k_store_write(float* __restrict__ table, uint32_t* __restrict__ written,
                              const uint32_t* __restrict__ ids, const float* __restrict__ rows,
                              const uint8_t* __restrict__ mask, long long n, const long long* d_n, int dim,
                              int32_t* __restrict__ loc) {
  n = load_count(n, d_n);
  const bool v4 = (dim & 3) == 0;
  const int q = v4 ? dim >> 2 : dim;
  const long long total = n * q;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total; i0 += stride * kIlp) {
    float4 v[kIlp];
    long long dst[kIlp];
#pragma unroll
    for (int r = 0; r < kIlp; ++r) {
      const long long i = i0 + r * stride;
      dst[r] = -1;
      if (i < total) {
        const long long row = i / q;
        const int c = (int)(i - row * q);
        if (mask && !mask[row]) continue;
        const long long g = ids[row];
        dst[r] = g * q + c;
        if (v4) v[r] = reinterpret_cast<const float4*>(rows)[i];
        else v[r].x = rows[i];
        if (c == 0) {
          atomicOr(&written[g >> 5], 1u << (g & 31));
          if (loc) loc[g] = -1;  // the table copy is now the newest
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kIlp; ++r) {
      if (dst[r] < 0) continue;
      if (v4) __stcs(reinterpret_cast<float4*>(table) + dst[r], v[r]);
      else __stcs(table + dst[r], v[r].x);
    }
  }
}

// Log commit after the DMA append of a chunk at log position p0: the chunk's
// dirty rows become the newest copies of their ids (last write wins: chunks
// are committed in link-stream order); clean rows are dead log entries.
__global__ void k_log_commit(const uint32_t* __restrict__ ids, const uint8_t* __restrict__ dirty, long long m,
                             long long p0, int32_t* __restrict__ loc, uint32_t* __restrict__ log_ids,
                             uint32_t* __restrict__ written) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t g = ids[i];
    log_ids[p0 + i] = g;
    if (dirty && !dirty[i]) continue;
    loc[g] = (int32_t)(p0 + i);
    atomicOr(&written[g >> 5], 1u << (g & 31));
  }
}

// Compaction: every log entry that is still the newest copy of its row is
// copied into the table (host memory both sides, zero-copy) and the row
// points back at the table.  Off the hot path: when the log is full, and
// before host-side readers (digest, dumps, table views).
__global__ void k_log_compact(const float4* __restrict__ log, float4* __restrict__ table,
                              const uint32_t* __restrict__ log_ids, long long used, int q,
                              int32_t* __restrict__ loc) {
  const long long total = used * q;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / q;
    const int c = (int)(i - p * q);
    const uint32_t g = log_ids[p];
    if (loc[g] != (int32_t)p) continue;
    table[(long long)g * q + c] = log[i];
  }
}

__global__ void k_log_reset(const uint32_t* __restrict__ log_ids, long long used, int32_t* __restrict__ loc) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < used; p += (long long)gridDim.x * blockDim.x)
    loc[log_ids[p]] = -1;
}

static cudaError_t link_attrs() {
  static int done_smem = -1;
  if (done_smem == g_link_smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_store_fetch_v4, cudaFuncAttributeMaxDynamicSharedMemorySize, g_link_smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_store_write, cudaFuncAttributeMaxDynamicSharedMemorySize, g_link_smem);
  if (e == cudaSuccess) done_smem = g_link_smem;
  return e;
}

}  // namespace bp

extern "C" int bp_store_create_ex(bp_ctx* ctx, const bp_schema* sc, uint64_t seed, int32_t init_dims,
                                  bp_stream_t stream, bp_store** out);

extern "C" int bp_store_create(bp_ctx* ctx, const bp_schema* sc, uint64_t seed, bp_stream_t stream, bp_store** out) {
  return bp_store_create_ex(ctx, sc, seed, sc->emb_dim, stream, out);
}

// init_dims < emb_dim: components >= init_dims start at 0 (optimizer state
// stored next to the weights, e.g. Adagrad accumulators).
extern "C" int bp_store_create_ex(bp_ctx* ctx, const bp_schema* sc, uint64_t seed, int32_t init_dims,
                                  bp_stream_t stream, bp_store** out) {
  using namespace bp;
  cudaStream_t s = (cudaStream_t)stream;
  bp_store* st = new bp_store();
  st->ctx = ctx;
  st->sc = sc;
  st->seed = seed;
  st->dim = sc->emb_dim;
  st->init_dims = init_dims;
  const size_t bytes = (size_t)sc->total_rows * sc->emb_dim * sizeof(float);
  BP_CUDA_TRY(cudaHostAlloc((void**)&st->h_table, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  BP_CUDA_TRY(cudaHostGetDevicePointer((void**)&st->d_table, st->h_table, 0));
  const long long words = (sc->total_rows + 31) / 32;
  BP_CUDA_TRY(cudaMalloc(&st->d_written, words * sizeof(uint32_t)));
  BP_CUDA_TRY(cudaMemsetAsync(st->d_written, 0, words * sizeof(uint32_t), s));
  BP_CUDA_TRY(cudaMalloc(&st->d_link_rows, 2 * sizeof(unsigned long long)));
  BP_CUDA_TRY(cudaMemsetAsync(st->d_link_rows, 0, 2 * sizeof(unsigned long long), s));
  const int chunks = (sc->emb_dim + 3) / 4;
  for (int t = 0; t < sc->num_tables; ++t) {
    const long long rows = sc->h_table_base[t + 1] - sc->h_table_base[t];
    k_store_init<<<grid_for(rows * chunks, 256, kNumSMs * 32), 256, 0, s>>>(st->d_table, sc->h_table_base[t], rows,
                                                                            (uint32_t)t, seed, sc->emb_dim,
                                                                            init_dims);
  }
  BP_LAUNCH_CHECK();
  BP_CUDA_TRY(cudaStreamSynchronize(s));
  *out = st;
  return BP_OK;
}

extern "C" int bp_store_destroy(bp_store* st) {
  if (!st) return BP_OK;
  cudaFreeHost(st->h_table);
  cudaFree(st->d_written);
  cudaFree(st->d_link_rows);
  if (st->h_log) cudaFreeHost(st->h_log);
  cudaFree(st->d_loc);
  cudaFree(st->d_log_ids);
  delete st;
  return BP_OK;
}

extern "C" float* bp_store_host_table(bp_store* st) { return st->h_table; }
extern "C" uint8_t* bp_store_written_bitmap(bp_store* st) { return (uint8_t*)st->d_written; }

extern "C" int bp_store_fetch(bp_store* st, const uint32_t* d_ids, int64_t n, const int64_t* d_n, float* d_out,
                              bp_stream_t stream) {
  using namespace bp;
  if (n <= 0 || (g_skip_link & 1)) return BP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int dim = st->dim;
  if ((dim & 3) == 0) {
    const int q = dim >> 2;
    BP_CUDA_TRY(link_attrs());
    k_store_fetch_v4<<<grid_for(n * q, g_link_threads * kIlp, g_link_blocks), g_link_threads, g_link_smem, s>>>(
        reinterpret_cast<const float4*>(st->d_table), d_ids, n, (const long long*)d_n, q,
        reinterpret_cast<float4*>(d_out), reinterpret_cast<const float4*>(st->d_log), st->d_loc);
  } else {
    k_store_fetch_scalar<<<grid_for(n * dim, 256, kNumSMs * 32), 256, 0, s>>>(st->d_table, d_ids, n,
                                                                             (const long long*)d_n, dim, d_out);
  }
  BP_LAUNCH_CHECK();
  return BP_OK;
}

// Lazy variant of bp_store_fetch: d_keys[i] is the packed key of d_ids[i].
extern "C" int bp_store_fetch_lazy(bp_store* st, const uint32_t* d_ids, const uint64_t* d_keys, int64_t n,
                                   const int64_t* d_n, float* d_out, bp_stream_t stream) {
  using namespace bp;
  if (n <= 0 || (g_skip_link & 1)) return BP_OK;
  if ((st->dim & 3) != 0) return bp_store_fetch(st, d_ids, n, d_n, d_out, stream);
  const int q = st->dim >> 2;
  BP_CUDA_TRY(link_attrs());
  k_store_fetch_lazy_v4<<<grid_for(n * q, g_link_threads * kIlp, g_link_blocks), g_link_threads, g_link_smem,
                          (cudaStream_t)stream>>>(reinterpret_cast<const float4*>(st->d_table), st->d_written, d_ids,
                                                  d_keys, n, (const long long*)d_n, q, st->seed, st->init_dims,
                                                  reinterpret_cast<float4*>(d_out), st->d_link_rows,
                                                  reinterpret_cast<const float4*>(st->d_log), st->d_loc);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

// Lazy-fetch counters since creation: h_out[0] rows read over the host link,
// h_out[1] rows computed on the GPU (never written).  Synchronises the device.
extern "C" int bp_store_link_counters(bp_store* st, int64_t* h_out) {
  BP_CUDA_TRY(cudaDeviceSynchronize());
  BP_CUDA_TRY(cudaMemcpy(h_out, st->d_link_rows, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
  return BP_OK;
}

extern "C" int bp_store_write(bp_store* st, const uint32_t* d_ids, const float* d_rows, int64_t n, const int64_t* d_n,
                              bp_stream_t stream) {
  using namespace bp;
  if (n <= 0) return BP_OK;
  const int q = (st->dim & 3) == 0 ? st->dim / 4 : st->dim;
  BP_CUDA_TRY(link_attrs());
  k_store_write<<<grid_for(n * q, g_link_threads * kIlp, g_link_blocks), g_link_threads, g_link_smem,
                  (cudaStream_t)stream>>>(
      st->d_table, st->d_written, d_ids, d_rows, nullptr, n, (const long long*)d_n, st->dim, st->d_loc);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_store_write_masked(bp_store* st, const uint32_t* d_ids, const float* d_rows, const uint8_t* d_mask,
                                     int64_t n, const int64_t* d_n, bp_stream_t stream) {
  using namespace bp;
  if (n <= 0 || (g_skip_link & 2)) return BP_OK;
  const int q = (st->dim & 3) == 0 ? st->dim / 4 : st->dim;
  BP_CUDA_TRY(link_attrs());
  k_store_write<<<grid_for(n * q, g_link_threads * kIlp, g_write_blocks ? g_write_blocks : g_link_blocks),
                  g_link_threads, g_link_smem, (cudaStream_t)stream>>>(
      st->d_table, st->d_written, d_ids, d_rows, d_mask, n, (const long long*)d_n, st->dim, st->d_loc);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_init_values(uint64_t seed, int32_t dim, const uint64_t* d_keys, int64_t n, float* d_out,
                              bp_stream_t stream) {
  using namespace bp;
  if (n <= 0) return BP_OK;
  k_init_values<<<grid_for(n * dim, 256), 256, 0, (cudaStream_t)stream>>>(seed, dim, d_keys, n, d_out);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_set_link_blocks(int32_t blocks) {
  if (blocks < 1 || blocks > 4096) return BP_ERR_INVALID;
  bp::g_link_blocks = blocks;
  return BP_OK;
}

extern "C" int bp_set_link_config(int32_t blocks, int32_t threads, int32_t smem_bytes) {
  if (blocks < 1 || blocks > 4096 || threads < 32 || threads > 1024 || (threads & 31) || smem_bytes < 0 ||
      smem_bytes > (227 << 10))
    return BP_ERR_INVALID;
  bp::g_link_blocks = blocks;
  bp::g_link_threads = threads;
  bp::g_link_smem = smem_bytes;
  return BP_OK;
}

extern "C" int bp_store_enable_log(bp_store* st, int64_t log_rows, bp_stream_t stream) {
  using namespace bp;
  if (st->log_rows) return log_rows == st->log_rows ? BP_OK : BP_ERR_INVALID;
  if (log_rows <= 0 || (st->dim & 3) != 0 || log_rows > INT32_MAX) return BP_ERR_INVALID;
  const long long rows = st->sc->total_rows;
  BP_CUDA_TRY(cudaHostAlloc((void**)&st->h_log, (size_t)log_rows * st->dim * sizeof(float),
                            cudaHostAllocMapped | cudaHostAllocPortable));
  BP_CUDA_TRY(cudaHostGetDevicePointer((void**)&st->d_log, st->h_log, 0));
  BP_CUDA_TRY(cudaMalloc(&st->d_loc, (size_t)rows * sizeof(int32_t)));
  BP_CUDA_TRY(cudaMalloc(&st->d_log_ids, (size_t)log_rows * sizeof(uint32_t)));
  BP_CUDA_TRY(cudaMemsetAsync(st->d_loc, 0xFF, (size_t)rows * sizeof(int32_t), (cudaStream_t)stream));
  st->log_rows = log_rows;
  st->log_pos = 0;
  return BP_OK;
}

extern "C" int bp_store_compact(bp_store* st, bp_stream_t stream) {
  using namespace bp;
  if (!st->log_rows || st->log_pos == 0) return BP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int q = st->dim / 4;
  k_log_compact<<<grid_for(st->log_pos * q, 256, kNumSMs * 4), 256, 0, s>>>(
      reinterpret_cast<const float4*>(st->d_log), reinterpret_cast<float4*>(st->d_table), st->d_log_ids, st->log_pos,
      q, st->d_loc);
  k_log_reset<<<grid_for(st->log_pos, 256), 256, 0, s>>>(st->d_log_ids, st->log_pos, st->d_loc);
  BP_LAUNCH_CHECK();
  st->log_pos = 0;
  return BP_OK;
}

namespace bp {
// The append with an optional event waited for between the row DMA and the
// commit: the engine's write-back stream DMAs into fresh log rows while an
// earlier-enqueued fetch still reads the store, and publishes the rows only
// after that fetch (so it reads exactly what it would have in stream order).
int store_log_append_fenced(bp_store* st, const uint32_t* d_ids, const float* d_rows, const uint8_t* d_dirty,
                            int64_t m, cudaStream_t s, cudaEvent_t before_commit) {
  if (!st->log_rows || m > st->log_rows) return BP_ERR_INVALID;
  if (m <= 0) return BP_OK;
  if (st->log_pos + m > st->log_rows) {
    // compaction rewrites the table and recycles log rows: fenced as a whole
    if (before_commit) BP_CUDA_TRY(cudaStreamWaitEvent(s, before_commit, 0));
    before_commit = nullptr;
    const int rc = bp_store_compact(st, s);
    if (rc) return rc;
  }
  const size_t rb = (size_t)st->dim * sizeof(float);
  BP_CUDA_TRY(cudaMemcpyAsync(st->h_log + (size_t)st->log_pos * st->dim, d_rows, (size_t)m * rb,
                              cudaMemcpyDeviceToHost, s));
  if (before_commit) BP_CUDA_TRY(cudaStreamWaitEvent(s, before_commit, 0));
  k_log_commit<<<grid_for(m, 256), 256, 0, s>>>(d_ids, d_dirty, m, st->log_pos, st->d_loc, st->d_log_ids,
                                                st->d_written);
  BP_LAUNCH_CHECK();
  st->log_pos += m;
  return BP_OK;
}
}  // namespace bp

extern "C" int bp_store_log_append(bp_store* st, const uint32_t* d_ids, const float* d_rows, const uint8_t* d_dirty,
                                   int64_t m, bp_stream_t stream) {
  return bp::store_log_append_fenced(st, d_ids, d_rows, d_dirty, m, (cudaStream_t)stream, nullptr);
}

extern "C" int64_t bp_store_log_rows(bp_store* st) { return st->log_rows; }



extern "C" int bp_set_write_blocks(int32_t blocks) {
  if (blocks < 0 || blocks > 4096) return BP_ERR_INVALID;
  bp::g_write_blocks = blocks;
  return BP_OK;
}

extern "C" int bp_debug_skip_link(int32_t skip) {
  bp::g_skip_link = skip;
  return BP_OK;
}
