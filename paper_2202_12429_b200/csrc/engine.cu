// Native engine runtime for the pipelined BagPipe iteration.
//
// The reference's per-iteration loop (engine.py:487-649) is split in two:
// the host keeps the scalar control flow (window length, dispatch gate,
// flush cadence, simulated clock -- integer/float bookkeeping that must stay
// byte-identical to the reference), and this runtime owns every device
// buffer and issues every kernel, a few coarse calls per iteration:
//
//   bp_engine_add_batch  upload (host or device keys) + batch prep
//   bp_engine_refill/pop planner window step into a ring plan slot
//   bp_engine_fetch      prefetch gather on the host-link stream
//   bp_engine_train      insert + TTL + lookup + mark + fused trainer +
//                        eviction into a ring chunk slot, counters D2H,
//                        one synchronisation of the compute stream
//   bp_engine_flush      dirty write-back of chunk slots on the link stream
//
// All buffers are allocated once (plan/staging/chunk rings sized for the
// largest batch), so the steady state performs no allocation.  The compute
// and link streams are ordered by events exactly as the reference orders
// fetches and write-backs: prefetch of plan x waits for its pop; training of
// x waits for the prefetch; write-backs and prefetches share the link stream
// in dispatch order, which is the consistency gate (engine.py:302-377).
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "hostpool.h"

#include <cuda.h>
#include <thread>

#include <atomic>
#include <mutex>
#include <chrono>

struct bp_store;
struct bp_cache;
struct bp_planner;

extern "C" {
int bp_store_create(bp_ctx*, const bp_schema*, uint64_t, bp_stream_t, bp_store**);
int bp_store_destroy(bp_store*);
int bp_store_fetch(bp_store*, const uint32_t*, int64_t, const int64_t*, float*, bp_stream_t);
int bp_store_write_masked(bp_store*, const uint32_t*, const float*, const uint8_t*, int64_t, const int64_t*,
                          bp_stream_t);
int bp_cache_create(bp_ctx*, const bp_schema*, int64_t, int32_t, bp_cache**);
int bp_cache_destroy(bp_cache*);
int bp_cache_insert(bp_cache*, const uint64_t*, const uint32_t*, const float*, const int64_t*, int64_t,
                    const int64_t*, int64_t, bp_stream_t);
int bp_cache_apply_resolve(bp_cache*, bp_prep*, const int64_t*, uint64_t, int32_t, int32_t*, bp_stream_t);
int bp_cache_evict(bp_cache*, int64_t, int32_t, const bp_evict_buffers*, int64_t, bp_stream_t);
int bp_cache_evict_planned(bp_cache*, const uint64_t*, const uint32_t*, const int64_t*, int64_t, const int64_t*,
                           int64_t, const bp_evict_buffers*, bp_stream_t);
int bp_cache_get_view(const bp_cache*, bp_cache_view*);
int bp_planner_create(bp_ctx*, const bp_schema*, int64_t, bp_planner**);
int bp_planner_destroy(bp_planner*);
int bp_planner_refill(bp_planner*, bp_prep*, bp_stream_t);
int bp_planner_pop(bp_planner*, bp_prep*, const bp_plan_buffers*, bp_stream_t);
int bp_mark_ids(bp_prep*, int64_t*, int64_t, bp_stream_t);
int bp_prep_create_columnar(bp_ctx*, const bp_schema*, const uint64_t*, const uint8_t*, int64_t, int32_t,
                            const int32_t*, const int64_t*, int32_t, int64_t, int32_t, bp_stream_t, bp_prep**);
int bp_stub_step(bp_ctx*, bp_prep*, float*, const int32_t*, uint8_t*, int32_t, float, float, float, int32_t, float*,
                 const int64_t*, int64_t, int64_t*, bp_stream_t);
int bp_store_create_ex(bp_ctx*, const bp_schema*, uint64_t, int32_t, bp_stream_t, bp_store**);
int bp_embbag_forward_peer(bp_prep*, const float*, int32_t, const int32_t*, int32_t, const bp_peer_xchg*, bp_stream_t);
int bp_embbag_backward_peer(bp_prep*, const bp_peer_xchg*, float, float*, int32_t, const int32_t*, uint8_t*, int32_t,
                            int32_t, float, float, int64_t*, bp_stream_t);
int bp_embbag_forward(bp_prep*, const float*, int32_t, const int32_t*, int32_t, const int64_t*, int64_t, int32_t,
                      const uint32_t*, float*, bp_stream_t);
int bp_embbag_backward(bp_prep*, const float*, const int64_t*, const float*, float*, int32_t, const int32_t*,
                       uint8_t*, int32_t, int32_t, float, float, int64_t*, bp_stream_t);
}

namespace bp {

struct PlanSlot {
  uint64_t* keys;
  uint32_t* ids;
  int64_t* ttls;
  int64_t* ttl_k;
  uint64_t* evict_keys;
  uint32_t* evict_ids;
  int64_t* counts;   // [5] device
  int64_t* h_counts;  // [5] pinned
  float* staging;    // [max_occ, dim]
  int64_t* n_ins;    // device: counts[0] - dropped
  cudaEvent_t popped, fetched, consumed;
  long long prep_pos;
};

struct ChunkSlot {
  uint64_t* keys;
  uint32_t* ids;
  float* rows;
  uint8_t* dirty;
  int64_t* count;  // [2] device
  long long h_count = -1;  // rows, known on the host after the step that filled it
  cudaEvent_t flushed;
  bool pending;
};

// DMA host-link mode (see hostpool.h): one pinned staging set per direction,
// reused in link-stream order; host callbacks gather / scatter rows.
struct LinkJob {
  HostPool* pool;
  const float* table_src;  // gather: host table
  float* table_dst;        // scatter: host table
  const uint32_t* ids;
  const uint8_t* dirty;    // scatter only: rows with dirty == 0 are skipped
  const float* rows_src;
  float* rows_dst;
  long long n;
  size_t row_bytes;
  // copy jobs (batch uploads into pinned memory): up to two (src, dst, bytes)
  int copies = 0;
  const void* csrc[2];
  void* cdst[2];
  size_t cbytes[2];
};

static void host_copy(const LinkJob* j) {
  for (int c = 0; c < j->copies; ++c) {
    const char* src = static_cast<const char*>(j->csrc[c]);
    char* dst = static_cast<char*>(j->cdst[c]);
    const size_t bytes = j->cbytes[c];
    constexpr size_t kPiece = 256 << 10;
    j->pool->parallel_for((long long)((bytes + kPiece - 1) / kPiece), [&](long long a, long long b) {
      const size_t lo = (size_t)a * kPiece, hi = std::min(bytes, (size_t)b * kPiece);
      if (hi > lo) std::memcpy(dst + lo, src + lo, hi - lo);
    });
  }
}

// Debug counters of the host-link callbacks (bp_debug_link_cb_stats).
static std::atomic<long long> g_cb_ns[3], g_cb_calls[3], g_cb_rows[3];

struct CbTimer {
  int k;
  long long n;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  ~CbTimer() {
    g_cb_ns[k] += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    g_cb_calls[k] += 1;
    g_cb_rows[k] += n;
  }
};

static void CUDART_CB link_gather_cb(void* p) {
  const LinkJob* j = static_cast<const LinkJob*>(p);
  CbTimer timer{0, j->n};
  const size_t rb = j->row_bytes;
  const char* table = reinterpret_cast<const char*>(j->table_src);
  char* out = reinterpret_cast<char*>(j->rows_dst);
  j->pool->parallel_for(j->n, [&](long long a, long long b) {
    for (long long i = a; i < b; ++i) {
      if (i + 8 < b) __builtin_prefetch(table + (size_t)j->ids[i + 8] * rb);
      std::memcpy(out + (size_t)i * rb, table + (size_t)j->ids[i] * rb, rb);
    }
  });
}

static void CUDART_CB link_scatter_cb(void* p) {
  const LinkJob* j = static_cast<const LinkJob*>(p);
  CbTimer timer{1, j->n};
  const size_t rb = j->row_bytes;
  char* table = reinterpret_cast<char*>(j->table_dst);
  const char* in = reinterpret_cast<const char*>(j->rows_src);
  j->pool->parallel_for(j->n, [&](long long a, long long b) {
    for (long long i = a; i < b; ++i) {
      if (i + 8 < b) __builtin_prefetch(table + (size_t)j->ids[i + 8] * rb, 1);
      if (j->dirty[i]) std::memcpy(table + (size_t)j->ids[i] * rb, in + (size_t)i * rb, rb);
    }
  });
}

// Host worker for the DMA link mode, driven by stream memory operations
// instead of cudaLaunchHostFunc (whose callbacks serialise with the
// launching thread's CUDA calls): the link stream writes the job's sequence
// number into pinned memory (cuStreamWriteValue32) and then waits
// (cuStreamWaitValue32 >=) until this thread, which polls that word, has run
// the job's gather/scatter on the pool and published the same number.
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct LinkWorker {
  static constexpr int kRing = 256;
  HostPool pool;
  std::vector<LinkJob> jobs = std::vector<LinkJob>(kRing);
  volatile uint32_t* flags = nullptr;  // pinned, mapped: [0] ready (GPU writes), [32] done (CPU writes)
  CUdeviceptr d_ready = 0, d_done = 0;
  uint32_t issued = 0;  // host-enqueued jobs
  std::atomic<bool> stop{false};
  std::thread thr;
  WriteValueFn write_value = nullptr;
  WaitValueFn wait_value = nullptr;

  explicit LinkWorker(int threads) : pool(threads) {}

  cudaError_t init() {
    cudaError_t e = cudaHostAlloc((void**)&flags, 256, cudaHostAllocMapped);
    if (e != cudaSuccess) return e;
    flags[0] = 0;
    flags[32] = 0;
    void* d = nullptr;
    e = cudaHostGetDevicePointer(&d, (void*)flags, 0);
    if (e != cudaSuccess) return e;
    d_ready = (CUdeviceptr)d;
    d_done = (CUdeviceptr)((char*)d + 128);
    cudaDriverEntryPointQueryResult q;
    e = cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&write_value, cudaEnableDefault, &q);
    if (e != cudaSuccess || !write_value) return e != cudaSuccess ? e : cudaErrorNotSupported;
    e = cudaGetDriverEntryPoint("cuStreamWaitValue32", (void**)&wait_value, cudaEnableDefault, &q);
    if (e != cudaSuccess || !wait_value) return e != cudaSuccess ? e : cudaErrorNotSupported;
    thr = std::thread([this] { loop(); });
    return cudaSuccess;
  }

  ~LinkWorker() {
    stop = true;
    if (thr.joinable()) thr.join();
    if (flags) cudaFreeHost((void*)flags);
  }

  void loop() {
    uint32_t processed = 0;
    unsigned idle = 0;
    while (!stop.load(std::memory_order_relaxed)) {
      const uint32_t ready = flags[0];
      if ((int32_t)(ready - processed) <= 0) {
        if (++idle > 4096) std::this_thread::yield();
        continue;
      }
      idle = 0;
      ++processed;
      LinkJob& j = jobs[processed % kRing];
      if (j.copies) {
        CbTimer timer{2, (long long)(j.cbytes[0] + j.cbytes[1])};
        host_copy(&j);
      }
      else if (j.table_src)
        link_gather_cb(&j);
      else
        link_scatter_cb(&j);
      std::atomic_thread_fence(std::memory_order_seq_cst);  // table writes before the flag
      flags[32] = processed;
    }
  }

  // Host: the job the link stream will hand over next (call before enqueue()).
  LinkJob* next() {
    while ((int32_t)(issued + 1 - flags[32]) >= kRing) std::this_thread::yield();  // ring full
    return &jobs[(issued + 1) % kRing];
  }

  // Stream side: publish the job and wait until the worker finished it.
  int enqueue(cudaStream_t s) {
    ++issued;
    if (write_value((CUstream)s, d_ready, issued, 0) != CUDA_SUCCESS) return BP_ERR_CUDA;
    if (wait_value((CUstream)s, d_done, issued, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) return BP_ERR_CUDA;
    return BP_OK;
  }
};

__global__ void k_mark_written(const uint32_t* __restrict__ ids, const uint8_t* __restrict__ dirty, long long n,
                               uint32_t* __restrict__ written) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (dirty[i]) atomicOr(&written[ids[i] >> 5], 1u << (ids[i] & 31));
}

struct UploadSlot {
  uint8_t* host;  // pinned
  size_t bytes;
  cudaEvent_t done;
  bool used;
};

}  // namespace bp

namespace bp {
// Optional per-stage CUDA-event timing (cfg.timing): pairs recorded on the
// stream that runs the stage, summed on demand by bp_engine_stage_times.
// kStageTrainer: the stub trainer, or the DLRM EmbeddingBag forward;
// kStageTrainerBwd: the DLRM EmbeddingBag backward + optimizer
enum Stage { kStagePrep = 0, kStagePlanner, kStageFetch, kStageApply, kStageTrainer, kStageEvict, kStageFlush,
             kStageTrainerBwd, kNumStages };
struct StageTimer {
  std::mutex mu;  // the planner thread (prep/planner stages) and the training thread record concurrently
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> spans[kNumStages];
  cudaEvent_t open[kNumStages] = {};
  // recycled events: a span's begin event is recorded right before the
  // stage's first launch, with no event creation on the host in between
  std::vector<cudaEvent_t> pool;
  cudaEvent_t take() {
    if (pool.empty()) {
      cudaEvent_t ev;
      cudaEventCreate(&ev);
      return ev;
    }
    cudaEvent_t ev = pool.back();
    pool.pop_back();
    return ev;
  }
};
}  // namespace bp

struct bp_engine {
  bp::StageTimer timer;
  bp_ctx* ctx;
  const bp_schema* sc;
  bp_engine_config cfg;
  bp_store* store;
  bp_cache* cache;
  bp_planner* planner;
  cudaStream_t compute, link, planq;
  // write-back appends (link mode 0) on their own stream: the copy-engine
  // D2H of evicted rows overlaps the prefetch's zero-copy reads (opposite
  // link directions).  Fetches wait for the latest commit (wb_done); a
  // commit, a compaction or a direct table write waits for the latest fetch
  // (fetch_done) -- every fetch reads exactly what it reads in stream order.
  cudaStream_t wb = nullptr;
  cudaEvent_t wb_done = nullptr, fetch_done = nullptr;
  bool wb_pending = false, fetch_pending = false;
  cudaStream_t prepq;  // batch uploads + preps, ahead of and apart from the planner
  std::vector<bp_prep*> preps;  // ring indexed by position
  std::vector<cudaEvent_t> prep_ready;  // per prep slot, recorded on planq
  std::vector<bp::PlanSlot> plans;
  std::vector<bp::ChunkSlot> chunks;
  std::vector<bp::UploadSlot> uploads;
  int next_plan;
  int next_upload;
  int32_t* slots_s;
  int64_t* mark;
  int64_t* stats;  // [2]
  int64_t* h_result;  // pinned + mapped, [kStepRing][16]: counters [0..8), error record [8..)
  int64_t* d_result;  // device alias of h_result
  int32_t* d_col_tables;  // table id per column of columnar batches
  std::vector<int32_t> h_col_tables;
  uint64_t* d_keys_staging[2];
  uint8_t* d_labels_staging[2];
  // compact columnar uploads (bp_engine_add_batch_packed), allocated on first use
  uint32_t* d_planes_staging[2] = {nullptr, nullptr};  // row-id planes (u32 | u16 | u8)
  uint8_t* d_exlab_staging[2] = {nullptr, nullptr};
  cudaEvent_t staging_free[2];
  cudaEvent_t join_ev[3];  // bp_engine_join: planq, link, prepq
  // steps enqueued by engine_finish_begin and not yet ended: a FIFO ring, so
  // the host can enqueue iteration x+1 before reading iteration x's counters
  static constexpr int kStepRing = 2;
  cudaEvent_t step_done[kStepRing];
  int step_chunk[kStepRing], step_drain[kStepRing];
  int step_head = 0, step_count = 0;
  void* l2_flush_buf = nullptr;  // bp_engine_set_l2_flush (benchmarks)
  size_t l2_flush_bytes = 0;
  int l2_flush_exclusive = 0;
  cudaEvent_t flush_ev = nullptr;
  // link gate (DLRM mode): prefetches wait for the latest EmbeddingBag
  // forward, so their zero-copy reads run under the dense step instead of
  // beside the embedding kernels
  // persistent scratch of the sorted EmbeddingBag backward (zeroed once)
  void* bwd_scratch = nullptr;
  size_t bwd_scratch_bytes = 0;
  float* peer_rows = nullptr;  // key-sorted peer gradient rows (sorted peer backward)
  size_t peer_rows_bytes = 0;
  bool link_gate = false;
  bool side_gate = false;  // the same for batch preps and planner passes
  cudaEvent_t gate_ev = nullptr;
  // DMA host-link mode
  int link_mode = 0;  // 0: zero-copy kernels, 1: copy engines + host pool
  bp::LinkWorker* worker = nullptr;
  bp::LinkWorker* upload_worker = nullptr;  // host-batch uploads: copies into the pinned ring off the caller's thread
  uint32_t* h_fetch_ids = nullptr;
  float* h_fetch_rows = nullptr;
  uint32_t* h_flush_ids = nullptr;
  uint8_t* h_flush_dirty = nullptr;
  float* h_flush_rows = nullptr;

  int staging_i;
  long long chunk_cap;
};

namespace bp {

static int engine_prep_slot(bp_engine* e, long long pos) { return (int)(pos % (long long)e->preps.size()); }

static void stage_begin(bp_engine* e, int stage, cudaStream_t s) {
  if (!e->cfg.timing) return;
  std::lock_guard<std::mutex> lk(e->timer.mu);
  cudaEvent_t ev = e->timer.take();
  cudaEventRecord(ev, s);
  e->timer.open[stage] = ev;
}

static void stage_end(bp_engine* e, int stage, cudaStream_t s) {
  if (!e->cfg.timing) return;
  std::lock_guard<std::mutex> lk(e->timer.mu);
  if (!e->timer.open[stage]) return;
  cudaEvent_t ev = e->timer.take();
  cudaEventRecord(ev, s);
  e->timer.spans[stage].emplace_back(e->timer.open[stage], ev);
  e->timer.open[stage] = nullptr;
}

}  // namespace bp

// Sum of the recorded stage spans (ms) and their counts since the last call;
// synchronises the device, then clears the record.
extern "C" int bp_engine_stage_times(bp_engine* e, double* h_ms, int64_t* h_counts) {
  BP_CUDA_TRY(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lk(e->timer.mu);
  for (int st = 0; st < bp::kNumStages; ++st) {
    double total = 0;
    for (auto& pr : e->timer.spans[st]) {
      float ms = 0;
      cudaEventElapsedTime(&ms, pr.first, pr.second);
      total += ms;
      e->timer.pool.push_back(pr.first);
      e->timer.pool.push_back(pr.second);
    }
    h_ms[st] = total;
    h_counts[st] = (int64_t)e->timer.spans[st].size();
    e->timer.spans[st].clear();
  }
  return BP_OK;
}

extern "C" int bp_engine_create(bp_ctx* ctx, const bp_schema* sc, const bp_engine_config* cfg, bp_engine** out) {
  using namespace bp;
  if (!sc || cfg->capacity < 1 || cfg->dim != sc->emb_dim || cfg->max_occ < 1 || cfg->plan_slots < 2 ||
      cfg->chunk_slots < 2 || cfg->prep_slots < 2)
    return BP_ERR_INVALID;
  bp_engine* e = new bp_engine();
  e->ctx = ctx;
  e->sc = sc;
  e->cfg = *cfg;
  int lo = 0, hi = 0;
  BP_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // Compute at the highest priority: the host-link kernels only wait on PCIe
  // and must not delay the critical path's CTAs.
  // With a green-context SM partition (bp_set_green_sms) every engine stream
  // lives in the rest partition and the hot-key chains get the hot one.
  cudaStream_t gs = nullptr;
  green_auto(cfg->dim);  // the partition's size by the row width (unless set)
  {
    int grc = green_stream(0, hi, &gs);
    if (grc) return grc;
  }
  if (gs && green_link_mode()) {
    // the small partition runs the host-link streams, everything else the rest
    e->compute = gs;
    int grc = green_stream(1, lo, &e->link);
    if (!grc) grc = green_stream(1, lo, &e->wb);
    if (!grc) grc = green_stream(0, hi < lo ? hi + 1 : hi, &e->planq);
    if (!grc) grc = green_stream(0, hi < lo ? hi + 1 : hi, &e->prepq);
    if (grc) return grc;
  } else if (gs) {
    e->compute = gs;
    int grc = green_stream(0, lo, &e->link);
    if (!grc) grc = green_stream(0, lo, &e->wb);
    if (!grc) grc = green_stream(0, hi < lo ? hi + 1 : hi, &e->planq);
    if (!grc) grc = green_stream(0, hi < lo ? hi + 1 : hi, &e->prepq);
    cudaStream_t hs = nullptr;
    if (!grc) grc = green_stream(1, hi, &hs);
    if (grc) return grc;
    set_long_stream(hs);
  } else {
    BP_CUDA_TRY(cudaStreamCreateWithPriority(&e->compute, cudaStreamNonBlocking, hi));
    BP_CUDA_TRY(cudaStreamCreateWithPriority(&e->link, cudaStreamNonBlocking, lo));
    BP_CUDA_TRY(cudaStreamCreateWithPriority(&e->wb, cudaStreamNonBlocking, lo));
    // Batch prep and the planner window step of batches entering the window run
    // on their own stream: they depend only on the trace, so they overlap the
    // training of the iterations ahead of them.
    BP_CUDA_TRY(cudaStreamCreateWithPriority(&e->planq, cudaStreamNonBlocking, hi < lo ? hi + 1 : hi));
    BP_CUDA_TRY(cudaStreamCreateWithPriority(&e->prepq, cudaStreamNonBlocking, hi < lo ? hi + 1 : hi));
  }
  int rc = bp_store_create_ex(ctx, sc, cfg->seed, cfg->init_dims > 0 ? cfg->init_dims : sc->emb_dim, e->compute,
                              &e->store);
  if (rc) return rc;
  rc = bp_cache_create(ctx, sc, cfg->capacity, cfg->dim, &e->cache);
  if (rc) return rc;
  rc = bp_planner_create(ctx, sc, cfg->capacity, &e->planner);
  if (rc) return rc;
  const long long n = cfg->max_occ;
  const int dim = cfg->dim;
  e->preps.assign(cfg->prep_slots, nullptr);
  e->prep_ready.resize(cfg->prep_slots);
  for (auto& ev : e->prep_ready) BP_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  e->plans.resize(cfg->plan_slots);
  for (auto& p : e->plans) {
    BP_CUDA_TRY(cudaMalloc(&p.keys, n * sizeof(uint64_t)));
    BP_CUDA_TRY(cudaMalloc(&p.ids, n * sizeof(uint32_t)));
    BP_CUDA_TRY(cudaMalloc(&p.ttls, n * sizeof(int64_t)));
    BP_CUDA_TRY(cudaMalloc(&p.ttl_k, n * sizeof(int64_t)));
    BP_CUDA_TRY(cudaMalloc(&p.evict_keys, n * sizeof(uint64_t)));
    BP_CUDA_TRY(cudaMalloc(&p.evict_ids, n * sizeof(uint32_t)));
    BP_CUDA_TRY(cudaMalloc(&p.counts, 5 * sizeof(int64_t)));
    BP_CUDA_TRY(cudaMallocHost(&p.h_counts, 5 * sizeof(int64_t)));
    BP_CUDA_TRY(cudaMalloc(&p.staging, n * dim * sizeof(float)));
    BP_CUDA_TRY(cudaMalloc(&p.n_ins, sizeof(int64_t)));
    BP_CUDA_TRY(cudaEventCreateWithFlags(&p.popped, cudaEventDisableTiming));
    BP_CUDA_TRY(cudaEventCreateWithFlags(&p.fetched, cudaEventDisableTiming));
    BP_CUDA_TRY(cudaEventCreateWithFlags(&p.consumed, cudaEventDisableTiming));
    BP_CUDA_TRY(cudaEventRecord(p.consumed, e->compute));
    BP_CUDA_TRY(cudaEventRecord(p.popped, e->compute));
    p.prep_pos = -1;
  }
  e->chunk_cap = cfg->capacity < n ? cfg->capacity : n;
  const long long cc = cfg->capacity;  // a drain may return every resident entry
  e->chunks.resize(cfg->chunk_slots);
  for (auto& c : e->chunks) {
    BP_CUDA_TRY(cudaMalloc(&c.keys, cc * sizeof(uint64_t)));
    BP_CUDA_TRY(cudaMalloc(&c.ids, cc * sizeof(uint32_t)));
    BP_CUDA_TRY(cudaMalloc(&c.rows, cc * dim * sizeof(float)));
    BP_CUDA_TRY(cudaMalloc(&c.dirty, cc));
    BP_CUDA_TRY(cudaMalloc(&c.count, 2 * sizeof(int64_t)));
    BP_CUDA_TRY(cudaEventCreateWithFlags(&c.flushed, cudaEventDisableTiming));
    BP_CUDA_TRY(cudaEventRecord(c.flushed, e->link));
    c.pending = false;
  }
  e->uploads.resize(8);
  for (auto& u : e->uploads) {
    u.bytes = (size_t)n * 9 + 64;
    BP_CUDA_TRY(cudaMallocHost(&u.host, u.bytes));
    BP_CUDA_TRY(cudaEventCreateWithFlags(&u.done, cudaEventDisableTiming));
    u.used = false;
  }
  for (int i = 0; i < 2; ++i) {
    BP_CUDA_TRY(cudaMalloc(&e->d_keys_staging[i], n * sizeof(uint64_t)));
    BP_CUDA_TRY(cudaMalloc(&e->d_labels_staging[i], n + 16));
    BP_CUDA_TRY(cudaEventCreateWithFlags(&e->staging_free[i], cudaEventDisableTiming));
    BP_CUDA_TRY(cudaEventCreateWithFlags(&e->join_ev[i], cudaEventDisableTiming));
    if (i == 0) BP_CUDA_TRY(cudaEventCreateWithFlags(&e->wb_done, cudaEventDisableTiming));
    if (i == 0) BP_CUDA_TRY(cudaEventCreateWithFlags(&e->fetch_done, cudaEventDisableTiming));
    if (i == 0) BP_CUDA_TRY(cudaEventCreateWithFlags(&e->join_ev[2], cudaEventDisableTiming));
    BP_CUDA_TRY(cudaEventCreateWithFlags(&e->step_done[i], cudaEventDisableTiming));
    BP_CUDA_TRY(cudaEventRecord(e->staging_free[i], e->prepq));
  }
  e->staging_i = 0;
  e->next_plan = 0;
  e->next_upload = 0;
  BP_CUDA_TRY(cudaMalloc(&e->slots_s, n * sizeof(int32_t)));
  BP_CUDA_TRY(cudaMalloc(&e->mark, sc->total_rows * sizeof(int64_t)));
  BP_CUDA_TRY(cudaMemsetAsync(e->mark, 0xC0, sc->total_rows * sizeof(int64_t), e->compute));  // never a tag
  BP_CUDA_TRY(cudaMalloc(&e->stats, 2 * sizeof(int64_t)));
  BP_CUDA_TRY(cudaHostAlloc(&e->h_result, bp_engine::kStepRing * 16 * sizeof(int64_t), cudaHostAllocMapped));
  BP_CUDA_TRY(cudaHostGetDevicePointer((void**)&e->d_result, e->h_result, 0));
  BP_CUDA_TRY(cudaMalloc(&e->d_col_tables, sc->num_tables * sizeof(int32_t)));
  // Reserve the stream-ordered pool's memory up front (its release threshold
  // is infinite, bp_ctx_create): the per-batch prep arenas and scratch then
  // never grow the pool inside the iteration loop -- a growth maps memory on
  // the host thread and stalled a step for milliseconds.
  {
    const size_t reserve = std::min<size_t>((size_t)4 << 30, std::max<size_t>((size_t)512 << 20,
                                             (size_t)(cfg->prep_slots > 0 ? cfg->prep_slots : 8) *
                                                 (size_t)n * 160));
    void* tmp = nullptr;
    if (cudaMallocAsync(&tmp, reserve, e->prepq) == cudaSuccess) cudaFreeAsync(tmp, e->prepq);
    else cudaGetLastError();
    // and a block freed on the compute stream for its own per-call scratch
    // (reused on the same stream without a cross-stream dependency)
    if (cudaMallocAsync(&tmp, (size_t)256 << 20, e->compute) == cudaSuccess) cudaFreeAsync(tmp, e->compute);
    else cudaGetLastError();
  }
  BP_CUDA_TRY(cudaStreamSynchronize(e->compute));
  BP_CUDA_TRY(cudaStreamSynchronize(e->planq));
  BP_CUDA_TRY(cudaStreamSynchronize(e->prepq));
  *out = e;
  return BP_OK;
}

extern "C" int bp_engine_destroy(bp_engine* e) {
  if (!e) return BP_OK;
  cudaDeviceSynchronize();
  delete e->worker;
  delete e->upload_worker;
  if (e->flush_ev) cudaEventDestroy(e->flush_ev);
  if (e->gate_ev) cudaEventDestroy(e->gate_ev);
  if (e->bwd_scratch) cudaFree(e->bwd_scratch);
  if (e->peer_rows) cudaFree(e->peer_rows);
  for (auto& spans : e->timer.spans)
    for (auto& pr : spans) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  for (auto ev : e->timer.open)
    if (ev) cudaEventDestroy(ev);
  for (auto ev : e->timer.pool) cudaEventDestroy(ev);
  cudaFreeHost(e->h_fetch_ids);
  cudaFreeHost(e->h_fetch_rows);
  cudaFreeHost(e->h_flush_ids);
  cudaFreeHost(e->h_flush_dirty);
  cudaFreeHost(e->h_flush_rows);
  for (auto* p : e->preps)
    if (p) bp_prep_destroy(p);
  for (auto& p : e->plans) {
    cudaFree(p.keys);
    cudaFree(p.ids);
    cudaFree(p.ttls);
    cudaFree(p.ttl_k);
    cudaFree(p.evict_keys);
    cudaFree(p.evict_ids);
    cudaFree(p.counts);
    cudaFreeHost(p.h_counts);
    cudaFree(p.staging);
    cudaFree(p.n_ins);
    cudaEventDestroy(p.popped);
    cudaEventDestroy(p.fetched);
    cudaEventDestroy(p.consumed);
  }
  for (auto& c : e->chunks) {
    cudaFree(c.keys);
    cudaFree(c.ids);
    cudaFree(c.rows);
    cudaFree(c.dirty);
    cudaFree(c.count);
    cudaEventDestroy(c.flushed);
  }
  for (auto& u : e->uploads) {
    cudaFreeHost(u.host);
    cudaEventDestroy(u.done);
  }
  for (int i = 0; i < 2; ++i) {
    cudaFree(e->d_keys_staging[i]);
    cudaFree(e->d_labels_staging[i]);
    if (e->d_planes_staging[i]) cudaFree(e->d_planes_staging[i]);
    if (e->d_exlab_staging[i]) cudaFree(e->d_exlab_staging[i]);
    cudaEventDestroy(e->staging_free[i]);
    cudaEventDestroy(e->join_ev[i]);
    if (i == 0) cudaEventDestroy(e->join_ev[2]);
    cudaEventDestroy(e->step_done[i]);
  }
  cudaFree(e->slots_s);
  cudaFree(e->mark);
  cudaFree(e->stats);
  cudaFreeHost(e->h_result);
  cudaFree(e->d_col_tables);
  bp_planner_destroy(e->planner);
  bp_cache_destroy(e->cache);
  bp_store_destroy(e->store);
  for (auto& ev : e->prep_ready) cudaEventDestroy(ev);
  cudaStreamDestroy(e->compute);
  cudaStreamDestroy(e->link);
  if (e->wb) cudaStreamDestroy(e->wb);
  if (e->wb_done) cudaEventDestroy(e->wb_done);
  if (e->fetch_done) cudaEventDestroy(e->fetch_done);
  cudaStreamDestroy(e->planq);
  cudaStreamDestroy(e->prepq);
  delete e;
  return BP_OK;
}

extern "C" int bp_engine_parts(bp_engine* e, bp_engine_parts_t* out) {
  out->store = e->store;
  out->cache = e->cache;
  out->planner = e->planner;
  out->compute_stream = e->compute;
  out->link_stream = e->link;
  return BP_OK;
}

static bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Batch entering the window: upload (host keys go through a pinned ring and
// one H2D copy each for keys and labels -- or straight from the caller's
// arrays when they are pinned) and device prep on the prep stream.
static int engine_add(bp_engine* e, int64_t pos, int64_t iteration, const uint64_t* keys, const uint8_t* labels,
                      int64_t n_occ, int64_t n_ex, int32_t n_cols, const int32_t* h_tables,
                      const int64_t* h_rank_bounds, int32_t num_ranks, int32_t keys_on_host) {
  using namespace bp;
  if (n_occ > e->cfg.max_occ) return BP_ERR_INVALID;
  const int slot = engine_prep_slot(e, pos);
  cudaStream_t q = e->prepq;
  if (e->preps[slot]) {
    bp_prep_destroy(e->preps[slot]);
    e->preps[slot] = nullptr;
  }
  const uint64_t* d_keys = keys;
  const uint8_t* d_labels = labels;
  int si = -1;
  if (keys_on_host && n_occ > 0 && host_pinned(keys) && host_pinned(labels)) {
    // the caller's arrays are pinned already: DMA them straight from there
    // (no copy into the upload ring; they stay alive until release)
    si = e->staging_i;
    e->staging_i ^= 1;
    BP_CUDA_TRY(cudaStreamWaitEvent(q, e->staging_free[si], 0));
    BP_CUDA_TRY(cudaMemcpyAsync(e->d_keys_staging[si], keys, n_occ * sizeof(uint64_t), cudaMemcpyHostToDevice, q));
    BP_CUDA_TRY(cudaMemcpyAsync(e->d_labels_staging[si], labels, n_occ, cudaMemcpyHostToDevice, q));
    d_keys = e->d_keys_staging[si];
    d_labels = e->d_labels_staging[si];
  } else if (keys_on_host && n_occ > 0) {
    UploadSlot& u = e->uploads[e->next_upload];
    e->next_upload = (e->next_upload + 1) % (int)e->uploads.size();
    if (u.used) BP_CUDA_TRY(cudaEventSynchronize(u.done));
    if (!e->upload_worker) {
      e->upload_worker = new bp::LinkWorker(1);  // measured: one thread copies fastest on the 16-vCPU box
      const cudaError_t err = e->upload_worker->init();
      if (err != cudaSuccess) {
        delete e->upload_worker;
        e->upload_worker = nullptr;
        BP_CUDA_TRY(err);
      }
    }
    si = e->staging_i;
    e->staging_i ^= 1;
    BP_CUDA_TRY(cudaStreamWaitEvent(q, e->staging_free[si], 0));
    // the copy into the pinned slot runs on the upload worker thread;
    // the stream waits for it, the caller does not (its arrays must stay
    // alive until bp_engine_release_batch)
    bp::LinkJob* j = e->upload_worker->next();
    *j = bp::LinkJob{&e->upload_worker->pool, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0};
    j->copies = 2;
    j->csrc[0] = keys;
    j->cdst[0] = u.host;
    j->cbytes[0] = n_occ * sizeof(uint64_t);
    j->csrc[1] = labels;
    j->cdst[1] = u.host + n_occ * sizeof(uint64_t);
    j->cbytes[1] = n_occ;
    {
      const int wrc = e->upload_worker->enqueue(q);
      if (wrc) return wrc;
    }
    BP_CUDA_TRY(cudaMemcpyAsync(e->d_keys_staging[si], u.host, n_occ * sizeof(uint64_t), cudaMemcpyHostToDevice, q));
    BP_CUDA_TRY(cudaMemcpyAsync(e->d_labels_staging[si], u.host + n_occ * sizeof(uint64_t), n_occ,
                                cudaMemcpyHostToDevice, q));
    BP_CUDA_TRY(cudaEventRecord(u.done, q));
    u.used = true;
    d_keys = e->d_keys_staging[si];
    d_labels = e->d_labels_staging[si];
  }
  if (e->side_gate) BP_CUDA_TRY(cudaStreamWaitEvent(q, e->gate_ev, 0));
  int rc;
  if (n_cols > 0) {
    if (n_cols > e->sc->num_tables) return BP_ERR_INVALID;
    if ((int)e->h_col_tables.size() != n_cols ||
        std::memcmp(e->h_col_tables.data(), h_tables, n_cols * sizeof(int32_t)) != 0) {
      e->h_col_tables.assign(h_tables, h_tables + n_cols);
      BP_CUDA_TRY(cudaStreamSynchronize(q));  // previous preps may still read the old ids
      BP_CUDA_TRY(cudaMemcpy(e->d_col_tables, h_tables, n_cols * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    stage_begin(e, kStagePrep, q);
    rc = bp_prep_create_columnar(e->ctx, e->sc, d_keys, d_labels, n_ex, n_cols, e->d_col_tables, h_rank_bounds,
                                 num_ranks, iteration, e->cfg.prep_flags, q, &e->preps[slot]);
  } else {
    stage_begin(e, kStagePrep, q);
    rc = bp_prep_create(e->ctx, e->sc, d_keys, d_labels, n_occ, h_rank_bounds, num_ranks, iteration,
                        e->cfg.prep_flags, 0, 0, q, &e->preps[slot]);
  }
  stage_end(e, kStagePrep, q);
  if (rc) return rc;
  if (si >= 0) BP_CUDA_TRY(cudaEventRecord(e->staging_free[si], q));  // prep consumed the staging copy
  BP_CUDA_TRY(cudaEventRecord(e->prep_ready[slot], q));
  return BP_OK;
}

namespace bp {
// Column map of a packed columnar upload: table id and (plane, index) of
// every column (plane 0: u32 rows, 1: u16, 2: u8).
struct PackedCols {
  int32_t table[64];
  int32_t where[64];  // plane << 16 | index within the plane
  int32_t n[3];       // columns per plane
};

// Packed keys (table << 44 | row) and per-occurrence labels of a columnar
// batch from its row-id planes and per-example labels.
__global__ void k_expand_packed(const uint8_t* __restrict__ planes, long long n_ex, int n_cols, PackedCols m,
                                const uint8_t* __restrict__ ex_labels, uint64_t* __restrict__ keys,
                                uint8_t* __restrict__ labels) {
  const uint32_t* r32 = reinterpret_cast<const uint32_t*>(planes);
  const uint16_t* r16 = reinterpret_cast<const uint16_t*>(planes + (size_t)n_ex * m.n[0] * 4);
  const uint8_t* r8 = planes + (size_t)n_ex * (m.n[0] * 4 + m.n[1] * 2);
  const long long n = n_ex * n_cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long ex = i / n_cols;
    const int c = (int)(i - ex * n_cols);
    const int w = m.where[c], plane = w >> 16, j = w & 0xFFFF;
    const uint32_t row = plane == 0 ? r32[ex * m.n[0] + j] : plane == 1 ? (uint32_t)r16[ex * m.n[1] + j]
                                                                        : (uint32_t)r8[ex * m.n[2] + j];
    keys[i] = ((uint64_t)(uint32_t)m.table[c] << kKeyTableShift) | (uint64_t)row;
    labels[i] = ex_labels[ex];
  }
}
}  // namespace bp

// Compact columnar upload (reference Batch.rows / Batch.labels of a
// Criteo-layout batch, traces.py): the row ids as planes of u32, u16 and u8
// columns ([n_ex][n] each, in that order, one buffer) and one label per
// example -- a CK batch is 1.0 MB over the link instead of 3.83 MB of packed
// u64 keys + per-occurrence labels -- expanded to packed keys + occurrence
// labels by one kernel on the prep stream, then the columnar prep.
// planes / ex_labels: pinned host memory (DMA'd) or device memory.
extern "C" int bp_engine_add_batch_packed(bp_engine* e, int64_t pos, int64_t iteration, const void* planes,
                                          const uint8_t* ex_labels, int64_t n_ex, int32_t n_cols,
                                          const int32_t* h_tables, const int8_t* h_widths,
                                          const int64_t* h_rank_bounds, int32_t num_ranks, int32_t on_host) {
  using namespace bp;
  const long long n_occ = n_ex * n_cols;
  if (n_occ > e->cfg.max_occ || n_cols < 1 || n_cols > e->sc->num_tables || n_cols > 64) return BP_ERR_INVALID;
  PackedCols m{};
  for (int c = 0; c < n_cols; ++c) {
    const int plane = h_widths[c] == 4 ? 0 : h_widths[c] == 2 ? 1 : h_widths[c] == 1 ? 2 : -1;
    if (plane < 0) return BP_ERR_INVALID;
    m.table[c] = h_tables[c];
    m.where[c] = (plane << 16) | m.n[plane]++;
  }
  const size_t plane_bytes = (size_t)n_ex * (m.n[0] * 4 + m.n[1] * 2 + m.n[2]);
  cudaStream_t q = e->prepq;
  const int si = e->staging_i;
  e->staging_i ^= 1;
  BP_CUDA_TRY(cudaStreamWaitEvent(q, e->staging_free[si], 0));
  const uint8_t* d_planes = static_cast<const uint8_t*>(planes);
  const uint8_t* d_lab = ex_labels;
  if (on_host) {
    if (!e->d_planes_staging[si]) {
      BP_CUDA_TRY(cudaStreamSynchronize(q));
      BP_CUDA_TRY(cudaMalloc(&e->d_planes_staging[si], (size_t)e->cfg.max_occ * sizeof(uint32_t)));
      BP_CUDA_TRY(cudaMalloc(&e->d_exlab_staging[si], (size_t)e->cfg.max_occ + 16));
    }
    BP_CUDA_TRY(cudaMemcpyAsync(e->d_planes_staging[si], planes, plane_bytes, cudaMemcpyHostToDevice, q));
    BP_CUDA_TRY(cudaMemcpyAsync(e->d_exlab_staging[si], ex_labels, n_ex, cudaMemcpyHostToDevice, q));
    d_planes = reinterpret_cast<const uint8_t*>(e->d_planes_staging[si]);
    d_lab = e->d_exlab_staging[si];
  }
  if (n_occ > 0) {
    k_expand_packed<<<grid_for(n_occ, 256), 256, 0, q>>>(d_planes, n_ex, n_cols, m, d_lab, e->d_keys_staging[si],
                                                         e->d_labels_staging[si]);
    BP_LAUNCH_CHECK();
  }
  const int rc = engine_add(e, pos, iteration, e->d_keys_staging[si], e->d_labels_staging[si], n_occ, n_ex, n_cols,
                            h_tables, h_rank_bounds, num_ranks, 0);
  if (rc) return rc;
  BP_CUDA_TRY(cudaEventRecord(e->staging_free[si], q));  // the prep consumed the staging buffers
  return BP_OK;
}

extern "C" int bp_engine_add_batch(bp_engine* e, int64_t pos, int64_t iteration, const uint64_t* keys,
                                   const uint8_t* labels, int64_t n_occ, const int64_t* h_rank_bounds,
                                   int32_t num_ranks, int32_t keys_on_host) {
  return engine_add(e, pos, iteration, keys, labels, n_occ, 0, 0, nullptr, h_rank_bounds, num_ranks, keys_on_host);
}

// Columnar batch (one key per table per example, h_tables[c] = table of
// column c, strictly increasing): per-column shared-memory sort in the prep.
extern "C" int bp_engine_add_batch_columnar(bp_engine* e, int64_t pos, int64_t iteration, const uint64_t* keys,
                                            const uint8_t* labels, int64_t n_ex, int32_t n_cols,
                                            const int32_t* h_tables, const int64_t* h_rank_bounds, int32_t num_ranks,
                                            int32_t keys_on_host) {
  return engine_add(e, pos, iteration, keys, labels, n_ex * n_cols, n_ex, n_cols, h_tables, h_rank_bounds,
                    num_ranks, keys_on_host);
}

extern "C" int bp_engine_prep(bp_engine* e, int64_t pos, bp_prep** out) {
  *out = e->preps[bp::engine_prep_slot(e, pos)];
  return *out ? BP_OK : BP_ERR_ENGINE;
}

extern "C" int bp_engine_release_batch(bp_engine* e, int64_t pos) {
  const int slot = bp::engine_prep_slot(e, pos);
  if (e->preps[slot]) {
    // The prep's memory is freed in stream order on the prep stream, after
    // the compute stream's last use (its training; the planner's uses
    // precede it through the fetch/popped events).
    cudaEvent_t done;
    BP_CUDA_TRY(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    BP_CUDA_TRY(cudaEventRecord(done, e->compute));
    BP_CUDA_TRY(cudaStreamWaitEvent(e->prepq, done, 0));
    cudaEventDestroy(done);
    bp_prep_destroy(e->preps[slot]);
    e->preps[slot] = nullptr;
  }
  return BP_OK;
}

extern "C" int bp_engine_refill(bp_engine* e, int64_t pos) {
  const int pslot = bp::engine_prep_slot(e, pos);
  bp_prep* P = e->preps[pslot];
  if (!P) return BP_ERR_ENGINE;
  BP_CUDA_TRY(cudaStreamWaitEvent(e->planq, e->prep_ready[pslot], 0));
  if (e->side_gate) BP_CUDA_TRY(cudaStreamWaitEvent(e->planq, e->gate_ev, 0));
  bp::stage_begin(e, bp::kStagePlanner, e->planq);
  const int rc = bp_planner_refill(e->planner, P, e->planq);
  bp::stage_end(e, bp::kStagePlanner, e->planq);
  return rc;
}

// Pop the planner window for the batch at ``pos`` into the next plan slot.
extern "C" int bp_engine_pop(bp_engine* e, int64_t pos, int32_t* slot_out) {
  using namespace bp;
  bp_prep* P = e->preps[engine_prep_slot(e, pos)];
  if (!P) return BP_ERR_ENGINE;
  const int slot = e->next_plan;
  e->next_plan = (e->next_plan + 1) % (int)e->plans.size();
  PlanSlot& ps = e->plans[slot];
  // The slot's previous plan must have been consumed by training.
  BP_CUDA_TRY(cudaStreamWaitEvent(e->planq, ps.consumed, 0));
  BP_CUDA_TRY(cudaStreamWaitEvent(e->planq, e->prep_ready[engine_prep_slot(e, pos)], 0));
  bp_plan_buffers b{ps.keys, ps.ids, ps.ttls, ps.ttl_k, ps.evict_keys, ps.evict_ids, ps.counts};
  stage_begin(e, kStagePlanner, e->planq);
  int rc = bp_planner_pop(e->planner, P, &b, e->planq);
  stage_end(e, kStagePlanner, e->planq);
  if (rc) return rc;
  BP_CUDA_TRY(cudaMemcpyAsync(ps.h_counts, ps.counts, 5 * sizeof(int64_t), cudaMemcpyDeviceToHost, e->planq));
  BP_CUDA_TRY(cudaEventRecord(ps.popped, e->planq));
  ps.prep_pos = pos;
  *slot_out = slot;
  return BP_OK;
}

// Host copy of a plan slot's counters (n_prefetch, n_evict, projected,
// resident_before); waits for that pop only.
extern "C" int bp_engine_plan_counts(bp_engine* e, int32_t slot, int64_t* out4) {
  bp::PlanSlot& ps = e->plans[slot];
  BP_CUDA_TRY(cudaEventSynchronize(ps.popped));
  std::memcpy(out4, ps.h_counts, 4 * sizeof(int64_t));
  return BP_OK;
}

// 1 if the pop of plan slot `slot` has completed on the device, else 0
// (non-blocking: lets the host emit plans ahead without stalling).
extern "C" int bp_engine_plan_ready(bp_engine* e, int32_t slot, int32_t* out) {
  const cudaError_t q = cudaEventQuery(e->plans[slot].popped);
  if (q == cudaErrorNotReady) {
    *out = 0;
    return BP_OK;
  }
  BP_CUDA_TRY(q);
  *out = 1;
  return BP_OK;
}

extern "C" int bp_engine_plan_view(bp_engine* e, int32_t slot, bp_plan_buffers* out, float** staging) {
  bp::PlanSlot& ps = e->plans[slot];
  *out = bp_plan_buffers{ps.keys, ps.ids, ps.ttls, ps.ttl_k, ps.evict_keys, ps.evict_ids, ps.counts};
  if (staging) *staging = ps.staging;
  return BP_OK;
}

// Prefetch of a plan on the link stream: zero-copy gather of its rows from
// the pinned store, after the plan's pop and after every earlier write-back
// issued on the same stream (the gate).
// Host-link mode of the engine: 0 = zero-copy row kernels (SM-driven PCIe
// gathers/scatters), 1 = copy engines + a pool of `threads` host threads
// gathering/scattering rows in pinned staging (no SM time on the link),
// 2 = zero-copy prefetch gathers, write-back by copy engine + host scatter
// (zero-copy scatters are the worst interferers: tools/mb/interfere.cu).
extern "C" int bp_engine_set_link_mode(bp_engine* e, int32_t mode, int32_t threads) {
  if (mode < 0 || mode > 2) return BP_ERR_INVALID;
  BP_CUDA_TRY(cudaStreamSynchronize(e->wb));
  BP_CUDA_TRY(cudaStreamSynchronize(e->link));
  if (mode != 0) {  // the host worker paths read / write the table itself
    const int rc = bp_store_compact(e->store, e->link);
    if (rc) return rc;
    BP_CUDA_TRY(cudaStreamSynchronize(e->link));
  }
  e->link_mode = mode;
  if (mode == 0) return BP_OK;
  if (threads < 1) {
    const unsigned hw = std::thread::hardware_concurrency();
    threads = (int)std::max(2u, std::min(16u, hw / 4));
  }
  if (!e->worker || e->worker->pool.size() != threads) {
    delete e->worker;
    e->worker = new bp::LinkWorker(threads);
    const cudaError_t err = e->worker->init();
    if (err != cudaSuccess) {
      delete e->worker;
      e->worker = nullptr;
      e->link_mode = 0;
      BP_CUDA_TRY(err);
    }
  }
  const size_t rb = (size_t)e->cfg.dim * sizeof(float);
  if (!e->h_fetch_ids) {
    BP_CUDA_TRY(cudaMallocHost(&e->h_fetch_ids, (size_t)e->cfg.max_occ * sizeof(uint32_t)));
    BP_CUDA_TRY(cudaMallocHost(&e->h_fetch_rows, (size_t)e->cfg.max_occ * rb));
    BP_CUDA_TRY(cudaMallocHost(&e->h_flush_ids, (size_t)e->chunk_cap * sizeof(uint32_t)));
    BP_CUDA_TRY(cudaMallocHost(&e->h_flush_dirty, (size_t)e->chunk_cap));
    BP_CUDA_TRY(cudaMallocHost(&e->h_flush_rows, (size_t)e->chunk_cap * rb));
  }
  return BP_OK;
}

// Write-back log of the engine's store (mode 0): log_rows pinned rows that
// flushes append to by DMA (0: zero-copy scatter into the table).
extern "C" int bp_engine_set_write_log(bp_engine* e, int64_t log_rows) {
  if (log_rows <= 0) return BP_OK;
  BP_CUDA_TRY(cudaStreamSynchronize(e->wb));
  return bp_store_enable_log(e->store, log_rows, e->link);
}

// bit 0: prefetches, bit 1: batch preps and planner passes wait for the
// latest EmbeddingBag forward (deadlock-free: the awaited forward is always
// enqueued before, everything waiting on the gated work after it)
extern "C" int bp_engine_set_link_gate(bp_engine* e, int32_t on) {
  if (on && !e->gate_ev) BP_CUDA_TRY(cudaEventCreateWithFlags(&e->gate_ev, cudaEventDisableTiming));
  e->link_gate = (on & 1) != 0;
  e->side_gate = (on & 2) != 0;
  return BP_OK;
}

extern "C" int bp_engine_fetch(bp_engine* e, int32_t slot) {
  bp::PlanSlot& ps = e->plans[slot];
  BP_CUDA_TRY(cudaStreamWaitEvent(e->link, ps.popped, 0));
  // rows written back by every flush enqueued before this fetch are visible
  if (e->wb_pending) BP_CUDA_TRY(cudaStreamWaitEvent(e->link, e->wb_done, 0));
  // the waited-for forward was enqueued before this fetch and everything
  // that waits on the fetch (the plan's apply) is enqueued after it: no cycle
  if (e->link_gate) BP_CUDA_TRY(cudaStreamWaitEvent(e->link, e->gate_ev, 0));
  bp::stage_begin(e, bp::kStageFetch, e->link);
  if (e->link_mode == 1) {
    // prefetch count on the host (the pop finished long before dispatch)
    BP_CUDA_TRY(cudaEventSynchronize(ps.popped));
    const long long n = ps.h_counts[0];
    if (n > 0) {
      const size_t rb = (size_t)e->cfg.dim * sizeof(float);
      BP_CUDA_TRY(cudaMemcpyAsync(e->h_fetch_ids, ps.ids, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, e->link));
      bp::LinkJob* j = e->worker->next();
      *j = bp::LinkJob{&e->worker->pool, bp_store_host_table(e->store), nullptr, e->h_fetch_ids, nullptr, nullptr,
                       e->h_fetch_rows, n, rb};
      const int rc = e->worker->enqueue(e->link);
      if (rc) return rc;
      BP_CUDA_TRY(cudaMemcpyAsync(ps.staging, e->h_fetch_rows, n * rb, cudaMemcpyHostToDevice, e->link));
    }
  } else {
    int rc = bp_store_fetch_lazy(e->store, ps.ids, ps.keys, e->cfg.max_occ, ps.counts, ps.staging, e->link);
    if (rc) return rc;
  }
  bp::stage_end(e, bp::kStageFetch, e->link);
  BP_CUDA_TRY(cudaEventRecord(ps.fetched, e->link));
  BP_CUDA_TRY(cudaEventRecord(e->fetch_done, e->link));
  e->fetch_pending = true;
  return BP_OK;
}

static int g_split_wb = 1;  // bp_set_split_writeback

extern "C" int bp_set_split_writeback(int32_t on) {
  g_split_wb = on != 0;
  return BP_OK;
}

// Dirty write-back of chunk slots, in order (last write wins), on the link stream.
extern "C" int bp_engine_flush(bp_engine* e, const int32_t* chunk_slots, int32_t n) {
  // link mode 0: the write-back stream (see bp_engine.wb); host-worker modes
  // keep everything on the link stream
  cudaStream_t ws = (g_split_wb && e->link_mode == 0) ? e->wb : e->link;
  bp::stage_begin(e, bp::kStageFlush, ws);
  for (int i = 0; i < n; ++i) {
    bp::ChunkSlot& c = e->chunks[chunk_slots[i]];
    if (e->link_mode >= 1 && c.h_count >= 0) {
      const long long m = c.h_count;
      if (m > 0) {
        const size_t rb = (size_t)e->cfg.dim * sizeof(float);
        BP_CUDA_TRY(cudaMemcpyAsync(e->h_flush_ids, c.ids, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, e->link));
        BP_CUDA_TRY(cudaMemcpyAsync(e->h_flush_dirty, c.dirty, m, cudaMemcpyDeviceToHost, e->link));
        BP_CUDA_TRY(cudaMemcpyAsync(e->h_flush_rows, c.rows, m * rb, cudaMemcpyDeviceToHost, e->link));
        bp::k_mark_written<<<bp::grid_for(m, 256), 256, 0, e->link>>>(
            c.ids, c.dirty, m, reinterpret_cast<uint32_t*>(bp_store_written_bitmap(e->store)));
        BP_LAUNCH_CHECK();
        bp::LinkJob* j = e->worker->next();
        *j = bp::LinkJob{&e->worker->pool, nullptr, bp_store_host_table(e->store), e->h_flush_ids, e->h_flush_dirty,
                         e->h_flush_rows, nullptr, m, rb};
        const int wrc = e->worker->enqueue(e->link);
        if (wrc) return wrc;
      }
    } else if (e->link_mode == 0 && c.h_count >= 0 && c.h_count <= bp_store_log_rows(e->store)) {
      // write-back log: one copy-engine append of the chunk + a commit kernel
      // (no zero-copy scatter stalling the compute stream)
      // split stream: the DMA overlaps the fetch enqueued before this flush,
      // the commit (or a compaction) waits for it
      int rc = bp::store_log_append_fenced(e->store, c.ids, c.rows, c.dirty, c.h_count, ws,
                                           (ws != e->link && e->fetch_pending) ? e->fetch_done : nullptr);
      if (rc) return rc;
    } else {
      if (ws != e->link && e->fetch_pending) BP_CUDA_TRY(cudaStreamWaitEvent(ws, e->fetch_done, 0));
      int rc = bp_store_write_masked(e->store, c.ids, c.rows, c.dirty, e->cfg.capacity, c.count, ws);
      if (rc) return rc;
    }
    BP_CUDA_TRY(cudaEventRecord(c.flushed, ws));
    c.pending = false;
  }
  bp::stage_end(e, bp::kStageFlush, ws);
  if (ws != e->link && n > 0) {
    BP_CUDA_TRY(cudaEventRecord(e->wb_done, ws));
    e->wb_pending = true;
  }
  return BP_OK;
}

namespace bp {

// Apply plan x (insert of its staged rows minus an optional dropped first
// key), TTL updates + lookup into slots_s, and stamp the next batch's keys.
// A cross-stream dependency the host has already seen complete needs no
// device-side wait: everything before the event is finished and visible to
// work enqueued after the query.  (The fetch, the next batch's prep and the
// chunk's previous write-back normally finished steps ago.)
static cudaError_t wait_pending(cudaStream_t s, cudaEvent_t ev) {
  const cudaError_t q = cudaEventQuery(ev);
  if (q == cudaSuccess) return cudaSuccess;
  if (q != cudaErrorNotReady) return q;
  return cudaStreamWaitEvent(s, ev, 0);
}

static int engine_apply(bp_engine* e, bp_prep* P, PlanSlot& ps, int64_t next_pos, uint64_t skip_key,
                        int32_t has_skip, bp_prep** next_out) {
  cudaStream_t s = e->compute;
  const int dim = e->cfg.dim;
  if (e->l2_flush_buf) {
    // benchmark hygiene (bp_engine_set_l2_flush): every iteration starts on a
    // cold L2; exclusive = no other engine work overlaps the flush write
    if (e->l2_flush_exclusive) {
      BP_CUDA_TRY(cudaEventRecord(e->join_ev[0], e->planq));
      BP_CUDA_TRY(cudaEventRecord(e->join_ev[1], e->link));
      BP_CUDA_TRY(cudaEventRecord(e->join_ev[2], e->prepq));
      BP_CUDA_TRY(cudaStreamWaitEvent(s, e->join_ev[0], 0));
      BP_CUDA_TRY(cudaStreamWaitEvent(s, e->join_ev[1], 0));
      BP_CUDA_TRY(cudaStreamWaitEvent(s, e->join_ev[2], 0));
      BP_CUDA_TRY(cudaEventRecord(e->join_ev[1], e->wb));
      BP_CUDA_TRY(cudaStreamWaitEvent(s, e->join_ev[1], 0));
    }
    BP_CUDA_TRY(cudaMemsetAsync(e->l2_flush_buf, 0, e->l2_flush_bytes, s));
    if (e->l2_flush_exclusive) {
      BP_CUDA_TRY(cudaEventRecord(e->flush_ev, s));
      BP_CUDA_TRY(cudaStreamWaitEvent(e->planq, e->flush_ev, 0));
      BP_CUDA_TRY(cudaStreamWaitEvent(e->link, e->flush_ev, 0));
      BP_CUDA_TRY(cudaStreamWaitEvent(e->wb, e->flush_ev, 0));
      BP_CUDA_TRY(cudaStreamWaitEvent(e->prepq, e->flush_ev, 0));
    }
  }
  BP_CUDA_TRY(wait_pending(s, ps.fetched));
  stage_begin(e, kStageApply, s);
  const int off = has_skip ? 1 : 0;
  // insert counts[0] - off rows; the count lands in ps.n_ins for the step record
  int rc = cache_insert_sub(e->cache, ps.keys + off, ps.ids + off, ps.staging + (size_t)off * dim, ps.ttls + off,
                            e->cfg.max_occ - off, ps.counts, off, ps.n_ins, P->iteration, s);
  if (rc) return rc;
  bp_prep* N = next_pos >= 0 ? e->preps[engine_prep_slot(e, next_pos)] : nullptr;
  if (N) {
    // this batch's TTL + lookup and the next batch's id stamp in one launch
    // (it also zeroes the step stats)
    BP_CUDA_TRY(wait_pending(s, e->prep_ready[engine_prep_slot(e, next_pos)]));
    rc = apply_resolve_mark(e->cache, P, ps.ttl_k, skip_key, has_skip, e->slots_s, N, e->mark, N->iteration,
                            e->stats, s);
    if (rc) return rc;
  } else {
    rc = bp_cache_apply_resolve(e->cache, P, ps.ttl_k, skip_key, has_skip, e->slots_s, s);
    if (rc) return rc;
    BP_CUDA_TRY(cudaMemsetAsync(e->stats, 0, 2 * sizeof(int64_t), s));
  }
  stage_end(e, kStageApply, s);
  *next_out = N;
  return BP_OK;
}

__global__ void k_step_counters(const uint64_t* num_unique, const uint64_t* n_ins, const uint64_t* stats,
                                const uint64_t* chunk_count, const uint64_t* drain_count, const uint64_t* err,
                                uint64_t* out) {
  if (threadIdx.x == 0) {
    out[0] = *num_unique;
    out[1] = *n_ins;
    out[2] = stats[0];
    out[3] = stats[1];
    out[4] = chunk_count[0];
    out[5] = chunk_count[1];
    out[6] = drain_count ? drain_count[0] : 0;
    out[7] = drain_count ? drain_count[1] : 0;
  }
  constexpr int kErrWords = sizeof(bp_error_t) / sizeof(uint64_t);
  static_assert(sizeof(bp_error_t) % sizeof(uint64_t) == 0 && kErrWords <= 8, "error record layout");
  if (threadIdx.x < kErrWords) out[8 + threadIdx.x] = err[threadIdx.x];
  __threadfence_system();
}

__global__ void k_count_critical(const uint32_t* __restrict__ ids, const long long* __restrict__ d_U,
                                 const int64_t* __restrict__ mark, long long tag, unsigned long long* stats) {
  const long long U = *d_U;
  unsigned long long c = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < U; i += (long long)gridDim.x * blockDim.x)
    c += mark[ids[i]] == tag;
  cta_add(stats, c);
}

// Eviction of ttl <= iteration into chunk_slot (+ full drain into drain_slot
// on the last iteration), counters to the host, one synchronisation.
static int engine_finish_begin(bp_engine* e, bp_prep* P, PlanSlot& ps, int32_t chunk_slot, int32_t drain_slot) {
  if (e->step_count == bp_engine::kStepRing) return BP_ERR_ENGINE;
  const int rs = (e->step_head + e->step_count) % bp_engine::kStepRing;
  e->step_chunk[rs] = chunk_slot;
  e->step_drain[rs] = drain_slot;
  cudaStream_t s = e->compute;
  BP_CUDA_TRY(cudaEventRecord(ps.consumed, s));
  ChunkSlot& c = e->chunks[chunk_slot];
  BP_CUDA_TRY(wait_pending(s, c.flushed));  // its previous contents are durable
  bp_evict_buffers eb{e->cfg.record_keys ? c.keys : nullptr, c.ids, c.rows, c.dirty, c.count};
  stage_begin(e, kStageEvict, s);
  // The planner's key-sorted evict set is exactly {ttl <= iteration}
  // (checked: the occupancy must then equal the mirror size after the pop);
  // key order makes the later write-back walk the host table ascending.
  // Without a drain, the eviction kernel's last block also writes the step
  // record (all counters + the error record) into mapped pinned memory.
  StepRecord rec;
  if (drain_slot < 0) {
    rec.num_unique = (const unsigned long long*)P->d_num_unique;
    rec.n_ins = (const long long*)ps.n_ins;
    rec.stats = (const unsigned long long*)e->stats;
    rec.out = (uint64_t*)(e->d_result + 16 * rs);
  }
  int rc = cache_evict_planned_rec(e->cache, ps.evict_keys, ps.evict_ids, ps.counts + 1, e->chunk_cap, ps.counts + 4,
                                   P->iteration, &eb, rec, s);
  stage_end(e, kStageEvict, s);
  if (rc) return rc;
  c.pending = true;
  if (drain_slot >= 0) {
    ChunkSlot& d = e->chunks[drain_slot];
    BP_CUDA_TRY(wait_pending(s, d.flushed));
    bp_evict_buffers db{e->cfg.record_keys ? d.keys : nullptr, d.ids, d.rows, d.dirty, d.count};
    rc = bp_cache_evict(e->cache, P->iteration, 1, &db, e->cfg.capacity, s);
    if (rc) return rc;
    d.pending = true;
    // all step counters + the error record in ONE kernel writing mapped
    // pinned memory, then one synchronisation
    k_step_counters<<<1, 32, 0, s>>>((const uint64_t*)P->d_num_unique, (const uint64_t*)ps.n_ins,
                                     (const uint64_t*)e->stats, (const uint64_t*)c.count, (const uint64_t*)d.count,
                                     (const uint64_t*)e->ctx->d_err, (uint64_t*)(e->d_result + 16 * rs));
    BP_LAUNCH_CHECK();
  }
  BP_CUDA_TRY(cudaEventRecord(e->step_done[rs], s));
  ++e->step_count;
  return BP_OK;
}

// Waits for the step enqueued by engine_finish_begin and reads its counters.
static int engine_finish_end(bp_engine* e, bp_step_result* out) {
  if (e->step_count == 0) return BP_ERR_ENGINE;
  const int rs = e->step_head;
  e->step_head = (e->step_head + 1) % bp_engine::kStepRing;
  --e->step_count;
  BP_CUDA_TRY(cudaEventSynchronize(e->step_done[rs]));
  volatile int64_t* h = e->h_result + 16 * rs;
  bp_error_t err;
  std::memcpy(&err, (const void*)(h + 8), sizeof(bp_error_t));
  if (err.code != 0) {
    BP_CUDA_TRY(cudaMemsetAsync(e->ctx->d_err, 0, sizeof(bp_error_t), e->compute));
    BP_CUDA_TRY(cudaStreamSynchronize(e->compute));
  }
  out->unique = h[0];
  out->inserted = h[1];
  out->critical = h[2];
  out->dirty_keys = h[3];
  out->evicted = h[4];
  out->evicted_dirty = h[5];
  out->drained = h[6];
  out->drained_dirty = h[7];
  out->err = err;
  if (e->step_chunk[rs] >= 0) e->chunks[e->step_chunk[rs]].h_count = h[4];
  if (e->step_drain[rs] >= 0) e->chunks[e->step_drain[rs]].h_count = h[6];
  return BP_OK;
}

static int engine_finish(bp_engine* e, bp_prep* P, PlanSlot& ps, int32_t chunk_slot, int32_t drain_slot,
                         bp_step_result* out) {
  const int rc = engine_finish_begin(e, P, ps, chunk_slot, drain_slot);
  return rc ? rc : engine_finish_end(e, out);
}

}  // namespace bp

// One stub-mode training iteration on the compute stream (reference
// engine.py:525-606): apply plan + lookup + next-batch stamp, fused trainer,
// eviction; synchronises once and fills ``out`` (device contract violations
// come back in out->err).
extern "C" int bp_engine_train_begin(bp_engine* e, int64_t pos, int32_t plan_slot, int64_t next_pos,
                                     uint64_t skip_key, int32_t has_skip, int32_t chunk_slot, int32_t drain_slot) {
  using namespace bp;
  if (e->step_count == bp_engine::kStepRing) return BP_ERR_ENGINE;
  bp_prep* P = e->preps[engine_prep_slot(e, pos)];
  if (!P) return BP_ERR_ENGINE;
  PlanSlot& ps = e->plans[plan_slot];
  bp_prep* N = nullptr;
  int rc = engine_apply(e, P, ps, next_pos, skip_key, has_skip, &N);
  if (rc) return rc;
  bp_cache_view cv;
  bp_cache_get_view(e->cache, &cv);
  stage_begin(e, kStageTrainer, e->compute);
  rc = bp_stub_step(e->ctx, P, cv.d_values, e->slots_s, cv.d_dirty, e->cfg.dim, e->cfg.c_value, e->cfg.c_label,
                    e->cfg.lr, BP_STUB_SGD, nullptr, N ? e->mark : nullptr, N ? N->iteration : 0, e->stats,
                    e->compute);
  stage_end(e, kStageTrainer, e->compute);
  if (rc) return rc;
  return engine_finish_begin(e, P, ps, chunk_slot, drain_slot);
}

extern "C" int bp_engine_train_end(bp_engine* e, bp_step_result* out) { return bp::engine_finish_end(e, out); }

extern "C" int bp_engine_train(bp_engine* e, int64_t pos, int32_t plan_slot, int64_t next_pos, uint64_t skip_key,
                               int32_t has_skip, int32_t chunk_slot, int32_t drain_slot, bp_step_result* out) {
  const int rc = bp_engine_train_begin(e, pos, plan_slot, next_pos, skip_key, has_skip, chunk_slot, drain_slot);
  return rc ? rc : bp_engine_train_end(e, out);
}

// DLRM mode, part 1: apply plan x and gather the batch's pooled embeddings
// (single-key bags) into d_pooled[n_occ][model_dim] on the compute stream.
extern "C" int bp_engine_dlrm_forward(bp_engine* e, int64_t pos, int32_t plan_slot, int64_t next_pos,
                                      uint64_t skip_key, int32_t has_skip, int32_t model_dim, float* d_pooled) {
  using namespace bp;
  bp_prep* P = e->preps[engine_prep_slot(e, pos)];
  if (!P) return BP_ERR_ENGINE;
  PlanSlot& ps = e->plans[plan_slot];
  bp_prep* N = nullptr;
  int rc = engine_apply(e, P, ps, next_pos, skip_key, has_skip, &N);
  if (rc) return rc;
  if (N) {
    k_count_critical<<<grid_for(P->n_occ, 256), 256, 0, e->compute>>>(P->d_uniq_id_s, P->d_num_unique, e->mark,
                                                                      N->iteration,
                                                                      (unsigned long long*)e->stats);
    BP_LAUNCH_CHECK();
  }
  bp_cache_view cv;
  bp_cache_get_view(e->cache, &cv);
  stage_begin(e, kStageTrainer, e->compute);
  rc = bp_embbag_forward(P, cv.d_values, e->cfg.dim, e->slots_s, model_dim, nullptr, P->n_occ, 0, nullptr, d_pooled,
                         e->compute);
  stage_end(e, kStageTrainer, e->compute);
  if (!rc && (e->link_gate || e->side_gate)) BP_CUDA_TRY(cudaEventRecord(e->gate_ev, e->compute));
  return rc;
}

// DLRM mode, part 2: EmbeddingBag backward + optimizer in place on the cached
// rows (gradient of the pooled rows in d_grad, produced by the dense model on
// the compute stream), then eviction and counters as bp_engine_train.
extern "C" int bp_engine_dlrm_backward(bp_engine* e, int64_t pos, int32_t plan_slot, const float* d_grad,
                                       int32_t model_dim, int32_t opt, float lr, float eps, int32_t chunk_slot,
                                       int32_t drain_slot, bp_step_result* out) {
  using namespace bp;
  bp_prep* P = e->preps[engine_prep_slot(e, pos)];
  if (!P) return BP_ERR_ENGINE;
  PlanSlot& ps = e->plans[plan_slot];
  bp_cache_view cv;
  bp_cache_get_view(e->cache, &cv);
  stage_begin(e, kStageTrainerBwd, e->compute);
  int rc = bp_embbag_backward(P, d_grad, nullptr, nullptr, cv.d_values, e->cfg.dim, e->slots_s, cv.d_dirty,
                              model_dim, opt, lr, eps, e->stats, e->compute);
  stage_end(e, kStageTrainerBwd, e->compute);
  if (rc) return rc;
  return engine_finish(e, P, ps, chunk_slot, drain_slot, out);
}

// Sorted-gradient variant: d_out[p] = key-sorted position of occurrence p of
// batch `pos` (compute stream), for the dense model's interaction backward
// to store the pooled-row gradients in that order; bp_engine_dlrm_backward_
// sorted then reduces them as a contiguous stream.
extern "C" int bp_engine_dlrm_grad_rows(bp_engine* e, int64_t pos, uint32_t* d_out) {
  using namespace bp;
  bp_prep* P = e->preps[engine_prep_slot(e, pos)];
  if (!P) return BP_ERR_ENGINE;
  return bp_prep_occ_rank(P, d_out, e->compute);
}

extern "C" int bp_engine_dlrm_backward_sorted(bp_engine* e, int64_t pos, int32_t plan_slot,
                                              const float* d_grad_sorted, int32_t model_dim, int32_t opt, float lr,
                                              float eps, int32_t chunk_slot, int32_t drain_slot,
                                              bp_step_result* out) {
  using namespace bp;
  bp_prep* P = e->preps[engine_prep_slot(e, pos)];
  if (!P) return BP_ERR_ENGINE;
  PlanSlot& ps = e->plans[plan_slot];
  bp_cache_view cv;
  bp_cache_get_view(e->cache, &cv);
  stage_begin(e, kStageTrainerBwd, e->compute);
  int rc = bp_embbag_backward_sorted(P, d_grad_sorted, cv.d_values, e->cfg.dim, e->slots_s, cv.d_dirty, model_dim,
                                     opt, lr, eps, e->stats, e->compute);
  stage_end(e, kStageTrainerBwd, e->compute);
  if (rc) return rc;
  return engine_finish(e, P, ps, chunk_slot, drain_slot, out);
}

// Asynchronous DLRM part 2: the backward + eviction + counters enqueued only
// (grad_sorted: rows in key-sorted order, else occurrence order);
// bp_engine_train_end waits and reads the counters, so the host can enqueue
// the next iteration's forward and dense step first.
extern "C" int bp_engine_dlrm_backward_begin(bp_engine* e, int64_t pos, int32_t plan_slot, const float* d_grad,
                                             int32_t grad_sorted, int32_t model_dim, int32_t opt, float lr, float eps,
                                             int32_t chunk_slot, int32_t drain_slot) {
  using namespace bp;
  if (e->step_count == bp_engine::kStepRing) return BP_ERR_ENGINE;
  bp_prep* P = e->preps[engine_prep_slot(e, pos)];
  if (!P) return BP_ERR_ENGINE;
  PlanSlot& ps = e->plans[plan_slot];
  bp_cache_view cv;
  bp_cache_get_view(e->cache, &cv);
  stage_begin(e, kStageTrainerBwd, e->compute);
  if (grad_sorted) {
    const size_t need = (size_t)bp_embbag_bwd_scratch_bytes(P->n_occ, model_dim);
    if (need > e->bwd_scratch_bytes) {
      BP_CUDA_TRY(cudaStreamSynchronize(e->compute));
      if (e->bwd_scratch) BP_CUDA_TRY(cudaFree(e->bwd_scratch));
      e->bwd_scratch = nullptr;
      e->bwd_scratch_bytes = 0;
      BP_CUDA_TRY(cudaMalloc(&e->bwd_scratch, need));
      BP_CUDA_TRY(cudaMemset(e->bwd_scratch, 0, need));
      e->bwd_scratch_bytes = need;
    }
  }
  int rc = grad_sorted ? bp_embbag_backward_sorted_scratch(P, d_grad, cv.d_values, e->cfg.dim, e->slots_s,
                                                           cv.d_dirty, model_dim, opt, lr, eps, e->stats,
                                                           e->bwd_scratch, (int64_t)e->bwd_scratch_bytes, e->compute)
                       : bp_embbag_backward(P, d_grad, nullptr, nullptr, cv.d_values, e->cfg.dim, e->slots_s,
                                            cv.d_dirty, model_dim, opt, lr, eps, e->stats, e->compute);
  stage_end(e, kStageTrainerBwd, e->compute);
  if (rc) return rc;
  return engine_finish_begin(e, P, ps, chunk_slot, drain_slot);
}

// DLRM hybrid parallel over NVLink peer memory (csrc/peer.cu): the same two
// halves, the forward storing pooled rows into the example owners' buffers,
// the backward loading gradient rows from them.
extern "C" int bp_engine_dlrm_forward_peer(bp_engine* e, int64_t pos, int32_t plan_slot, int64_t next_pos,
                                           uint64_t skip_key, int32_t has_skip, int32_t model_dim,
                                           const bp_peer_xchg* rows) {
  using namespace bp;
  bp_prep* P = e->preps[engine_prep_slot(e, pos)];
  if (!P) return BP_ERR_ENGINE;
  PlanSlot& ps = e->plans[plan_slot];
  bp_prep* N = nullptr;
  int rc = engine_apply(e, P, ps, next_pos, skip_key, has_skip, &N);
  if (rc) return rc;
  if (N) {
    k_count_critical<<<grid_for(P->n_occ, 256), 256, 0, e->compute>>>(P->d_uniq_id_s, P->d_num_unique, e->mark,
                                                                      N->iteration,
                                                                      (unsigned long long*)e->stats);
    BP_LAUNCH_CHECK();
  }
  bp_cache_view cv;
  bp_cache_get_view(e->cache, &cv);
  stage_begin(e, kStageTrainer, e->compute);
  rc = bp_embbag_forward_peer(P, cv.d_values, e->cfg.dim, e->slots_s, model_dim, rows, e->compute);
  stage_end(e, kStageTrainer, e->compute);
  return rc;
}

namespace bp {

static int g_peer_sorted = 1;  // bp_set_peer_sorted: 1 = gather into key order + staged backward

// The peer backward: the key-sorted form (gradient rows pulled over NVLink
// into key order, then the staged segmented reduce) or the reduce-by-key
// gather straight from the peers' buffers.
static int engine_backward_peer(bp_engine* e, bp_prep* P, const bp_peer_xchg* grads, float scale,
                                const bp_cache_view& cv, int32_t model_dim, int32_t opt, float lr, float eps) {
  const bool sorted = g_peer_sorted && P->d_seg_of && (model_dim == 4 || model_dim == 8 || model_dim == 16 ||
                                                       model_dim == 32);
  if (!sorted)
    return bp_embbag_backward_peer(P, grads, scale, cv.d_values, e->cfg.dim, e->slots_s, cv.d_dirty, model_dim, opt,
                                   lr, eps, e->stats, e->compute);
  const size_t need = (size_t)bp_embbag_bwd_scratch_bytes(P->n_occ, model_dim);
  const size_t rows = (size_t)P->n_occ * model_dim * sizeof(float);
  if (need > e->bwd_scratch_bytes || rows > e->peer_rows_bytes) {
    BP_CUDA_TRY(cudaStreamSynchronize(e->compute));
    if (need > e->bwd_scratch_bytes) {
      if (e->bwd_scratch) BP_CUDA_TRY(cudaFree(e->bwd_scratch));
      e->bwd_scratch = nullptr;
      e->bwd_scratch_bytes = 0;
      BP_CUDA_TRY(cudaMalloc(&e->bwd_scratch, need));
      BP_CUDA_TRY(cudaMemset(e->bwd_scratch, 0, need));
      e->bwd_scratch_bytes = need;
    }
    if (rows > e->peer_rows_bytes) {
      if (e->peer_rows) BP_CUDA_TRY(cudaFree(e->peer_rows));
      e->peer_rows = nullptr;
      e->peer_rows_bytes = 0;
      BP_CUDA_TRY(cudaMalloc(&e->peer_rows, rows));
      e->peer_rows_bytes = rows;
    }
  }
  return bp_embbag_backward_peer_sorted(P, grads, scale, cv.d_values, e->cfg.dim, e->slots_s, cv.d_dirty, model_dim,
                                        opt, lr, eps, e->stats, e->peer_rows, e->bwd_scratch,
                                        (int64_t)e->bwd_scratch_bytes, e->compute);
}

}  // namespace bp

extern "C" int bp_set_peer_sorted(int32_t on) {
  bp::g_peer_sorted = on ? 1 : 0;
  return BP_OK;
}

extern "C" int bp_engine_dlrm_backward_peer(bp_engine* e, int64_t pos, int32_t plan_slot, const bp_peer_xchg* grads,
                                            float scale, int32_t model_dim, int32_t opt, float lr, float eps,
                                            int32_t chunk_slot, int32_t drain_slot, bp_step_result* out) {
  using namespace bp;
  bp_prep* P = e->preps[engine_prep_slot(e, pos)];
  if (!P) return BP_ERR_ENGINE;
  PlanSlot& ps = e->plans[plan_slot];
  bp_cache_view cv;
  bp_cache_get_view(e->cache, &cv);
  stage_begin(e, kStageTrainerBwd, e->compute);
  int rc = engine_backward_peer(e, P, grads, scale, cv, model_dim, opt, lr, eps);
  stage_end(e, kStageTrainerBwd, e->compute);
  if (rc) return rc;
  return engine_finish(e, P, ps, chunk_slot, drain_slot, out);
}

// Asynchronous form of bp_engine_dlrm_backward_peer: enqueue only (the
// device-side peer barriers order the ranks' buffer reuse across iterations);
// bp_engine_train_end reads the counters.
extern "C" int bp_engine_dlrm_backward_peer_begin(bp_engine* e, int64_t pos, int32_t plan_slot,
                                                  const bp_peer_xchg* grads, float scale, int32_t model_dim,
                                                  int32_t opt, float lr, float eps, int32_t chunk_slot,
                                                  int32_t drain_slot) {
  using namespace bp;
  if (e->step_count == bp_engine::kStepRing) return BP_ERR_ENGINE;
  bp_prep* P = e->preps[engine_prep_slot(e, pos)];
  if (!P) return BP_ERR_ENGINE;
  PlanSlot& ps = e->plans[plan_slot];
  bp_cache_view cv;
  bp_cache_get_view(e->cache, &cv);
  stage_begin(e, kStageTrainerBwd, e->compute);
  int rc = engine_backward_peer(e, P, grads, scale, cv, model_dim, opt, lr, eps);
  stage_end(e, kStageTrainerBwd, e->compute);
  if (rc) return rc;
  return engine_finish_begin(e, P, ps, chunk_slot, drain_slot);
}

// Evicted keys of a chunk (device -> host), for event logs.
extern "C" int bp_engine_chunk_keys(bp_engine* e, int32_t chunk_slot, uint64_t* h_out, int64_t n) {
  if (n <= 0) return BP_OK;
  if (!e->cfg.record_keys) return BP_ERR_INVALID;
  BP_CUDA_TRY(cudaMemcpy(h_out, e->chunks[chunk_slot].keys, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return BP_OK;
}

extern "C" int bp_engine_chunk_view(bp_engine* e, int32_t chunk_slot, bp_evict_buffers* out) {
  bp::ChunkSlot& c = e->chunks[chunk_slot];
  *out = bp_evict_buffers{c.keys, c.ids, c.rows, c.dirty, c.count};
  return BP_OK;
}

// Per-stage event timing on/off (cfg.timing at creation); spans recorded so
// far are kept until bp_engine_stage_times.
extern "C" int bp_engine_set_timing(bp_engine* e, int32_t on) {
  std::lock_guard<std::mutex> lk(e->timer.mu);
  e->cfg.timing = on ? 1 : 0;
  for (auto& ev : e->timer.open) {
    if (ev) e->timer.pool.push_back(ev);
    ev = nullptr;
  }
  return BP_OK;
}

// Benchmark hygiene: every iteration first writes `bytes` of `d_buf` (larger
// than L2) on the compute stream; exclusive != 0 also fences the plan and
// host-link streams around that write so nothing overlaps it.  NULL disables.
extern "C" int bp_engine_set_l2_flush(bp_engine* e, void* d_buf, int64_t bytes, int32_t exclusive) {
  if (d_buf && bytes <= 0) return BP_ERR_INVALID;
  if (!e->flush_ev) BP_CUDA_TRY(cudaEventCreateWithFlags(&e->flush_ev, cudaEventDisableTiming));
  e->l2_flush_buf = d_buf;
  e->l2_flush_bytes = (size_t)bytes;
  e->l2_flush_exclusive = exclusive;
  return BP_OK;
}

extern "C" int bp_engine_join(bp_engine* e, bp_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  // the write-back stream first folds into the link stream
  BP_CUDA_TRY(cudaEventRecord(e->join_ev[1], e->wb));
  BP_CUDA_TRY(cudaStreamWaitEvent(e->link, e->join_ev[1], 0));
  BP_CUDA_TRY(cudaEventRecord(e->join_ev[0], e->planq));
  BP_CUDA_TRY(cudaEventRecord(e->join_ev[1], e->link));
  BP_CUDA_TRY(cudaEventRecord(e->join_ev[2], e->prepq));
  BP_CUDA_TRY(cudaStreamWaitEvent(s, e->join_ev[0], 0));
  BP_CUDA_TRY(cudaStreamWaitEvent(s, e->join_ev[1], 0));
  BP_CUDA_TRY(cudaStreamWaitEvent(s, e->join_ev[2], 0));
  if (s != e->compute) {
    cudaEvent_t c = e->join_ev[0];
    BP_CUDA_TRY(cudaEventRecord(c, e->compute));
    BP_CUDA_TRY(cudaStreamWaitEvent(s, c, 0));
  }
  return BP_OK;
}

extern "C" int bp_engine_sync(bp_engine* e) {
  BP_CUDA_TRY(cudaStreamSynchronize(e->compute));
  BP_CUDA_TRY(cudaStreamSynchronize(e->planq));
  BP_CUDA_TRY(cudaStreamSynchronize(e->prepq));
  BP_CUDA_TRY(cudaStreamSynchronize(e->wb));
  BP_CUDA_TRY(cudaStreamSynchronize(e->link));
  return BP_OK;
}

// Host-side row gather (op 0) / scatter (op 1) rate of the DMA link mode's
// worker pool, for tools/hostlink_peak.py: n random rows of `dim` floats
// between `table` and a scratch buffer; wall seconds in *seconds.
extern "C" int bp_host_rows_bench(float* table, int32_t dim, const uint32_t* ids, int64_t n, int32_t threads, int32_t op,
                                  double* seconds) {
  if (n <= 0 || dim <= 0 || threads < 1) return BP_ERR_INVALID;
  std::vector<float> scratch((size_t)n * dim);
  std::vector<uint8_t> dirty((size_t)n, 1);
  bp::HostPool pool(threads);
  bp::LinkJob j{&pool, table, table, ids, dirty.data(), scratch.data(), scratch.data(), n, (size_t)dim * sizeof(float)};
  if (op == 1) {  // scatter the rows' current values back (content unchanged)
    bp::link_gather_cb(&j);
  }
  const auto t0 = std::chrono::steady_clock::now();
  if (op == 0) bp::link_gather_cb(&j);
  else bp::link_scatter_cb(&j);
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return BP_OK;
}

// Debug: {gather ns, calls, rows, scatter ns, calls, rows} of the DMA link
// mode's host callbacks since the last call (reset).
extern "C" int bp_debug_link_cb_stats(int64_t* out6) {
  for (int k = 0; k < 3; ++k) {
    out6[3 * k] = bp::g_cb_ns[k].exchange(0);  // out6 holds 9 values
    out6[3 * k + 1] = bp::g_cb_calls[k].exchange(0);
    out6[3 * k + 2] = bp::g_cb_rows[k].exchange(0);
  }
  return BP_OK;
}
