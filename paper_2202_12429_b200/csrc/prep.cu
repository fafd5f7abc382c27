// Batch prep: dedupe + grouping of one batch's occurrences on the device.
//
// Replaces Batch.unique_keys (reference traces.py:91-103) and _prep_batch
// (reference engine.py:142-182).  One stable LSD radix sort of
// (sort key, occurrence position) yields, for free:
//   * key-sorted unique keys (segment heads) -- the order of plan.prefetch
//     and of every store call (reference lookahead.py:108, engine.py:150),
//   * each key's occurrences in occurrence order (stability) -- the order in
//     which np.add.at accumulates (reference trainer.py:48-53),
// and one scan over "first occurrence" flags scattered back to occurrence
// positions gives the first-occurrence order of ttl_updates.
//
// Sort key: schema mode -> dense id g = table_base[t] + row (u32, monotone in
// (table,row)); registry mode -> the packed u64 key sorted on its two live
// bit ranges (rows: [0,row_bits), tables: [44, 44+table_bits)).
#include <algorithm>

#include <cooperative_groups.h>

#include "internal.cuh"

namespace bp {

// Debug switch (bp_debug_prep_cluster): 0 forces the single-CTA column sort.
static int g_prep_cluster = 1;

struct ColumnarInfo {
  int n_ex, n_cols, row_bits;
  const int32_t* d_tables;
  bool cluster;  // k_col_cluster_prep applies (see cs_shape)
};

__global__ void k_prep_keys_schema(const uint64_t* __restrict__ keys, long long n, const int64_t* base,
                                   const int64_t* rows, int num_tables, uint32_t* __restrict__ sk,
                                   uint32_t* __restrict__ val, ErrorRecord* err, long long iteration) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    uint32_t id = schema_id(base, rows, num_tables, keys[i]);
    if (id == kNoId) {
      raise_error(err, BP_ERR_STORE_KEY, iteration, i, keys[i]);
      id = 0;
    }
    sk[i] = id;
    val[i] = (uint32_t)i;
  }
}

__global__ void k_prep_keys_packed(const uint64_t* __restrict__ keys, long long n, uint64_t* __restrict__ sk,
                                   uint32_t* __restrict__ val) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    sk[i] = keys[i];
    val[i] = (uint32_t)i;
  }
}

template <typename K>
__global__ void k_prep_heads(const K* __restrict__ sk, long long n, uint32_t* __restrict__ head) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
    head[j] = (j == 0 || sk[j] != sk[j - 1]) ? 1u : 0u;
}

__device__ __forceinline__ int rank_of(long long p, const long long* __restrict__ rb, int num_ranks) {
  int r = 0;
  while (r + 1 < num_ranks && p >= rb[r + 1]) ++r;
  return r;
}

// Segment heads: CSR start, unique key/id (sorted order), first-occurrence
// flag at the head's position (the smallest position of the key: stable sort).
// Every occurrence's label byte carries bit 7 = "first occurrence of this key
// in its trainer rank", so the trainer streams one byte per occurrence and
// closes a rank partial on the flag (reference combine order, trainer.py:92-105).
template <typename K>
__global__ void k_prep_segments(const K* __restrict__ sk, const uint32_t* __restrict__ pos,
                                const uint32_t* __restrict__ head, const uint32_t* __restrict__ segx, long long n,
                                const uint64_t* __restrict__ keys, const uint8_t* __restrict__ labels,
                                int schema_mode, uint32_t* __restrict__ seg_start, uint64_t* __restrict__ uniq_key_s,
                                uint32_t* __restrict__ uniq_id_s, uint32_t* __restrict__ first_flag,
                                uint8_t* __restrict__ occ_label, const long long* d_num_unique,
                                const long long* __restrict__ rank_bounds, int num_ranks, ErrorRecord* err,
                                long long iteration) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const uint32_t p = pos[j];
    const uint8_t lab = labels[p];
    if (lab > 127) raise_error(err, BP_ERR_CONFIG, iteration, p, 0);
    bool rank_start = head[j] != 0;
    if (!rank_start && num_ranks > 1)
      rank_start = rank_of(p, rank_bounds, num_ranks) != rank_of(pos[j - 1], rank_bounds, num_ranks);
    occ_label[j] = (uint8_t)((lab & 0x7f) | (rank_start ? 0x80 : 0));
    if (head[j]) {
      const uint32_t s = segx[j];
      seg_start[s] = (uint32_t)j;
      uniq_key_s[s] = keys[p];
      uniq_id_s[s] = schema_mode ? (uint32_t)sk[j] : kNoId;
      first_flag[p] = 1u;
    }
    if (j == n - 1) seg_start[*d_num_unique] = (uint32_t)n;
  }
}

__global__ void k_prep_perm(const uint32_t* __restrict__ pos, const uint32_t* __restrict__ head,
                            const uint32_t* __restrict__ segx, const uint32_t* __restrict__ first_rank, long long n,
                            const uint64_t* __restrict__ uniq_key_s, uint32_t* __restrict__ perm_s2k,
                            uint32_t* __restrict__ perm_k2s, uint64_t* __restrict__ uniq_key_k,
                            const uint32_t* __restrict__ seg_start, uint32_t* __restrict__ long_list,
                            unsigned long long* num_long, long long long_cap) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    if (!head[j]) continue;
    const uint32_t s = segx[j];
    const uint32_t k = first_rank[pos[j]];
    perm_s2k[s] = k;
    perm_k2s[k] = s;
    uniq_key_k[k] = uniq_key_s[s];
    const uint32_t len = seg_start[s + 1] - seg_start[s];
    if (len >= kVeryLongSeg) long_list[atomicAdd(&num_long[0], 1ull)] = s;
    else if (len >= kLongSeg) long_list[long_cap - 1 - (long long)atomicAdd(&num_long[1], 1ull)] = s;
  }
}

__global__ void k_prep_occ_k(const uint32_t* __restrict__ pos, const uint32_t* __restrict__ head,
                             const uint32_t* __restrict__ segx, long long n, const uint32_t* __restrict__ perm_s2k,
                             uint32_t* __restrict__ occ_k, uint32_t* __restrict__ occ_s,
                             uint32_t* __restrict__ seg_of, uint32_t* __restrict__ occ_rank) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const uint32_t s = segx[j] + head[j] - 1u;  // inclusive segment index
    const uint32_t p = pos[j];
    if (occ_k) occ_k[p] = perm_s2k[s];
    if (occ_s) occ_s[p] = s;
    if (seg_of) seg_of[j] = s;
    if (occ_rank) occ_rank[p] = (uint32_t)j;
  }
}

// Columnar fast path (one key per table per example: the Criteo layout of
// every columnar batch).  A key of table t only occurs in column t, so the
// global (g, position) sort decomposes into one independent sort per column
// by row, each small enough for one CTA's shared memory (B <= 16384
// examples).  Elements (row << 14 | example) live in registers, 16 per thread;
// each 8-bit LSD pass ranks digits per warp with __match_any_sync (stable),
// scans the per-warp digit counts and scatters through one 128 KB smem
// buffer.  Column blocks are written in table order, so the output is
// identical to the generic radix sort's -- sorted by (g, position) -- with
// 26 CTAs and no global passes instead of 3 x (histogram, scan, scatter).
constexpr int kColThreads = 1024;
constexpr int kColIpt = 16;
constexpr int kColMax = kColThreads * kColIpt;  // 16384 examples
constexpr int kColWarps = kColThreads / 32;
constexpr int kColMaxChunks = 64;  // columnar path up to 64 x 16,384 examples

// Batches of more than kColMax examples (N-GPU weak scaling: N x 16,384):
// CTA (column c, chunk k) sorts examples [k*kColMax, (k+1)*kColMax) of the
// column, then k_prep_col_merge places every element at its rank in the
// column's merged order.
__global__ void __launch_bounds__(kColThreads, 1) k_prep_table_sort(const uint64_t* __restrict__ keys, int n_ex,
                                                                     int n_cols, const int64_t* __restrict__ base,
                                                                     const int32_t* __restrict__ col_tables,
                                                                     int row_bits, uint32_t* __restrict__ sk_out,
                                                                     uint32_t* __restrict__ pos_out) {
  extern __shared__ unsigned long long col_smem[];
  unsigned long long* buf = col_smem;                                             // [kColMax]
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(col_smem + kColMax);               // [kColWarps][256]
  uint32_t* dtot = wcnt + kColWarps * 256;                                        // [256]
  const int c = blockIdx.x;
  const int t = col_tables[c];
  const int ex0 = blockIdx.y * kColMax;  // this CTA's chunk of examples
  const int n_chunk = min(kColMax, n_ex - ex0);
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  unsigned long long e[kColIpt];
#pragma unroll
  for (int r = 0; r < kColIpt; ++r) {
    const int ex = warp * (32 * kColIpt) + r * 32 + lane;
    e[r] = ex < n_chunk ? (((keys[(long long)(ex0 + ex) * n_cols + c] & kRowMask) << 14) | (unsigned long long)ex)
                        : ~0ull;  // padding sorts last
  }
  for (int shift = 14; shift < 14 + row_bits; shift += 8) {
    for (int i = lane; i < 256; i += 32) wcnt[warp * 256 + i] = 0;
    __syncwarp();
    uint32_t rank[kColIpt];
#pragma unroll
    for (int r = 0; r < kColIpt; ++r) {
      const uint32_t d = (uint32_t)((e[r] >> shift) & 0xFFull);
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const unsigned below = peers & ((1u << lane) - 1u);
      const uint32_t prev = wcnt[warp * 256 + d];
      rank[r] = prev + (uint32_t)__popc(below);
      __syncwarp();
      if (below == 0) wcnt[warp * 256 + d] = prev + (uint32_t)__popc(peers);
      __syncwarp();
    }
    __syncthreads();
    if (threadIdx.x < 256) {  // per digit: exclusive prefix over warps, total
      uint32_t run = 0;
      for (int w = 0; w < kColWarps; ++w) {
        const uint32_t x = wcnt[w * 256 + threadIdx.x];
        wcnt[w * 256 + threadIdx.x] = run;
        run += x;
      }
      dtot[threadIdx.x] = run;
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the 256 digit totals (8 per lane)
      uint32_t v[8], sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[i] = dtot[lane * 8 + i];
        sum += v[i];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += y;
      }
      uint32_t run = incl - sum;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        dtot[lane * 8 + i] = run;
        run += v[i];
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kColIpt; ++r) {
      const uint32_t d = (uint32_t)((e[r] >> shift) & 0xFFull);
      buf[dtot[d] + wcnt[warp * 256 + d] + rank[r]] = e[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kColIpt; ++r) e[r] = buf[warp * (32 * kColIpt) + r * 32 + lane];
    __syncthreads();
  }
  const long long out0 = (long long)c * n_ex + ex0;  // columns are in increasing table order
#pragma unroll
  for (int r = 0; r < kColIpt; ++r) {
    const int i = warp * (32 * kColIpt) + r * 32 + lane;
    if (i < n_chunk) {
      const unsigned long long x = e[r];
      const long long ex = ex0 + (long long)(x & 0x3FFFull);
      sk_out[out0 + i] = (uint32_t)(base[t] + (long long)(x >> 14));
      pos_out[out0 + i] = (uint32_t)(ex * n_cols + c);
    }
  }
}

// Stable merge of a column's sorted chunks: element i of chunk k goes to
// (its index in chunk k) + (# keys <= it in earlier chunks) + (# keys < it in
// later chunks) -- earlier chunks hold smaller positions, so equal keys keep
// position order, exactly the single-sort output.
__global__ void k_prep_col_merge(const uint32_t* __restrict__ sk_in, const uint32_t* __restrict__ pos_in, int n_ex,
                                 int n_cols, int n_chunks, uint32_t* __restrict__ sk_out,
                                 uint32_t* __restrict__ pos_out) {
  const long long total = (long long)n_ex * n_cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long c = i / n_ex;
    const int j = (int)(i - c * n_ex);
    const int k = j / kColMax;
    const uint32_t key = sk_in[i];
    const uint32_t* col = sk_in + c * n_ex;
    long long dst = j - (long long)k * kColMax;
    for (int k2 = 0; k2 < n_chunks; ++k2) {
      if (k2 == k) continue;
      const int lo0 = k2 * kColMax, hi0 = min(n_ex, lo0 + kColMax);
      int lo = lo0, hi = hi0;
      if (k2 < k) {  // upper bound: keys <= key
        while (lo < hi) {
          const int m = (lo + hi) >> 1;
          if (col[m] <= key) lo = m + 1;
          else hi = m;
        }
      } else {  // lower bound: keys < key
        while (lo < hi) {
          const int m = (lo + hi) >> 1;
          if (col[m] < key) lo = m + 1;
          else hi = m;
        }
      }
      dst += lo - lo0;
    }
    sk_out[c * n_ex + dst] = key;
    pos_out[c * n_ex + dst] = pos_in[i];
  }
}

constexpr size_t kColSmem = sizeof(unsigned long long) * kColMax + sizeof(uint32_t) * (kColWarps * 256 + 256);

struct RankBounds {
  static constexpr int kMax = 64;
  long long v[kMax];
};

// ---------------------------------------------------------------------------
// Columnar prep on thread-block clusters (the default for Criteo-layout
// batches of up to 65,536 examples and 32 columns).
//
// One cluster of CS CTAs (CS = 1..16) sorts one column: CTA r of the cluster
// owns the column's examples [r*M, (r+1)*M) (M = 256 x IPT).  Elements
//   e = row << 27 | label << 20 | example
// live in registers; each 8-bit LSD pass over the column's OWN row bits
// ranks digits per warp with __match_any_sync (stable), publishes the CTA's
// 256 digit counts in shared memory, reads every CTA's counts through
// distributed shared memory (DSMEM) to get the column-wide digit offsets,
// and scatters each element straight into the shared memory of the CTA that
// owns its destination slot (st.shared::cluster).  After the last pass CTA r
// holds sorted positions [r*M, (r+1)*M) of the column -- no global
// temporaries, no merge pass, and every column occupies CS SMs instead of
// one.  Small tables take fewer passes (a 3-row table: one; a 1-row table:
// none).
//
// The same kernel then finds segment heads (row != previous row; the
// neighbour CTA's last element via DSMEM), numbers them with a block scan, a
// cluster prefix over the CTA totals and a decoupled look-back over the
// columns (column c's first segment index = distinct keys of columns < c,
// since dense ids of table t precede those of any later table), and writes
// every per-occurrence and per-segment output of the prep directly:
// key-sorted occurrence positions (column c's occurrences are sorted slots
// [c*n_ex, (c+1)*n_ex): every column holds exactly n_ex occurrences), the
// label byte with its rank-start bit, CSR offsets, sorted unique keys/ids,
// and, per first occurrence, its segment index plus one bit in a per-example
// mask from which k_first_order derives the first-occurrence order.
// ---------------------------------------------------------------------------
constexpr int kCsThreads = 256;
constexpr int kCsWarps = kCsThreads / 32;
constexpr int kCsRowShift = 27;  // row << 27 | label (7 bits) << 20 | example (20 bits)
constexpr unsigned long long kCsExMask = (1ull << 20) - 1;
constexpr int kCsMaxRowBits = 64 - kCsRowShift;
constexpr int kCsMaxCols = 32;
constexpr int kCsMaxCluster = 16;
constexpr int kFirstThreads = 256;  // k_first_order: one example per thread

struct ColPrepArgs {
  const uint64_t* keys;
  const uint8_t* labels;
  int n_ex, n_cols;
  const int32_t* col_tables;
  const int64_t* base;
  const int64_t* rows;
  RankBounds rb;
  int num_ranks;
  long long iteration;
  ErrorRecord* err;
  // outputs
  uint32_t* occ_pos;
  uint8_t* occ_label;
  uint32_t* seg_start;
  uint64_t* uniq_key_s;
  uint32_t* uniq_id_s;
  uint32_t* first_s;   // [n_occ] segment index at each first occurrence (only those written)
  uint32_t* ex_mask;   // [n_ex] bit c = column c's key is first seen at this example (zeroed)
  unsigned long long* col_state;  // [n_cols] look-back words (zeroed)
  uint32_t epoch;
  long long* num_unique;
  long long* rank_bounds;
  uint32_t* occ_s;     // optional: occurrence -> key-sorted unique index
  uint32_t* seg_of;    // optional: sorted position -> key-sorted unique index
  uint32_t* occ_rank;  // optional: occurrence -> sorted position
  uint32_t* long_list;
  unsigned long long* num_long;
  long long long_cap;
};

__device__ __forceinline__ int rank_of_rb(long long p, const RankBounds& rb, int num_ranks) {
  int r = 0;
  while (r + 1 < num_ranks && p >= rb.v[r + 1]) ++r;
  return r;
}

// Debug (bp_debug_phase_trace 0): %globaltimer stamps of every CTA's phases,
// [column][16 CTAs][16 stamps].
__device__ unsigned long long* g_prep_trace = nullptr;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int IPT>
__global__ void __launch_bounds__(kCsThreads, 2) k_col_cluster_prep(const __grid_constant__ ColPrepArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int M = kCsThreads * IPT;
  extern __shared__ unsigned long long cs_smem[];
  unsigned long long* recv = cs_smem;                           // [M] this CTA's slice of the column
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(recv + M);       // [warps][256]
  uint32_t* hist = wcnt + kCsWarps * 256;                       // [256] published per-CTA counts
  uint32_t* off = hist + 256;                                   // [256]
  uint32_t* misc = off + 256;                                   // [32]
  uint32_t* headpos = misc + 32;                                // [M] slice index of the CTA's h-th head
  uint32_t* loff = headpos + M;                                 // [256] local digit offsets
  unsigned long long* stage = reinterpret_cast<unsigned long long*>(loff + 256);  // [M] locally sorted
  const int CS = (int)cluster.num_blocks();
  const int me = (int)cluster.block_rank();
  const int c = blockIdx.y;
  const int t = a.col_tables[c];
  const long long rows_t = a.rows[t];
  const long long base_t = a.base[t];
  const int bits = rows_t > 1 ? 64 - __clzll((unsigned long long)(rows_t - 1)) : 0;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const int n_ex = a.n_ex, n_cols = a.n_cols;
  unsigned long long* tr = g_prep_trace ? g_prep_trace + ((long long)c * 16 + me) * 16 : nullptr;
#define BP_STAMP(k) \
  if (tr && threadIdx.x == 0) tr[k] = gtimer()
  BP_STAMP(0);

  if (blockIdx.x == 0 && c == 0 && (int)threadIdx.x <= a.num_ranks) a.rank_bounds[threadIdx.x] = a.rb.v[threadIdx.x];

  // every key and label load in flight at once (the checks below may call
  // the error path, which would otherwise serialise the loads)
  unsigned long long e[IPT];
  uint32_t lab[IPT];
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const int ex = me * M + (int)(warp * (32 * IPT) + r * 32 + lane);
    const long long p = (long long)(ex < n_ex ? ex : 0) * n_cols + c;
    e[r] = __ldg(a.keys + p);
    lab[r] = __ldg(a.labels + p);
  }
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const int ex = me * M + (int)(warp * (32 * IPT) + r * 32 + lane);
    if (ex < n_ex) {
      const uint64_t key = e[r];
      uint64_t row = key & kRowMask;
      const bool bad_key = (int)(key >> kKeyTableShift) != t || (long long)row >= rows_t;
      if (bad_key || lab[r] > 127) {
        const long long p = (long long)ex * n_cols + c;
        if (bad_key) raise_error(a.err, BP_ERR_STORE_KEY, a.iteration, p, key);
        else raise_error(a.err, BP_ERR_CONFIG, a.iteration, p, 0);
        if (bad_key) row = 0;
      }
      e[r] = (row << kCsRowShift) | ((unsigned long long)(lab[r] & 0x7f) << 20) | (unsigned long long)ex;
    } else {
      e[r] = ~0ull;  // padding sorts last (stable: after any real all-ones digit)
    }
  }
  BP_STAMP(1);
  int pass = 0;

  for (int shift = kCsRowShift; shift < kCsRowShift + bits; shift += 8) {
    for (int i = lane; i < 256; i += 32) wcnt[warp * 256 + i] = 0;
    __syncwarp();
    uint32_t rank[IPT];
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
      const uint32_t d = (uint32_t)((e[r] >> shift) & 0xFFull);
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const unsigned below = peers & ((1u << lane) - 1u);
      const uint32_t prev = wcnt[warp * 256 + d];
      rank[r] = prev + (uint32_t)__popc(below);
      __syncwarp();
      if (below == 0) wcnt[warp * 256 + d] = prev + (uint32_t)__popc(peers);
      __syncwarp();
    }
    __syncthreads();
    {  // per digit: exclusive prefix over warps; the CTA's count is published
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < kCsWarps; ++w) {
        const uint32_t x = wcnt[w * 256 + threadIdx.x];
        wcnt[w * 256 + threadIdx.x] = run;
        run += x;
      }
      hist[threadIdx.x] = run;
    }
    cluster.sync();
    {  // column-wide offset of digit d in this CTA: all CTAs' smaller digits + lower CTAs' d
      uint32_t h[kCsMaxCluster];
#pragma unroll
      for (int r = 0; r < kCsMaxCluster; ++r)  // independent remote loads
        h[r] = r < CS ? *cluster.map_shared_rank(&hist[threadIdx.x], r) : 0u;
      uint32_t tot = 0, before = 0;
#pragma unroll
      for (int r = 0; r < kCsMaxCluster; ++r) {
        tot += h[r];
        before += r < me ? h[r] : 0u;
      }
      uint32_t block_total;
      const uint32_t incl = block_inclusive_scan_256(tot, misc, &block_total);
      off[threadIdx.x] = incl - tot + before;
      const uint32_t mine = hist[threadIdx.x];
      loff[threadIdx.x] = block_inclusive_scan_256(mine, misc, &block_total) - mine;
    }
    __syncthreads();
    // stable local sort by digit, then the slice is streamed out in local
    // order: consecutive threads hold consecutive elements of one digit's run,
    // whose destinations are consecutive too (coalesced DSMEM stores)
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
      const uint32_t d = (uint32_t)((e[r] >> shift) & 0xFFull);
      stage[loff[d] + wcnt[warp * 256 + d] + rank[r]] = e[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
      const uint32_t li = threadIdx.x + r * kCsThreads;
      const unsigned long long x = stage[li];
      const uint32_t d = (uint32_t)((x >> shift) & 0xFFull);
      const uint32_t dest = off[d] + (li - loff[d]);
      unsigned long long* rp = cluster.map_shared_rank(recv, (int)(dest / M));
      rp[dest % M] = x;
    }
    cluster.sync();
#pragma unroll
    for (int r = 0; r < IPT; ++r) e[r] = recv[warp * (32 * IPT) + r * 32 + lane];
    BP_STAMP(2 + (pass < 4 ? pass : 3));
    ++pass;
  }
  if (bits == 0) {
#pragma unroll
    for (int r = 0; r < IPT; ++r) recv[warp * (32 * IPT) + r * 32 + lane] = e[r];
  }
  cluster.sync();  // final slices visible to the neighbours
  BP_STAMP(6);

  // ---- segment heads and their numbering
  const unsigned long long left = me > 0 ? *cluster.map_shared_rank(&recv[M - 1], me - 1) : ~0ull;
  bool head[IPT];
  uint32_t pre[IPT];
  uint32_t wsum = 0;
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const int i = (int)(warp * (32 * IPT) + r * 32 + lane);
    const int j = me * M + i;
    const unsigned long long prev = i > 0 ? recv[i - 1] : left;
    head[r] = j < n_ex && (j == 0 || (prev >> kCsRowShift) != (e[r] >> kCsRowShift));
    const unsigned b = __ballot_sync(0xffffffffu, head[r]);
    pre[r] = wsum + (uint32_t)__popc(b & ((1u << lane) - 1u));
    wsum += (uint32_t)__popc(b);
  }
  if (lane == 0) off[warp] = wsum;
  if (threadIdx.x == 0) hist[1] = 0xFFFFFFFFu;  // column index of this CTA's first head (none yet)
  __syncthreads();
  uint32_t wbefore = 0, cta_heads = 0;
#pragma unroll
  for (int w = 0; w < kCsWarps; ++w) {
    const uint32_t x = off[w];
    wbefore += w < (int)warp ? x : 0u;
    cta_heads += x;
  }
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    if (!head[r]) continue;
    const uint32_t i = warp * (32 * IPT) + r * 32 + lane;
    headpos[wbefore + pre[r]] = i;
    if (wbefore + pre[r] == 0) hist[1] = (uint32_t)(me * M) + i;
  }
  if (threadIdx.x == 0) hist[0] = cta_heads;
  cluster.sync();
  uint32_t cbefore = 0, col_heads = 0;
  uint32_t next_first = (uint32_t)n_ex;  // first head after this CTA's slice: where its last segment ends
  {
    uint32_t h[kCsMaxCluster], f[kCsMaxCluster];
#pragma unroll
    for (int r = 0; r < kCsMaxCluster; ++r) {
      h[r] = r < CS ? *cluster.map_shared_rank(&hist[0], r) : 0u;
      f[r] = r < CS && r > me ? *cluster.map_shared_rank(&hist[1], r) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int r = 0; r < kCsMaxCluster; ++r) {
      col_heads += h[r];
      cbefore += r < me ? h[r] : 0u;
      next_first = f[r] < next_first ? f[r] : next_first;
    }
  }
  BP_STAMP(7);
  if (me == 0 && warp == 0) {
    // distinct keys of the columns before this one (decoupled look-back over
    // columns, one warp), broadcast to the cluster's CTAs
    const uint32_t colp = warp_lookback(a.col_state, c, a.epoch, col_heads);
    if (lane < (unsigned)CS) *cluster.map_shared_rank(&misc[16], (int)lane) = colp;
  }
  // ---- position outputs (independent of the segment numbering: written
  // while CTA 0 waits for the columns in front)
  const long long col0 = (long long)c * n_ex;
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const int i = (int)(warp * (32 * IPT) + r * 32 + lane);
    const int j = me * M + i;
    if (j >= n_ex) continue;
    const unsigned long long x = e[r];
    const long long p = (long long)(x & kCsExMask) * n_cols + c;
    const long long J = col0 + j;
    bool rs = head[r];
    if (!rs && a.num_ranks > 1) {
      const unsigned long long px = i > 0 ? recv[i - 1] : left;
      rs = rank_of_rb(p, a.rb, a.num_ranks) !=
           rank_of_rb((long long)(px & kCsExMask) * n_cols + c, a.rb, a.num_ranks);
    }
    a.occ_pos[J] = (uint32_t)p;
    a.occ_label[J] = (uint8_t)(((x >> 20) & 0x7f) | (rs ? 0x80 : 0));
    if (a.occ_rank) a.occ_rank[p] = (uint32_t)J;
  }
  cluster.sync();
  const uint32_t seg0 = misc[16] + cbefore + wbefore;
  BP_STAMP(8);

  // ---- segment outputs
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const int i = (int)(warp * (32 * IPT) + r * 32 + lane);
    const int j = me * M + i;
    if (j >= n_ex) continue;
    const unsigned long long x = e[r];
    const uint32_t ex = (uint32_t)(x & kCsExMask);
    const long long p = (long long)ex * n_cols + c;
    const long long J = col0 + j;
    const uint32_t s = seg0 + pre[r] + (head[r] ? 0u : (uint32_t)-1);  // inclusive segment index
    if (head[r]) {
      const uint64_t row = x >> kCsRowShift;
      a.seg_start[s] = (uint32_t)J;
      a.uniq_key_s[s] = ((uint64_t)t << kKeyTableShift) | row;
      a.uniq_id_s[s] = (uint32_t)(base_t + (long long)row);
      a.first_s[p] = s;
      atomicOr(&a.ex_mask[ex], 1u << c);
      // segment length from the next head (this slice's, else the first
      // head of a later slice of the column, else the column's end)
      const uint32_t lh = wbefore + pre[r];
      const uint32_t end = lh + 1 < cta_heads ? (uint32_t)(me * M) + headpos[lh + 1] : next_first;
      const uint32_t len = end - (uint32_t)j;
      if (len >= kVeryLongSeg) a.long_list[atomicAdd(&a.num_long[0], 1ull)] = s;
      else if (len >= kLongSeg) a.long_list[a.long_cap - 1 - (long long)atomicAdd(&a.num_long[1], 1ull)] = s;
    }
    if (a.occ_s) a.occ_s[p] = s;
    if (a.seg_of) a.seg_of[J] = s;
    if (c == n_cols - 1 && j == n_ex - 1) {
      const uint32_t U = misc[16] + col_heads;
      *a.num_unique = U;
      a.seg_start[U] = (uint32_t)((long long)n_cols * n_ex);
    }
  }
  BP_STAMP(9);
  BP_STAMP(10);
#undef BP_STAMP
}

// First-occurrence order (reference traces.py:91-103: examples in order, an
// example's keys in column order): k of the first occurrence at (ex, c) =
// first occurrences in earlier examples (block scan of the per-example mask
// popcounts + decoupled look-back over tiles of 256 examples) + set bits
// below c.  The tile's positions are then walked in order by all threads
// (coalesced, independent loads) to fill both permutations and the
// first-order keys (read from the batch itself: the key at position p).
__global__ void __launch_bounds__(kFirstThreads) k_first_order(const uint32_t* __restrict__ ex_mask,
                                                               const uint32_t* __restrict__ first_s,
                                                               const uint64_t* __restrict__ keys, int n_ex,
                                                               int n_cols, unsigned long long* state, uint32_t epoch,
                                                               uint32_t* __restrict__ perm_s2k,
                                                               uint32_t* __restrict__ perm_k2s,
                                                               uint64_t* __restrict__ uniq_key_k) {
  __shared__ uint32_t sh_warp[kFirstThreads / 32];
  __shared__ uint32_t sh_mask[kFirstThreads];
  __shared__ uint32_t sh_pfx[kFirstThreads];
  __shared__ uint32_t sh_prefix;
  const int ex0 = blockIdx.x * kFirstThreads;
  const int ex = ex0 + threadIdx.x;
  const uint32_t m = ex < n_ex ? ex_mask[ex] : 0u;
  const uint32_t cnt = (uint32_t)__popc(m);
  uint32_t block_total;
  const uint32_t excl = block_inclusive_scan_256(cnt, sh_warp, &block_total) - cnt;
  if (threadIdx.x < 32) {
    const uint32_t pfx = warp_lookback(state, blockIdx.x, epoch, block_total);
    if (threadIdx.x == 0) sh_prefix = pfx;
  }
  sh_mask[threadIdx.x] = m;
  sh_pfx[threadIdx.x] = excl;
  __syncthreads();
  const uint32_t tile_k0 = sh_prefix;
  // warp w walks examples [32w, 32w+32) of the tile, lane c = column c: the
  // loads of one example are consecutive positions, all issued up front
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const bool col_ok = (int)lane < n_cols;
  uint32_t sv[32];
  uint64_t kv[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int e = (int)warp * 32 + i;
    const bool first = col_ok && ex0 + e < n_ex && ((sh_mask[e] >> lane) & 1u);
    const long long p = (long long)(ex0 + e) * n_cols + lane;
    sv[i] = first ? __ldg(first_s + p) : 0u;
    kv[i] = first ? __ldg(keys + p) : 0ull;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int e = (int)warp * 32 + i;
    const uint32_t mm = sh_mask[e];
    if (!col_ok || ex0 + e >= n_ex || !((mm >> lane) & 1u)) continue;
    const uint32_t k = tile_k0 + sh_pfx[e] + (uint32_t)__popc(mm & ((1u << lane) - 1u));
    perm_s2k[sv[i]] = k;
    perm_k2s[k] = sv[i];
    uniq_key_k[k] = kv[i];
  }
}

__global__ void k_occ_k_from_s(const uint32_t* __restrict__ occ_s, long long n, const uint32_t* __restrict__ perm_s2k,
                               uint32_t* __restrict__ occ_k) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    occ_k[p] = perm_s2k[occ_s[p]];
}

static size_t cs_smem_bytes(int ipt) {
  return 2 * sizeof(unsigned long long) * kCsThreads * ipt +
         sizeof(uint32_t) * (kCsWarps * 256 + 256 + 256 + 32 + kCsThreads * ipt + 256);
}

// Cluster size and items per thread for n_ex examples per column; 0 if the
// cluster path does not apply.
static int g_prep_ipt_min = 8;  // debug knob (bp_debug_prep_shape): smallest items per thread tried

static bool cs_shape(int n_ex, int* cs, int* ipt) {
  for (int i : {4, 8, 16}) {
    if (i < g_prep_ipt_min) continue;
    for (int c = 1; c <= kCsMaxCluster; c <<= 1) {
      if ((long long)c * kCsThreads * i >= n_ex && (i != 8 || c <= 8)) {
        *cs = c;
        *ipt = i;
        return true;
      }
    }
  }
  return false;
}

__global__ void k_set_rank_bounds(RankBounds rb, int n, long long* out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = rb.v[i];
}

// Columnar prep on clusters: one memset (example masks, look-back words,
// long-list counters), the cluster sort-and-number kernel, the
// first-occurrence kernel (+ the occurrence -> first-order index on request).
static int prep_build_cluster(bp_prep* P, const bp_schema* sc, const uint64_t* d_keys, const uint8_t* d_labels,
                              const ColumnarInfo* col, const int64_t* h_rank_bounds, cudaStream_t s) {
  int cs = 0, ipt = 0;
  cs_shape(col->n_ex, &cs, &ipt);
  ColPrepArgs a;
  a.keys = d_keys;
  a.labels = d_labels;
  a.n_ex = col->n_ex;
  a.n_cols = col->n_cols;
  a.col_tables = col->d_tables;
  a.base = sc->d_table_base;
  a.rows = sc->d_rows;
  for (int i = 0; i <= P->num_ranks; ++i) a.rb.v[i] = h_rank_bounds[i];
  a.num_ranks = P->num_ranks;
  a.iteration = P->iteration;
  a.err = P->ctx ? P->ctx->d_err : nullptr;
  a.occ_pos = P->d_occ_pos;
  a.occ_label = P->d_occ_label;
  a.seg_start = P->d_seg_start;
  a.uniq_key_s = P->d_uniq_key_s;
  a.uniq_id_s = P->d_uniq_id_s;
  a.first_s = P->t_first_flag;
  a.ex_mask = P->t_ex_mask;
  a.col_state = P->t_col_state;
  a.epoch = next_scan_epoch();
  a.num_unique = P->d_num_unique;
  a.rank_bounds = P->d_rank_bounds;
  const bool occ_s_needed = (P->flags & (BP_PREP_OCC_INDEX | BP_PREP_OCC_SORTED)) != 0;
  a.occ_s = occ_s_needed ? (P->d_occ_s ? P->d_occ_s : P->t_va) : nullptr;
  a.seg_of = P->d_seg_of;
  a.occ_rank = P->d_occ_rank;
  a.long_list = P->d_long;
  a.num_long = (unsigned long long*)P->d_num_long;
  a.long_cap = P->long_cap;
  BP_CUDA_TRY(cudaMemsetAsync(P->d_num_long, 0, P->zero_bytes, s));
  const size_t smem = cs_smem_bytes(ipt);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, col->n_cols, 1);
  cfg.blockDim = dim3(kCsThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static bool attr_set = false;
  if (!attr_set) {
    BP_CUDA_TRY(cudaFuncSetAttribute(k_col_cluster_prep<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)cs_smem_bytes(8)));
    BP_CUDA_TRY(cudaFuncSetAttribute(k_col_cluster_prep<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)cs_smem_bytes(16)));
    BP_CUDA_TRY(cudaFuncSetAttribute(k_col_cluster_prep<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    BP_CUDA_TRY(cudaFuncSetAttribute(k_col_cluster_prep<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)cs_smem_bytes(4)));
    BP_CUDA_TRY(cudaFuncSetAttribute(k_col_cluster_prep<4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_set = true;
  }
  if (ipt == 4) BP_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_col_cluster_prep<4>, a));
  else if (ipt == 8) BP_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_col_cluster_prep<8>, a));
  else BP_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_col_cluster_prep<16>, a));
  const int tiles = (col->n_ex + kFirstThreads - 1) / kFirstThreads;
  k_first_order<<<tiles, kFirstThreads, 0, s>>>(P->t_ex_mask, P->t_first_flag, d_keys, col->n_ex, col->n_cols,
                                                P->t_tile_state, next_scan_epoch(), P->d_perm_s2k, P->d_perm_k2s,
                                                P->d_uniq_key_k);
  if (P->flags & BP_PREP_OCC_INDEX)
    k_occ_k_from_s<<<grid_for(P->n_occ, 256), 256, 0, s>>>(a.occ_s, P->n_occ, P->d_perm_s2k, P->d_occ_k);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

template <typename K>
static int prep_build(bp_prep* P, const bp_schema* sc, const uint64_t* d_keys, const uint8_t* d_labels,
                      int row_bits, int table_bits, cudaStream_t s, const ColumnarInfo* col) {
  const long long n = P->n_occ;
  K* ka = static_cast<K*>(P->t_ka);
  K* kb = static_cast<K*>(P->t_kb);
  uint32_t *va = P->t_va, *vb = P->t_vb, *hist = P->t_hist, *head = P->t_head, *segx = P->t_segx;
  uint32_t *first_flag = P->t_first_flag, *first_rank = P->t_first_rank, *partials = P->t_partials;
  const int g = grid_for(n, 256);
  int which = 0;
  if (col) {
    static bool attr_set = false;
    if (!attr_set) {
      BP_CUDA_TRY(cudaFuncSetAttribute(k_prep_table_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kColSmem));
      attr_set = true;
    }
    const int n_chunks = (col->n_ex + kColMax - 1) / kColMax;
    if (n_chunks == 1) {
      k_prep_table_sort<<<col->n_cols, kColThreads, kColSmem, s>>>(d_keys, col->n_ex, col->n_cols,
                                                                    sc->d_table_base, col->d_tables, col->row_bits,
                                                                    (uint32_t*)ka, va);
    } else {
      k_prep_table_sort<<<dim3(col->n_cols, n_chunks), kColThreads, kColSmem, s>>>(
          d_keys, col->n_ex, col->n_cols, sc->d_table_base, col->d_tables, col->row_bits, (uint32_t*)kb, vb);
      k_prep_col_merge<<<grid_for(n, 256), 256, 0, s>>>((const uint32_t*)kb, vb, col->n_ex, col->n_cols, n_chunks,
                                                        (uint32_t*)ka, va);
    }
    which = 0;
  } else if (P->schema_mode) {
    k_prep_keys_schema<<<g, 256, 0, s>>>(d_keys, n, sc->d_table_base, sc->d_rows, sc->num_tables,
                                         (uint32_t*)ka, va, P->ctx ? P->ctx->d_err : nullptr, P->iteration);
    BP_CUDA_TRY(radix_sort_pairs<K>(ka, va, kb, vb, n, nullptr, 0, sc->id_bits, hist, partials, &which, s));
  } else {
    k_prep_keys_packed<<<g, 256, 0, s>>>(d_keys, n, (uint64_t*)ka, va);
    int w1 = 0, w2 = 0;
    BP_CUDA_TRY(radix_sort_pairs<K>(ka, va, kb, vb, n, nullptr, 0, row_bits, hist, partials, &w1, s));
    K* k1 = w1 ? kb : ka;
    uint32_t* v1 = w1 ? vb : va;
    K* k2 = w1 ? ka : kb;
    uint32_t* v2 = w1 ? va : vb;
    BP_CUDA_TRY(radix_sort_pairs<K>(k1, v1, k2, v2, n, nullptr, kKeyTableShift, kKeyTableShift + table_bits, hist,
                                    partials, &w2, s));
    which = w1 ^ w2;
  }
  const K* skey = which ? kb : ka;
  const uint32_t* spos = which ? vb : va;
  BP_CUDA_TRY(cudaMemcpyAsync(P->d_occ_pos, spos, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));

  k_prep_heads<K><<<g, 256, 0, s>>>(skey, n, head);
  BP_CUDA_TRY(exclusive_scan(head, segx, n, nullptr, partials, nullptr, P->d_num_unique, s));
  BP_CUDA_TRY(cudaMemsetAsync(first_flag, 0, n * sizeof(uint32_t), s));
  k_prep_segments<K><<<g, 256, 0, s>>>(skey, P->d_occ_pos, head, segx, n, d_keys, d_labels, P->schema_mode,
                                       P->d_seg_start, P->d_uniq_key_s, P->d_uniq_id_s, first_flag,
                                       P->d_occ_label, P->d_num_unique, P->d_rank_bounds, P->num_ranks,
                                       P->ctx ? P->ctx->d_err : nullptr, P->iteration);
  BP_CUDA_TRY(exclusive_scan(first_flag, first_rank, n, nullptr, partials, nullptr, nullptr, s));
  BP_CUDA_TRY(cudaMemsetAsync(P->d_num_long, 0, 2 * sizeof(long long), s));
  k_prep_perm<<<g, 256, 0, s>>>(P->d_occ_pos, head, segx, first_rank, n, P->d_uniq_key_s, P->d_perm_s2k,
                                P->d_perm_k2s, P->d_uniq_key_k, P->d_seg_start, P->d_long,
                                (unsigned long long*)P->d_num_long, P->long_cap);
  if (P->flags & (BP_PREP_OCC_INDEX | BP_PREP_OCC_SORTED))
    k_prep_occ_k<<<g, 256, 0, s>>>(P->d_occ_pos, head, segx, n, P->d_perm_s2k, P->d_occ_k, P->d_occ_s,
                                   P->d_seg_of, P->d_occ_rank);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

// Byte layout of a prep's arena (base == nullptr: size only).
struct Carve {
  char* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

static size_t prep_layout(bp_prep* P, char* base, long long n, int num_ranks, int flags, const ColumnarInfo* cl) {
  Carve c{base};
  P->d_num_unique = c.take<long long>(1);
  P->d_uniq_key_s = c.take<uint64_t>(n);
  P->d_uniq_id_s = c.take<uint32_t>(n);
  P->d_uniq_key_k = c.take<uint64_t>(n);
  P->d_perm_s2k = c.take<uint32_t>(n);
  P->d_perm_k2s = c.take<uint32_t>(n);
  P->d_seg_start = c.take<uint32_t>(n + 1);
  P->d_occ_pos = c.take<uint32_t>(n);
  P->d_occ_label = c.take<uint8_t>(n + 16);  // read as 16-byte chunks
  P->d_occ_k = (flags & BP_PREP_OCC_INDEX) ? c.take<uint32_t>(n) : nullptr;
  P->d_occ_s = (flags & BP_PREP_OCC_SORTED) ? c.take<uint32_t>(n) : nullptr;
  P->d_seg_of = (flags & BP_PREP_OCC_SORTED) ? c.take<uint32_t>(n) : nullptr;
  P->d_occ_rank = (flags & BP_PREP_OCC_SORTED) ? c.take<uint32_t>(n) : nullptr;
  P->d_rank_bounds = c.take<long long>(num_ranks + 1);
  P->long_cap = n / kLongSeg + 1;
  P->d_long = c.take<uint32_t>(P->long_cap);
  if (cl) {
    // cluster path: the temporaries are one segment index per occurrence and
    // a zeroed block (long-list counters, example masks, look-back words)
    // cleared by ONE memset starting at d_num_long
    const size_t zero0 = c.off = (c.off + 255) & ~size_t(255);
    P->d_num_long = reinterpret_cast<long long*>(base ? base + c.off : nullptr);
    c.off += 2 * sizeof(long long);
    P->t_ex_mask = c.take<uint32_t>(cl->n_ex);
    P->t_col_state = c.take<unsigned long long>((size_t)cl->n_cols * kLookbackStride);
    P->t_tile_state = c.take<unsigned long long>((size_t)((cl->n_ex + kFirstThreads - 1) / kFirstThreads) *
                                                 kLookbackStride);
    P->zero_bytes = c.off - zero0;
    P->t_first_flag = c.take<uint32_t>(n);
    P->t_va = (flags & BP_PREP_OCC_INDEX) && !(flags & BP_PREP_OCC_SORTED) ? c.take<uint32_t>(n) : nullptr;
    P->t_ka = P->t_kb = nullptr;
    P->t_vb = P->t_hist = P->t_head = P->t_segx = P->t_first_rank = P->t_partials = nullptr;
    return c.off;
  }
  P->d_num_long = c.take<long long>(2);
  P->t_ex_mask = nullptr;
  P->t_col_state = P->t_tile_state = nullptr;
  P->zero_bytes = 0;
  P->t_ka = c.take<uint64_t>(n);
  P->t_kb = c.take<uint64_t>(n);
  P->t_va = c.take<uint32_t>(n);
  P->t_vb = c.take<uint32_t>(n);
  P->t_hist = c.take<uint32_t>(sort_hist_words(n));
  P->t_head = c.take<uint32_t>(n);
  P->t_segx = c.take<uint32_t>(n);
  P->t_first_flag = c.take<uint32_t>(n);
  P->t_first_rank = c.take<uint32_t>(n);
  P->t_partials = c.take<uint32_t>((long long)sort_partials_words(n) + scan_state_words(n));
  return c.off;
}

}  // namespace bp

static int prep_create_impl(bp_ctx* ctx, const bp_schema* sc, const uint64_t* d_keys, const uint8_t* d_labels,
                            int64_t n_occ, const int64_t* h_rank_bounds, int32_t num_ranks, int64_t iteration,
                            int32_t flags, int32_t row_bits, int32_t table_bits, bp_stream_t stream, bp_prep** out,
                            const bp::ColumnarInfo* col) {
  using namespace bp;
  if (n_occ < 0 || num_ranks < 1 || n_occ >= (int64_t)kNoId) return BP_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  bp_prep* P = new bp_prep();
  P->ctx = ctx;
  P->n_occ = n_occ;
  P->iteration = iteration;
  P->num_ranks = num_ranks;
  P->flags = flags;
  P->schema_mode = sc != nullptr;
  P->stream = s;
  P->h_num_unique = n_occ == 0 ? 0 : -1;
  const long long n = n_occ > 0 ? n_occ : 1;
  const ColumnarInfo* cl = (col && n_occ > 0 && col->cluster) ? col : nullptr;
  const size_t bytes = prep_layout(P, nullptr, n, num_ranks, flags, cl);
  void* arena = nullptr;
  BP_CUDA_TRY(cudaMallocAsync(&arena, bytes, s));
  P->d_arena = arena;
  prep_layout(P, static_cast<char*>(arena), n, num_ranks, flags, cl);
  if (cl) {
    const int rc = prep_build_cluster(P, sc, d_keys, d_labels, cl, h_rank_bounds, s);
    if (rc != BP_OK) return rc;
    *out = P;
    return BP_OK;
  }
  if (num_ranks + 1 <= RankBounds::kMax) {
    // by value as a kernel parameter: a pageable H2D copy would first wait
    // for the whole stream (host-blocking)
    RankBounds rb;
    for (int i = 0; i <= num_ranks; ++i) rb.v[i] = h_rank_bounds[i];
    k_set_rank_bounds<<<1, 32, 0, s>>>(rb, num_ranks + 1, P->d_rank_bounds);
  } else {
    // The pageable H2D copy is staged by the driver before returning, so the
    // caller's rank-bounds array may be released immediately.
    BP_CUDA_TRY(cudaMemcpyAsync(P->d_rank_bounds, h_rank_bounds, sizeof(long long) * (num_ranks + 1),
                                cudaMemcpyHostToDevice, s));
  }
  if (n_occ == 0) {
    BP_CUDA_TRY(cudaMemsetAsync(P->d_num_long, 0, 2 * sizeof(long long), s));
    BP_CUDA_TRY(cudaMemsetAsync(P->d_num_unique, 0, sizeof(long long), s));
    BP_CUDA_TRY(cudaMemsetAsync(P->d_seg_start, 0, sizeof(uint32_t), s));
    *out = P;
    return BP_OK;
  }
  int rc;
  if (sc) {
    rc = prep_build<uint32_t>(P, sc, d_keys, d_labels, 0, 0, s, col);
  } else {
    if (row_bits < 1) row_bits = 1;
    if (table_bits < 1) table_bits = 1;
    if (row_bits > kKeyTableShift || table_bits > 64 - kKeyTableShift) return BP_ERR_INVALID;
    rc = prep_build<uint64_t>(P, nullptr, d_keys, d_labels, row_bits, table_bits, s, nullptr);
  }
  if (rc != BP_OK) return rc;
  *out = P;
  return BP_OK;
}

extern "C" int bp_prep_create(bp_ctx* ctx, const bp_schema* sc, const uint64_t* d_keys, const uint8_t* d_labels,
                              int64_t n_occ, const int64_t* h_rank_bounds, int32_t num_ranks, int64_t iteration,
                              int32_t flags, int32_t row_bits, int32_t table_bits, bp_stream_t stream,
                              bp_prep** out) {
  return prep_create_impl(ctx, sc, d_keys, d_labels, n_occ, h_rank_bounds, num_ranks, iteration, flags, row_bits,
                          table_bits, stream, out, nullptr);
}

// Columnar batch: keys laid out [n_ex][n_cols], column c holding table
// h_tables[c] (strictly increasing).  Takes the per-column shared-memory
// sort (chunks of 16,384 examples merged by rank above that), else the
// generic path.
extern "C" int bp_prep_create_columnar(bp_ctx* ctx, const bp_schema* sc, const uint64_t* d_keys,
                                       const uint8_t* d_labels, int64_t n_ex, int32_t n_cols, const int32_t* d_tables,
                                       const int64_t* h_rank_bounds, int32_t num_ranks, int64_t iteration,
                                       int32_t flags, bp_stream_t stream, bp_prep** out) {
  using namespace bp;
  if (!sc || n_cols < 1 || n_ex < 0) return BP_ERR_INVALID;
  const int64_t n_occ = n_ex * n_cols;
  if (n_ex > kColMax * kColMaxChunks || n_ex == 0)
    return prep_create_impl(ctx, sc, d_keys, d_labels, n_occ, h_rank_bounds, num_ranks, iteration, flags, 0, 0,
                            stream, out, nullptr);
  int64_t max_rows = 1;
  for (int t = 0; t < sc->num_tables; ++t)
    max_rows = std::max<int64_t>(max_rows, sc->h_table_base[t + 1] - sc->h_table_base[t]);
  const int row_bits = std::max(1, bit_width_u64((unsigned long long)(max_rows - 1)));
  if (row_bits > 44 - 14) return BP_ERR_INVALID;
  int cs = 0, ipt = 0;
  const bool cluster = g_prep_cluster && n_cols <= kCsMaxCols && row_bits <= kCsMaxRowBits &&
                       num_ranks + 1 <= RankBounds::kMax && cs_shape((int)n_ex, &cs, &ipt);
  const ColumnarInfo col{(int)n_ex, n_cols, row_bits, d_tables, cluster};
  return prep_create_impl(ctx, sc, d_keys, d_labels, n_occ, h_rank_bounds, num_ranks, iteration, flags, 0, 0, stream,
                          out, &col);
}

extern "C" int bp_prep_destroy(bp_prep* P) {
  if (!P) return BP_OK;
  cudaFreeAsync(P->d_arena, P->stream);
  delete P;
  return BP_OK;
}

extern "C" int bp_prep_get_view(const bp_prep* P, bp_prep_view* v) {
  v->n_occ = P->n_occ;
  v->iteration = P->iteration;
  v->num_ranks = P->num_ranks;
  v->pad = 0;
  v->d_num_unique = (const int64_t*)P->d_num_unique;
  v->d_uniq_key_s = P->d_uniq_key_s;
  v->d_uniq_id_s = P->d_uniq_id_s;
  v->d_uniq_key_k = P->d_uniq_key_k;
  v->d_perm_s2k = P->d_perm_s2k;
  v->d_perm_k2s = P->d_perm_k2s;
  v->d_seg_start = P->d_seg_start;
  v->d_occ_pos = P->d_occ_pos;
  v->d_occ_label = P->d_occ_label;
  v->d_occ_k = P->d_occ_k;
  v->d_rank_bounds = (const int64_t*)P->d_rank_bounds;
  return BP_OK;
}

extern "C" int bp_prep_num_unique(bp_prep* P, bp_stream_t stream, int64_t* h_out) {
  if (P->h_num_unique < 0) {
    long long u = 0;
    BP_CUDA_TRY(cudaMemcpyAsync(&u, P->d_num_unique, sizeof(long long), cudaMemcpyDeviceToHost,
                                (cudaStream_t)stream));
    BP_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    P->h_num_unique = u;
  }
  *h_out = P->h_num_unique;
  return BP_OK;
}

// 1 (default): Criteo-layout batches use the cluster prep; 0: the per-column
// single-CTA sort (kept as the reference implementation for tests).
// Debug: phase timestamps (%globaltimer, ns) of kernel `which` into d_buf
// (NULL disables): 0 = k_col_cluster_prep [column][16][16], 1 = k_pop_fused
// [tile][8].
extern "C" int bp_debug_phase_trace(int32_t which, void* d_buf) {
  if (which == 0) BP_CUDA_TRY(cudaMemcpyToSymbol(bp::g_prep_trace, &d_buf, sizeof(void*)));
  else if (which == 1) return bp_debug_pop_trace(d_buf);
  else return BP_ERR_INVALID;
  return BP_OK;
}

extern "C" int bp_debug_prep_cluster(int32_t on) {
  bp::g_prep_cluster = on ? 1 : 0;
  return BP_OK;
}

// Debug/tuning: smallest items per thread of the cluster prep (4, 8 or 16;
// with 4 a 16,384-example column is spread over 16 CTAs instead of 8).
extern "C" int bp_debug_prep_shape(int32_t ipt_min) {
  if (ipt_min != 4 && ipt_min != 8 && ipt_min != 16) return BP_ERR_INVALID;
  bp::g_prep_ipt_min = ipt_min;
  return BP_OK;
}
