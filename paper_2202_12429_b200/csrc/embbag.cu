// EmbeddingBag forward / backward + sparse optimizer over the HBM cache
// (north-star piece 4, DLRM mode).  The reference has no model (its trainer
// is the stub of trainer.py), so parity for this mode is against a PyTorch
// fp32 CPU model (nn.EmbeddingBag + the same MLPs) within a tolerance.
//
// Both kernels walk the batch prep's key-sorted CSR (prep.cu): every cached
// row is read (forward) or read-modified-written (backward) exactly once per
// batch, however many times the key occurs.
//
//   forward, single-key bags (Criteo layout: one key per table per example,
//   bag = occurrence position): one G-lane group per unique key loads the
//   row once and scatters it to all of the key's occurrence rows of
//   pooled[n_occ][dim] -- N_occ x 64 B of writes, U x 64 B of reads.
//   forward, multi-key bags: per bag, sum (or mean) of its keys' rows.
//   backward: per unique key, g = sum over its occurrences of the bag
//   gradient rows (x 1/|bag| for mean), then SGD (v -= lr g) or Adagrad
//   (a += g^2; v -= lr g / (sqrt(a) + eps)) in place; optimizer state lives
//   in the second half of the row (row stride 2*dim), so it travels with the
//   row through eviction and write-back.  Keys with >= kLongSeg occurrences
//   are reduced by whole CTAs (16 partial sums, fixed-order tree: run-to-run
//   deterministic).
#include "internal.cuh"

namespace bp {

constexpr int kBagLongBlocks = 128;
constexpr int kSpanWarpTiles = 32;         // spanning keys up to this many tiles: a warp each
constexpr int kSpanSmallBlocks = 148 * 2;  // CTAs of k_embbag_bwd_span on those (the rest: a CTA per key)

// Single-key bags: pooled[p] = cached row of occurrence p's key, one 16-byte
// lane per (occurrence, 4 components): coalesced pooled writes in occurrence
// order, row reads from the (L2-resident) cache arena, no per-key serial loop
// (a Zipf-hot key has ~9K occurrences per Criteo-Kaggle batch).
template <int QT>  // QT > 0: the float4s per row at compile time (shifts instead of divisions); 0: runtime q
__global__ void __launch_bounds__(256) k_embbag_fwd_rows_v4(const uint32_t* __restrict__ occ_s,
                                                           const int32_t* __restrict__ slots_s,
                                                           const float4* __restrict__ values, int q_rt,
                                                           int row_q, long long n, float4* __restrict__ out) {
  // 4 elements per thread, their three dependent loads (unique index, slot,
  // row) issued as batches so the latency chain is paid once per 4 rows
  constexpr int U = 4;
  const int q = QT > 0 ? QT : q_rt;
  const long long total = n * q;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total; i0 += stride * U) {
    uint32_t u[U];
    int32_t sl[U];
    float4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = i0 + k * stride;
      u[k] = i < total ? __ldg(occ_s + i / q) : 0u;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) sl[k] = i0 + k * stride < total ? __ldg(slots_s + u[k]) : -1;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = i0 + k * stride;
      const int c = (int)(i % q);
      v[k] = sl[k] >= 0 ? values[(long long)sl[k] * row_q + c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = i0 + k * stride;
      if (i < total) out[i] = v[k];
    }
  }
}

// Same output from the key-sorted side: one float4 lane per (sorted position
// j, 4 components); segment id and slot loads are coalesced (consecutive j
// share a key, so its row is read once into L1 and broadcast), and the row
// is stored to its occurrence position occ_pos[j] -- 64-byte scattered
// stores, which never stall the thread, instead of a random 4-byte slot
// gather per occurrence.
__global__ void __launch_bounds__(256) k_embbag_fwd_sorted_v4(const uint32_t* __restrict__ seg_of,
                                                             const uint32_t* __restrict__ occ_pos,
                                                             const int32_t* __restrict__ slots_s,
                                                             const float4* __restrict__ values, int q, int row_q,
                                                             long long n, float4* __restrict__ out) {
  constexpr int U = 4;
  const long long total = n * q;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total; i0 += stride * U) {
    uint32_t sg[U], pos[U];
    int32_t sl[U];
    float4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = i0 + k * stride;
      const long long j = i / q;
      sg[k] = i < total ? seg_of[j] : 0u;
      pos[k] = i < total ? occ_pos[j] : 0u;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) sl[k] = i0 + k * stride < total ? slots_s[sg[k]] : -1;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = i0 + k * stride;
      const int c = (int)(i - (i / q) * q);
      v[k] = sl[k] >= 0 ? values[(long long)sl[k] * row_q + c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = i0 + k * stride;
      if (i < total) out[(long long)pos[k] * q + (i - (i / q) * q)] = v[k];
    }
  }
}

static int g_fwd_variant = 0;  // debug: 0 = occurrence-order gather, 1 = key-sorted scatter

extern "C" int bp_debug_fwd_variant(int32_t v) {
  g_fwd_variant = v;
  return BP_OK;
}

// Gradient / row source in a peer example owner's [bl][t_global][Q] buffer
// (csrc/peer.cu); rows == nullptr: local gradient rows.
struct PeerSrc {
  float4* const* rows;
  const int32_t* col_tables;
  long long bl;
  int t_global;
  int n_cols;
  float scale;
};

__device__ __forceinline__ float4* peer_row(const PeerSrc& ps, long long p, int q) {
  const long long b = p / ps.n_cols;
  const int j = (int)(p - b * ps.n_cols);
  const long long r = b / ps.bl;
  return ps.rows[r] + ((b - r * ps.bl) * ps.t_global + ps.col_tables[j]) * q;
}

// Forward fused with the all-to-all: pooled row of occurrence p (example b,
// local column j) stored straight into example owner b / bl's buffer at its
// global-table column, over NVLink.
template <int QT>  // QT > 0: float4s per row at compile time; 0: runtime q
__global__ void __launch_bounds__(256) k_embbag_fwd_peer_v4(const uint32_t* __restrict__ occ_s,
                                                           const int32_t* __restrict__ slots_s,
                                                           const float4* __restrict__ values, int q_rt, int row_q,
                                                           long long n, PeerSrc dst) {
  constexpr int U = 4;  // four independent (index, slot, row) chains per thread
  const int q = QT > 0 ? QT : q_rt;
  const long long total = n * q;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total; i0 += stride * U) {
    int32_t sl[U];
    float4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = i0 + k * stride;
      sl[k] = i < total ? __ldg(slots_s + __ldg(occ_s + i / q)) : -1;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = i0 + k * stride;
      v[k] = sl[k] >= 0 ? values[(long long)sl[k] * row_q + (int)(i % q)] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = i0 + k * stride;
      if (i < total) peer_row(dst, i / q, q)[i % q] = v[k];
    }
  }
}

template <int G, int DPL>
__global__ void __launch_bounds__(256) k_embbag_fwd_gather(const uint32_t* __restrict__ occ_s,
                                                           const int32_t* __restrict__ slots_s,
                                                           const float* __restrict__ values,
                                                           const int64_t* __restrict__ bag_offsets, long long n_bags,
                                                           int dim, int row_stride, int mean,
                                                           float* __restrict__ out) {
  const int lane_g = (int)(threadIdx.x & (G - 1));
  const long long groups_total = (long long)gridDim.x * (blockDim.x / G);
  for (long long bag = (long long)blockIdx.x * (blockDim.x / G) + threadIdx.x / G; bag < n_bags;
       bag += groups_total) {
    const long long lo = bag_offsets[bag], hi = bag_offsets[bag + 1];
    float acc[DPL];
#pragma unroll
    for (int q = 0; q < DPL; ++q) acc[q] = 0.f;
    for (long long p = lo; p < hi; ++p) {
      const int32_t slot = slots_s[occ_s[p]];
      if (slot < 0) continue;
#pragma unroll
      for (int q = 0; q < DPL; ++q) {
        const int d = lane_g + q * G;
        if (d < dim) acc[q] = __fadd_rn(acc[q], values[(long long)slot * row_stride + d]);
      }
    }
    const float scale = (mean && hi > lo) ? __frcp_rn((float)(hi - lo)) : 1.f;
#pragma unroll
    for (int q = 0; q < DPL; ++q) {
      const int d = lane_g + q * G;
      if (d < dim) out[bag * dim + d] = mean ? __fmul_rn(acc[q], scale) : acc[q];
    }
  }
}

struct BagGrad {
  const float* grad;        // [n_bags][dim]
  const int64_t* occ_bag;   // bag of each occurrence position (NULL: identity)
  const float* bag_scale;   // per bag multiplier (NULL: 1), e.g. 1/|bag| for mean
};

__device__ __forceinline__ float grad_at(const BagGrad& g, long long p, int d, int dim) {
  const long long bag = g.occ_bag ? g.occ_bag[p] : p;
  const float x = g.grad[bag * dim + d];
  return g.bag_scale ? __fmul_rn(x, g.bag_scale[bag]) : x;
}

template <int DPL>
__device__ __forceinline__ void apply_update(float* __restrict__ row, const float (&g)[DPL], int lane_g, int G, int dim,
                                             int opt, float lr, float eps, bool& nonzero) {
#pragma unroll
  for (int q = 0; q < DPL; ++q) {
    const int d = lane_g + q * G;
    if (d >= dim) continue;
    nonzero |= g[q] != 0.f;
    const float v = row[d];
    if (opt == BP_OPT_ADAGRAD) {
      const float a = __fadd_rn(row[dim + d], __fmul_rn(g[q], g[q]));
      row[dim + d] = a;
      row[d] = __fsub_rn(v, __fdiv_rn(__fmul_rn(lr, g[q]), __fadd_rn(__fsqrt_rn(a), eps)));
    } else {
      row[d] = __fsub_rn(v, __fmul_rn(lr, g[q]));
    }
  }
}

template <int G, int DPL>
__global__ void __launch_bounds__(256) k_embbag_bwd(const uint32_t* __restrict__ seg_start,
                                                    const uint32_t* __restrict__ occ_pos,
                                                    const long long* __restrict__ d_U,
                                                    const uint32_t* __restrict__ long_list,
                                                    const long long* __restrict__ d_num_long, long long long_cap,
                                                    BagGrad bg, float* __restrict__ values,
                                                    const int32_t* __restrict__ slots_s, uint8_t* __restrict__ dirty,
                                                    int dim, int row_stride, int opt, float lr, float eps,
                                                    unsigned long long* __restrict__ stats) {
  const unsigned lane = threadIdx.x & 31u;
  if (blockIdx.x < kBagLongBlocks) {
    // whole-CTA reduction of a long segment: 256/G partial sums, fixed tree
    __shared__ float part[256 / 1 * 4];
    const long long n_vlong = d_num_long[0], n_long = n_vlong + d_num_long[1];
    const int groups = 256 / G;
    const int grp = threadIdx.x / G, lane_g = threadIdx.x & (G - 1);
    for (long long li = blockIdx.x; li < n_long; li += kBagLongBlocks) {
      const uint32_t s = li < n_vlong ? long_list[li] : long_list[long_cap - 1 - (li - n_vlong)];
      const uint32_t a = seg_start[s], b = seg_start[s + 1];
      const int32_t slot = slots_s[s];
      if (slot < 0) continue;
      float acc[DPL];
#pragma unroll
      for (int q = 0; q < DPL; ++q) acc[q] = 0.f;
      for (uint32_t j = a + grp; j < b; j += groups) {
        const long long p = occ_pos[j];
#pragma unroll
        for (int q = 0; q < DPL; ++q) {
          const int d = lane_g + q * G;
          if (d < dim) acc[q] = __fadd_rn(acc[q], grad_at(bg, p, d, dim));
        }
      }
#pragma unroll
      for (int q = 0; q < DPL; ++q) part[(grp * G + lane_g) * DPL + q] = acc[q];
      __syncthreads();
      for (int width = groups / 2; width > 0; width >>= 1) {
        if (grp < width) {
#pragma unroll
          for (int q = 0; q < DPL; ++q)
            part[(grp * G + lane_g) * DPL + q] =
                __fadd_rn(part[(grp * G + lane_g) * DPL + q], part[((grp + width) * G + lane_g) * DPL + q]);
        }
        __syncthreads();
      }
      if (threadIdx.x < 32) {
        bool nonzero = false;
        if (threadIdx.x < G) {
          float g[DPL];
#pragma unroll
          for (int q = 0; q < DPL; ++q) g[q] = part[threadIdx.x * DPL + q];
          apply_update<DPL>(values + (long long)slot * row_stride, g, threadIdx.x, G, dim, opt, lr, eps, nonzero);
        }
        const bool nz = __ballot_sync(0xffffffffu, nonzero) != 0;
        if (threadIdx.x == 0) {
          if (nz && dirty) dirty[slot] = 1;
          if (nz && stats) atomicAdd(&stats[1], 1ull);
        }
      }
      __syncthreads();
    }
    return;
  }
  const long long U = *d_U;
  const int lane_g = (int)(lane & (G - 1));
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(unsigned)(G - 1)));
  const long long groups_per_block = blockDim.x / G;
  const long long groups_total = (long long)(gridDim.x - kBagLongBlocks) * groups_per_block;
  const long long warp_first =
      (long long)(blockIdx.x - kBagLongBlocks) * groups_per_block + (threadIdx.x >> 5) * (32 / G);
  for (long long base = warp_first; base < U; base += groups_total) {
    const long long s = base + (long long)(lane / G);
    bool active = s < U;
    uint32_t a = 0, b = 0;
    int32_t slot = -1;
    if (active) {
      a = seg_start[s];
      b = seg_start[s + 1];
      slot = slots_s[s];
      active = slot >= 0 && b - a < kLongSeg;
    }
    bool nonzero = false;
    if (active) {
      float g[DPL];
#pragma unroll
      for (int q = 0; q < DPL; ++q) g[q] = 0.f;
      for (uint32_t j = a; j < b; ++j) {
        const long long p = occ_pos[j];
#pragma unroll
        for (int q = 0; q < DPL; ++q) {
          const int d = lane_g + q * G;
          if (d < dim) g[q] = __fadd_rn(g[q], grad_at(bg, p, d, dim));
        }
      }
      apply_update<DPL>(values + (long long)slot * row_stride, g, lane_g, G, dim, opt, lr, eps, nonzero);
    }
    const unsigned nz = __ballot_sync(0xffffffffu, nonzero) & gmask;
    if (active && lane_g == 0 && nz && dirty) dirty[slot] = 1;
    if (stats) {
      const unsigned dm = __ballot_sync(0xffffffffu, active && lane_g == 0 && nz != 0);
      if (lane == 0 && dm) atomicAdd(&stats[1], (unsigned long long)__popc(dm));
    }
  }
}

// Backward as a tiled reduce-by-key over the key-sorted occurrence order
// (dim % 4 == 0; needs the prep's seg_of, BP_PREP_OCC_SORTED).  Tile b holds
// sorted positions [b*T, b*T+T) (T*dim/4 = 2048 float4 = 32 KB): the CTA
// gathers the T gradient rows into shared memory (16-byte loads, all issued
// before any add), runs a segmented Hillis-Steele scan, and at the last row
// of every key in the tile holds that key's partial sum.  A key wholly inside
// the tile is updated right there; a key spanning tiles (the Zipf-hot rows:
// ~9K occurrences = 18 tiles at Criteo-Kaggle) leaves one partial per tile
// that k_embbag_bwd_span combines in a fixed order and applies.  Every summation order is fixed by the data, not by
// scheduling, so the result is run-to-run deterministic; all occurrence work
// is parallel (no per-key dependent chains as in the stub trainer, whose
// order is pinned by the reference).
constexpr int kBwdTileF4 = 2048;
constexpr int kBwdPer = kBwdTileF4 / 256;

__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

__device__ __forceinline__ float upd1(float v, float& a, float g, int opt, float lr, float eps) {
  if (opt == BP_OPT_ADAGRAD) {
    a = __fadd_rn(a, __fmul_rn(g, g));
    return __fsub_rn(v, __fdiv_rn(__fmul_rn(lr, g), __fadd_rn(__fsqrt_rn(a), eps)));
  }
  return __fsub_rn(v, __fmul_rn(lr, g));
}

__device__ __forceinline__ bool apply_row4(float* __restrict__ row, int dim, int c, float4 g, int opt, float lr,
                                           float eps) {
  float4* v4 = reinterpret_cast<float4*>(row) + c;
  float4 v = *v4;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  float4* a4 = reinterpret_cast<float4*>(row + dim) + c;
  if (opt == BP_OPT_ADAGRAD) a = *a4;
  v.x = upd1(v.x, a.x, g.x, opt, lr, eps);
  v.y = upd1(v.y, a.y, g.y, opt, lr, eps);
  v.z = upd1(v.z, a.z, g.z, opt, lr, eps);
  v.w = upd1(v.w, a.w, g.w, opt, lr, eps);
  *v4 = v;
  if (opt == BP_OPT_ADAGRAD) *a4 = a;
  return g.x != 0.f || g.y != 0.f || g.z != 0.f || g.w != 0.f;
}

__global__ void __launch_bounds__(256) k_embbag_bwd_tiles(
    const uint32_t* __restrict__ occ_pos, const uint32_t* __restrict__ seg_of, const uint32_t* __restrict__ seg_start,
    long long n, int q, int T, const float4* __restrict__ grad, const int64_t* __restrict__ occ_bag,
    const float* __restrict__ bag_scale, float* __restrict__ values, int row_stride,
    const int32_t* __restrict__ slots_s, uint8_t* __restrict__ dirty, int opt, float lr, float eps,
    float4* __restrict__ parts, unsigned long long* __restrict__ stats, uint32_t* __restrict__ span_list,
    unsigned int* __restrict__ span_count, long long span_cap) {
  extern __shared__ float4 tile[];  // [T*q] gradient rows, then [T] segment ids
  uint32_t* seg = reinterpret_cast<uint32_t*>(tile + kBwdTileF4);
  __shared__ unsigned int n_dirty;
  const long long t0 = (long long)blockIdx.x * T;
  const int rows = (int)min((long long)T, n - t0);
  const int dim = 4 * q;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  long long pk[kBwdPer];
#pragma unroll
  for (int k = 0; k < kBwdPer; ++k) {
    const int i = threadIdx.x + k * 256, r = i / q;
    pk[k] = r < rows ? (long long)occ_pos[t0 + r] : -1;
  }
  if (occ_bag) {
#pragma unroll
    for (int k = 0; k < kBwdPer; ++k)
      if (pk[k] >= 0) pk[k] = occ_bag[pk[k]];
  }
  float4 v[kBwdPer];
#pragma unroll
  for (int k = 0; k < kBwdPer; ++k) {
    const int i = threadIdx.x + k * 256, c = i - (i / q) * q;
    v[k] = pk[k] >= 0 ? grad[pk[k] * q + c] : zero;
  }
  if (bag_scale) {
#pragma unroll
    for (int k = 0; k < kBwdPer; ++k)
      if (pk[k] >= 0) {
        const float sc = bag_scale[pk[k]];
        v[k] = make_float4(__fmul_rn(v[k].x, sc), __fmul_rn(v[k].y, sc), __fmul_rn(v[k].z, sc), __fmul_rn(v[k].w, sc));
      }
  }
#pragma unroll
  for (int k = 0; k < kBwdPer; ++k) tile[threadIdx.x + k * 256] = v[k];
  for (int r = threadIdx.x; r < T; r += 256) seg[r] = r < rows ? seg_of[t0 + r] : 0xffffffffu;
  if (threadIdx.x == 0) n_dirty = 0;
  __syncthreads();
  for (int off = 1; off < rows; off <<= 1) {
    bool take[kBwdPer];
#pragma unroll
    for (int k = 0; k < kBwdPer; ++k) {
      const int i = threadIdx.x + k * 256, r = i / q;
      take[k] = r >= off && r < rows && seg[r - off] == seg[r];
      if (take[k]) v[k] = tile[i - off * q];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kBwdPer; ++k) {
      const int i = threadIdx.x + k * 256;
      if (take[k]) tile[i] = f4_add(tile[i], v[k]);
    }
    __syncthreads();
  }
  unsigned my_dirty = 0;
  for (int r = threadIdx.x; r < rows; r += 256) {
    const uint32_t s = seg[r];
    if (r + 1 < rows && seg[r + 1] == s) continue;  // not this key's last row in the tile
    const int32_t slot = slots_s[s];
    if (slot < 0) continue;
    const long long a = seg_start[s], b = seg_start[s + 1];
    float* row = values + (long long)slot * row_stride;
    bool nz = false;
    if (a >= t0 && b <= t0 + rows) {
      for (int c = 0; c < q; ++c) nz |= apply_row4(row, dim, c, tile[r * q + c], opt, lr, eps);
    } else {  // spans tiles: leave this tile's partial for k_embbag_bwd_span
      float4* dst = parts + ((long long)blockIdx.x * 2 + (s == seg[0] ? 0 : 1)) * q;
      for (int c = 0; c < q; ++c) dst[c] = tile[r * q + c];
      if (a >= t0) {  // the key's first tile: list it for k_embbag_bwd_span
        const bool big = (b - 1) / T - (long long)blockIdx.x + 1 > kSpanWarpTiles;
        span_list[(big ? span_cap : 0) + atomicAdd(span_count + (big ? 1 : 0), 1u)] = blockIdx.x;
      }
    }
    if (nz) {
      if (dirty) dirty[slot] = 1;
      ++my_dirty;
    }
  }
  if (stats && my_dirty) atomicAdd(&n_dirty, my_dirty);
  __syncthreads();
  if (stats && threadIdx.x == 0 && n_dirty) atomicAdd(&stats[1], (unsigned long long)n_dirty);
}

// Warp tiles (dim 4..32, the DLRM shapes): one warp reduces T = 32 * R
// sorted positions (R = 8 / Q rows per lane, Q float4 per row), entirely in
// registers: per-lane segmented sum over its R rows, then a segmented
// Hillis-Steele scan of the lanes' last-segment partials with shuffles
// (element (has_head, value), earlier + later), then the carry-in of each
// lane's first segment.  No shared memory, no barriers; every order is fixed.
template <int Q>
__global__ void __launch_bounds__(256) k_embbag_bwd_warp(
    const uint32_t* __restrict__ occ_pos, const uint32_t* __restrict__ seg_of, const uint32_t* __restrict__ seg_start,
    long long n, const float4* __restrict__ grad, const int64_t* __restrict__ occ_bag,
    const float* __restrict__ bag_scale, float* __restrict__ values, int row_stride,
    const int32_t* __restrict__ slots_s, uint8_t* __restrict__ dirty, int opt, float lr, float eps,
    float4* __restrict__ parts, unsigned long long* __restrict__ stats, PeerSrc src,
    uint32_t* __restrict__ span_list, unsigned int* __restrict__ span_count, long long span_cap) {
  constexpr int R = 8 / Q, T = 32 * R;
  const unsigned lane = threadIdx.x & 31u;
  const long long tile = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long t0 = tile * T;
  if (t0 >= n) return;
  const long long r0 = t0 + (long long)lane * R;
  uint32_t sg[R];
  long long pk[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const bool ok = r0 + j < n;
    sg[j] = ok ? seg_of[r0 + j] : 0xffffffffu;
    pk[j] = ok ? (long long)occ_pos[r0 + j] : -1;
  }
  if (occ_bag) {
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (pk[j] >= 0) pk[j] = occ_bag[pk[j]];
  }
  // which of this lane's rows end a key's run in the tile, and that key's
  // slot / CSR bounds: loaded now, in flight with the gradient loads, and the
  // cached row pulled into L2 -- the update after the scan then waits on L2
  // instead of a chain of DRAM round trips
  const uint32_t next_first = __shfl_down_sync(0xffffffffu, sg[0], 1);
  bool endj[R];
  int32_t slotj[R];
  long long aj[R], bj[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    endj[j] = r0 + j < n &&
              ((j < R - 1) ? sg[j + 1] != sg[j] : (lane == 31 || r0 + j + 1 >= n || next_first != sg[j]));
    slotj[j] = endj[j] ? slots_s[sg[j]] : -1;
    aj[j] = endj[j] ? (long long)seg_start[sg[j]] : 0;
    bj[j] = endj[j] ? (long long)seg_start[sg[j] + 1] : 0;
  }
  float4 v[R][Q];
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  if (src.rows) {  // gradient rows in the example owners' buffers (NVLink loads)
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const float4* row = pk[j] >= 0 ? peer_row(src, pk[j], Q) : nullptr;
#pragma unroll
      for (int c = 0; c < Q; ++c) v[j][c] = row ? row[c] : zero;
    }
    if (src.scale != 1.f) {
#pragma unroll
      for (int j = 0; j < R; ++j)
#pragma unroll
        for (int c = 0; c < Q; ++c)
          v[j][c] = make_float4(__fmul_rn(v[j][c].x, src.scale), __fmul_rn(v[j][c].y, src.scale),
                                __fmul_rn(v[j][c].z, src.scale), __fmul_rn(v[j][c].w, src.scale));
    }
  } else {
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int c = 0; c < Q; ++c) v[j][c] = pk[j] >= 0 ? grad[pk[j] * Q + c] : zero;
  }
  if (bag_scale) {
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (pk[j] >= 0) {
        const float sc = bag_scale[pk[j]];
#pragma unroll
        for (int c = 0; c < Q; ++c)
          v[j][c] = make_float4(__fmul_rn(v[j][c].x, sc), __fmul_rn(v[j][c].y, sc), __fmul_rn(v[j][c].z, sc),
                                __fmul_rn(v[j][c].w, sc));
      }
  }
#pragma unroll
  for (int j = 0; j < R; ++j)
    if (slotj[j] >= 0)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(values + (long long)slotj[j] * row_stride));
  // per-lane inclusive segmented sums
  bool inner_head = false;
#pragma unroll
  for (int j = 1; j < R; ++j) {
    if (sg[j] == sg[j - 1]) {
#pragma unroll
      for (int c = 0; c < Q; ++c) v[j][c] = f4_add(v[j - 1][c], v[j][c]);
    } else {
      inner_head = true;
    }
  }
  const uint32_t prev_last = __shfl_up_sync(0xffffffffu, sg[R - 1], 1);
  const bool first_head = lane == 0 || sg[0] != prev_last;
  // segmented inclusive scan over lanes of (flag, last-segment partial)
  bool flag = first_head || inner_head;
  float4 agg[Q];
#pragma unroll
  for (int c = 0; c < Q; ++c) agg[c] = v[R - 1][c];
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const bool fo = __shfl_up_sync(0xffffffffu, flag ? 1 : 0, off) != 0;
#pragma unroll
    for (int c = 0; c < Q; ++c) {
      float4 o;
      o.x = __shfl_up_sync(0xffffffffu, agg[c].x, off);
      o.y = __shfl_up_sync(0xffffffffu, agg[c].y, off);
      o.z = __shfl_up_sync(0xffffffffu, agg[c].z, off);
      o.w = __shfl_up_sync(0xffffffffu, agg[c].w, off);
      if (lane >= (unsigned)off && !flag) agg[c] = f4_add(o, agg[c]);
    }
    if (lane >= (unsigned)off) flag = flag || fo;
  }
  // carry-in for the first segment of this lane = previous lane's inclusive aggregate
  float4 carry[Q];
#pragma unroll
  for (int c = 0; c < Q; ++c) {
    carry[c].x = __shfl_up_sync(0xffffffffu, agg[c].x, 1);
    carry[c].y = __shfl_up_sync(0xffffffffu, agg[c].y, 1);
    carry[c].z = __shfl_up_sync(0xffffffffu, agg[c].z, 1);
    carry[c].w = __shfl_up_sync(0xffffffffu, agg[c].w, 1);
  }
  if (!first_head) {
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (sg[j] == sg[0]) {
#pragma unroll
        for (int c = 0; c < Q; ++c) v[j][c] = f4_add(carry[c], v[j][c]);
      }
  }
  const uint32_t tile_first = __shfl_sync(0xffffffffu, sg[0], 0);
  const long long rows = min((long long)T, n - t0);
  const int dim = 4 * Q;
  unsigned n_nz = 0;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (!endj[j]) continue;
    const uint32_t s = sg[j];
    const int32_t slot = slotj[j];
    if (slot < 0) continue;
    const long long a = aj[j], b = bj[j];
    if (a >= t0 && b <= t0 + rows) {
      float* row = values + (long long)slot * row_stride;
      bool nz = false;
#pragma unroll
      for (int c = 0; c < Q; ++c) nz |= apply_row4(row, dim, c, v[j][c], opt, lr, eps);
      if (nz) {
        if (dirty) dirty[slot] = 1;
        ++n_nz;
      }
    } else {  // spans tiles: this tile's partial for k_embbag_bwd_span
      float4* dst = parts + (tile * 2 + (s == tile_first ? 0 : 1)) * Q;
#pragma unroll
      for (int c = 0; c < Q; ++c) dst[c] = v[j][c];
      if (a >= t0) {  // the key's first tile: list it for k_embbag_bwd_span
        const bool big = (b - 1) / T - tile + 1 > kSpanWarpTiles;
        span_list[(big ? span_cap : 0) + atomicAdd(span_count + (big ? 1 : 0), 1u)] = (uint32_t)tile;
      }
    }
  }
  if (stats) {
    for (int off = 16; off > 0; off >>= 1) n_nz += __shfl_down_sync(0xffffffffu, n_nz, off);
    if (lane == 0 && n_nz) atomicAdd(&stats[1], (unsigned long long)n_nz);
  }
}

// Backward over gradient rows already in key-sorted order: the producer (the
// fused interaction backward, csrc/interact.cu) stored occurrence p's row at
// its sorted position occ_rank[p], so the random 64-byte gradient gather of
// k_embbag_bwd_warp becomes a contiguous stream and the kernel is a pure
// segmented reduce.  Warp tile = T = G * R sorted rows; lane = (row group g,
// float4 column c): Q lanes per row, G = 32 / Q groups of R consecutive rows,
// so every load instruction covers G whole rows with fully used sectors.
// Per lane a sequential segmented sum over its R rows, a segmented scan
// across the groups (shuffles by Q), the carry-in of each group's first run;
// each key ending in the tile is then updated by its Q lanes (one 16-byte
// column each).  Only the tile's first and last runs can span tiles; their
// bounds come from two broadcast loads.  A spanning key leaves one partial
// per tile and counts its tiles on an arrival counter at its first tile: the
// warp that completes the count sums all partials in ascending tile order
// (groups stride the tiles, fixed shuffle tree) and applies the update -- no
// second launch, and the order is fixed by the data: run-to-run
// deterministic.
constexpr int kSortedRows = 8;  // rows per lane group in k_embbag_bwd_sorted

template <int Q>
__device__ __forceinline__ bool span_combine(const float4* __restrict__ parts, uint32_t ft, uint32_t nt, bool mid,
                                             int g, int c, float* __restrict__ row, int opt, float lr, float eps) {
  constexpr int G = 32 / Q;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 acc = zero;
  bool any = false;
  for (uint32_t k = g; k < nt; k += G) {
    const uint32_t half = (k == 0 && mid) ? 1u : 0u;
    const float4 x = __ldcg(parts + (size_t)((ft + k) * 2 + half) * Q + c);
    acc = any ? f4_add(acc, x) : x;
    any = true;
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) {
    float4 o;
    o.x = __shfl_down_sync(0xffffffffu, acc.x, off * Q);
    o.y = __shfl_down_sync(0xffffffffu, acc.y, off * Q);
    o.z = __shfl_down_sync(0xffffffffu, acc.z, off * Q);
    o.w = __shfl_down_sync(0xffffffffu, acc.w, off * Q);
    const bool ao = __shfl_down_sync(0xffffffffu, any ? 1 : 0, off * Q) != 0;
    if (g < off && ao) {
      acc = any ? f4_add(acc, o) : o;
      any = true;
    }
  }
  return g == 0 && apply_row4(row, 4 * Q, c, acc, opt, lr, eps);
}

template <int Q, int R, int MINB>
__global__ void __launch_bounds__(256, MINB) k_embbag_bwd_sorted(
    const uint32_t* __restrict__ seg_of, const uint32_t* __restrict__ seg_start, uint32_t n,
    const float4* __restrict__ grad, float* __restrict__ values, int row_stride, const int32_t* __restrict__ slots_s,
    uint8_t* __restrict__ dirty, int opt, float lr, float eps, float4* __restrict__ parts,
    unsigned int* __restrict__ arrivals, unsigned long long* __restrict__ stats) {
  constexpr int G = 32 / Q, T = G * R;
  const unsigned lane = threadIdx.x & 31u;
  const int c = (int)lane % Q, g = (int)lane / Q;
  const uint32_t tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint32_t t0 = tile * T;
  if (t0 >= n) return;
  const uint32_t rows = min((uint32_t)T, n - t0);
  const uint32_t r0 = t0 + g * R;  // first row of this lane's group
  uint32_t sg[R];
  if (r0 + R <= n) {
    if constexpr (R % 4 == 0) {
#pragma unroll
      for (int k = 0; k < R / 4; ++k) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(seg_of + r0) + k);
        sg[4 * k] = x.x, sg[4 * k + 1] = x.y, sg[4 * k + 2] = x.z, sg[4 * k + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < R; ++j) sg[j] = seg_of[r0 + j];
    }
  } else {
#pragma unroll
    for (int j = 0; j < R; ++j) sg[j] = r0 + j < n ? seg_of[r0 + j] : 0xffffffffu;
  }
  const uint32_t tile_first = seg_of[t0], tile_last = seg_of[t0 + rows - 1];
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 v[R];
#pragma unroll
  for (int j = 0; j < R; ++j) v[j] = r0 + j < n ? __ldcs(grad + (size_t)(r0 + j) * Q + c) : zero;
  // bounds of the two runs that may span tiles (broadcast loads)
  const uint32_t fa = seg_start[tile_first], fb = seg_start[tile_first + 1];
  const uint32_t la = seg_start[tile_last], lb = seg_start[tile_last + 1];
  // rows ending a key's run in the tile: slot loaded now, the cached row
  // pulled into L2 while the scan runs
  const uint32_t next_first = __shfl_down_sync(0xffffffffu, sg[0], Q);
  int32_t slotj[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const bool e = r0 + j < n && ((j < R - 1) ? sg[j + 1] != sg[j] : (g == G - 1 || next_first != sg[j]));
    slotj[j] = e ? slots_s[sg[j]] : -1;
  }
#pragma unroll
  for (int j = 0; j < R; ++j)
    if (c == 0 && slotj[j] >= 0)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(values + (size_t)slotj[j] * row_stride));
  bool inner_head = false;
#pragma unroll
  for (int j = 1; j < R; ++j) {
    if (sg[j] == sg[j - 1]) v[j] = f4_add(v[j - 1], v[j]);
    else inner_head = true;
  }
  const uint32_t prev_last = __shfl_up_sync(0xffffffffu, sg[R - 1], Q);
  const bool first_head = g == 0 || sg[0] != prev_last;
  bool flag = first_head || inner_head;
  float4 agg = v[R - 1];
#pragma unroll
  for (int off = 1; off < G; off <<= 1) {
    const bool fo = __shfl_up_sync(0xffffffffu, flag ? 1 : 0, off * Q) != 0;
    float4 o;
    o.x = __shfl_up_sync(0xffffffffu, agg.x, off * Q);
    o.y = __shfl_up_sync(0xffffffffu, agg.y, off * Q);
    o.z = __shfl_up_sync(0xffffffffu, agg.z, off * Q);
    o.w = __shfl_up_sync(0xffffffffu, agg.w, off * Q);
    if (g >= off && !flag) agg = f4_add(o, agg);
    if (g >= off) flag = flag || fo;
  }
  float4 carry;
  carry.x = __shfl_up_sync(0xffffffffu, agg.x, Q);
  carry.y = __shfl_up_sync(0xffffffffu, agg.y, Q);
  carry.z = __shfl_up_sync(0xffffffffu, agg.z, Q);
  carry.w = __shfl_up_sync(0xffffffffu, agg.w, Q);
  if (!first_head) {
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (sg[j] == sg[0]) v[j] = f4_add(carry, v[j]);
  }
  const unsigned gm = (Q == 32 ? 0xffffffffu : ((1u << Q) - 1u)) << (g * Q);
  // spanning keys: the tile's first run if its key extends past either tile
  // edge, the last run (a different key) if it continues in a later tile
  const bool span1 = fa < t0 || fb > t0 + rows;
  const bool span2 = tile_last != tile_first && lb > t0 + rows;
  // spanning partials first, then their arrivals: the release fence waits
  // only for these stores, not for the row updates below
  bool wrote = false;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (slotj[j] >= 0 && (sg[j] == tile_first ? span1 : (sg[j] == tile_last && span2))) {
      parts[(size_t)(tile * 2 + (sg[j] == tile_first ? 0 : 1)) * Q + c] = v[j];
      slotj[j] = -1;  // not an in-tile update
      wrote = true;
    }
  }
  unsigned last = 0;  // bit k: this warp completed spanning key k's arrivals
  if (span1 || span2) {
    if (wrote) __threadfence();
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (!(k == 0 ? span1 : span2)) continue;
        // a key not in the cache (slot < 0) is skipped on every tile: no partials, no arrivals
        if (slots_s[k == 0 ? tile_first : tile_last] < 0) continue;
        const uint32_t a = k == 0 ? fa : la, b = k == 0 ? fb : lb;
        const uint32_t ft = a / T, nt = (b - 1) / T - ft + 1;
        if (atomicAdd(arrivals + ft, 1u) == nt - 1) last |= 1u << k;
      }
    }
    last = __shfl_sync(0xffffffffu, last, 0);
  }
  // in-tile keys: the row loads of a batch of end rows issued before any of
  // its stores (the compiler cannot move loads across possibly aliasing stores)
  unsigned n_nz = 0;
  constexpr int B = R < 4 ? R : 4;
#pragma unroll
  for (int j0 = 0; j0 < R; j0 += B) {
    float4 w[B], acc[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int32_t sl = slotj[j0 + u];
      const float4* row = reinterpret_cast<const float4*>(values + (size_t)(sl >= 0 ? sl : 0) * row_stride);
      w[u] = sl >= 0 ? row[c] : zero;
      acc[u] = (sl >= 0 && opt == BP_OPT_ADAGRAD) ? row[Q + c] : zero;
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int32_t sl = slotj[j0 + u];
      bool nz = false;
      if (sl >= 0) {
        const float4 gg = v[j0 + u];
        float4 x = w[u], a = acc[u];
        x.x = upd1(x.x, a.x, gg.x, opt, lr, eps);
        x.y = upd1(x.y, a.y, gg.y, opt, lr, eps);
        x.z = upd1(x.z, a.z, gg.z, opt, lr, eps);
        x.w = upd1(x.w, a.w, gg.w, opt, lr, eps);
        float4* row = reinterpret_cast<float4*>(values + (size_t)sl * row_stride);
        row[c] = x;
        if (opt == BP_OPT_ADAGRAD) row[Q + c] = a;
        nz = gg.x != 0.f || gg.y != 0.f || gg.z != 0.f || gg.w != 0.f;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, nz);
      if (sl >= 0 && c == 0 && (bal & gm)) {
        if (dirty) dirty[sl] = 1;
        ++n_nz;
      }
    }
  }
  // the warp that completed a spanning key's arrivals combines its partials
  // (ascending tiles, fixed tree) and applies the update
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    if (!((last >> k) & 1u)) continue;  // warp-uniform
    __threadfence();
    const uint32_t key = k == 0 ? tile_first : tile_last;
    const uint32_t a = k == 0 ? fa : la, b = k == 0 ? fb : lb;
    const uint32_t ft = a / T, nt = (b - 1) / T - ft + 1;
    const int32_t slot = slots_s[key];
    const bool nz = span_combine<Q>(parts, ft, nt, a != ft * T, g, c, values + (size_t)slot * row_stride, opt, lr,
                                    eps);
    if (__ballot_sync(0xffffffffu, nz) != 0 && lane == 0) {
      if (dirty) dirty[slot] = 1;
      ++n_nz;
    }
  }
  if (stats) {
    for (int off = 16; off > 0; off >>= 1) n_nz += __shfl_down_sync(0xffffffffu, n_nz, off);
    if (lane == 0 && n_nz) atomicAdd(&stats[1], (unsigned long long)n_nz);
  }
}

// Staged backward over sorted gradients (the default of
// bp_embbag_backward_sorted): a CTA owns a 32 KB tile of T = 2048/Q sorted
// rows, pulled into shared memory by one bulk async copy (TMA engine,
// mbarrier completion) together with its segment ids -- no per-thread load
// queues.  While the copy is in flight the CTA stages the cache slots of the
// tile's keys (a contiguous range of unique ids) in shared memory and pulls
// their rows into L2.  In shared memory: 256/Q lane groups of T/(256/Q)
// consecutive rows turn their rows into running segmented sums in place; a
// two-level segmented scan of the group totals (warp shuffles, then the 8
// warp totals in a fixed sequential order) gives each group its carry-in;
// then every (row, column) item of a key's last row in the tile applies the
// update (cache-row loads batched ahead of their stores).  Spanning keys:
// partials + arrival counters as in k_embbag_bwd_sorted.  Fixed orders
// throughout: run-to-run deterministic.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

constexpr int kStagedF4 = 2048;  // float4 per k_embbag_bwd_staged tile (32 KB)

template <int Q, int NT = 256, int F4 = kStagedF4, bool ENDS = true>
__global__ void __launch_bounds__(NT, 3 * 256 / NT) k_embbag_bwd_staged(
    const uint32_t* __restrict__ seg_of, const uint32_t* __restrict__ seg_start, uint32_t n,
    const float4* __restrict__ grad, float* __restrict__ values, int row_stride, const int32_t* __restrict__ slots_s,
    uint8_t* __restrict__ dirty, int opt, float lr, float eps, float4* __restrict__ parts,
    unsigned int* __restrict__ arrivals, unsigned long long* __restrict__ stats) {
  constexpr int T = F4 / Q, NG = NT / Q, RPG = T / NG, GW = 32 / Q, NW = NT / 32;
  extern __shared__ __align__(128) unsigned char st_smem[];
  float4* tile = reinterpret_cast<float4*>(st_smem);          // [T][Q]
  uint32_t* sgs = reinterpret_cast<uint32_t*>(tile + T * Q);  // [T]
  int32_t* tslot = reinterpret_cast<int32_t*>(sgs + T);          // [T] cache slots of the tile's keys
  __shared__ __align__(8) uint64_t bar;
  __shared__ float4 gcarry[NG][Q];
  __shared__ float4 wagg[NW][Q];
  __shared__ int wflag[NW][Q];
  __shared__ uint8_t ghead[NG];
  // rows that end a key's run inside the tile (pass 1 records them, pass 3
  // walks only those: ~T/6 at Criteo-Kaggle shape instead of every row)
  __shared__ uint16_t ends[ENDS ? T : 1];
  __shared__ uint32_t n_ends;
  const uint32_t t0 = blockIdx.x * T;
  const uint32_t rows = min((uint32_t)T, n - t0);
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    if (ENDS) n_ends = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const uint32_t seg_bytes = (rows / 4) * 16;  // whole 16-byte chunks of segment ids
  if (tid == 0) {
    const uint32_t gbytes = rows * Q * 16;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"(gbytes + seg_bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(tile)),
                 "l"(grad + (size_t)t0 * Q), "r"(gbytes), "r"(smem_u32(&bar))
                 : "memory");
    if (seg_bytes)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(sgs)),
                   "l"(seg_of + t0), "r"(seg_bytes), "r"(smem_u32(&bar))
                   : "memory");
  }
  // meanwhile: the bounds of the tile's first and last runs, and the cache
  // slots of its keys -- a contiguous range of unique ids -- staged in shared
  // memory, their rows pulled into L2 for the updates
  const uint32_t tile_first = seg_of[t0], tile_last = seg_of[t0 + rows - 1];
  const uint32_t fa = seg_start[tile_first], fb = seg_start[tile_first + 1];
  const uint32_t la = seg_start[tile_last], lb = seg_start[tile_last + 1];
  const uint32_t nu = tile_last - tile_first + 1;
  for (uint32_t i = tid; i < nu; i += NT) {
    const int32_t sl = slots_s[tile_first + i];
    tslot[i] = sl;
    if (sl >= 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(values + (size_t)sl * row_stride));
  }
  if (tid < rows - seg_bytes / 4) sgs[seg_bytes / 4 + tid] = seg_of[t0 + seg_bytes / 4 + tid];  // < 4 tail ids
  asm volatile(
      "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT%=;\n}\n" ::"r"(
          smem_u32(&bar))
      : "memory");
  __syncthreads();  // the tail segment ids
  const int c = (int)(tid % Q), gi = (int)(tid / Q), w = (int)(tid >> 5), gw = (int)((tid & 31) / Q);
  const uint32_t r0 = gi * RPG;
  // pass 1: running segmented sums of the group's rows, in place
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 acc = zero;
  bool flag = false;
  if (r0 < rows) {
    uint32_t ps = sgs[r0];
    acc = tile[r0 * Q + c];
    flag = r0 == 0 || sgs[r0 - 1] != ps;
    if (c == 0) ghead[gi] = flag ? 1 : 0;
    const uint32_t re = min(r0 + RPG, rows);
    for (uint32_t r = r0 + 1; r < re; ++r) {
      const uint32_t sr = sgs[r];
      const float4 x = tile[r * Q + c];
      if (sr == ps) {
        acc = f4_add(acc, x);
      } else {
        if (ENDS && c == 0) ends[atomicAdd(&n_ends, 1u)] = (uint16_t)(r - 1);  // row r-1 ends its run
        acc = x;
        flag = true;
      }
      tile[r * Q + c] = acc;
      ps = sr;
    }
    if (ENDS && c == 0 && (re == rows || sgs[re] != ps)) ends[atomicAdd(&n_ends, 1u)] = (uint16_t)(re - 1);
  } else if (c == 0) {
    ghead[gi] = 1;
  }
  // pass 2: segmented scan of the group totals; warp level first
  float4 inc = acc;
  bool finc = flag;
#pragma unroll
  for (int off = 1; off < GW; off <<= 1) {
    const bool fo = __shfl_up_sync(0xffffffffu, finc ? 1 : 0, off * Q) != 0;
    float4 o;
    o.x = __shfl_up_sync(0xffffffffu, inc.x, off * Q);
    o.y = __shfl_up_sync(0xffffffffu, inc.y, off * Q);
    o.z = __shfl_up_sync(0xffffffffu, inc.z, off * Q);
    o.w = __shfl_up_sync(0xffffffffu, inc.w, off * Q);
    if (gw >= off && !finc) inc = f4_add(o, inc);
    if (gw >= off) finc = finc || fo;
  }
  if (gw == GW - 1) {
    wagg[w][c] = inc;
    wflag[w][c] = finc ? 1 : 0;
  }
  // exclusive (within the warp) value for this group
  float4 ex;
  ex.x = __shfl_up_sync(0xffffffffu, inc.x, Q);
  ex.y = __shfl_up_sync(0xffffffffu, inc.y, Q);
  ex.z = __shfl_up_sync(0xffffffffu, inc.z, Q);
  ex.w = __shfl_up_sync(0xffffffffu, inc.w, Q);
  const bool fex = __shfl_up_sync(0xffffffffu, finc ? 1 : 0, Q) != 0;
  __syncthreads();
  // carry into this warp: the warp totals before it, in order
  float4 cw = zero;
  for (int k = 0; k < w; ++k) cw = wflag[k][c] ? wagg[k][c] : f4_add(cw, wagg[k][c]);
  const float4 carry = gw == 0 ? cw : (fex ? ex : f4_add(cw, ex));
  gcarry[gi][c] = carry;
  __syncthreads();
  // spanning keys of the tile
  const bool span1 = fa < t0 || fb > t0 + rows;
  const bool span2 = tile_last != tile_first && lb > t0 + rows;
  // pass 3: (row, column) items; a key's last row in the tile holds its sum
  unsigned my_nz = 0;
  bool wrote = false;
  constexpr int ITEMS = T * Q / NT, B = 4;
  const int n_items = ENDS ? (int)((n_ends + NG - 1) / NG) : ITEMS;
#pragma unroll 1
  for (int k0 = 0; k0 < n_items; k0 += B) {
    int32_t sl[B];
    float4 val[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      sl[u] = -1;
      uint32_t r;
      if (ENDS) {
        const uint32_t e = (uint32_t)(tid / Q) + (uint32_t)(k0 + u) * NG;
        if (e >= n_ends) continue;
        r = ends[e];
      } else {
        r = (uint32_t)(tid / Q) + (uint32_t)(k0 + u) * NG;
      }
      if (r >= rows) continue;
      const uint32_t s = sgs[r];
      if (!ENDS && r + 1 < rows && sgs[r + 1] == s) continue;  // not the last row of its run
      const int32_t slot = tslot[s - tile_first];
      if (slot < 0) continue;
      const uint32_t g = r / RPG;
      float4 x = tile[r * Q + c];
      if (!ghead[g] && s == sgs[g * RPG]) x = f4_add(gcarry[g][c], x);
      if (s == tile_first ? span1 : (s == tile_last && span2)) {
        parts[(size_t)(blockIdx.x * 2 + (s == tile_first ? 0 : 1)) * Q + c] = x;
        wrote = true;
        continue;
      }
      sl[u] = slot;
      val[u] = x;
    }
    float4 wv[B], av[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const float4* row = reinterpret_cast<const float4*>(values + (size_t)(sl[u] >= 0 ? sl[u] : 0) * row_stride);
      wv[u] = sl[u] >= 0 ? row[c] : zero;
      av[u] = (sl[u] >= 0 && opt == BP_OPT_ADAGRAD) ? row[Q + c] : zero;
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      bool nz = false;
      if (sl[u] >= 0) {
        const float4 gg = val[u];
        float4 x = wv[u], a = av[u];
        x.x = upd1(x.x, a.x, gg.x, opt, lr, eps);
        x.y = upd1(x.y, a.y, gg.y, opt, lr, eps);
        x.z = upd1(x.z, a.z, gg.z, opt, lr, eps);
        x.w = upd1(x.w, a.w, gg.w, opt, lr, eps);
        float4* row = reinterpret_cast<float4*>(values + (size_t)sl[u] * row_stride);
        row[c] = x;
        if (opt == BP_OPT_ADAGRAD) row[Q + c] = a;
        nz = gg.x != 0.f || gg.y != 0.f || gg.z != 0.f || gg.w != 0.f;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, nz);
      const unsigned gm = (Q == 32 ? 0xffffffffu : ((1u << Q) - 1u)) << ((tid & 31) / Q * Q);
      if (sl[u] >= 0 && c == 0 && (bal & gm)) {
        if (dirty) dirty[sl[u]] = 1;
        ++my_nz;
      }
    }
  }
  // stats: one atomic per CTA (same-address atomics serialise in L2)
  if (stats) cta_add(&stats[1], my_nz);
  if (span1 || span2) {
    // partials visible device-wide, then warp 0 alone counts the arrivals and
    // (if it completed a key) combines; the other warps are done
    if (wrote) __threadfence();
    __syncthreads();
    if (w != 0) return;
    unsigned lst = 0;
    if (tid == 0) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (!(k == 0 ? span1 : span2)) continue;
        if (tslot[k == 0 ? 0 : nu - 1] < 0) continue;
        const uint32_t a = k == 0 ? fa : la, b = k == 0 ? fb : lb;
        const uint32_t ft = a / T, nt = (b - 1) / T - ft + 1;
        if (atomicAdd(arrivals + ft, 1u) == nt - 1) {
          lst |= 1u << k;
          arrivals[ft] = 0;  // every arrival is in: the counter is free again (persistent scratch)
        }
      }
    }
    lst = __shfl_sync(0xffffffffu, lst, 0);
    if (!lst) return;
    __threadfence();
    unsigned n_comb = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!((lst >> k) & 1u)) continue;
      const uint32_t key = k == 0 ? tile_first : tile_last;
      const uint32_t a = k == 0 ? fa : la, b = k == 0 ? fb : lb;
      const uint32_t ft = a / T, nt = (b - 1) / T - ft + 1;
      const int32_t slot = tslot[key - tile_first];
      const bool nz = span_combine<Q>(parts, ft, nt, a != ft * T, (int)(tid / Q), c,
                                      values + (size_t)slot * row_stride, opt, lr, eps);
      if (__ballot_sync(0xffffffffu, nz) != 0 && tid == 0) {
        if (dirty) dirty[slot] = 1;
        ++n_comb;
      }
    }
    if (stats && tid == 0 && n_comb) atomicAdd(&stats[1], (unsigned long long)n_comb);
  }
}

// Persistent, pipelined form of k_embbag_bwd_staged (variant 5): a grid
// of 2 CTAs per SM walks the tiles t = blockIdx.x + k * gridDim.x with
// kPipeStages shared-memory stages.  Thread 0 keeps kPipeStages bulk copies
// (TMA, one mbarrier per stage, phase parity per reuse) in flight, so tile
// k+1..k+S-1 stream in while tile k is reduced and applied -- the one-shot
// kernel left every CTA idle on its single copy.  The per-tile work (running
// segmented sums in shared memory, two-level carry scan, in-place
// SGD/Adagrad of the keys ending in the tile, partials + arrival counters for
// spanning keys) is the same, so results are bit-identical.
constexpr int kPipeStages = 3;

template <int Q>
__global__ void __launch_bounds__(256, 2) k_embbag_bwd_pipe(
    const uint32_t* __restrict__ seg_of, const uint32_t* __restrict__ seg_start, uint32_t n, uint32_t n_tiles,
    const float4* __restrict__ grad, float* __restrict__ values, int row_stride, const int32_t* __restrict__ slots_s,
    uint8_t* __restrict__ dirty, int opt, float lr, float eps, float4* __restrict__ parts,
    unsigned int* __restrict__ arrivals, unsigned long long* __restrict__ stats) {
  constexpr int T = kStagedF4 / Q, NG = 256 / Q, RPG = T / NG, GW = 32 / Q;
  extern __shared__ __align__(128) unsigned char st_smem[];
  float4* tiles_sm = reinterpret_cast<float4*>(st_smem);                          // [S][T][Q]
  uint32_t* sgs_sm = reinterpret_cast<uint32_t*>(tiles_sm + kPipeStages * T * Q);  // [S][T]
  int32_t* tslot = reinterpret_cast<int32_t*>(sgs_sm + kPipeStages * T);          // [T]
  __shared__ __align__(8) uint64_t bar[kPipeStages];
  __shared__ float4 gcarry[NG][Q];
  __shared__ float4 wagg[8][Q];
  __shared__ int wflag[8][Q];
  __shared__ uint8_t ghead[NG];
  const uint32_t tid = threadIdx.x;
  const uint32_t G = gridDim.x;
  auto issue = [&](uint32_t tile, int st) {  // thread 0: bulk copies of one tile into stage st
    const uint32_t t0 = tile * T;
    const uint32_t rows = min((uint32_t)T, n - t0);
    const uint32_t gbytes = rows * Q * 16, seg_bytes = (rows / 4) * 16;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])),
                 "r"(gbytes + seg_bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(tiles_sm + (size_t)st * T * Q)),
                 "l"(grad + (size_t)t0 * Q), "r"(gbytes), "r"(smem_u32(&bar[st]))
                 : "memory");
    if (seg_bytes)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(sgs_sm + (size_t)st * T)),
                   "l"(seg_of + t0), "r"(seg_bytes), "r"(smem_u32(&bar[st]))
                   : "memory");
  };
  if (tid == 0) {
#pragma unroll
    for (int st = 0; st < kPipeStages; ++st)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[st])));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
    for (int st = 0; st < kPipeStages; ++st)
      if (blockIdx.x + st * G < n_tiles) issue(blockIdx.x + st * G, st);
  }
  __syncthreads();
  const int c = (int)(tid % Q), gi = (int)(tid / Q), w = (int)(tid >> 5), gw = (int)((tid & 31) / Q);
  const uint32_t r0 = gi * RPG;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  unsigned my_nz = 0;
  uint32_t k = 0;
  for (uint32_t tile_id = blockIdx.x; tile_id < n_tiles; tile_id += G, ++k) {
    const int st = (int)(k % kPipeStages);
    const uint32_t phase = (k / kPipeStages) & 1u;
    float4* tile = tiles_sm + (size_t)st * T * Q;
    uint32_t* sgs = sgs_sm + (size_t)st * T;
    const uint32_t t0 = tile_id * T;
    const uint32_t rows = min((uint32_t)T, n - t0);
    const uint32_t seg_bytes = (rows / 4) * 16;
    // while the copy is in flight: run bounds, slots of the tile's keys (rows
    // pulled into L2 for the update), the < 4 tail segment ids
    const uint32_t tile_first = seg_of[t0], tile_last = seg_of[t0 + rows - 1];
    const uint32_t fa = seg_start[tile_first], fb = seg_start[tile_first + 1];
    const uint32_t la = seg_start[tile_last], lb = seg_start[tile_last + 1];
    const uint32_t nu = tile_last - tile_first + 1;
    for (uint32_t i = tid; i < nu; i += 256) {
      const int32_t sl = slots_s[tile_first + i];
      tslot[i] = sl;
      if (sl >= 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(values + (size_t)sl * row_stride));
    }
    if (tid < rows - seg_bytes / 4) sgs[seg_bytes / 4 + tid] = seg_of[t0 + seg_bytes / 4 + tid];
    asm volatile(
        "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT%=;\n}\n" ::"r"(
            smem_u32(&bar[st])),
        "r"(phase)
        : "memory");
    __syncthreads();
    // pass 1: running segmented sums of the group's rows, in place
    float4 acc = zero;
    bool flag = false;
    if (r0 < rows) {
      uint32_t ps = sgs[r0];
      acc = tile[r0 * Q + c];
      flag = r0 == 0 || sgs[r0 - 1] != ps;
      if (c == 0) ghead[gi] = flag ? 1 : 0;
      const uint32_t re = min(r0 + RPG, rows);
      for (uint32_t r = r0 + 1; r < re; ++r) {
        const uint32_t sr = sgs[r];
        const float4 x = tile[r * Q + c];
        if (sr == ps) {
          acc = f4_add(acc, x);
        } else {
          acc = x;
          flag = true;
        }
        tile[r * Q + c] = acc;
        ps = sr;
      }
    } else if (c == 0) {
      ghead[gi] = 1;
    }
    // pass 2: segmented scan of the group totals; warp level first
    float4 inc = acc;
    bool finc = flag;
#pragma unroll
    for (int off = 1; off < GW; off <<= 1) {
      const bool fo = __shfl_up_sync(0xffffffffu, finc ? 1 : 0, off * Q) != 0;
      float4 o;
      o.x = __shfl_up_sync(0xffffffffu, inc.x, off * Q);
      o.y = __shfl_up_sync(0xffffffffu, inc.y, off * Q);
      o.z = __shfl_up_sync(0xffffffffu, inc.z, off * Q);
      o.w = __shfl_up_sync(0xffffffffu, inc.w, off * Q);
      if (gw >= off && !finc) inc = f4_add(o, inc);
      if (gw >= off) finc = finc || fo;
    }
    if (gw == GW - 1) {
      wagg[w][c] = inc;
      wflag[w][c] = finc ? 1 : 0;
    }
    float4 ex;
    ex.x = __shfl_up_sync(0xffffffffu, inc.x, Q);
    ex.y = __shfl_up_sync(0xffffffffu, inc.y, Q);
    ex.z = __shfl_up_sync(0xffffffffu, inc.z, Q);
    ex.w = __shfl_up_sync(0xffffffffu, inc.w, Q);
    const bool fex = __shfl_up_sync(0xffffffffu, finc ? 1 : 0, Q) != 0;
    __syncthreads();
    float4 cw = zero;
    for (int kk = 0; kk < w; ++kk) cw = wflag[kk][c] ? wagg[kk][c] : f4_add(cw, wagg[kk][c]);
    const float4 carry = gw == 0 ? cw : (fex ? ex : f4_add(cw, ex));
    gcarry[gi][c] = carry;
    __syncthreads();
    const bool span1 = fa < t0 || fb > t0 + rows;
    const bool span2 = tile_last != tile_first && lb > t0 + rows;
    // pass 3: (row, column) items; a key's last row in the tile holds its sum
    bool wrote = false;
    constexpr int ITEMS = T * Q / 256, B = 4;
#pragma unroll 1
    for (int k0 = 0; k0 < ITEMS; k0 += B) {
      int32_t sl[B];
      float4 val[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const uint32_t r = (uint32_t)(tid / Q) + (uint32_t)(k0 + u) * NG;
        sl[u] = -1;
        if (r >= rows) continue;
        const uint32_t sg = sgs[r];
        if (r + 1 < rows && sgs[r + 1] == sg) continue;  // not the last row of its run
        const int32_t slot = tslot[sg - tile_first];
        if (slot < 0) continue;
        const uint32_t g = r / RPG;
        float4 x = tile[r * Q + c];
        if (!ghead[g] && sg == sgs[g * RPG]) x = f4_add(gcarry[g][c], x);
        if (sg == tile_first ? span1 : (sg == tile_last && span2)) {
          parts[(size_t)(tile_id * 2 + (sg == tile_first ? 0 : 1)) * Q + c] = x;
          wrote = true;
          continue;
        }
        sl[u] = slot;
        val[u] = x;
      }
      float4 wv[B], av[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const float4* row = reinterpret_cast<const float4*>(values + (size_t)(sl[u] >= 0 ? sl[u] : 0) * row_stride);
        wv[u] = sl[u] >= 0 ? row[c] : zero;
        av[u] = (sl[u] >= 0 && opt == BP_OPT_ADAGRAD) ? row[Q + c] : zero;
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        bool nz = false;
        if (sl[u] >= 0) {
          const float4 gg = val[u];
          float4 x = wv[u], a = av[u];
          x.x = upd1(x.x, a.x, gg.x, opt, lr, eps);
          x.y = upd1(x.y, a.y, gg.y, opt, lr, eps);
          x.z = upd1(x.z, a.z, gg.z, opt, lr, eps);
          x.w = upd1(x.w, a.w, gg.w, opt, lr, eps);
          float4* row = reinterpret_cast<float4*>(values + (size_t)sl[u] * row_stride);
          row[c] = x;
          if (opt == BP_OPT_ADAGRAD) row[Q + c] = a;
          nz = gg.x != 0.f || gg.y != 0.f || gg.z != 0.f || gg.w != 0.f;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, nz);
        const unsigned gm = (Q == 32 ? 0xffffffffu : ((1u << Q) - 1u)) << ((tid & 31) / Q * Q);
        if (sl[u] >= 0 && c == 0 && (bal & gm)) {
          if (dirty) dirty[sl[u]] = 1;
          ++my_nz;
        }
      }
    }
    const int32_t slot_first = tslot[0], slot_last = tslot[nu - 1];
    if (wrote) __threadfence();  // partials visible device-wide before the arrival count
    __syncthreads();             // every thread is done with this stage and with tslot
    if (tid == 0 && tile_id + kPipeStages * G < n_tiles) {
      // the stage was read and written through the generic proxy: order that
      // before the async-proxy (TMA) refill
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile_id + kPipeStages * G, st);
    }
    if ((span1 || span2) && w == 0) {
      // warp 0 counts the arrivals and, when it completed a spanning key,
      // combines its partials in tile order; the other warps move on
      unsigned lst = 0;
      if (tid == 0) {
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          if (!(kk == 0 ? span1 : span2)) continue;
          if ((kk == 0 ? slot_first : slot_last) < 0) continue;
          const uint32_t a = kk == 0 ? fa : la, b = kk == 0 ? fb : lb;
          const uint32_t ft = a / T, nt = (b - 1) / T - ft + 1;
          if (atomicAdd(arrivals + ft, 1u) == nt - 1) {
            lst |= 1u << kk;
            arrivals[ft] = 0;  // every arrival is in: the counter is free again (persistent scratch)
          }
        }
      }
      lst = __shfl_sync(0xffffffffu, lst, 0);
      if (lst) {
        __threadfence();
        unsigned n_comb = 0;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          if (!((lst >> kk) & 1u)) continue;
          const uint32_t a = kk == 0 ? fa : la, b = kk == 0 ? fb : lb;
          const uint32_t ft = a / T, nt = (b - 1) / T - ft + 1;
          const int32_t slot = kk == 0 ? slot_first : slot_last;
          const bool nz = span_combine<Q>(parts, ft, nt, a != ft * T, (int)(tid / Q), c,
                                          values + (size_t)slot * row_stride, opt, lr, eps);
          if (__ballot_sync(0xffffffffu, nz) != 0 && tid == 0) {
            if (dirty) dirty[slot] = 1;
            ++n_comb;
          }
        }
        if (tid == 0) my_nz += n_comb;
      }
    }
  }
  if (stats) cta_add(&stats[1], my_nz);
}

// Two-kernel backward (variant 4; measured slower inside the step than the
// fused one-shot kernel, kept for comparison): the reduction and the update
// are split so neither waits on the other's latency.
//
// k_bwd_reduce: a streaming segmented reduction of the key-sorted gradient
// rows.  Persistent CTAs (2 per SM) keep kPipeStages bulk copies (TMA +
// mbarrier) of 16 KB tiles in flight; per tile the running segmented sums,
// the two-level carry scan (fixed order) and, for every key ending in the
// tile, ONE float4 store of its sum into gsum[s] (keys are consecutive, so
// the stores are too) -- no cache-row access, no dependent global loads.  A
// key that continues from the previous tile or into the next one leaves its
// tile partial in parts[tile][0 | 1] (first | last key of the tile).
//
// k_bwd_apply: one Q-lane group per unique key (fully parallel, latency
// hidden by occupancy): g = gsum[s], or for a key spanning tiles its
// partials summed in tile order, then SGD/Adagrad in place on its cached row,
// dirty mark and the non-zero count.
constexpr int kRedF4 = 1024;  // float4 per k_bwd_reduce tile (16 KB): 4 CTAs x 3 stages per SM

template <int Q>
__global__ void __launch_bounds__(256, 4) k_bwd_reduce(const uint32_t* __restrict__ seg_of, uint32_t n,
                                                       uint32_t n_tiles, const float4* __restrict__ grad,
                                                       float4* __restrict__ gsum, float4* __restrict__ parts) {
  constexpr int T = kRedF4 / Q, NG = 256 / Q, RPG = T / NG, GW = 32 / Q;
  extern __shared__ __align__(128) unsigned char st_smem[];
  float4* tiles_sm = reinterpret_cast<float4*>(st_smem);                          // [S][T][Q]
  uint32_t* sgs_sm = reinterpret_cast<uint32_t*>(tiles_sm + kPipeStages * T * Q);  // [S][T]
  __shared__ __align__(8) uint64_t bar[kPipeStages];
  __shared__ float4 gcarry[NG][Q];
  __shared__ float4 wagg[8][Q];
  __shared__ int wflag[8][Q];
  __shared__ uint8_t ghead[NG];
  const uint32_t tid = threadIdx.x;
  const uint32_t G = gridDim.x;
  auto issue = [&](uint32_t tile, int st) {
    const uint32_t t0 = tile * T;
    const uint32_t rows = min((uint32_t)T, n - t0);
    const uint32_t gbytes = rows * Q * 16, seg_bytes = (rows / 4) * 16;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])),
                 "r"(gbytes + seg_bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(tiles_sm + (size_t)st * T * Q)),
                 "l"(grad + (size_t)t0 * Q), "r"(gbytes), "r"(smem_u32(&bar[st]))
                 : "memory");
    if (seg_bytes)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(sgs_sm + (size_t)st * T)),
                   "l"(seg_of + t0), "r"(seg_bytes), "r"(smem_u32(&bar[st]))
                   : "memory");
  };
  if (tid == 0) {
#pragma unroll
    for (int st = 0; st < kPipeStages; ++st)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[st])));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
    for (int st = 0; st < kPipeStages; ++st)
      if (blockIdx.x + st * G < n_tiles) issue(blockIdx.x + st * G, st);
  }
  __syncthreads();
  const int c = (int)(tid % Q), gi = (int)(tid / Q), w = (int)(tid >> 5), gw = (int)((tid & 31) / Q);
  const uint32_t r0 = gi * RPG;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t k = 0;
  for (uint32_t tile_id = blockIdx.x; tile_id < n_tiles; tile_id += G, ++k) {
    const int st = (int)(k % kPipeStages);
    const uint32_t phase = (k / kPipeStages) & 1u;
    float4* tile = tiles_sm + (size_t)st * T * Q;
    uint32_t* sgs = sgs_sm + (size_t)st * T;
    const uint32_t t0 = tile_id * T;
    const uint32_t rows = min((uint32_t)T, n - t0);
    const uint32_t seg_bytes = (rows / 4) * 16;
    // the neighbours' segment ids tell whether the tile's first / last key
    // continues across its edges (independent loads, in flight with the copy)
    const uint32_t prev_id = t0 > 0 ? seg_of[t0 - 1] : 0xFFFFFFFFu;
    const uint32_t next_id = t0 + rows < n ? seg_of[t0 + rows] : 0xFFFFFFFFu;
    if (tid < rows - seg_bytes / 4) sgs[seg_bytes / 4 + tid] = seg_of[t0 + seg_bytes / 4 + tid];
    asm volatile(
        "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT%=;\n}\n" ::"r"(
            smem_u32(&bar[st])),
        "r"(phase)
        : "memory");
    __syncthreads();
    float4 acc = zero;
    bool flag = false;
    if (r0 < rows) {
      uint32_t ps = sgs[r0];
      acc = tile[r0 * Q + c];
      flag = r0 == 0 || sgs[r0 - 1] != ps;
      if (c == 0) ghead[gi] = flag ? 1 : 0;
      const uint32_t re = min(r0 + RPG, rows);
      for (uint32_t r = r0 + 1; r < re; ++r) {
        const uint32_t sr = sgs[r];
        const float4 x = tile[r * Q + c];
        if (sr == ps) {
          acc = f4_add(acc, x);
        } else {
          acc = x;
          flag = true;
        }
        tile[r * Q + c] = acc;
        ps = sr;
      }
    } else if (c == 0) {
      ghead[gi] = 1;
    }
    float4 inc = acc;
    bool finc = flag;
#pragma unroll
    for (int off = 1; off < GW; off <<= 1) {
      const bool fo = __shfl_up_sync(0xffffffffu, finc ? 1 : 0, off * Q) != 0;
      float4 o;
      o.x = __shfl_up_sync(0xffffffffu, inc.x, off * Q);
      o.y = __shfl_up_sync(0xffffffffu, inc.y, off * Q);
      o.z = __shfl_up_sync(0xffffffffu, inc.z, off * Q);
      o.w = __shfl_up_sync(0xffffffffu, inc.w, off * Q);
      if (gw >= off && !finc) inc = f4_add(o, inc);
      if (gw >= off) finc = finc || fo;
    }
    if (gw == GW - 1) {
      wagg[w][c] = inc;
      wflag[w][c] = finc ? 1 : 0;
    }
    float4 ex;
    ex.x = __shfl_up_sync(0xffffffffu, inc.x, Q);
    ex.y = __shfl_up_sync(0xffffffffu, inc.y, Q);
    ex.z = __shfl_up_sync(0xffffffffu, inc.z, Q);
    ex.w = __shfl_up_sync(0xffffffffu, inc.w, Q);
    const bool fex = __shfl_up_sync(0xffffffffu, finc ? 1 : 0, Q) != 0;
    __syncthreads();
    float4 cw = zero;
    for (int kk = 0; kk < w; ++kk) cw = wflag[kk][c] ? wagg[kk][c] : f4_add(cw, wagg[kk][c]);
    const float4 carry = gw == 0 ? cw : (fex ? ex : f4_add(cw, ex));
    gcarry[gi][c] = carry;
    __syncthreads();
    const uint32_t first = sgs[0], last = sgs[rows - 1];
    const bool cont_in = prev_id == first, cont_out = next_id == last;
    constexpr int ITEMS = T * Q / 256;
#pragma unroll 4
    for (int kk = 0; kk < ITEMS; ++kk) {
      const uint32_t r = (uint32_t)(tid / Q) + (uint32_t)kk * NG;
      if (r >= rows) continue;
      const uint32_t sg = sgs[r];
      if (r + 1 < rows && sgs[r + 1] == sg) continue;  // not the last row of its run
      const uint32_t g = r / RPG;
      float4 x = tile[r * Q + c];
      if (!ghead[g] && sg == sgs[g * RPG]) x = f4_add(gcarry[g][c], x);
      if (sg == first && cont_in) parts[(size_t)(tile_id * 2) * Q + c] = x;
      else if (sg == last && cont_out) parts[(size_t)(tile_id * 2 + 1) * Q + c] = x;
      else gsum[(size_t)sg * Q + c] = x;
    }
    __syncthreads();  // every thread is done with this stage
    if (tid == 0 && tile_id + kPipeStages * G < n_tiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile_id + kPipeStages * G, st);
    }
  }
}

// Register-resident reduce of the key-sorted gradient rows (variant 8, the
// first half of the split backward; k_bwd_apply is the second).  A CTA owns
// kRegTileF4 / Q sorted rows, each of its 8 warps 16 rows per lane group
// (Q lanes, one float4 column each; the 16 loads of a lane are issued
// together).  A group sums its rows in order, branch-free, and stores every
// key that starts and ends inside them straight to gsum.  Two left-to-right
// chains in fixed order complete the keys crossing group boundaries (through
// shuffles) and warp boundaries (through shared memory); a key crossing the
// CTA tile boundary leaves its partial in the tile's parts slot (1 at the
// key's first tile, 0 at every later one) for k_bwd_apply.  No atomics,
// one barrier; ncu on the staged and split kernels: 6.9M warp instructions
// per CK batch, most of them in shared-memory passes and per-thread carry
// loops.
constexpr int kRegTileF4 = 4096;  // float4 per k_bwd_reduce_reg CTA tile (64 KB of gradient rows)

// one segment of a chain: its first key (+ that key's sum, complete when the
// segment holds more than one key) and its last key (+ sum); nk = keys seen
struct ChainSeg {
  uint32_t fk, lk;
  int nk;
  float4 fv, lv;
};

// Left-to-right merge of the open key (ok, ov) with the next segment:
// returns through emit the keys it completes.  first: the open key is the
// chain's first key.
template <typename Emit>
__device__ __forceinline__ void chain_step(uint32_t& ok, float4& ov, bool& first, const ChainSeg& sg, Emit&& emit) {
  if (sg.nk == 0) return;
  if (sg.fk == ok) {
    if (sg.nk == 1) {
      ov = f4_add(ov, sg.lv);
      return;
    }
    emit(ok, f4_add(ov, sg.fv), first);
  } else {
    emit(ok, ov, first);
    if (sg.nk >= 2) emit(sg.fk, sg.fv, false);
  }
  first = false;
  ok = sg.lk;
  ov = sg.lv;
}

// TMA = true (variant 10): the CTA's tile of gradient rows and segment ids
// arrives by one bulk async copy (TMA engine, mbarrier completion) into
// shared memory instead of per-lane loads: the bytes in flight no longer
// cost registers, so ~6 CTAs per SM stream their tiles at once.
template <int Q, int R = 16, int NW = 8, bool TMA = false>
__global__ void __launch_bounds__(NW * 32, TMA ? 6 : (R == 16 ? 2 : 3) * 8 / NW) k_bwd_reduce_reg(
    const uint32_t* __restrict__ seg_of, uint32_t n, const float4* __restrict__ grad, float4* __restrict__ gsum,
    float4* __restrict__ parts, uint32_t* __restrict__ span_list, unsigned* __restrict__ span_count) {
  constexpr int G = 32 / Q, WT = G * R, T = NW * WT;
  static_assert(T * Q == 32 * NW * R, "tile of k_bwd_apply");
  const unsigned lane = threadIdx.x & 31u;
  const int w = (int)(threadIdx.x >> 5), g = (int)(lane / Q), c = (int)(lane % Q);
  const long long t0 = (long long)blockIdx.x * T;
  const long long w0 = t0 + (long long)w * WT;
  const long long r0 = w0 + (long long)g * R;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const long long t_end = t0 + T < (long long)n ? t0 + T : (long long)n;
  // neighbours of the CTA tile: does its first key come from the previous
  // tile, does its last key go on into the next one
  const uint32_t before = t0 > 0 ? seg_of[t0 - 1] : 0xFFFFFFFFu;
  const uint32_t after = t_end < (long long)n ? seg_of[t_end] : 0xFFFFFFFEu;
  // the lane's 16 rows, all loads in flight together
  uint32_t sg[R];
  float4 x[R];
  if constexpr (TMA) {
    extern __shared__ __align__(128) unsigned char rt_smem[];
    float4* tile = reinterpret_cast<float4*>(rt_smem);            // [T][Q]
    uint32_t* sgs = reinterpret_cast<uint32_t*>(tile + T * Q);     // [T]
    __shared__ __align__(8) uint64_t bar;
    const uint32_t rows = (uint32_t)(t_end - t0);
    const uint32_t seg_bytes = (rows / 4) * 16;
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                   "r"(rows * Q * 16 + seg_bytes)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(tile)),
                   "l"(grad + t0 * Q), "r"(rows * Q * 16), "r"(smem_u32(&bar))
                   : "memory");
      if (seg_bytes)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sgs)),
                     "l"(seg_of + t0), "r"(seg_bytes), "r"(smem_u32(&bar))
                     : "memory");
    }
    if (threadIdx.x < rows - seg_bytes / 4) sgs[seg_bytes / 4 + threadIdx.x] = seg_of[t0 + seg_bytes / 4 + threadIdx.x];
    __syncthreads();  // the barrier is initialised, the tail ids are in
    asm volatile(
        "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT%=;\n}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
    const int lr0 = (int)(r0 - t0);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const bool ok = (uint32_t)(lr0 + j) < rows;
      sg[j] = ok ? sgs[lr0 + j] : 0xFFFFFFFFu;
      x[j] = ok ? tile[(lr0 + j) * Q + c] : zero;
    }
  } else if (r0 + R <= (long long)n) {
#pragma unroll
    for (int j = 0; j < R; j += 4) {
      const uint4 q4 = *reinterpret_cast<const uint4*>(seg_of + r0 + j);
      sg[j] = q4.x;
      sg[j + 1] = q4.y;
      sg[j + 2] = q4.z;
      sg[j + 3] = q4.w;
    }
#pragma unroll
    for (int j = 0; j < R; ++j) x[j] = __ldcs(grad + (r0 + j) * Q + c);
  } else {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const bool ok = r0 + j < (long long)n;
      sg[j] = ok ? seg_of[r0 + j] : 0xFFFFFFFFu;
      x[j] = ok ? __ldcs(grad + (r0 + j) * Q + c) : zero;
    }
  }
  // in-order segmented sum, branch-free: a key that closes as the group's
  // second or later key started and ended here -> gsum
  ChainSeg me;
  me.fk = 0xFFFFFFFFu;
  me.nk = 0;
  me.fv = zero;
  uint32_t cur = 0xFFFFFFFFu;
  float4 acc = zero;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const bool valid = sg[j] != 0xFFFFFFFFu;
    const bool same = sg[j] == cur;
    const bool opens = valid && !same;
    if (opens && me.nk >= 2) gsum[(size_t)cur * Q + c] = acc;
    if (opens && me.nk == 1) me.fv = acc;
    if (opens && me.nk == 0) me.fk = sg[j];
    me.nk += opens ? 1 : 0;
    const float4 sum = f4_add(acc, x[j]);
    acc = !valid ? acc : (same ? sum : x[j]);
    cur = valid ? sg[j] : cur;
  }
  me.lk = cur;
  me.lv = acc;
  // chain 1: the warp's groups, left to right (every lane runs it for its
  // column; group 0's lanes store).  The warp's first and last keys stay
  // open for chain 2.
  ChainSeg ws;
  {
    ChainSeg s0;
    s0.nk = __shfl_sync(0xffffffffu, me.nk, c);
    s0.fk = __shfl_sync(0xffffffffu, me.fk, c);
    s0.lk = __shfl_sync(0xffffffffu, me.lk, c);
    s0.fv.x = __shfl_sync(0xffffffffu, me.fv.x, c);
    s0.fv.y = __shfl_sync(0xffffffffu, me.fv.y, c);
    s0.fv.z = __shfl_sync(0xffffffffu, me.fv.z, c);
    s0.fv.w = __shfl_sync(0xffffffffu, me.fv.w, c);
    s0.lv.x = __shfl_sync(0xffffffffu, me.lv.x, c);
    s0.lv.y = __shfl_sync(0xffffffffu, me.lv.y, c);
    s0.lv.z = __shfl_sync(0xffffffffu, me.lv.z, c);
    s0.lv.w = __shfl_sync(0xffffffffu, me.lv.w, c);
    ws = s0;  // fk / fv / nk describe the warp's first key until it closes
    uint32_t ok_ = s0.lk;
    float4 ov = s0.lv;
    bool first = s0.nk <= 1;
    int keys = s0.nk;
    const bool leader = g == 0;
#pragma unroll
    for (int k = 1; k < G; ++k) {
      const int src = k * Q + c;
      ChainSeg sk;
      sk.nk = __shfl_sync(0xffffffffu, me.nk, src);
      sk.fk = __shfl_sync(0xffffffffu, me.fk, src);
      sk.lk = __shfl_sync(0xffffffffu, me.lk, src);
      sk.fv.x = __shfl_sync(0xffffffffu, me.fv.x, src);
      sk.fv.y = __shfl_sync(0xffffffffu, me.fv.y, src);
      sk.fv.z = __shfl_sync(0xffffffffu, me.fv.z, src);
      sk.fv.w = __shfl_sync(0xffffffffu, me.fv.w, src);
      sk.lv.x = __shfl_sync(0xffffffffu, me.lv.x, src);
      sk.lv.y = __shfl_sync(0xffffffffu, me.lv.y, src);
      sk.lv.z = __shfl_sync(0xffffffffu, me.lv.z, src);
      sk.lv.w = __shfl_sync(0xffffffffu, me.lv.w, src);
      keys += sk.nk > 0 ? sk.nk - (sk.fk == ok_ ? 1 : 0) : 0;
      chain_step(ok_, ov, first, sk, [&](uint32_t key, float4 val, bool is_first) {
        if (is_first) {
          ws.fv = val;  // the warp's first key closes: chain 2 decides
        } else if (leader) {
          gsum[(size_t)key * Q + c] = val;
        }
      });
    }
    ws.nk = keys;
    ws.lk = ok_;
    ws.lv = ov;
    if (keys <= 1) ws.fv = ov;
  }
  // chain 2: the CTA's warps, left to right, in shared memory
  __shared__ ChainSeg wseg[NW][Q];
  if (g == 0) wseg[w][c] = ws;
  __syncthreads();
  if (w != 0 || g != 0) return;
  const ChainSeg s0 = wseg[0][c];
  if (s0.nk == 0) return;
  const bool cont_in = before == s0.fk;
  const auto emit = [&](uint32_t key, float4 val, bool is_first) {
    if (is_first && cont_in) parts[(size_t)(blockIdx.x * 2) * Q + c] = val;
    else gsum[(size_t)key * Q + c] = val;
  };
  uint32_t ok_ = s0.lk;
  float4 ov = s0.lv;
  bool first = s0.nk <= 1;
  if (s0.nk >= 2) emit(s0.fk, s0.fv, true);
#pragma unroll 1
  for (int k = 1; k < NW; ++k) chain_step(ok_, ov, first, wseg[k][c], emit);
  // the tile's last key
  if (after == ok_) {
    parts[(size_t)(blockIdx.x * 2 + ((first && cont_in) ? 0 : 1)) * Q + c] = ov;
    // the key's first tile lists it: k_bwd_apply gives it a whole warp
    if (span_list && c == 0 && !(first && cont_in)) span_list[atomicAdd(span_count, 1u)] = ok_;
  }
  else emit(ok_, ov, first);
}

template <int Q, int TF4 = kRedF4>
__global__ void __launch_bounds__(256) k_bwd_apply(const uint32_t* __restrict__ seg_start, const long long* d_U,
                                                   const float4* __restrict__ gsum, const float4* __restrict__ parts,
                                                   float* __restrict__ values, int row_stride,
                                                   const int32_t* __restrict__ slots_s, uint8_t* __restrict__ dirty,
                                                   int opt, float lr, float eps,
                                                   unsigned long long* __restrict__ stats,
                                                   const uint32_t* __restrict__ span_list = nullptr,
                                                   const unsigned* __restrict__ span_count = nullptr) {
  constexpr int T = TF4 / Q;
  const long long U = *d_U;
  unsigned long long my_nz = 0;
  if (span_count) {
    // keys spanning tiles (listed by k_bwd_reduce_reg): a warp each, one
    // lane per tile partial (all loaded at once), a fixed xor tree over the
    // lanes, then the update by the first Q lanes
    const unsigned nspan = *span_count;
    const unsigned lane = threadIdx.x & 31u;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long wi = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); wi < nspan; wi += warps) {
      const uint32_t key = span_list[wi];
      const uint32_t ft = seg_start[key] / T, lt = (seg_start[key + 1] - 1) / T;
      float4 part[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) part[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (uint32_t t = ft + lane; t <= lt; t += 32) {  // lanes: ascending tiles; rounds: in order
        const float4* pt = parts + (size_t)(t * 2 + (t == ft ? 1 : 0)) * Q;
#pragma unroll
        for (int q = 0; q < Q; ++q) part[q] = f4_add(part[q], __ldcg(pt + q));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          float4 y;
          y.x = __shfl_xor_sync(0xffffffffu, part[q].x, o);
          y.y = __shfl_xor_sync(0xffffffffu, part[q].y, o);
          y.z = __shfl_xor_sync(0xffffffffu, part[q].z, o);
          y.w = __shfl_xor_sync(0xffffffffu, part[q].w, o);
          part[q] = (lane & o) ? f4_add(y, part[q]) : f4_add(part[q], y);  // same order on both lanes
        }
      const int32_t slot = slots_s[key];
      bool nz = false;
      if (slot >= 0 && lane < (unsigned)Q) {
        float4 gv = part[0];
#pragma unroll
        for (int q = 1; q < Q; ++q)
          if (lane == (unsigned)q) gv = part[q];
        float* row = values + (size_t)slot * row_stride;
        float4 x = reinterpret_cast<const float4*>(row)[lane];
        float4 a = opt == BP_OPT_ADAGRAD ? reinterpret_cast<const float4*>(row)[Q + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
        x.x = upd1(x.x, a.x, gv.x, opt, lr, eps);
        x.y = upd1(x.y, a.y, gv.y, opt, lr, eps);
        x.z = upd1(x.z, a.z, gv.z, opt, lr, eps);
        x.w = upd1(x.w, a.w, gv.w, opt, lr, eps);
        reinterpret_cast<float4*>(row)[lane] = x;
        if (opt == BP_OPT_ADAGRAD) reinterpret_cast<float4*>(row)[Q + lane] = a;
        nz = gv.x != 0.f || gv.y != 0.f || gv.z != 0.f || gv.w != 0.f;
      }
      if (__ballot_sync(0xffffffffu, nz) && lane == 0) {
        if (dirty) dirty[slot] = 1;
        ++my_nz;
      }
    }
  }
  // grid-stride over (key, column) items: the grid is sized for the
  // machine, not for the n_occ bound on U
  for (long long base = (long long)blockIdx.x * blockDim.x; base < U * Q; base += (long long)gridDim.x * blockDim.x) {
  const long long i = base + threadIdx.x;
  const long long s = i / Q;
  const int c = (int)(i % Q);
  bool nz = false;
  if (s < U) {
    // independent loads first: slot, CSR bounds, the in-tile sum
    const int32_t slot = slots_s[s];
    const uint32_t a = seg_start[s], b = seg_start[s + 1];
    float4 g = __ldcg(gsum + (size_t)s * Q + c);
    const uint32_t ft = a / T, lt = (b - 1) / T;
    // a listed spanning key is done by its warp above
    if (slot >= 0 && !(ft != lt && span_count)) {
      float* row = values + (size_t)slot * row_stride;
      float4 x = reinterpret_cast<const float4*>(row)[c];
      float4 acc = opt == BP_OPT_ADAGRAD ? reinterpret_cast<const float4*>(row)[Q + c] : make_float4(0.f, 0.f, 0.f, 0.f);
      if (ft != lt) {  // tile partials in tile order: the key continues out of
                       // its first tile (slot 1 there) and into every later one (slot 0)
        g = __ldcg(parts + (size_t)(ft * 2 + 1) * Q + c);
        // 8 partial loads in flight per round (a Zipf-hot key spans dozens of
        // tiles), summed in tile order
        for (uint32_t t0 = ft + 1; t0 <= lt; t0 += 8) {
          float4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            v[u] = t0 + u <= lt ? __ldcg(parts + (size_t)((t0 + u) * 2) * Q + c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (t0 + u <= lt) g = f4_add(g, v[u]);
        }
      }
      x.x = upd1(x.x, acc.x, g.x, opt, lr, eps);
      x.y = upd1(x.y, acc.y, g.y, opt, lr, eps);
      x.z = upd1(x.z, acc.z, g.z, opt, lr, eps);
      x.w = upd1(x.w, acc.w, g.w, opt, lr, eps);
      reinterpret_cast<float4*>(row)[c] = x;
      if (opt == BP_OPT_ADAGRAD) reinterpret_cast<float4*>(row)[Q + c] = acc;
      nz = g.x != 0.f || g.y != 0.f || g.z != 0.f || g.w != 0.f;
    }
  }
  // a key is dirty if any of its Q lanes saw a non-zero component
  const unsigned lane = threadIdx.x & 31u;
  const unsigned bal = __ballot_sync(0xffffffffu, nz);
  const unsigned gm = (Q == 32 ? 0xffffffffu : ((1u << Q) - 1u)) << (lane / Q * Q);
  const bool key_nz = (bal & gm) != 0 && c == 0 && s < U;
  if (key_nz && dirty) dirty[slots_s[s]] = 1;
  my_nz += key_nz ? 1ull : 0ull;
  }
  if (stats) cta_add(&stats[1], my_nz);
}

// Keys spanning several tiles, listed by the tile kernels at the key's first
// tile: up to kSpanWarpTiles tiles (the many keys that merely cross a tile
// boundary) one warp per key, longer ones (the Zipf-hot rows) one CTA per
// key.  Lanes / threads split (tile, float4): each sums its tiles in
// ascending order (four independent accumulators, combined in a fixed
// order), then a fixed xor-shuffle or shared-memory tree over the tile lanes
// -- every order is data-independent -- and the first tile lane applies the
// update.

__device__ __forceinline__ void span_sum(const float4* __restrict__ parts, long long t, long long nt, long long a,
                                         int T, int q, int c, int tl, int per, float4& acc, bool& any) {
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 acc4[4] = {zero, zero, zero, zero};
  bool any4[4] = {false, false, false, false};
  for (long long k0 = tl; tl < per && k0 < nt; k0 += 4 * per) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long k = k0 + (long long)u * per;
      if (k < nt) {
        const int half = (k == 0 && a != t * T) ? 1 : 0;
        const float4 x = __ldcg(parts + ((t + k) * 2 + half) * q + c);
        acc4[u] = any4[u] ? f4_add(acc4[u], x) : x;
        any4[u] = true;
      }
    }
  }
  acc = acc4[0];
#pragma unroll
  for (int u = 1; u < 4; ++u)
    if (any4[u]) acc = f4_add(acc, acc4[u]);  // any4[u] implies any4[0]
  any = any4[0];
}

__global__ void __launch_bounds__(256) k_embbag_bwd_span(
    const uint32_t* __restrict__ seg_of, const uint32_t* __restrict__ seg_start, long long n, int q, int T,
    const uint32_t* __restrict__ small_list, const unsigned int* __restrict__ small_count,
    const uint32_t* __restrict__ big_list, const unsigned int* __restrict__ big_count,
    const float4* __restrict__ parts, float* __restrict__ values, int row_stride,
    const int32_t* __restrict__ slots_s, uint8_t* __restrict__ dirty, int opt, float lr, float eps,
    unsigned long long* __restrict__ stats) {
  __shared__ float4 red[256];
  __shared__ int any_nz;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  if (blockIdx.x < kSpanSmallBlocks) {  // warp per key
    const unsigned lane = threadIdx.x & 31u;
    int per = 1;
    while (per * 2 * q <= 32) per *= 2;
    const int c = (int)lane % q, tl = (int)lane / q;
    const long long warps = (long long)kSpanSmallBlocks * (blockDim.x >> 5);
    const long long n_span = *small_count;
    for (long long li = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); li < n_span; li += warps) {
      const long long t = small_list[li];
      const long long last = min((t + 1) * (long long)T, n) - 1;
      const uint32_t s = seg_of[last];
      const long long a = seg_start[s], b = seg_start[s + 1];
      const int32_t slot = slots_s[s];
      if (slot < 0) continue;  // warp-uniform
      float4 acc;
      bool any;
      span_sum(parts, t, (b - 1) / T - t + 1, a, T, q, c, tl, per, acc, any);
      if (!any) acc = zero;
      for (int off = per / 2; off > 0; off >>= 1) {
        float4 o;
        o.x = __shfl_down_sync(0xffffffffu, acc.x, off * q);
        o.y = __shfl_down_sync(0xffffffffu, acc.y, off * q);
        o.z = __shfl_down_sync(0xffffffffu, acc.z, off * q);
        o.w = __shfl_down_sync(0xffffffffu, acc.w, off * q);
        if (tl < off) acc = f4_add(acc, o);
      }
      bool nz = false;
      if (tl == 0) nz = apply_row4(values + (long long)slot * row_stride, 4 * q, c, acc, opt, lr, eps);
      if (__ballot_sync(0xffffffffu, nz) != 0 && lane == 0) {
        if (dirty) dirty[slot] = 1;
        if (stats) atomicAdd(&stats[1], 1ull);
      }
    }
    return;
  }
  int per = 1;  // CTA per key: the largest power of two with per * q <= 256 (others idle)
  while (per * 2 * q <= 256) per *= 2;
  const int c = threadIdx.x % q, tl = threadIdx.x / q;
  const long long n_span = *big_count;
  for (long long li = blockIdx.x - kSpanSmallBlocks; li < n_span; li += gridDim.x - kSpanSmallBlocks) {
    const long long t = big_list[li];
    const long long last = min((t + 1) * (long long)T, n) - 1;
    const uint32_t s = seg_of[last];
    const long long a = seg_start[s], b = seg_start[s + 1];
    const int32_t slot = slots_s[s];
    if (slot < 0) continue;  // block-uniform
    float4 acc;
    bool any;
    span_sum(parts, t, (b - 1) / T - t + 1, a, T, q, c, tl, per, acc, any);
    red[threadIdx.x] = any ? acc : zero;
    if (threadIdx.x == 0) any_nz = 0;
    __syncthreads();
    for (int off = per / 2; off > 0; off >>= 1) {
      if (tl < off) red[threadIdx.x] = f4_add(red[threadIdx.x], red[threadIdx.x + off * q]);
      __syncthreads();
    }
    if (tl == 0 && apply_row4(values + (long long)slot * row_stride, 4 * q, c, red[c], opt, lr, eps)) any_nz = 1;
    __syncthreads();
    if (threadIdx.x == 0 && any_nz) {
      if (dirty) dirty[slot] = 1;
      if (stats) atomicAdd(&stats[1], 1ull);
    }
    __syncthreads();
  }
}

// occ_s[p] = key-sorted unique index of occurrence p (segment of sorted slot j
// found by binary search over the CSR offsets).
__global__ void k_occ_sorted_index(const uint32_t* __restrict__ seg_start, const uint32_t* __restrict__ occ_pos,
                                   const long long* __restrict__ d_U, long long n, uint32_t* __restrict__ occ_s) {
  const long long U = *d_U;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = U;  // largest s with seg_start[s] <= j
    while (hi - lo > 1) {
      const long long mid = (lo + hi) >> 1;
      if (seg_start[mid] <= (uint32_t)j) lo = mid;
      else hi = mid;
    }
    occ_s[occ_pos[j]] = (uint32_t)lo;
  }
}

static inline void shape_of(int dim, int* G, int* dpl) {
  int g = 1;
  while (g < dim && g < 32) g <<= 1;
  *G = g;
  *dpl = (dim + g - 1) / g;
}

}  // namespace bp

#define BP_BAG_DISPATCH(G, DPL, CALL)                                  \
  switch (G * 16 + DPL) {                                               \
    case 1 * 16 + 1: { constexpr int g_ = 1, d_ = 1; CALL; break; }   \
    case 2 * 16 + 1: { constexpr int g_ = 2, d_ = 1; CALL; break; }   \
    case 4 * 16 + 1: { constexpr int g_ = 4, d_ = 1; CALL; break; }   \
    case 8 * 16 + 1: { constexpr int g_ = 8, d_ = 1; CALL; break; }   \
    case 16 * 16 + 1: { constexpr int g_ = 16, d_ = 1; CALL; break; } \
    case 32 * 16 + 1: { constexpr int g_ = 32, d_ = 1; CALL; break; } \
    case 32 * 16 + 2: { constexpr int g_ = 32, d_ = 2; CALL; break; } \
    case 32 * 16 + 3: { constexpr int g_ = 32, d_ = 3; CALL; break; } \
    case 32 * 16 + 4: { constexpr int g_ = 32, d_ = 4; CALL; break; } \
    default: return BP_ERR_INVALID;                                     \
  }

extern "C" int bp_embbag_forward(bp_prep* P, const float* d_values, int32_t row_stride, const int32_t* d_slots_s,
                                 int32_t dim, const int64_t* d_bag_offsets, int64_t n_bags, int32_t mode,
                                 const uint32_t* d_occ_s, float* d_out, bp_stream_t stream) {
  using namespace bp;
  if (dim < 1 || dim > 128) return BP_ERR_INVALID;
  if (P->n_occ == 0) return BP_OK;
  int G, dpl;
  shape_of(dim, &G, &dpl);
  cudaStream_t s = (cudaStream_t)stream;
  if (!d_occ_s) d_occ_s = P->d_occ_s;
  if (!d_occ_s) return BP_ERR_INVALID;
  if (!d_bag_offsets && (dim & 3) == 0 && (row_stride & 3) == 0 && g_fwd_variant == 1 && P->d_seg_of &&
      d_occ_s == P->d_occ_s) {
    const int q = dim / 4;
    k_embbag_fwd_sorted_v4<<<grid_for(P->n_occ * q, 256 * 4, kNumSMs * 8), 256, 0, s>>>(
        P->d_seg_of, P->d_occ_pos, d_slots_s, reinterpret_cast<const float4*>(d_values), q, row_stride / 4,
        P->n_occ, reinterpret_cast<float4*>(d_out));
  } else if (!d_bag_offsets && (dim & 3) == 0 && (row_stride & 3) == 0) {
    const int q = dim / 4;
    const int fg = grid_for(P->n_occ * q, 256 * 4, kNumSMs * 8);
    const float4* vals4 = reinterpret_cast<const float4*>(d_values);
    float4* out4 = reinterpret_cast<float4*>(d_out);
    switch (q) {
      case 1: k_embbag_fwd_rows_v4<1><<<fg, 256, 0, s>>>(d_occ_s, d_slots_s, vals4, q, row_stride / 4, P->n_occ, out4); break;
      case 2: k_embbag_fwd_rows_v4<2><<<fg, 256, 0, s>>>(d_occ_s, d_slots_s, vals4, q, row_stride / 4, P->n_occ, out4); break;
      case 4: k_embbag_fwd_rows_v4<4><<<fg, 256, 0, s>>>(d_occ_s, d_slots_s, vals4, q, row_stride / 4, P->n_occ, out4); break;
      case 8: k_embbag_fwd_rows_v4<8><<<fg, 256, 0, s>>>(d_occ_s, d_slots_s, vals4, q, row_stride / 4, P->n_occ, out4); break;
      case 16: k_embbag_fwd_rows_v4<16><<<fg, 256, 0, s>>>(d_occ_s, d_slots_s, vals4, q, row_stride / 4, P->n_occ, out4); break;
      default: k_embbag_fwd_rows_v4<0><<<fg, 256, 0, s>>>(d_occ_s, d_slots_s, vals4, q, row_stride / 4, P->n_occ, out4); break;
    }
  } else {
    if (!d_bag_offsets) return BP_ERR_INVALID;
    const int blocks = grid_for(n_bags * G, 256, kNumSMs * 8);
    BP_BAG_DISPATCH(G, dpl,
                    (k_embbag_fwd_gather<g_, d_><<<blocks, 256, 0, s>>>(d_occ_s, d_slots_s, d_values, d_bag_offsets,
                                                                        n_bags, dim, row_stride, mode, d_out)));
  }
  BP_LAUNCH_CHECK();
  return BP_OK;
}

static int embbag_backward_impl(bp_prep* P, const float* d_grad, const int64_t* d_occ_bag, const float* d_bag_scale,
                                float* d_values, int32_t row_stride, const int32_t* d_slots_s, uint8_t* d_dirty,
                                int32_t dim, int32_t opt, float lr, float eps, int64_t* d_stats, bp_stream_t stream,
                                const bp::PeerSrc* peer_src) {
  using namespace bp;
  if (dim < 1 || dim > 128) return BP_ERR_INVALID;
  if (opt == BP_OPT_ADAGRAD && row_stride < 2 * dim) return BP_ERR_INVALID;
  if (P->n_occ == 0) return BP_OK;
  int G, dpl;
  shape_of(dim, &G, &dpl);
  cudaStream_t s = (cudaStream_t)stream;
  if (P->d_seg_of && (dim & 3) == 0 && (row_stride & 3) == 0 && dim <= 32 && (32 % dim) == 0) {
    const int q = dim / 4, T = 32 * (8 / q);
    const long long tiles = (P->n_occ + T - 1) / T;
    const PeerSrc psrc = peer_src ? *peer_src : PeerSrc{nullptr, nullptr, 1, 1, 1, 1.f};
    // one allocation: tile partials, the spanning-key list and its count
    const size_t parts_bytes = ((size_t)tiles * 2 * q * sizeof(float4) + 255) & ~size_t(255);
    const size_t list_bytes = ((size_t)2 * tiles * sizeof(uint32_t) + 255) & ~size_t(255);
    char* scratch = nullptr;
    BP_CUDA_TRY(pool_alloc(&scratch, parts_bytes + list_bytes + 256, s));
    float4* parts = reinterpret_cast<float4*>(scratch);
    uint32_t* span_list = reinterpret_cast<uint32_t*>(scratch + parts_bytes);
    unsigned int* span_count = reinterpret_cast<unsigned int*>(scratch + parts_bytes + list_bytes);
    BP_CUDA_TRY(cudaMemsetAsync(span_count, 0, 2 * sizeof(unsigned int), s));
    const unsigned blocks = (unsigned)((tiles + 7) / 8);
#define BP_BWD_WARP(QQ)                                                                                        \
  k_embbag_bwd_warp<QQ><<<blocks, 256, 0, s>>>(P->d_occ_pos, P->d_seg_of, P->d_seg_start, P->n_occ,              \
                                               reinterpret_cast<const float4*>(d_grad), d_occ_bag, d_bag_scale,  \
                                               d_values, row_stride, d_slots_s, d_dirty, opt, lr, eps, parts,    \
                                               (unsigned long long*)d_stats, psrc, span_list, span_count, tiles)
    switch (q) {
      case 1: BP_BWD_WARP(1); break;
      case 2: BP_BWD_WARP(2); break;
      case 4: BP_BWD_WARP(4); break;
      default: BP_BWD_WARP(8); break;
    }
#undef BP_BWD_WARP
    k_embbag_bwd_span<<<kSpanSmallBlocks + kNumSMs, 256, 0, s>>>(
        P->d_seg_of, P->d_seg_start, P->n_occ, q, T, span_list, span_count, span_list + tiles, span_count + 1, parts,
        d_values, row_stride, d_slots_s, d_dirty, opt, lr, eps, (unsigned long long*)d_stats);
    BP_LAUNCH_CHECK();
    cudaFreeAsync(scratch, s);
    return BP_OK;
  }
  if (peer_src) return BP_ERR_INVALID;  // the peer source needs the warp-tile path
  if (P->d_seg_of && (dim & 3) == 0 && (row_stride & 3) == 0 && dim <= 128) {
    const int q = dim / 4, T = kBwdTileF4 / q;
    const long long tiles = (P->n_occ + T - 1) / T;
    const size_t parts_bytes = ((size_t)tiles * 2 * q * sizeof(float4) + 255) & ~size_t(255);
    const size_t list_bytes = ((size_t)2 * tiles * sizeof(uint32_t) + 255) & ~size_t(255);
    char* scratch = nullptr;
    BP_CUDA_TRY(pool_alloc(&scratch, parts_bytes + list_bytes + 256, s));
    float4* parts = reinterpret_cast<float4*>(scratch);
    uint32_t* span_list = reinterpret_cast<uint32_t*>(scratch + parts_bytes);
    unsigned int* span_count = reinterpret_cast<unsigned int*>(scratch + parts_bytes + list_bytes);
    BP_CUDA_TRY(cudaMemsetAsync(span_count, 0, 2 * sizeof(unsigned int), s));
    const size_t smem = sizeof(float4) * kBwdTileF4 + sizeof(uint32_t) * T;
    static bool attr = false;
    if (!attr) {
      BP_CUDA_TRY(cudaFuncSetAttribute(k_embbag_bwd_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10));
      attr = true;
    }
    k_embbag_bwd_tiles<<<(unsigned)tiles, 256, smem, s>>>(
        P->d_occ_pos, P->d_seg_of, P->d_seg_start, P->n_occ, q, T, reinterpret_cast<const float4*>(d_grad), d_occ_bag,
        d_bag_scale, d_values, row_stride, d_slots_s, d_dirty, opt, lr, eps, parts, (unsigned long long*)d_stats,
        span_list, span_count, tiles);
    k_embbag_bwd_span<<<kSpanSmallBlocks + kNumSMs, 256, 0, s>>>(
        P->d_seg_of, P->d_seg_start, P->n_occ, q, T, span_list, span_count, span_list + tiles, span_count + 1, parts,
        d_values, row_stride, d_slots_s, d_dirty, opt, lr, eps, (unsigned long long*)d_stats);
    BP_LAUNCH_CHECK();
    cudaFreeAsync(scratch, s);
    return BP_OK;
  }
  const BagGrad bg{d_grad, d_occ_bag, d_bag_scale};
  const int blocks = kBagLongBlocks + grid_for(P->n_occ * G, 256, kNumSMs * 6);
  BP_BAG_DISPATCH(G, dpl,
                  (k_embbag_bwd<g_, d_><<<blocks, 256, 0, s>>>(P->d_seg_start, P->d_occ_pos, P->d_num_unique,
                                                               P->d_long, P->d_num_long, P->long_cap, bg, d_values,
                                                               d_slots_s, d_dirty, dim, row_stride, opt, lr, eps,
                                                               (unsigned long long*)d_stats)));
  BP_LAUNCH_CHECK();
  return BP_OK;
}

// debug: the kernels behind bp_embbag_backward_sorted (0: the one-shot fused
// k_embbag_bwd_staged, 32 KB tiles -- the default, fastest inside the DLRM
// step; 6: the same with 16 KB tiles x 128 threads; 4: the split
// k_bwd_reduce + k_bwd_apply; 5: the persistent 3-stage k_embbag_bwd_pipe;
// warp tiles: 1: R=8 x 3 CTAs/SM, 2: R=4 x 4, 3: R=8 x 2).  Measured at CK
// shape (tools/embbag_instep.py, profiles/round2): in the step 0 = 6 = 30.7
// us, 4: 35.8 us, 5: slower still; isolated 24-25 us for 0/6, 28-31 us for 4/5.
// Sorted-gradient backward launch shape (bp_debug_bwd_variant; -1 = the
// default).  9 (default): register-resident reduce in 512-row CTA tiles +
// the per-key update (in-step CUPTI 19.5 us at CK shape against 26.7 us for
// the staged one-kernel form, variant 0).
constexpr int kBwdDefault = 9;
static int g_bwd_variant = kBwdDefault;

extern "C" int bp_debug_bwd_variant(int32_t v) {
  if (v < -1 || v > 10) return BP_ERR_INVALID;
  g_bwd_variant = v < 0 ? kBwdDefault : v;
  return BP_OK;
}

template <int R, int MINB>
static int launch_bwd_sorted(bp_prep* P, const float* d_grad_sorted, float* d_values, int32_t row_stride,
                             const int32_t* d_slots_s, uint8_t* d_dirty, int32_t dim, int32_t opt, float lr,
                             float eps, int64_t* d_stats, cudaStream_t s) {
  using namespace bp;
  const int q = dim / 4, T = (32 / q) * R;
  const long long tiles = (P->n_occ + T - 1) / T;
  // one allocation: tile partials (2 per tile) and the arrival counters
  const size_t parts_bytes = ((size_t)tiles * 2 * q * sizeof(float4) + 255) & ~size_t(255);
  char* scratch = nullptr;
  BP_CUDA_TRY(pool_alloc(&scratch, parts_bytes + tiles * sizeof(unsigned int) + 256, s));
  float4* parts = reinterpret_cast<float4*>(scratch);
  unsigned int* arrivals = reinterpret_cast<unsigned int*>(scratch + parts_bytes);
  BP_CUDA_TRY(cudaMemsetAsync(arrivals, 0, tiles * sizeof(unsigned int), s));
  const unsigned blocks = (unsigned)((tiles + 7) / 8);
#define BP_BWD_SORTED(QQ)                                                                                         \
  k_embbag_bwd_sorted<QQ, R, MINB><<<blocks, 256, 0, s>>>(P->d_seg_of, P->d_seg_start, (uint32_t)P->n_occ,        \
                                                          reinterpret_cast<const float4*>(d_grad_sorted), d_values, \
                                                          row_stride, d_slots_s, d_dirty, opt, lr, eps, parts,  \
                                                          arrivals, (unsigned long long*)d_stats)
  switch (q) {
    case 1: BP_BWD_SORTED(1); break;
    case 2: BP_BWD_SORTED(2); break;
    case 4: BP_BWD_SORTED(4); break;
    default: BP_BWD_SORTED(8); break;
  }
#undef BP_BWD_SORTED
  BP_LAUNCH_CHECK();
  cudaFreeAsync(scratch, s);
  return BP_OK;
}

// Scratch of the staged backward for n_occ occurrences: tile partials, then
// the arrival counters (zero between calls: the last arriver resets them).
extern "C" int64_t bp_embbag_bwd_scratch_bytes(int64_t n_occ, int32_t dim) {
  if (dim < 4 || (dim & 3) != 0) return 0;
  const int q = dim / 4, T = bp::kStagedF4 / 2 / q;  // the smaller staged tiles (variant 6): most tiles
  const long long tiles = (n_occ + T - 1) / T;
  const long long rtiles = (n_occ + bp::kRedF4 / q - 1) / (bp::kRedF4 / q);
  // parts [tiles][2][q] float4 | arrival counters | gsum [n_occ][q] float4 |
  // k_bwd_reduce parts [rtiles][2][q] float4
  // ... | spanning-key count + list of the register-resident reduce
  return (((long long)tiles * 2 * q * 16 + 255) & ~255ll) + ((tiles * 4 + 255) & ~255ll) + n_occ * q * 16 +
         rtiles * 2 * q * 16 + ((64 + rtiles) * 4 + 255) / 256 * 256 + 256;
}

static int embbag_backward_sorted_impl(bp_prep* P, const float* d_grad_sorted, float* d_values, int32_t row_stride,
                                       const int32_t* d_slots_s, uint8_t* d_dirty, int32_t dim, int32_t opt,
                                       float lr, float eps, int64_t* d_stats, bp_stream_t stream, char* own_scratch,
                                       size_t own_bytes);

extern "C" int bp_embbag_backward_sorted(bp_prep* P, const float* d_grad_sorted, float* d_values, int32_t row_stride,
                                         const int32_t* d_slots_s, uint8_t* d_dirty, int32_t dim, int32_t opt,
                                         float lr, float eps, int64_t* d_stats, bp_stream_t stream) {
  return embbag_backward_sorted_impl(P, d_grad_sorted, d_values, row_stride, d_slots_s, d_dirty, dim, opt, lr, eps,
                                     d_stats, stream, nullptr, 0);
}

// With a caller-owned scratch (bp_embbag_bwd_scratch_bytes, zeroed once):
// no per-call stream-ordered allocation (whose reuse of memory freed on
// another stream can make this stream wait for that one) and no memset.
extern "C" int bp_embbag_backward_sorted_scratch(bp_prep* P, const float* d_grad_sorted, float* d_values,
                                                 int32_t row_stride, const int32_t* d_slots_s, uint8_t* d_dirty,
                                                 int32_t dim, int32_t opt, float lr, float eps, int64_t* d_stats,
                                                 void* d_scratch, int64_t scratch_bytes, bp_stream_t stream) {
  return embbag_backward_sorted_impl(P, d_grad_sorted, d_values, row_stride, d_slots_s, d_dirty, dim, opt, lr, eps,
                                     d_stats, stream, static_cast<char*>(d_scratch), (size_t)scratch_bytes);
}

static int embbag_backward_sorted_impl(bp_prep* P, const float* d_grad_sorted, float* d_values, int32_t row_stride,
                                       const int32_t* d_slots_s, uint8_t* d_dirty, int32_t dim, int32_t opt,
                                       float lr, float eps, int64_t* d_stats, bp_stream_t stream, char* own_scratch,
                                       size_t own_bytes) {
  using namespace bp;
  if (!P->d_seg_of || (dim & 3) != 0 || (row_stride & 3) != 0 || dim > 32 || (32 % dim) != 0) return BP_ERR_INVALID;
  if (opt == BP_OPT_ADAGRAD && row_stride < 2 * dim) return BP_ERR_INVALID;
  if (P->n_occ == 0) return BP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  switch (g_bwd_variant) {
    case 0:
    case 4:
    case 5:
    case 6:
    case 7:
    case 8:
    case 9:
    case 10: {
      const int q = dim / 4, T = kStagedF4 / 2 / q;  // scratch layout of the smallest tiles
      const unsigned tiles = (unsigned)((P->n_occ + T - 1) / T);
      const size_t parts_bytes = ((size_t)tiles * 2 * q * sizeof(float4) + 255) & ~size_t(255);
      const bool own = own_scratch && own_bytes >= (size_t)bp_embbag_bwd_scratch_bytes(P->n_occ, dim);
      char* scratch = own ? own_scratch : nullptr;
      if (!own) BP_CUDA_TRY(pool_alloc(&scratch, (size_t)bp_embbag_bwd_scratch_bytes(P->n_occ, dim), s));
      float4* parts = reinterpret_cast<float4*>(scratch);
      unsigned int* arrivals = reinterpret_cast<unsigned int*>(scratch + parts_bytes);
      if (!own) BP_CUDA_TRY(cudaMemsetAsync(arrivals, 0, tiles * sizeof(unsigned int), s));
      if ((g_bwd_variant == 8 || g_bwd_variant == 9 || g_bwd_variant == 10) &&
          (reinterpret_cast<uintptr_t>(P->d_seg_of) & 15) == 0 &&
          (reinterpret_cast<uintptr_t>(d_grad_sorted) & 15) == 0) {
        // register-resident reduce + apply (k_bwd_reduce_reg, k_bwd_apply)
        float4* gsum = reinterpret_cast<float4*>(scratch + parts_bytes + ((tiles * sizeof(unsigned int) + 255) & ~size_t(255)));
        const bool r8 = g_bwd_variant == 9 || g_bwd_variant == 10;  // 4-warp CTAs: 2 KB tiles, more CTAs per SM
        const bool tma = g_bwd_variant == 10;
        const int Tr = (r8 ? kRegTileF4 / 2 : kRegTileF4) / q;
        const size_t tsmem = (size_t)Tr * q * sizeof(float4) + (size_t)Tr * sizeof(uint32_t);
        const unsigned rgrid = (unsigned)((P->n_occ + Tr - 1) / Tr);
        float4* rparts = gsum + (size_t)P->n_occ * q;
        // spanning-key list after the k_bwd_reduce tile partials
        const long long rtiles_max = (P->n_occ + kRedF4 / q - 1) / (kRedF4 / q);
        unsigned* span_count = reinterpret_cast<unsigned*>(rparts + (size_t)rtiles_max * 2 * q);
        uint32_t* span_list = span_count + 64;
        BP_CUDA_TRY(cudaMemsetAsync(span_count, 0, sizeof(unsigned), s));
        const int agrid = grid_for(P->n_occ * q, 256, kNumSMs * 8);
#define BP_BWD_REG(QQ)                                                                                        \
  if (tma) {                                                                                                  \
    static bool attr = false;                                                                                 \
    if (!attr) {                                                                                              \
      BP_CUDA_TRY(cudaFuncSetAttribute(k_bwd_reduce_reg<QQ, 16, 4, true>,                                     \
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem));             \
      attr = true;                                                                                            \
    }                                                                                                         \
    k_bwd_reduce_reg<QQ, 16, 4, true><<<rgrid, 128, tsmem, s>>>(P->d_seg_of, (uint32_t)P->n_occ,               \
                                                  reinterpret_cast<const float4*>(d_grad_sorted), gsum, rparts, \
                                                  span_list, span_count);                                      \
    k_bwd_apply<QQ, kRegTileF4 / 2><<<agrid, 256, 0, s>>>(P->d_seg_start, P->d_num_unique, gsum, rparts,       \
                                                          d_values, row_stride, d_slots_s, d_dirty, opt, lr,   \
                                                          eps, (unsigned long long*)d_stats, span_list,        \
                                                          span_count);                                         \
  } else if (r8) {                                                                                            \
    k_bwd_reduce_reg<QQ, 16, 4><<<rgrid, 128, 0, s>>>(P->d_seg_of, (uint32_t)P->n_occ,                          \
                                                  reinterpret_cast<const float4*>(d_grad_sorted), gsum, rparts, \
                                                  span_list, span_count);                                      \
    k_bwd_apply<QQ, kRegTileF4 / 2><<<agrid, 256, 0, s>>>(P->d_seg_start, P->d_num_unique, gsum, rparts,       \
                                                          d_values, row_stride, d_slots_s, d_dirty, opt, lr,   \
                                                          eps, (unsigned long long*)d_stats, span_list,        \
                                                          span_count);                                         \
  } else {                                                                                                    \
    k_bwd_reduce_reg<QQ><<<rgrid, 256, 0, s>>>(P->d_seg_of, (uint32_t)P->n_occ,                                 \
                                               reinterpret_cast<const float4*>(d_grad_sorted), gsum, rparts,   \
                                               span_list, span_count);                                         \
    k_bwd_apply<QQ, kRegTileF4><<<agrid, 256, 0, s>>>(P->d_seg_start, P->d_num_unique, gsum, rparts, d_values, \
                                                      row_stride, d_slots_s, d_dirty, opt, lr, eps,            \
                                                      (unsigned long long*)d_stats, span_list, span_count);    \
  }
        switch (q) {
          case 1: BP_BWD_REG(1); break;
          case 2: BP_BWD_REG(2); break;
          case 4: BP_BWD_REG(4); break;
          default: BP_BWD_REG(8); break;
        }
#undef BP_BWD_REG
        BP_LAUNCH_CHECK();
        if (!own) cudaFreeAsync(scratch, s);
        return BP_OK;
      }
      if (g_bwd_variant == 4) {
        float4* gsum = reinterpret_cast<float4*>(scratch + parts_bytes + ((tiles * sizeof(unsigned int) + 255) & ~size_t(255)));
        const int Tr = kRedF4 / q;
        const unsigned rtiles = (unsigned)((P->n_occ + Tr - 1) / Tr);
        float4* rparts = gsum + (size_t)P->n_occ * q;  // [rtiles][2][q] after gsum
        const size_t rsmem = (size_t)kPipeStages * ((size_t)Tr * q * sizeof(float4) + (size_t)Tr * sizeof(uint32_t));
        const unsigned grid = rtiles < 4u * kNumSMs ? rtiles : 4u * kNumSMs;
        const int agrid = grid_for(P->n_occ * q, 256, kNumSMs * 8);
#define BP_BWD_SPLIT(QQ)                                                                                       \
  {                                                                                                            \
    static bool attr = false;                                                                                  \
    if (!attr) {                                                                                               \
      BP_CUDA_TRY(cudaFuncSetAttribute(k_bwd_reduce<QQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,          \
                                       (int)rsmem));                                                           \
      attr = true;                                                                                             \
    }                                                                                                          \
    k_bwd_reduce<QQ><<<grid, 256, rsmem, s>>>(P->d_seg_of, (uint32_t)P->n_occ, rtiles,                          \
                                              reinterpret_cast<const float4*>(d_grad_sorted), gsum, rparts);   \
    k_bwd_apply<QQ><<<agrid, 256, 0, s>>>(P->d_seg_start, P->d_num_unique, gsum, rparts, d_values, row_stride, \
                                          d_slots_s, d_dirty, opt, lr, eps, (unsigned long long*)d_stats);     \
  }
        switch (q) {
          case 1: BP_BWD_SPLIT(1); break;
          case 2: BP_BWD_SPLIT(2); break;
          case 4: BP_BWD_SPLIT(4); break;
          default: BP_BWD_SPLIT(8); break;
        }
#undef BP_BWD_SPLIT
        BP_LAUNCH_CHECK();
        if (!own) cudaFreeAsync(scratch, s);
        return BP_OK;
      }
      if (g_bwd_variant == 5) {
        const int Tp = kStagedF4 / q;
        const size_t psmem = (size_t)kPipeStages * ((size_t)Tp * q * sizeof(float4) + (size_t)Tp * sizeof(uint32_t)) +
                             (size_t)Tp * sizeof(int32_t);
        const unsigned ptiles = (unsigned)((P->n_occ + kStagedF4 / q - 1) / (kStagedF4 / q));
        const unsigned grid = ptiles < 2u * kNumSMs ? ptiles : 2u * kNumSMs;
#define BP_BWD_PIPE(QQ)                                                                                        \
  {                                                                                                            \
    static bool attr = false;                                                                                  \
    if (!attr) {                                                                                               \
      BP_CUDA_TRY(cudaFuncSetAttribute(k_embbag_bwd_pipe<QQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                       (int)psmem));                                                           \
      attr = true;                                                                                             \
    }                                                                                                          \
    k_embbag_bwd_pipe<QQ><<<grid, 256, psmem, s>>>(P->d_seg_of, P->d_seg_start, (uint32_t)P->n_occ, ptiles,     \
                                                   reinterpret_cast<const float4*>(d_grad_sorted), d_values,    \
                                                   row_stride, d_slots_s, d_dirty, opt, lr, eps, parts,         \
                                                   arrivals, (unsigned long long*)d_stats);                     \
  }
        switch (q) {
          case 1: BP_BWD_PIPE(1); break;
          case 2: BP_BWD_PIPE(2); break;
          case 4: BP_BWD_PIPE(4); break;
          default: BP_BWD_PIPE(8); break;
        }
#undef BP_BWD_PIPE
        BP_LAUNCH_CHECK();
        if (!own) cudaFreeAsync(scratch, s);
        return BP_OK;
      }
      // one-shot staged tiles: 32 KB x 256 threads (variant 4) or 16 KB x 128
      // threads (variant 6: twice the CTAs resident per SM)
      const bool small = g_bwd_variant == 6;
      const bool no_ends = g_bwd_variant == 7;  // the round-1 pass 3 over every row
      const int Ts = (small ? kStagedF4 / 2 : kStagedF4) / q;
      const unsigned stiles = (unsigned)((P->n_occ + Ts - 1) / Ts);
      const size_t smem = (size_t)Ts * q * sizeof(float4) + 2 * (size_t)Ts * sizeof(uint32_t);
#define BP_BWD_STAGED(QQ, NT, F4, ...)                                                                         \
  {                                                                                                            \
    static bool attr = false;                                                                                  \
    if (!attr) {                                                                                               \
      BP_CUDA_TRY(cudaFuncSetAttribute(k_embbag_bwd_staged<QQ, NT, F4, ##__VA_ARGS__>,                         \
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));               \
      attr = true;                                                                                             \
    }                                                                                                          \
    k_embbag_bwd_staged<QQ, NT, F4, ##__VA_ARGS__><<<stiles, NT, smem, s>>>(                                   \
        P->d_seg_of, P->d_seg_start, (uint32_t)P->n_occ, reinterpret_cast<const float4*>(d_grad_sorted),       \
        d_values, row_stride, d_slots_s, d_dirty, opt, lr, eps, parts, arrivals,                               \
        (unsigned long long*)d_stats);                                                                         \
  }
      if (no_ends) {
        switch (q) {
          case 1: BP_BWD_STAGED(1, 256, kStagedF4, false); break;
          case 2: BP_BWD_STAGED(2, 256, kStagedF4, false); break;
          case 4: BP_BWD_STAGED(4, 256, kStagedF4, false); break;
          default: BP_BWD_STAGED(8, 256, kStagedF4, false); break;
        }
      } else if (small) {
        switch (q) {
          case 1: BP_BWD_STAGED(1, 128, kStagedF4 / 2); break;
          case 2: BP_BWD_STAGED(2, 128, kStagedF4 / 2); break;
          case 4: BP_BWD_STAGED(4, 128, kStagedF4 / 2); break;
          default: BP_BWD_STAGED(8, 128, kStagedF4 / 2); break;
        }
      } else {
        switch (q) {
          case 1: BP_BWD_STAGED(1, 256, kStagedF4); break;
          case 2: BP_BWD_STAGED(2, 256, kStagedF4); break;
          case 4: BP_BWD_STAGED(4, 256, kStagedF4); break;
          default: BP_BWD_STAGED(8, 256, kStagedF4); break;
        }
      }
#undef BP_BWD_STAGED
      BP_LAUNCH_CHECK();
      if (!own) cudaFreeAsync(scratch, s);
      return BP_OK;
    }
    case 1: return launch_bwd_sorted<8, 3>(P, d_grad_sorted, d_values, row_stride, d_slots_s, d_dirty, dim, opt, lr,
                                           eps, d_stats, s);
    case 2: return launch_bwd_sorted<4, 4>(P, d_grad_sorted, d_values, row_stride, d_slots_s, d_dirty, dim, opt, lr,
                                           eps, d_stats, s);
    default: return launch_bwd_sorted<8, 2>(P, d_grad_sorted, d_values, row_stride, d_slots_s, d_dirty, dim, opt, lr,
                                            eps, d_stats, s);  // 3
  }
}

extern "C" int bp_prep_occ_rank(bp_prep* P, uint32_t* d_out, bp_stream_t stream) {
  if (!P->d_occ_rank) return BP_ERR_INVALID;
  if (P->n_occ == 0) return BP_OK;
  BP_CUDA_TRY(cudaMemcpyAsync(d_out, P->d_occ_rank, P->n_occ * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                              (cudaStream_t)stream));
  return BP_OK;
}

extern "C" int bp_prep_occ_sorted_index(bp_prep* P, uint32_t* d_occ_s, bp_stream_t stream) {
  using namespace bp;
  if (P->n_occ == 0) return BP_OK;
  k_occ_sorted_index<<<grid_for(P->n_occ, 256), 256, 0, (cudaStream_t)stream>>>(P->d_seg_start, P->d_occ_pos,
                                                                                 P->d_num_unique, P->n_occ, d_occ_s);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_embbag_backward(bp_prep* P, const float* d_grad, const int64_t* d_occ_bag,
                                  const float* d_bag_scale, float* d_values, int32_t row_stride,
                                  const int32_t* d_slots_s, uint8_t* d_dirty, int32_t dim, int32_t opt, float lr,
                                  float eps, int64_t* d_stats, bp_stream_t stream) {
  return embbag_backward_impl(P, d_grad, d_occ_bag, d_bag_scale, d_values, row_stride, d_slots_s, d_dirty, dim, opt,
                              lr, eps, d_stats, stream, nullptr);
}

extern "C" int bp_embbag_backward_peer(bp_prep* P, const bp_peer_xchg* x, float scale, float* d_values,
                                       int32_t row_stride, const int32_t* d_slots_s, uint8_t* d_dirty, int32_t dim,
                                       int32_t opt, float lr, float eps, int64_t* d_stats, bp_stream_t stream) {
  using namespace bp;
  if (!x || !P->d_seg_of || (dim & 3) != 0 || dim > 32 || (32 % dim) != 0 || x->n_cols < 1 || x->bl < 1)
    return BP_ERR_INVALID;
  if (P->n_occ != x->bl * x->world * x->n_cols) return BP_ERR_INVALID;
  const PeerSrc ps{reinterpret_cast<float4* const*>(x->d_peer_rows), x->d_col_tables, x->bl, x->t_global, x->n_cols,
                   scale};
  return embbag_backward_impl(P, nullptr, nullptr, nullptr, d_values, row_stride, d_slots_s, d_dirty, dim, opt, lr,
                              eps, d_stats, stream, &ps);
}

namespace bp {

// Peer gradient rows pulled into key-sorted order: sorted position j (one
// float4 lane per (j, 4 components): coalesced stores) takes the gradient
// row of occurrence occ_pos[j] from its example owner's buffer over NVLink,
// scaled.  The staged sorted backward then streams the local buffer.
template <int QT>
__global__ void __launch_bounds__(256) k_peer_gather_sorted(const uint32_t* __restrict__ occ_pos, int q_rt,
                                                           long long n, PeerSrc src, float4* __restrict__ out) {
  constexpr int U = 4;
  const int q = QT > 0 ? QT : q_rt;
  const long long total = n * q;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total; i0 += stride * U) {
    float4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = i0 + k * stride;
      v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < total) v[k] = peer_row(src, __ldg(occ_pos + i / q), q)[i % q];
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long i = i0 + k * stride;
      if (i < total) {
        float4 x = v[k];
        if (src.scale != 1.f) {
          x.x = __fmul_rn(x.x, src.scale);
          x.y = __fmul_rn(x.y, src.scale);
          x.z = __fmul_rn(x.z, src.scale);
          x.w = __fmul_rn(x.w, src.scale);
        }
        out[i] = x;
      }
    }
  }
}

}  // namespace bp

// Peer backward through the key-sorted path: the gradient rows of the rank's
// occurrences gathered from the example owners into d_sorted (n_occ x dim
// floats, caller-owned) in key-sorted order, then the staged sorted backward
// (d_scratch: bp_embbag_bwd_scratch_bytes, zeroed once).
extern "C" int bp_embbag_backward_peer_sorted(bp_prep* P, const bp_peer_xchg* x, float scale, float* d_values,
                                              int32_t row_stride, const int32_t* d_slots_s, uint8_t* d_dirty,
                                              int32_t dim, int32_t opt, float lr, float eps, int64_t* d_stats,
                                              float* d_sorted, void* d_scratch, int64_t scratch_bytes,
                                              bp_stream_t stream) {
  using namespace bp;
  if (!x || !P->d_seg_of || (dim & 3) != 0 || dim > 32 || (32 % dim) != 0 || x->n_cols < 1 || x->bl < 1)
    return BP_ERR_INVALID;
  if (P->n_occ != x->bl * x->world * x->n_cols) return BP_ERR_INVALID;
  if (P->n_occ == 0) return BP_OK;
  const int q = dim / 4;
  const PeerSrc ps{reinterpret_cast<float4* const*>(x->d_peer_rows), x->d_col_tables, x->bl, x->t_global, x->n_cols,
                   scale};
  const int gg = grid_for(P->n_occ * q, 256 * 4, kNumSMs * 8);
  float4* out4 = reinterpret_cast<float4*>(d_sorted);
  cudaStream_t gs = (cudaStream_t)stream;
  switch (q) {
    case 1: k_peer_gather_sorted<1><<<gg, 256, 0, gs>>>(P->d_occ_pos, q, P->n_occ, ps, out4); break;
    case 2: k_peer_gather_sorted<2><<<gg, 256, 0, gs>>>(P->d_occ_pos, q, P->n_occ, ps, out4); break;
    case 4: k_peer_gather_sorted<4><<<gg, 256, 0, gs>>>(P->d_occ_pos, q, P->n_occ, ps, out4); break;
    default: k_peer_gather_sorted<8><<<gg, 256, 0, gs>>>(P->d_occ_pos, q, P->n_occ, ps, out4); break;
  }
  BP_LAUNCH_CHECK();
  return bp_embbag_backward_sorted_scratch(P, d_sorted, d_values, row_stride, d_slots_s, d_dirty, dim, opt, lr, eps,
                                           d_stats, d_scratch, scratch_bytes, stream);
}

extern "C" int bp_embbag_forward_peer(bp_prep* P, const float* d_values, int32_t row_stride, const int32_t* d_slots_s,
                                      int32_t dim, const bp_peer_xchg* x, bp_stream_t stream) {
  using namespace bp;
  if (!x || !P->d_occ_s || (dim & 3) != 0 || (row_stride & 3) != 0 || x->n_cols < 1 || x->bl < 1)
    return BP_ERR_INVALID;
  if (P->n_occ != x->bl * x->world * x->n_cols) return BP_ERR_INVALID;
  if (P->n_occ == 0) return BP_OK;
  const int q = dim / 4;
  const PeerSrc dst{reinterpret_cast<float4* const*>(x->d_peer_rows), x->d_col_tables, x->bl, x->t_global, x->n_cols,
                    1.f};
  const int fg = grid_for(P->n_occ * q, 256 * 4, kNumSMs * 8);
  const float4* vals4 = reinterpret_cast<const float4*>(d_values);
  cudaStream_t fs = (cudaStream_t)stream;
  switch (q) {
    case 1: k_embbag_fwd_peer_v4<1><<<fg, 256, 0, fs>>>(P->d_occ_s, d_slots_s, vals4, q, row_stride / 4, P->n_occ, dst); break;
    case 2: k_embbag_fwd_peer_v4<2><<<fg, 256, 0, fs>>>(P->d_occ_s, d_slots_s, vals4, q, row_stride / 4, P->n_occ, dst); break;
    case 4: k_embbag_fwd_peer_v4<4><<<fg, 256, 0, fs>>>(P->d_occ_s, d_slots_s, vals4, q, row_stride / 4, P->n_occ, dst); break;
    case 8: k_embbag_fwd_peer_v4<8><<<fg, 256, 0, fs>>>(P->d_occ_s, d_slots_s, vals4, q, row_stride / 4, P->n_occ, dst); break;
    default: k_embbag_fwd_peer_v4<0><<<fg, 256, 0, fs>>>(P->d_occ_s, d_slots_s, vals4, q, row_stride / 4, P->n_occ, dst); break;
  }
  BP_LAUNCH_CHECK();
  return BP_OK;
}
