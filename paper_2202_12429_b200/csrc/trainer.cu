// Fused stub backward + rank-ordered combine + SGD (the reference's whole
// "EmbeddingBag backward + sparse optimizer": trainer.py:37-53, 92-105,
// 140-146, driven by engine.py:545-579 / 706-718).
//
// Bit-exactness: np.add.at accumulates sequentially, per key, in occurrence
// order, starting from +0.0; the cross-rank combine is a second sequential
// sum in ascending rank.  A tree or warp reduction would change the float32
// rounding, so each (key, component) is one sequential chain here: a group of
// G lanes owns a key (lane = component), walks the key's occurrence list (the
// stable sort in prep.cu keeps it in occurrence order) rank by rank, and
// applies SGD in place.  Parallelism comes from the ~75K keys x 16 components
// of a Criteo-Kaggle batch; the longest chain (a 3-row table's hot key,
// ~9K occurrences per batch) bounds the kernel at a few tens of microseconds.
// Every multiply/add uses an explicit _rn intrinsic: no FMA contraction.
#include "internal.cuh"

namespace bp {

// Accumulate the occurrence bytes [lo, hi) of one 16-byte chunk into the
// per-component chains.  Byte = label (7 bits) | rank-start flag (bit 7);
// ``first_q`` is the chunk offset of the key's first occurrence (16 if the
// key does not start in this chunk): its flag opens the chain, every other
// flag closes the running rank partial into ``comb``.
template <int DPL>
__device__ __forceinline__ void chain_chunk(const uint32_t (&word)[4], uint32_t lo, uint32_t hi, uint32_t first_q,
                                            float (&acc)[DPL], float (&comb)[DPL], const float (&t0)[DPL],
                                            const float (&t1)[DPL], const float (&sc)[DPL], float c_label) {
  const uint32_t big = (word[0] | word[1] | word[2] | word[3]) & 0x7E7E7E7Eu;
  const uint32_t flags_hi = (word[1] | word[2] | word[3]) & 0x80808080u;
  const uint32_t flags_lo = word[0] & 0x80808080u;
  if (lo == 0 && hi == 16 && !big && !flags_hi && (flags_lo == 0 || (first_q == 0 && flags_lo == 0x80u))) {
    // 16 occurrences, labels 0/1, no rank change: one select + one add each.
    if constexpr (DPL == 1) {
      // all 16 selects first (independent of the chain), then the 16
      // dependent adds back to back: the chain runs at the add latency
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = ((word[i >> 2] >> ((i & 3) * 8)) & 1u) ? t1[0] : t0[0];
      float a = acc[0];
#pragma unroll
      for (int i = 0; i < 16; ++i) a = __fadd_rn(a, v[i]);
      acc[0] = a;
    } else {
#pragma unroll
      for (int wi = 0; wi < 4; ++wi) {
#pragma unroll
        for (int bi = 0; bi < 4; ++bi) {
          const bool one = (word[wi] >> (bi * 8)) & 1u;
#pragma unroll
          for (int q = 0; q < DPL; ++q) acc[q] = __fadd_rn(acc[q], one ? t1[q] : t0[q]);
        }
      }
    }
    return;
  }
  for (uint32_t q8 = lo; q8 < hi; ++q8) {
    const uint32_t byte = (word[q8 >> 2] >> ((q8 & 3) * 8)) & 0xFFu;
    const uint32_t lab = byte & 0x7Fu;
    if ((byte & 0x80u) && q8 != first_q) {
#pragma unroll
      for (int q = 0; q < DPL; ++q) {
        comb[q] = __fadd_rn(comb[q], acc[q]);
        acc[q] = 0.f;
      }
    }
#pragma unroll
    for (int q = 0; q < DPL; ++q) {
      const float t = lab == 0 ? t0[q]
                    : lab == 1 ? t1[q]
                               : __fadd_rn(sc[q], __fmul_rn(c_label, __fsub_rn((float)lab, 0.5f)));
      acc[q] = __fadd_rn(acc[q], t);
    }
  }
}

constexpr int kLongBlocks = 148;       // CTAs of the long-segment launch (one per SM)
// Optional per-CTA phase timestamps of k_stub_step_long (tools/kernel_bench.py;
// nullptr in production): [cta][8] = start, setup, window staged, chain
// done, end, segment length.
__device__ unsigned long long* g_long_trace = nullptr;
// Unused dynamic shared memory that keeps the long-segment CTAs one per SM:
// the block scheduler would otherwise pack several 128-thread CTAs onto one
// SM and their chain warps would share issue slots.
constexpr int kLongSmemPad = 120 << 10;
// bp_set_stub_long_smem: the pad in bytes (default kLongSmemPad); the
// largest pad keeps short-kernel CTAs off the chain's SM altogether
static int g_long_smem = kLongSmemPad;
constexpr int kLongWindowChunks = 1024;  // 16 KB of occurrence bytes staged in smem

// Fused trainer, two launches.  k_stub_step_long (first) takes the keys whose
// segment has >= kLongSeg occurrences (the Zipf-hot rows of tiny tables, up
// to ~9K per batch at Criteo-Kaggle), longest first: the CTA stages the key's
// occurrence bytes in shared memory with coalesced 16-byte loads, then one
// warp runs the per-component chains from shared memory (broadcast reads, no
// global latency inside the chain).  Running alone keeps the chain warp's
// issue slots free (3 instructions per occurrence on a 4-cycle add chain).
// k_stub_step then handles the short segments with one group of G lanes per
// key (lane = component, DPL components per lane when dim > 32): every
// per-key load that does not depend on another is issued up front, and the
// label chunks are prefetched two rounds ahead.
template <int G, int DPL>
__global__ void __launch_bounds__(1024) k_stub_step_long(
    const uint32_t* __restrict__ seg_start, const uint8_t* __restrict__ occ_label,
    const long long* __restrict__ d_U, const uint32_t* __restrict__ long_list,
    const long long* __restrict__ d_num_long, long long long_cap, float* __restrict__ rows, const int32_t* __restrict__ row_index,
    uint8_t* __restrict__ dirty, int dim, float c_value, float c_label, float lr, int mode,
    float* __restrict__ grad_out, const uint32_t* __restrict__ my_ids, const int64_t* __restrict__ next_mark,
    long long next_tag, unsigned long long* __restrict__ stats, const uint32_t* __restrict__ occ_pos,
    const long long* __restrict__ rank_bounds, int num_ranks, float* __restrict__ rank_parts) {
  const unsigned lane = threadIdx.x & 31u;
  const uint4* __restrict__ chunks = reinterpret_cast<const uint4*>(occ_label);
  const float b0 = __fmul_rn(c_label, -0.5f), b1 = __fmul_rn(c_label, 0.5f);

  {
    __shared__ uint4 win[kLongWindowChunks];
    __shared__ uint32_t winfo[kLongWindowChunks];
    const long long n_vlong = d_num_long[0], n_long = n_vlong + d_num_long[1];
    const bool chain_lane = threadIdx.x < G;  // warp 0, lanes [0, G)
    // very long segments first (front of the list), then the others (back)
    unsigned long long* tr = g_long_trace ? g_long_trace + blockIdx.x * 8 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = clock64();
    // rank split (rank_parts != nullptr, num_ranks > 1): one work item per
    // (key, rank) -- the rank's run of the key's occurrences is an
    // independent sequential chain; k_stub_long_combine adds the rank
    // partials in ascending rank order, which is exactly the reference's
    // combine (a rank without occurrences contributes +0.0, an exact no-op)
    const int T = rank_parts ? num_ranks : 1;
    for (long long it = blockIdx.x; it < n_long * T; it += gridDim.x) {
      const long long li = it / T;
      const int rk = (int)(it - li * T);
      const uint32_t s = li < n_vlong ? long_list[li] : long_list[long_cap - 1 - (li - n_vlong)];
      uint32_t a = seg_start[s], b = seg_start[s + 1];
      const int32_t row = row_index ? row_index[s] : (int32_t)s;
      if (row < 0) continue;  // block-uniform: the miss is already recorded
      if (T > 1) {
        // the rank's occurrences: positions ascend within the key's run
        uint32_t lo = a, hi = b;
        if (rk > 0) {
          const long long bound = rank_bounds[rk];
          uint32_t l = a, h = b;
          while (l < h) {
            const uint32_t m = (l + h) >> 1;
            if ((long long)occ_pos[m] < bound) l = m + 1;
            else h = m;
          }
          lo = l;
        }
        if (rk + 1 < T) {
          const long long bound = rank_bounds[rk + 1];
          uint32_t l = lo, h = b;
          while (l < h) {
            const uint32_t m = (l + h) >> 1;
            if ((long long)occ_pos[m] < bound) l = m + 1;
            else h = m;
          }
          hi = l;
        }
        if (lo >= hi) {  // block-uniform: no occurrence in this rank
          for (int d = threadIdx.x; d < dim; d += blockDim.x) rank_parts[(it)*dim + d] = 0.f;
          continue;
        }
        a = lo;
        b = hi;
      }
      if (tr && threadIdx.x == 0) tr[5] = b - a;
      float v[DPL], t0[DPL], t1[DPL], sc[DPL], acc[DPL], comb[DPL];
#pragma unroll
      for (int q = 0; q < DPL; ++q) {
        const int d = (int)threadIdx.x + q * G;
        v[q] = (chain_lane && d < dim) ? rows[(long long)row * dim + d] : 0.f;
        sc[q] = __fmul_rn(c_value, v[q]);
        t0[q] = __fadd_rn(sc[q], b0);
        t1[q] = __fadd_rn(sc[q], b1);
        acc[q] = 0.f;
        comb[q] = 0.f;
      }
      const uint32_t c0 = a >> 4, c_end = ((b - 1) >> 4) + 1;
      if (tr && threadIdx.x == 0) tr[1] = clock64() + 0 * (unsigned long long)__float_as_uint(t0[0]);
      for (uint32_t wc = c0; wc < c_end; wc += kLongWindowChunks) {
        const uint32_t nchunk = min((uint32_t)kLongWindowChunks, c_end - wc);
        // all warps stage the bytes and classify each chunk: info = 16-bit
        // label mask | (1 << 16) when the chunk is a plain run (16 of this
        // key's occurrences, labels 0/1, no rank change) -- so the chain warp
        // does only select + add on those
        for (uint32_t k = threadIdx.x; k < nchunk; k += blockDim.x) {
          const uint4 w4 = chunks[wc + k];
          win[k] = w4;
          const uint32_t cbase = (wc + k) << 4;
          const uint32_t word[4] = {w4.x, w4.y, w4.z, w4.w};
          const uint32_t big = (w4.x | w4.y | w4.z | w4.w) & 0x7E7E7E7Eu;
          const uint32_t flags_hi = (w4.y | w4.z | w4.w) & 0x80808080u;
          const uint32_t flags_lo = w4.x & 0x80808080u;
          const bool full = a <= cbase && b >= cbase + 16;
          const bool plain = full && !big && !flags_hi && (flags_lo == 0 || (a == cbase && flags_lo == 0x80u));
          uint32_t m = 0;
#pragma unroll
          for (int i = 0; i < 16; ++i) m |= ((word[i >> 2] >> ((i & 3) * 8)) & 1u) << i;
          winfo[k] = m | (plain ? 0x10000u : 0u);
        }
        __syncthreads();
        if (tr && threadIdx.x == 0) tr[2] = clock64();
        if (chain_lane) {
          uint32_t k = 0;
          while (k < nchunk) {
            uint32_t info = winfo[k];
            if constexpr (DPL == 1) {
              if (info & 0x10000u) {
                // a run of plain chunks, four at a time: one basic block of
                // 64 selects + 64 dependent adds, so the scheduler hides the
                // selects (and the R2P label unpacking) under the add chain
                // instead of paying them in front of every 16 adds (measured
                // 7.6 cycles per add for one chunk per iteration).  The next
                // quad's chunk infos are loaded a quad ahead.
                float a0 = acc[0];
                const auto ld = [&](uint32_t j) { return j < nchunk ? winfo[j] : 0u; };
                uint32_t c0 = info, c1 = ld(k + 1), c2 = ld(k + 2), c3 = ld(k + 3);
                for (;;) {
                  const uint32_t n0 = ld(k + 4), n1 = ld(k + 5), n2 = ld(k + 6), n3 = ld(k + 7);
                  if (c0 & c1 & c2 & c3 & 0x10000u) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) a0 = __fadd_rn(a0, ((c0 >> i) & 1u) ? t1[0] : t0[0]);
#pragma unroll
                    for (int i = 0; i < 16; ++i) a0 = __fadd_rn(a0, ((c1 >> i) & 1u) ? t1[0] : t0[0]);
#pragma unroll
                    for (int i = 0; i < 16; ++i) a0 = __fadd_rn(a0, ((c2 >> i) & 1u) ? t1[0] : t0[0]);
#pragma unroll
                    for (int i = 0; i < 16; ++i) a0 = __fadd_rn(a0, ((c3 >> i) & 1u) ? t1[0] : t0[0]);
                    k += 4;
                    c0 = n0;
                    c1 = n1;
                    c2 = n2;
                    c3 = n3;
                  } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) a0 = __fadd_rn(a0, ((c0 >> i) & 1u) ? t1[0] : t0[0]);
                    k += 1;
                    c0 = c1;
                    c1 = c2;
                    c2 = c3;
                    c3 = n0;
                  }
                  if (!(c0 & 0x10000u)) break;
                }
                acc[0] = a0;
                continue;
              }
            }
            const uint4 w4 = win[k];
            const uint32_t word[4] = {w4.x, w4.y, w4.z, w4.w};
            const uint32_t cbase = (wc + k) << 4;
            const uint32_t lo = a > cbase ? a - cbase : 0u;
            const uint32_t hi = b - cbase < 16u ? b - cbase : 16u;
            const uint32_t first_q = (a >= cbase && a < cbase + 16) ? a - cbase : 16u;
            chain_chunk<DPL>(word, lo, hi, first_q, acc, comb, t0, t1, sc, c_label);
            ++k;
          }
          if (tr && threadIdx.x == 0) tr[3] = clock64() + 0 * (unsigned long long)__float_as_uint(acc[0]);
        }
        __syncthreads();
      }
      if (T > 1) {  // the rank partial, for k_stub_long_combine
        if (chain_lane) {
#pragma unroll
          for (int q = 0; q < DPL; ++q) {
            const int d = (int)threadIdx.x + q * G;
            if (d < dim) rank_parts[it * dim + d] = __fadd_rn(comb[q], acc[q]);
          }
        }
        continue;
      }
      if (threadIdx.x < 32) {
        bool nonzero = false;
#pragma unroll
        for (int q = 0; q < DPL; ++q) {
          comb[q] = __fadd_rn(comb[q], acc[q]);
          const int d = (int)threadIdx.x + q * G;
          if (chain_lane && d < dim) {
            nonzero |= comb[q] != 0.f;
            if (mode == BP_STUB_SGD) rows[(long long)row * dim + d] = __fsub_rn(v[q], __fmul_rn(lr, comb[q]));
            else grad_out[(long long)s * dim + d] = comb[q];
          }
        }
        const bool nz = __ballot_sync(0xffffffffu, nonzero) != 0;
        if (threadIdx.x == 0) {
          if (nz && dirty && mode == BP_STUB_SGD) dirty[row] = 1;
          if (stats) {
            if (next_mark && next_mark[my_ids[s]] == next_tag) atomicAdd(&stats[0], 1ull);
            if (nz) atomicAdd(&stats[1], 1ull);
          }
        }
      }
    }
    if (tr && threadIdx.x == 0) tr[4] = clock64();
    return;
  }

}

template <int G, int DPL>
__global__ void __launch_bounds__(256, 6) k_stub_step(
    const uint32_t* __restrict__ seg_start, const uint8_t* __restrict__ occ_label,
    const long long* __restrict__ d_U, const uint32_t* __restrict__ long_list,
    const long long* __restrict__ d_num_long, long long long_cap, float* __restrict__ rows, const int32_t* __restrict__ row_index,
    uint8_t* __restrict__ dirty, int dim, float c_value, float c_label, float lr, int mode,
    float* __restrict__ grad_out, const uint32_t* __restrict__ my_ids, const int64_t* __restrict__ next_mark,
    long long next_tag, unsigned long long* __restrict__ stats) {
  const unsigned lane = threadIdx.x & 31u;
  const uint4* __restrict__ chunks = reinterpret_cast<const uint4*>(occ_label);
  const float b0 = __fmul_rn(c_label, -0.5f), b1 = __fmul_rn(c_label, 0.5f);

  const long long U = *d_U;
  const int lane_g = (int)(lane & (G - 1));
  const unsigned gbase = lane & ~(unsigned)(G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
  const long long groups_per_block = blockDim.x / G;
  const long long groups_total = (long long)gridDim.x * groups_per_block;
  const long long warp_first = (long long)blockIdx.x * groups_per_block + (threadIdx.x >> 5) * (32 / G);
  // the counters are summed per CTA in shared memory: one global atomic per
  // CTA instead of one per warp and key round on the same two addresses
  __shared__ unsigned int cta_stats[2];
  if (threadIdx.x < 2) cta_stats[threadIdx.x] = 0u;
  __syncthreads();

  for (long long base = warp_first; base < U; base += groups_total) {
    const long long s = base + (long long)(lane / G);
    bool active = s < U;
    uint32_t a = 0, b = 0;
    int32_t row = 0;
    bool crit = false;
    if (active) {
      a = seg_start[s];
      b = seg_start[s + 1];
      row = row_index ? row_index[s] : (int32_t)s;
      if (next_mark && lane_g == 0) crit = next_mark[my_ids[s]] == next_tag;
      active = row >= 0 && b - a < kLongSeg;  // long segments belong to the long CTAs
    }
    bool nonzero = false;
    if (active) {
      float v[DPL], t0[DPL], t1[DPL], sc[DPL], acc[DPL], comb[DPL];
#pragma unroll
      for (int q = 0; q < DPL; ++q) {
        const int d = lane_g + q * G;
        v[q] = d < dim ? rows[(long long)row * dim + d] : 0.f;
        sc[q] = __fmul_rn(c_value, v[q]);
        t0[q] = __fadd_rn(sc[q], b0);
        t1[q] = __fadd_rn(sc[q], b1);
        acc[q] = 0.f;
        comb[q] = 0.f;
      }
      const uint32_t c_first = a >> 4;
      const uint32_t n_chunks = ((b - 1) >> 4) - c_first + 1;
      const uint4 zero4 = make_uint4(0, 0, 0, 0);
      uint4 w0 = lane_g < (int)n_chunks ? chunks[c_first + lane_g] : zero4;
      uint4 w1 = lane_g + G < (int)n_chunks ? chunks[c_first + G + lane_g] : zero4;
      for (uint32_t r0 = 0; r0 < n_chunks; r0 += G) {
        const uint32_t nxt = r0 + 2 * G + lane_g;
        const uint4 w2 = nxt < n_chunks ? chunks[c_first + nxt] : zero4;
        const uint32_t in_round = min((uint32_t)G, n_chunks - r0);
        for (uint32_t i = 0; i < in_round; ++i) {
          uint32_t word[4];
          word[0] = __shfl_sync(gmask, w0.x, (int)i, G);
          word[1] = __shfl_sync(gmask, w0.y, (int)i, G);
          word[2] = __shfl_sync(gmask, w0.z, (int)i, G);
          word[3] = __shfl_sync(gmask, w0.w, (int)i, G);
          const uint32_t cbase = (c_first + r0 + i) << 4;
          const uint32_t lo = a > cbase ? a - cbase : 0u;
          const uint32_t hi = b - cbase < 16u ? b - cbase : 16u;
          const uint32_t first_q = (a >= cbase && a < cbase + 16) ? a - cbase : 16u;
          chain_chunk<DPL>(word, lo, hi, first_q, acc, comb, t0, t1, sc, c_label);
        }
        w0 = w1;
        w1 = w2;
      }
#pragma unroll
      for (int q = 0; q < DPL; ++q) {
        comb[q] = __fadd_rn(comb[q], acc[q]);
        const int d = lane_g + q * G;
        if (d < dim) {
          nonzero |= comb[q] != 0.f;
          if (mode == BP_STUB_SGD) rows[(long long)row * dim + d] = __fsub_rn(v[q], __fmul_rn(lr, comb[q]));
          else grad_out[s * dim + d] = comb[q];
        }
      }
    }
    const unsigned nz = __ballot_sync(0xffffffffu, nonzero) & gmask;
    // critical = needed by the next batch (reference engine.py:560-564): the
    // next batch's ids carry its iteration tag in a dense mark array.
    crit = crit && active;
    if (active && lane_g == 0 && nz && dirty && mode == BP_STUB_SGD) dirty[row] = 1;
    if (stats) {
      const unsigned cm = __ballot_sync(0xffffffffu, crit);
      const unsigned dm = __ballot_sync(0xffffffffu, active && lane_g == 0 && nz != 0);
      if (lane == 0) {
        if (cm) atomicAdd(&cta_stats[0], (unsigned)__popc(cm));
        if (dm) atomicAdd(&cta_stats[1], (unsigned)__popc(dm));
      }
    }
  }
  if (stats) {
    __syncthreads();
    if (threadIdx.x < 2 && cta_stats[threadIdx.x]) atomicAdd(&stats[threadIdx.x], (unsigned long long)cta_stats[threadIdx.x]);
  }
}

// Rank partials of the long keys -> per key ((0 + G_0) + G_1) + ... in rank
// order, then the SGD update / gradient output, dirty and counters (the tail
// of k_stub_step_long for the rank-split case).  A warp per long key.
template <int G, int DPL>
__global__ void __launch_bounds__(256) k_stub_long_combine(
    const long long* __restrict__ d_num_long, const uint32_t* __restrict__ long_list, long long long_cap, int T,
    const float* __restrict__ rank_parts, float* __restrict__ rows, const int32_t* __restrict__ row_index,
    uint8_t* __restrict__ dirty, int dim, float lr, int mode, float* __restrict__ grad_out,
    const uint32_t* __restrict__ my_ids, const int64_t* __restrict__ next_mark, long long next_tag,
    unsigned long long* __restrict__ stats) {
  const long long n_vlong = d_num_long[0], n_long = n_vlong + d_num_long[1];
  const unsigned lane = threadIdx.x & 31u;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long li = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); li < n_long; li += warps) {
    const uint32_t s = li < n_vlong ? long_list[li] : long_list[long_cap - 1 - (li - n_vlong)];
    const int32_t row = row_index ? row_index[s] : (int32_t)s;
    if (row < 0) continue;  // warp-uniform
    bool nonzero = false;
#pragma unroll
    for (int q = 0; q < DPL; ++q) {
      const int d = (int)lane + q * G;
      if (lane < (unsigned)G && d < dim) {
        float comb = 0.f;
        for (int r = 0; r < T; ++r) comb = __fadd_rn(comb, rank_parts[(li * T + r) * dim + d]);
        nonzero |= comb != 0.f;
        if (mode == BP_STUB_SGD) {
          const float v = rows[(long long)row * dim + d];
          rows[(long long)row * dim + d] = __fsub_rn(v, __fmul_rn(lr, comb));
        } else {
          grad_out[(long long)s * dim + d] = comb;
        }
      }
    }
    const bool nz = __ballot_sync(0xffffffffu, nonzero) != 0;
    if (lane == 0) {
      if (nz && dirty && mode == BP_STUB_SGD) dirty[row] = 1;
      if (stats) {
        if (next_mark && next_mark[my_ids[s]] == next_tag) atomicAdd(&stats[0], 1ull);
        if (nz) atomicAdd(&stats[1], 1ull);
      }
    }
  }
}

// np.add.at(out, idx, vals) for row blocks, sequential per index in input
// order (combine_core, reference trainer.py:92-105).  Groups over the CSR of
// a registry-mode prep whose keys are the indices.
template <int G, int DPL>
__global__ void __launch_bounds__(256) k_add_at_rows(const uint32_t* __restrict__ seg_start,
                                                     const uint32_t* __restrict__ occ_pos,
                                                     const uint64_t* __restrict__ uniq_key_s,
                                                     const long long* __restrict__ d_U, const float* __restrict__ vals,
                                                     int dim, float* __restrict__ out) {
  const long long U = *d_U;
  const int lane_g = (int)(threadIdx.x & (G - 1));
  const long long groups_total = (long long)gridDim.x * (blockDim.x / G);
  for (long long s = (long long)blockIdx.x * (blockDim.x / G) + threadIdx.x / G; s < U; s += groups_total) {
    const uint32_t a = seg_start[s], b = seg_start[s + 1];
    const long long dst = (long long)row_of(uniq_key_s[s]);
    float acc[DPL];
#pragma unroll
    for (int q = 0; q < DPL; ++q) acc[q] = 0.f;
    for (uint32_t j = a; j < b; ++j) {
      const long long src = occ_pos[j];
#pragma unroll
      for (int q = 0; q < DPL; ++q) {
        const int d = lane_g + q * G;
        if (d < dim) acc[q] = __fadd_rn(acc[q], vals[src * dim + d]);
      }
    }
#pragma unroll
    for (int q = 0; q < DPL; ++q) {
      const int d = lane_g + q * G;
      if (d < dim) out[dst * dim + d] = acc[q];
    }
  }
}

__global__ void k_sgd(const float* __restrict__ v, const float* __restrict__ g, float lr, long long n,
                      float* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __fsub_rn(v[i], __fmul_rn(lr, g[i]));
}

__global__ void k_key_rows(const uint64_t* __restrict__ keys, const long long* d_U, int32_t* __restrict__ out) {
  const long long U = *d_U;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < U; i += (long long)gridDim.x * blockDim.x)
    out[i] = (int32_t)row_of(keys[i]);
}

__global__ void k_mark_ids(const uint32_t* __restrict__ ids, const long long* __restrict__ d_U, int64_t* mark,
                           long long tag, int64_t* zero2) {
  if (zero2 && blockIdx.x == 0 && threadIdx.x < 2) zero2[threadIdx.x] = 0;  // the step's stats (no memset)
  const long long U = *d_U;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < U; i += (long long)gridDim.x * blockDim.x)
    mark[ids[i]] = tag;
}

static inline void group_shape(int dim, int* G, int* dpl) {
  int g = 1;
  while (g < dim && g < 32) g <<= 1;
  *G = g;
  *dpl = (dim + g - 1) / g;
}

}  // namespace bp

#define BP_DISPATCH_GD(G, DPL, CALL)                      \
  switch (G * 16 + DPL) {                                 \
    case 1 * 16 + 1: { constexpr int g_ = 1, d_ = 1; CALL; break; }   \
    case 2 * 16 + 1: { constexpr int g_ = 2, d_ = 1; CALL; break; }   \
    case 4 * 16 + 1: { constexpr int g_ = 4, d_ = 1; CALL; break; }   \
    case 8 * 16 + 1: { constexpr int g_ = 8, d_ = 1; CALL; break; }   \
    case 16 * 16 + 1: { constexpr int g_ = 16, d_ = 1; CALL; break; } \
    case 32 * 16 + 1: { constexpr int g_ = 32, d_ = 1; CALL; break; } \
    case 32 * 16 + 2: { constexpr int g_ = 32, d_ = 2; CALL; break; } \
    case 32 * 16 + 3: { constexpr int g_ = 32, d_ = 3; CALL; break; } \
    case 32 * 16 + 4: { constexpr int g_ = 32, d_ = 4; CALL; break; } \
    default: return BP_ERR_INVALID;                       \
  }

extern "C" int bp_mark_ids(bp_prep* P, int64_t* d_mark, int64_t tag, bp_stream_t stream) {
  return bp::mark_ids_zero(P, d_mark, tag, nullptr, (cudaStream_t)stream);
}

// bp_mark_ids that also zeroes two counters (the engine's step stats).
int bp::mark_ids_zero(bp_prep* P, int64_t* d_mark, int64_t tag, int64_t* d_zero2, cudaStream_t stream) {
  using namespace bp;
  if (!P->schema_mode) return BP_ERR_INVALID;
  if (P->n_occ == 0) {
    if (d_zero2) BP_CUDA_TRY(cudaMemsetAsync(d_zero2, 0, 2 * sizeof(int64_t), stream));
    return BP_OK;
  }
  k_mark_ids<<<grid_for(P->n_occ, 256), 256, 0, (cudaStream_t)stream>>>(P->d_uniq_id_s, P->d_num_unique, d_mark,
                                                                         tag, d_zero2);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

// Side stream of the calling thread for the long-segment kernel (created on
// first use, high priority: its chains are the trainer's critical path).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  float* parts = nullptr;  // rank partials of the long keys (grow-only; no per-step allocation)
  size_t parts_cap = 0;
  SideStream() {
    int lo = 0, hi = 0;
    cudaStream_t gs = nullptr;
    // with the host-link green partition the side stream stays out of it
    if (bp::green_link_mode() && bp::green_stream(0, 0, &gs) == BP_OK && gs) {
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      cudaStreamDestroy(gs);
      if (bp::green_stream(0, hi, &gs) == BP_OK && gs) s = gs;
    }
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess ||
        (!s && cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi) != cudaSuccess) ||
        cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&join, cudaEventDisableTiming) != cudaSuccess)
      s = nullptr;
  }
};

static SideStream& side_stream() {
  thread_local SideStream side;
  return side;
}

// 0: both kernels on the caller's stream; 1: hot-key chains on a side stream;
// 2 (default): chains on the caller's stream, launched first, and the short
// kernel on the side stream -- the chain CTAs then reach their SMs before the
// short kernel's grid fills them, instead of racing a cross-stream event
static int g_fork_long = 2;
static cudaStream_t g_long_stream = nullptr;  // engine-provided stream for the chains (green partition)
static int g_short_ctas = 5;  // tuning knob (bp_set_stub_short_ctas): short-kernel CTAs per SM
// threads of a long-segment CTA (bp_set_stub_long_threads): one warp runs the
// chain, the others stage occurrence bytes.  With the chains launched first
// (fork mode 2) 128 measured best (0.1699 vs 0.171 ms/step for 1024 over 6
// runs each, profiles/round2/stub_knobs2/)
static int g_long_threads = 128;

static int g_short_carveout = 100;  // tuning knob: shared-memory carveout (%) of the short kernel

template <int G, int DPL>
static void long_attr() {
  static int done = -1;
  if (done != bp::g_long_smem) {
    cudaFuncSetAttribute(bp::k_stub_step_long<G, DPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, bp::g_long_smem);
    // the short kernel's SMs keep the shared-memory carveout a long CTA
    // needs: with a small carveout an SM running short CTAs would have to
    // drain before it could take a long one (measured: the hot-key chains
    // then started ~25 us after the short kernel instead of beside it)
    cudaFuncSetAttribute(bp::k_stub_step<G, DPL>, cudaFuncAttributePreferredSharedMemoryCarveout, g_short_carveout);
    done = bp::g_long_smem;
  }
}

extern "C" int bp_stub_step(bp_ctx* ctx, bp_prep* P, float* d_rows, const int32_t* d_row_index, uint8_t* d_dirty,
                            int32_t dim, float c_value, float c_label, float lr, int32_t mode, float* d_grad_out,
                            const int64_t* d_next_mark, int64_t next_tag, int64_t* d_stats, bp_stream_t stream) {
  using namespace bp;
  (void)ctx;
  if (dim < 1 || dim > 128) return BP_ERR_INVALID;
  if (P->n_occ == 0) return BP_OK;
  int G, dpl;
  group_shape(dim, &G, &dpl);
  cudaStream_t s = (cudaStream_t)stream;
  const long long groups = P->n_occ;  // upper bound on U
  const int threads = 256;
  // grid: g_short_ctas CTAs per SM (grid-stride).  5 (default) of the 6 that
  // fit leave every SM room for one long-segment CTA, so the hot-key chains
  // start when they are launched instead of after the whole short kernel
  const int blocks = grid_for(groups * G, threads, kNumSMs * g_short_ctas);
  // the long-segment kernel (a few sequential hot-key chains) runs on a side
  // stream beside the short-segment kernel: the two touch disjoint keys
  cudaStream_t ls = s, ss = s;
  if (g_fork_long) {
    SideStream& side = side_stream();
    if (!side.s) return BP_ERR_CUDA;
    if (g_fork_long == 2 && !g_long_stream) ss = side.s;
    else ls = g_long_stream ? g_long_stream : side.s;
    cudaStream_t forked = ls != s ? ls : ss;
    BP_CUDA_TRY(cudaEventRecord(side.fork, s));
    BP_CUDA_TRY(cudaStreamWaitEvent(forked, side.fork, 0));
  }
  // T > 1: the long keys' rank runs are separate chains (rank partials in a
  // stream-ordered scratch), combined in rank order by k_stub_long_combine
  const int T = P->num_ranks;
  float* parts = nullptr;
  if (T > 1) {
    SideStream& side = side_stream();
    const size_t need = (size_t)P->long_cap * T * dim;
    if (need > side.parts_cap) {
      BP_CUDA_TRY(cudaDeviceSynchronize());  // the old buffer may still be read
      if (side.parts) BP_CUDA_TRY(cudaFree(side.parts));
      side.parts = nullptr;
      side.parts_cap = 0;
      BP_CUDA_TRY(cudaMalloc(&side.parts, need * sizeof(float)));
      side.parts_cap = need;
    }
    parts = side.parts;
  }
  BP_DISPATCH_GD(G, dpl,
                 (long_attr<g_, d_>(), k_stub_step_long<g_, d_><<<kLongBlocks, g_long_threads, g_long_smem, ls>>>(
                     P->d_seg_start, P->d_occ_label, P->d_num_unique, P->d_long, P->d_num_long, P->long_cap, d_rows,
                     d_row_index, d_dirty, dim, c_value, c_label, lr, mode, d_grad_out, P->d_uniq_id_s, d_next_mark,
                     next_tag, (unsigned long long*)d_stats, P->d_occ_pos, P->d_rank_bounds, T, parts)));
  if (T > 1) {
    BP_DISPATCH_GD(G, dpl,
                   (k_stub_long_combine<g_, d_><<<kNumSMs, 256, 0, ls>>>(
                       P->d_num_long, P->d_long, P->long_cap, T, parts, d_rows, d_row_index, d_dirty, dim, lr, mode,
                       d_grad_out, P->d_uniq_id_s, d_next_mark, next_tag, (unsigned long long*)d_stats)));
  }
  BP_DISPATCH_GD(G, dpl,
                 (k_stub_step<g_, d_><<<blocks, threads, 0, ss>>>(
                     P->d_seg_start, P->d_occ_label, P->d_num_unique, P->d_long, P->d_num_long, P->long_cap, d_rows,
                     d_row_index, d_dirty, dim, c_value,
                     c_label, lr, mode, d_grad_out, P->d_uniq_id_s, d_next_mark, next_tag,
                     (unsigned long long*)d_stats)));
  BP_LAUNCH_CHECK();
  if (ls != s || ss != s) {
    SideStream& side = side_stream();
    BP_CUDA_TRY(cudaEventRecord(side.join, ls != s ? ls : ss));
    BP_CUDA_TRY(cudaStreamWaitEvent(s, side.join, 0));
  }
  return BP_OK;
}

namespace bp {
void set_long_stream(cudaStream_t s) { g_long_stream = s; }
}  // namespace bp

extern "C" int bp_set_stub_long_threads(int32_t threads) {
  if (threads < 64 || threads > 1024 || (threads & 31)) return BP_ERR_INVALID;
  g_long_threads = threads;
  return BP_OK;
}

extern "C" int bp_set_stub_long_smem(int32_t bytes) {
  if (bytes < 0 || bytes > (227 << 10)) return BP_ERR_INVALID;
  bp::g_long_smem = bytes;
  return BP_OK;
}

extern "C" int bp_set_stub_carveout(int32_t percent) {
  if (percent < -1 || percent > 100) return BP_ERR_INVALID;
  g_short_carveout = percent;
  return BP_OK;
}

extern "C" int bp_set_stub_short_ctas(int32_t per_sm) {
  if (per_sm < 1 || per_sm > 6) return BP_ERR_INVALID;
  g_short_ctas = per_sm;
  return BP_OK;
}

extern "C" int bp_set_stub_fork(int32_t mode) {
  if (mode < 0 || mode > 2) return BP_ERR_INVALID;
  g_fork_long = mode;
  return BP_OK;
}

extern "C" int bp_add_at_rows(bp_prep* P, const float* d_vals, int32_t dim, float* d_out, bp_stream_t stream) {
  using namespace bp;
  if (dim < 1 || dim > 128) return BP_ERR_INVALID;
  if (P->n_occ == 0) return BP_OK;
  int G, dpl;
  group_shape(dim, &G, &dpl);
  const int blocks = grid_for(P->n_occ * G, 256, kNumSMs * 8);
  cudaStream_t s = (cudaStream_t)stream;
  BP_DISPATCH_GD(G, dpl,
                 (k_add_at_rows<g_, d_><<<blocks, 256, 0, s>>>(P->d_seg_start, P->d_occ_pos, P->d_uniq_key_s,
                                                                P->d_num_unique, d_vals, dim, d_out)));
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_prep_key_rows(bp_prep* P, int32_t* d_out, bp_stream_t stream) {
  using namespace bp;
  if (P->n_occ == 0) return BP_OK;
  k_key_rows<<<grid_for(P->n_occ, 256), 256, 0, (cudaStream_t)stream>>>(P->d_uniq_key_s, P->d_num_unique, d_out);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_sgd(const float* d_values, const float* d_grads, float lr, int64_t count, float* d_out,
                      bp_stream_t stream) {
  using namespace bp;
  if (count <= 0) return BP_OK;
  k_sgd<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(d_values, d_grads, lr, count, d_out);
  BP_LAUNCH_CHECK();
  return BP_OK;
}

extern "C" int bp_debug_long_trace(void* d_buf) {
  BP_CUDA_TRY(cudaMemcpyToSymbol(bp::g_long_trace, &d_buf, sizeof(void*)));
  return BP_OK;
}
