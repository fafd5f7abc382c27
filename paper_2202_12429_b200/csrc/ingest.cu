// EMTRC1 binary trace ingest on the device (reference
// traces.py:231-296).  A trace is a header followed by packed records
// "<B{num_dense}f{num_tables}Q" (label byte, dense floats, one row id per
// table, no padding: a Criteo-Kaggle record is 261 bytes, so no field is
// aligned).  The host streams the record bytes from the file into pinned
// chunks and copies them to HBM; this kernel turns a chunk into the engine's
// device batch layout in one pass:
//   keys[e * T + t]       = (t << 44) | row     (occurrence order: the engine's packed keys)
//   occ_labels[e * T + t] = label               (one label byte per occurrence)
//   labels[e], dense[e * D + d]                 (the DLRM inputs)
// One thread per 8-byte row field (its bytes are read individually and
// assembled: the field is unaligned), consecutive threads reading consecutive
// bytes of the same records -- the loads coalesce into whole sectors.
#include "internal.cuh"

namespace bp {

__global__ void k_trace_decode(const uint8_t* __restrict__ rec, long long n, int num_dense, int num_tables,
                               uint64_t* __restrict__ keys, uint8_t* __restrict__ occ_labels,
                               uint8_t* __restrict__ labels, float* __restrict__ dense) {
  const int rb = 1 + 4 * num_dense + 8 * num_tables;
  const long long n_keys = n * num_tables;
  const long long n_dense = n * num_dense;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_keys; i += stride) {
    const long long e = i / num_tables;
    const int t = (int)(i - e * num_tables);
    const uint8_t* r = rec + e * rb;
    const uint8_t* f = r + 1 + 4 * num_dense + 8 * t;
    uint64_t row = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) row |= (uint64_t)f[b] << (8 * b);
    keys[i] = ((uint64_t)t << kKeyTableShift) | (row & kRowMask);
    const uint8_t lab = r[0];
    occ_labels[i] = lab;
    if (t == 0 && labels) labels[e] = lab;
  }
  if (!dense) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_dense; i += stride) {
    const long long e = i / num_dense;
    const int d = (int)(i - e * num_dense);
    const uint8_t* f = rec + e * rb + 1 + 4 * d;
    const uint32_t w = (uint32_t)f[0] | ((uint32_t)f[1] << 8) | ((uint32_t)f[2] << 16) | ((uint32_t)f[3] << 24);
    dense[i] = __uint_as_float(w);
  }
}

}  // namespace bp

extern "C" int bp_trace_decode(const uint8_t* d_records, int64_t n, int32_t num_dense, int32_t num_tables,
                               uint64_t* d_keys, uint8_t* d_occ_labels, uint8_t* d_labels, float* d_dense,
                               bp_stream_t stream) {
  using namespace bp;
  if (n < 0 || num_dense < 0 || num_tables < 1) return BP_ERR_INVALID;
  if (n == 0) return BP_OK;
  const long long work = n * (long long)(num_tables > num_dense ? num_tables : num_dense);
  k_trace_decode<<<grid_for(work, 256), 256, 0, (cudaStream_t)stream>>>(d_records, n, num_dense, num_tables, d_keys,
                                                                       d_occ_labels, d_labels, d_dense);
  BP_LAUNCH_CHECK();
  return BP_OK;
}
