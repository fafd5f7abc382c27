// Host-link interference microbenchmark (tools/mb): how much does concurrent
// host-link traffic slow an HBM-bound victim kernel, by link mechanism?
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/interfere tools/mb/interfere.cu -lcuda
//   /tmp/interfere
//
// victims (stream A, high priority): random 64 B row gather from a 64 MB
// device table (latency-bound, like the cache lookups), and a 256 MB
// streaming copy (bandwidth-bound).
// aggressors (stream B, looping for the victim's duration): zero-copy random
// 64 B row gather from a 2 GB pinned host table (blocks x threads x ILP),
// zero-copy scatter, a bulk copy-engine H2D memcpy.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__global__ void k_gather(const float4* __restrict__ tab, const uint32_t* __restrict__ ids, long long n, float4* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n * 4; i += (long long)gridDim.x * blockDim.x)
    out[i] = tab[(long long)ids[i >> 2] * 4 + (i & 3)];
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <int ILP>
__global__ void k_zc_gather(const float4* __restrict__ host, const uint32_t* __restrict__ ids, long long n,
                            float4* __restrict__ out, volatile int* stop) {
  const long long total = n * 4, stride = (long long)gridDim.x * blockDim.x;
  do {
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total; i0 += stride * ILP) {
      float4 v[ILP];
#pragma unroll
      for (int r = 0; r < ILP; ++r) {
        const long long i = i0 + r * stride;
        if (i < total) v[r] = __ldcs(host + (long long)ids[i >> 2] * 4 + (i & 3));
      }
#pragma unroll
      for (int r = 0; r < ILP; ++r) {
        const long long i = i0 + r * stride;
        if (i < total) out[i] = v[r];
      }
    }
  } while (!*stop);
}

__global__ void k_zc_scatter(float4* __restrict__ host, const uint32_t* __restrict__ ids, long long n,
                             const float4* __restrict__ src, volatile int* stop) {
  const long long total = n * 4, stride = (long long)gridDim.x * blockDim.x;
  do {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += stride)
      __stcs(host + (long long)ids[i >> 2] * 4 + (i & 3), src[i]);
  } while (!*stop);
}

static float time_victim(int which, cudaStream_t s, const float4* tab, const uint32_t* ids, long long n, float4* out,
                         const float4* big_a, float4* big_b, long long big_n) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, s));
  for (int r = 0; r < 10; ++r) {
    if (which == 0) k_gather<<<148 * 8, 256, 0, s>>>(tab, ids, n, out);
    else k_copy<<<148 * 8, 256, 0, s>>>(big_a, big_b, big_n);
  }
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms * 100.f;  // us per victim launch
}

int main() {
  CK(cudaSetDevice(0));
  int lo, hi;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  cudaStream_t sa, sb;
  CK(cudaStreamCreateWithPriority(&sa, cudaStreamNonBlocking, hi));
  CK(cudaStreamCreateWithPriority(&sb, cudaStreamNonBlocking, lo));
  const long long tab_rows = 1 << 20, n = 400000;
  float4 *tab, *out, *big_a, *big_b, *zc_out, *zc_src;
  uint32_t *ids, *hids;
  const long long big_n = (256ll << 20) / 16;
  CK(cudaMalloc(&tab, tab_rows * 64));
  CK(cudaMalloc(&out, n * 64));
  CK(cudaMalloc(&big_a, big_n * 16));
  CK(cudaMalloc(&big_b, big_n * 16));
  CK(cudaMemset(big_a, 1, big_n * 16));
  CK(cudaMalloc(&ids, n * 4));
  const long long host_rows = (2ll << 30) / 64, zn = 35000;
  CK(cudaMalloc(&hids, zn * 4));
  CK(cudaMalloc(&zc_out, zn * 64));
  CK(cudaMalloc(&zc_src, zn * 64));
  std::vector<uint32_t> h(n), hz(zn);
  srand(1);
  for (auto& x : h) x = (uint32_t)(((long long)rand() * 7919) % tab_rows);
  for (auto& x : hz) x = (uint32_t)(((long long)rand() * 104729 + rand()) % host_rows);
  CK(cudaMemcpy(ids, h.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(hids, hz.data(), zn * 4, cudaMemcpyHostToDevice));
  float4* host;
  CK(cudaHostAlloc((void**)&host, host_rows * 64, cudaHostAllocMapped));
  memset(host, 0, 1 << 20);
  float4* dhost;
  CK(cudaHostGetDevicePointer((void**)&dhost, host, 0));
  int* stop;
  CK(cudaHostAlloc((void**)&stop, 4, cudaHostAllocMapped));
  int* dstop;
  CK(cudaHostGetDevicePointer((void**)&dstop, stop, 0));
  float4* hbuf;
  CK(cudaHostAlloc((void**)&hbuf, 64 << 20, 0));
  float4* dbuf;
  CK(cudaMalloc(&dbuf, 64 << 20));
  const char* vname[2] = {"gather64B", "copy256MB"};
  for (int v = 0; v < 2; ++v) {
    time_victim(v, sa, tab, ids, n, out, big_a, big_b, big_n);
    const float base = time_victim(v, sa, tab, ids, n, out, big_a, big_b, big_n);
    printf("{\"victim\": \"%s\", \"aggressor\": \"none\", \"us\": %.2f}\n", vname[v], base);
    struct Cfg { int kind, blocks, threads, ilp; };
    const Cfg cfgs[] = {{0, 32, 256, 4}, {0, 8, 256, 4}, {0, 4, 256, 4}, {0, 2, 256, 4}, {0, 1, 256, 4},
                        {0, 8, 1024, 1}, {0, 16, 128, 1}, {1, 32, 256, 1}, {1, 4, 256, 1}, {2, 0, 0, 0}};
    for (const Cfg& c : cfgs) {
      *stop = 0;
      cudaEvent_t ea, eb;
      CK(cudaEventCreate(&ea));
      CK(cudaEventCreate(&eb));
      CK(cudaEventRecord(ea, sb));
      int iters = 0;
      if (c.kind == 0) {
        if (c.ilp == 4) k_zc_gather<4><<<c.blocks, c.threads, 0, sb>>>(dhost, hids, zn, zc_out, dstop);
        else k_zc_gather<1><<<c.blocks, c.threads, 0, sb>>>(dhost, hids, zn, zc_out, dstop);
      } else if (c.kind == 1) {
        k_zc_scatter<<<c.blocks, c.threads, 0, sb>>>(dhost, hids, zn, zc_src, dstop);
      } else if (c.kind == 2) {
        for (int r = 0; r < 40; ++r) CK(cudaMemcpyAsync(dbuf, hbuf, 64 << 20, cudaMemcpyHostToDevice, sb));
        iters = 40;
      }
      CK(cudaEventRecord(eb, sb));
      // let the aggressor ramp up
      CK(cudaStreamSynchronize(sa));
      const float t = time_victim(v, sa, tab, ids, n, out, big_a, big_b, big_n);
      *stop = 1;
      CK(cudaStreamSynchronize(sb));
      float agg_ms;
      CK(cudaEventElapsedTime(&agg_ms, ea, eb));
      const char* kn[3] = {"zc_gather", "zc_scatter", "ce_bulk_h2d_64MB"};
      double gbs = 0;
      if (c.kind == 2) gbs = 40.0 * (64 << 20) / (agg_ms * 1e-3) / 1e9;
      printf("{\"victim\": \"%s\", \"aggressor\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ilp\": %d, \"us\": %.2f, "
             "\"slowdown\": %.2f, \"aggressor_gbs\": %.2f}\n",
             vname[v], kn[c.kind], c.blocks, c.threads, c.ilp, t, t / base, gbs);
      fflush(stdout);
    }
  }
  // zero-copy gather rates alone (one pass, per config)
  for (int blocks : {1, 2, 4, 8, 32}) {
    *stop = 1;
    cudaEvent_t ea, eb;
    CK(cudaEventCreate(&ea));
    CK(cudaEventCreate(&eb));
    k_zc_gather<4><<<blocks, 256, 0, sb>>>(dhost, hids, zn, zc_out, dstop);
    CK(cudaEventRecord(ea, sb));
    for (int r = 0; r < 5; ++r) k_zc_gather<4><<<blocks, 256, 0, sb>>>(dhost, hids, zn, zc_out, dstop);
    CK(cudaEventRecord(eb, sb));
    CK(cudaEventSynchronize(eb));
    float ms;
    CK(cudaEventElapsedTime(&ms, ea, eb));
    printf("{\"zc_gather_alone\": {\"blocks\": %d, \"us\": %.1f, \"gbs\": %.2f}}\n", blocks, ms * 200.f,
           5.0 * zn * 64 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
