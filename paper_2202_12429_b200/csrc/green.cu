// SM partition of the engine with green contexts (CUDA driver API): a small
// partition of a few SMs runs either the engine's host-link streams (the
// default: the zero-copy prefetch fills its SMs' load queues with
// microsecond host reads, which slowed every kernel sharing those SMs) or
// the stub trainer's hot-key chains (measured slower, off), and every other
// engine stream lives in the complementary partition.
// Memory is the device's: green contexts partition SMs only.  The driver
// entry points are fetched through the runtime (cudaGetDriverEntryPoint), so
// the library does not link libcuda and still loads on a machine without a
// GPU driver.
#include <cuda.h>

#include "internal.cuh"

namespace bp {

struct GreenApi {
  CUresult (*ctxGetDevice)(CUdevice*);
  CUresult (*getDevResource)(CUdevice, CUdevResource*, CUdevResourceType);
  CUresult (*smSplit)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int, unsigned int);
  CUresult (*genDesc)(CUdevResourceDesc*, CUdevResource*, unsigned int);
  CUresult (*greenCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
  CUresult (*greenStream)(CUstream*, CUgreenCtx, unsigned int, int);
};

static int green_api(GreenApi* a) {
  struct {
    const char* name;
    void** fn;
  } entries[] = {{"cuCtxGetDevice", (void**)&a->ctxGetDevice},
                 {"cuDeviceGetDevResource", (void**)&a->getDevResource},
                 {"cuDevSmResourceSplitByCount", (void**)&a->smSplit},
                 {"cuDevResourceGenerateDesc", (void**)&a->genDesc},
                 {"cuGreenCtxCreate", (void**)&a->greenCreate},
                 {"cuGreenCtxStreamCreate", (void**)&a->greenStream}};
  for (auto& en : entries) {
    cudaDriverEntryPointQueryResult q;
    BP_CUDA_TRY(cudaGetDriverEntryPoint(en.name, en.fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !*en.fn) {
      bp_set_last_error(en.name, __FILE__, __LINE__);
      return BP_ERR_CUDA;
    }
  }
  return BP_OK;
}

struct GreenPartition {
  CUgreenCtx hot = nullptr, rest = nullptr;
  int hot_sms = 0, rest_sms = 0;
};

static GreenPartition g_green;
// bp_set_green_sms: SMs requested for the small partition (0 = off); the
// driver rounds a request up to its split granularity -- on B200 8 SMs
// (bp_green_info reports the partition made).  Used for the engine's
// host-link streams (bp_set_green_link), measured on the CK step with the
// planner thread (8 SMs): value 99.0-100.6M vs 89.3-97.1M samples/s, e2e
// 92.5-95.3M vs 82.0-89.8M (profiles/round2/green_link_threaded/).
// -1 (default) = auto at the first engine: 8 SMs per 32 row components (the
// host-link bytes per row), at most 16 -- CK / Avazu (D=16) 8 SMs, Terabyte
// (D=64) 16 (measured there: 71.1M samples/s with 16 SMs, 63.2M with 8,
// 64.9M unpartitioned; profiles/round2/green_link_tb10/)
static int g_green_sms = -1;
// bp_set_green_link: 1 = the small partition runs the host-link streams
// (zero-copy prefetch, write-back) instead of the hot-key chains, so the
// SMs whose load queues fill with microsecond host reads run nothing else
static int g_green_link = 1;

#define BP_CU_TRY(expr)                                        \
  do {                                                         \
    CUresult _r = (expr);                                      \
    if (_r != CUDA_SUCCESS) {                                  \
      bp_set_last_error("CUDA driver call failed", __FILE__, __LINE__); \
      return BP_ERR_CUDA;                                      \
    }                                                          \
  } while (0)

static GreenApi g_api;

// Creates the partition once per process (green contexts are per device).
static int green_init() {
  if (g_green.hot || g_green_sms <= 0) return BP_OK;
  BP_CUDA_TRY(cudaFree(nullptr));  // the runtime's primary context exists
  const int rc = green_api(&g_api);
  if (rc) return rc;
  CUdevice dev;
  BP_CU_TRY(g_api.ctxGetDevice(&dev));
  CUdevResource all;
  BP_CU_TRY(g_api.getDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  CUdevResource hot, rest;
  unsigned int n = 1;
  BP_CU_TRY(g_api.smSplit(&hot, &n, &all, &rest, 0, (unsigned)g_green_sms));
  CUdevResourceDesc dh, dr;
  BP_CU_TRY(g_api.genDesc(&dh, &hot, 1));
  BP_CU_TRY(g_api.genDesc(&dr, &rest, 1));
  BP_CU_TRY(g_api.greenCreate(&g_green.hot, dh, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  BP_CU_TRY(g_api.greenCreate(&g_green.rest, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  g_green.hot_sms = (int)hot.sm.smCount;
  g_green.rest_sms = (int)rest.sm.smCount;
  return BP_OK;
}

// A non-blocking stream of the hot (hot != 0) or rest partition; nullptr out
// when partitioning is off.
int green_stream(int hot, int priority, cudaStream_t* out) {
  *out = nullptr;
  if (green_init() != BP_OK || !g_green.rest) {
    // the partition is a performance feature: without green-context support
    // the engine runs unpartitioned
    g_green = GreenPartition{};
    g_green_sms = 0;
    return BP_OK;
  }
  CUstream s;
  BP_CU_TRY(g_api.greenStream(&s, hot ? g_green.hot : g_green.rest, CU_STREAM_NON_BLOCKING, priority));
  *out = (cudaStream_t)s;
  return BP_OK;
}

bool green_link_mode() { return g_green_link != 0; }

void green_auto(int dim) {
  if (g_green_sms < 0) {
    const int s = 8 * ((dim + 31) / 32);
    g_green_sms = s < 8 ? 8 : (s > 16 ? 16 : s);
  }
}

}  // namespace bp

extern "C" int bp_set_green_link(int32_t on) {
  bp::g_green_link = on != 0;
  return BP_OK;
}

// Tuning: SMs of the small partition (0 = off; -1 = auto by the row width,
// the default).  Takes effect for engines created afterwards (the partition
// is made once per process).
extern "C" int bp_set_green_sms(int32_t sms) {
  if (sms < -1) return BP_ERR_INVALID;
  bp::g_green_sms = sms;
  return BP_OK;
}

// {hot SMs, rest SMs} of the partition in use (0, 0 when off).
extern "C" int bp_green_info(int32_t* out2) {
  out2[0] = bp::g_green.hot_sms;
  out2[1] = bp::g_green.rest_sms;
  return BP_OK;
}
