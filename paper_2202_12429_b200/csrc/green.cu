// Optional SM partition of the engine with green contexts (CUDA driver API):
// a "hot" partition of a few SMs runs the stub trainer's hot-key chains
// (k_stub_step_long, sequential per-key f32 adds) and every other engine
// stream lives in the complementary partition, so the chains never share an
// SM with the short-segment kernel (measured in the step: the two kernels
// slowed each other from 47 + 25 us isolated to ~55 us side by side).
// Memory is the device's: green contexts partition SMs only.
#include <cuda.h>

#include "internal.cuh"

namespace bp {

struct GreenPartition {
  CUgreenCtx hot = nullptr, rest = nullptr;
  int hot_sms = 0, rest_sms = 0;
};

static GreenPartition g_green;
static int g_green_sms = 0;  // bp_set_green_sms: SMs of the hot partition (0 = off)

#define BP_CU_TRY(expr)                                               \
  do {                                                                \
    CUresult _r = (expr);                                             \
    if (_r != CUDA_SUCCESS) {                                         \
      const char* _m = nullptr;                                       \
      cuGetErrorString(_r, &_m);                                      \
      bp_set_last_error(_m ? _m : "driver error", __FILE__, __LINE__); \
      return BP_ERR_CUDA;                                             \
    }                                                                 \
  } while (0)

// Creates the partition once per process (green contexts are per device).
static int green_init() {
  if (g_green.hot || g_green_sms <= 0) return BP_OK;
  BP_CUDA_TRY(cudaFree(nullptr));  // the runtime's primary context exists
  CUdevice dev;
  BP_CU_TRY(cuCtxGetDevice(&dev));
  CUdevResource all;
  BP_CU_TRY(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  CUdevResource hot, rest;
  unsigned int n = 1;
  BP_CU_TRY(cuDevSmResourceSplitByCount(&hot, &n, &all, &rest, 0, (unsigned)g_green_sms));
  CUdevResourceDesc dh, dr;
  BP_CU_TRY(cuDevResourceGenerateDesc(&dh, &hot, 1));
  BP_CU_TRY(cuDevResourceGenerateDesc(&dr, &rest, 1));
  BP_CU_TRY(cuGreenCtxCreate(&g_green.hot, dh, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  BP_CU_TRY(cuGreenCtxCreate(&g_green.rest, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  g_green.hot_sms = (int)hot.sm.smCount;
  g_green.rest_sms = (int)rest.sm.smCount;
  return BP_OK;
}

// A non-blocking stream of the hot (hot != 0) or rest partition; nullptr out
// when partitioning is off.
int green_stream(int hot, int priority, cudaStream_t* out) {
  *out = nullptr;
  const int rc = green_init();
  if (rc || !g_green.hot) return rc;
  CUstream s;
  BP_CU_TRY(cuGreenCtxStreamCreate(&s, hot ? g_green.hot : g_green.rest, CU_STREAM_NON_BLOCKING, priority));
  *out = (cudaStream_t)s;
  return BP_OK;
}

}  // namespace bp

// Tuning: SMs of the hot-key partition (0 = off, the default; on B200 a
// multiple of 8).  Takes effect for engines created afterwards.
extern "C" int bp_set_green_sms(int32_t sms) {
  if (sms < 0) return BP_ERR_INVALID;
  bp::g_green_sms = sms;
  return BP_OK;
}

// {hot SMs, rest SMs} of the partition in use (0, 0 when off).
extern "C" int bp_green_info(int32_t* out2) {
  out2[0] = bp::g_green.hot_sms;
  out2[1] = bp::g_green.rest_sms;
  return BP_OK;
}
