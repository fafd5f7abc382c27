// NVLink peer-memory exchange for DLRM hybrid parallelism.
//
// Instead of an NCCL all-to-all after the EmbeddingBag forward and another
// before its backward, the kernels themselves move the rows over NVLink:
//
//   forward   the table owner's EmbeddingBag forward stores each pooled row
//             straight into the example owner's [bl][T][D] input buffer,
//             at its global-table column (no send buffer, no reorder);
//   backward  the table owner's reduce-by-key backward loads each gradient
//             row straight from the example owner's [bl][T][D] gradient
//             buffer (peer loads, 8 rows per lane in flight).
//
// Buffers are plain cudaMalloc allocations shared with CUDA IPC handles
// (exchanged by the host over torch.distributed).  A flag barrier orders the
// phases: every rank stores its epoch into every peer's flag array after a
// system-scope fence and spins (bounded, with an error instead of a hang) on
// its own array.  Two barriers per iteration (rows ready, gradients ready)
// also protect buffer reuse across iterations.
#include <cstring>

#include "internal.cuh"

namespace bp {

__global__ void k_peer_barrier(uint32_t* const* __restrict__ peer_flags, uint32_t* my_flags, int rank, int world,
                               uint32_t epoch, ErrorRecord* err) {
  if (threadIdx.x != 0) return;
  __threadfence_system();  // this stream's earlier peer stores before the flag
  for (int q = 0; q < world; ++q) {
    volatile uint32_t* f = peer_flags[q];
    f[rank] = epoch;
  }
  __threadfence_system();
  for (int q = 0; q < world; ++q) {
    volatile uint32_t* f = my_flags;
    long long spins = 0;
    while ((int)(f[q] - epoch) < 0) {
      __nanosleep(128);
      if (++spins > (1ll << 25)) {  // ~5 s: a peer never arrived
        raise_error(err, BP_ERR_ENGINE, (long long)epoch, q, 0);
        return;
      }
    }
  }
  __threadfence_system();
}

}  // namespace bp

extern "C" int bp_ipc_alloc(int64_t bytes, void** d_ptr, uint8_t* handle) {
  if (bytes <= 0) return BP_ERR_INVALID;
  BP_CUDA_TRY(cudaMalloc(d_ptr, (size_t)bytes));
  BP_CUDA_TRY(cudaMemset(*d_ptr, 0, (size_t)bytes));
  cudaIpcMemHandle_t h;
  BP_CUDA_TRY(cudaIpcGetMemHandle(&h, *d_ptr));
  static_assert(sizeof(cudaIpcMemHandle_t) == BP_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof(h));
  return BP_OK;
}

extern "C" int bp_ipc_open(const uint8_t* handle, void** d_ptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  BP_CUDA_TRY(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return BP_OK;
}

extern "C" int bp_ipc_close(void* d_ptr) {
  BP_CUDA_TRY(cudaIpcCloseMemHandle(d_ptr));
  return BP_OK;
}

extern "C" int bp_ipc_free(void* d_ptr) {
  BP_CUDA_TRY(cudaFree(d_ptr));
  return BP_OK;
}

extern "C" int bp_peer_barrier(bp_ctx* ctx, const bp_peer_xchg* x, uint32_t epoch, bp_stream_t stream) {
  using namespace bp;
  if (!x || x->world < 1 || x->rank < 0 || x->rank >= x->world) return BP_ERR_INVALID;
  k_peer_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(x->d_peer_flags, x->d_flags, x->rank, x->world, epoch,
                                                    ctx ? ctx->d_err : nullptr);
  BP_LAUNCH_CHECK();
  return BP_OK;
}
