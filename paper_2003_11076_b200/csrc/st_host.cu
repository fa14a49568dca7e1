// Host-side helpers of the streaming runtime (reconstruct_stream): one C call
// per frame for the copies that would otherwise be many Python-level calls,
// made through ctypes, which releases the GIL for their duration -- the
// stream's two host threads then overlap instead of taking turns.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "st_common.cuh"

extern "C" {

// dst + dst_off[i] <- srcs[i] (sizes[i] bytes), host memory to host memory
// (the pinned staging block of a frame's triangulation tables).
int st_host_gather(void* dst, const void* const* srcs, const int64_t* dst_off,
                   const int64_t* sizes, int32_t n) {
  if (!dst || (n > 0 && (!srcs || !dst_off || !sizes))) {
    sthost::set_error("st_host_gather: null argument");
    return ST_EINVAL;
  }
  for (int32_t i = 0; i < n; ++i)
    if (sizes[i] > 0) memcpy((char*)dst + dst_off[i], srcs[i], (size_t)sizes[i]);
  return ST_OK;
}

// dst_dev + dst_off[i] <- srcs[i] (sizes[i] bytes, host; pinned sources copy
// by DMA), each an asynchronous copy on `stream` (one call per frame for a
// frame's K views and K priors).
int st_h2d_gather(void* dst_dev, const void* const* srcs, const int64_t* dst_off,
                  const int64_t* sizes, int32_t n, void* stream) {
  if (!dst_dev || (n > 0 && (!srcs || !dst_off || !sizes))) {
    sthost::set_error("st_h2d_gather: null argument");
    return ST_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  for (int32_t i = 0; i < n; ++i)
    if (sizes[i] > 0)
      ST_CUDA_CHECK(cudaMemcpyAsync((char*)dst_dev + dst_off[i], srcs[i], (size_t)sizes[i],
                                    cudaMemcpyHostToDevice, s));
  return ST_OK;
}

}  // extern "C"
