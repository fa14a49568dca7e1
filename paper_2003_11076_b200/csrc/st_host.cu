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

extern "C" {

// L2 residency control (B200: 126 MB L2): reserve `bytes` of L2 for
// persisting accesses (0 = release) -- device-wide, cudaLimitPersistingL2CacheSize.
int st_l2_set_aside(int64_t bytes) {
  int dev = 0;
  ST_CUDA_CHECK(cudaGetDevice(&dev));
  int max_persist = 0;
  ST_CUDA_CHECK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
  size_t b = (size_t)(bytes < 0 ? 0 : bytes);
  if (b > (size_t)max_persist) b = (size_t)max_persist;
  ST_CUDA_CHECK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, b));
  return ST_OK;
}

// Kernels launched on `stream` treat [base, base + bytes) as persisting in L2
// (hit_ratio of its lines; the rest streaming); bytes = 0 clears the window.
int st_stream_l2_window(void* stream, void* base, int64_t bytes, float hit_ratio) {
  cudaStreamAttrValue attr = {};
  attr.accessPolicyWindow.base_ptr = base;
  attr.accessPolicyWindow.num_bytes = (size_t)(bytes < 0 ? 0 : bytes);
  attr.accessPolicyWindow.hitRatio = hit_ratio;
  attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  ST_CUDA_CHECK(cudaStreamSetAttribute((cudaStream_t)stream, cudaStreamAttributeAccessPolicyWindow,
                                       &attr));
  return ST_OK;
}

}  // extern "C"
