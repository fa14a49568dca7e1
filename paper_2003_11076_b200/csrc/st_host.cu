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

// ---------------------------------------------------------------------------
// Clock sampler for the benchmark's timed regions: a native thread polling
// NVML (dlopen'd, no link dependency) for the SM clock and the clock-event
// (throttle) reasons, so sampling never competes with the enqueueing Python
// thread for the GIL.

#include <dlfcn.h>

#include <atomic>
#include <chrono>
#include <mutex>
#include <thread>
#include <vector>

namespace {

typedef int (*NvmlInit)(void);
typedef int (*NvmlByPci)(const char*, void**);
typedef int (*NvmlClock)(void*, int, unsigned int*);
typedef int (*NvmlReasons)(void*, unsigned long long*);

struct ClockSampler {
  std::thread th;
  std::atomic<bool> stop{false};
  std::mutex mu;
  std::vector<unsigned> sm, mx;
  std::vector<unsigned long long> reasons;
  bool running = false;
};

ClockSampler& sampler() {
  static ClockSampler s;
  return s;
}

}  // namespace

extern "C" {

// Start sampling every interval_us on the current CUDA device.  0 = started,
// ST_EINVAL when NVML is unavailable.
int st_clocks_start(int32_t interval_us) {
  ClockSampler& S = sampler();
  if (S.running) {
    sthost::set_error("st_clocks_start: already running");
    return ST_EINVAL;
  }
  void* h = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    sthost::set_error("st_clocks_start: libnvidia-ml.so.1 not found");
    return ST_EINVAL;
  }
  auto init = (NvmlInit)dlsym(h, "nvmlInit_v2");
  auto by_pci = (NvmlByPci)dlsym(h, "nvmlDeviceGetHandleByPciBusId_v2");
  auto clock = (NvmlClock)dlsym(h, "nvmlDeviceGetClockInfo");
  auto maxclock = (NvmlClock)dlsym(h, "nvmlDeviceGetMaxClockInfo");
  auto reasons = (NvmlReasons)dlsym(h, "nvmlDeviceGetCurrentClocksEventReasons");
  if (!reasons) reasons = (NvmlReasons)dlsym(h, "nvmlDeviceGetCurrentClocksThrottleReasons");
  int dev = 0;
  char bus[64] = {0};
  void* nd = nullptr;
  if (!init || !by_pci || !clock || !maxclock || !reasons || init() != 0 ||
      cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetPCIBusId(bus, sizeof(bus), dev) != cudaSuccess ||
      by_pci(bus, &nd) != 0) {
    sthost::set_error("st_clocks_start: NVML initialisation failed");
    return ST_EINVAL;
  }
  {
    std::lock_guard<std::mutex> lock(S.mu);
    S.sm.clear();
    S.mx.clear();
    S.reasons.clear();
  }
  S.stop = false;
  S.running = true;
  const int us = interval_us > 0 ? interval_us : 2000;
  auto sample = [&S, nd, clock, maxclock, reasons]() {
    unsigned a = 0, b = 0;
    unsigned long long r = 0;
    if (clock(nd, 1 /* NVML_CLOCK_SM */, &a) == 0 && maxclock(nd, 1, &b) == 0 &&
        reasons(nd, &r) == 0) {
      std::lock_guard<std::mutex> lock(S.mu);
      S.sm.push_back(a);
      S.mx.push_back(b);
      S.reasons.push_back(r);
    }
  };
  sample();
  S.th = std::thread([&S, us, sample]() {
    while (!S.stop.load()) {
      std::this_thread::sleep_for(std::chrono::microseconds(us));
      sample();
    }
    sample();
  });
  return ST_OK;
}

// Stop; copy up to cap samples (SM MHz, max SM MHz, reason bits) and return
// how many were taken (< 0: not running).
int64_t st_clocks_stop(uint32_t* sm_mhz, uint32_t* max_mhz, uint64_t* reason_bits,
                       int64_t cap) {
  ClockSampler& S = sampler();
  if (!S.running) return -1;
  S.stop = true;
  S.th.join();
  S.running = false;
  std::lock_guard<std::mutex> lock(S.mu);
  const int64_t n = (int64_t)S.sm.size();
  for (int64_t i = 0; i < n && i < cap; ++i) {
    sm_mhz[i] = S.sm[i];
    max_mhz[i] = S.mx[i];
    reason_bits[i] = S.reasons[i];
  }
  return n;
}

}  // extern "C"
