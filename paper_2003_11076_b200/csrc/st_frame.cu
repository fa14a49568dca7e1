// One frame of the reference pipeline's compute stages in one call
// (pipeline.py:247-261: DisparitySolver(...).solve() + synthesize(...)), for
// the host runtime of reconstruct_stream: the whole frame is enqueued with no
// host synchronisation and no per-stage Python, so one host thread keeps the
// GPU fed while the next frame's inputs are prepared.
//
//   side  stream : st_mu_raster (Qhull-walk replay, a long pointer chase)
//   side2 stream : st_descriptors, st_support_build
//   main  stream : st_solve_async, st_synthesize
//   out   stream : D2H of the artefacts into one pinned block
#include <cuda_runtime.h>
#include <stdint.h>

#include "st_common.cuh"

namespace {

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

extern "C" {

int st_frame_plan_init(st_frame_plan* plan) {
  if (!plan) {
    sthost::set_error("st_frame_plan_init: null plan");
    return ST_EINVAL;
  }
  for (int i = 0; i < 4; ++i) {
    if (plan->events[i]) continue;
    cudaEvent_t e;
    ST_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    plan->events[i] = (void*)e;
  }
  return ST_OK;
}

int st_frame_plan_destroy(st_frame_plan* plan) {
  if (!plan) return ST_OK;
  for (int i = 0; i < 4; ++i) {
    if (plan->events[i]) cudaEventDestroy((cudaEvent_t)plan->events[i]);
    plan->events[i] = nullptr;
  }
  return ST_OK;
}

int64_t st_frame_host_bytes(int32_t W, int32_t H) {
  const size_t n = (size_t)W * H;
  return (int64_t)(align256(n * 4) + align256(n) + align256(n * 4) + align256(n * 4) +
                   align256(n * 3) + align256(n) + align256(n) + align256(sizeof(st_stats)));
}

int st_frame_run(st_frame_plan* P, const st_tri* tri, const double* support_uv,
                 const double* support_d, int32_t n_support, void* ready, void* host_block,
                 void* done) {
  if (!P || !P->events[0] || !tri) {
    sthost::set_error("st_frame_run: plan not initialised (st_frame_plan_init)");
    return ST_EINVAL;
  }
  cudaStream_t m = (cudaStream_t)P->main_stream;
  cudaStream_t s1 = (cudaStream_t)P->side_stream;
  cudaStream_t s2 = (cudaStream_t)P->side2_stream;
  cudaStream_t so = (cudaStream_t)P->out_stream;
  cudaEvent_t* ev = (cudaEvent_t*)P->events;
  const int W = P->rig.width, H = P->rig.height, K = P->rig.num_views;
  if (st_mu_raster_workspace(W, H, tri->n_tri) > P->mu_ws_bytes ||
      st_support_workspace(n_support, W, H, P->params.neighborhood_radius) > P->sup_ws_bytes) {
    sthost::set_error("st_frame_run: workspace too small for this triangulation");
    return ST_ENOMEM;
  }
  cudaEvent_t r = (cudaEvent_t)ready;
  if (!r) {
    ST_CUDA_CHECK(cudaEventRecord(ev[0], m));
    r = ev[0];
  }
  int rc;
  // surface raster (side)
  ST_CUDA_CHECK(cudaStreamWaitEvent(s1, r, 0));
  if ((rc = st_mu_raster(tri, W, H, P->params.d_max, (double*)P->frame.mu, P->mu_ws,
                         P->mu_ws_bytes, s1)))
    return rc;
  ST_CUDA_CHECK(cudaEventRecord(ev[1], s1));
  // descriptors + support candidate groups (side2)
  ST_CUDA_CHECK(cudaStreamWaitEvent(s2, r, 0));
  if (P->descriptors_ready) {
    ST_CUDA_CHECK(cudaEventRecord(ev[2], m));  // written on the main stream
    ST_CUDA_CHECK(cudaStreamWaitEvent(s2, ev[2], 0));
  } else if ((rc = st_descriptors(P->frame.images, K, H, W, 3, (uint8_t*)P->frame.desc, nullptr,
                                  nullptr, s2))) {
    return rc;
  }
  P->descriptors_ready = 0;
  if ((rc = st_support_build(support_uv, support_d, n_support, W, H, &P->params, &P->frame,
                             P->sup_ws, P->sup_ws_bytes, nullptr, s2)))
    return rc;
  ST_CUDA_CHECK(cudaEventRecord(ev[2], s2));
  // EM + refocus (main)
  ST_CUDA_CHECK(cudaStreamWaitEvent(m, ev[2], 0));
  ST_CUDA_CHECK(cudaStreamWaitEvent(m, ev[1], 0));
  if ((rc = st_solve_async(&P->frame, &P->rig, &P->params, P->values, P->status, P->static_bits,
                           P->valid_bits, P->stats_dev, P->solve_ws, P->solve_ws_bytes, m)))
    return rc;
  if ((rc = st_synthesize(P->frame.images, &P->rig, P->values, P->status, P->static_bits,
                          P->params.min_static_rays, P->median_radius, nullptr, P->image,
                          P->prov, P->n_rays, P->scratch, m)))
    return rc;
  // artefacts to the host
  if (host_block) {  // (a null out stream is the legacy default stream)
    ST_CUDA_CHECK(cudaEventRecord(ev[3], m));
    ST_CUDA_CHECK(cudaStreamWaitEvent(so, ev[3], 0));
    const size_t n = (size_t)W * H;
    const void* src[8] = {P->values, P->status, P->static_bits, P->valid_bits,
                          P->image, P->prov, P->n_rays, P->stats_dev};
    const size_t bytes[8] = {n * 4, n, n * 4, n * 4, n * 3, n, n, sizeof(st_stats)};
    char* dst = (char*)host_block;
    for (int i = 0; i < 8; ++i) {
      ST_CUDA_CHECK(cudaMemcpyAsync(dst, src[i], bytes[i], cudaMemcpyDeviceToHost, so));
      dst += align256(bytes[i]);
    }
    if (done) ST_CUDA_CHECK(cudaEventRecord((cudaEvent_t)done, so));
  } else if (done) {
    ST_CUDA_CHECK(cudaEventRecord((cudaEvent_t)done, m));
  }
  return ST_OK;
}

}  // extern "C"
