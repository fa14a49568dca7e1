// np.mean of the finite values of a float64 array, bit for bit, as a C-ABI
// entry point (solver.py:466 `finite.mean()`): the same kernel the EM
// statistics use (k_em_stats, numpy's pairwise summation order, st_pw.cuh),
// run over one array with its record written to the workspace.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "st_common.cuh"
#include "st_em.cuh"

namespace st {

__global__ void k_finish_mean(const Partial* __restrict__ rec, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    *out = rec->n_fin > 0 ? ddiv(rec->sum_e, (double)rec->n_fin) : NAN;
}

}  // namespace st

namespace {
size_t al(size_t x) { return (x + 255) & ~(size_t)255; }
}  // namespace

extern "C" int64_t st_numpy_mean_workspace(int64_t n) {
  const int64_t m = n > 0 ? n : 1;
  const int nb = 1 << st::stats_depth(m);
  return (int64_t)(al(2 * sizeof(st::Partial)) + al(64) + al(nb * sizeof(st::Partial)) +
                   al(sizeof(double) * m) + al(sizeof(double) * st::pw_val_size(m)));
}

extern "C" int st_numpy_mean(const double* x, int64_t n, double* out, void* workspace,
                             int64_t workspace_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (workspace_bytes < st_numpy_mean_workspace(n)) {
    sthost::set_error("st_numpy_mean: workspace too small");
    return ST_ENOMEM;
  }
  const int64_t m = n > 0 ? n : 1;
  const int D = st::stats_depth(m);
  char* ws = (char*)workspace;
  st::Partial* reduced = (st::Partial*)ws;           // [0] unused, [1] the record
  uint32_t* misc = (uint32_t*)(ws + al(2 * sizeof(st::Partial)));  // done, counts
  st::Partial* parts = (st::Partial*)((char*)misc + al(64));
  double* scratch = (double*)((char*)parts + al((1 << D) * sizeof(st::Partial)));
  double* val = (double*)((char*)scratch + al(sizeof(double) * m));
  ST_CUDA_CHECK(cudaMemsetAsync(misc, 0, 64, s));
  st::StatsTail tail = {};
  tail.on = 1;
  tail.it = 1;
  tail.done = misc;
  tail.reduced = reduced;
  tail.counts = misc + 4;
  tail.record_only = 1;
  tail.keep_counts = 1;
  tail.pw_depth = D;
  tail.pw_scratch = scratch;
  tail.pw_val = val;
  st::k_em_stats<<<1u << D, STATS_BLOCK, 0, s>>>(n > 0 ? n : 0, 0, x, x, nullptr, nullptr, 0,
                                                 parts, nullptr, tail);
  ST_LAUNCH_CHECK("k_em_stats");
  st::k_finish_mean<<<1, 32, 0, s>>>(reduced + 1, out);
  ST_LAUNCH_CHECK("k_finish_mean");
  return ST_OK;
}
