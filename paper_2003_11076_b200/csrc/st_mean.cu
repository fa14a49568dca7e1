// numpy's float64 mean, bit for bit, for the EM statistics (solver.py:466
// `finite.mean()` of the M-step energies and :471 of the previous-disparity
// energies; written to em_stats.txt by pipeline.py:292-302 with repr()).
//
// np.add.reduce over a contiguous float64 array evaluates
//     0.0 + pairwise_sum(a, n)
// (numpy loops_utils.h.src): a block of n <= 128 values is summed with
// eight strided accumulators r[j] += a[8i + j] combined as
// ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)), then the n % 8 tail in
// order (n < 8: a plain running sum from 0.0); a larger block splits at
// n2 = n/2 rounded down to a multiple of 8 and adds the two halves' sums.
// The mean is that sum / n (IEEE division).  The identity start and the
// split rule are pinned against numpy itself in tests/test_oracle.py.
//
// Device form: the top D levels of the recursion assign one node (~4k
// values) per block; a block enumerates its node's leaves, sums them in
// parallel (one thread per leaf), then replays the node's additions in
// recursion order; the last block to finish replays the top D levels over
// the blocks' sums.  The sequence is the FINITE values in slot order: when
// a value is non-finite (never for d_max >= 1: the coarse sweep always has
// a finite candidate) one block first compacts them into scratch.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include <cub/block/block_scan.cuh>

#include "st_common.cuh"
#include "st_em.cuh"

namespace st {

#define PW_LEAF 128
#define PW_THREADS 256

__device__ __forceinline__ int64_t pw_split(int64_t n) {
  const int64_t h = n / 2;
  return h - h % 8;
}

__device__ double pw_leaf(const double* __restrict__ a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = dadd(r, a[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = dadd(r[j], a[i + j]);
  }
  double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
  for (; i < n; ++i) res = dadd(res, a[i]);
  return res;
}

struct PwSeq {
  const double* src;
  int64_t m;
};

// Rare path: compact the finite values (slot order) into scratch when the
// statistics found a non-finite one; otherwise point at the input.
__global__ void __launch_bounds__(1024) k_pw_prepare(const double* __restrict__ e,
                                                     const double* __restrict__ pe, int64_t n,
                                                     const Partial* __restrict__ rec,
                                                     double* __restrict__ scratch, PwSeq* seq,
                                                     int with_prev, int it,
                                                     const st_stats* __restrict__ stats) {
  if (stats->iterations_run != it) return;  // the iteration did not run (converged before)
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t base;
  for (int y = 0; y < 1 + with_prev; ++y) {
    const double* x = y ? pe : e;
    const int64_t m = y ? rec->n_pfin : rec->n_fin;
    if (m == n) {
      if (threadIdx.x == 0) seq[y] = PwSeq{x, n};
      continue;
    }
    double* out = scratch + (size_t)y * n;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    for (int64_t c = 0; c < n; c += 1024) {
      const int64_t i = c + threadIdx.x;
      const int f = (i < n && isfinite(x[i])) ? 1 : 0;
      int off, tot;
      Scan(tmp).ExclusiveSum(f, off, tot);
      if (f) out[base + off] = x[i];
      __syncthreads();
      if (threadIdx.x == 0) base += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) seq[y] = PwSeq{out, base};
    __syncthreads();
  }
}

// Node (s, n) at depth t along the t low bits of `path` (MSB first) below
// (s0, n0); false when an ancestor is already a leaf (size <= PW_LEAF).
__device__ __forceinline__ bool pw_descend(int64_t s0, int64_t n0, int t, unsigned path,
                                           int64_t& s, int64_t& n) {
  s = s0;
  n = n0;
  for (int d = 0; d < t; ++d) {
    if (n <= PW_LEAF) return false;
    const int64_t n2 = pw_split(n);
    if ((path >> (t - 1 - d)) & 1u) {
      s += n2;
      n -= n2;
    } else {
      n = n2;
    }
  }
  return true;
}

#define PW_MAX_LEVELS 11  // node depth below a block root / top depth D: <= 10

// The recursion below (s0, n0) evaluated level by level, deepest first: node
// (t, p) = val[2^t - 1 + p] is a leaf sum when its size is <= PW_LEAF (or
// when t == cut, with its value from `cut_val(p)`), else the sum of its two
// children.  Every addition is the recursion's own (left + right).
template <typename CutVal>
__device__ double pw_levels(const double* __restrict__ a, int64_t s0, int64_t n0, int cut,
                            CutVal cut_val, double* val) {
  int depth = 0;  // deepest level with a node
  {
    int64_t n = n0;
    while (n > PW_LEAF && depth < cut) {
      n = n - pw_split(n);  // the right child is the larger half
      ++depth;
    }
  }
  for (int t = depth; t >= 0; --t) {
    const unsigned cnt = 1u << t;
    for (unsigned p = threadIdx.x; p < cnt; p += blockDim.x) {
      int64_t s, n;
      if (!pw_descend(s0, n0, t, p, s, n)) continue;
      double v;
      if (t == cut)
        v = cut_val(p);
      else if (n <= PW_LEAF)
        v = a ? pw_leaf(a + s, n) : cut_val(p << (cut - t));
      else
        v = dadd(val[(2u << t) - 1 + 2 * p], val[(2u << t) + 2 * p]);
      val[cnt - 1 + p] = v;
    }
    __syncthreads();
  }
  return val[0];
}

// gridDim.x = 2^D nodes, gridDim.y = 1 (E) or 2 (E and previous E).
__global__ void __launch_bounds__(PW_THREADS) k_pw_mean(const PwSeq* __restrict__ seq, int D,
                                                        int it, double* __restrict__ partial,
                                                        unsigned* __restrict__ done,
                                                        st_stats* __restrict__ stats) {
  if (stats->iterations_run != it) return;  // the iteration did not run (converged before)
  __shared__ double val[(1 << PW_MAX_LEVELS) - 1];
  const int y = blockIdx.y;
  const PwSeq q = seq[y];
  const int nb = gridDim.x;
  // this block's node: D levels down along its index; an early leaf belongs
  // to the lowest path under it
  int64_t s = 0, n = q.m;
  bool own = true;
  {
    int d = 0;
    while (d < D && n > PW_LEAF) {
      const int64_t n2 = pw_split(n);
      if ((blockIdx.x >> (D - 1 - d)) & 1u) {
        s += n2;
        n -= n2;
      } else {
        n = n2;
      }
      ++d;
    }
    if (d < D && (blockIdx.x & ((1u << (D - d)) - 1u)) != 0) own = false;
  }
  if (own) {
    const double v = q.m > 0 ? pw_levels(q.src, s, n, PW_MAX_LEVELS - 1,
                                         [&](unsigned) { return 0.0; }, val)
                             : 0.0;
    if (threadIdx.x == 0) partial[(size_t)y * nb + blockIdx.x] = v;
  }
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(done + y, 1u) == (unsigned)nb - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the top D levels over the blocks' sums (a top-level leaf at depth t, path
  // p, was written by block p << (D - t))
  const double* part = partial + (size_t)y * nb;
  const double total = pw_levels(nullptr, 0, q.m, D,
                                 [&](unsigned p) { return part[p]; }, val);
  if (threadIdx.x == 0) {
    done[y] = 0u;
    const double mean = q.m > 0 ? ddiv(dadd(0.0, total), (double)q.m) : NAN;
    if (y == 0)
      stats->mean_energy[it - 1] = mean;
    else
      stats->prev_energy[it - 2] = mean;
  }
}

}  // namespace st

// Host launcher used by the asynchronous solve (st_api.cu).
int st_pw_means(const double* e, const double* pe, int64_t n, const void* rec, void* scratch,
                void* seq, double* partial, unsigned* done, int it, st_stats* stats,
                cudaStream_t s) {
  if (n <= 0) return ST_OK;
  const int with_prev = it > 1 ? 1 : 0;
  st::k_pw_prepare<<<1, 1024, 0, s>>>(e, pe, n, (const st::Partial*)rec, (double*)scratch,
                                       (st::PwSeq*)seq, with_prev, it, stats);
  ST_LAUNCH_CHECK("k_pw_prepare");
  int D = 0;  // <= 10 top levels: nodes of ~4k values (<= 128 k up to 2^27 values)
  while (D < 10 && (n >> D) > 4096) ++D;
  st::k_pw_mean<<<dim3(1u << D, 1 + with_prev), PW_THREADS, 0, s>>>(
      (const st::PwSeq*)seq, D, it, partial, done, stats);
  ST_LAUNCH_CHECK("k_pw_mean");
  return ST_OK;
}

namespace st {
__global__ void k_count_finite(const double* __restrict__ x, int64_t n, Partial* rec,
                               st_stats* stats) {
  long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += isfinite(x[i]) ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long*)&rec->n_fin, (unsigned long long)c);
  if (blockIdx.x == 0 && threadIdx.x == 0) stats->iterations_run = 1;
}
}  // namespace st

extern "C" int64_t st_numpy_mean_workspace(int64_t n) {
  return (int64_t)(1024 + sizeof(st_stats) + sizeof(double) * 2 * (1 << ST_PW_MAX_DEPTH) +
                   sizeof(double) * (n > 0 ? n : 1) + 256 * 4);
}

// np.mean of the finite values of x (n float64, device), bit for bit: the
// device form of solver.py:466 `finite.mean()` (NaN when none is finite).
extern "C" int st_numpy_mean(const double* x, int64_t n, double* out, void* workspace,
                             int64_t workspace_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (workspace_bytes < st_numpy_mean_workspace(n)) {
    sthost::set_error("st_numpy_mean: workspace too small");
    return ST_ENOMEM;
  }
  char* ws = (char*)workspace;
  st::Partial* rec = (st::Partial*)ws;                     // 0..255
  void* seq = ws + 256;                                     // 256..511
  unsigned* done = (unsigned*)(ws + 512);                   // 512..767
  st_stats* stats = (st_stats*)(ws + 1024);
  double* partial = (double*)(ws + 1024 + ((sizeof(st_stats) + 255) & ~(size_t)255));
  double* scratch = partial + 2 * (1 << ST_PW_MAX_DEPTH);
  ST_CUDA_CHECK(cudaMemsetAsync(ws, 0, 1024, s));
  ST_CUDA_CHECK(cudaMemsetAsync(stats, 0, sizeof(st_stats), s));
  if (n > 0) {
    st::k_count_finite<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, s>>>(
        x, n, rec, stats);
    ST_LAUNCH_CHECK("k_count_finite");
    int rc = st_pw_means(x, x, n, rec, scratch, seq, partial, done, 1, stats, s);
    if (rc) return rc;
    ST_CUDA_CHECK(cudaMemcpyAsync(out, &stats->mean_energy[0], sizeof(double),
                                  cudaMemcpyDeviceToDevice, s));
  } else {
    const double nan = NAN;
    ST_CUDA_CHECK(cudaMemcpyAsync(out, &nan, sizeof(double), cudaMemcpyHostToDevice, s));
    ST_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  return ST_OK;
}
