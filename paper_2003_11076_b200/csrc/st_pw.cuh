// numpy's float64 summation order on the device (block-level building blocks).
//
// np.add.reduce over a contiguous float64 array evaluates 0.0 +
// pairwise_sum(a, n) (numpy/_core/src/umath/loops_utils.h.src):
//   n < 8     : a running sum from 0.0,
//   n <= 128  : eight strided accumulators r[j] = a[j] + a[8+j] + ... (in
//               order), combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then
//               the n % 8 tail added in order,
//   otherwise : split at n2 = n/2 rounded down to a multiple of 8, sum of the
//               two halves' sums.
// The identity start and the split rule are pinned against numpy itself
// (tests/test_oracle.py, oracle.numpy_sum_order).  The tree below a node is
// evaluated level by level, deepest first, so every addition is the
// recursion's own (left + right); leaves are summed by 8-lane groups, lane j
// owning accumulator r[j], and the r-tree is two xor-shuffles and one more
// (IEEE addition is commutative, every lane ends with the same bits).
#pragma once

#include <stdint.h>

#include "st_common.cuh"

namespace st {

#define PW_LEAF 128
#define PW_MAX_LEVELS 11  // levels kept in shared memory: node depth <= 10

__device__ __forceinline__ int64_t pw_split(int64_t n) {
  const int64_t h = n / 2;
  return h - h % 8;
}

// Node (s, n) at depth t along the t low bits of `path` (MSB first) below
// (s0, n0); false when an ancestor is already a leaf.
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

// Deepest level holding a node below a root of size n0 (levels < cap).
__device__ __forceinline__ int pw_depth_of(int64_t n0, int cap) {
  int depth = 0;
  int64_t n = n0;
  while (n > PW_LEAF && depth < cap) {
    n -= pw_split(n);  // the right child is the larger half
    ++depth;
  }
  return depth;
}

// A leaf (n <= 128 values at a) summed by the 8 lanes of `g` (lane j of the
// group = accumulator j); every lane returns the leaf's sum.
__device__ __forceinline__ double pw_leaf8(const double* __restrict__ a, int64_t n, int j,
                                           unsigned gmask) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = dadd(r, a[i]);
    return r;  // (every lane computes it)
  }
  const int64_t body = n - (n % 8);
  double r = a[j];
  for (int64_t i = 8 + j; i < body; i += 8) r = dadd(r, a[i]);
  r = dadd(r, __shfl_xor_sync(gmask, r, 1));  // (r0 + r1), (r2 + r3), ...
  r = dadd(r, __shfl_xor_sync(gmask, r, 2));  // (r0 + r1) + (r2 + r3), ...
  r = dadd(r, __shfl_xor_sync(gmask, r, 4));
  for (int64_t i = body; i < n; ++i) r = dadd(r, a[i]);
  return r;
}

// Sum of node (s0, n0) of the tree over `a` by the whole block (blockDim.x a
// multiple of 32): level by level in `val` (2^(levels) - 1 doubles; shared
// or global), leaves by 8-lane groups.  Every thread returns the sum.
__device__ __forceinline__ double pw_block_sum(const double* __restrict__ a, int64_t s0,
                                               int64_t n0, double* val, int levels) {
  const int depth = pw_depth_of(n0, levels - 1);
  const int lane8 = threadIdx.x & 7;
  const unsigned gmask = 0xFFu << (threadIdx.x & 24);
  const int groups = blockDim.x >> 3, grp = threadIdx.x >> 3;
  for (int t = depth; t >= 0; --t) {
    const unsigned cnt = 1u << t;
    for (unsigned p0 = 0; p0 < cnt; p0 += groups) {
      const unsigned p = p0 + grp;
      int64_t s = 0, n = 0;
      const bool ok = p < cnt && pw_descend(s0, n0, t, p, s, n);
      if (ok && n <= PW_LEAF) {
        const double v = pw_leaf8(a + s, n, lane8, gmask);
        if (lane8 == 0) val[cnt - 1 + p] = v;
      } else if (ok && lane8 == 0) {
        val[cnt - 1 + p] = dadd(val[(2u << t) - 1 + 2 * p], val[(2u << t) + 2 * p]);
      }
    }
    __syncthreads();
  }
  const double r = val[0];
  __syncthreads();
  return r;
}

// The top D levels of the tree of n values, whose nodes at depth D (or
// leaves above it) were summed into node_sum(path << (D - t)): by one block.
template <typename NodeSum>
__device__ __forceinline__ double pw_top_sum(int64_t n, int D, NodeSum node_sum, double* val) {
  const int depth = pw_depth_of(n, D);
  for (int t = depth; t >= 0; --t) {
    const unsigned cnt = 1u << t;
    for (unsigned p = threadIdx.x; p < cnt; p += blockDim.x) {
      int64_t s, m;
      if (!pw_descend(0, n, t, p, s, m)) continue;
      val[cnt - 1 + p] = (t == D || m <= PW_LEAF)
                             ? node_sum(p << (D - t))
                             : dadd(val[(2u << t) - 1 + 2 * p], val[(2u << t) + 2 * p]);
    }
    __syncthreads();
  }
  const double r = val[0];
  __syncthreads();
  return r;
}

// Block `b` of a 2^D grid: its node (s, n) of the tree of n0 values; false
// for a block under an early leaf (that leaf belongs to the lowest path).
__device__ __forceinline__ bool pw_block_node(int64_t n0, int D, unsigned b, int64_t& s,
                                              int64_t& n) {
  s = 0;
  n = n0;
  int d = 0;
  while (d < D && n > PW_LEAF) {
    const int64_t n2 = pw_split(n);
    if ((b >> (D - 1 - d)) & 1u) {
      s += n2;
      n -= n2;
    } else {
      n = n2;
    }
    ++d;
  }
  return !(d < D && (b & ((1u << (D - d)) - 1u)) != 0);
}

}  // namespace st
