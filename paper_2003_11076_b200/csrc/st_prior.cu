// Per-frame support candidate lists on the device (solver.py:286-321).
#include <cuda_runtime.h>
#include <float.h>
#include <math.h>
#include <stdint.h>

#include <cub/cub.cuh>

#include <algorithm>

#include "st_common.cuh"

namespace st {

// ---------------------------------------------------------------------------
// support candidate lists.  A record is (fp32 disparity, packed u|v) in the
// bucket of every 32x8 tile its radius-r disk bbox touches.  Each bucket is
// sorted by value in shared memory and its records grouped by value, so a
// pixel dedups candidates by walking value groups (solver.py:316-321 keeps
// unique (pixel, value) pairs) and tests one coverage bit per group.

struct SupGeom {
  int W, H, tiles_x, tiles_y, ir;
  double d_max;
  int ty_lo, ty_hi;  // tile rows built (a row band's; all otherwise)
};

__device__ __forceinline__ bool sup_range(const SupGeom& g, double su, double sv, double sd,
                                          int& tx0, int& tx1, int& ty0, int& ty1, float& val,
                                          int& pu, int& pv) {
  val = (float)sd;                                  // solver.py:308 (float32 values)
  const double dv = (double)val;
  if (!(dv > 0.0 && dv <= g.d_max)) return false;   // solver.py:380
  pu = (int)trunc(su);                              // .astype(np.int64)
  pv = (int)trunc(sv);
  const int x0 = max(pu - g.ir, 0), x1 = min(pu + g.ir, g.W - 1);
  const int y0 = max(pv - g.ir, 0), y1 = min(pv + g.ir, g.H - 1);
  if (x0 > x1 || y0 > y1) return false;
  tx0 = x0 / ST_TW;
  tx1 = x1 / ST_TW;
  ty0 = max(y0 / ST_TH, g.ty_lo);
  ty1 = min(y1 / ST_TH, g.ty_hi);
  return ty0 <= ty1;
}

// One point's 32x8 coverage rows in tile (tx, ty): the pixels inside its
// disk (solver.py:290-308: du^2 + dv^2 <= r^2, |du|, |dv| <= floor(r), in the
// image), dx range compared in double like numpy.
__device__ __forceinline__ uint32_t cover_row(const SupGeom& g, double r2, int tx, int ty,
                                              int pu, int pv, int r) {
  const int y = ty * ST_TH + r;
  if (y >= g.H) return 0u;
  const int dy = y - pv;
  if (abs(dy) > g.ir) return 0u;
  int dxm = (int)floor(sqrt(fmax(r2 - (double)(dy * dy), 0.0)));
  while ((double)((dxm + 1) * (dxm + 1) + dy * dy) <= r2) ++dxm;
  while (dxm >= 0 && (double)(dxm * dxm + dy * dy) > r2) --dxm;
  if (dxm < 0) return 0u;
  dxm = min(dxm, g.ir);
  const int x0 = max(max(pu - dxm, tx * ST_TW), 0);
  const int x1 = min(min(pu + dxm, tx * ST_TW + ST_TW - 1), g.W - 1);
  if (x0 > x1) return 0u;
  const int c0 = x0 - tx * ST_TW, nbits = x1 - x0 + 1;
  return (nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u)) << c0;
}

// Records per tile: every support point whose disk bbox touches the tile.
__global__ void k_tile_count(const double* __restrict__ uv, const double* __restrict__ d, int n,
                             SupGeom g, uint32_t* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int tx0, tx1, ty0, ty1, pu, pv;
  float val;
  if (!sup_range(g, uv[2 * i], uv[2 * i + 1], d[i], tx0, tx1, ty0, ty1, val, pu, pv)) return;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(cnt + ty * g.tiles_x + tx, 1u);
}

// Scatter the records into their tile's bucket (order inside a bucket is
// irrelevant: the bucket is sorted by value next).
__global__ void k_tile_fill(const double* __restrict__ uv, const double* __restrict__ d, int n,
                            SupGeom g, const uint32_t* __restrict__ off,
                            uint32_t* __restrict__ fill, unsigned long long* __restrict__ recs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int tx0, tx1, ty0, ty1, pu, pv;
  float val;
  if (!sup_range(g, uv[2 * i], uv[2 * i + 1], d[i], tx0, tx1, ty0, ty1, val, pu, pv)) return;
  const uint32_t packed = ((uint32_t)(uint16_t)(int16_t)pu) | ((uint32_t)(uint16_t)(int16_t)pv << 16);
  const unsigned long long rec = ((unsigned long long)__float_as_uint(val) << 32) | packed;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) {
      const int t = ty * g.tiles_x + tx;
      recs[off[t] + atomicAdd(fill + t, 1u)] = rec;
    }
}

#define TILE_CAP 2048  // records sorted in shared memory (more: in place, global)

// In-block bitonic sort of n keys (padded to a power of two with ~0).
__device__ void block_sort(unsigned long long* k, int n) {
  int p2 = 1;
  while (p2 < n) p2 <<= 1;
  for (int i = n + threadIdx.x; i < p2; i += blockDim.x) k[i] = ~0ull;
  __syncthreads();
  for (int size = 2; size <= p2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < p2 / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long a = k[lo], b = k[hi];
        if ((a > b) == up) {
          k[lo] = b;
          k[hi] = a;
        }
      }
      __syncthreads();
    }
}

// One block per tile: sort its records by (value, point), one group per
// distinct value, each record ORs its disk rows into its group's mask.
// Groups land at the tile's record offset (scratch); ngroups per tile.
__global__ void k_tile_groups(SupGeom g, double r2, const uint32_t* __restrict__ cnt,
                              const uint32_t* __restrict__ off, unsigned long long* recs,
                              float* __restrict__ tvalue, uint32_t* __restrict__ tmask,
                              uint32_t* __restrict__ ngroups) {
  extern __shared__ unsigned long long sh[];
  __shared__ uint32_t s_ng;
  const int t = blockIdx.x;
  const int n = (int)cnt[t];
  const uint32_t base = off[t];
  if (n == 0) {
    if (threadIdx.x == 0) ngroups[t] = 0u;
    return;
  }
  const bool in_smem = n <= TILE_CAP;
  unsigned long long* k = in_smem ? sh : recs + base;  // large buckets: sort in place
  uint32_t* gid = reinterpret_cast<uint32_t*>(sh + TILE_CAP);
  if (in_smem) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) k[i] = recs[base + i];
    block_sort(k, n);
  } else {
    // odd-even transposition sort in place in global memory: buckets this
    // large do not occur for de-duplicated support sets (at most one point
    // per pixel); kept correct, not fast
    for (int round = 0; round < n; ++round) {
      for (int i = 2 * threadIdx.x + (round & 1); i + 1 < n; i += 2 * blockDim.x) {
        const unsigned long long a = k[i], b = k[i + 1];
        if (a > b) {
          k[i] = b;
          k[i + 1] = a;
        }
      }
      __syncthreads();
    }
  }
  // group ids (value = high 32 bits): the number of value changes up to
  // each record -- a block-wide scan of the head flags over contiguous
  // per-thread ranges (large buckets: counted on the fly below)
  if (in_smem) {
    __shared__ uint32_t s_wsum[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int i0 = min(n, (int)threadIdx.x * per), i1 = min(n, i0 + per);
    uint32_t c = 0;
    for (int i = i0; i < i1; ++i) c += (i > 0 && (k[i] >> 32) != (k[i - 1] >> 32)) ? 1u : 0u;
    uint32_t x = c;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t acc = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        const uint32_t v = s_wsum[w];
        s_wsum[w] = acc;
        acc += v;
      }
      s_ng = acc + 1;
    }
    __syncthreads();
    uint32_t gcur = s_wsum[wid] + (x - c);
    for (int i = i0; i < i1; ++i) {
      if (i > 0 && (k[i] >> 32) != (k[i - 1] >> 32)) ++gcur;
      gid[i] = gcur;
    }
  } else if (threadIdx.x == 0) {
    uint32_t gcur = 0;
    for (int i = 1; i < n; ++i) gcur += (k[i] >> 32) != (k[i - 1] >> 32);
    s_ng = gcur + 1;
  }
  __syncthreads();
  const uint32_t ng = s_ng;
  const int tx = t % g.tiles_x, ty = t / g.tiles_x;
  // masks: tmask (scratch, at the tile's record offset) zeroed, then ORed
  for (uint32_t i = threadIdx.x; i < ng * ST_TH; i += blockDim.x) tmask[(size_t)base * ST_TH + i] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    uint32_t grp;
    if (in_smem) {
      grp = gid[i];
    } else {  // first record of this value = number of distinct values before it
      grp = 0;
      for (int j = 1; j <= i; ++j) grp += (k[j] >> 32) != (k[j - 1] >> 32);
    }
    const uint32_t uv = (uint32_t)(k[i] & 0xffffffffull);
    const int pu = (int)(int16_t)(uv & 0xffffu), pv = (int)(int16_t)(uv >> 16);
    if (i == 0 || (k[i] >> 32) != (k[i - 1] >> 32))
      tvalue[base + grp] = __uint_as_float((uint32_t)(k[i] >> 32));
#pragma unroll
    for (int r = 0; r < ST_TH; ++r) {
      const uint32_t bits = cover_row(g, r2, tx, ty, pu, pv, r);
      if (bits) atomicOr(tmask + ((size_t)base + grp) * ST_TH + r, bits);
    }
  }
  if (threadIdx.x == 0) ngroups[t] = ng;
}

// Compact every tile's groups to the scanned group offsets.
__global__ void k_tile_compact(const uint32_t* __restrict__ off, const uint32_t* __restrict__ ngroups,
                               const uint32_t* __restrict__ gstart, const float* __restrict__ tvalue,
                               const uint32_t* __restrict__ tmask, float* __restrict__ gvalue,
                               uint32_t* __restrict__ gmask) {
  const int t = blockIdx.x;
  const uint32_t ng = ngroups[t], src = off[t], dst = gstart[t];
  for (uint32_t i = threadIdx.x; i < ng; i += blockDim.x) gvalue[dst + i] = tvalue[src + i];
  for (uint32_t i = threadIdx.x; i < ng * ST_TH; i += blockDim.x)
    gmask[(size_t)dst * ST_TH + i] = tmask[(size_t)src * ST_TH + i];
}

}  // namespace st

// ---------------------------------------------------------------------------
// host side

namespace {

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct SupLayout {
  size_t cnt, off, fill, ng, gstart, recs, tvalue, tmask, gvalue, gmask, cub, total;
  size_t cub_bytes;
  int64_t max_rec;
  int tiles_x, tiles_y;
};

int tiles_per_point_max(int ir) {
  const int span = 2 * ir + 1;
  return ((span + ST_TW - 2) / ST_TW + 1) * ((span + ST_TH - 2) / ST_TH + 1);
}

SupLayout sup_layout(int n, int W, int H, double radius) {
  SupLayout L;
  const int ir = (int)floor(radius);
  L.tiles_x = (W + ST_TW - 1) / ST_TW;
  L.tiles_y = (H + ST_TH - 1) / ST_TH;
  const int n_tiles = L.tiles_x * L.tiles_y;
  L.max_rec = (int64_t)n * tiles_per_point_max(ir < 0 ? 0 : ir);
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                n_tiles + 1);
  L.cub_bytes = scan_bytes;
  const size_t R = (size_t)L.max_rec + 1, T = (size_t)n_tiles + 1;
  size_t o = 0;
  L.cnt = o;    o += align_up(sizeof(uint32_t) * T);
  L.fill = o;   o += align_up(sizeof(uint32_t) * T);
  L.off = o;    o += align_up(sizeof(uint32_t) * T);
  L.ng = o;     o += align_up(sizeof(uint32_t) * T);
  L.gstart = o; o += align_up(sizeof(uint32_t) * T);
  L.recs = o;   o += align_up(sizeof(unsigned long long) * R);
  L.tvalue = o; o += align_up(sizeof(float) * R);
  L.tmask = o;  o += align_up(sizeof(uint32_t) * ST_TH * R);
  L.gvalue = o; o += align_up(sizeof(float) * R);
  L.gmask = o;  o += align_up(sizeof(uint32_t) * ST_TH * R);
  L.cub = o;    o += align_up(L.cub_bytes);
  L.total = o;
  return L;
}

}  // namespace

extern "C" int64_t st_support_workspace(int32_t n, int32_t W, int32_t H, double radius) {
  return (int64_t)sup_layout(n, W, H, radius).total;
}

extern "C" int st_support_build_rows(const double* support_uv, const double* support_d,
                                     int32_t n, int32_t W, int32_t H, const st_params* p,
                                     st_frame* frame, void* workspace, int64_t workspace_bytes,
                                     int64_t* n_records, int32_t row0, int32_t row1,
                                     void* stream);

extern "C" int st_support_build(const double* support_uv, const double* support_d, int32_t n,
                                int32_t W, int32_t H, const st_params* p, st_frame* frame,
                                void* workspace, int64_t workspace_bytes, int64_t* n_records,
                                void* stream) {
  return st_support_build_rows(support_uv, support_d, n, W, H, p, frame, workspace,
                               workspace_bytes, n_records, 0, H, stream);
}

extern "C" int st_support_build_rows(const double* support_uv, const double* support_d,
                                     int32_t n, int32_t W, int32_t H, const st_params* p,
                                     st_frame* frame, void* workspace, int64_t workspace_bytes,
                                     int64_t* n_records, int32_t row0, int32_t row1,
                                     void* stream) {
  if (!(0 <= row0 && row0 < row1 && row1 <= H)) {
    sthost::set_error("st_support_build_rows: bad rows [%d, %d) of %d", row0, row1, H);
    return ST_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  SupLayout L = sup_layout(n, W, H, p->neighborhood_radius);
  if ((int64_t)L.total > workspace_bytes) {
    sthost::set_error("support workspace too small (%lld < %lld)", (long long)workspace_bytes,
                      (long long)L.total);
    return ST_ENOMEM;
  }
  {
    // lay the record arrays out for the largest support count the workspace
    // holds: the group tables' addresses (st_frame.sup_*) then do not move
    // with the frame's support count, so the EM's cached graph (st_api.cu)
    // serves every frame of a stream
    const int ir = (int)floor(p->neighborhood_radius);
    const int64_t tpp = tiles_per_point_max(ir < 0 ? 0 : ir);
    const int64_t per_rec = 16 + 8 * ST_TH;
    const int64_t fixed = (int64_t)L.recs + (int64_t)align_up(L.cub_bytes) + 6 * 256;
    if (workspace_bytes > fixed) {
      int64_t ncap = ((workspace_bytes - fixed) / per_rec - 1) / tpp;
      ncap = std::min<int64_t>(ncap, (int64_t)1 << 28);
      for (int tries = 0; tries < 4 && ncap > n; ++tries, ncap -= 64) {
        const SupLayout L2 = sup_layout((int)ncap, W, H, p->neighborhood_radius);
        if ((int64_t)L2.total <= workspace_bytes) {
          L = L2;
          break;
        }
      }
    }
  }
  char* ws = (char*)workspace;
  uint32_t* cnt = (uint32_t*)(ws + L.cnt);
  uint32_t* fill = (uint32_t*)(ws + L.fill);
  uint32_t* off = (uint32_t*)(ws + L.off);
  uint32_t* ng = (uint32_t*)(ws + L.ng);
  uint32_t* gstart = (uint32_t*)(ws + L.gstart);
  auto* recs = (unsigned long long*)(ws + L.recs);
  float* tvalue = (float*)(ws + L.tvalue);
  uint32_t* tmask = (uint32_t*)(ws + L.tmask);
  float* gvalue = (float*)(ws + L.gvalue);
  uint32_t* gmask = (uint32_t*)(ws + L.gmask);
  const int n_tiles = L.tiles_x * L.tiles_y;

  st::SupGeom g;
  g.W = W;
  g.H = H;
  g.tiles_x = L.tiles_x;
  g.tiles_y = L.tiles_y;
  g.ir = (int)floor(p->neighborhood_radius);
  g.d_max = p->d_max;
  g.ty_lo = row0 / ST_TH;
  g.ty_hi = (row1 - 1) / ST_TH;
  const double r = p->neighborhood_radius;

  // per-tile buckets: count, scan, fill -- no host round trip
  ST_CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (n_tiles + 1), s));
  ST_CUDA_CHECK(cudaMemsetAsync(fill, 0, sizeof(uint32_t) * (n_tiles + 1), s));
  if (n > 0) {
    st::k_tile_count<<<(n + 255) / 256, 256, 0, s>>>(support_uv, support_d, n, g, cnt);
    ST_LAUNCH_CHECK("k_tile_count");
  }
  size_t tb = L.cub_bytes;
  ST_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ws + L.cub, tb, cnt, off, n_tiles + 1, s));
  sthost::count_launch();
  if (n > 0) {
    st::k_tile_fill<<<(n + 255) / 256, 256, 0, s>>>(support_uv, support_d, n, g, off, fill, recs);
    ST_LAUNCH_CHECK("k_tile_fill");
  }
  // per tile: sort by value, one group per distinct value, coverage masks
  const int smem = TILE_CAP * (int)(sizeof(unsigned long long) + sizeof(uint32_t));
  st::k_tile_groups<<<n_tiles, 128, smem, s>>>(g, r * r, cnt, off, recs, tvalue, tmask, ng);
  ST_LAUNCH_CHECK("k_tile_groups");
  ST_CUDA_CHECK(cudaMemsetAsync(ng + n_tiles, 0, sizeof(uint32_t), s));
  tb = L.cub_bytes;
  ST_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ws + L.cub, tb, ng, gstart, n_tiles + 1, s));
  sthost::count_launch();
  st::k_tile_compact<<<n_tiles, 64, 0, s>>>(off, ng, gstart, tvalue, tmask, gvalue, gmask);
  ST_LAUNCH_CHECK("k_tile_compact");
  frame->sup_tile_start = gstart;
  frame->sup_value = gvalue;
  frame->sup_mask = gmask;
  if (n_records) {  // diagnostics only: one host round trip
    uint32_t total = 0;
    ST_CUDA_CHECK(cudaMemcpyAsync(&total, off + n_tiles, sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost, s));
    ST_CUDA_CHECK(cudaStreamSynchronize(s));
    *n_records = total;
  }
  return ST_OK;
}
