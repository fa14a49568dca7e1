// Per-frame support candidate lists on the device (solver.py:286-321).
#include <cuda_runtime.h>
#include <float.h>
#include <math.h>
#include <stdint.h>

#include <cub/cub.cuh>

#include "st_common.cuh"

namespace st {

// ---------------------------------------------------------------------------
// support candidate lists.  A record is (tile, fp32 disparity, packed u|v)
// for every support point whose radius-r disk bbox touches the tile.  After
// a radix sort on (tile, value) each tile's records are grouped by value, so
// a pixel dedups candidates by walking value groups (solver.py:316-321 keeps
// unique (pixel, value) pairs).

struct SupGeom {
  int W, H, tiles_x, tiles_y, ir;
  double d_max;
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
  ty0 = y0 / ST_TH;
  ty1 = y1 / ST_TH;
  return true;
}

__global__ void k_sup_count(const double* __restrict__ uv, const double* __restrict__ d, int n,
                            SupGeom g, uint32_t* __restrict__ counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int tx0, tx1, ty0, ty1, pu, pv;
  float val;
  counts[i] = sup_range(g, uv[2 * i], uv[2 * i + 1], d[i], tx0, tx1, ty0, ty1, val, pu, pv)
                  ? (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1))
                  : 0u;
}

__global__ void k_sup_emit(const double* __restrict__ uv, const double* __restrict__ d, int n,
                           SupGeom g, const uint32_t* __restrict__ offs,
                           unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int tx0, tx1, ty0, ty1, pu, pv;
  float val;
  if (!sup_range(g, uv[2 * i], uv[2 * i + 1], d[i], tx0, tx1, ty0, ty1, val, pu, pv)) return;
  uint32_t o = offs[i];
  const uint32_t packed = ((uint32_t)(uint16_t)(int16_t)pu) | ((uint32_t)(uint16_t)(int16_t)pv << 16);
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx, ++o) {
      keys[o] = ((unsigned long long)(ty * g.tiles_x + tx) << 32) | __float_as_uint(val);
      vals[o] = packed;
    }
}

// After the sort: records with equal (tile, value) form one group.  heads[i]
// flags the first record of each group.
// n_dev (nullable): the record count on the device -- launches sized by an
// upper bound then clear the flags of the padding records.
__global__ void k_sup_heads(const unsigned long long* __restrict__ keys, int64_t n_rec,
                            uint32_t* __restrict__ heads, const uint32_t* n_dev) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rec) return;
  const int64_t n = n_dev ? (int64_t)*n_dev : n_rec;
  heads[i] = i < n && (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

// Each record ORs the pixels of its tile inside its disk (solver.py:290-308:
// du^2 + dv^2 <= r^2, |du|, |dv| <= floor(r), in the image) into its group's
// 32x8 coverage mask; group heads also publish the group's key and value.
__global__ void k_sup_cover(const unsigned long long* __restrict__ keys,
                            const uint32_t* __restrict__ vals, const uint32_t* __restrict__ gid_incl,
                            int64_t n_rec, SupGeom g, double r2,
                            unsigned long long* __restrict__ gkey, float* __restrict__ gvalue,
                            uint32_t* __restrict__ gmask, const uint32_t* n_dev) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (n_dev ? (int64_t)*n_dev : n_rec)) return;
  const unsigned long long key = keys[i];
  const uint32_t grp = gid_incl[i] - 1;
  if (i == 0 || keys[i - 1] != key) {
    gkey[grp] = key;
    gvalue[grp] = __uint_as_float((uint32_t)(key & 0xffffffffull));
  }
  const int tile = (int)(key >> 32);
  const int tx = tile % g.tiles_x, ty = tile / g.tiles_x;
  const uint32_t uv = vals[i];
  const int pu = (int)(int16_t)(uv & 0xffffu), pv = (int)(int16_t)(uv >> 16);
  for (int r = 0; r < ST_TH; ++r) {
    const int y = ty * ST_TH + r;
    if (y >= g.H) break;
    const int dy = y - pv;
    if (abs(dy) > g.ir) continue;
    // largest |dx| with dx^2 + dy^2 <= r^2 (compared in double like numpy)
    int dxm = (int)floor(sqrt(fmax(r2 - (double)(dy * dy), 0.0)));
    while ((double)((dxm + 1) * (dxm + 1) + dy * dy) <= r2) ++dxm;
    while (dxm >= 0 && (double)(dxm * dxm + dy * dy) > r2) --dxm;
    if (dxm < 0) continue;
    dxm = min(dxm, g.ir);
    const int x0 = max(max(pu - dxm, tx * ST_TW), 0);
    const int x1 = min(min(pu + dxm, tx * ST_TW + ST_TW - 1), g.W - 1);
    if (x0 > x1) continue;
    const int c0 = x0 - tx * ST_TW, nbits = x1 - x0 + 1;
    const uint32_t bits = (nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u)) << c0;
    atomicOr(gmask + (size_t)grp * ST_TH + r, bits);
  }
}

__global__ void k_sup_group_start(const unsigned long long* __restrict__ gkey,
                                  const uint32_t* __restrict__ n_groups_ptr, int n_tiles,
                                  uint32_t* __restrict__ tile_start) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n_tiles) return;
  // lower_bound of tile i in the sorted group keys
  int64_t lo = 0, hi = n_groups_ptr ? (int64_t)*n_groups_ptr : 0;
  const unsigned long long want = (unsigned long long)i << 32;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (gkey[mid] < want)
      lo = mid + 1;
    else
      hi = mid;
  }
  tile_start[i] = (uint32_t)lo;
}

}  // namespace st

// ---------------------------------------------------------------------------
// host side

namespace {

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct SupLayout {
  size_t counts, offs, keys_in, keys_out, vals_in, vals_out, heads, gid, gkey, gvalue, gmask,
      tile_start, cub, total;
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
  size_t scan_bytes = 0, sort_bytes = 0, incl_bytes = 0;
  const int mr = (int)(L.max_rec > 0 ? L.max_rec : 1);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                n + 1);
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, mr);
  cub::DeviceScan::InclusiveSum(nullptr, incl_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr, mr);
  L.cub_bytes = std::max(scan_bytes, std::max(sort_bytes, incl_bytes));
  const size_t R = (size_t)L.max_rec + 1;
  size_t o = 0;
  L.counts = o;     o += align_up(sizeof(uint32_t) * (n + 1));
  L.offs = o;       o += align_up(sizeof(uint32_t) * (n + 1));
  L.keys_in = o;    o += align_up(sizeof(unsigned long long) * R);
  L.keys_out = o;   o += align_up(sizeof(unsigned long long) * R);
  L.vals_in = o;    o += align_up(sizeof(uint32_t) * R);
  L.vals_out = o;   o += align_up(sizeof(uint32_t) * R);
  L.heads = o;      o += align_up(sizeof(uint32_t) * R);
  L.gid = o;        o += align_up(sizeof(uint32_t) * R);
  L.gkey = o;       o += align_up(sizeof(unsigned long long) * R);
  L.gvalue = o;     o += align_up(sizeof(float) * R);
  L.gmask = o;      o += align_up(sizeof(uint32_t) * ST_TH * R);
  L.tile_start = o; o += align_up(sizeof(uint32_t) * (n_tiles + 1));
  L.cub = o;        o += align_up(L.cub_bytes);
  L.total = o;
  return L;
}

}  // namespace

extern "C" int64_t st_support_workspace(int32_t n, int32_t W, int32_t H, double radius) {
  return (int64_t)sup_layout(n, W, H, radius).total;
}

extern "C" int st_support_build(const double* support_uv, const double* support_d, int32_t n,
                                int32_t W, int32_t H, const st_params* p, st_frame* frame,
                                void* workspace, int64_t workspace_bytes, int64_t* n_records,
                                void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const SupLayout L = sup_layout(n, W, H, p->neighborhood_radius);
  if ((int64_t)L.total > workspace_bytes) {
    sthost::set_error("support workspace too small (%lld < %lld)", (long long)workspace_bytes,
                      (long long)L.total);
    return ST_ENOMEM;
  }
  char* ws = (char*)workspace;
  uint32_t* counts = (uint32_t*)(ws + L.counts);
  uint32_t* offs = (uint32_t*)(ws + L.offs);
  auto* keys_in = (unsigned long long*)(ws + L.keys_in);
  auto* keys_out = (unsigned long long*)(ws + L.keys_out);
  uint32_t* vals_in = (uint32_t*)(ws + L.vals_in);
  uint32_t* vals_out = (uint32_t*)(ws + L.vals_out);
  uint32_t* tile_start = (uint32_t*)(ws + L.tile_start);
  uint32_t* heads = (uint32_t*)(ws + L.heads);
  uint32_t* gid = (uint32_t*)(ws + L.gid);
  auto* gkey = (unsigned long long*)(ws + L.gkey);
  float* gvalue = (float*)(ws + L.gvalue);
  uint32_t* gmask = (uint32_t*)(ws + L.gmask);
  void* cub_tmp = ws + L.cub;
  const int n_tiles = L.tiles_x * L.tiles_y;

  st::SupGeom g;
  g.W = W;
  g.H = H;
  g.tiles_x = L.tiles_x;
  g.tiles_y = L.tiles_y;
  g.ir = (int)floor(p->neighborhood_radius);
  g.d_max = p->d_max;

  int64_t total = 0;
  if (n > 0) {
    ST_CUDA_CHECK(cudaMemsetAsync(counts + n, 0, sizeof(uint32_t), s));
    st::k_sup_count<<<(n + 255) / 256, 256, 0, s>>>(support_uv, support_d, n, g, counts);
    ST_LAUNCH_CHECK("k_sup_count");
    size_t tb = L.cub_bytes;
    ST_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, counts, offs, n + 1, s));
    sthost::count_launch();
    // n_records == NULL: no host round trip -- every later launch is sized
    // by the bound max_rec, padding keys (all ones) sort after the real
    // records and the kernels read the real count offs[n] on the device.
    const bool async = n_records == nullptr;
    const uint32_t* total_dev = async ? offs + n : nullptr;
    if (async) {
      total = L.max_rec;
      ST_CUDA_CHECK(cudaMemsetAsync(keys_in, 0xff, sizeof(unsigned long long) * (size_t)total, s));
    } else {
      uint32_t host_total = 0;
      ST_CUDA_CHECK(cudaMemcpyAsync(&host_total, offs + n, sizeof(uint32_t),
                                    cudaMemcpyDeviceToHost, s));
      ST_CUDA_CHECK(cudaStreamSynchronize(s));
      total = host_total;
    }
    if (total > 0) {
      st::k_sup_emit<<<(n + 255) / 256, 256, 0, s>>>(support_uv, support_d, n, g, offs, keys_in,
                                                      vals_in);
      ST_LAUNCH_CHECK("k_sup_emit");
      int tile_bits = 1;
      while ((1ll << tile_bits) <= n_tiles) ++tile_bits;
      tb = L.cub_bytes;
      ST_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, keys_in, keys_out, vals_in,
                                                    vals_out, (int)total, 0, 32 + tile_bits, s));
      sthost::count_launch();
      // (tile, value) groups and their 32x8 pixel coverage masks
      const unsigned rb = (unsigned)((total + 255) / 256);
      st::k_sup_heads<<<rb, 256, 0, s>>>(keys_out, total, heads, total_dev);
      ST_LAUNCH_CHECK("k_sup_heads");
      tb = L.cub_bytes;
      ST_CUDA_CHECK(cub::DeviceScan::InclusiveSum(cub_tmp, tb, heads, gid, (int)total, s));
      sthost::count_launch();
      ST_CUDA_CHECK(cudaMemsetAsync(gmask, 0, sizeof(uint32_t) * ST_TH * (size_t)total, s));
      const double r = p->neighborhood_radius;
      st::k_sup_cover<<<rb, 256, 0, s>>>(keys_out, vals_out, gid, total, g, r * r, gkey, gvalue,
                                         gmask, total_dev);
      ST_LAUNCH_CHECK("k_sup_cover");
    }
  }
  st::k_sup_group_start<<<(unsigned)((n_tiles + 1 + 255) / 256), 256, 0, s>>>(
      gkey, total > 0 ? gid + total - 1 : nullptr, n_tiles, tile_start);
  ST_LAUNCH_CHECK("k_sup_group_start");
  frame->sup_tile_start = tile_start;
  frame->sup_value = gvalue;
  frame->sup_mask = gmask;
  if (n_records) *n_records = total;
  return ST_OK;
}

