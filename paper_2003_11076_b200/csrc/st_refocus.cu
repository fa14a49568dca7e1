// See-through composition (refocus.py:24-148) on the device.
//
// k_refocus: per reference pixel, the Eq. 2 fp64 average of the static,
// in-bounds rays' bilinear colours (view order), provenance and n_rays.
// k_median: per-channel median over the clipped (2r+1)^2 window, applied to
// every non-COPIED pixel.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "st_common.cuh"

namespace st {

struct RefocusOut {
  double tot[3];
  int count;
};

// gather_static_colors for one pixel (refocus.py:24-49).
// rectified: every view has A = I, b = (bx, 0, 0); then warp_ab's roundings
// reduce to pu = u + d bx, pv = v exactly (as the EM kernels' warp_ctx).
__device__ __forceinline__ RefocusOut gather_colors(const uint8_t* __restrict__ images,
                                                    const st_rig& rig, int W, int H, double u,
                                                    double v, double d, uint32_t bits,
                                                    bool rectified = false) {
  RefocusOut r;
  r.tot[0] = r.tot[1] = r.tot[2] = 0.0;
  r.count = 0;
  const size_t plane = (size_t)W * H * 3;
  for (int k = 0; k < rig.num_views; ++k) {
    if (!((bits >> k) & 1u)) continue;
    WarpOut w;
    if (rectified) {
      w.pu = dadd(u, dmul(d, rig.warp_b[k][0]));
      w.pv = v;
      w.front = true;
    } else {
      w = warp_to(rig, k, u, v, d);
    }
    // refocus.py:42: margin 0 against the frame size
    if (!(w.front && w.pu >= 0.0 && w.pu <= (double)W - 1.0 && w.pv >= 0.0 &&
          w.pv <= (double)H - 1.0))
      continue;
    const Taps t = taps_of(w.pu, w.pv, W, H);
    const uint8_t* img = images + k * plane;
    const size_t b = ((size_t)t.iv * W + t.iu) * 3;
    const size_t bu = b + (size_t)t.su * 3;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      double f = lerp_u8(img[b + ch], img[bu + ch], t.fu);
      if (t.fv != 0.0) {
        const size_t bv = b + (size_t)t.sv * 3, bvu = bu + (size_t)t.sv * 3;
        const double bot = lerp_u8(img[bv + ch], img[bvu + ch], t.fu);
        f = dadd(f, dmul(t.fv, dsub(bot, f)));
      }
      r.tot[ch] = dadd(r.tot[ch], f);
    }
    ++r.count;
  }
  return r;
}

__device__ __forceinline__ uint8_t round_u8(double x) {
  // np.clip(np.rint(x), 0, 255).astype(uint8)
  return (uint8_t)fmin(fmax(rint(x), 0.0), 255.0);
}

// total / count correctly rounded for a small positive integer count: the
// 3-FMA Markstein step with r = RN(1/n) (st_common.cuh div_small, checked
// against __ddiv_rn by st_selftest).
__device__ __forceinline__ double div_count(double x, int n) {
  const double nn = (double)n;
  return div_small(x, nn, __drcp_rn(nn));
}

__global__ void k_refocus(const uint8_t* __restrict__ images, st_rig rig, int W, int H,
                          const float* __restrict__ values, const uint8_t* __restrict__ status,
                          const uint32_t* __restrict__ static_bits, int min_static_rays,
                          const uint8_t* __restrict__ copy_mask, uint8_t* __restrict__ out,
                          uint8_t* __restrict__ prov, uint8_t* __restrict__ n_rays,
                          int rectified, int64_t p0, int64_t p1) {
  // pixels [p0, p1) (a row band's rows; the whole frame otherwise)
  const int64_t p = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= p1) return;
  const uint8_t* ref = images + (size_t)rig.ref_index * W * H * 3 + (size_t)p * 3;
  uint8_t c0 = ref[0], c1 = ref[1], c2 = ref[2];
  const bool copied = copy_mask && copy_mask[p];
  uint8_t pv = copied ? ST_PROV_COPIED : ST_PROV_FALLBACK;
  uint8_t nr = 0;
  if (!copied && status[p] == ST_STATUS_VALID) {
    const double d = (double)values[p];  // refocus.py:133
    const RefocusOut r = gather_colors(images, rig, W, H, (double)(p % W), (double)(p / W), d,
                                       static_bits[p], rectified != 0);
    nr = (uint8_t)min(r.count, 255);
    if (r.count >= min_static_rays) {
      c0 = round_u8(div_count(r.tot[0], r.count));
      c1 = round_u8(div_count(r.tot[1], r.count));
      c2 = round_u8(div_count(r.tot[2], r.count));
      pv = ST_PROV_REFOCUSED;
    }
  }
  out[(size_t)p * 3] = c0;
  out[(size_t)p * 3 + 1] = c1;
  out[(size_t)p * 3 + 2] = c2;
  prov[p] = pv;
  n_rays[p] = nr;
}

// refocus_pixel, batched (refocus.py:52-65).
__global__ void k_refocus_pixels(const uint8_t* __restrict__ images, st_rig rig, int W, int H,
                                 const int64_t* __restrict__ pix, const double* __restrict__ d,
                                 const uint32_t* __restrict__ bits, int64_t n,
                                 int min_static_rays, uint8_t* __restrict__ rgb,
                                 int32_t* __restrict__ count, uint8_t* __restrict__ prov,
                                 double* __restrict__ totals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t p = pix[i];
  const RefocusOut r = gather_colors(images, rig, W, H, (double)(p % W), (double)(p / W), d[i],
                                     bits[i]);
  count[i] = r.count;
  if (totals)
    for (int ch = 0; ch < 3; ++ch) totals[3 * i + ch] = r.tot[ch];
  if (r.count >= min_static_rays) {
    const double c = (double)r.count;
    for (int ch = 0; ch < 3; ++ch) rgb[3 * i + ch] = round_u8(ddiv(r.tot[ch], c));
    prov[i] = ST_PROV_REFOCUSED;
  } else {
    const uint8_t* ref = images + (size_t)rig.ref_index * W * H * 3 + (size_t)p * 3;
    for (int ch = 0; ch < 3; ++ch) rgb[3 * i + ch] = ref[ch];
    prov[i] = ST_PROV_FALLBACK;
  }
}

// Median of the clipped window: the values are uint8, so the i-th smallest
// is found by counting (no sort), then 0.5 * (v[i0] + v[i1]) in fp32 and
// rint half-even -- refocus.py:98-105.
__device__ __forceinline__ int kth_smallest(const uint8_t* __restrict__ img, int W, int C, int ch,
                                            int ylo, int yhi, int xlo, int xhi, int kth) {
  // smallest value v with count(<= v) > kth
  int lo = 0, hi = 255;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    int cnt = 0;
    for (int y = ylo; y <= yhi; ++y)
      for (int x = xlo; x <= xhi; ++x) cnt += img[((size_t)y * W + x) * C + ch] <= mid;
    if (cnt > kth)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

__global__ void k_median_small(const uint8_t* __restrict__ src, int H, int W, int C, int radius,
                               const uint8_t* __restrict__ prov, uint8_t* __restrict__ out,
                               int64_t p0, int64_t p1) {
  const int64_t p = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= p1) return;
  const int x = (int)(p % W), y = (int)(p / W);
  if (prov && prov[p] == ST_PROV_COPIED) {
    for (int ch = 0; ch < C; ++ch) out[(size_t)p * C + ch] = src[(size_t)p * C + ch];
    return;
  }
  const int ylo = max(y - radius, 0), yhi = min(y + radius, H - 1);
  const int xlo = max(x - radius, 0), xhi = min(x + radius, W - 1);
  const int cnt = (yhi - ylo + 1) * (xhi - xlo + 1);
  if (radius == 1 && cnt == 9) {
    // full 3x3 window: v[(9-1)//2] == v[9//2], so 0.5*(v+v) and rint give
    // the middle value itself -- a fixed 19-exchange median-of-9 network
    // in registers (no data-dependent sort)
    for (int ch = 0; ch < C; ++ch) {
      int v[9];
#pragma unroll
      for (int j = 0; j < 9; ++j)
        v[j] = __ldg(src + ((size_t)(y - 1 + j / 3) * W + (x - 1 + j % 3)) * C + ch);
      auto cx = [&](int a, int b) {
        const int lo = min(v[a], v[b]), hi = max(v[a], v[b]);
        v[a] = lo;
        v[b] = hi;
      };
      cx(1, 2); cx(4, 5); cx(7, 8);
      cx(0, 1); cx(3, 4); cx(6, 7);
      cx(1, 2); cx(4, 5); cx(7, 8);
      cx(0, 3); cx(5, 8); cx(4, 7);
      cx(3, 6); cx(1, 4); cx(2, 5);
      cx(4, 7); cx(4, 2); cx(6, 4);
      cx(4, 2);
      out[(size_t)p * C + ch] = (uint8_t)v[4];
    }
    return;
  }
  for (int ch = 0; ch < C; ++ch) {
    int v0, v1;
    if (radius == 1) {
      // <= 9 values: insertion sort in registers
      int a[9];
      int n = 0;
      for (int yy = ylo; yy <= yhi; ++yy)
        for (int xx = xlo; xx <= xhi; ++xx) {
          int val = src[((size_t)yy * W + xx) * C + ch];
          int j = n++;
          while (j > 0 && a[j - 1] > val) {
            a[j] = a[j - 1];
            --j;
          }
          a[j] = val;
        }
      v0 = a[(cnt - 1) / 2];
      v1 = a[cnt / 2];
    } else {
      v0 = kth_smallest(src, W, C, ch, ylo, yhi, xlo, xhi, (cnt - 1) / 2);
      v1 = kth_smallest(src, W, C, ch, ylo, yhi, xlo, xhi, cnt / 2);
    }
    const float m = __fmul_rn(0.5f, __fadd_rn((float)v0, (float)v1));
    out[(size_t)p * C + ch] = (uint8_t)fminf(fmaxf(rintf(m), 0.0f), 255.0f);
  }
}

// radius-1 median of an RGB image with a 32x8 output tile per block: the
// tile and its 1-pixel halo are staged in shared memory with 32-bit loads,
// interior pixels take the median-of-9 network from there; pixels whose
// window is clipped (the image border) run k_median_small's general path.
#define MT_W 32
#define MT_H 8
__device__ __forceinline__ void med9(int (&v)[9]) {
  auto cx = [&](int a, int b) {
    const int lo = min(v[a], v[b]), hi = max(v[a], v[b]);
    v[a] = lo;
    v[b] = hi;
  };
  cx(1, 2); cx(4, 5); cx(7, 8);
  cx(0, 1); cx(3, 4); cx(6, 7);
  cx(1, 2); cx(4, 5); cx(7, 8);
  cx(0, 3); cx(5, 8); cx(4, 7);
  cx(3, 6); cx(1, 4); cx(2, 5);
  cx(4, 7); cx(4, 2); cx(6, 4);
  cx(4, 2);
}

__global__ void __launch_bounds__(MT_W * MT_H) k_median_rgb_tile(
    const uint8_t* __restrict__ src, int H, int W, const uint8_t* __restrict__ prov,
    uint8_t* __restrict__ out, int row0, int row1) {
  // output rows [row0, row1); the staged halo rows must hold refocused pixels
  __shared__ uint8_t tile[MT_H + 2][(MT_W + 2) * 3 + 2];
  const int x0 = blockIdx.x * MT_W, y0 = row0 + blockIdx.y * MT_H;
  const int tid = threadIdx.y * MT_W + threadIdx.x;
  for (int i = tid; i < (MT_H + 2) * (MT_W + 2) * 3; i += MT_W * MT_H) {
    const int r = i / ((MT_W + 2) * 3), cb = i % ((MT_W + 2) * 3);
    const int yy = min(max(y0 - 1 + r, 0), H - 1);
    const int xx = min(max(x0 - 1 + cb / 3, 0), W - 1);
    tile[r][cb] = src[((size_t)yy * W + xx) * 3 + cb % 3];
  }
  __syncthreads();
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  if (x >= W || y >= row1) return;
  const size_t p = (size_t)y * W + x;
  if (prov && prov[p] == ST_PROV_COPIED) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) out[p * 3 + ch] = src[p * 3 + ch];
    return;
  }
  if (x == 0 || y == 0 || x == W - 1 || y == H - 1) {
    // clipped window (4 or 6 values): insertion sort, 0.5 (v0 + v1), rint
    const int ylo = max(y - 1, 0), yhi = min(y + 1, H - 1);
    const int xlo = max(x - 1, 0), xhi = min(x + 1, W - 1);
    const int cnt = (yhi - ylo + 1) * (xhi - xlo + 1);
    for (int ch = 0; ch < 3; ++ch) {
      int a[9];
      int n = 0;
      for (int yy = ylo; yy <= yhi; ++yy)
        for (int xx = xlo; xx <= xhi; ++xx) {
          const int val = tile[yy - y0 + 1][(xx - x0 + 1) * 3 + ch];
          int j = n++;
          while (j > 0 && a[j - 1] > val) {
            a[j] = a[j - 1];
            --j;
          }
          a[j] = val;
        }
      const float m = __fmul_rn(0.5f, __fadd_rn((float)a[(cnt - 1) / 2], (float)a[cnt / 2]));
      out[p * 3 + ch] = (uint8_t)fminf(fmaxf(rintf(m), 0.0f), 255.0f);
    }
    return;
  }
  // full 3x3 window: the median-of-9 value itself (see k_median_small)
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    int v[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) v[j] = tile[threadIdx.y + j / 3][(threadIdx.x + j % 3) * 3 + ch];
    med9(v);
    out[p * 3 + ch] = (uint8_t)v[4];
  }
}

}  // namespace st

extern "C" int st_median(const uint8_t* image, int32_t H, int32_t W, int32_t C, int32_t radius,
                         uint8_t* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npx = (int64_t)W * H;
  if (radius <= 0) {
    ST_CUDA_CHECK(cudaMemcpyAsync(out, image, (size_t)npx * C, cudaMemcpyDeviceToDevice, s));
    return ST_OK;
  }
  st::k_median_small<<<(unsigned)((npx + 255) / 256), 256, 0, s>>>(image, H, W, C, radius,
                                                                   nullptr, out, 0, npx);
  ST_LAUNCH_CHECK("k_median_small");
  return ST_OK;
}

static int synthesize_rows(const uint8_t* images, const st_rig* rig, const float* values,
                           const uint8_t* status, const uint32_t* static_bits,
                           int32_t min_static_rays, int32_t median_radius,
                           const uint8_t* copy_mask, uint8_t* image_out, uint8_t* prov_out,
                           uint8_t* n_rays_out, uint8_t* scratch, int row0, int row1, int ext0,
                           int ext1, cudaStream_t s) {
  const int W = rig->width, H = rig->height;
  const int64_t e0 = (int64_t)ext0 * W, e1 = (int64_t)ext1 * W;
  uint8_t* stage = median_radius > 0 ? scratch : image_out;
  int rectified = 1;
  for (int k = 0; k < rig->num_views; ++k) {
    const double* a = rig->warp_a[k];
    const double* b = rig->warp_b[k];
    if (!(a[0] == 1.0 && a[1] == 0.0 && a[2] == 0.0 && a[3] == 0.0 && a[4] == 1.0 &&
          a[5] == 0.0 && a[6] == 0.0 && a[7] == 0.0 && a[8] == 1.0 && b[1] == 0.0 &&
          b[2] == 0.0 && fabs(b[0]) < 1e300))
      rectified = 0;
  }
  if (e1 > e0) {
    st::k_refocus<<<(unsigned)((e1 - e0 + 127) / 128), 128, 0, s>>>(
        images, *rig, W, H, values, status, static_bits, min_static_rays, copy_mask, stage,
        prov_out, n_rays_out, rectified, e0, e1);
    ST_LAUNCH_CHECK("k_refocus");
  }
  if (median_radius <= 0 || row1 <= row0) return ST_OK;
  if (median_radius == 1) {
    dim3 grid((W + MT_W - 1) / MT_W, (row1 - row0 + MT_H - 1) / MT_H);
    st::k_median_rgb_tile<<<grid, dim3(MT_W, MT_H), 0, s>>>(scratch, H, W, prov_out, image_out,
                                                            row0, row1);
    ST_LAUNCH_CHECK("k_median_rgb_tile");
  } else {
    const int64_t p0 = (int64_t)row0 * W, p1 = (int64_t)row1 * W;
    st::k_median_small<<<(unsigned)((p1 - p0 + 255) / 256), 256, 0, s>>>(
        scratch, H, W, 3, median_radius, prov_out, image_out, p0, p1);
    ST_LAUNCH_CHECK("k_median_small");
  }
  return ST_OK;
}

extern "C" int st_synthesize(const uint8_t* images, const st_rig* rig, const float* values,
                             const uint8_t* status, const uint32_t* static_bits,
                             int32_t min_static_rays, int32_t median_radius,
                             const uint8_t* copy_mask, uint8_t* image_out, uint8_t* prov_out,
                             uint8_t* n_rays_out, uint8_t* scratch, void* stream) {
  return synthesize_rows(images, rig, values, status, static_bits, min_static_rays,
                         median_radius, copy_mask, image_out, prov_out, n_rays_out, scratch, 0,
                         rig->height, 0, rig->height, (cudaStream_t)stream);
}

extern "C" int st_synthesize_rows(const uint8_t* images, const st_rig* rig, const float* values,
                                  const uint8_t* status, const uint32_t* static_bits,
                                  int32_t min_static_rays, int32_t median_radius,
                                  const uint8_t* copy_mask, uint8_t* image_out,
                                  uint8_t* prov_out, uint8_t* n_rays_out, uint8_t* scratch,
                                  int32_t row0, int32_t row1, int32_t ext0, int32_t ext1,
                                  void* stream) {
  const int H = rig->height;
  const int r = median_radius > 0 ? median_radius : 0;
  if (!(0 <= ext0 && ext0 <= row0 && row0 <= row1 && row1 <= ext1 && ext1 <= H) ||
      ext0 > std::max(row0 - r, 0) || ext1 < std::min(row1 + r, H)) {
    sthost::set_error("st_synthesize_rows: rows [%d, %d) need the refocused rows [%d, %d) "
                      "(got [%d, %d))", row0, row1, std::max(row0 - r, 0),
                      std::min(row1 + r, H), ext0, ext1);
    return ST_EINVAL;
  }
  return synthesize_rows(images, rig, values, status, static_bits, min_static_rays,
                         median_radius, copy_mask, image_out, prov_out, n_rays_out, scratch,
                         row0, row1, ext0, ext1, (cudaStream_t)stream);
}

namespace st {
// pipeline.py:254-255: copy_mask = ref prior >= threshold (float32 compare, NEP 50)
__global__ void k_copy_mask(const float* __restrict__ prior, int64_t n, float thr,
                            uint8_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = prior[i] >= thr ? 1 : 0;
}
}  // namespace st

extern "C" int st_copy_mask(const float* ref_prior, int64_t n, double threshold, uint8_t* out,
                            void* stream) {
  if (n <= 0) return ST_OK;
  st::k_copy_mask<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      ref_prior, n, (float)threshold, out);
  ST_LAUNCH_CHECK("k_copy_mask");
  return ST_OK;
}

extern "C" int st_refocus_pixels(const uint8_t* images, const st_rig* rig, const int64_t* pix,
                                 const double* d, const uint32_t* bits, int64_t n,
                                 int32_t min_static_rays, uint8_t* rgb, int32_t* count,
                                 uint8_t* prov, double* totals, void* stream) {
  if (n <= 0) return ST_OK;
  st::k_refocus_pixels<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      images, *rig, rig->width, rig->height, pix, d, bits, n, min_static_rays, rgb, count, prov,
      totals);
  ST_LAUNCH_CHECK("k_refocus_pixels");
  return ST_OK;
}
