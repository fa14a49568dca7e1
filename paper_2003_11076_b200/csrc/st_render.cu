// Device renderer for the synthetic light fields: the
// reference's `render` (synth.py:244-309) -- per-view nearest-surface ray
// cast (synth.py:174-230), value-noise + sinusoid textures (synth.py:25-82),
// 4x supersampled billboard edges, the reference view's background and
// disparity ground truth -- and `corrupt_prior` (synth.py:314-346): seeded
// label flips (numpy's PCG64 stream, advanced per chunk on the device) and
// the clipped box blur.  Everything follows the reference's operation order
// without FMA contraction; the flips and the blur are exact integer work.
//
// Layout: one thread per pixel, images (H, W, 3) u8 and masks / priors
// (H, W) row-major, exactly the reference's arrays.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "st_common.cuh"

namespace {

using st::dadd;
using st::ddiv;
using st::dmul;
using st::dsub;

constexpr uint64_t LAT_M1 = 0x9E3779B97F4A7C15ull;
constexpr uint64_t LAT_M2 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t LAT_M3 = 0x94D049BB133111EBull;

struct RenderArgs {
  st_scene sc;
  double center[3];
  double rot[9];  // row-major; dirs = (b0, b1, 1) @ rot
  int with_occluders;
};

// synth.py:25-36: per-lattice-point hash in [0, 1)
__device__ __forceinline__ double lattice(int64_t ix, int64_t iy, uint64_t seed32) {
  uint64_t h = ((uint64_t)ix * LAT_M1) ^ ((uint64_t)iy * LAT_M2) ^ (seed32 * LAT_M3);
  h ^= h >> 30;
  h *= LAT_M2;
  h ^= h >> 27;
  h *= LAT_M3;
  h ^= h >> 31;
  return ddiv((double)(h >> 11), 9007199254740992.0);
}

// synth.py:39-56: smoothstep-interpolated lattice noise in [-1, 1]
__device__ double value_noise(double x, double y, uint64_t seed32) {
  const double x0 = floor(x), y0 = floor(y);
  const double tx = dsub(x, x0), ty = dsub(y, y0);
  const int64_t i = (int64_t)x0, j = (int64_t)y0;
  const double wx = dmul(dmul(tx, tx), dsub(3.0, dmul(2.0, tx)));
  const double wy = dmul(dmul(ty, ty), dsub(3.0, dmul(2.0, ty)));
  const double a = lattice(i, j, seed32), b = lattice(i + 1, j, seed32);
  const double c = lattice(i, j + 1, seed32), d = lattice(i + 1, j + 1, seed32);
  const double upper = dadd(a, dmul(wx, dsub(b, a)));
  const double lower = dadd(c, dmul(wx, dsub(d, c)));
  return dsub(dmul(2.0, dadd(upper, dmul(wy, dsub(lower, upper)))), 1.0);
}

// synth.py:59-82 at one world point; the rng-drawn constants come from the
// host (numpy's own draws and scalar cos/sin)
__device__ void surface_color(const st_surface& s, double px, double py, double out[3]) {
  const double x = dmul(px, s.frequency), y = dmul(py, s.frequency);
  const double nz = value_noise(dadd(x, 13.7), dadd(y, 7.31), (uint64_t)(uint32_t)s.seed);
  double arg[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) arg[i] = dmul(s.c0[i], dadd(dmul(x, s.ca[i]), dmul(y, s.sa[i])));
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) acc = dadd(acc, sin(dadd(arg[i], s.ph[i][c])));
    const double v = dadd(s.base, dmul(s.amplitude, dadd(dmul(dsub(1.0, s.nw[c]), ddiv(acc, 3.0)),
                                                         dmul(s.nw[c], nz))));
    out[c] = fmin(fmax(v, 0.0), 255.0);
  }
}

// synth.py:174-230 for one ray through sensor point (su, sv): the first
// surface hit in trace order (occluders by depth, then planes by depth).
// Returns the surface index, or -1 when the ray hits nothing.
__device__ int trace(const RenderArgs& A, double su, double sv, double color[3]) {
  const st_scene& sc = A.sc;
  const double b0 = ddiv(dsub(su, sc.cx), sc.fx), b1 = ddiv(dsub(sv, sc.cy), sc.fy);
  const double* R = A.rot;
  const double dx = dadd(dadd(dmul(b0, R[0]), dmul(b1, R[3])), R[6]);
  const double dy = dadd(dadd(dmul(b0, R[1]), dmul(b1, R[4])), R[7]);
  const double dz = dadd(dadd(dmul(b0, R[2]), dmul(b1, R[5])), R[8]);
  if (!(dz > 0.0)) return -1;  // every surface test needs a forward ray
  for (int k = 0; k < sc.n_surfaces; ++k) {
    const st_surface& s = sc.surf[k];
    if (s.is_occluder && !A.with_occluders) continue;
    const double t = ddiv(dsub(s.depth, A.center[2]), dz);
    const double px = dadd(A.center[0], dmul(t, dx));
    const double py = dadd(A.center[1], dmul(t, dy));
    bool hit;
    if (s.is_occluder) {
      hit = fabs(dsub(px, s.center_x)) <= s.half_w && fabs(dsub(py, s.center_y)) <= s.half_h;
    } else {
      hit = true;
      if (s.has_x_min) hit = hit && px >= s.x_min;
      if (s.has_x_max) hit = hit && px < s.x_max;
    }
    if (hit) {
      surface_color(s, px, py, color);
      return k;
    }
  }
  return -1;
}

__device__ __forceinline__ uint8_t to_u8(double v) {  // np.clip(np.rint(v), 0, 255)
  return (uint8_t)fmin(fmax(rint(v), 0.0), 255.0);
}

// One view (synth.py:251-286): image, occluder cover mask, and -- for the
// billboard edge pixels -- the 4-sample supersampled colour and cover.
__global__ void k_render_view(RenderArgs A, const double* __restrict__ rects, int n_rects,
                              uint8_t* __restrict__ image, uint8_t* __restrict__ mask,
                              int* __restrict__ fail) {
  const int W = A.sc.width, H = A.sc.height;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)W * H) return;
  const double su = (double)(p % W), sv = (double)(p / W);
  bool edge = false;
  for (int o = 0; o < n_rects; ++o) {
    const double u0 = rects[4 * o], u1 = rects[4 * o + 1];
    const double v0 = rects[4 * o + 2], v1 = rects[4 * o + 3];
    edge = edge || ((fabs(dsub(su, u0)) <= 0.5 || fabs(dsub(su, u1)) <= 0.5) &&
                    sv >= dsub(v0, 0.5) && sv <= dadd(v1, 0.5));
    edge = edge || ((fabs(dsub(sv, v0)) <= 0.5 || fabs(dsub(sv, v1)) <= 0.5) &&
                    su >= dsub(u0, 0.5) && su <= dadd(u1, 0.5));
  }
  double color[3];
  const int hit = trace(A, su, sv, color);
  if (hit < 0) {
    atomicExch(fail, 1);
    return;
  }
  bool covered = A.sc.surf[hit].is_occluder != 0;
  if (edge) {
    const double offs[4][2] = {{-0.25, -0.25}, {0.25, -0.25}, {-0.25, 0.25}, {0.25, 0.25}};
    double csum[3] = {0.0, 0.0, 0.0}, osum = 0.0;
    for (int q = 0; q < 4; ++q) {
      double c[3];
      const int h = trace(A, dadd(su, offs[q][0]), dadd(sv, offs[q][1]), c);
      if (h < 0) {
        atomicExch(fail, 1);
        return;
      }
      for (int ch = 0; ch < 3; ++ch) csum[ch] = dadd(csum[ch], c[ch]);
      osum = dadd(osum, A.sc.surf[h].is_occluder ? 1.0 : 0.0);
    }
    for (int ch = 0; ch < 3; ++ch) color[ch] = ddiv(csum[ch], 4.0);
    covered = ddiv(osum, 4.0) >= 0.5;
  }
  for (int ch = 0; ch < 3; ++ch) image[p * 3 + ch] = to_u8(color[ch]);
  mask[p] = covered ? 1 : 0;
}

// The reference view's ground truth (synth.py:287-290): the background
// without occluders and its disparity focal * unit_baseline / depth.
__global__ void k_render_background(RenderArgs A, double focal_baseline,
                                    uint8_t* __restrict__ image, float* __restrict__ disparity,
                                    int* __restrict__ fail) {
  const int W = A.sc.width, H = A.sc.height;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)W * H) return;
  double color[3];
  const int hit = trace(A, (double)(p % W), (double)(p / W), color);
  if (hit < 0) {
    atomicExch(fail, 1);
    return;
  }
  for (int ch = 0; ch < 3; ++ch) image[p * 3 + ch] = to_u8(color[ch]);
  disparity[p] = (float)ddiv(focal_baseline, A.sc.surf[hit].depth);
}

// numpy's PCG64 (XSL-RR 128/64): state = state * M + inc, output of the new
// state; random() = (next >> 11) * 2^-53 (numpy pcg64.h / distributions).
typedef unsigned __int128 u128;
__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

__device__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ double pcg_random(u128& state, u128 inc) {
  state = state * pcg_mult() + inc;
  const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
  const unsigned r = (unsigned)(state >> 122);
  const uint64_t out = (x >> r) | (x << ((64u - r) & 63u));
  return (double)(out >> 11) * (1.0 / 9007199254740992.0);
}

constexpr int FLIP_CHUNK = 32;

// synth.py:334-338: exact = 1 - cover; flips = rng.random(shape) < p_flip;
// value = flips ? 1 - exact : exact (0 or 1, kept as an integer)
__global__ void k_prior_flips(const uint8_t* __restrict__ mask, int64_t n, uint64_t s_hi,
                              uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, double p_flip,
                              uint8_t* __restrict__ value) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p0 = c * FLIP_CHUNK;
  if (p0 >= n) return;
  const u128 inc = ((u128)i_hi << 64) | i_lo;
  u128 st = pcg_advance(((u128)s_hi << 64) | s_lo, inc, (uint64_t)p0);
  const int64_t p1 = min(n, p0 + FLIP_CHUNK);
  for (int64_t p = p0; p < p1; ++p) {
    const bool flip = pcg_random(st, inc) < p_flip;
    const uint8_t exact = mask[p] ? 0 : 1;
    value[p] = flip ? (uint8_t)(1 - exact) : exact;
  }
}

// synth.py:314-331 box_blur on 0/1 values: the integral-image sums are exact
// integers, so clipped-window counts reproduce them; tot / count in fp64,
// clip, float32.  Horizontal then vertical window sums.
__global__ void k_blur_rows(const uint8_t* __restrict__ value, int W, int H, int r,
                            int32_t* __restrict__ rowsum) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)W * H) return;
  const int x = (int)(p % W);
  const int64_t row = p - x;
  const int c0 = max(x - r, 0), c1 = min(x + r + 1, W);
  int32_t s = 0;
  for (int c = c0; c < c1; ++c) s += value[row + c];
  rowsum[p] = s;
}

__global__ void k_blur_cols(const int32_t* __restrict__ rowsum, const uint8_t* __restrict__ value,
                            int W, int H, int r, float* __restrict__ prior) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)W * H) return;
  if (r <= 0) {
    prior[p] = (float)value[p];
    return;
  }
  const int x = (int)(p % W), y = (int)(p / W);
  const int r0 = max(y - r, 0), r1 = min(y + r + 1, H);
  const int c0 = max(x - r, 0), c1 = min(x + r + 1, W);
  int64_t tot = 0;
  for (int yy = r0; yy < r1; ++yy) tot += rowsum[(int64_t)yy * W + x];
  const double v = ddiv((double)tot, (double)((int64_t)(r1 - r0) * (c1 - c0)));
  prior[p] = (float)fmin(fmax(v, 0.0), 1.0);
}

int check_scene(const st_scene* sc) {
  if (!sc || sc->width <= 0 || sc->height <= 0 || sc->n_surfaces <= 0 ||
      sc->n_surfaces > ST_MAX_SURFACES) {
    sthost::set_error("st_render: bad scene (size or surface count)");
    return ST_EINVAL;
  }
  return ST_OK;
}

RenderArgs make_args(const st_scene* sc, const double* center, const double* rotation,
                     int with_occluders) {
  RenderArgs A;
  memset(&A, 0, sizeof(A));
  A.sc = *sc;
  for (int i = 0; i < 3; ++i) A.center[i] = center[i];
  for (int i = 0; i < 9; ++i) A.rot[i] = rotation[i];
  A.with_occluders = with_occluders;
  return A;
}

}  // namespace

extern "C" {

int st_render_view(const st_scene* scene, const double* center, const double* rotation,
                   const double* rects_dev, int32_t n_rects, uint8_t* image, uint8_t* mask,
                   int32_t* fail, void* stream) {
  int rc = check_scene(scene);
  if (rc) return rc;
  const int64_t n = (int64_t)scene->width * scene->height;
  const RenderArgs A = make_args(scene, center, rotation, 1);
  k_render_view<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      A, rects_dev, n_rects, image, mask, fail);
  ST_LAUNCH_CHECK("k_render_view");
  return ST_OK;
}

int st_render_background(const st_scene* scene, const double* center, const double* rotation,
                         double focal_baseline, uint8_t* image, float* disparity, int32_t* fail,
                         void* stream) {
  int rc = check_scene(scene);
  if (rc) return rc;
  const int64_t n = (int64_t)scene->width * scene->height;
  const RenderArgs A = make_args(scene, center, rotation, 0);
  k_render_background<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      A, focal_baseline, image, disparity, fail);
  ST_LAUNCH_CHECK("k_render_background");
  return ST_OK;
}

int64_t st_corrupt_prior_workspace(int32_t W, int32_t H) {
  const int64_t n = (int64_t)W * H;
  return ((n + 255) & ~(int64_t)255) + 4 * n;
}

int st_corrupt_prior(const uint8_t* mask, int32_t W, int32_t H, const uint64_t* pcg_state,
                     double p_flip, int32_t blur_radius, float* prior, void* workspace,
                     int64_t workspace_bytes, void* stream) {
  if (W <= 0 || H <= 0 || !pcg_state) {
    sthost::set_error("st_corrupt_prior: bad arguments");
    return ST_EINVAL;
  }
  if (workspace_bytes < st_corrupt_prior_workspace(W, H)) {
    sthost::set_error("st_corrupt_prior: workspace too small");
    return ST_ENOMEM;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = (int64_t)W * H;
  uint8_t* value = (uint8_t*)workspace;
  int32_t* rowsum = (int32_t*)((char*)workspace + ((n + 255) & ~(int64_t)255));
  const int64_t chunks = (n + FLIP_CHUNK - 1) / FLIP_CHUNK;
  k_prior_flips<<<(unsigned)((chunks + 127) / 128), 128, 0, s>>>(
      mask, n, pcg_state[0], pcg_state[1], pcg_state[2], pcg_state[3], p_flip, value);
  ST_LAUNCH_CHECK("k_prior_flips");
  const unsigned g = (unsigned)((n + 255) / 256);
  if (blur_radius > 0) {
    k_blur_rows<<<g, 256, 0, s>>>(value, W, H, blur_radius, rowsum);
    ST_LAUNCH_CHECK("k_blur_rows");
  }
  k_blur_cols<<<g, 256, 0, s>>>(rowsum, value, W, H, blur_radius, prior);
  ST_LAUNCH_CHECK("k_blur_cols");
  return ST_OK;
}

}  // extern "C"
