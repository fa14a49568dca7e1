// Shared device helpers for the seethrough_b200 kernels (sm_100a).
//
// Numerics follow the reference recipe bit for bit where IEEE allows it:
// every fp64 product/sum is an explicit __dmul_rn/__dadd_rn (no FMA
// contraction), evaluation order is the reference's left-to-right order.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/seethrough_b200.h"

#define ST_TW 32  // support tile width  (pixels)
#define ST_TH 8   // support tile height (pixels)

namespace st {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Exact small-integer -> double through the 2^52 magic constant: one DADD
// instead of an I2F conversion.  Valid for -2^31 < x < 2^31.
__device__ __forceinline__ double i2d_exact(int x) {
  return __dsub_rn(__hiloint2double(0x43300000, (unsigned)(x + 0x40000000)),
                   4503600701112320.0);  // 2^52 + 2^30
}
__device__ __forceinline__ double u8d(uint32_t word, int byte) {
  return __dsub_rn(__hiloint2double(0x43300000, __byte_perm(word, 0u, 0x4440 | byte)),
                   4503599627370496.0);  // 2^52
}

// geometry.py:204-219 -- h = A (u, v, 1) + d b, left to right, separate roundings.
struct WarpOut {
  double pu, pv;
  bool front;
};

__device__ __forceinline__ WarpOut warp_ab(const double* a, const double* b, double u, double v,
                                           double d) {
  double hx = dadd(dadd(dadd(dmul(a[0], u), dmul(a[1], v)), a[2]), dmul(d, b[0]));
  double hy = dadd(dadd(dadd(dmul(a[3], u), dmul(a[4], v)), a[5]), dmul(d, b[1]));
  double hz = dadd(dadd(dadd(dmul(a[6], u), dmul(a[7], v)), a[8]), dmul(d, b[2]));
  WarpOut o;
  o.front = hz > 0.0;
  if (hz == 1.0) {  // rectified rigs: x / 1 == x exactly
    o.pu = hx;
    o.pv = hy;
  } else {
    o.pu = ddiv(hx, hz);
    o.pv = ddiv(hy, hz);
  }
  return o;
}

__device__ __forceinline__ WarpOut warp_to(const st_rig& r, int k, double u, double v, double d) {
  return warp_ab(r.warp_a[k], r.warp_b[k], u, v, d);
}

// solver.py:197-204 -- descriptor-support margin test on rig dims.
__device__ __forceinline__ bool in_margin(const st_rig& r, int k, const WarpOut& w) {
  const double m = (double)ST_DESC_MARGIN;
  return w.front && w.pu >= m && w.pu <= (double)(r.view_w[k] - ST_DESC_MARGIN - 1) &&
         w.pv >= m && w.pv <= (double)(r.view_h[k] - ST_DESC_MARGIN - 1);
}

// sampling.py:21-55 tap selection: nan/inf -> 0, clip, floor, min(., n-2).
struct Taps {
  int iu, iv;        // top-left tap
  int su, sv;        // steps to the right / lower tap (0 on 1-px axes)
  double fu, fv;     // fp64 weights
};

__device__ __forceinline__ double clean_coord(double x, double hi) {
  if (!isfinite(x)) x = 0.0;   // nan_to_num(nan=0, posinf=0, neginf=0)
  return fmin(fmax(x, 0.0), hi);
}

__device__ __forceinline__ Taps taps_of(double u, double v, int w, int h) {
  Taps t;
  u = clean_coord(u, (double)w - 1.0);
  v = clean_coord(v, (double)h - 1.0);
  double fiu = w > 1 ? fmin(floor(u), (double)w - 2.0) : 0.0;
  double fiv = h > 1 ? fmin(floor(v), (double)h - 2.0) : 0.0;
  t.fu = dsub(u, fiu);
  t.fv = dsub(v, fiv);
  t.iu = (int)fiu;
  t.iv = (int)fiv;
  t.su = w > 1 ? 1 : 0;
  t.sv = h > 1 ? w : 0;
  return t;
}

// fp64 lerp of fp32 taps with an fp32 tap difference (sampling.py:49-55).
__device__ __forceinline__ double lerp_f32(float g0, float g1, double f) {
  return dadd((double)g0, dmul(f, (double)__fsub_rn(g1, g0)));
}

// One byte channel of a descriptor / colour, exact integer taps.
__device__ __forceinline__ double lerp_u8(int g0, int g1, double f) {
  return dadd(i2d_exact(g0), dmul(f, i2d_exact(g1 - g0)));
}

// Correctly rounded x / n for a small positive integer n with r = RN(1/n):
// q = RN(x r) is faithful, the residual x - q n is exact in one FMA, and
// RN(q + (x - q n) r) is the correctly rounded quotient (Markstein's final
// correction step).  Three DP ops instead of the generic __ddiv_rn sequence;
// st_selftest(1, ...) checks it against __ddiv_rn bit for bit.
__device__ __forceinline__ double div_small(double x, double n, double r) {
  const double q = __dmul_rn(x, r);
  const double e = __fma_rn(-q, n, x);
  return __fma_rn(e, r, q);
}

// prior.py:365-370 -- log(gamma + exp(-z^2/2)), z = (d - mu)/sigma.
// inv_sigma != 0 means sigma is a power of two and the division is an exact
// scaling.
__device__ __forceinline__ double log_prior(double d, double mu, double sigma, double gamma,
                                            double inv_sigma = 0.0) {
  const double dm = dsub(d, mu);
  const double z = inv_sigma != 0.0 ? dmul(dm, inv_sigma) : ddiv(dm, sigma);
  return log(dadd(gamma, exp(dmul(dmul(-0.5, z), z))));
}

// Pruning radius for the M-step: -log prior(d) = -log(gamma + exp(-z^2/2))
// grows with |d - mu|, so it exceeds the incumbent energy `best` exactly when
// |d - mu| > sigma sqrt(-2 ln(exp(-best) - gamma)).  Computed in fp32 once
// per incumbent change; callers prune only beyond the radius plus a margin
// (1e-4 relative + 0.01 absolute) far larger than the fp32 error (the
// argument is kept >= 1e-3, so |d ln x| < 1e-4), and run the exact fp64
// comparison for everything inside it.
__device__ __forceinline__ double prune_radius(double best, float sigma_f, float gamma_f) {
  if (!(best < 1e30)) return INFINITY;
  const float x = expf(-(float)best) - gamma_f;
  if (!(x >= 1e-3f)) return INFINITY;  // nothing prunable (best near -log gamma)
  // best at (or, by fp32 rounding, apparently below) the smallest bound:
  // only candidates within the absolute margin of mu can still tie
  if (x >= 1.0f) return 0.01;
  const float r = sigma_f * sqrtf(-2.0f * logf(x));
  return (double)r * (1.0 + 1e-4) + 0.01;
}

// 16-channel bilinear descriptor sample, fp64 recipe (sampling.py:49-55 on
// the float32 copy of the uint8 map: tap differences are exact integers).
// Calls `sink(c, f)` for each channel in order.
// Four channels of one 32-bit descriptor word pair: exact g0 and g1 - g0 as
// doubles via the 2^52 trick (one PRMT / paired 16-bit SIMD difference + one
// DADD each), then the fp64 lerp g0 + fu * (g1 - g0).
__device__ __forceinline__ void lerp_word(uint32_t wa, uint32_t wb, double fu, double (&f)[4]) {
  const uint32_t ea = wa & 0x00ff00ffu, eb = wb & 0x00ff00ffu;
  const uint32_t oa = (wa >> 8) & 0x00ff00ffu, ob = (wb >> 8) & 0x00ff00ffu;
  const uint32_t de = eb + 0x01000100u - ea;  // bytes 0 and 2: (g1 - g0 + 256) per 16-bit lane
  const uint32_t dodd = ob + 0x01000100u - oa;  // bytes 1 and 3
  const uint32_t lanes[4] = {__byte_perm(de, 0u, 0x4410), __byte_perm(dodd, 0u, 0x4410),
                             __byte_perm(de, 0u, 0x4432), __byte_perm(dodd, 0u, 0x4432)};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double g0 = __dsub_rn(__hiloint2double(0x43300000, __byte_perm(wa, 0u, 0x4440 | j)),
                                4503599627370496.0);          // 2^52
    const double df = __dsub_rn(__hiloint2double(0x43300000, lanes[j]),
                                4503599627370752.0);          // 2^52 + 256
    f[j] = dadd(g0, dmul(fu, df));
  }
}

template <typename Sink>
__device__ __forceinline__ void sample_desc(const uint4* __restrict__ plane, int W, const Taps& t,
                                            Sink&& sink) {
  const size_t base = (size_t)t.iv * W + t.iu;
  const uint4 a = __ldg(plane + base);
  const uint4 b = __ldg(plane + base + t.su);
  const uint32_t aw[4] = {a.x, a.y, a.z, a.w};
  const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
  if (t.fv == 0.0) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      double f[4];
      lerp_word(aw[w], bw[w], t.fu, f);
#pragma unroll
      for (int j = 0; j < 4; ++j) sink(4 * w + j, f[j]);
    }
  } else {
    const uint4 e = __ldg(plane + base + t.sv);
    const uint4 g = __ldg(plane + base + t.sv + t.su);
    const uint32_t ew[4] = {e.x, e.y, e.z, e.w};
    const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int sh = 8 * (c & 3);
      const double top = lerp_u8((aw[c >> 2] >> sh) & 0xff, (bw[c >> 2] >> sh) & 0xff, t.fu);
      const double bot = lerp_u8((ew[c >> 2] >> sh) & 0xff, (gw[c >> 2] >> sh) & 0xff, t.fu);
      sink(c, dadd(top, dmul(t.fv, dsub(bot, top))));
    }
  }
}

__device__ __forceinline__ double variance_ceiling() { return 16.0 * 127.5 * 127.5; }

}  // namespace st

// CUDA error plumbing shared by the host side of every .cu file.
namespace sthost {
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);
void count_launch();
}  // namespace sthost

#define ST_CUDA_CHECK(call)                                       \
  do {                                                            \
    cudaError_t _e = (call);                                      \
    if (_e != cudaSuccess) return sthost::cuda_fail(_e, #call);   \
  } while (0)

// Every kernel launch site is followed by ST_LAUNCH_CHECK: it both checks the
// launch and counts it for st_launch_count().
#define ST_LAUNCH_CHECK(name)                                     \
  do {                                                            \
    sthost::count_launch();                                       \
    cudaError_t _e = cudaGetLastError();                          \
    if (_e != cudaSuccess) return sthost::cuda_fail(_e, name);    \
  } while (0)
