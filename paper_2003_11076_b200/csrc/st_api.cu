// C ABI entry points and the native EM driver (solver.py:436-508).
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <functional>
#include <mutex>
#include <cub/cub.cuh>
#include <vector>

#include "st_common.cuh"
#include "st_em.cuh"

#define ST_VERSION 10000

namespace sthost {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return ST_ECUDA;
}

}  // namespace sthost

namespace {

constexpr int ST_ASYNC_CHUNK = 16;

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

int check_views(int K) {
  if (K > ST_MAX_VIEWS) {
    sthost::set_error("mask enumeration is exponential; refusing %d views (limit %d)", K,
                      ST_MAX_VIEWS);
    return ST_EINVAL;
  }
  if (K < 2) {
    sthost::set_error("a light-field frame needs at least two views");
    return ST_EINVAL;
  }
  return ST_OK;
}

// solver.py:187-192: band offsets nearest-first, coarse sweep length.
int make_ctx(const st_frame* f, const st_rig* rig, const st_params* p, st::EmCtx& c) {
  int rc = check_views(rig->num_views);
  if (rc) return rc;
  memset(&c, 0, sizeof(c));
  c.rig = *rig;
  const int iters = p->forced_iters > 0 ? p->forced_iters : p->max_iters;
  if (iters > ST_MAX_ITERS) {
    sthost::set_error("max_iters %d exceeds the %d iterations the EM statistics hold", iters,
                      ST_MAX_ITERS);
    return ST_EINVAL;
  }
  c.p = *p;
  c.W = rig->width;
  c.H = rig->height;
  c.HW = (int64_t)c.W * c.H;
  c.desc = reinterpret_cast<const uint4*>(f->desc);
  c.priors = f->priors;
  c.mu = f->mu;
  const int jm = (int)floor(2.0 * p->sigma / 0.5 + 1e-12);
  if (2 * jm + 1 > ST_MAX_BAND) {
    sthost::set_error("sigma too large for the candidate band (%d offsets > %d)", 2 * jm + 1,
                      ST_MAX_BAND);
    return ST_EINVAL;
  }
  std::vector<double> band;
  for (int j = -jm; j <= jm; ++j) band.push_back(0.5 * j);
  std::stable_sort(band.begin(), band.end(), [](double a, double b) {
    return fabs(a) < fabs(b) || (fabs(a) == fabs(b) && a < b);
  });
  c.n_band = (int)band.size();
  for (int j = 0; j < c.n_band; ++j) c.band[j] = band[j];
  // len(np.arange(1.0, d_max + 1e-9, 4.0))
  const double span = ceil(((p->d_max + 1e-9) - 1.0) / 4.0);
  c.n_coarse = span > 0 ? (int)span : 0;
  c.sup_tile_start = f->sup_tile_start;
  c.sup_value = f->sup_value;
  c.sup_mask = f->sup_mask;
  c.tiles_x = (c.W + ST_TW - 1) / ST_TW;
  c.sup_ir = (int)floor(p->neighborhood_radius);
  c.sup_r2 = p->neighborhood_radius * p->neighborhood_radius;
  int ex = 0;
  const double mant = frexp(p->sigma, &ex);
  c.inv_sigma = (p->sigma > 0 && mant == 0.5) ? 1.0 / p->sigma : 0.0;  // exact scaling
  c.sigma_f = (float)p->sigma;
  c.gamma_f = (float)p->gamma;
  // rectified rig: h = (u + d bx, v, 1) exactly (the general left-to-right
  // formula reduces to these roundings when A = I and b_y = b_z = 0)
  c.rectified = 1;
  for (int k = 0; k < rig->num_views; ++k) {
    const double* a = rig->warp_a[k];
    const double* b = rig->warp_b[k];
    const bool eye = a[0] == 1.0 && a[1] == 0.0 && a[2] == 0.0 && a[3] == 0.0 && a[4] == 1.0 &&
                     a[5] == 0.0 && a[6] == 0.0 && a[7] == 0.0 && a[8] == 1.0;
    if (!eye || b[1] != 0.0 || b[2] != 0.0 || !(fabs(b[0]) < 1e300)) c.rectified = 0;
  }
  for (int n = 0; n <= ST_MAX_VIEWS; ++n) c.recip[n] = n ? 1.0 / (double)n : 0.0;
  // the M-step tap cache holds 32-bit descriptor indices
  if ((double)rig->num_views * (double)c.HW >= 4294967295.0) c.rectified = 0;
  c.view_bits = (uint32_t)((1u << rig->num_views) - 1u);
  // cross-check: evaluate every candidate (no pruning; same winner)
  c.exhaustive = getenv("ST_MSTEP_EXHAUSTIVE") != nullptr;
  return ST_OK;
}

unsigned blocks_for(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// Optional CUDA-event brackets around the solve's kernels (st_params.timing).
struct EventSet {
  bool on;
  cudaEvent_t e[6];
  explicit EventSet(bool enable) : on(enable) {
    if (on)
      for (auto& x : e) cudaEventCreate(&x);
  }
  ~EventSet() {
    if (on)
      for (auto& x : e) cudaEventDestroy(x);
  }
  void record(int i, cudaStream_t s) {
    if (on) cudaEventRecord(e[i], s);
  }
  double ms(int a, int b) {
    if (!on) return 0.0;
    float t = 0.f;
    cudaEventElapsedTime(&t, e[a], e[b]);
    return (double)t;
  }
};

int estep_smem(int K) { return ESTEP_BLOCK * K * 16 * (int)sizeof(double); }

// The opt-in above 48 KB of dynamic shared memory is a per-device function
// attribute: set once per device (K >= 7 E-step launches need it).
int prepare_estep_kernels() {
  static std::mutex mu;
  static uint64_t prepared = 0;  // bit d: device d done
  int dev = 0;
  ST_CUDA_CHECK(cudaGetDevice(&dev));
  const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
  std::lock_guard<std::mutex> lock(mu);
  if (bit && (prepared & bit)) return ST_OK;
  const int max_smem = estep_smem(ST_MAX_VIEWS);
  ST_CUDA_CHECK(cudaFuncSetAttribute(st::k_e_step_at,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
  ST_CUDA_CHECK(cudaFuncSetAttribute(st::k_e_step_rays,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
  prepared |= bit;
  return ST_OK;
}

// E-step launch: the register-resident screened kernel for K <= 5 views
// (templated on K and on the rectified-rig shortcut), the shared-memory
// enumeration for larger rigs.  `n` bounds the rows (list or dense).
template <int K>
void launch_taps(unsigned blocks, cudaStream_t s, const st::EmCtx& c, const st::EStepArgs& a) {
  if (c.rectified)
    st::k_e_step_taps<K, true><<<blocks, ESTEP_TAPS_BLOCK, 0, s>>>(c, a);
  else
    st::k_e_step_taps<K, false><<<blocks, ESTEP_TAPS_BLOCK, 0, s>>>(c, a);
}

template <int K>
void launch_cert(unsigned blocks, cudaStream_t s, const st::EmCtx& c, const st::EStepArgs& a) {
  if (c.rectified)
    st::k_e_step_cert<K, true><<<blocks, ESTEP_CERT_BLOCK, 0, s>>>(c, a);
  else
    st::k_e_step_cert<K, false><<<blocks, ESTEP_CERT_BLOCK, 0, s>>>(c, a);
}

// With a fallback list (args.flist, K <= 5): the certificate pass
// (k_e_step_cert) decides most rows without any fp64 score; the rows it
// cannot certify go through the screened kernel, one grid-stride wave.
void launch_e_step(int K, int64_t n, cudaStream_t s, const st::EmCtx& c,
                   const st::EStepArgs& args, bool count_cleared = false) {
  const bool exhaustive = getenv("ST_ESTEP_EXHAUSTIVE") != nullptr;  // cross-check
  st::EStepArgs a = args;
  a.exhaustive = exhaustive ? 1 : 0;
  if (a.flist && !exhaustive) {
    if (!count_cleared) cudaMemsetAsync(a.flist_count, 0, sizeof(uint32_t), s);
    const unsigned bc = blocks_for(n, ESTEP_CERT_BLOCK);
    switch (K) {
      case 2: launch_cert<2>(bc, s, c, a); break;
      case 3: launch_cert<3>(bc, s, c, a); break;
      case 4: launch_cert<4>(bc, s, c, a); break;
      case 5: launch_cert<5>(bc, s, c, a); break;
      default:  // 6 <= K <= 12: enumerated bounds, branch-and-bound fallback
        if (c.rectified)
          st::k_e_step_cert_big<true><<<bc, CERT_BIG_BLOCK, 0, s>>>(c, a);
        else
          st::k_e_step_cert_big<false><<<bc, CERT_BIG_BLOCK, 0, s>>>(c, a);
        break;
    }
    sthost::count_launch();
    if (getenv("ST_ESTEP_STATS")) {  // diagnostics: rows left for the fallback (synchronises)
      uint32_t nf = 0;
      cudaMemcpyAsync(&nf, a.flist_count, sizeof(nf), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      fprintf(stderr, "e-step certificate: %u rows to the fallback\n", nf);
    }
    a.list = a.flist;
    a.list_count = a.flist_count;
    n = std::min<int64_t>(n, K <= 5 ? 148 * ESTEP_MIN_BLOCKS * ESTEP_TAPS_BLOCK
                                     : 148 * 8 * ESTEP_BLOCK);
  }
  const unsigned bt = blocks_for(n, ESTEP_TAPS_BLOCK);
  switch (K) {
    case 2: launch_taps<2>(bt, s, c, a); break;
    case 3: launch_taps<3>(bt, s, c, a); break;
    case 4: launch_taps<4>(bt, s, c, a); break;
    case 5: launch_taps<5>(bt, s, c, a); break;
    default:
      // (ST_ESTEP_SMEM: the shared-memory ray staging, for cross-checks)
      if (c.rectified && !a.exhaustive && getenv("ST_ESTEP_SMEM") == nullptr)
        st::k_e_step_at_taps<<<blocks_for(n, ESTEP_BLOCK), ESTEP_BLOCK, 0, s>>>(c, a);
      else
        st::k_e_step_at<<<blocks_for(n, ESTEP_BLOCK), ESTEP_BLOCK, estep_smem(K), s>>>(c, a);
      break;
  }
}

// M-step launch: one thread per slot (`grid_slots`: slots the grid must
// cover; a wave of grid-stride blocks for worklists).
unsigned mstep_blocks(const st::EmCtx&, int64_t grid_slots) {
  return blocks_for(std::max<int64_t>(grid_slots, 1), EM_BLOCK);
}

void launch_m_step(const st::EmCtx& c, const st::MStepArgs& a, unsigned grid, cudaStream_t s) {
  st::k_m_step<<<grid, EM_BLOCK, 0, s>>>(c, a);
}

}  // namespace

namespace st {

__global__ void k_bilinear(const float* __restrict__ plane, int h, int w, int c,
                           const double* __restrict__ u, const double* __restrict__ v, int64_t n,
                           double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Taps t = taps_of(u[i], v[i], w, h);
  const size_t b = ((size_t)t.iv * w + t.iu) * c;
  const size_t bu = b + (size_t)t.su * c, bv = b + (size_t)t.sv * c, bvu = bu + (size_t)t.sv * c;
  for (int ch = 0; ch < c; ++ch) {
    double top = lerp_f32(plane[b + ch], plane[bu + ch], t.fu);
    if (t.fv != 0.0) {
      const double bot = lerp_f32(plane[bv + ch], plane[bvu + ch], t.fu);
      top = dadd(top, dmul(t.fv, dsub(bot, top)));
    }
    out[(size_t)i * c + ch] = top;
  }
}

__global__ void k_warp(st_rig rig, int k, const double* __restrict__ u,
                       const double* __restrict__ v, const double* __restrict__ d, int64_t n,
                       double* __restrict__ pu, double* __restrict__ pv, uint8_t* __restrict__ ok) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* a = rig.warp_a[k];
  const double* b = rig.warp_b[k];
  const double uu = u[i], vv = v[i], dd = d[i];
  const double hx = dadd(dadd(dadd(dmul(a[0], uu), dmul(a[1], vv)), a[2]), dmul(dd, b[0]));
  const double hy = dadd(dadd(dadd(dmul(a[3], uu), dmul(a[4], vv)), a[5]), dmul(dd, b[1]));
  const double hz = dadd(dadd(dadd(dmul(a[6], uu), dmul(a[7], vv)), a[8]), dmul(dd, b[2]));
  pu[i] = ddiv(hx, hz);
  pv[i] = ddiv(hy, hz);
  ok[i] = hz > 0.0 ? 1 : 0;
}

// Self-test of div_small against __ddiv_rn: x spans many binades and
// integer-valued / half-integer patterns, n = 1..12.
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_selftest_div(int64_t n, unsigned long long seed,
                               unsigned long long* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long h = mix64(seed ^ (unsigned long long)i);
  double x;
  const int kind = (int)(h & 3);
  if (kind == 0) {
    // random mantissa, exponent in [-60, 60]
    const unsigned long long m = (h >> 12) | 0x3ff0000000000000ull;
    x = ldexp(__longlong_as_double((long long)m) - 1.0 + 1.0, (int)((h >> 2) & 127) - 63);
  } else if (kind == 1) {
    x = (double)(long long)(h >> 20);  // large integers
  } else if (kind == 2) {
    x = (double)((h >> 40) & 0xffffff) * 0.5;  // half integers
  } else {
    x = __longlong_as_double((long long)((h >> 2) & 0x7fefffffffffffffull));  // any finite
    if (fabs(x) < 1e-300 || fabs(x) > 1e300) x = 1.0 + (double)(h & 0xffff);
  }
  for (int k = 1; k <= 12; ++k) {
    const double want = __ddiv_rn(x, (double)k);
    const double got = div_small(x, (double)k, 1.0 / (double)k);
    if (__double_as_longlong(want) != __double_as_longlong(got) && !(want == 0.0 && got == 0.0))
      atomicAdd(bad, 1ull);
  }
}

// FP64 throughput probe: 8 independent DFMA chains per thread (the pipe's
// latency hidden), 2 flops per DFMA.  Output kept live through `sink`.
__global__ void __launch_bounds__(256) k_fp64_peak(int iters, double seed, double* sink) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed + threadIdx.x * 1e-9 + j;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __fma_rn(a[j], m, c);
  }
  double t = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += a[j];
  if (t == 12345.678) *sink = t;
}

}  // namespace st

extern "C" {

int st_fp64_peak(double* tflops, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  double* sink = nullptr;
  ST_CUDA_CHECK(cudaMallocAsync(&sink, sizeof(double), s));
  cudaEvent_t e0, e1;
  ST_CUDA_CHECK(cudaEventCreate(&e0));
  ST_CUDA_CHECK(cudaEventCreate(&e1));
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  st::k_fp64_peak<<<blocks, threads, 0, s>>>(64, 1.0, sink);  // warm-up
  ST_LAUNCH_CHECK("k_fp64_peak");
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, s);
    st::k_fp64_peak<<<blocks, threads, 0, s>>>(iters, 1.0 + r, sink);
    ST_LAUNCH_CHECK("k_fp64_peak");
    cudaEventRecord(e1, s);
    ST_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ST_CUDA_CHECK(cudaFreeAsync(sink, s));
  ST_CUDA_CHECK(cudaStreamSynchronize(s));
  *tflops = 2.0 * 8.0 * (double)iters * blocks * threads / (best * 1e-3) / 1e12;
  return ST_OK;
}

int st_selftest(int32_t which, int64_t n, uint64_t seed, int64_t* mismatches, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (which != 1) {
    sthost::set_error("unknown self-test %d", which);
    return ST_EINVAL;
  }
  unsigned long long* bad = nullptr;
  ST_CUDA_CHECK(cudaMallocAsync(&bad, sizeof(*bad), s));
  ST_CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(*bad), s));
  st::k_selftest_div<<<blocks_for(n, 256), 256, 0, s>>>(n, seed, bad);
  ST_LAUNCH_CHECK("k_selftest_div");
  unsigned long long h = 0;
  ST_CUDA_CHECK(cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, s));
  ST_CUDA_CHECK(cudaFreeAsync(bad, s));
  ST_CUDA_CHECK(cudaStreamSynchronize(s));
  *mismatches = (int64_t)h;
  return ST_OK;
}

const char* st_last_error(void) { return sthost::g_err; }

int64_t st_struct_size(int32_t which) {
  switch (which) {
    case 0: return (int64_t)sizeof(st_rig);
    case 1: return (int64_t)sizeof(st_params);
    case 2: return (int64_t)sizeof(st_stats);
    case 3: return (int64_t)sizeof(st_frame);
    case 4: return (int64_t)sizeof(st_tri);
    case 5: return (int64_t)sizeof(st_cams);
    case 6: return (int64_t)sizeof(st_frame_plan);
    case 7: return (int64_t)sizeof(st_scene);
    default: return -1;
  }
}
int st_version(void) { return ST_VERSION; }
int64_t st_launch_count(void) { return sthost::g_launches.load(); }

int st_device_count(void) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    sthost::cuda_fail(e, "cudaGetDeviceCount");
    return 0;
  }
  return n;
}

int st_bilinear(const float* plane, int32_t h, int32_t w, int32_t c, const double* u,
                const double* v, int64_t n, double* out, void* stream) {
  if (n <= 0) return ST_OK;
  st::k_bilinear<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(plane, h, w, c, u, v, n,
                                                                        out);
  ST_LAUNCH_CHECK("k_bilinear");
  return ST_OK;
}

int st_warp(const st_rig* rig, int32_t k, const double* u, const double* v, const double* d,
            int64_t n, double* pu, double* pv, uint8_t* ok, void* stream) {
  if (k < 0 || k >= rig->num_views) {
    sthost::set_error("view index %d out of range", k);
    return ST_EINVAL;
  }
  if (n <= 0) return ST_OK;
  st::k_warp<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*rig, k, u, v, d, n, pu, pv,
                                                                    ok);
  ST_LAUNCH_CHECK("k_warp");
  return ST_OK;
}

int st_initial_masks(const st_frame* f, const st_rig* rig, const st_params* p, const int64_t* pix,
                     int64_t n, uint32_t* static_out, uint32_t* valid_out, void* stream) {
  st::EmCtx c;
  int rc = make_ctx(f, rig, p, c);
  if (rc) return rc;
  if (!pix) n = c.HW;
  if (n <= 0) return ST_OK;
  st::k_initial_masks<<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(c, pix, n, static_out,
                                                                             valid_out);
  ST_LAUNCH_CHECK("k_initial_masks");
  return ST_OK;
}

int st_gather_rays(const st_frame* f, const st_rig* rig, const int64_t* pix, const double* d,
                   int64_t n, double* desc, uint8_t* valid, double* q, void* stream) {
  st::EmCtx c;
  st_params p = {};
  p.sigma = 1.0;
  int rc = make_ctx(f, rig, &p, c);
  if (rc) return rc;
  if (n <= 0) return ST_OK;
  st::k_gather_rays<<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(c, pix, d, n, desc,
                                                                           valid, q);
  ST_LAUNCH_CHECK("k_gather_rays");
  return ST_OK;
}

int st_energy(const st_frame* f, const st_rig* rig, const st_params* p, const int64_t* pix,
              const double* d, const uint32_t* bits, int64_t n, double* energy, uint8_t* real,
              void* stream) {
  st::EmCtx c;
  int rc = make_ctx(f, rig, p, c);
  if (rc) return rc;
  if (n <= 0) return ST_OK;
  st::k_energy<<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(c, pix, d, bits, n, energy,
                                                                      real);
  ST_LAUNCH_CHECK("k_energy");
  return ST_OK;
}

int st_m_step(const st_frame* f, const st_rig* rig, const st_params* p, const int64_t* active,
              int64_t n, const uint32_t* static_all, double* d_out, double* e_out,
              uint8_t* status_out, void* stream) {
  st::EmCtx c;
  int rc = make_ctx(f, rig, p, c);
  if (rc) return rc;
  if (!active) n = c.HW;
  if (n <= 0) return ST_OK;
  st::MStepArgs a = {};
  a.active = active;
  a.n = n;
  a.static_all = static_all;
  a.first = 1;
  a.d = d_out;
  a.e = e_out;
  a.status = status_out;
  launch_m_step(c, a, mstep_blocks(c, n), (cudaStream_t)stream);
  ST_LAUNCH_CHECK("k_m_step");
  return ST_OK;
}

int st_e_step_at(const st_frame* f, const st_rig* rig, const st_params* p, const int64_t* pix,
                 const double* d, int64_t n, uint32_t* static_out, uint32_t* valid_out,
                 void* stream) {
  st::EmCtx c;
  int rc = make_ctx(f, rig, p, c);
  if (rc) return rc;
  if ((rc = prepare_estep_kernels())) return rc;
  if (!pix) n = c.HW;
  if (n <= 0) return ST_OK;
  st::EStepArgs a = {};
  a.pix = pix;
  a.n = n;
  a.d = d;
  a.static_out = static_out;
  a.valid_out = valid_out;
  a.scatter = 0;
  launch_e_step(rig->num_views, n, (cudaStream_t)stream, c, a);
  ST_LAUNCH_CHECK("k_e_step_at");
  return ST_OK;
}

int st_e_step(const double* desc, const uint8_t* valid, const double* q, int64_t n, int32_t K,
              const st_params* p, uint32_t* out, void* stream) {
  int rc = check_views(K);
  if (rc) return rc;
  if ((rc = prepare_estep_kernels())) return rc;
  if (n <= 0) return ST_OK;
  st::k_e_step_rays<<<blocks_for(n, ESTEP_BLOCK), ESTEP_BLOCK, estep_smem(K),
                      (cudaStream_t)stream>>>(desc, valid, q, n, K, *p, out);
  ST_LAUNCH_CHECK("k_e_step_rays");
  return ST_OK;
}

int st_masked_variance(const double* desc, const uint8_t* mask, int64_t n, int32_t K, double* out,
                       void* stream) {
  if (n <= 0) return ST_OK;
  st::k_masked_variance<<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(desc, mask, n, K,
                                                                               out);
  ST_LAUNCH_CHECK("k_masked_variance");
  return ST_OK;
}

// ---------------------------------------------------------------------------
// fused solve

struct SolveLayout {
  size_t d, e, pe, st_act, chg, mask_in, mlist, elist, counts, flist, active, flags, offs,
      work, parts, reduced, cub, pw_scratch, pw_val, total;
  size_t cub_bytes;
  int max_warps;
};

static SolveLayout solve_layout(int W, int H) {
  SolveLayout L;
  const int64_t npx = (int64_t)W * H;
  L.max_warps = (int)blocks_for(npx, EM_BLOCK) * (EM_BLOCK / 32);
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                (int)(npx + 1));
  L.cub_bytes = scan_bytes;
  size_t o = 0;
  L.d = o;        o += align_up(sizeof(double) * npx);
  L.e = o;        o += align_up(sizeof(double) * npx);
  L.pe = o;       o += align_up(sizeof(double) * npx);
  L.st_act = o;   o += align_up(npx);
  L.chg = o;      o += align_up(npx);
  L.mask_in = o;  o += align_up(sizeof(uint32_t) * npx);
  L.mlist = o;    o += align_up(sizeof(int32_t) * npx);
  L.elist = o;    o += align_up(sizeof(int32_t) * npx);
  L.counts = o;   o += align_up(sizeof(uint32_t) * 4 + sizeof(double) * 4 + 16);  // worklist counts, stop flag, eps logs, fallback count
  L.flist = o;    o += align_up(sizeof(int32_t) * npx);
  L.active = o;   o += align_up(sizeof(int64_t) * npx);
  L.flags = o;    o += align_up(sizeof(uint32_t) * (npx + 1));
  L.offs = o;     o += align_up(sizeof(uint32_t) * (npx + 1));
  L.work = o;     o += align_up(sizeof(st::Partial) * L.max_warps);
  L.parts = o;    o += align_up(sizeof(st::Partial) * L.max_warps);
  L.reduced = o;  o += align_up(sizeof(st::Partial) * (ST_MAX_ITERS + 2));
  L.cub = o;      o += align_up(L.cub_bytes);
  L.pw_scratch = o; o += align_up(sizeof(double) * npx);
  L.pw_val = o;   o += align_up(sizeof(double) * st::pw_val_size(npx));
  L.total = o;
  return L;
}

int64_t st_solve_workspace(int32_t W, int32_t H, int32_t K) {
  (void)K;
  return (int64_t)solve_layout(W, H).total;
}

int st_solve(const st_frame* f, const st_rig* rig, const st_params* p, int32_t dynamic_only,
             const uint8_t* active_mask, float* values, uint8_t* status, uint32_t* static_bits,
             uint32_t* valid_bits, st_stats* stats, void* workspace, int64_t workspace_bytes,
             st_reduce_fn reduce, void* reduce_user, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  st::EmCtx c;
  int rc = make_ctx(f, rig, p, c);
  if (rc) return rc;
  if ((rc = prepare_estep_kernels())) return rc;
  const int W = c.W, H = c.H;
  const int64_t npx = c.HW;
  const SolveLayout L = solve_layout(W, H);
  if ((int64_t)L.total > workspace_bytes) {
    sthost::set_error("solve workspace too small (%lld < %lld)", (long long)workspace_bytes,
                      (long long)L.total);
    return ST_ENOMEM;
  }
  char* ws = (char*)workspace;
  double* d_act = (double*)(ws + L.d);
  double* e_act = (double*)(ws + L.e);
  double* pe_act = (double*)(ws + L.pe);
  uint8_t* st_act = (uint8_t*)(ws + L.st_act);
  uint8_t* chg = (uint8_t*)(ws + L.chg);
  uint32_t* mask_in = (uint32_t*)(ws + L.mask_in);
  int32_t* mlist = (int32_t*)(ws + L.mlist);
  int32_t* elist = (int32_t*)(ws + L.elist);
  uint32_t* counts = (uint32_t*)(ws + L.counts);
  int64_t* active = (int64_t*)(ws + L.active);
  uint32_t* flags = (uint32_t*)(ws + L.flags);
  uint32_t* offs = (uint32_t*)(ws + L.offs);
  st::Partial* work = (st::Partial*)(ws + L.work);
  st::Partial* parts = (st::Partial*)(ws + L.parts);
  st::Partial* reduced = (st::Partial*)(ws + L.reduced);

  memset(stats, 0, sizeof(*stats));
  stats->converged_after = -1;
  EventSet ev(p->timing != 0);
  // the stats kernel's block counter (word 13) starts at zero
  ST_CUDA_CHECK(cudaMemsetAsync(counts + 12, 0, 4 * sizeof(uint32_t), s));
  double* eps_logs = (double*)(counts + 4);
  st::k_eps_logs<<<1, 32, 0, s>>>(p->epsilon_prior, eps_logs);
  ST_LAUNCH_CHECK("k_eps_logs");

  // initial masks for every pixel at the surface disparity (solver.py:455)
  ev.record(4, s);
  st::k_initial_masks<<<blocks_for(npx, 128), 128, 0, s>>>(c, nullptr, npx, static_bits,
                                                           valid_bits);
  ST_LAUNCH_CHECK("k_initial_masks");
  ev.record(5, s);
  stats->kernel_launches[2] += 1;

  // active set (solver.py:447-452)
  const bool dense = !dynamic_only && !active_mask;
  int64_t n_act = npx;
  if (!dense) {
    const float* ref_prior = f->priors + (size_t)rig->ref_index * npx;
    st::k_flag_active<<<blocks_for(npx, 256), 256, 0, s>>>(ref_prior, active_mask, npx,
                                                          p->threshold, flags, 0, npx);
    ST_LAUNCH_CHECK("k_flag_active");
    ST_CUDA_CHECK(cudaMemsetAsync(flags + npx, 0, sizeof(uint32_t), s));
    size_t tb = L.cub_bytes;
    ST_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ws + L.cub, tb, flags, offs, (int)(npx + 1), s));
    sthost::count_launch();
    st::k_scatter_active<<<blocks_for(npx, 256), 256, 0, s>>>(flags, offs, npx, active);
    ST_LAUNCH_CHECK("k_scatter_active");
    uint32_t cnt = 0;
    ST_CUDA_CHECK(cudaMemcpyAsync(&cnt, offs + npx, sizeof(cnt), cudaMemcpyDeviceToHost, s));
    ST_CUDA_CHECK(cudaStreamSynchronize(s));
    n_act = cnt;
  }
  stats->active_pixels = n_act;
  const int64_t* act_ptr = dense ? nullptr : active;

  // global active count across shards (for changed_fraction)
  double n_act_global = (double)n_act;
  if (reduce) {
    double v = n_act_global;
    if (reduce(&v, 1, reduce_user)) {
      sthost::set_error("shard reduction failed");
      return ST_EINVAL;
    }
    n_act_global = v;
  }

  const int iters = p->forced_iters > 0 ? p->forced_iters : p->max_iters;
  // worklist counts start cleared even on a shard whose band has no active pixel
  ST_CUDA_CHECK(cudaMemsetAsync(counts, 0, 2 * sizeof(uint32_t), s));
  const int nblk = (int)blocks_for(n_act, EM_BLOCK);
  bool solved = false;
  for (int it = 1; it <= iters; ++it) {
    if (n_act_global == 0) {
      stats->converged_after = 0;
      break;
    }
    stats->iterations_run = it;
    if (n_act > 0) {
      // Incremental EM (see k_m_step): iteration 1 solves every slot; later
      // iterations re-solve only slots whose mask changed, and re-run the
      // E-step only where d changed.  Both steps are pure per-pixel
      // functions of those inputs, so the result is bit-identical to a
      // full recomputation.
      ST_CUDA_CHECK(cudaMemsetAsync(counts, 0, 2 * sizeof(uint32_t), s));
      ev.record(0, s);
      if (it > 1) {
        st::k_flag_mstep<<<nblk, EM_BLOCK, 0, s>>>(act_ptr, n_act, 0, static_bits, mask_in, e_act,
                                                   pe_act, chg, mlist, counts);
        ST_LAUNCH_CHECK("k_flag_mstep");
      }
      st::MStepArgs a = {};
      a.active = act_ptr;
      a.n = n_act;
      a.list = it > 1 ? mlist : nullptr;
      a.list_count = counts;
      a.static_all = static_bits;
      a.first = it == 1;
      a.d = d_act;
      a.e = e_act;
      a.status = st_act;
      a.mask_in = mask_in;
      a.pe = pe_act;
      a.chg = chg;
      a.elist = elist;
      a.elist_count = counts + 1;
      a.partials = work;
      launch_m_step(c, a, mstep_blocks(c, n_act), s);
      ST_LAUNCH_CHECK("k_m_step");
      ev.record(1, s);
      st::EStepArgs e = {};
      e.pix = act_ptr;
      e.n = n_act;
      e.list = elist;
      e.list_count = counts + 1;
      e.d = d_act;
      e.status = st_act;
      e.static_out = static_bits;
      e.valid_out = valid_bits;
      e.scatter = 1;
      e.eps_logs = eps_logs;
      e.flist = (int32_t*)(ws + L.flist);
      e.flist_count = (uint32_t*)(eps_logs + 4);
      launch_e_step(rig->num_views, n_act, s, c, e);
      ST_LAUNCH_CHECK("k_e_step_at");
      ev.record(2, s);
      // statistics in numpy's summation order, folded by the last block into
      // reduced[it] (the host loop reads the worklist counts itself)
      st::StatsTail tail = {};
      tail.on = 1;
      tail.it = it;
      tail.done = counts + 13;
      tail.reduced = reduced;
      tail.counts = counts;
      tail.record_only = 1;
      tail.keep_counts = 1;
      tail.record_n_act = n_act;
      tail.record_slots = n_act;
      tail.pw_depth = st::stats_depth(n_act);
      tail.pw_scratch = (double*)(ws + L.pw_scratch);
      tail.pw_val = (double*)(ws + L.pw_val);
      st::k_em_stats<<<1 << tail.pw_depth, STATS_BLOCK, 0, s>>>(
          n_act, it > 1, e_act, pe_act, chg, work,
          (int)mstep_blocks(c, n_act) * (EM_BLOCK / 32), parts, nullptr, tail);
      ST_LAUNCH_CHECK("k_em_stats");
      ev.record(3, s);
      stats->kernel_launches[0] += 1;
      stats->kernel_launches[1] += 1;
      stats->kernel_launches[3] += it > 1 ? 3 : 2;
      solved = true;
    } else {
      ST_CUDA_CHECK(cudaMemsetAsync(reduced + it, 0, sizeof(st::Partial), s));
    }
    st::Partial r;
    uint32_t work_counts[2] = {0, 0};
    ST_CUDA_CHECK(cudaMemcpyAsync(&r, reduced + it, sizeof(r), cudaMemcpyDeviceToHost, s));
    ST_CUDA_CHECK(cudaMemcpyAsync(work_counts, counts, sizeof(work_counts),
                                  cudaMemcpyDeviceToHost, s));
    ST_CUDA_CHECK(cudaStreamSynchronize(s));
    stats->msteps += it > 1 ? work_counts[0] : n_act;
    stats->esteps += work_counts[1];
    if (it > 1) stats->prev_evals += work_counts[0];
    if (n_act > 0) {
      stats->kernel_ms[0] += ev.ms(0, 1);
      stats->kernel_ms[1] += ev.ms(1, 2);
      stats->kernel_ms[3] += ev.ms(2, 3);
    }
    if (it == 1) stats->kernel_ms[2] += ev.ms(4, 5);
    double v[7] = {r.sum_e, (double)r.n_fin, r.sum_pe, (double)r.n_pfin, (double)r.n_changed,
                   (double)r.n_cand, (double)r.n_eval};
    if (reduce && reduce(v, 7, reduce_user)) {
      sthost::set_error("shard reduction failed");
      return ST_EINVAL;
    }
    stats->mean_energy[it - 1] = v[1] > 0 ? v[0] / v[1] : NAN;
    stats->candidates_total += (int64_t)v[5];
    stats->energy_evals += (int64_t)v[6];
    stats->hopeless_msteps += r.n_hopeless;  // (diagnostics, this rank only)
    stats->energy_samples += r.n_samples;
    if (it > 1) {
      stats->prev_energy[it - 2] = v[3] > 0 ? v[2] / v[3] : NAN;
      const double changed = v[4] / n_act_global;
      stats->changed_fraction[it - 2] = changed;
      if (p->forced_iters <= 0 && changed < 1e-3) {
        stats->converged_after = it - 1;
        break;
      }
    }
  }

  // outputs (solver.py:491-500)
  if (dense) {
    st::k_pack_outputs<<<blocks_for(npx, 256), 256, 0, s>>>(
        f->mu, npx, 0, nullptr, npx, solved ? d_act : nullptr, st_act, values, status, 1);
    ST_LAUNCH_CHECK("k_pack_outputs");
  } else {
    st::k_fill_mu<<<blocks_for(npx, 256), 256, 0, s>>>(f->mu, npx, values, status);
    ST_LAUNCH_CHECK("k_fill_mu");
    if (solved && n_act > 0) {
      st::k_pack_outputs<<<blocks_for(n_act, 256), 256, 0, s>>>(f->mu, npx, 0, active, n_act, d_act,
                                                                st_act, values, status, 0);
      ST_LAUNCH_CHECK("k_pack_outputs");
    }
  }
  return ST_OK;
}

namespace {

// Iterations >= 3 as a CUDA graph: a WHILE conditional node whose body is
// one iteration's launches, captured once per argument set (TailGraphKey)
// and cached.  The statistics kernel keeps the iteration count on the device
// (counts[14]) and sets the loop condition.
struct TailGraphFields {
  cudaGraphConditionalHandle cond;
};

struct TailGraphKey {
  st::EmCtx c;
  const int64_t* active;
  int64_t n, cnt_lo, cnt_hi;
  const uint32_t* static_bits;
  const uint32_t* valid_bits;
  const st_stats* stats;
  const char* ws;
  const int32_t* mu_unsafe;
  const uint32_t* n_dev;
  int band, forced_iters, iters, wave_env, device;
};

struct TailGraph {
  TailGraphKey key;
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  long long launches;  // kernels per body run
  unsigned long long used;
};

constexpr size_t TAIL_GRAPH_CAP = 32;
std::mutex g_tail_mu;
std::vector<TailGraph>* g_tail = new std::vector<TailGraph>();  // (never freed: exit order)
unsigned long long g_tail_tick = 0;
std::atomic<long long> g_tail_builds{0};
std::atomic<long long> g_tail_launches{0};

// ST_NO_GRAPH: the plain launch loop.  The E-step's diagnostic / cross-check
// switches (launch_e_step) are read per launch, so they disable the graph.
bool tail_graphs_enabled() {
  return !getenv("ST_NO_GRAPH") && !getenv("ST_ESTEP_STATS") && !getenv("ST_ESTEP_EXHAUSTIVE") &&
         !getenv("ST_ESTEP_SMEM");
}

void destroy_tail_graph(TailGraph& t) {
  if (t.exec) cudaGraphExecDestroy(t.exec);  // (freed once in-flight launches finish)
  if (t.graph) cudaGraphDestroy(t.graph);
  t.exec = nullptr;
  t.graph = nullptr;
}

using TailBody = std::function<int(const TailGraphFields*, cudaStream_t)>;

int build_tail_graph(TailGraph& t, const TailBody& body_fn) {
  TailGraphFields fields;
  ST_CUDA_CHECK(cudaGraphCreate(&t.graph, 0));
  ST_CUDA_CHECK(cudaGraphConditionalHandleCreate(&fields.cond, t.graph, 1u,
                                                 cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = fields.cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  ST_CUDA_CHECK(cudaGraphAddNode(&node, t.graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaStream_t cs;
  ST_CUDA_CHECK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaError_t e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                                cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaStreamDestroy(cs);
    return sthost::cuda_fail(e, "cudaStreamBeginCaptureToGraph");
  }
  const long long l0 = sthost::g_launches.load();
  const int rc = body_fn(&fields, cs);
  t.launches = sthost::g_launches.load() - l0;
  sthost::g_launches.fetch_sub(t.launches);  // (counted per graph launch instead)
  cudaGraph_t captured = nullptr;
  e = cudaStreamEndCapture(cs, &captured);
  cudaStreamDestroy(cs);
  if (rc) return rc;
  if (e != cudaSuccess) return sthost::cuda_fail(e, "cudaStreamEndCapture");
  ST_CUDA_CHECK(cudaGraphInstantiate(&t.exec, t.graph, 0));
  g_tail_builds.fetch_add(1);
  return ST_OK;
}

int run_tail_graph(cudaStream_t s, TailGraphKey key, const TailBody& body_fn) {
  ST_CUDA_CHECK(cudaGetDevice(&key.device));
  std::lock_guard<std::mutex> lock(g_tail_mu);
  std::vector<TailGraph>& cache = *g_tail;
  TailGraph* hit = nullptr;
  for (TailGraph& t : cache)
    if (memcmp(&t.key, &key, sizeof(key)) == 0) hit = &t;
  if (!hit) {
    if (cache.size() >= TAIL_GRAPH_CAP) {  // least recently used out
      auto lru = std::min_element(
          cache.begin(), cache.end(),
          [](const TailGraph& a, const TailGraph& b) { return a.used < b.used; });
      destroy_tail_graph(*lru);
      cache.erase(lru);
    }
    TailGraph t;
    memset(&t, 0, sizeof(t));
    t.key = key;
    const int rc = build_tail_graph(t, body_fn);
    if (rc) {
      destroy_tail_graph(t);
      return rc;
    }
    cache.push_back(t);
    hit = &cache.back();
  }
  hit->used = ++g_tail_tick;
  ST_CUDA_CHECK(cudaGraphLaunch(hit->exec, s));
  sthost::g_launches.fetch_add(hit->launches);
  g_tail_launches.fetch_add(1);
  return ST_OK;
}

}  // namespace

int64_t st_tail_graph_count(int32_t which) {
  return which == 0 ? g_tail_builds.load() : which == 1 ? g_tail_launches.load() : -1;
}

// The asynchronous EM driver behind st_solve_async and st_solve_rows.
// Slots: i -> pixel pix0 + i (dense) or active[i] (a sorted list); slots
// [cnt_lo, cnt_hi) are this shard's own pixels (the statistics count only
// them; row bands also solve a halo of neighbour rows for the median).
struct AsyncSolve {
  int64_t pix0;
  const int64_t* active;
  int64_t n;
  int64_t cnt_lo, cnt_hi;
  int64_t init_pix0, init_n;   // initial masks: pixels [init_pix0, init_pix0 + init_n)
  bool band;                   // per-iteration record exchange + k_band_control
  st_exchange_fn exchange;     // nullable when world == 1
  void* user;
  int world;
  void* rec_send;
  void* rec_recv;
  // nullable: the slot count on the device (dynamic_only, one shard: no host
  // read-back); n and cnt_hi are then its upper bound (the grids)
  const uint32_t* n_dev;
};

static int solve_async_core(const st_frame* f, const st_rig* rig, const st_params* p,
                            st::EmCtx& c, const AsyncSolve& A, float* values, uint8_t* status,
                            uint32_t* static_bits, uint32_t* valid_bits, st_stats* stats_dev,
                            char* ws, const SolveLayout& L, cudaStream_t s) {
  const int64_t npx = c.HW;
  double* d_act = (double*)(ws + L.d);
  double* e_act = (double*)(ws + L.e);
  double* pe_act = (double*)(ws + L.pe);
  uint8_t* st_act = (uint8_t*)(ws + L.st_act);
  uint8_t* chg = (uint8_t*)(ws + L.chg);
  uint32_t* mask_in = (uint32_t*)(ws + L.mask_in);
  int32_t* mlist = (int32_t*)(ws + L.mlist);
  int32_t* elist = (int32_t*)(ws + L.elist);
  uint32_t* counts = (uint32_t*)(ws + L.counts);
  int* stop = (int*)(counts + 2);
  st::Partial* work = (st::Partial*)(ws + L.work);
  st::Partial* parts = (st::Partial*)(ws + L.parts);
  st::Partial* reduced = (st::Partial*)(ws + L.reduced);
  const int64_t n = A.n;
  const int64_t n_cnt = A.cnt_hi - A.cnt_lo;

  ST_CUDA_CHECK(cudaMemsetAsync(stats_dev, 0, sizeof(st_stats), s));
  ST_CUDA_CHECK(cudaMemsetAsync(counts, 0, 2 * sizeof(uint32_t) + sizeof(int), s));
  // E-step fallback count (byte 48) and the stats kernel's block counter (52)
  ST_CUDA_CHECK(cudaMemsetAsync(counts + 12, 0, 4 * sizeof(uint32_t), s));
  st::k_stats_init<<<1, 32, 0, s>>>(stats_dev, A.n_dev ? 0 : n_cnt);  // (band control sets it)
  ST_LAUNCH_CHECK("k_stats_init");
  double* eps_logs = (double*)(counts + 4);
  st::k_eps_logs<<<1, 32, 0, s>>>(p->epsilon_prior, eps_logs);
  ST_LAUNCH_CHECK("k_eps_logs");
  {
    st::EmCtx ci = c;
    ci.pix0 = A.init_pix0;
    // (k_initial_masks writes row i of its outputs: pixel init_pix0 + i)
    st::k_initial_masks<<<blocks_for(A.init_n, 128), 128, 0, s>>>(
        ci, nullptr, A.init_n, static_bits + A.init_pix0, valid_bits + A.init_pix0);
    ST_LAUNCH_CHECK("k_initial_masks");
  }
  c.pix0 = A.active ? 0 : A.pix0;

  const int iters = p->forced_iters > 0 ? p->forced_iters : p->max_iters;
  const int nblk = std::max(1, (int)blocks_for(n, EM_BLOCK));
  const int pw_d = st::stats_depth(n_cnt);
  const int sblk = 1 << pw_d;  // numpy's pairwise tree, top levels (st_pw.cuh)
  // iterations >= 2 work on device-counted worklists (a fraction of the
  // pixels) and do nothing once converged: a fixed grid of grid-stride
  // blocks (16 per SM measured best: the worklists' items are latency-bound)
  static const int wave_env = [] {
    const char* e = getenv("ST_WAVE_BLOCKS_PER_SM");
    return e ? atoi(e) : 16;
  }();
  const int wave2 = std::min(nblk, 148 * wave_env);
  const int mblk = (int)mstep_blocks(c, n);
  const int mwave2 = std::min(mblk, 148 * wave_env);
  uint32_t* it_off = counts + 14;  // (zeroed above with counts + 12 .. + 15)
  // everything the captured launches depend on: the cache key of the graph
  TailGraphKey graph_key;
  memset(&graph_key, 0, sizeof(graph_key));
  graph_key.c = c;
  graph_key.active = A.active;
  graph_key.n = n;
  graph_key.cnt_lo = A.cnt_lo;
  graph_key.cnt_hi = A.cnt_hi;
  graph_key.static_bits = static_bits;
  graph_key.valid_bits = valid_bits;
  graph_key.stats = stats_dev;
  graph_key.ws = ws;
  graph_key.mu_unsafe = f->mu_unsafe;
  graph_key.n_dev = A.n_dev;
  graph_key.band = A.band ? 1 : 0;
  graph_key.forced_iters = p->forced_iters;
  graph_key.iters = iters;
  graph_key.wave_env = wave_env;
  // One EM iteration's launches (M-step worklist, M-step, E-step, statistics
  // + control).  Every iteration >= 3 enqueues the same launches with the
  // same arguments; `g` (nullable) turns on the graph loop's fields of the
  // statistics kernel (the iteration counter and the WHILE condition).
  auto iteration = [&](int it, const TailGraphFields* g, cudaStream_t s) -> int {
    // iteration 2 re-solves the pixels whose mask changed at iteration 1
    // (~20 %); later iterations have far smaller worklists, or none once
    // converged (the launches then exit at once): a smaller grid
    const int wave = it <= 2 ? wave2 : std::min(nblk, 148 * 4);
    if (n > 0) {
    if (it > 1) {
      st::k_flag_mstep<<<wave, EM_BLOCK, 0, s>>>(A.active, n, c.pix0, static_bits, mask_in,
                                                 e_act, pe_act, chg, mlist, counts, stop,
                                                 A.n_dev);
      ST_LAUNCH_CHECK("k_flag_mstep");
    }
    st::MStepArgs a;
    memset(&a, 0, sizeof(a));
    a.active = A.active;
    a.n = n;
    a.list = it > 1 ? mlist : nullptr;
    a.list_count = counts;
    a.static_all = static_bits;
    a.first = it == 1;
    a.d = d_act;
    a.e = e_act;
    a.status = st_act;
    a.mask_in = mask_in;
    a.pe = pe_act;
    a.chg = chg;
    a.elist = elist;
    a.elist_count = counts + 1;
    a.partials = work;
    a.stop = stop;
    a.n_dev = A.n_dev;
    const int mgrid = it == 1 ? mblk : it == 2 ? mwave2 : std::min(mblk, 148 * 4);
    launch_m_step(c, a, mgrid, s);
    ST_LAUNCH_CHECK("k_m_step");
    st::EStepArgs e;
    memset(&e, 0, sizeof(e));
    e.pix = A.active;
    e.n = n;
    e.list = elist;
    e.list_count = counts + 1;
    e.d = d_act;
    e.status = st_act;
    e.static_out = static_bits;
    e.valid_out = valid_bits;
    e.scatter = 1;
    e.eps_logs = eps_logs;
    e.flist = (int32_t*)(ws + L.flist);
    e.flist_count = (uint32_t*)(eps_logs + 4);
    e.stop = stop;
    launch_e_step(rig->num_views,
                  it == 1 ? n : std::min<int64_t>(n, 148 * (it == 2 ? 8 : 4) * 128), s, c, e,
                  true);
    ST_LAUNCH_CHECK("k_e_step_at");
    }  // n > 0
    // statistics, their fixed-order reduction and the control in one launch
    // (the last block folds the partials; it also clears the fallback count)
    st::StatsTail tail;
    memset(&tail, 0, sizeof(tail));
    tail.on = 1;
    tail.it = it;
    tail.done = counts + 13;
    tail.reduced = reduced;
    tail.counts = counts;
    tail.n_act = n_cnt;
    tail.forced_iters = p->forced_iters;
    tail.stats = stats_dev;
    tail.stop_rw = stop;
    tail.flist_count = (uint32_t*)(eps_logs + 4);
    tail.record_only = A.band ? 1 : 0;
    tail.record_n_act = n_cnt;
    tail.record_slots = n;
    tail.pw_depth = pw_d;
    tail.pw_scratch = (double*)(ws + L.pw_scratch);
    tail.pw_val = (double*)(ws + L.pw_val);
    tail.mu_unsafe = A.band ? f->mu_unsafe : nullptr;
    tail.n_dev = A.n_dev;
    if (g) {
      tail.it_off = it_off;
      tail.use_cond = 1;
      tail.iters = iters;
      tail.cond = g->cond;
    }
    st::k_em_stats<<<sblk, STATS_BLOCK, 0, s>>>(
        n_cnt, it > 1, e_act + A.cnt_lo, pe_act + A.cnt_lo, chg + A.cnt_lo, work,
        (n > 0 ? (it == 1 ? mblk : it == 2 ? mwave2 : std::min(mblk, 148 * 4)) : 0) *
            (EM_BLOCK / 32),
        parts, stop, tail);
    ST_LAUNCH_CHECK("k_em_stats");
    if (A.band) {
      const st::Partial* recs = reduced + it;
      if (A.exchange) {
        ST_CUDA_CHECK(cudaMemcpyAsync(A.rec_send, reduced + it, sizeof(st::Partial),
                                      cudaMemcpyDeviceToDevice, s));
        if (A.exchange(s, A.user)) {
          sthost::set_error("row-band record exchange failed");
          return ST_EINVAL;
        }
        recs = (const st::Partial*)A.rec_recv;
      }
      st::BandLoop loop;
      memset(&loop, 0, sizeof(loop));
      if (g) {
        loop.it_off = it_off;
        loop.use_cond = 1;
        loop.iters = iters;
        loop.cond = g->cond;
      }
      st::k_band_control<<<1, 32, 0, s>>>(it, recs, A.exchange ? A.world : 1, p->forced_iters,
                                          stats_dev, stop, loop);
      ST_LAUNCH_CHECK("k_band_control");
    }
    return ST_OK;
  };
  // Iterations >= 3 of a one-device solve run as a CUDA-graph WHILE loop
  // (the statistics kernel sets its condition): the frame's converged
  // iterations cost no launches and no host round trip, whatever the cap.
  // (row bands exchanging records through the host callback keep the loop,
  // and so do active-pixel lists whose length the host passes: it is part of
  // the captured arguments and changes from frame to frame; a device-side
  // count (A.n_dev) keeps the captured arguments fixed)
  bool use_graph = !A.exchange && (!A.active || A.n_dev) && n > 0 && iters >= 3 &&
                   tail_graphs_enabled();
  // a row band with no active pixel still takes part in every exchange
  for (int it = 1; it <= iters && (n > 0 || A.band); ++it) {
    if (use_graph && it == 3) {
      const int rc = run_tail_graph(
          s, graph_key,
          [&](const TailGraphFields* g, cudaStream_t cs) { return iteration(3, g, cs); });
      if (rc == ST_OK) break;
      use_graph = false;  // (could not build the graph: the launch loop below)
      sthost::set_error("");
    }
    // long caps (max_iters > ST_ASYNC_CHUNK) and row bands: read the device
    // stop flag back before enqueueing more iterations, so a converged solve
    // does not enqueue max_iters rounds of (immediately exiting) launches and
    // exchanges (row bands check every iteration)
    const int chunk = A.band && A.exchange ? 1 : ST_ASYNC_CHUNK;
    if (it > chunk && (it - 1) % chunk == 0) {
      int h_stop = 0;
      ST_CUDA_CHECK(cudaMemcpyAsync(&h_stop, stop, sizeof(int), cudaMemcpyDeviceToHost, s));
      ST_CUDA_CHECK(cudaStreamSynchronize(s));
      if (h_stop == 2) {
        sthost::set_error("row band: whole-frame surface raster needed");
        return ST_EAGAIN;
      }
      if (h_stop) break;
    }
    const int rc = iteration(it, nullptr, s);
    if (rc) return rc;
  }
  if (A.band && A.exchange) {  // (max_iters == 1: the loop read no stop flag)
    int h_stop = 0;
    ST_CUDA_CHECK(cudaMemcpyAsync(&h_stop, stop, sizeof(int), cudaMemcpyDeviceToHost, s));
    ST_CUDA_CHECK(cudaStreamSynchronize(s));
    if (h_stop == 2) {
      sthost::set_error("row band: whole-frame surface raster needed");
      return ST_EAGAIN;
    }
  }
  if (A.active) {
    st::k_fill_mu<<<blocks_for(A.init_n, 256), 256, 0, s>>>(f->mu + A.init_pix0, A.init_n,
                                                             values + A.init_pix0,
                                                             status + A.init_pix0);
    ST_LAUNCH_CHECK("k_fill_mu");
    if (n > 0) {
      st::k_pack_outputs<<<blocks_for(n, 256), 256, 0, s>>>(f->mu, npx, 0, A.active, n, d_act,
                                                            st_act, values, status, 0, A.n_dev);
      ST_LAUNCH_CHECK("k_pack_outputs");
    }
  } else {
    st::k_pack_outputs<<<blocks_for(n, 256), 256, 0, s>>>(f->mu, n, A.pix0, nullptr, n, d_act,
                                                          st_act, values, status, 1);
    ST_LAUNCH_CHECK("k_pack_outputs");
  }
  return ST_OK;
}

static int solve_prologue(const st_frame* f, const st_rig* rig, const st_params* p,
                          st::EmCtx& c, int64_t workspace_bytes, SolveLayout& L) {
  int rc = make_ctx(f, rig, p, c);
  if (rc) return rc;
  if ((rc = prepare_estep_kernels())) return rc;
  L = solve_layout(c.W, c.H);
  if ((int64_t)L.total > workspace_bytes) {
    sthost::set_error("solve workspace too small (%lld < %lld)", (long long)workspace_bytes,
                      (long long)L.total);
    return ST_ENOMEM;
  }
  return ST_OK;
}

// st_solve for a dense solve on one device with no host synchronisation: the
// convergence test (solver.py:483-485) and the statistics run on the device
// (k_solve_control), and every kernel of the iterations after convergence
// exits at once on the device stop flag.  Results are identical to st_solve.
int st_solve_async(const st_frame* f, const st_rig* rig, const st_params* p, float* values,
                   uint8_t* status, uint32_t* static_bits, uint32_t* valid_bits,
                   st_stats* stats_dev, void* workspace, int64_t workspace_bytes,
                   void* stream) {
  st::EmCtx c;
  SolveLayout L;
  int rc = solve_prologue(f, rig, p, c, workspace_bytes, L);
  if (rc) return rc;
  if (!stats_dev) {
    sthost::set_error("st_solve_async: stats_dev is required");
    return ST_EINVAL;
  }
  AsyncSolve A = {};
  A.n = c.HW;
  A.cnt_hi = c.HW;
  A.init_n = c.HW;
  A.world = 1;
  return solve_async_core(f, rig, p, c, A, values, status, static_bits, valid_bits, stats_dev,
                          (char*)workspace, L, (cudaStream_t)stream);
}

int64_t st_band_record_bytes(void) { return (int64_t)sizeof(st::Partial); }

int st_solve_rows(const st_frame* f, const st_rig* rig, const st_params* p,
                  int32_t dynamic_only, int32_t row0, int32_t row1, int32_t ext0, int32_t ext1,
                  float* values, uint8_t* status, uint32_t* static_bits, uint32_t* valid_bits,
                  st_stats* stats_dev, void* workspace, int64_t workspace_bytes,
                  st_exchange_fn exchange, void* user, int32_t world, void* rec_send,
                  void* rec_recv, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  st::EmCtx c;
  SolveLayout L;
  int rc = solve_prologue(f, rig, p, c, workspace_bytes, L);
  if (rc) return rc;
  const int W = c.W, H = c.H;
  if (!stats_dev || !(0 <= ext0 && ext0 <= row0 && row0 <= row1 && row1 <= ext1 && ext1 <= H) ||
      world < 1 || (world > 1 && (!exchange || !rec_send || !rec_recv))) {
    sthost::set_error("st_solve_rows: need 0 <= ext0 <= row0 <= row1 <= ext1 <= H (%d), "
                      "stats_dev, and an exchange with its buffers when world > 1", H);
    return ST_EINVAL;
  }
  char* ws = (char*)workspace;
  AsyncSolve A = {};
  A.band = true;
  A.exchange = world > 1 || exchange ? exchange : nullptr;
  A.user = user;
  A.world = world;
  A.rec_send = rec_send;
  A.rec_recv = rec_recv;
  A.init_pix0 = (int64_t)ext0 * W;
  A.init_n = (int64_t)(ext1 - ext0) * W;
  if (!dynamic_only) {
    A.pix0 = A.init_pix0;
    A.n = A.init_n;
    A.cnt_lo = (int64_t)(row0 - ext0) * W;
    A.cnt_hi = (int64_t)(row1 - ext0) * W;
  } else {
    // active = ref prior < threshold inside the solved rows (solver.py:449-452):
    // one host read-back for the list size and this band's counted slots
    const int64_t npx = c.HW;
    uint32_t* flags = (uint32_t*)(ws + L.flags);
    uint32_t* offs = (uint32_t*)(ws + L.offs);
    int64_t* active = (int64_t*)(ws + L.active);
    const float* ref_prior = f->priors + (size_t)rig->ref_index * npx;
    st::k_flag_active<<<blocks_for(npx, 256), 256, 0, s>>>(ref_prior, nullptr, npx, p->threshold,
                                                          flags, A.init_pix0,
                                                          A.init_pix0 + A.init_n);
    ST_LAUNCH_CHECK("k_flag_active");
    ST_CUDA_CHECK(cudaMemsetAsync(flags + npx, 0, sizeof(uint32_t), s));
    size_t tb = L.cub_bytes;
    ST_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ws + L.cub, tb, flags, offs, (int)(npx + 1), s));
    sthost::count_launch();
    st::k_scatter_active<<<blocks_for(npx, 256), 256, 0, s>>>(flags, offs, npx, active);
    ST_LAUNCH_CHECK("k_scatter_active");
    A.active = active;
    if (world == 1 && row0 == 0 && row1 == H && ext0 == 0 && ext1 == H &&
        !getenv("ST_DYNAMIC_READBACK")) {
      // one shard over the whole frame: the count stays on the device (the
      // grids cover every pixel; the kernels read the count), no host sync
      A.n_dev = offs + npx;
      A.n = npx;
      A.cnt_lo = 0;
      A.cnt_hi = npx;
      return solve_async_core(f, rig, p, c, A, values, status, static_bits, valid_bits,
                              stats_dev, ws, L, s);
    }
    uint32_t h[3] = {0, 0, 0};
    ST_CUDA_CHECK(cudaMemcpyAsync(&h[0], offs + npx, 4, cudaMemcpyDeviceToHost, s));
    ST_CUDA_CHECK(cudaMemcpyAsync(&h[1], offs + (int64_t)row0 * W, 4, cudaMemcpyDeviceToHost, s));
    ST_CUDA_CHECK(cudaMemcpyAsync(&h[2], offs + (int64_t)row1 * W, 4, cudaMemcpyDeviceToHost, s));
    ST_CUDA_CHECK(cudaStreamSynchronize(s));
    A.active = active;
    A.n = h[0];
    A.cnt_lo = h[1];
    A.cnt_hi = h[2];
  }
  return solve_async_core(f, rig, p, c, A, values, status, static_bits, valid_bits, stats_dev,
                          ws, L, s);
}

}  // extern "C"
