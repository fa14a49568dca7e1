// Support-point harvest on the device (prior.py:51-260).
//
// Stages, one frame, all views at once:
//   k_hv_detect   one thread per stride-grid site: descriptor-valid interior,
//                 texture energy >= min_texture (features.py:114-117,
//                 prior.py:51-66) and the ring-eroded prior >= threshold
//                 (prior.py:215-230, 248-250).
//   (CUB select)  ordered compaction -> view-major, raster-ordered candidates.
//   k_hv_match    one warp per candidate: lanes sweep the disparity grid, the
//                 SAD costs stay in registers, a warp reduction gives the
//                 first argmin and the excluded second best (prior.py:69-98);
//                 the same warp then runs the reverse scan from the rounded
//                 landing pixel (:120-133) and, for non-reference views,
//                 reprojects the point into the reference (:146-180).
//   (CUB select)  ordered compaction of the surviving points.
// deduplicate (:183-212) is an order-dependent greedy pass and runs on the
// host (st_support_dedup below).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cub/cub.cuh>
#include <vector>

#include "st_common.cuh"

#define HV_MAXJ 16              // disparity slots per lane: n_d <= 512
#define HV_BLOCK 256

namespace st {

// SAMPLE_OFFSETS (features.py:24)
__constant__ int c_ring_du[8] = {0, 1, 2, 1, 0, -1, -2, -1};
__constant__ int c_ring_dv[8] = {-2, -1, 0, 1, 2, 1, 0, -1};

__global__ void k_hv_detect(const uint4* __restrict__ desc, const float* __restrict__ priors,
                            int K, int W, int H, int stride, int gw, int gh, double min_texture,
                            float thr, uint8_t* __restrict__ flags) {
  const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per_view = (int64_t)gw * gh;
  if (slot >= per_view * K) return;
  const int k = (int)(slot / per_view);
  const int r = (int)(slot % per_view);
  const int u = (r % gw) * stride, v = (r / gw) * stride;
  bool keep = u >= ST_DESC_MARGIN && u < W - ST_DESC_MARGIN && v >= ST_DESC_MARGIN &&
              v < H - ST_DESC_MARGIN;
  if (keep) {
    const uint4 q = __ldg(desc + (size_t)k * W * H + (size_t)v * W + u);
    const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
    int e = 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) e += abs((int)((w4[c >> 2] >> (8 * (c & 3))) & 0xff) - 128);
    keep = (double)e >= min_texture;
  }
  if (keep) {
    const float* p = priors + (size_t)k * W * H;
    float m = p[(size_t)v * W + u];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int sy = min(max(v + c_ring_dv[i], 0), H - 1);
      const int sx = min(max(u + c_ring_du[i], 0), W - 1);
      m = fminf(m, p[(size_t)sy * W + sx]);
    }
    keep = m >= thr;
  }
  flags[slot] = keep ? 1 : 0;
}

__device__ __forceinline__ bool desc_ok(double u, double v, int W, int H) {
  // sample_descriptors validity (features.py:131-132); NaN -> false
  return u >= (double)ST_DESC_MARGIN && u <= (double)(W - ST_DESC_MARGIN - 1) &&
         v >= (double)ST_DESC_MARGIN && v <= (double)(H - ST_DESC_MARGIN - 1);
}

__device__ __forceinline__ double grid_d(int j) { return dadd(0.5, dmul((double)j, 0.5)); }

// One warp: SAD scan of (u, v) in plane `src` against plane `dst` along the
// warp (a, b) over d_j = 0.5 + 0.5 j, then _best_with_ratio.  Returns the
// best disparity or NaN (uniform across the warp).
__device__ double warp_scan(const uint4* __restrict__ src, const uint4* __restrict__ dst, int W,
                            int H, const double* a, const double* b, double u, double v, int nd) {
  const int lane = threadIdx.x & 31;
  const bool ref_ok = desc_ok(u, v, W, H);
  double ref[16];
  sample_desc(src, W, taps_of(u, v, W, H), [&](int c, double x) { ref[c] = x; });
  double cost[HV_MAXJ];
#pragma unroll
  for (int r = 0; r < HV_MAXJ; ++r) {
    const int j = lane + 32 * r;
    cost[r] = INFINITY;
    if (j >= nd) continue;
    const WarpOut w = warp_ab(a, b, u, v, grid_d(j));
    if (!(ref_ok && w.front && desc_ok(w.pu, w.pv, W, H))) continue;
    // np.abs(ref - tgt).sum(axis=1): numpy's contiguous 16-term reduction
    double acc[8];
    sample_desc(dst, W, taps_of(w.pu, w.pv, W, H), [&](int c, double x) {
      const double t = fabs(dsub(ref[c], x));
      if (c < 8)
        acc[c] = t;
      else
        acc[c - 8] = dadd(acc[c - 8], t);
    });
    cost[r] = dadd(dadd(dadd(acc[0], acc[1]), dadd(acc[2], acc[3])),
                   dadd(dadd(acc[4], acc[5]), dadd(acc[6], acc[7])));
  }
  // first argmin (np.argmin; all-inf -> index 0): (cost, j) lexicographic
  double bc = INFINITY;
  int bj = 0x7fffffff;
#pragma unroll
  for (int r = 0; r < HV_MAXJ; ++r) {
    const int j = lane + 32 * r;
    if (j < nd && (bj == 0x7fffffff || cost[r] < bc)) {
      bc = cost[r];
      bj = j;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
    if (oc < bc || (oc == bc && oj < bj)) {
      bc = oc;
      bj = oj;
    }
  }
  if (bj == 0x7fffffff) bj = 0;  // empty grid: bc stays inf -> no match
  const double bd = grid_d(bj);
  // best among |d - best_d| > SECOND_BEST_EXCLUSION (prior.py:90-93)
  double sc = INFINITY;
#pragma unroll
  for (int r = 0; r < HV_MAXJ; ++r) {
    const int j = lane + 32 * r;
    if (j < nd && !(fabs(dsub(grid_d(j), bd)) <= 1.0)) sc = fmin(sc, cost[r]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sc = fmin(sc, __shfl_xor_sync(0xffffffffu, sc, o));
  const bool ok = isfinite(bc) && !(isfinite(sc) && bc > dmul(0.9, sc));
  return ok ? bd : NAN;
}

struct HvArgs {
  const uint4* desc;
  const float* priors;
  int K, W, H, stride, gw, gh, nd;
  double d_max;
  float thr;
  const int32_t* cand;        // candidate slots (view-major, raster)
  const int64_t* n_cand;
  int32_t* pu;                // per candidate: output point (valid where flag)
  int32_t* pv;
  double* pd;
  uint8_t* flag;
  int64_t* counters;          // nullable: [candidates, reverse scans]
};

__global__ void __launch_bounds__(HV_BLOCK) k_hv_match(st_cams cam, HvArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t n = *a.n_cand;
  const int64_t per_view = (int64_t)a.gw * a.gh;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t ci = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; ci < n;
       ci += nwarps) {
    const int32_t slot = a.cand[ci];
    const int s = (int)(slot / per_view);
    const int r = (int)(slot % per_view);
    const int iu = (r % a.gw) * a.stride, iv = (r / a.gw) * a.stride;
    const double u = (double)iu, v = (double)iv;
    const int dn = cam.nn[s];
    const uint4* ps = a.desc + (size_t)s * a.W * a.H;
    const uint4* pd = a.desc + (size_t)dn * a.W * a.H;
    bool keep = false;
    int ou = 0, ov = 0;
    double od = 0.0;
    const double best = warp_scan(ps, pd, a.W, a.H, cam.fw_a[s], cam.fw_b[s], u, v, a.nd);
    if (!isnan(best)) {
      // reverse match from the rounded landing pixel (prior.py:120-133)
      const WarpOut w = warp_ab(cam.fw_a[s], cam.fw_b[s], u, v, best);
      const double ru = rint(w.pu), rv = rint(w.pv);
      if (a.counters && lane == 0) atomicAdd((unsigned long long*)(a.counters + 1), 1ull);
      const double rb = warp_scan(pd, ps, a.W, a.H, cam.bw_a[s], cam.bw_b[s], ru, rv, a.nd);
      keep = !isnan(rb) && fabs(dsub(dmul(rb, cam.lr_scale[s]), best)) <= 1.0;
      if (keep && s == cam.ref_index) {
        keep = best <= a.d_max;  // prior.py:253
        ou = iu;
        ov = iv;
        od = best;
      } else if (keep) {
        // reproject_occluded_support (prior.py:160-179).  R^T (cam - t) as
        // the fused multiply-add chain numpy's dgemv evaluates.
        const double depth = ddiv(dmul(cam.fx[s], cam.unit_baseline), best);
        const double xc = dmul(ddiv(dsub(u, cam.cx[s]), cam.fx[s]), depth);
        const double yc = dmul(ddiv(dsub(v, cam.cy[s]), cam.fy[s]), depth);
        const double x0 = dsub(xc, cam.trans[s][0]);
        const double x1 = dsub(yc, cam.trans[s][1]);
        const double x2 = dsub(depth, cam.trans[s][2]);
        const double* R = cam.rot[s];
        double wd[3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
          wd[i] = __fma_rn(R[6 + i], x2, __fma_rn(R[3 + i], x1, dmul(R[i], x0)));
        keep = wd[2] > 0.0;
        const int ref = cam.ref_index;
        if (keep) {
          const double ur = dadd(ddiv(dmul(cam.fx[ref], wd[0]), wd[2]), cam.cx[ref]);
          const double vr = dadd(ddiv(dmul(cam.fy[ref], wd[1]), wd[2]), cam.cy[ref]);
          const double fu = rint(ur), fv = rint(vr);
          keep = fu >= 0.0 && fu < (double)a.W && fv >= 0.0 && fv < (double)a.H;
          if (keep) {
            ou = (int)fu;
            ov = (int)fv;
            keep = !(a.priors[(size_t)ref * a.W * a.H + (size_t)ov * a.W + ou] >= a.thr);
          }
          if (keep) {
            od = ddiv(dmul(cam.fx[ref], cam.unit_baseline), wd[2]);
            keep = od > 0.0 && od <= a.d_max;
          }
        }
      }
    }
    if (lane == 0) {
      a.flag[ci] = keep ? 1 : 0;
      a.pu[ci] = ou;
      a.pv[ci] = ov;
      a.pd[ci] = od;
    }
  }
}

__global__ void k_hv_gather(const int32_t* __restrict__ sel, const int64_t* __restrict__ n_sel,
                            const int32_t* __restrict__ cand, int64_t per_view,
                            const int32_t* __restrict__ pu, const int32_t* __restrict__ pv,
                            const double* __restrict__ pd, int32_t* __restrict__ ou,
                            int32_t* __restrict__ ov, double* __restrict__ od,
                            int32_t* __restrict__ osrc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *n_sel) return;
  const int32_t c = sel[i];
  ou[i] = pu[c];
  ov[i] = pv[c];
  od[i] = pd[c];
  osrc[i] = (int32_t)(cand[c] / per_view);
}

}  // namespace st

namespace {

int64_t grid_sites(int32_t W, int32_t H, int32_t stride, int32_t& gw, int32_t& gh) {
  gw = (W + stride - 1) / stride;
  gh = (H + stride - 1) / stride;
  return (int64_t)gw * gh;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct HvWs {
  uint8_t* flags;     // sites
  int32_t* cand;      // sites
  int64_t* n_cand;
  int32_t* pu;        // sites
  int32_t* pv;
  double* pd;
  uint8_t* pflag;
  int32_t* sel;
  void* cub;
  size_t cub_bytes;
  size_t total;
};

HvWs carve(void* base, int64_t sites) {
  HvWs w = {};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    void* p = base ? (void*)((char*)base + off) : nullptr;
    off += align256(bytes);
    return p;
  };
  w.flags = (uint8_t*)take(sites);
  w.cand = (int32_t*)take(sites * 4);
  w.n_cand = (int64_t*)take(8);
  w.pu = (int32_t*)take(sites * 4);
  w.pv = (int32_t*)take(sites * 4);
  w.pd = (double*)take(sites * 8);
  w.pflag = (uint8_t*)take(sites);
  w.sel = (int32_t*)take(sites * 4);
  size_t c1 = 0, c2 = 0;
  cub::DeviceSelect::Flagged(nullptr, c1, cub::CountingInputIterator<int32_t>(0),
                             (const uint8_t*)nullptr, (int32_t*)nullptr, (int64_t*)nullptr,
                             (int64_t)sites);
  cub::DeviceSelect::Flagged(nullptr, c2, cub::CountingInputIterator<int32_t>(0),
                             (const uint8_t*)nullptr, (int32_t*)nullptr, (int64_t*)nullptr,
                             (int64_t)sites);
  w.cub_bytes = std::max(c1, c2);
  w.cub = take(w.cub_bytes);
  w.total = off;
  return w;
}

}  // namespace

extern "C" {

int64_t st_harvest_capacity(int32_t K, int32_t W, int32_t H, int32_t stride) {
  int32_t gw, gh;
  if (stride < 1) return 0;
  return grid_sites(W, H, stride, gw, gh) * K;
}

int64_t st_harvest_workspace(int32_t K, int32_t W, int32_t H, int32_t stride) {
  int32_t gw, gh;
  if (stride < 1) return 0;
  return (int64_t)carve(nullptr, grid_sites(W, H, stride, gw, gh) * K).total;
}

int st_harvest(const uint8_t* desc, const float* priors, const st_cams* cams, double d_max,
               int32_t n_d, float threshold, int32_t stride, double min_texture,
               int32_t* out_u, int32_t* out_v, double* out_d, int32_t* out_src,
               int64_t* out_count, int64_t* counters, void* workspace, int64_t workspace_bytes,
               void* stream) {
  if (!cams || cams->num_views < 2 || cams->num_views > ST_MAX_VIEWS) {
    sthost::set_error("st_harvest: view count must be in [2, %d]", ST_MAX_VIEWS);
    return ST_EINVAL;
  }
  if (stride < 1 || n_d < 0 || n_d > 32 * HV_MAXJ) {
    sthost::set_error("st_harvest: stride >= 1 and disparity grid <= %d required",
                      32 * HV_MAXJ);
    return ST_EINVAL;
  }
  const int K = cams->num_views, W = cams->width, H = cams->height;
  if (W < 2 * ST_DESC_MARGIN + 1 || H < 2 * ST_DESC_MARGIN + 1) {
    sthost::set_error("st_harvest: image too small for descriptors");
    return ST_EINVAL;
  }
  int32_t gw, gh;
  const int64_t per_view = grid_sites(W, H, stride, gw, gh);
  const int64_t sites = per_view * K;
  if (sites >= (int64_t)1 << 31) {
    sthost::set_error("st_harvest: too many grid sites");
    return ST_EINVAL;
  }
  HvWs w = carve(workspace, sites);
  if (!workspace || workspace_bytes < (int64_t)w.total) {
    sthost::set_error("st_harvest: workspace too small (%lld < %lld)",
                      (long long)workspace_bytes, (long long)w.total);
    return ST_ENOMEM;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const uint4* d4 = reinterpret_cast<const uint4*>(desc);
  st::k_hv_detect<<<(unsigned)((sites + 255) / 256), 256, 0, s>>>(
      d4, priors, K, W, H, stride, gw, gh, min_texture, threshold, w.flags);
  ST_LAUNCH_CHECK("k_hv_detect");
  size_t cb = w.cub_bytes;
  ST_CUDA_CHECK(cub::DeviceSelect::Flagged(w.cub, cb, cub::CountingInputIterator<int32_t>(0),
                                           w.flags, w.cand, w.n_cand, sites, s));
  sthost::count_launch();
  st::HvArgs a;
  a.desc = d4;
  a.priors = priors;
  a.K = K;
  a.W = W;
  a.H = H;
  a.stride = stride;
  a.gw = gw;
  a.gh = gh;
  a.nd = n_d;
  a.d_max = d_max;
  a.thr = threshold;
  a.cand = w.cand;
  a.n_cand = w.n_cand;
  a.pu = w.pu;
  a.pv = w.pv;
  a.pd = w.pd;
  a.flag = w.pflag;
  a.counters = counters;
  if (counters) {
    ST_CUDA_CHECK(cudaMemcpyAsync(counters, w.n_cand, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    ST_CUDA_CHECK(cudaMemsetAsync(counters + 1, 0, sizeof(int64_t), s));
  }
  // one warp per candidate (grid-stride; the count stays on the device)
  ST_CUDA_CHECK(cudaMemsetAsync(w.pflag, 0, (size_t)sites, s));
  const int64_t warps = std::max<int64_t>(sites, 1);
  const unsigned blocks = (unsigned)std::min<int64_t>((warps + 7) / 8, 148 * 64);
  st::k_hv_match<<<blocks, HV_BLOCK, 0, s>>>(*cams, a);
  ST_LAUNCH_CHECK("k_hv_match");
  cb = w.cub_bytes;
  ST_CUDA_CHECK(cub::DeviceSelect::Flagged(w.cub, cb, cub::CountingInputIterator<int32_t>(0),
                                           w.pflag, w.sel, out_count, sites, s));
  sthost::count_launch();
  st::k_hv_gather<<<(unsigned)((sites + 255) / 256), 256, 0, s>>>(
      w.sel, out_count, w.cand, per_view, w.pu, w.pv, w.pd, out_u, out_v, out_d, out_src);
  ST_LAUNCH_CHECK("k_hv_gather");
  return ST_OK;
}

int st_support_dedup(const int32_t* u, const int32_t* v, const double* d, const int32_t* src,
                     int64_t n, int32_t ref_index, int32_t W, int32_t H, int64_t* keep,
                     int64_t* n_keep) {
  if (n < 0 || W < 1 || H < 1 || !n_keep) {
    sthost::set_error("st_support_dedup: bad arguments");
    return ST_EINVAL;
  }
  std::vector<int64_t> order((size_t)n);
  for (int64_t i = 0; i < n; ++i) order[(size_t)i] = i;
  // sorted(points, key=(source_view != ref, d, v, u)) -- stable
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    const int ra = src[a] != ref_index, rb = src[b] != ref_index;
    if (ra != rb) return ra < rb;
    if (d[a] != d[b]) return d[a] < d[b];
    if (v[a] != v[b]) return v[a] < v[b];
    return u[a] < u[b];
  });
  // taken: pixel -> accepted point (points may sit anywhere the reference
  // lets them; out-of-image neighbours simply have no entry)
  std::vector<int64_t> taken((size_t)W * H, -1);
  auto at = [&](int64_t x, int64_t y) -> int64_t {
    if (x < 0 || y < 0 || x >= W || y >= H) return -1;
    return taken[(size_t)y * W + x];
  };
  std::vector<int64_t> acc;
  acc.reserve((size_t)n);
  for (int64_t p : order) {
    const int64_t x = u[p], y = v[p];
    if (x < 0 || y < 0 || x >= W || y >= H) {
      sthost::set_error("st_support_dedup: point (%lld, %lld) outside the image",
                        (long long)x, (long long)y);
      return ST_EINVAL;
    }
    if (at(x, y) >= 0) continue;
    bool conflict = false;
    for (int du = -1; du <= 1 && !conflict; ++du)
      for (int dv = -1; dv <= 1; ++dv) {
        const int64_t q = at(x + du, y + dv);
        if (q >= 0 && fabs(d[q] - d[p]) > 2.0) {
          conflict = true;
          break;
        }
      }
    if (conflict) continue;
    taken[(size_t)y * W + x] = p;
    acc.push_back(p);
  }
  // accepted.sort(key=(v, u, d)) -- one point per pixel, so (v, u) decides
  std::sort(acc.begin(), acc.end(), [&](int64_t a, int64_t b) {
    if (v[a] != v[b]) return v[a] < v[b];
    if (u[a] != u[b]) return u[a] < u[b];
    return d[a] < d[b];
  });
  for (size_t i = 0; i < acc.size(); ++i) keep[i] = acc[i];
  *n_keep = (int64_t)acc.size();
  return ST_OK;
}

}  // extern "C"
