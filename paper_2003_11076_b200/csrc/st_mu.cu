// Surface raster mu on the device (prior.py:276-310 disparity_map, then the
// solver's clip, solver.py:185-186) -- bit-exact with the reference.
//
// The reference evaluates the plane of the triangle scipy's Qhull
// `find_simplex` returns.  ~40 % of pixel centres lie on triangle edges or
// vertices (support points sit on an integer grid), and which of the touching
// triangles Qhull returns depends on its directed walk, which starts from the
// simplex found for the PREVIOUS query point (raster order).  The planes of
// the touching triangles differ by ulps, and those ulps move warped rays
// across the integer margin boundaries downstream, so the walk is emulated
// exactly:
//   1. k_claim: every triangle tests the pixel centres in its bbox with
//      Qhull's barycentric inclusion test (eps = 100 DBL_EPSILON, same
//      arithmetic); per pixel we keep the claim count and min/max claimer.
//      A pixel with exactly one claimer has a start-independent answer.
//   2. k_walk_chunks: runs of ambiguous pixels are cut into chunks at pixels
//      whose predecessor has <= 2 claimers; each chunk is walked once per
//      possible incoming start (the predecessor's claimers), replaying
//      _find_simplex / _find_simplex_directed step by step.
//      When both speculative walks end in the same simplex (the usual case)
//      the next chunk's start is decided right there.
//   3. k_resolve_chunks: the remaining links are followed forward from every
//      decided chunk (a few lookups each).
//   4. k_mu_eval: pick the resolved simplex, evaluate its plane left to
//      right, clip.
#include <cuda_runtime.h>
#include <float.h>
#include <limits.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include <cub/cub.cuh>

#include "st_common.cuh"

namespace st {

#define MU_CHUNK 8
#define QH_EPS (100.0 * DBL_EPSILON)

struct TriDev {
  const double *pts, *disp, *planes, *transform, *equations;
  const double* nb_eq;  // (n_tri, 3, 4): the neighbours' lifted facet equations (0 for none)
  double cen0, cen1;    // points.mean(axis=0) (numpy, host): the off-hull nudge target
  const int32_t *simp, *nb;
  int n_pts, n_tri;
  double ps, psh, lo0, lo1, hi0, hi1;
};

struct MuWs {
  unsigned *cnt, *tmin, *tmax;
  int32_t *res0, *res1, *final_s, *chunk_of, *len, *end0, *end1;
  uint8_t* chosen;
  unsigned long long *vmin, *vmax;  // range of the claimers' plane values (order keys)
  int32_t *chunks, *runs;  // worklists of chunk starts / run starts
  unsigned* counts;        // [0] chunks, [1] runs
  int chunk;  // chunk length for the speculative walks (MU_CHUNK, env ST_MU_CHUNK)
  unsigned* miss_bits;  // pixels the raster walk left outside the triangulation
  int32_t* miss_list;   // ... in pixel order (k_mu_nudge)
  // row window (st_mu_raster_rows): pixels [p_lo, p_hi) are rastered (the
  // band's rows plus a halo above), mu is written for [b_lo, p_hi); the whole
  // frame otherwise (p_lo = b_lo = 0, p_hi = W*H)
  int64_t p_lo, p_hi, b_lo;
};

// prior.py:296: pl[:, 0] * u + pl[:, 1] * v + pl[:, 2], left to right.
__device__ __forceinline__ double plane_at(const TriDev& d, int t, double u, double v) {
  const double* pl = d.planes + 3 * t;
  return dadd(dadd(dmul(pl[0], u), dmul(pl[1], v)), pl[2]);
}

// Doubles as unsigned keys with the same order (for atomicMin/atomicMax).
__device__ __forceinline__ unsigned long long order_key(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// scipy _barycentric_inside (ndim = 2), same operation order.
__device__ __forceinline__ bool bary_inside(const double* __restrict__ T, double x0, double x1) {
  const double eps = QH_EPS;
  double c2 = 1.0;
  double c0 = 0.0;
  c0 = dadd(c0, dmul(T[0], dsub(x0, T[4])));
  c0 = dadd(c0, dmul(T[1], dsub(x1, T[5])));
  c2 = dsub(c2, c0);
  if (!(-eps <= c0 && c0 <= 1.0 + eps)) return false;
  double c1 = 0.0;
  c1 = dadd(c1, dmul(T[2], dsub(x0, T[4])));
  c1 = dadd(c1, dmul(T[3], dsub(x1, T[5])));
  c2 = dsub(c2, c1);
  if (!(-eps <= c1 && c1 <= 1.0 + eps)) return false;
  return -eps <= c2 && c2 <= 1.0 + eps;
}

// Pixel-centre bbox of every triangle (empty for degenerate simplices) and
// its pixel count, scanned afterwards so the claim tests can be spread
// evenly over the grid (a few corner-anchor triangles span most of the
// image; one thread per triangle would serialise them).
__global__ void k_tri_bbox(TriDev d, int W, int H, int y_lo, int y_hi, int4* __restrict__ bbox,
                           unsigned long long* __restrict__ area) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.n_tri) return;
  const int a = d.simp[3 * t], b = d.simp[3 * t + 1], c = d.simp[3 * t + 2];
  const double ax = d.pts[2 * a], ay = d.pts[2 * a + 1];
  const double bx = d.pts[2 * b], by = d.pts[2 * b + 1];
  const double cx = d.pts[2 * c], cy = d.pts[2 * c + 1];
  const double* T = d.transform + 6 * t;
  int4 bb;
  bb.x = max(0, (int)ceil(fmin(ax, fmin(bx, cx)) - 1e-6));
  bb.z = min(W - 1, (int)floor(fmax(ax, fmax(bx, cx)) + 1e-6));
  bb.y = max(y_lo, (int)ceil(fmin(ay, fmin(by, cy)) - 1e-6));
  bb.w = min(y_hi - 1, (int)floor(fmax(ay, fmax(by, cy)) + 1e-6));
  unsigned long long n = 0;
  if (T[0] == T[0] && bb.x <= bb.z && bb.y <= bb.w)  // nan transform: degenerate simplex
    n = (unsigned long long)(bb.z - bb.x + 1) * (unsigned long long)(bb.w - bb.y + 1);
  bbox[t] = bb;
  area[t] = n;
}

#define CLAIM_ITEMS 16

// Flattened (triangle, bbox pixel) work items; `start` is the exclusive scan
// of the bbox areas (n_tri + 1 entries, start[n_tri] = total).
__global__ void k_claim(TriDev d, int W, const int4* __restrict__ bbox,
                        const unsigned long long* __restrict__ start, MuWs w) {
  const unsigned long long total = start[d.n_tri];
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x * CLAIM_ITEMS;
  for (unsigned long long i0 =
           ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) * CLAIM_ITEMS;
       i0 < total; i0 += stride) {
    // triangle owning item i0: last t with start[t] <= i0
    int lo = 0, hi = d.n_tri - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (start[mid] <= i0)
        lo = mid;
      else
        hi = mid - 1;
    }
    int t = lo;
    const unsigned long long i1 = min(i0 + CLAIM_ITEMS, total);
    for (unsigned long long i = i0; i < i1; ++i) {
      while (i >= start[t + 1]) ++t;
      const int4 bb = bbox[t];
      const int bw = bb.z - bb.x + 1;
      const unsigned long long local = i - start[t];
      const int x = bb.x + (int)(local % bw), y = bb.y + (int)(local / bw);
      if (bary_inside(d.transform + 6 * t, (double)x, (double)y)) {
        const size_t p = (size_t)y * W + x;
        atomicAdd(w.cnt + p, 1u);
        atomicMin(w.tmin + p, (unsigned)t);
        atomicMax(w.tmax + p, (unsigned)t);
        // range of the claimers' plane values at this pixel (order-preserving keys)
        const unsigned long long key = order_key(plane_at(d, t, (double)x, (double)y));
        atomicMin(w.vmin + p, key);
        atomicMax(w.vmax + p, key);
      }
    }
  }
}

// Neighbour equations gathered per simplex, so a paraboloid sweep reads
// them from its own simplex's row (one dependent load round per walk step
// instead of two: nb, then the neighbour's equation).
__global__ void k_nb_equations(TriDev d, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.n_tri) return;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int m = d.nb[3 * t + k];
#pragma unroll
    for (int i = 0; i < 4; ++i) out[12 * t + 4 * k + i] = m >= 0 ? d.equations[4 * m + i] : 0.0;
  }
}

// scipy _distplane on the lifted point, equation at e.
__device__ __forceinline__ double distplane_eq(const double* __restrict__ e, double z0, double z1,
                                               double z2) {
  double dist = __ldg(e + 3);
  dist = dadd(dist, dmul(__ldg(e), z0));
  dist = dadd(dist, dmul(__ldg(e + 1), z1));
  dist = dadd(dist, dmul(__ldg(e + 2), z2));
  return dist;
}

// scipy _distplane on the lifted point.
__device__ __forceinline__ double distplane(const TriDev& d, int s, double z0, double z1,
                                            double z2) {
  const double* e = d.equations + 4 * s;
  double dist = e[3];
  dist = dadd(dist, dmul(e[0], z0));
  dist = dadd(dist, dmul(e[1], z1));
  dist = dadd(dist, dmul(e[2], z2));
  return dist;
}

// The current simplex's walk tables, kept in registers across consecutive
// queries: along a run of edge pixels the walk almost always stays in (or
// returns to) the same simplex, so most steps need no memory access.
struct TriCache {
  int s = -1;
  double e0, e1, e2, e3;      // lifted facet equation
  double t0, t1, t2, t3, t4, t5;  // barycentric transform
  int n0, n1, n2;             // neighbours
  __device__ __forceinline__ void ensure(const TriDev& d, int t) {
    if (t == s) return;
    s = t;
    const double2* ep = reinterpret_cast<const double2*>(d.equations + 4 * t);
    const double2 a = __ldg(ep), b = __ldg(ep + 1);
    e0 = a.x; e1 = a.y; e2 = b.x; e3 = b.y;
    const double2* tp = reinterpret_cast<const double2*>(d.transform + 6 * t);
    const double2 x = __ldg(tp), y = __ldg(tp + 1), z = __ldg(tp + 2);
    t0 = x.x; t1 = x.y; t2 = y.x; t3 = y.y; t4 = z.x; t5 = z.y;
    n0 = __ldg(d.nb + 3 * t);
    n1 = __ldg(d.nb + 3 * t + 1);
    n2 = __ldg(d.nb + 3 * t + 2);
  }
  __device__ __forceinline__ int nb(int k) const { return k == 0 ? n0 : (k == 1 ? n1 : n2); }
  __device__ __forceinline__ double dist(double z0, double z1, double z2) const {
    double v = e3;
    v = dadd(v, dmul(e0, z0));
    v = dadd(v, dmul(e1, z1));
    v = dadd(v, dmul(e2, z2));
    return v;
  }
};

// _find_simplex + _find_simplex_directed for one query; `start` in/out.
// The brute-force fallback (lowest-index including simplex) is the claim
// pass's tmin.
// scipy _find_simplex_bruteforce for a point that is not a pixel centre
// (the nudged off-hull queries): the lowest-index simplex with a valid
// transform whose barycentric test passes.
__device__ int brute_force_simplex(const TriDev& d, double x0, double x1) {
  for (int t = 0; t < d.n_tri; ++t) {
    const double* T = d.transform + 6 * t;
    if (T[0] == T[0] && bary_inside(T, x0, x1)) return t;
  }
  return -1;
}

// p >= 0: pixel centre p (its claims give the brute-force answer);
// p < 0: any point (brute force: bf_hint when given, else by scanning the
// simplices).
__device__ int find_simplex(const TriDev& d, const MuWs& w, int64_t p, double x0, double x1,
                            int& start, TriCache& tc, int bf_hint = INT_MIN) {
  const double eps = QH_EPS;
  if (x0 < d.lo0 - eps || x0 > d.hi0 + eps || x1 < d.lo1 - eps || x1 > d.hi1 + eps) return -1;
  if (d.n_tri <= 0) return -1;
  double z2 = 0.0;
  z2 = dadd(z2, dmul(x0, x0));
  z2 = dadd(z2, dmul(x1, x1));
  z2 = dmul(z2, d.ps);
  z2 = dadd(z2, d.psh);
  int s = start;
  if (s < 0 || s >= d.n_tri) s = 0;
  tc.ensure(d, s);
  double best = tc.dist(x0, x1, z2);
  bool changed = true;
  while (changed) {
    if (best > 0.0) break;
    changed = false;
    // the three neighbours' distances, fetched in parallel; used as long as
    // s has not moved inside this sweep (scipy reads the neighbours of the
    // CURRENT s at every k)
    tc.ensure(d, s);
    const int s0 = s;
    double pre[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) pre[k] = distplane_eq(d.nb_eq + 12 * s0 + 4 * k, x0, x1, z2);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      tc.ensure(d, s);
      const int m = tc.nb(k);
      if (m == -1) continue;
      const double dd = s == s0 ? pre[k] : distplane_eq(d.nb_eq + 12 * s + 4 * k, x0, x1, z2);
      if (dd > dadd(best, dmul(eps, dadd(1.0, fabs(best))))) {
        s = m;
        best = dd;
        changed = true;
      }
    }
  }
  start = s;
  const int cycles = 1 + d.n_tri / 4;
  // Brent cycle detection: the directed step depends on s alone, so a
  // revisited simplex means the walk loops until the cap above and then
  // takes the brute-force answer -- which we can return at once.
  int saved = s, power = 1, lam = 0;
  for (int cyc = 0; cyc < cycles; ++cyc) {
    if (s == -1) {
      start = s;
      return s;
    }
    tc.ensure(d, s);
    int inside = 1;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;
    for (int k = 0; k < 3; ++k) {
      double ck;
      if (k == 0) {
        c0 = dadd(c0, dmul(tc.t0, dsub(x0, tc.t4)));
        c0 = dadd(c0, dmul(tc.t1, dsub(x1, tc.t5)));
        ck = c0;
      } else if (k == 1) {
        c1 = dadd(c1, dmul(tc.t2, dsub(x0, tc.t4)));
        c1 = dadd(c1, dmul(tc.t3, dsub(x1, tc.t5)));
        ck = c1;
      } else {
        c2 = 1.0;
        c2 = dsub(c2, c0);
        c2 = dsub(c2, c1);
        ck = c2;
      }
      if (ck < -eps) {
        const int m = tc.nb(k);
        if (m == -1) {
          start = s;  // outside the triangulation: bail out
          return -1;
        }
        s = m;
        inside = -1;
        break;
      } else if (ck <= 1.0 + eps) {
        // inside along this coordinate
      } else {
        inside = 0;  // outside or nan (degenerate)
      }
    }
    if (inside == -1) {
      if (s == saved) break;  // cycle: same result as exhausting the cap
      if (++lam == power) {
        saved = s;
        power <<= 1;
        lam = 0;
      }
      continue;
    }
    if (inside == 1) {
      start = s;
      return s;
    }
    s = p < 0 ? (bf_hint != INT_MIN ? bf_hint : brute_force_simplex(d, x0, x1))
              : w.cnt[p] ? (int)w.tmin[p] : -1;  // brute force
    start = s;
    return s;
  }
  // walk did not converge: brute force
  s = p < 0 ? (bf_hint != INT_MIN ? bf_hint : brute_force_simplex(d, x0, x1))
            : w.cnt[p] ? (int)w.tmin[p] : -1;
  start = s;
  return s;
}

__device__ __forceinline__ bool ambiguous(const MuWs& w, int64_t p) { return w.cnt[p] != 1u; }

// A chunk starts at an ambiguous pixel whose predecessor is unambiguous, at
// pixel 0, or every MU_CHUNK pixels where the predecessor has exactly two
// claimers (then the incoming start is one of those two).
__device__ __forceinline__ bool chunk_start(const MuWs& w, int64_t p) {
  if (!ambiguous(w, p)) return false;
  if (p == w.p_lo) return true;  // (pixel 0, or a row window's first pixel)
  if (!ambiguous(w, p - 1)) return true;
  return (p % w.chunk) == 0 && w.cnt[p - 1] == 2u;
}

// Dense worklists of chunk starts and run starts (warp-aggregated appends;
// list order is irrelevant: every entry owns disjoint pixels).
__device__ __forceinline__ void append_lane(bool want, int32_t v, int32_t* list,
                                            unsigned* count) {
  const unsigned ballot = __ballot_sync(0xffffffffu, want);
  if (!ballot) return;
  const int lane = threadIdx.x & 31, leader = __ffs(ballot) - 1;
  unsigned base = 0;
  if (lane == leader) base = atomicAdd(count, (unsigned)__popc(ballot));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (want) list[base + __popc(ballot & ((1u << lane) - 1))] = v;
}

// Per-pixel workspace reset (one pass instead of seven memsets): no claims,
// empty claimer/value ranges, every chunk undecided.
__global__ void k_mu_init(int64_t npx, MuWs w) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  (void)npx;
  for (int64_t p = w.p_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < w.p_hi;
       p += stride) {
    w.cnt[p] = 0u;
    w.tmin[p] = 0xffffffffu;
    w.tmax[p] = 0u;
    w.vmin[p] = ~0ull;
    w.vmax[p] = 0ull;
    w.chosen[p] = 0xff;
    if ((p & 31) == 0 || p == w.p_lo) w.miss_bits[p >> 5] = 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x < 8) w.counts[threadIdx.x] = 0u;
}

__global__ void k_mu_lists(int64_t npx, MuWs w) {
  (void)npx;
  const int64_t p = w.p_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = p < w.p_hi;
  const bool cs = in && chunk_start(w, p);
  append_lane(cs, (int32_t)p, w.chunks, w.counts);
}

#ifndef WALK_MIN_BLOCKS
#define WALK_MIN_BLOCKS 5  // <= 102 registers: no spills, measured best
#endif
__global__ void __launch_bounds__(128, WALK_MIN_BLOCKS)
    k_walk_chunks(TriDev d, int W, int64_t npx, MuWs w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)w.counts[0]) return;
  const int64_t p = w.chunks[t];
  int opts[2];
  int nopt;
  if (p == 0) {
    opts[0] = 0;  // find_simplex starts every batch at simplex 0
    nopt = 1;
  } else if (p == w.p_lo) {
    // a row window's first pixel: its predecessor was not rastered.  Any
    // start is a guess; k_mu_window_check flags the window when this run
    // reaches the band's own rows (the caller then rasters the whole frame)
    opts[0] = 0;
    nopt = 1;
  } else if (!ambiguous(w, p - 1)) {
    opts[0] = (int)w.tmin[p - 1];
    nopt = 1;
  } else {
    opts[0] = (int)w.tmin[p - 1];
    opts[1] = (int)w.tmax[p - 1];
    nopt = 2;
  }
  // A chunk whose pixels get bit-identical plane values from every claiming
  // simplex, and that ends its run (so no later walk starts from its end
  // state), cannot influence mu: skip the walk.  This is the common case
  // (including the image-corner vertices, whose walks start a full row away).
  int64_t end;
  bool ends_run;
  {
    int64_t q = p;
    bool agnostic = true;
    do {
      agnostic = agnostic && w.cnt[q] > 0 && w.vmin[q] == w.vmax[q];
      w.chunk_of[q] = (int32_t)p;
      ++q;
    } while (q < w.p_hi && ambiguous(w, q) && !chunk_start(w, q));
    end = q;
    ends_run = q >= w.p_hi || !ambiguous(w, q);
    if (agnostic && ends_run) {
      w.len[p] = (int32_t)(q - p);
      w.end0[p] = w.end1[p] = -1;  // never read: the run ends here
      return;
    }
  }
  if (nopt == 1) w.chosen[p] = 0;  // a run start: its incoming start is known
  // the chunk's extent is known from the scan: no per-pixel reload in the walk
  int st0 = opts[0], st1 = nopt > 1 ? opts[1] : 0;
  TriCache tc0, tc1;
  for (int64_t q = p; q < end; ++q) {
    const double x0 = (double)(q % W), x1 = (double)(q / W);
    w.res0[q] = find_simplex(d, w, q, x0, x1, st0, tc0);
    if (nopt > 1) w.res1[q] = find_simplex(d, w, q, x0, x1, st1, tc1);
  }
  const int64_t q = end;
  w.len[p] = (int32_t)(q - p);
  w.end0[p] = st0;
  w.end1[p] = nopt > 1 ? st1 : st0;
  // Both speculative walks ended in the same simplex (the usual, "sticky"
  // case): the next chunk's incoming start no longer depends on this
  // chunk's choice, so decide it here.
  if (w.end0[p] == w.end1[p] && !ends_run) {
    if ((int)w.tmin[q - 1] == st0)
      w.chosen[q] = 0;
    else if ((int)w.tmax[q - 1] == st0)
      w.chosen[q] = 1;
  }
}

// Links the chunks the walk kernel could not decide locally: from every
// decided chunk, follow the run forward while the next chunk is undecided.
__global__ void k_resolve_chunks(TriDev d, int W, int64_t npx, MuWs w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)w.counts[0]) return;
  int64_t c = w.chunks[t];
  uint8_t ch = w.chosen[c];
  if (ch == 0xff) return;  // undecided: resolved by the thread of a decided predecessor
  for (;;) {
    const int64_t nxt = c + w.len[c];
    if (nxt >= w.p_hi || !ambiguous(w, nxt) || w.chosen[nxt] != 0xff) break;
    const int carry = ch == 1 ? w.end1[c] : w.end0[c];  // (a replayed chunk keeps its end in end0)
    uint8_t pick;
    if ((int)w.tmin[nxt - 1] == carry) {
      pick = 0;
    } else if ((int)w.tmax[nxt - 1] == carry) {
      pick = 1;
    } else {
      // the incoming start is not a claimer of the predecessor (never seen
      // in practice): replay this chunk sequentially from the true start
      int st = carry;
      const int64_t e = nxt + w.len[nxt];
      TriCache tc;
      for (int64_t q = nxt; q < e; ++q)
        w.final_s[q] = find_simplex(d, w, q, (double)(q % W), (double)(q / W), st, tc);
      w.end0[nxt] = st;
      pick = 2;
    }
    w.chosen[nxt] = pick;
    c = nxt;
    ch = pick;
  }
}

__global__ void k_mu_eval(TriDev d, int W, int64_t npx, MuWs w, double clip_dmax,
                          double* __restrict__ mu) {
  (void)npx;
  const int64_t p = w.b_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= w.p_hi) return;
  int s;
  bool agnostic = false;
  if (!ambiguous(w, p)) {
    s = (int)w.tmin[p];
  } else if (w.cnt[p] > 0 && w.vmin[p] == w.vmax[p]) {
    s = 0;
    agnostic = true;  // every claimer yields the same value: no walk needed
  } else {
    const int64_t c = w.chunk_of[p];
    const uint8_t ch = w.chosen[c];
    s = ch == 0 ? w.res0[p] : ch == 1 ? w.res1[p] : w.final_s[p];
  }
  const double u = (double)(p % W), v = (double)(p / W);
  double m;
  if (agnostic) {
    m = key_value(w.vmin[p]);
    if (clip_dmax > 0.0) m = fmin(fmax(m, 1e-6), clip_dmax);
    mu[p] = m;
    return;
  }
  if (s >= 0) {
    // prior.py:296: pl[:, 0] * u + pl[:, 1] * v + pl[:, 2]
    const double* pl = d.planes + 3 * s;
    m = dadd(dadd(dmul(pl[0], u), dmul(pl[1], v)), pl[2]);
  } else {
    // off the hull after the raster walk: k_mu_nudge (prior.py:287-301)
    atomicOr(w.miss_bits + (p >> 5), 1u << (p & 31));
    w.counts[6] = 1u;  // (any miss: k_mu_nudge has work)
    return;
  }
  if (clip_dmax > 0.0) m = fmin(fmax(m, 1e-6), clip_dmax);
  mu[p] = m;
}

// prior.py:287-301 for the pixels the raster walk left outside the
// triangulation (s < 0): a second find_simplex batch on the points nudged
// 1e-9 toward the vertex centroid -- in pixel order, the walk start carried
// from one query to the next and starting at simplex 0, like scipy's -- and
// the nearest vertex for what is still outside.  The plane is evaluated at
// the original pixel centre.  One block: the bitmap is compacted in pixel
// order (block scan), then thread 0 walks the list.
#define NUDGE_CAP 16384
__global__ void __launch_bounds__(1024) k_mu_nudge(TriDev d, int W, int64_t npx, MuWs w,
                                                   double clip_dmax, double* __restrict__ mu) {
  __shared__ unsigned s_cnt[1024];
  if (w.counts[6] == 0u) return;  // the common case: every pixel found its simplex
  // The nudged batch carries its walk start from one off-hull pixel to the
  // next in pixel order, from simplex 0.  A window from pixel 0 replays its
  // own misses exactly (later ones cannot affect them).  A window further
  // down does not know the start its first miss inherits: its results are
  // still exact when every nudged point has at most one claiming triangle
  // (then any walk ends there, or outside for the nearest-vertex fallback),
  // which the block checks below; otherwise the window is flagged.
  const bool windowed = w.p_lo > 0;
  const int64_t word_lo = w.p_lo >> 5;
  const int64_t words = (w.p_hi + 31) / 32;
  const int64_t nw = words - word_lo;
  const int64_t per = (nw + blockDim.x - 1) / blockDim.x;
  const int64_t w0 = word_lo + (int64_t)threadIdx.x * per, w1 = min(w0 + per, words);
  const unsigned lo_mask = ~0u << (unsigned)(w.p_lo & 31);  // (bits below p_lo are stale)
  auto miss_word = [&](int64_t i) {
    const unsigned b = w.miss_bits[i];
    return i == word_lo ? (b & lo_mask) : b;
  };
  unsigned c = 0;
  for (int64_t i = w0; i < w1; ++i) c += __popc(miss_word(i));
  s_cnt[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scan (1024 entries)
    unsigned acc = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const unsigned x = s_cnt[i];
      s_cnt[i] = acc;
      acc += x;
    }
    w.counts[7] = acc;
  }
  __syncthreads();
  const unsigned total = w.counts[7];
  if (total == 0) return;
  if (total <= NUDGE_CAP) {
    unsigned o = s_cnt[threadIdx.x];
    for (int64_t i = w0; i < w1; ++i)
      for (unsigned b = miss_word(i); b; b &= b - 1) w.miss_list[o++] = (int32_t)(i * 32 + __ffs(b) - 1);
  } else if (windowed) {
    if (threadIdx.x == 0) w.counts[5] = 1u;  // (never seen) flag the window
    return;
  }
  __syncthreads();
  // vertex centroid (NaN from the host: integer coordinates, exact sums in
  // any order, then one division like numpy's mean)
  __shared__ double s_sum[2][1024];
  TriDev dd = d;
  if (!(d.cen0 == d.cen0)) {
    double a0 = 0.0, a1 = 0.0;
    for (int i = threadIdx.x; i < d.n_pts; i += blockDim.x) {
      a0 += d.pts[2 * i];
      a1 += d.pts[2 * i + 1];
    }
    s_sum[0][threadIdx.x] = a0;
    s_sum[1][threadIdx.x] = a1;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
      if ((int)threadIdx.x < h) {
        s_sum[0][threadIdx.x] += s_sum[0][threadIdx.x + h];
        s_sum[1][threadIdx.x] += s_sum[1][threadIdx.x + h];
      }
      __syncthreads();
    }
    dd.cen0 = ddiv(s_sum[0][0], (double)d.n_pts);
    dd.cen1 = ddiv(s_sum[1][0], (double)d.n_pts);
  }
  if (windowed) {
    // claimers of every nudged point (Qhull's inclusion test, as k_claim)
    __shared__ unsigned s_multi;
    if (threadIdx.x == 0) s_multi = 0u;
    __syncthreads();
    for (unsigned j = 0; j < total; ++j) {
      const int64_t p = w.miss_list[j];
      const double u = (double)(p % W), v = (double)(p / W);
      const double x0 = dadd(u, dmul(1e-9, dsub(dd.cen0, u)));
      const double x1 = dadd(v, dmul(1e-9, dsub(dd.cen1, v)));
      unsigned k = 0;
      for (int t = threadIdx.x; t < d.n_tri; t += blockDim.x)
        k += bary_inside(d.transform + 6 * t, x0, x1) ? 1u : 0u;
      k = __reduce_add_sync(0xffffffffu, k);
      if ((threadIdx.x & 31) == 0 && k) atomicAdd(&s_multi, k);
      __syncthreads();
      if (threadIdx.x == 0) {
        if (s_multi >= 2u) w.counts[5] = 1u;
        s_multi = 0u;
      }
      __syncthreads();
    }
  }
  if (threadIdx.x != 0) return;
  int start = 0;
  TriCache tc;
  int64_t wi = 0;
  unsigned bits = 0;
  for (unsigned j = 0; j < total; ++j) {
    int64_t p;
    if (total <= NUDGE_CAP) {
      p = w.miss_list[j];
    } else {  // (never seen in practice) scan the bitmap in order
      while (!bits) bits = w.miss_bits[wi++];
      p = (wi - 1) * 32 + __ffs(bits) - 1;
      bits &= bits - 1;
    }
    const double u = (double)(p % W), v = (double)(p / W);
    // q + 1e-9 * (centroid - q), numpy's elementwise order
    const double x0 = dadd(u, dmul(1e-9, dsub(dd.cen0, u)));
    const double x1 = dadd(v, dmul(1e-9, dsub(dd.cen1, v)));
    const int s = find_simplex(d, w, -1, x0, x1, start, tc);
    double m;
    if (s >= 0) {
      m = plane_at(d, s, u, v);
    } else {
      // cKDTree nearest vertex of the original point (first minimum)
      double best = INFINITY;
      int bi = 0;
      for (int i = 0; i < d.n_pts; ++i) {
        const double dx = d.pts[2 * i] - u, dy = d.pts[2 * i + 1] - v;
        const double d2 = dx * dx + dy * dy;
        if (d2 < best) {
          best = d2;
          bi = i;
        }
      }
      m = d.disp[bi];
    }
    if (clip_dmax > 0.0) m = fmin(fmax(m, 1e-6), clip_dmax);
    mu[p] = m;
  }
}

}  // namespace st

namespace {

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct MuLayout {
  size_t off[16];
  size_t bbox, area, start, nb_eq, miss_bits, miss_list, cub, cub_bytes;
  size_t total;
};

MuLayout mu_layout(int W, int H, int n_tri) {
  MuLayout L;
  const size_t npx = (size_t)W * H;
  size_t o = 0;
  const size_t sz[16] = {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 1, 4, 4, 0, 8, 8};
  for (int i = 0; i < 16; ++i) {
    L.off[i] = o;
    o += align_up(sz[i] ? sz[i] * npx : 256);  // the counts slot is fixed-size
  }
  const size_t nt = (size_t)(n_tri > 0 ? n_tri : 1) + 1;
  L.bbox = o;  o += align_up(sizeof(int4) * nt);
  L.area = o;  o += align_up(sizeof(unsigned long long) * nt);
  L.start = o; o += align_up(sizeof(unsigned long long) * nt);
  L.nb_eq = o; o += align_up(sizeof(double) * 12 * nt);
  L.miss_bits = o; o += align_up(sizeof(unsigned) * ((npx + 31) / 32));
  L.miss_list = o; o += align_up(sizeof(int32_t) * NUDGE_CAP);
  L.cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, L.cub_bytes, (unsigned long long*)nullptr,
                                (unsigned long long*)nullptr, (int)nt);
  L.cub = o;   o += align_up(L.cub_bytes);
  L.total = o;
  return L;
}

}  // namespace

// ---------------------------------------------------------------------------
// per-triangle LAPACK tables (see st_tri_tables in the header)

namespace st {

__global__ void k_tri_tables(const double* __restrict__ pts, const double* __restrict__ disp,
                             const int32_t* __restrict__ simp, int n_tri,
                             double* __restrict__ planes, double* __restrict__ transform,
                             int32_t* __restrict__ flags) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tri) return;
  int vtx[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) vtx[i] = simp[3 * t + i];
  // planes: dgesv on A = [u v 1] (rows = vertices), b = d
  double A[3][3], b[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    A[i][0] = pts[2 * vtx[i]];
    A[i][1] = pts[2 * vtx[i] + 1];
    A[i][2] = 1.0;
    b[i] = disp[vtx[i]];
  }
  int piv[3];
  bool zero_pivot = false;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
#pragma unroll
    for (int i = 0; i < j; ++i) {  // earlier row interchanges on column j
      if (piv[i] != i) {
        const double x = A[i][j];
        A[i][j] = A[piv[i]][j];
        A[piv[i]][j] = x;
      }
    }
#pragma unroll
    for (int i = 1; i < j; ++i) {  // U part: b[i] -= dot(L[i, :i], b[:i])
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) acc = __fma_rn(A[i][k], A[k][j], acc);
      A[i][j] = dsub(A[i][j], acc);
    }
    if (j > 0) {
#pragma unroll
      for (int i = j; i < 3; ++i) {  // gemv tail rows: dot, then subtract
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < j; ++k) acc = __fma_rn(A[i][k], A[k][j], acc);
        A[i][j] = dsub(A[i][j], acc);
      }
    }
    int p = j;  // idamax: first largest magnitude
#pragma unroll
    for (int i = j + 1; i < 3; ++i)
      if (fabs(A[i][j]) > fabs(A[p][j])) p = i;
    piv[j] = p;
    if (p != j) {
#pragma unroll
      for (int k = 0; k <= j; ++k) {
        const double x = A[j][k];
        A[j][k] = A[p][k];
        A[p][k] = x;
      }
    }
    if (A[j][j] == 0.0) {
      zero_pivot = true;
    } else {
      const double r = ddiv(1.0, A[j][j]);
#pragma unroll
      for (int i = j + 1; i < 3; ++i) A[i][j] = dmul(A[i][j], r);
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (piv[i] != i) {
      const double x = b[i];
      b[i] = b[piv[i]];
      b[piv[i]] = x;
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)  // trsv, unit lower
#pragma unroll
    for (int k = i + 1; k < 3; ++k) b[k] = __fma_rn(-b[i], A[k][i], b[k]);
#pragma unroll
  for (int i = 2; i >= 0; --i) {  // trsv, upper: divide, then axpy
    b[i] = ddiv(b[i], A[i][i]);
#pragma unroll
    for (int k = 0; k < i; ++k) b[k] = __fma_rn(-b[i], A[k][i], b[k]);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) planes[3 * t + i] = b[i];
  if (zero_pivot) atomicOr(flags, 1);

  // transform: M = T^T, M[j][i] = points[s[j]][i] - points[s[2]][i]
  const double r0 = pts[2 * vtx[2]], r1 = pts[2 * vtx[2] + 1];
  double m00 = dsub(pts[2 * vtx[0]], r0), m01 = dsub(pts[2 * vtx[0] + 1], r1);
  double m10 = dsub(pts[2 * vtx[1]], r0), m11 = dsub(pts[2 * vtx[1] + 1], r1);
  // integer coordinates: flat <=> exact determinant 0 (scipy: NaN rows)
  const long long det = (long long)m00 * (long long)m11 - (long long)m10 * (long long)m01;
  double* T = transform + 6 * t;
  if (det == 0) {
#pragma unroll
    for (int i = 0; i < 6; ++i) T[i] = NAN;
    return;
  }
  const bool sw = fabs(m10) > fabs(m00);
  if (sw) {
    double x = m00;
    m00 = m10;
    m10 = x;
    x = m01;
    m01 = m11;
    m11 = x;
  }
  const double l = dmul(m10, ddiv(1.0, m00));
  const double u11 = dsub(m11, dmul(l, m01));
  const double iu00 = ddiv(1.0, m00), iu11 = ddiv(1.0, u11);
  double X[2][2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    double y0 = c == 0 ? 1.0 : 0.0, y1 = c == 1 ? 1.0 : 0.0;
    if (sw) {
      const double x = y0;
      y0 = y1;
      y1 = x;
    }
    y1 = __fma_rn(-y0, l, y1);
    y1 = dmul(y1, iu11);
    y0 = __fma_rn(-y1, m01, y0);
    y0 = dmul(y0, iu00);
    X[0][c] = y0;
    X[1][c] = y1;
  }
  T[0] = X[0][0];
  T[1] = X[1][0];
  T[2] = X[0][1];
  T[3] = X[1][1];
  T[4] = r0;
  T[5] = r1;
}

}  // namespace st

extern "C" int st_tri_tables(const st_tri* tri, double* planes_out, double* transform_out,
                             int32_t* flags, void* stream) {
  if (!tri || tri->n_tri < 0) {
    sthost::set_error("st_tri_tables: bad triangulation");
    return ST_EINVAL;
  }
  if (tri->n_tri == 0) return ST_OK;
  st::k_tri_tables<<<(tri->n_tri + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
      tri->points, tri->disparities, tri->simplices, tri->n_tri, planes_out, transform_out,
      flags);
  ST_LAUNCH_CHECK("k_tri_tables");
  return ST_OK;
}

namespace st {
// A row window is exact when the run of ambiguous pixels that starts at its
// first pixel (whose walk start was guessed) ends before the band's rows;
// otherwise flag it (counts[5]).  One thread: at most the halo rows.
__global__ void k_mu_window_check(MuWs w, int32_t* __restrict__ unsafe_out, int force) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned bad = w.counts[5] | (unsigned)force;
  if (w.p_lo > 0 && w.p_lo < w.b_lo) {
    int64_t q = w.p_lo;
    while (q < w.b_lo && ambiguous(w, q)) ++q;
    if (q >= w.b_lo) bad = 1u;
  } else if (w.p_lo > 0) {
    bad = 1u;  // no halo at all
  }
  w.counts[5] = bad;
  if (unsafe_out) *unsafe_out = (int32_t)bad;
}
}  // namespace st

extern "C" int64_t st_mu_raster_workspace(int32_t W, int32_t H, int32_t n_tri) {
  return (int64_t)mu_layout(W, H, n_tri).total;
}

extern "C" int st_mu_raster_rows(const st_tri* tri, int32_t W, int32_t H, double clip_dmax,
                                 double* mu_out, void* workspace, int64_t workspace_bytes,
                                 int32_t row0, int32_t row1, int32_t* unsafe_out,
                                 void* stream);

extern "C" int st_mu_raster(const st_tri* tri, int32_t W, int32_t H, double clip_dmax,
                            double* mu_out, void* workspace, int64_t workspace_bytes,
                            void* stream) {
  return st_mu_raster_rows(tri, W, H, clip_dmax, mu_out, workspace, workspace_bytes, 0, H,
                           nullptr, stream);
}

#define MU_HALO_ROWS 2  // rows rastered above a band (their walks seed the band's)

extern "C" int st_mu_raster_rows(const st_tri* tri, int32_t W, int32_t H, double clip_dmax,
                                 double* mu_out, void* workspace, int64_t workspace_bytes,
                                 int32_t row0, int32_t row1, int32_t* unsafe_out,
                                 void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!(0 <= row0 && row0 < row1 && row1 <= H)) {
    sthost::set_error("st_mu_raster_rows: bad rows [%d, %d) of %d", row0, row1, H);
    return ST_EINVAL;
  }
  const MuLayout L = mu_layout(W, H, tri->n_tri);
  if ((int64_t)L.total > workspace_bytes) {
    sthost::set_error("mu raster workspace too small");
    return ST_ENOMEM;
  }
  if (tri->n_pts < 1) {
    sthost::set_error("degenerate support set: no support points");
    return ST_EINVAL;
  }
  if (!tri->neighbors || !tri->transform || !tri->equations) {
    sthost::set_error("st_mu_raster needs the Delaunay walk tables (neighbors, transform, "
                      "equations)");
    return ST_EINVAL;
  }
  char* ws = (char*)workspace;
  st::MuWs w;
  w.cnt = (unsigned*)(ws + L.off[0]);
  w.tmin = (unsigned*)(ws + L.off[1]);
  w.tmax = (unsigned*)(ws + L.off[2]);
  w.res0 = (int32_t*)(ws + L.off[3]);
  w.res1 = (int32_t*)(ws + L.off[4]);
  w.final_s = (int32_t*)(ws + L.off[5]);
  w.chunk_of = (int32_t*)(ws + L.off[6]);
  w.len = (int32_t*)(ws + L.off[7]);
  w.end0 = (int32_t*)(ws + L.off[8]);
  w.end1 = (int32_t*)(ws + L.off[9]);
  w.chosen = (uint8_t*)(ws + L.off[10]);
  w.chunks = (int32_t*)(ws + L.off[11]);
  w.runs = (int32_t*)(ws + L.off[12]);
  w.counts = (unsigned*)(ws + L.off[13]);
  w.vmin = (unsigned long long*)(ws + L.off[14]);
  w.vmax = (unsigned long long*)(ws + L.off[15]);
  w.miss_bits = (unsigned*)(ws + L.miss_bits);
  w.miss_list = (int32_t*)(ws + L.miss_list);
  const int y_lo = row0 > 0 ? std::max(0, row0 - MU_HALO_ROWS) : 0;
  w.p_lo = (int64_t)y_lo * W;
  w.b_lo = (int64_t)row0 * W;
  w.p_hi = (int64_t)row1 * W;
  static const int chunk_env = [] {
    const char* e = getenv("ST_MU_CHUNK");
    const int v = e ? atoi(e) : 0;
    return v >= 2 ? v : MU_CHUNK;
  }();
  w.chunk = chunk_env;
  st::TriDev d;
  d.pts = tri->points;
  d.disp = tri->disparities;
  d.planes = tri->planes;
  d.transform = tri->transform;
  d.equations = tri->equations;
  d.simp = tri->simplices;
  d.nb = tri->neighbors;
  d.n_pts = tri->n_pts;
  d.n_tri = tri->n_tri;
  d.ps = tri->paraboloid_scale;
  d.psh = tri->paraboloid_shift;
  d.lo0 = tri->min_bound[0];
  d.lo1 = tri->min_bound[1];
  d.hi0 = tri->max_bound[0];
  d.hi1 = tri->max_bound[1];
  d.nb_eq = (const double*)(ws + L.nb_eq);
  d.cen0 = tri->centroid[0];
  d.cen1 = tri->centroid[1];
  const int64_t npx = (int64_t)W * H;
  static const bool prof_on = getenv("ST_MU_PROFILE") != nullptr;  // diagnostics
  cudaEvent_t pev[8];
  int npev = 0;
  auto prof = [&]() {
    if (prof_on && npev < 8) {
      cudaEventCreate(&pev[npev]);
      cudaEventRecord(pev[npev++], s);
    }
  };
  prof();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  st::k_mu_init<<<sms * 8, 256, 0, s>>>(npx, w);
  ST_LAUNCH_CHECK("k_mu_init");
  if (d.n_tri > 0) {
    int4* bbox = (int4*)(ws + L.bbox);
    auto* area = (unsigned long long*)(ws + L.area);
    auto* start = (unsigned long long*)(ws + L.start);
    prof();
    ST_CUDA_CHECK(cudaMemsetAsync(area + d.n_tri, 0, sizeof(unsigned long long), s));
    st::k_tri_bbox<<<(d.n_tri + 127) / 128, 128, 0, s>>>(d, W, H, y_lo, row1, bbox, area);
    ST_LAUNCH_CHECK("k_tri_bbox");
    st::k_nb_equations<<<(d.n_tri + 127) / 128, 128, 0, s>>>(d, (double*)(ws + L.nb_eq));
    ST_LAUNCH_CHECK("k_nb_equations");
    size_t tb = L.cub_bytes;
    ST_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ws + L.cub, tb, area, start, d.n_tri + 1, s));
    sthost::count_launch();
    st::k_claim<<<sms * 8, 256, 0, s>>>(d, W, bbox, start, w);
    ST_LAUNCH_CHECK("k_claim");
  }
  const int64_t wpx = w.p_hi - w.p_lo;  // rastered pixels
  const unsigned blocks = (unsigned)((wpx + 255) / 256);
  prof();
  st::k_mu_lists<<<blocks, 256, 0, s>>>(npx, w);
  ST_LAUNCH_CHECK("k_mu_lists");
  prof();
  // worklist grids are sized for the worst case; surplus threads exit at once
  st::k_walk_chunks<<<(unsigned)((wpx + 127) / 128), 128, 0, s>>>(d, W, npx, w);
  ST_LAUNCH_CHECK("k_walk_chunks");
  prof();
  st::k_resolve_chunks<<<(unsigned)((wpx + 127) / 128), 128, 0, s>>>(d, W, npx, w);
  ST_LAUNCH_CHECK("k_resolve_chunks");
  prof();
  st::k_mu_eval<<<(unsigned)((w.p_hi - w.b_lo + 255) / 256), 256, 0, s>>>(d, W, npx, w,
                                                                          clip_dmax, mu_out);
  ST_LAUNCH_CHECK("k_mu_eval");
  st::k_mu_nudge<<<1, 1024, 0, s>>>(d, W, npx, w, clip_dmax, mu_out);
  ST_LAUNCH_CHECK("k_mu_nudge");
  if (row0 > 0 || row1 < H || unsafe_out) {
    // (ST_MU_FORCE_UNSAFE: test hook for the whole-frame retry of row bands)
    static const int force = getenv("ST_MU_FORCE_UNSAFE") != nullptr ? 1 : 0;
    st::k_mu_window_check<<<1, 32, 0, s>>>(w, unsafe_out, (row0 > 0 || row1 < H) ? force : 0);
    ST_LAUNCH_CHECK("k_mu_window_check");
  }
  prof();
  if (prof_on && npev > 1) {
    cudaEventSynchronize(pev[npev - 1]);
    fprintf(stderr, "mu_raster stages (ms): memset/bbox/claim/lists/walk/resolve/eval:");
    for (int i = 1; i < npev; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, pev[i - 1], pev[i]);
      fprintf(stderr, " %.4f", ms);
    }
    unsigned cnts[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpy(cnts, w.counts, sizeof(cnts), cudaMemcpyDeviceToHost);
    fprintf(stderr, "  chunks %u off-hull %u\n", cnts[0], cnts[7]);
    for (int i = 0; i < npev; ++i) cudaEventDestroy(pev[i]);
  }
  return ST_OK;
}
