// EM core of the seethrough_b200 hot path (sm_100a).
//
// Reference: solver.py (DisparitySolver) -- gather_rays :206-227, _energy
// :229-260, m_step :325-407, e_step :115-157, e_step_at :409-419,
// initial_masks :421-432.  One thread owns one reference pixel (the
// reference's per-pixel independence, solver.py:30-32); candidate energies
// never leave registers (no cost volume in HBM).
#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <stdint.h>

#include "st_common.cuh"
#include "st_em.cuh"
#include "st_pw.cuh"

#include <cub/block/block_scan.cuh>

namespace st {

// ---------------------------------------------------------------------------
// sampling

// Prior-plane sample (float32 plane, one channel).
__device__ __forceinline__ double sample_prior(const float* __restrict__ plane, int W,
                                               const Taps& t) {
  const size_t base = (size_t)t.iv * W + t.iu;
  const double top = lerp_f32(__ldg(plane + base), __ldg(plane + base + t.su), t.fu);
  if (t.fv == 0.0) return top;
  const double bot =
      lerp_f32(__ldg(plane + base + t.sv), __ldg(plane + base + t.sv + t.su), t.fu);
  return dadd(top, dmul(t.fv, dsub(bot, top)));
}

// Warp with the rectified-rig shortcut (identical roundings, see make_ctx).
__device__ __forceinline__ WarpOut warp_ctx(const EmCtx& c, int k, double u, double v,
                                            double d) {
  if (c.rectified) {
    WarpOut o;
    o.pu = dadd(u, dmul(d, c.rig.warp_b[k][0]));
    o.pv = v;
    o.front = true;
    return o;
  }
  return warp_to(c.rig, k, u, v, d);
}

// Tap selection for an in-margin ray.  On rectified rigs the clip and the
// min(., n - 2) of sampling.py are no-ops inside the margin and v is an
// integer row, so the taps reduce to floor(pu) and a zero vertical weight.
__device__ __forceinline__ Taps taps_ctx(const EmCtx& c, const WarpOut& w) {
  if (c.rectified) {
    Taps t;
    const double fl = floor(w.pu);
    t.iu = (int)fl;
    t.fu = dsub(w.pu, fl);
    t.iv = (int)w.pv;
    t.fv = 0.0;
    t.su = 1;
    t.sv = c.W;
    return t;
  }
  return taps_of(w.pu, w.pv, c.W, c.H);
}

// ---------------------------------------------------------------------------
// energy (solver.py:229-260)

struct Energy {
  double e;
  bool real;
  int n;  // descriptor samples taken (static in-margin rays of a real candidate)
};

#ifdef ENERGY_TWO_PASS
// Channels 4p..4p+3 and 8+4p..8+4p+3 of one descriptor sample (words p and
// p + 2), with exactly sample_desc's arithmetic.
__device__ __forceinline__ void sample_words(const uint4* __restrict__ plane, int W,
                                             const Taps& t, int p, double (&f)[8]) {
  const size_t base = (size_t)t.iv * W + t.iu;
  const uint4 a = __ldg(plane + base), b = __ldg(plane + base + t.su);
  const uint32_t aw[2] = {p ? a.y : a.x, p ? a.w : a.z};
  const uint32_t bw[2] = {p ? b.y : b.x, p ? b.w : b.z};
  if (t.fv == 0.0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double g[4];
      lerp_word(aw[h], bw[h], t.fu, g);
#pragma unroll
      for (int j = 0; j < 4; ++j) f[4 * h + j] = g[j];
    }
  } else {
    const uint4 e = __ldg(plane + base + t.sv), g = __ldg(plane + base + t.sv + t.su);
    const uint32_t ew[2] = {p ? e.y : e.x, p ? e.w : e.z};
    const uint32_t gw[2] = {p ? g.y : g.x, p ? g.w : g.z};
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int sh = 8 * j;
        const double top = lerp_u8((aw[h] >> sh) & 0xff, (bw[h] >> sh) & 0xff, t.fu);
        const double bot = lerp_u8((ew[h] >> sh) & 0xff, (gw[h] >> sh) & 0xff, t.fu);
        f[4 * h + j] = dadd(top, dmul(t.fv, dsub(bot, top)));
      }
  }
}

// Same result as the single-pass form below with half the live channel
// sums: a cheap count of the static in-margin rays first (too few -> the
// penalty energy without sampling), then numpy's reduction tree in two
// passes -- words {0, 2} give r0..r3, words {1, 3} give r4..r7.
__device__ __forceinline__ Energy energy_at(const EmCtx& c, double u, double v, double d,
                                            uint32_t bits, double lp) {
  int cnt = 0;
  for (int k = 0; k < c.rig.num_views; ++k)
    if (((bits >> k) & 1u) && in_margin(c.rig, k, warp_ctx(c, k, u, v, d))) ++cnt;
  Energy out;
  out.real = cnt >= c.p.min_static_rays;
  out.n = out.real ? cnt : 0;
  if (!out.real) {
    out.e = dsub(dmul(c.p.beta, variance_ceiling()), lp);
    return out;
  }
  const double nn = (double)cnt;
  const double rn = c.recip[cnt];
  double half[2];
#pragma unroll 1
  for (int p = 0; p < 2; ++p) {
    double s1[8], s2[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s1[i] = 0.0;
      s2[i] = 0.0;
    }
    for (int k = 0; k < c.rig.num_views; ++k) {
      if (!((bits >> k) & 1u)) continue;
      const WarpOut w = warp_ctx(c, k, u, v, d);
      if (!in_margin(c.rig, k, w)) continue;
      double f[8];
      sample_words(c.desc + (size_t)k * c.HW, c.W, taps_ctx(c, w), p, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s1[i] = dadd(s1[i], f[i]);
        s2[i] = dadd(s2[i], dmul(f[i], f[i]));
      }
    }
    double r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      r[j] = dadd(dsub(s2[j], div_small(dmul(s1[j], s1[j]), nn, rn)),
                  dsub(s2[4 + j], div_small(dmul(s1[4 + j], s1[4 + j]), nn, rn)));
    half[p] = dadd(dadd(r[0], r[1]), dadd(r[2], r[3]));
  }
  const double var = fmax(div_small(dadd(half[0], half[1]), nn, rn), 0.0);
  out.e = dsub(dmul(c.p.beta, var), lp);
  return out;
}
#else
__device__ __forceinline__ Energy energy_at(const EmCtx& c, double u, double v, double d,
                                            uint32_t bits, double lp) {
  double s1[16], s2[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    s1[i] = 0.0;
    s2[i] = 0.0;
  }
  int cnt = 0;
  for (int k = 0; k < c.rig.num_views; ++k) {
    if (!((bits >> k) & 1u)) continue;
    const WarpOut w = warp_ctx(c, k, u, v, d);
    if (!in_margin(c.rig, k, w)) continue;
    const Taps t = taps_ctx(c, w);
    sample_desc(c.desc + (size_t)k * c.HW, c.W, t, [&](int ch, double f) {
      s1[ch] = dadd(s1[ch], f);
      s2[ch] = dadd(s2[ch], dmul(f, f));
    });
    ++cnt;
  }
  Energy out;
  out.real = cnt >= c.p.min_static_rays;
  out.n = cnt;
  double var;
  if (out.real) {
    const double nn = (double)cnt;
    const double rn = c.recip[cnt];
    double t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = dsub(s2[i], div_small(dmul(s1[i], s1[i]), nn, rn));
    // numpy's contiguous 16-wide reduction: r_j = t_j + t_{j+8}, then the
    // ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)) tree.
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = dadd(t[j], t[j + 8]);
    const double sum = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])),
                            dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
    var = fmax(div_small(sum, nn, rn), 0.0);
  } else {
    var = variance_ceiling();
  }
  out.e = dsub(dmul(c.p.beta, var), lp);
  return out;
}
#endif

// ---------------------------------------------------------------------------
// Rectified rigs: cached taps (k_m_step).
//
// On a rectified rig a ray's bilinear taps are one descriptor index and a
// horizontal weight.  The count pass that decides `real` (solver.py:244-250)
// stores them per thread in shared memory (column `threadIdx.x`, stride
// EM_BLOCK), so the two channel passes of the energy do not re-warp.

struct TapCol {
  uint32_t* off;  // k * HW + row * W + floor(pu), static in-margin views in view order
  double* f64;    // fu = pu - floor(pu)
};

__device__ __forceinline__ int rect_taps(const EmCtx& c, double u, double v, double d,
                                         uint32_t bits, const TapCol& t) {
  int cnt = 0;
  const uint32_t row = (uint32_t)v * (uint32_t)c.W;
  for (int k = 0; k < c.rig.num_views; ++k) {
    if (!((bits >> k) & 1u)) continue;
    const WarpOut w = warp_ctx(c, k, u, v, d);
    if (!in_margin(c.rig, k, w)) continue;
    const double fl = floor(w.pu);
    const double fu = dsub(w.pu, fl);
    t.off[cnt * EM_BLOCK] = (uint32_t)k * (uint32_t)c.HW + row + (uint32_t)(int)fl;
    t.f64[cnt * EM_BLOCK] = fu;
    ++cnt;
  }
  return cnt;
}

// Exact energy of a real candidate from the cached taps: the arithmetic of
// energy_at (two passes along numpy's reduction tree) on the same samples.
__device__ __forceinline__ double rect_energy(const EmCtx& c, int cnt, const TapCol& t,
                                              double lp) {
  const double nn = (double)cnt;
  const double rn = c.recip[cnt];
  double half[2];
#pragma unroll 1
  for (int p = 0; p < 2; ++p) {
    double s1[8], s2[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s1[i] = 0.0;
      s2[i] = 0.0;
    }
    for (int j = 0; j < cnt; ++j) {
      const uint4* pl = c.desc + t.off[j * EM_BLOCK];
      const uint4 a = __ldg(pl), b = __ldg(pl + 1);
      const double fu = t.f64[j * EM_BLOCK];
      const uint32_t aw[2] = {p ? a.y : a.x, p ? a.w : a.z};
      const uint32_t bw[2] = {p ? b.y : b.x, p ? b.w : b.z};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double g[4];
        lerp_word(aw[h], bw[h], fu, g);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          s1[4 * h + q] = dadd(s1[4 * h + q], g[q]);
          s2[4 * h + q] = dadd(s2[4 * h + q], dmul(g[q], g[q]));
        }
      }
    }
    double r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      r[j] = dadd(dsub(s2[j], div_small(dmul(s1[j], s1[j]), nn, rn)),
                  dsub(s2[4 + j], div_small(dmul(s1[4 + j], s1[4 + j]), nn, rn)));
    half[p] = dadd(dadd(r[0], r[1]), dadd(r[2], r[3]));
  }
  const double var = fmax(div_small(dadd(half[0], half[1]), nn, rn), 0.0);
  return dsub(dmul(c.p.beta, var), lp);
}

// ---------------------------------------------------------------------------
// block-deterministic reductions

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  return x;
}

// Warp-aggregated append of `slot` to a worklist (one atomic per warp).  The
// list order depends on scheduling; every consumer's per-slot result does
// not, and statistics are summed per slot elsewhere, so results stay
// deterministic.
__device__ __forceinline__ void list_append(bool want, int32_t slot, int32_t* list,
                                            uint32_t* count) {
  const unsigned ballot = __ballot_sync(0xffffffffu, want);
  if (!ballot) return;
  const int lane = threadIdx.x & 31;
  unsigned base = 0;
  if (lane == __ffs(ballot) - 1) base = atomicAdd(count, (unsigned)__popc(ballot));
  base = __shfl_sync(0xffffffffu, base, __ffs(ballot) - 1);
  if (want) list[base + __popc(ballot & ((1u << lane) - 1))] = slot;
}

// ---------------------------------------------------------------------------
// M-step (solver.py:325-407).  Incremental EM: m_step is a pure function of
// (pixel, static mask) -- the candidate set is fixed per solve -- so from the
// second iteration on only slots whose mask changed since their last M-step
// are recomputed (k_flag_mstep builds that worklist); the others keep d, E and
// status bit for bit, and the previous-disparity energy of solve()
// (solver.py:468-471) equals their stored E.  Worked slots also get the
// previous-disparity energy and the |d - d_prev| > 0.5 flag here, and append
// themselves to the E-step worklist when their d changed (e_step_at is a pure
// function of (pixel, d)).

__global__ void MSTEP_BOUNDS k_m_step(EmCtx c, MStepArgs a) {
  if (a.stop && *a.stop) return;  // converged (st_solve_async)
  const int64_t n_work = a.list ? (int64_t)*a.list_count : a.n_dev ? (int64_t)*a.n_dev : a.n;
  long long n_cand = 0, n_eval = 0, n_hopeless = 0, n_samples = 0;
  __shared__ uint32_t s_off[ST_MAX_VIEWS * EM_BLOCK];
  __shared__ double s_f64[ST_MAX_VIEWS * EM_BLOCK];
  const TapCol tc = {s_off + threadIdx.x, s_f64 + threadIdx.x};
  // penalty energy term beta * VARIANCE_CEILING (solver.py:44, 252-256)
  const double pen = dmul(c.p.beta, variance_ceiling());
  // Exact energy (and `real`) of one candidate.  A pixel whose static mask
  // has fewer than min_static_rays views (`hopeless`) can have no real
  // candidate: every energy is the penalty minus the log prior, no sampling.
  auto energy = [&](double u, double v, double d, uint32_t bits, bool hopeless, double lp,
                    Energy& E) {
    if (hopeless) {
      E.real = false;
      E.n = 0;
      E.e = dsub(pen, lp);
    } else if (!c.rectified) {
      E = energy_at(c, u, v, d, bits, lp);
    } else {
      const int cnt = rect_taps(c, u, v, d, bits, tc);
      E.real = cnt >= c.p.min_static_rays;
      E.n = E.real ? cnt : 0;
      E.e = E.real ? rect_energy(c, cnt, tc, lp) : dsub(pen, lp);
    }
    n_samples += E.n;
  };
  // block-uniform grid-stride loop: one wave of blocks can cover a worklist
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_work;
       base += (int64_t)gridDim.x * blockDim.x) {
  const int64_t t = base + threadIdx.x;
  const bool live = t < n_work;
  const int64_t i = live ? (a.list ? (int64_t)a.list[t] : t) : 0;
  bool want_e = false;

  if (live) {
    const int64_t pix = a.active ? a.active[i] : c.pix0 + i;
    const int x = (int)(pix % c.W), y = (int)(pix / c.W);
    const double u = (double)x, v = (double)y;
    const double mu = c.mu[pix];
    const uint32_t bits = a.static_all[pix];
    const double dmax = c.p.d_max;
    const bool hopeless = __popc(bits & c.view_bits) < c.p.min_static_rays;
    n_hopeless += hopeless;
    // Pruning radius of an incumbent energy.  Real candidates: E >= -lp
    // (var >= 0, solver.py:341-347).  Hopeless pixels: E = fl(pen - lp), and
    // fl is monotone, so a candidate can only tie the incumbent when
    // -lp <= (be - pen) + one rounding of pen (the slack), i.e. only
    // candidates within a hair of the best prior survive.
    auto radius = [&](double best) -> double {
      if (c.exhaustive) return INFINITY;
      if (!hopeless) return prune_radius(best, c.sigma_f, c.gamma_f);
      return prune_radius(dadd(dsub(best, pen), 1e-12 * (1.0 + fabs(pen))), c.sigma_f,
                          c.gamma_f);
    };

    double be = INFINITY, bd = INFINITY;
    bool br = false;
    double lim = INFINITY;  // pruning radius of the current incumbent
    // Iterations >= 2: the previous disparity is one of this pixel's
    // candidates (the set is fixed per solve) and its energy under the new
    // mask is needed for the statistics anyway (solver.py:468-471).  The
    // winner is the order-independent lexicographic (E, d) minimum, so
    // evaluating it first only seeds the incumbent -- and the pruning.
    double dp = NAN, pe = NAN;
    if (!a.first) {
      dp = a.d[i];  // previous disparity (in place)
      if (!isnan(dp)) {
        Energy E;
        energy(u, v, dp, bits, hopeless, log_prior(dp, mu, c.p.sigma, c.p.gamma, c.inv_sigma),
               E);
        pe = E.e;
        be = E.e;
        bd = dp;
        br = E.real;
        lim = radius(be);
      }
    }
    auto offer = [&](double d) {
      ++n_cand;
      // -log prior bounds the energy from below (var >= 0): exact pruning
      // (solver.py:341-347).  Candidates beyond the incumbent's radius are
      // certainly pruned; the rest get the exact fp64 comparison.
      if (fabs(d - mu) > lim || d == bd) return;  // (d == bd: same energy, no change)
      const double lp = log_prior(d, mu, c.p.sigma, c.p.gamma, c.inv_sigma);
      if (!(-lp <= be) && !c.exhaustive) return;
      ++n_eval;
      Energy E;
      energy(u, v, d, bits, hopeless, lp, E);
      if (E.e < be || (E.e == be && d < bd)) {
        be = E.e;
        bd = d;
        br = E.real;
        lim = radius(be);
      }
    };

    // support disparities within the radius (solver.py:286-321, 373-400)
    auto support = [&]() {
      if (!c.sup_tile_start) return;
      // one bit test per distinct support value of the pixel's tile
      const int tile = (y / ST_TH) * c.tiles_x + (x / ST_TW);
      const uint32_t g1 = __ldg(c.sup_tile_start + tile + 1);
      const int row = y % ST_TH, col = x % ST_TW;
      for (uint32_t g = __ldg(c.sup_tile_start + tile); g < g1; ++g)
        if ((__ldg(c.sup_mask + (size_t)g * ST_TH + row) >> col) & 1u)
          offer((double)__ldg(c.sup_value + g));
    };
    // band mu + 0.5 j, nearest first (solver.py:187-191, 360-363)
    for (int j = 0; j < c.n_band; ++j) {
      const double d = dadd(mu, c.band[j]);
      if (d > 0.0 && d <= dmax) offer(d);
    }
    // coarse sweep 1, 5, 9, ... (solver.py:192, 364-365)
    for (int j = 0; j < c.n_coarse; ++j) offer(dadd(1.0, dmul(4.0, (double)j)));
    support();

    uint8_t status = ST_STATUS_VALID;
    if (!isfinite(be)) {
      status = ST_STATUS_LOW_TEXTURE;
      bd = NAN;
    } else if (!br) {
      status = ST_STATUS_NO_STATIC_EVIDENCE;
    }
    if (!a.first) {
      a.pe[i] = pe;
      // |d - d_prev| > 0.5 with NaN -> False (solver.py:472-475)
      a.chg[i] = fabs(bd - dp) > 0.5 ? 1 : 0;
      want_e = status != ST_STATUS_LOW_TEXTURE &&
               __double_as_longlong(bd) != __double_as_longlong(dp);
    } else {
      want_e = status != ST_STATUS_LOW_TEXTURE;
    }
    a.d[i] = bd;
    a.e[i] = be;
    a.status[i] = status;
    if (a.mask_in) a.mask_in[i] = bits;
  }
  if (a.elist) list_append(want_e, (int32_t)i, a.elist, a.elist_count);
  }
  if (a.partials) {
    const long long c_cand = warp_sum(n_cand);
    const long long c_eval = warp_sum(n_eval);
    const long long c_hopeless = warp_sum(n_hopeless);
    const long long c_samples = warp_sum(n_samples);
    if ((threadIdx.x & 31) == 0) {
      Partial& P = a.partials[(blockIdx.x * blockDim.x + threadIdx.x) >> 5];
      P.n_cand = c_cand;
      P.n_eval = c_eval;
      P.n_hopeless = c_hopeless;
      P.n_samples = c_samples;
    }
  }
}

// Iteration >= 2: which slots need a new M-step (mask changed since their
// last one).  The others carry their previous-disparity energy (= their E)
// and changed = 0 into the statistics.
__global__ void k_flag_mstep(const int64_t* __restrict__ active, int64_t n, int64_t pix0,
                             const uint32_t* __restrict__ static_all,
                             const uint32_t* __restrict__ mask_in, const double* __restrict__ e,
                             double* __restrict__ pe, uint8_t* __restrict__ chg,
                             int32_t* __restrict__ list, uint32_t* __restrict__ count,
                             const int* stop, const uint32_t* n_dev) {
  if (stop && *stop) return;
  if (n_dev) n = *n_dev;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool want = false;
    if (i < n) {
      const int64_t pix = active ? active[i] : pix0 + i;
      want = static_all[pix] != mask_in[i];
      if (!want) {
        pe[i] = e[i];
        chg[i] = 0;
      }
    }
    list_append(want, (int32_t)i, list, count);
  }
}

// Per-iteration statistics over every active slot, as fixed-order per-warp
// partials (solver.py:463-475: mean of finite E, mean of finite previous
// energies, changed count).
__device__ void solve_control(int it, const Partial* __restrict__ reduced,
                              uint32_t* __restrict__ counts, int64_t n_act, int forced_iters,
                              st_stats* __restrict__ stats, int* __restrict__ stop);

// Per-iteration statistics (solver.py:463-475).  solver.py:466/471 take
// `finite.mean()`: the grid is the top `pw_depth` levels of numpy's pairwise
// tree over the slots (st_pw.cuh), each block sums its node of E (and of
// the previous-disparity energies) exactly, and the last block adds the
// nodes up the same tree.  Should a value be non-finite (never for
// d_max >= 1), the last block compacts the finite values and sums them
// itself (the slow path: numpy's tree over the compacted sequence).
#ifndef STATS_NODE
#define STATS_NODE 4096
#endif
__host__ __device__ int stats_depth(int64_t n) {
  int D = 0;  // nodes of ~STATS_NODE values per block, <= 1024 blocks
  while (D < 10 && (n >> D) > STATS_NODE) ++D;
  return D;
}

int64_t pw_val_size(int64_t n) {  // the slow path's levels for n values
  int depth = 0;
  while (n > PW_LEAF) {
    n -= n / 2 - (n / 2) % 8;
    ++depth;
  }
  return ((int64_t)2 << depth) + 64;
}

__device__ double pw_sum_compacted(const double* __restrict__ x, int64_t n,
                                   double* __restrict__ scratch, double* __restrict__ val,
                                   int64_t* m_out) {
  typedef cub::BlockScan<int, STATS_BLOCK> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t c = 0; c < n; c += STATS_BLOCK) {
    const int64_t i = c + threadIdx.x;
    const int f = (i < n && isfinite(x[i])) ? 1 : 0;
    int off, tot;
    Scan(tmp).ExclusiveSum(f, off, tot);
    if (f) scratch[base + off] = x[i];
    __syncthreads();
    if (threadIdx.x == 0) base += tot;
    __syncthreads();
  }
  const int64_t m = base;
  *m_out = m;
  const int levels = pw_depth_of(m, 62) + 1;
  return m > 0 ? pw_block_sum(scratch, 0, m, val, levels) : 0.0;
}

__global__ void __launch_bounds__(STATS_BLOCK) k_em_stats(
    int64_t n, int with_prev, const double* __restrict__ e, const double* __restrict__ pe,
    const uint8_t* __restrict__ chg, const Partial* __restrict__ work, int n_work_parts,
    Partial* __restrict__ parts, const int* stop, StatsTail tail) {
  if (stop && *stop) {
    // (in the graph loop every body run must set the condition, else the
    // WHILE node would keep its last value)
    if (tail.use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(tail.cond, 0u);
    return;
  }
  __shared__ double val[(1 << PW_MAX_LEVELS) - 1];
  if (tail.n_dev) n = *tail.n_dev;  // (the grid covers the upper bound's tree)
  const int D = tail.n_dev ? stats_depth(n) : tail.pw_depth;
  int64_t s0, nn;
  const bool own = blockIdx.x < (1u << D) && pw_block_node(n, D, blockIdx.x, s0, nn);
  double se = 0.0, spe = 0.0;
  if (own && nn > 0) {
    se = pw_block_sum(e, s0, nn, val, PW_MAX_LEVELS);
    if (with_prev) spe = pw_block_sum(pe, s0, nn, val, PW_MAX_LEVELS);
  }
  long long nf = 0, npf = 0, nch = 0;
  if (own) {
    for (int64_t i = s0 + threadIdx.x; i < s0 + nn; i += blockDim.x) {
      nf += isfinite(e[i]) ? 1 : 0;
      if (with_prev) {
        npf += isfinite(pe[i]) ? 1 : 0;
        nch += chg[i];
      }
    }
  }
  // the M-step's per-warp work counters (integers: any order is exact)
  long long wc = 0, we = 0, wh = 0, ws = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n_work_parts;
       w += (int64_t)gridDim.x * blockDim.x) {
    wc += work[w].n_cand;
    we += work[w].n_eval;
    wh += work[w].n_hopeless;
    ws += work[w].n_samples;
  }
  __shared__ long long si[7][STATS_BLOCK / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long v7[7] = {nf, npf, nch, wc, we, wh, ws};
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const long long x = warp_sum(v7[k]);
    if (lane == 0) si[k][wid] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Partial B = {};
    B.sum_e = se;
    B.sum_pe = spe;
    long long t7[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j < (int)(blockDim.x >> 5); ++j)
      for (int k = 0; k < 7; ++k) t7[k] += si[k][j];
    B.n_fin = t7[0];
    B.n_pfin = t7[1];
    B.n_changed = t7[2];
    B.n_cand = t7[3];
    B.n_eval = t7[4];
    B.n_hopeless = t7[5];
    B.n_samples = t7[6];
    parts[blockIdx.x] = B;
  }
  if (!tail.on) return;
  // the last block to finish folds the blocks' records and runs the control
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(tail.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // integer counts: any order
  const int nb = gridDim.x;
  long long c7[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const Partial& P = parts[b];
    c7[0] += P.n_fin;
    c7[1] += P.n_pfin;
    c7[2] += P.n_changed;
    c7[3] += P.n_cand;
    c7[4] += P.n_eval;
    c7[5] += P.n_hopeless;
    c7[6] += P.n_samples;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const long long x = warp_sum(c7[k]);
    if (lane == 0) si[k][wid] = x;
  }
  __syncthreads();
  __shared__ long long tot7[7];
  if (threadIdx.x < 7) {
    long long x = 0;
    for (int j = 0; j < (int)(blockDim.x >> 5); ++j) x += si[threadIdx.x][j];
    tot7[threadIdx.x] = x;
  }
  __syncthreads();
  // the energy sums in numpy's order
  double sum_e, sum_pe = 0.0;
  int64_t m_e = tot7[0], m_pe = tot7[1];
  if (m_e == n) {
    sum_e = pw_top_sum(n, D, [&](unsigned p) { return parts[p].sum_e; }, val);
  } else {
    sum_e = pw_sum_compacted(e, n, tail.pw_scratch, tail.pw_val, &m_e);
  }
  if (with_prev) {
    if (m_pe == n)
      sum_pe = pw_top_sum(n, D, [&](unsigned p) { return parts[p].sum_pe; }, val);
    else
      sum_pe = pw_sum_compacted(pe, n, tail.pw_scratch, tail.pw_val, &m_pe);
  }
  if (threadIdx.x != 0) return;
  Partial r = {};
  r.sum_e = dadd(0.0, sum_e);  // np.add.reduce: the identity, then the pairwise sum
  r.sum_pe = dadd(0.0, sum_pe);
  r.n_fin = tot7[0];
  r.n_pfin = tot7[1];
  r.n_changed = tot7[2];
  r.n_cand = tot7[3];
  r.n_eval = tot7[4];
  r.n_hopeless = tot7[5];
  r.n_samples = tot7[6];
  *tail.done = 0u;
  const int it = tail.it + (tail.it_off ? (int)*tail.it_off : 0);
  if (tail.record_only) {
    r.n_act = tail.n_dev ? (long long)n : tail.record_n_act;
    r.n_mwork = it > 1 ? (long long)tail.counts[0] : tail.n_dev ? (long long)n : tail.record_slots;
    r.n_ework = (long long)tail.counts[1];
    r.n_unsafe = tail.mu_unsafe ? (long long)(*tail.mu_unsafe != 0) : 0;
    tail.reduced[it] = r;
    if (!tail.keep_counts) {
      tail.counts[0] = 0;  // next iteration's worklists
      tail.counts[1] = 0;
    }
    if (tail.flist_count) *tail.flist_count = 0u;
    return;
  }
  tail.reduced[it] = r;
  __threadfence();
  solve_control(it, tail.reduced, tail.counts, tail.n_act, tail.forced_iters, tail.stats,
                tail.stop_rw);
  if (tail.flist_count) *tail.flist_count = 0u;
  if (tail.it_off) *tail.it_off += 1u;
  if (tail.use_cond)
    cudaGraphSetConditional(tail.cond, (*tail.stop_rw == 0 && it + 1 <= tail.iters) ? 1u : 0u);
}

// ---------------------------------------------------------------------------
// E-step (solver.py:115-157)

// Gathered ray state for one pixel; descriptors live in shared memory,
// element (k, ch) of thread t at smem[(k * 16 + ch) * blockDim + t].
struct RayPriors {
  double l1[ST_MAX_VIEWS];
  double l0[ST_MAX_VIEWS];
};

// log of the clamped Bernoulli factors (solver.py:137-140).
__device__ __forceinline__ void clamp_logs(double q, double eps, double& l1, double& l0) {
  const double qc = fmin(fmax(q, eps), dsub(1.0, eps));  // np.clip(q, eps, 1 - eps)
  l1 = log(qc);
  l0 = log(dsub(1.0, qc));
}

// Same values; rays clamped to eps or 1 - eps take the precomputed logs
// (eps_logs = log(eps), log(1 - eps), log(1 - (1 - eps))).
__device__ __forceinline__ void clamp_logs(double q, double eps, const double* eps_logs,
                                           double& l1, double& l0) {
  const double hi = dsub(1.0, eps);
  const double qc = fmin(fmax(q, eps), hi);
  if (eps_logs && qc == eps) {
    l1 = __ldg(eps_logs);
    l0 = __ldg(eps_logs + 1);
  } else if (eps_logs && qc == hi) {
    l1 = __ldg(eps_logs + 1);
    l0 = __ldg(eps_logs + 2);
  } else {
    l1 = log(qc);
    l0 = log(dsub(1.0, qc));
  }
}

__global__ void k_eps_logs(double eps, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double hi = dsub(1.0, eps);
    out[0] = log(eps);
    out[1] = log(hi);
    out[2] = log(dsub(1.0, hi));
  }
}

// Mask preference (solver.py:110-112, 156): higher score, then larger
// popcount, then smaller encoding -- the first maximum in _mask_order.
__device__ __forceinline__ bool prefer(double s, int pop, uint32_t m, double bs, int bpop,
                                       uint32_t bm) {
  if (s > bs) return true;
  if (s < bs || !(s == bs)) return false;
  if (pop != bpop) return pop > bpop;
  return m < bm;
}

__constant__ double c_recip[13] = {0.0,       1.0 / 1,  1.0 / 2,  1.0 / 3, 1.0 / 4,
                                   1.0 / 5,   1.0 / 6,  1.0 / 7,  1.0 / 8, 1.0 / 9,
                                   1.0 / 10,  1.0 / 11, 1.0 / 12};

__device__ __forceinline__ double div_n(double x, int n) {
  // powers of two scale exactly; other counts use the exact small divisor
  switch (n) {
    case 1: return x;
    case 2: return dmul(x, 0.5);
    case 4: return dmul(x, 0.25);
    case 8: return dmul(x, 0.125);
    default: return div_small(x, (double)n, c_recip[n]);
  }
}

__host__ __device__ constexpr int popc_c(int x) { return x ? (x & 1) + popc_c(x >> 1) : 0; }

template <int N>
__device__ __forceinline__ double div_c(double x) {
  if constexpr (N == 1) return x;
  else if constexpr ((N & (N - 1)) == 0) return dmul(x, 1.0 / N);  // exact scaling
  else return div_small(x, (double)N, 1.0 / N);                      // RN(1/N) folded at compile time
}

// fp32 screening sums: every non-empty mask's per-channel prefix b1 in
// depth-first order (C = M | 1 << KB extends its prefix M by view KB),
// accumulating b1^2; sum_c b2 is recovered later from per-view totals.
template <int K, int M, int KB>
__device__ __forceinline__ void mask_dfs32(const float (&g)[K], float a1, float (&acc)[1 << K]) {
  if constexpr (KB < K) {
    constexpr int C = M | (1 << KB);
    const float b1 = M == 0 ? g[KB] : a1 + g[KB];
    if constexpr (popc_c(C) >= 2) acc[C] = fmaf(b1, b1, acc[C]);
    mask_dfs32<K, C, KB + 1>(g, b1, acc);  // supersets of C
    mask_dfs32<K, M, KB + 1>(g, a1, acc);  // M with a later view instead
  }
}

// Exact score of one mask in the reference's arithmetic order: per channel
// the in-order sums over the selected views (BLAS dgemm with a 0/1 operand,
// solver.py:148-149), (s2 - s1*s1/n) summed over channels in order, then
// prior - beta * var (solver.py:150-156).  `load(k, w, f)` yields channels
// 4w..4w+3 of view k exactly as gather_rays samples them.
template <int K, typename Load>
__device__ __forceinline__ double score_exact(uint32_t m, Load& load, const double* l1,
                                              const double* l0, const st_params& p) {
  const int pop = __popc(m);
  double vr;
  if (pop < p.min_static_rays) {
    vr = variance_ceiling();
  } else if (pop == 0) {
    vr = 0.0;
  } else {
    double acc = 0.0;
#pragma unroll 1
    for (int w = 0; w < 4; ++w) {
      double a1[4], a2[4];
      bool first = true;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!((m >> k) & 1)) continue;
        double x[4];
        load(k, w, x);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double x2 = dmul(x[j], x[j]);
          a1[j] = first ? x[j] : dadd(a1[j], x[j]);
          a2[j] = first ? x2 : dadd(a2[j], x2);
        }
        first = false;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) acc = dadd(acc, dsub(a2[j], div_n(dmul(a1[j], a1[j]), pop)));
    }
    vr = fmax(div_n(acc, pop), 0.0);
  }
  double a = 0.0, b = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if ((m >> k) & 1)
      a = dadd(a, l1[k]);
    else
      b = dadd(b, l0[k]);
  }
  return dsub(dadd(a, b), dmul(p.beta, vr));
}

// E-step argmax for K <= 5 (<= 32 masks): screen in fp32, decide in fp64.
//
// Every mask is scored in fp32 on data centred at the first valid view
// (variance is shift-invariant), with sum_c b2 = sum_{k in m} Q_k taken from
// per-view totals, so one mask-channel costs an FADD and an FFMA.  D below
// majorises |score32(m) - score64(m)| for every admissible mask: variance
// numerator error <= 50u*S2c (u = 2^-24, S2c = centred sum of squares over
// the valid views), the fp64 recipe's own error <= 2^-47*S2u, the prior sum
// <= (K+3)u*L, beta*v rounding <= 2u*beta*max(ceiling, S2c), all doubled.
// The reference's argmax m* therefore has score32(m*) >= best32 - 2D, and
// only the masks in that window are re-scored exactly (score_exact) under
// the reference's tie rules -- normally one.  `exhaustive` re-scores every
// admissible mask (the cross-check behind ST_ESTEP_EXHAUSTIVE).
template <int K, typename Load, typename Load32>
__device__ __forceinline__ uint32_t estep_small(Load& load, Load32& load32, float eps32,
                                                const double* l1, const double* l0,
                                                uint32_t vbits, const st_params& p,
                                                bool exhaustive) {
  constexpr int M = 1 << K;
  constexpr float U = 5.9604645e-08f;  // 2^-24
  if (!vbits) return 0;                // only the empty mask is admissible
  const int k0 = __ffs(vbits) - 1;
  float acc[M];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m] = 0.0f;
  float q[K];
#pragma unroll
  for (int k = 0; k < K; ++k) q[k] = 0.0f;
  float s2u = 0.0f;
#pragma unroll 1
  for (int w = 0; w < 4; ++w) {
    // fp32 samples straight from the taps (|error| <= eps32 each); the
    // first valid view's error is a common shift the variance ignores
    float ref[4];
#pragma unroll
    for (int k = 0; k < K; ++k)  // compile-time view index keeps the taps in registers
      if (k == k0) load32(k, w, ref);
    float g[K][4];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float x[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // invalid rays hold 0
      if ((vbits >> k) & 1) load32(k, w, x);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        g[k][j] = x[j] - ref[j];
        q[k] = fmaf(g[k][j], g[k][j], q[k]);
        s2u = fmaf(x[j], x[j], s2u);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float gj[K];
#pragma unroll
      for (int k = 0; k < K; ++k) gj[k] = g[k][j];
      mask_dfs32<K, 0, 0>(gj, 0.0f, acc);
    }
  }
  float s2c = 0.0f, lsum = 0.0f, l0tot = 0.0f, dl[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if ((vbits >> k) & 1) s2c += q[k];
    const float f1 = __double2float_rn(l1[k]), f0 = __double2float_rn(l0[k]);
    dl[k] = f1 - f0;
    l0tot += f0;
    lsum += fabsf(f1) + fabsf(f0);
  }
  const float beta = (float)p.beta;
  const float ceil32 = (float)variance_ceiling();
  constexpr float inv_n[6] = {1.0f, 1.0f, 0.5f, 1.0f / 3.0f, 0.25f, 0.2f};
  float sc[M];
  float best32 = -INFINITY;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int pop = __popc(m);
    float v;
    if (pop < p.min_static_rays) {
      v = ceil32;
    } else if (pop < 2) {
      v = 0.0f;
    } else {
      float qs = 0.0f;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if ((m >> k) & 1) qs += q[k];
      v = fmaxf((qs - acc[m] * inv_n[pop]) * inv_n[pop], 0.0f);
    }
    float pr = l0tot;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if ((m >> k) & 1) pr += dl[k];
    sc[m] = pr - beta * v;
    if (!((uint32_t)m & ~vbits)) best32 = fmaxf(best32, sc[m]);
  }
  // + sample perturbation: |d t_c| <= 2 eps sqrt(n t_c) + n eps^2, summed
  // over 16 channels, n <= 5 (not divided by n: conservative)
  const float D = 2.0f * (fabsf(beta) * (64.0f * U * s2c + 2.0f * U * fmaxf(ceil32, s2c) +
                                         7.1054274e-15f * s2u + 2.0f * U * ceil32 +
                                         2.0f * eps32 * sqrtf(80.0f * s2c) +
                                         80.0f * eps32 * eps32) +
                          (2.0f * K + 6.0f) * U * lsum);
  const float thr = best32 - 2.0f * D;
  const bool all = exhaustive || !(thr > -INFINITY);  // non-finite bound: decide exhaustively
  uint32_t cand = 0;
#pragma unroll
  for (int m = 0; m < M; ++m)
    if (all || sc[m] >= thr) cand |= 1u << m;
  double best = -INFINITY;
  int bpop = -1;
  uint32_t bm = 0;
  for (; cand; cand &= cand - 1) {
    const uint32_t m = __ffs(cand) - 1;
    if (m & ~vbits) continue;  // touches an invalid ray
    const double s = score_exact<K>(m, load, l1, l0, p);
    const int pop = __popc(m);
    if (prefer(s, pop, m, best, bpop, bm)) {
      best = s;
      bpop = pop;
      bm = m;
    }
  }
  return bm;
}

// Generic path for 6 <= K <= 12: one mask at a time, same arithmetic order.
__device__ uint32_t estep_generic(int K, const double* __restrict__ f, int stride,
                                  const double* l1, const double* l0, uint32_t vbits,
                                  const st_params& p) {
  const uint32_t M = 1u << K;
  double best = -INFINITY;
  int bpop = -1;
  uint32_t bm = 0;
  for (uint32_t m = 0; m < M; ++m) {
    if (m & ~vbits) continue;
    const int pop = __popc(m);
    double vr;
    if (pop < p.min_static_rays) {
      vr = variance_ceiling();
    } else {
      double acc = 0.0;
      for (int ch = 0; ch < 16; ++ch) {
        double a1 = 0.0, a2 = 0.0;
        int n = 0;
        for (uint32_t r = m; r; r &= r - 1) {
          const int k = __ffs(r) - 1;
          const double x = f[(k * 16 + ch) * stride];
          a1 = n ? dadd(a1, x) : x;
          const double x2 = dmul(x, x);
          a2 = n ? dadd(a2, x2) : x2;
          ++n;
        }
        acc = dadd(acc, dsub(a2, div_n(dmul(a1, a1), n)));
      }
      vr = fmax(div_n(acc, pop), 0.0);
    }
    double a = 0.0, b = 0.0;
    for (int k = 0; k < K; ++k) {
      if ((m >> k) & 1)
        a = dadd(a, l1[k]);
      else
        b = dadd(b, l0[k]);
    }
    const double s = dsub(dadd(a, b), dmul(p.beta, vr));
    if (prefer(s, pop, m, best, bpop, bm)) {
      best = s;
      bpop = pop;
      bm = m;
    }
  }
  return bm;
}

// Same argmax by bounding (6 <= K <= 12).  P(m) = fl(a + b), the prior sum
// in the reference's order, bounds score(m) = fl(P(m) - fl(beta v(m)))
// from above (v >= 0, fl monotone) and equals it up to the constant penalty
// when pop(m) < min_static_rays.  The bounds are evaluated as exact integer
// sums of the logs rounded to 2^-20 units, |Pq/2^20 - P| <= (K/2 + 3) 2^-20
// (rounding of each term, the fp64 sum's own roundings).  The mask with the
// largest bound is scored exactly first; every other admissible mask is
// scored exactly only if its bound can still reach the best exact score, so
// no skipped mask can tie or win.  Normally one or two exact scores instead
// of 2^K.
__device__ double score_generic(uint32_t m, int K, const double* __restrict__ f, int stride,
                                const double* l1, const double* l0, const st_params& p) {
  const int pop = __popc(m);
  double vr;
  if (pop < p.min_static_rays) {
    vr = variance_ceiling();
  } else {
    double acc = 0.0;
    for (int ch = 0; ch < 16; ++ch) {
      double a1 = 0.0, a2 = 0.0;
      int n = 0;
      for (uint32_t r = m; r; r &= r - 1) {
        const int k = __ffs(r) - 1;
        const double x = f[(k * 16 + ch) * stride];
        a1 = n ? dadd(a1, x) : x;
        const double x2 = dmul(x, x);
        a2 = n ? dadd(a2, x2) : x2;
        ++n;
      }
      acc = dadd(acc, dsub(a2, div_n(dmul(a1, a1), n)));
    }
    vr = fmax(div_n(acc, pop), 0.0);
  }
  double a = 0.0, b = 0.0;
  for (int k = 0; k < K; ++k) {
    if ((m >> k) & 1)
      a = dadd(a, l1[k]);
    else
      b = dadd(b, l0[k]);
  }
  return dsub(dadd(a, b), dmul(p.beta, vr));
}

template <typename Score>
__device__ uint32_t estep_bnb_core(int K, const double* l1, const double* l0, uint32_t vbits,
                                   const st_params& p, Score score) {
  constexpr double QS = 1048576.0;  // 2^20
  long long dq[ST_MAX_VIEWS];
  long long base = 0;
  double lmax = 0.0;
#pragma unroll
  for (int k = 0; k < ST_MAX_VIEWS; ++k) {
    dq[k] = 0;
    if (k < K) {
      const long long q1 = __double2ll_rn(l1[k] * QS), q0 = __double2ll_rn(l0[k] * QS);
      dq[k] = q1 - q0;
      base += q0;
      lmax = fmax(lmax, fmax(fabs(l1[k]), fabs(l0[k])));
    }
  }
  const long long penq = __double2ll_rn(fmin(dmul(p.beta, variance_ceiling()) * QS, 1e15));
  const double errq = 0.5 * K + 3.0 + 1e-12 * K * lmax * QS;
  auto bound = [&](uint32_t m) -> long long {
    long long ub = base;
#pragma unroll
    for (int k = 0; k < ST_MAX_VIEWS; ++k)
      if ((m >> k) & 1) ub += dq[k];
    return __popc(m) < p.min_static_rays ? ub - penq : ub;
  };
  // the largest bound first
  uint32_t mtop = 0;
  long long btop = bound(0);
  for (uint32_t m = vbits; m; m = (m - 1) & vbits) {
    const long long ub = bound(m);
    if (ub > btop) {
      btop = ub;
      mtop = m;
    }
  }
  double best = score(mtop);
  int bpop = __popc(mtop);
  uint32_t bm = mtop;
  auto consider = [&](uint32_t mm) {
    const double sc = score(mm);
    const int pop = __popc(mm);
    if (prefer(sc, pop, mm, best, bpop, bm)) {
      best = sc;
      bpop = pop;
      bm = mm;
    }
  };
  // The masks whose bound can still reach the best score, visited in
  // decreasing bound order: the winner is usually among the first, and the
  // rising best score then ends the visit early.  (More than BNB_LIST such
  // masks: all of them are scored, in enumeration order.)
  constexpr int BNB_LIST = 48;
  uint32_t lm[BNB_LIST];
  long long lb[BNB_LIST];
  int nl = 0;
  bool overflow = false;
  const double thr0 = best * QS - errq;
  uint32_t m = 0;
  do {
    if (m != mtop) {
      const long long ub = bound(m);
      if ((double)ub >= thr0) {
        if (nl < BNB_LIST) {
          int q = nl++;  // insertion, descending bound
          while (q > 0 && lb[q - 1] < ub) {
            lb[q] = lb[q - 1];
            lm[q] = lm[q - 1];
            --q;
          }
          lb[q] = ub;
          lm[q] = m;
        } else {
          overflow = true;
        }
      }
    }
    m = (m - vbits) & vbits;
  } while (m != 0);
  if (!overflow) {
    for (int q = 0; q < nl; ++q) {
      if ((double)lb[q] + errq < best * QS) break;  // every later bound is lower still
      consider(lm[q]);
    }
    return bm;
  }
  m = 0;
  do {
    if (m != mtop && (double)bound(m) + errq >= best * QS) consider(m);
    m = (m - vbits) & vbits;
  } while (m != 0);
  return bm;
}

__device__ uint32_t estep_bnb(int K, const double* __restrict__ f, int stride, const double* l1,
                              const double* l0, uint32_t vbits, const st_params& p) {
  return estep_bnb_core(K, l1, l0, vbits, p, [&](uint32_t m) {
    return score_generic(m, K, f, stride, l1, l0, p);
  });
}

// Loader over rays staged in shared memory: element (k, ch) of thread t at
// smem[(k * 16 + ch) * stride + t].
struct SmemRays {
  const double* f;
  int stride;
  __device__ __forceinline__ void operator()(int k, int w, double (&x)[4]) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = f[(k * 16 + 4 * w + j) * stride];
  }
};

// fp32 view of the same rays: one rounding, |error| <= 2^-24 * 255 < 256u
struct SmemRays32 {
  const double* f;
  int stride;
  __device__ __forceinline__ void operator()(int k, int w, float (&x)[4]) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = __double2float_rn(f[(k * 16 + 4 * w + j) * stride]);
  }
};

__device__ __forceinline__ uint32_t estep_dispatch(int K, const double* f, int stride,
                                                   const double* l1, const double* l0,
                                                   uint32_t vbits, const st_params& p) {
  SmemRays ld{f, stride};
  SmemRays32 ld32{f, stride};
  const float eps = 512.0f * 5.9604645e-08f;
  switch (K) {
    case 2: return estep_small<2>(ld, ld32, eps, l1, l0, vbits, p, false);
    case 3: return estep_small<3>(ld, ld32, eps, l1, l0, vbits, p, false);
    case 4: return estep_small<4>(ld, ld32, eps, l1, l0, vbits, p, false);
    case 5: return estep_small<5>(ld, ld32, eps, l1, l0, vbits, p, false);
    default: return estep_generic(K, f, stride, l1, l0, vbits, p);
  }
}

// Channels 4w..4w+3 of one descriptor sample, recomputed from the uint8 map
// with exactly sample_desc's arithmetic (sampling.py:49-55).
template <bool RECT>
__device__ __forceinline__ void desc_word(const uint32_t* __restrict__ plane, int idx, int su,
                                          int sv, double fu, double fv, int w,
                                          double (&f)[4]) {
  const uint32_t* p = plane + (size_t)idx * 4 + w;
  const uint32_t a = __ldg(p), b = __ldg(p + 4 * su);
  if (RECT || fv == 0.0) {
    lerp_word(a, b, fu, f);
  } else {
    const uint32_t e = __ldg(p + 4 * (size_t)sv), g = __ldg(p + 4 * ((size_t)sv + su));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int sh = 8 * j;
      const double top = lerp_u8((a >> sh) & 0xff, (b >> sh) & 0xff, fu);
      const double bot = lerp_u8((e >> sh) & 0xff, (g >> sh) & 0xff, fu);
      f[j] = dadd(top, dmul(fv, dsub(bot, top)));
    }
  }
}

// fp32 counterpart of desc_word for the screen: exact integer taps via the
// 2^23 trick, one FFMA per lerp.  |f32 - f| <= 511u for one lerp (u = 2^-24,
// taps <= 255), <= 2300u for the bilinear case.
__device__ __forceinline__ void lerp_word32(uint32_t wa, uint32_t wb, float fu, float (&f)[4]) {
  const uint32_t ea = wa & 0x00ff00ffu, eb = wb & 0x00ff00ffu;
  const uint32_t oa = (wa >> 8) & 0x00ff00ffu, ob = (wb >> 8) & 0x00ff00ffu;
  const uint32_t de = eb + 0x01000100u - ea;
  const uint32_t dodd = ob + 0x01000100u - oa;
  const uint32_t lanes[4] = {__byte_perm(de, 0u, 0x4410), __byte_perm(dodd, 0u, 0x4410),
                             __byte_perm(de, 0u, 0x4432), __byte_perm(dodd, 0u, 0x4432)};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float g0 = __fsub_rn(__uint_as_float(__byte_perm(wa, 0x4b000000u, 0x7440 | j)),
                               8388608.0f);  // 2^23 + byte, exact
    const float df = __fsub_rn(__uint_as_float(0x4b000000u | lanes[j]), 8388864.0f);
    f[j] = fmaf(fu, df, g0);
  }
}

template <bool RECT>
__device__ __forceinline__ void desc_word32(const uint32_t* __restrict__ plane, int idx, int su,
                                            int sv, float fu, float fv, int w, float (&f)[4]) {
  const uint32_t* p = plane + (size_t)idx * 4 + w;
  lerp_word32(__ldg(p), __ldg(p + 4 * su), fu, f);
  if (!RECT && fv != 0.0f) {
    float bot[4];
    lerp_word32(__ldg(p + 4 * (size_t)sv), __ldg(p + 4 * ((size_t)sv + su)), fu, bot);
#pragma unroll
    for (int j = 0; j < 4; ++j) f[j] = fmaf(fv, bot[j] - f[j], f[j]);
  }
}

// E-step at the solver's disparities for K <= 5 views (solver.py:409-419).
// No ray staging: each view keeps only its tap (index, weights) in
// registers and the screen / exact re-score re-read the 16-byte descriptor
// words (L1-resident), so occupancy is bounded by registers alone.  RECT:
// rectified rig, vertical weight identically 0.
template <int KT, bool RECT>
__global__ void __launch_bounds__(ESTEP_TAPS_BLOCK, ESTEP_MIN_BLOCKS) k_e_step_taps(EmCtx c, EStepArgs a) {
  if (a.stop && *a.stop) return;  // converged (st_solve_async)
  const int64_t n_work = a.list ? (int64_t)*a.list_count : a.n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_work;
       t += (int64_t)gridDim.x * blockDim.x) {
  const int64_t i = a.list ? (int64_t)a.list[t] : t;
  if (a.status && a.status[i] == ST_STATUS_LOW_TEXTURE) continue;  // solver.py:476-478
  const int64_t pix = a.pix ? a.pix[i] : c.pix0 + i;
  const double u = (double)(pix % c.W), v = (double)(pix / c.W);
  const double d = a.d[i];
  int idx[KT];
  double fu[KT], fv[KT], l1[KT], l0[KT];
  uint32_t vb = 0;
  // gather_rays (solver.py:206-227): invalid rays carry q 0.5
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    const WarpOut w = warp_ctx(c, k, u, v, d);
    double q = 0.5;
    idx[k] = 0;
    fu[k] = 0.0;
    fv[k] = 0.0;
    if (in_margin(c.rig, k, w)) {
      const Taps tp = taps_ctx(c, w);
      idx[k] = tp.iv * c.W + tp.iu;
      fu[k] = tp.fu;
      if (!RECT) fv[k] = tp.fv;
      q = sample_prior(c.priors + (size_t)k * c.HW, c.W, tp);
      vb |= 1u << k;
    }
    clamp_logs(q, c.p.epsilon_prior, a.eps_logs, l1[k], l0[k]);
  }
  const int su = c.W > 1 ? 1 : 0, sv = c.H > 1 ? c.W : 0;  // taps_of's steps
  const uint32_t* desc = reinterpret_cast<const uint32_t*>(c.desc);
  auto load = [&](int k, int w, double (&x)[4]) {
    desc_word<RECT>(desc + (size_t)k * c.HW * 4, idx[k], su, sv, fu[k], RECT ? 0.0 : fv[k], w,
                    x);
  };
  auto load32 = [&](int k, int w, float (&x)[4]) {
    desc_word32<RECT>(desc + (size_t)k * c.HW * 4, idx[k], su, sv, (float)fu[k],
                      RECT ? 0.0f : (float)fv[k], w, x);
  };
  const float eps = (RECT ? 1024.0f : 4096.0f) * 5.9604645e-08f;
  const uint32_t m = estep_small<KT>(load, load32, eps, l1, l0, vb, c.p, a.exhaustive != 0);
  const int64_t o = a.scatter ? pix : i;
  a.static_out[o] = m;
  a.valid_out[o] = vb;
  }
}

template __global__ void k_e_step_taps<2, false>(EmCtx, EStepArgs);
template __global__ void k_e_step_taps<3, false>(EmCtx, EStepArgs);
template __global__ void k_e_step_taps<4, false>(EmCtx, EStepArgs);
template __global__ void k_e_step_taps<5, false>(EmCtx, EStepArgs);
template __global__ void k_e_step_taps<2, true>(EmCtx, EStepArgs);
template __global__ void k_e_step_taps<3, true>(EmCtx, EStepArgs);
template __global__ void k_e_step_taps<4, true>(EmCtx, EStepArgs);
template __global__ void k_e_step_taps<5, true>(EmCtx, EStepArgs);

// E-step certificate pass for K <= 5 views (prior dominance, exact).
//
// score(m) = fl(P(m) - fl(beta v(m))) <= P(m) - [pop(m) < min_static_rays]
// beta * ceiling, P(m) the prior sum (v >= 0, fl monotone).  Those bounds
// need no descriptor samples.  The admissible mask m1 with the largest
// bound is scored in fp32 with the screen's error bound D (estep_small);
// if the lower end of that score beats every other mask's bound, m1 is the
// reference's argmax -- uniquely, so its tie rules cannot intervene.  Rows
// without such a certificate go to a fallback list for k_e_step_taps.
//
// Everything here is fp32 except the warp (validity is an output and must
// be exact).  The priors' log factors are fp32 too; against the fp64
// recipe (sample_prior, clamp_logs) each log differs by at most
//   E_l = (6u + 2u) / eps * 1.01 + 2 ulp32(max(|log eps|, 1)),
// (q lerp in fp32 <= 6u, clip bound and 1 - q roundings 2u, |d log q| <=
// |dq| / eps, logf <= 2 ulp), so every P(m) moves by <= K E_l.
template <int KT, bool RECT>
__global__ void __launch_bounds__(ESTEP_CERT_BLOCK, ESTEP_CERT_MIN_BLOCKS)
    k_e_step_cert(EmCtx c, EStepArgs a) {
  if (a.stop && *a.stop) return;  // converged (st_solve_async)
  constexpr int M = 1 << KT;
  constexpr float U = 5.9604645e-08f;  // 2^-24
  const int64_t n_work = a.list ? (int64_t)*a.list_count : a.n;
  const float eps = (float)c.p.epsilon_prior;
  const float hi = (float)dsub(1.0, c.p.epsilon_prior);
  const float lmax = fmaxf(fabsf(logf(eps)), 1.0f);
  const float e_l = (8.0f * U) / eps * 1.01f + 4.0f * U * 2.0f * lmax;
  const float beta = (float)c.p.beta;
  const float ceil32 = (float)variance_ceiling();
  const float pen = beta * ceil32;
  const float eps32 = (RECT ? 1024.0f : 4096.0f) * U;  // descriptor sample error (desc_word32)
  const uint32_t* desc = reinterpret_cast<const uint32_t*>(c.desc);
  const int su = c.W > 1 ? 1 : 0, sv = c.H > 1 ? c.W : 0;  // taps_of's steps
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_work;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = base + threadIdx.x;
    bool fail = false;
    int64_t i = 0;
    if (t < n_work) {
      i = a.list ? (int64_t)a.list[t] : t;
      if (!(a.status && a.status[i] == ST_STATUS_LOW_TEXTURE)) {  // solver.py:476-478
        const int64_t pix = a.pix ? a.pix[i] : c.pix0 + i;
        const double u = (double)(pix % c.W), v = (double)(pix / c.W);
        const double d = a.d[i];
        int idx[KT];
        float fu[KT], fv[KT], l1[KT], l0[KT];
        uint32_t vb = 0;
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          const WarpOut w = warp_ctx(c, k, u, v, d);
          float q = 0.5f;  // invalid rays (solver.py:206-227)
          idx[k] = 0;
          fu[k] = 0.0f;
          fv[k] = 0.0f;
          if (in_margin(c.rig, k, w)) {
            const Taps tp = taps_ctx(c, w);
            idx[k] = tp.iv * c.W + tp.iu;
            fu[k] = (float)tp.fu;
            if (!RECT) fv[k] = (float)tp.fv;
            const float* pl = c.priors + (size_t)k * c.HW + idx[k];
            const float p0 = __ldg(pl), p1 = __ldg(pl + tp.su);
            q = fmaf(fu[k], __fsub_rn(p1, p0), p0);
            if (!RECT && tp.fv != 0.0) {
              const float p2 = __ldg(pl + tp.sv), p3 = __ldg(pl + tp.sv + tp.su);
              const float bot = fmaf(fu[k], __fsub_rn(p3, p2), p2);
              q = fmaf(fv[k], bot - q, q);
            }
            vb |= 1u << k;
          }
          const float qc = fminf(fmaxf(q, eps), hi);
          l1[k] = logf(qc);
          l0[k] = logf(1.0f - qc);
        }
        uint32_t m1 = 0;
        if (vb) {
          float l0t = 0.0f, lsum = 0.0f, dl[KT];
#pragma unroll
          for (int k = 0; k < KT; ++k) {
            dl[k] = l1[k] - l0[k];
            l0t += l0[k];
            lsum += fabsf(l1[k]) + fabsf(l0[k]);
          }
          float ub1 = -INFINITY, ub2 = -INFINITY;
#pragma unroll
          for (int m = 0; m < M; ++m) {
            if ((uint32_t)m & ~vb) continue;
            float ub = l0t;
#pragma unroll
            for (int k = 0; k < KT; ++k)
              if ((m >> k) & 1) ub += dl[k];
            if (__popc(m) < c.p.min_static_rays) ub -= pen;
            if (ub > ub1) {
              ub2 = ub1;
              ub1 = ub;
              m1 = (uint32_t)m;
            } else {
              ub2 = fmaxf(ub2, ub);
            }
          }
          // |bound32 - bound64| <= K E_l + fp32 sums and penalty roundings
          const float errp = 2.0f * (KT * e_l + (2.0f * KT + 8.0f) * U * (lsum + pen));
          if (__popc(m1) < c.p.min_static_rays) {
            fail = !(ub1 - errp > ub2 + errp);
          } else {
            const int k0 = __ffs(vb) - 1;
            float qs = 0.0f, ac = 0.0f, s2u = 0.0f;
#pragma unroll 1
            for (int w = 0; w < 4; ++w) {
              float ref[4];
#pragma unroll
              for (int k = 0; k < KT; ++k)
                if (k == k0)
                  desc_word32<RECT>(desc + (size_t)k * c.HW * 4, idx[k], su, sv, fu[k], fv[k], w,
                                    ref);
              float b1[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
              for (int k = 0; k < KT; ++k) {
                if (!((m1 >> k) & 1)) continue;
                float x[4];
                desc_word32<RECT>(desc + (size_t)k * c.HW * 4, idx[k], su, sv, fu[k], fv[k], w,
                                  x);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float g = x[j] - ref[j];
                  b1[j] += g;
                  qs = fmaf(g, g, qs);
                  s2u = fmaf(x[j], x[j], s2u);
                }
              }
#pragma unroll
              for (int j = 0; j < 4; ++j) ac = fmaf(b1[j], b1[j], ac);
            }
            const float rn = 1.0f / (float)__popc(m1);
            const float var = fmaxf((qs - ac * rn) * rn, 0.0f);
            const float s32 = ub1 - beta * var;
            // estep_small's D on the in-mask sums
            const float D = 2.0f * (fabsf(beta) * (64.0f * U * qs + 2.0f * U * fmaxf(ceil32, qs) +
                                                   7.1054274e-15f * s2u + 2.0f * U * ceil32 +
                                                   2.0f * eps32 * sqrtf(80.0f * qs) +
                                                   80.0f * eps32 * eps32) +
                                    (2.0f * KT + 6.0f) * U * lsum);
            fail = !(s32 - D - errp > ub2 + errp);
          }
        }
        if (!fail) {
          const int64_t o = a.scatter ? pix : i;
          a.static_out[o] = m1;
          a.valid_out[o] = vb;
        }
      }
    }
    list_append(fail, (int32_t)i, a.flist, a.flist_count);
  }
}

// Certificate pass for 6 <= K <= 12 views: k_e_step_cert's argument with
// the mask bounds enumerated instead of unrolled.  The fp32 log factors are
// rounded to fixed point (2^-20 units), so every bound over the 2^popc(valid)
// admissible masks is an exact integer sum; the top two bounds come from the
// views sorted by their log ratio (per-thread table in shared memory).
// |bound_q / 2^20 - bound64| <= K (E_l + 2^-21) + penalty rounding.
template <bool RECT>
__global__ void __launch_bounds__(CERT_BIG_BLOCK, 4) k_e_step_cert_big(EmCtx c, EStepArgs a) {
  __shared__ int s_dl[ST_MAX_VIEWS][CERT_BIG_BLOCK];
  if (a.stop && *a.stop) return;  // converged (st_solve_async)
  constexpr float U = 5.9604645e-08f;  // 2^-24
  constexpr float QS = 1048576.0f;     // 2^20
  const int K = c.rig.num_views;
  const int64_t n_work = a.list ? (int64_t)*a.list_count : a.n;
  const float eps = (float)c.p.epsilon_prior;
  const float hi = (float)dsub(1.0, c.p.epsilon_prior);
  const float lmax = fmaxf(fabsf(logf(eps)), 1.0f);
  const float e_l = (8.0f * U) / eps * 1.01f + 4.0f * U * 2.0f * lmax;
  const bool fits = (float)K * lmax * QS < 1.0e9f;  // integer sums cannot overflow
  const float beta = (float)c.p.beta;
  const float ceil32 = (float)variance_ceiling();
  const float pen = beta * ceil32;
  const int penq = __float2int_rn(fminf(pen * QS, 1.0e9f));
  const float eps32 = (RECT ? 1024.0f : 4096.0f) * U;
  const uint32_t* desc = reinterpret_cast<const uint32_t*>(c.desc);
  const int su = c.W > 1 ? 1 : 0, sv = c.H > 1 ? c.W : 0;
  int* dlq = &s_dl[0][threadIdx.x];
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_work;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = base + threadIdx.x;
    bool fail = false;
    int64_t i = 0;
    if (t < n_work) {
      i = a.list ? (int64_t)a.list[t] : t;
      if (!(a.status && a.status[i] == ST_STATUS_LOW_TEXTURE)) {  // solver.py:476-478
        const int64_t pix = a.pix ? a.pix[i] : c.pix0 + i;
        const double u = (double)(pix % c.W), v = (double)(pix / c.W);
        const double d = a.d[i];
        int idx[ST_MAX_VIEWS];
        float fu[ST_MAX_VIEWS], fv[ST_MAX_VIEWS];
        uint32_t vb = 0;
        int baseq = 0;
        float lsum = 0.0f;
#pragma unroll
        for (int k = 0; k < ST_MAX_VIEWS; ++k) {
          idx[k] = 0;
          fu[k] = 0.0f;
          fv[k] = 0.0f;
          if (k >= K) continue;
          const WarpOut w = warp_ctx(c, k, u, v, d);
          float q = 0.5f;  // invalid rays (solver.py:206-227)
          if (in_margin(c.rig, k, w)) {
            const Taps tp = taps_ctx(c, w);
            idx[k] = tp.iv * c.W + tp.iu;
            fu[k] = (float)tp.fu;
            if (!RECT) fv[k] = (float)tp.fv;
            const float* pl = c.priors + (size_t)k * c.HW + idx[k];
            const float p0 = __ldg(pl), p1 = __ldg(pl + tp.su);
            q = fmaf(fu[k], __fsub_rn(p1, p0), p0);
            if (!RECT && tp.fv != 0.0) {
              const float p2 = __ldg(pl + tp.sv), p3 = __ldg(pl + tp.sv + tp.su);
              const float bot = fmaf(fu[k], __fsub_rn(p3, p2), p2);
              q = fmaf(fv[k], bot - q, q);
            }
            vb |= 1u << k;
          }
          const float qc = fminf(fmaxf(q, eps), hi);
          const float l1 = logf(qc), l0 = logf(1.0f - qc);
          const int q1 = __float2int_rn(l1 * QS), q0 = __float2int_rn(l0 * QS);
          dlq[k * CERT_BIG_BLOCK] = q1 - q0;
          baseq += q0;
          lsum += fabsf(l1) + fabsf(l0);
        }
        uint32_t m1 = 0;
        int b1 = 0, b2 = 0;
        if (!fits) {
          fail = true;
        } else if (vb) {
          // Exact top two of bound(m) = base + sum_{k in m} dl_k - penq [pop(m) <
          // min] over the submasks of vb: for each size p the best mask takes
          // the p largest dl (views sorted descending), the runner-up of that
          // size swaps its weakest member for the strongest outsider.
          int dv[ST_MAX_VIEWS], kv[ST_MAX_VIEWS];
#pragma unroll
          for (int k = 0; k < ST_MAX_VIEWS; ++k) {
            const bool in = k < K && ((vb >> k) & 1);
            dv[k] = in ? dlq[k * CERT_BIG_BLOCK] : INT_MIN / 4;
            kv[k] = k;
          }
#pragma unroll
          for (int r = 0; r < ST_MAX_VIEWS - 1; ++r)
#pragma unroll
            for (int j = 0; j < ST_MAX_VIEWS - 1 - r; ++j)
              if (dv[j] < dv[j + 1]) {
                const int td = dv[j], tk = kv[j];
                dv[j] = dv[j + 1];
                kv[j] = kv[j + 1];
                dv[j + 1] = td;
                kv[j + 1] = tk;
              }
          const int nv = __popc(vb);
          int vp[ST_MAX_VIEWS + 1];
          int pre = 0;
          vp[0] = baseq - (0 < c.p.min_static_rays ? penq : 0);
#pragma unroll
          for (int q = 1; q <= ST_MAX_VIEWS; ++q) {
            pre += q <= nv ? dv[q - 1] : 0;
            vp[q] = q <= nv ? baseq + pre - (q < c.p.min_static_rays ? penq : 0) : INT_MIN;
          }
          int ps = 0;
#pragma unroll
          for (int q = 1; q <= ST_MAX_VIEWS; ++q)
            if (vp[q] > vp[ps]) ps = q;
          b1 = vp[ps];
          b2 = INT_MIN;
#pragma unroll
          for (int q = 0; q <= ST_MAX_VIEWS; ++q)
            if (q != ps) b2 = max(b2, vp[q]);
#pragma unroll
          for (int q = 1; q < ST_MAX_VIEWS; ++q)
            if (q == ps && q < nv) b2 = max(b2, b1 - dv[q - 1] + dv[q]);
          m1 = 0;
#pragma unroll
          for (int q = 0; q < ST_MAX_VIEWS; ++q)
            if (q < ps) m1 |= 1u << kv[q];
          // quantised bounds vs the fp64 ones: K (E_l + 2^-21) + 1 unit for
          // the penalty, doubled; in 2^-20 units
          const float errq = 2.0f * (K * (e_l * QS + 0.5f) + 1.0f) + (2.0f * K + 8.0f) * U * lsum * QS;
          const float gap = (float)(b1 - b2);  // exact integer difference (both >= -2^30)
          if (__popc(m1) < c.p.min_static_rays) {
            fail = !(gap > 2.0f * errq);
          } else {
            const int k0 = __ffs(vb) - 1;
            float qs = 0.0f, ac = 0.0f, s2u = 0.0f;
#pragma unroll 1
            for (int w = 0; w < 4; ++w) {
              float ref[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
              for (int k = 0; k < ST_MAX_VIEWS; ++k)
                if (k == k0)
                  desc_word32<RECT>(desc + (size_t)k * c.HW * 4, idx[k], su, sv, fu[k], fv[k], w,
                                    ref);
              float b1s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
              for (int k = 0; k < ST_MAX_VIEWS; ++k) {
                if (!((m1 >> k) & 1)) continue;
                float x[4];
                desc_word32<RECT>(desc + (size_t)k * c.HW * 4, idx[k], su, sv, fu[k], fv[k], w, x);
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                  const float gdev = x[jj] - ref[jj];
                  b1s[jj] += gdev;
                  qs = fmaf(gdev, gdev, qs);
                  s2u = fmaf(x[jj], x[jj], s2u);
                }
              }
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) ac = fmaf(b1s[jj], b1s[jj], ac);
            }
            const float n = (float)__popc(m1);
            const float rn = 1.0f / n;
            const float var = fmaxf((qs - ac * rn) * rn, 0.0f);
            // estep_small's D generalised to n <= 12 rays (16 n samples)
            const float D = 2.0f * (fabsf(beta) * ((4.0f * n + 44.0f) * U * qs +
                                                   2.0f * U * fmaxf(ceil32, qs) +
                                                   7.1054274e-15f * s2u + 2.0f * U * ceil32 +
                                                   2.0f * eps32 * sqrtf(16.0f * n * qs) +
                                                   16.0f * n * eps32 * eps32));
            fail = !(gap / QS - beta * var - D > 2.0f * errq / QS);
          }
        }
        if (!fail) {
          const int64_t o = a.scatter ? pix : i;
          a.static_out[o] = m1;
          a.valid_out[o] = vb;
        }
      }
    }
    list_append(fail, (int32_t)i, a.flist, a.flist_count);
  }
}

template __global__ void k_e_step_cert_big<false>(EmCtx, EStepArgs);
template __global__ void k_e_step_cert_big<true>(EmCtx, EStepArgs);

template __global__ void k_e_step_cert<2, false>(EmCtx, EStepArgs);
template __global__ void k_e_step_cert<3, false>(EmCtx, EStepArgs);
template __global__ void k_e_step_cert<4, false>(EmCtx, EStepArgs);
template __global__ void k_e_step_cert<5, false>(EmCtx, EStepArgs);
template __global__ void k_e_step_cert<2, true>(EmCtx, EStepArgs);
template __global__ void k_e_step_cert<3, true>(EmCtx, EStepArgs);
template __global__ void k_e_step_cert<4, true>(EmCtx, EStepArgs);
template __global__ void k_e_step_cert<5, true>(EmCtx, EStepArgs);

// E-step for 6 <= K <= 12 views: rays staged in shared memory, masks
// enumerated one at a time (estep_generic).
__global__ void __launch_bounds__(ESTEP_BLOCK) k_e_step_at(EmCtx c, EStepArgs a) {
  extern __shared__ double sh_f[];
  if (a.stop && *a.stop) return;  // converged (st_solve_async)
  const int64_t n_work = a.list ? (int64_t)*a.list_count : a.n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_work;
       t += (int64_t)gridDim.x * blockDim.x) {
  const int64_t i = a.list ? (int64_t)a.list[t] : t;
  if (a.status && a.status[i] == ST_STATUS_LOW_TEXTURE) continue;  // solver.py:476-478
  const int64_t pix = a.pix ? a.pix[i] : c.pix0 + i;
  const double u = (double)(pix % c.W), v = (double)(pix / c.W);
  const double d = a.d[i];
  double* f = sh_f + threadIdx.x;
  const int stride = blockDim.x;
  const int K = c.rig.num_views;
  double l1[ST_MAX_VIEWS], l0[ST_MAX_VIEWS];
  uint32_t vb = 0;
  // gather_rays (solver.py:206-227): invalid rays carry desc 0 and q 0.5
  for (int k = 0; k < K; ++k) {
    const WarpOut w = warp_ctx(c, k, u, v, d);
    double q = 0.5;
    if (in_margin(c.rig, k, w)) {
      const Taps tp = taps_ctx(c, w);
      sample_desc(c.desc + (size_t)k * c.HW, c.W, tp,
                  [&](int ch, double x) { f[(k * 16 + ch) * stride] = x; });
      q = sample_prior(c.priors + (size_t)k * c.HW, c.W, tp);
      vb |= 1u << k;
    } else {
#pragma unroll
      for (int ch = 0; ch < 16; ++ch) f[(k * 16 + ch) * stride] = 0.0;
    }
    clamp_logs(q, c.p.epsilon_prior, a.eps_logs, l1[k], l0[k]);
  }
  const uint32_t m = a.exhaustive ? estep_generic(K, f, stride, l1, l0, vb, c.p)
                                  : estep_bnb(K, f, stride, l1, l0, vb, c.p);
  const int64_t o = a.scatter ? pix : i;
  a.static_out[o] = m;
  a.valid_out[o] = vb;
  }
}

// The K >= 6 fallback on rectified rigs without the shared-memory ray
// staging: each ray keeps only its tap (descriptor index, horizontal
// weight) in shared memory (12 B instead of 128 B of fp64 samples), and a
// mask's exact score re-samples its rays' descriptors (L1/L2 hits) with the
// arithmetic of gather_rays + score_generic: channels 0-7 then 8-15 (two
// passes of 8 accumulators), each channel's sums over the mask's views in
// view order, the 16 channel terms added in channel order.  Same outputs as
// k_e_step_at with ~10x less shared memory per pixel (occupancy).
#ifndef ESTEP_AT_TAPS_MIN_BLOCKS
#define ESTEP_AT_TAPS_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(ESTEP_BLOCK, ESTEP_AT_TAPS_MIN_BLOCKS)
    k_e_step_at_taps(EmCtx c, EStepArgs a) {
  __shared__ uint32_t s_off[ST_MAX_VIEWS * ESTEP_BLOCK];
  __shared__ double s_fu[ST_MAX_VIEWS * ESTEP_BLOCK];
  if (a.stop && *a.stop) return;  // converged (st_solve_async)
  const int64_t n_work = a.list ? (int64_t)*a.list_count : a.n;
  const int K = c.rig.num_views;
  uint32_t* toff = s_off + threadIdx.x;
  double* tfu = s_fu + threadIdx.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_work;
       t += (int64_t)gridDim.x * blockDim.x) {
  const int64_t i = a.list ? (int64_t)a.list[t] : t;
  if (a.status && a.status[i] == ST_STATUS_LOW_TEXTURE) continue;  // solver.py:476-478
  const int64_t pix = a.pix ? a.pix[i] : c.pix0 + i;
  const int x = (int)(pix % c.W), y = (int)(pix / c.W);
  const double u = (double)x, v = (double)y;
  const double d = a.d[i];
  const uint32_t row = (uint32_t)y * (uint32_t)c.W;
  double l1[ST_MAX_VIEWS], l0[ST_MAX_VIEWS];
  uint32_t vb = 0;
  // gather_rays (solver.py:206-227): taps of the valid rays, priors at them
  for (int k = 0; k < K; ++k) {
    const WarpOut w = warp_ctx(c, k, u, v, d);
    double q = 0.5;
    if (in_margin(c.rig, k, w)) {
      const Taps tp = taps_ctx(c, w);
      toff[k * ESTEP_BLOCK] = (uint32_t)k * (uint32_t)c.HW + row + (uint32_t)tp.iu;
      tfu[k * ESTEP_BLOCK] = tp.fu;
      q = sample_prior(c.priors + (size_t)k * c.HW, c.W, tp);
      vb |= 1u << k;
    }
    clamp_logs(q, c.p.epsilon_prior, a.eps_logs, l1[k], l0[k]);
  }
  auto score = [&](uint32_t m) -> double {
    const int pop = __popc(m);
    double vr;
    if (pop < c.p.min_static_rays) {
      vr = variance_ceiling();
    } else {
      double acc = 0.0;
#pragma unroll 1
      for (int ps = 0; ps < 2; ++ps) {
        double a1[8], a2[8];
        int n = 0;
        for (uint32_t r = m; r; r &= r - 1) {
          const int k = __ffs(r) - 1;
          const uint4* pl = c.desc + toff[k * ESTEP_BLOCK];
          const uint4 ta = __ldg(pl), tb = __ldg(pl + 1);
          const double fu = tfu[k * ESTEP_BLOCK];
          double xv[8];
          lerp_word(ps ? ta.z : ta.x, ps ? tb.z : tb.x, fu, *reinterpret_cast<double(*)[4]>(xv));
          lerp_word(ps ? ta.w : ta.y, ps ? tb.w : tb.y, fu,
                    *reinterpret_cast<double(*)[4]>(xv + 4));
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const double x2 = dmul(xv[j], xv[j]);
            a1[j] = n ? dadd(a1[j], xv[j]) : xv[j];
            a2[j] = n ? dadd(a2[j], x2) : x2;
          }
          ++n;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc = dadd(acc, dsub(a2[j], div_n(dmul(a1[j], a1[j]), n)));
      }
      vr = fmax(div_n(acc, pop), 0.0);
    }
    double sa = 0.0, sb = 0.0;
    for (int k = 0; k < K; ++k) {
      if ((m >> k) & 1)
        sa = dadd(sa, l1[k]);
      else
        sb = dadd(sb, l0[k]);
    }
    return dsub(dadd(sa, sb), dmul(c.p.beta, vr));
  };
  const uint32_t m = estep_bnb_core(K, l1, l0, vb, c.p, score);
  const int64_t o = a.scatter ? pix : i;
  a.static_out[o] = m;
  a.valid_out[o] = vb;
  }
}

// initial_masks (solver.py:421-432): valid & q >= threshold at mu.
__global__ void k_initial_masks(EmCtx c, const int64_t* __restrict__ pix_list, int64_t n,
                                uint32_t* __restrict__ static_out,
                                uint32_t* __restrict__ valid_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t pix = pix_list ? pix_list[i] : c.pix0 + i;
  const double u = (double)(pix % c.W), v = (double)(pix / c.W);
  const double d = c.mu[pix];
  uint32_t sb = 0, vb = 0;
  for (int k = 0; k < c.rig.num_views; ++k) {
    const WarpOut w = warp_ctx(c, k, u, v, d);
    if (!in_margin(c.rig, k, w)) continue;
    const Taps t = taps_ctx(c, w);
    const double q = sample_prior(c.priors + (size_t)k * c.HW, c.W, t);
    vb |= 1u << k;
    if (q >= c.p.threshold) sb |= 1u << k;
  }
  static_out[i] = sb;
  valid_out[i] = vb;
}

// gather_rays API (solver.py:206-227).
__global__ void k_gather_rays(EmCtx c, const int64_t* __restrict__ pix, const double* __restrict__ d,
                              int64_t n, double* __restrict__ desc, uint8_t* __restrict__ valid,
                              double* __restrict__ q) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int K = c.rig.num_views;
  const int64_t p = pix[i];
  const double u = (double)(p % c.W), v = (double)(p / c.W);
  for (int k = 0; k < K; ++k) {
    double* out = desc + ((size_t)i * K + k) * 16;
    const WarpOut w = warp_to(c.rig, k, u, v, d[i]);
    if (in_margin(c.rig, k, w)) {
      const Taps t = taps_ctx(c, w);
      sample_desc(c.desc + (size_t)k * c.HW, c.W, t, [&](int ch, double x) { out[ch] = x; });
      q[(size_t)i * K + k] = sample_prior(c.priors + (size_t)k * c.HW, c.W, t);
      valid[(size_t)i * K + k] = 1;
    } else {
      for (int ch = 0; ch < 16; ++ch) out[ch] = 0.0;
      q[(size_t)i * K + k] = 0.5;
      valid[(size_t)i * K + k] = 0;
    }
  }
}

// _energy API (solver.py:229-260) on explicit (pixel, d, mask) triples.
__global__ void k_energy(EmCtx c, const int64_t* __restrict__ pix, const double* __restrict__ d,
                         const uint32_t* __restrict__ bits, int64_t n, double* __restrict__ e,
                         uint8_t* __restrict__ real) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t p = pix[i];
  const double lp = log_prior(d[i], c.mu[p], c.p.sigma, c.p.gamma, c.inv_sigma);
  const Energy E = energy_at(c, (double)(p % c.W), (double)(p / c.W), d[i], bits[i], lp);
  e[i] = E.e;
  real[i] = E.real ? 1 : 0;
}

// Standalone e_step on caller-gathered rays (n, K, 16) f64.
__global__ void __launch_bounds__(ESTEP_BLOCK) k_e_step_rays(const double* __restrict__ desc,
                                                             const uint8_t* __restrict__ valid,
                                                             const double* __restrict__ q, int64_t n,
                                                             int K, st_params p,
                                                             uint32_t* __restrict__ out) {
  extern __shared__ double sh_f[];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* f = sh_f + threadIdx.x;
  double l1[ST_MAX_VIEWS], l0[ST_MAX_VIEWS];
  uint32_t vb = 0;
  for (int k = 0; k < K; ++k) {
    for (int ch = 0; ch < 16; ++ch) f[(k * 16 + ch) * blockDim.x] = desc[((size_t)i * K + k) * 16 + ch];
    if (valid[(size_t)i * K + k]) vb |= 1u << k;
    clamp_logs(q[(size_t)i * K + k], p.epsilon_prior, l1[k], l0[k]);
  }
  out[i] = estep_dispatch(K, f, blockDim.x, l1, l0, vb, p);
}

// masked_variance (solver.py:93-107): two-pass in double precision.
__global__ void k_masked_variance(const double* __restrict__ desc, const uint8_t* __restrict__ mask,
                                  int64_t n, int K, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int cnt = 0;
  for (int k = 0; k < K; ++k) cnt += mask[(size_t)i * K + k] ? 1 : 0;
  if (cnt == 0) {
    out[i] = NAN;
    return;
  }
  // sel.sum(axis=0) / n: pairwise over rows is sequential for < 8 rows;
  // numpy sums axis 0 of a (n, 16) array row by row.
  double mean[16];
  for (int ch = 0; ch < 16; ++ch) mean[ch] = 0.0;
  bool first = true;
  for (int k = 0; k < K; ++k) {
    if (!mask[(size_t)i * K + k]) continue;
    for (int ch = 0; ch < 16; ++ch) {
      const double x = desc[((size_t)i * K + k) * 16 + ch];
      mean[ch] = first ? x : dadd(mean[ch], x);
    }
    first = false;
  }
  for (int ch = 0; ch < 16; ++ch) mean[ch] = ddiv(mean[ch], (double)cnt);
  // ((sel - mean) ** 2).sum(): one contiguous reduction over cnt*16 values
  // (numpy pairwise: 8 accumulators over blocks of 128, then the tree).
  double acc[8];
  for (int j = 0; j < 8; ++j) acc[j] = 0.0;
  const int total = cnt * 16;
  int idx = 0;
  double tail = 0.0;
  bool tail_first = true;
  const int main_n = total < 8 ? 0 : total - (total % 8);
  for (int k = 0; k < K; ++k) {
    if (!mask[(size_t)i * K + k]) continue;
    for (int ch = 0; ch < 16; ++ch, ++idx) {
      const double dlt = dsub(desc[((size_t)i * K + k) * 16 + ch], mean[ch]);
      const double sq = dmul(dlt, dlt);
      if (idx < main_n) {
        acc[idx & 7] = idx < 8 ? sq : dadd(acc[idx & 7], sq);
      } else {
        tail = tail_first ? sq : dadd(tail, sq);
        tail_first = false;
      }
    }
  }
  double s = dadd(dadd(dadd(acc[0], acc[1]), dadd(acc[2], acc[3])),
                  dadd(dadd(acc[4], acc[5]), dadd(acc[6], acc[7])));
  if (!tail_first) s = dadd(s, tail);
  out[i] = ddiv(s, (double)cnt);
}

// solve() output packing (solver.py:491-500).
// dense: slots 0..npx-1 are pixels pix0 + i.
__global__ void k_pack_outputs(const double* __restrict__ mu, int64_t npx, int64_t pix0,
                               const int64_t* __restrict__ active, int64_t n_active,
                               const double* __restrict__ d_act,
                               const uint8_t* __restrict__ st_act, float* __restrict__ values,
                               uint8_t* __restrict__ status, int dense, const uint32_t* n_dev) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n_dev) n_active = *n_dev;
  if (dense) {
    if (i >= npx) return;
    const int64_t p = pix0 + i;
    if (d_act) {
      const double d = d_act[i];
      values[p] = isnan(d) ? 0.0f : (float)d;
      status[p] = st_act[i];
    } else {
      values[p] = (float)mu[p];
      status[p] = ST_STATUS_VALID;
    }
    return;
  }
  // sparse: first pass (fill) is done by k_fill_mu; scatter active results
  if (i >= n_active || !d_act) return;
  const int64_t p = active[i];
  const double d = d_act[i];
  values[p] = isnan(d) ? 0.0f : (float)d;
  status[p] = st_act[i];
}

__global__ void k_fill_mu(const double* __restrict__ mu, int64_t npx, float* __restrict__ values,
                          uint8_t* __restrict__ status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npx) return;
  values[i] = (float)mu[i];
  status[i] = ST_STATUS_VALID;
}


// dynamic_only / explicit active-set compaction: count then scatter, in
// pixel order (the reference's `active` is ascending).
__global__ void k_flag_active(const float* __restrict__ ref_prior, const uint8_t* __restrict__ mask,
                              int64_t npx, double threshold, uint32_t* __restrict__ flags,
                              int64_t lo, int64_t hi) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npx) return;
  // numpy compares the float32 prior against the Python float in float32 (NEP 50);
  // [lo, hi): the pixel window of a row band (the whole frame otherwise)
  const bool on = mask ? mask[i] != 0 : ref_prior[i] < (float)threshold;
  flags[i] = (on && i >= lo && i < hi) ? 1u : 0u;
}

__global__ void k_scatter_active(const uint32_t* __restrict__ flags,
                                 const uint32_t* __restrict__ offs, int64_t npx,
                                 int64_t* __restrict__ active) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npx) return;
  if (flags[i]) active[offs[i]] = i;
}

__global__ void k_stats_init(st_stats* stats, int64_t n_act) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    stats->converged_after = -1;
    stats->active_pixels = n_act;
    stats->kernel_launches[2] = 1;  // k_initial_masks
  }
}

// Device-side EM control (solver.py:463-485): one thread.  `r` is the
// iteration's (all-shard) record, n_act the (global) active count.
__device__ void control_step(int it, const Partial& r, int64_t n_act, long long mwork,
                             long long ework, int forced_iters, st_stats* __restrict__ stats,
                             int* __restrict__ stop) {
  stats->iterations_run = it;
  stats->msteps += mwork;
  stats->esteps += ework;
  if (it > 1) stats->prev_evals += mwork;
  stats->kernel_launches[0] += 1;
  stats->kernel_launches[1] += 1;
  stats->kernel_launches[3] += it > 1 ? 3 : 2;
  const double nf = (double)r.n_fin;
  stats->mean_energy[it - 1] = nf > 0 ? r.sum_e / nf : NAN;
  stats->candidates_total += r.n_cand;
  stats->energy_evals += r.n_eval;
  stats->hopeless_msteps += r.n_hopeless;
  stats->energy_samples += r.n_samples;
  if (it > 1) {
    const double npf = (double)r.n_pfin;
    stats->prev_energy[it - 2] = npf > 0 ? r.sum_pe / npf : NAN;
    const double changed = (double)r.n_changed / (double)n_act;
    stats->changed_fraction[it - 2] = changed;
    if (forced_iters <= 0 && changed < 1e-3) {  // solver.py:483-485
      stats->converged_after = it - 1;
      *stop = 1;
    }
  }
}

__device__ void solve_control(int it, const Partial* __restrict__ reduced,
                              uint32_t* __restrict__ counts, int64_t n_act, int forced_iters,
                              st_stats* __restrict__ stats, int* __restrict__ stop) {
  const Partial r = reduced[it];
  control_step(it, r, n_act, it > 1 ? (long long)counts[0] : (long long)n_act,
               (long long)counts[1], forced_iters, stats, stop);
  counts[0] = 0;  // next iteration's worklists
  counts[1] = 0;
}

__device__ void band_control(int it, const Partial* __restrict__ gathered, int world,
                             int forced_iters, st_stats* __restrict__ stats,
                             int* __restrict__ stop) {
  Partial r = gathered[0];
  for (int w = 1; w < world; ++w) {  // rank order: identical on every shard
    const Partial& g = gathered[w];
    r.sum_e += g.sum_e;
    r.sum_pe += g.sum_pe;
    r.n_fin += g.n_fin;
    r.n_pfin += g.n_pfin;
    r.n_changed += g.n_changed;
    r.n_cand += g.n_cand;
    r.n_eval += g.n_eval;
    r.n_hopeless += g.n_hopeless;
    r.n_samples += g.n_samples;
    r.n_act += g.n_act;
    r.n_mwork += g.n_mwork;
    r.n_ework += g.n_ework;
    r.n_unsafe += g.n_unsafe;
  }
  if (r.n_unsafe > 0) {  // a shard's surface raster was not exact: redo the frame
    *stop = 2;
    return;
  }
  if (it == 1) stats->active_pixels = r.n_act;
  if (r.n_act == 0) {  // solver.py:486-488: no active pixel anywhere
    stats->converged_after = 0;
    *stop = 1;
    return;
  }
  control_step(it, r, r.n_act, r.n_mwork, r.n_ework, forced_iters, stats, stop);
}

__global__ void k_band_control(int it, const Partial* __restrict__ gathered, int world,
                               int forced_iters, st_stats* __restrict__ stats,
                               int* __restrict__ stop, BandLoop loop) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (*stop) {
    if (loop.use_cond) cudaGraphSetConditional(loop.cond, 0u);
    return;
  }
  if (loop.it_off) {  // the graph loop: the iteration and its record on the device
    it += (int)*loop.it_off;
    gathered += *loop.it_off;
  }
  band_control(it, gathered, world, forced_iters, stats, stop);
  if (loop.it_off) *loop.it_off += 1u;
  if (loop.use_cond) cudaGraphSetConditional(loop.cond, (*stop == 0 && it + 1 <= loop.iters) ? 1u : 0u);
}


}  // namespace st
