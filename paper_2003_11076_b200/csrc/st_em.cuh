// Kernel-side context and kernel declarations of the EM core.
#pragma once

#include <stdint.h>

#include "st_common.cuh"

#define EM_BLOCK 128
// M-step energies in two passes of 8 channel sums (energy_at), 5 resident
// blocks per SM (<= 96 registers): measured fastest on B200
#ifndef ENERGY_SINGLE_PASS
#define ENERGY_TWO_PASS
#endif
#ifndef MSTEP_MIN_BLOCKS
#define MSTEP_MIN_BLOCKS 5
#endif
#define MSTEP_BOUNDS __launch_bounds__(EM_BLOCK, MSTEP_MIN_BLOCKS)
#define STATS_BLOCK 256
#define ESTEP_BLOCK 64
#define ESTEP_TAPS_BLOCK 128
#define ESTEP_CERT_BLOCK 128
#define CERT_BIG_BLOCK 128
#ifndef ESTEP_CERT_MIN_BLOCKS
#define ESTEP_CERT_MIN_BLOCKS 8  // <= 64 registers (no spills; measured best)
#endif
#ifndef ESTEP_MIN_BLOCKS
#define ESTEP_MIN_BLOCKS 4  // <= 128 registers
#endif
#define ST_MAX_BAND 64

namespace st {

// Everything a pixel thread needs, passed by value (lands in the constant bank).
struct EmCtx {
  st_rig rig;
  st_params p;
  int W, H;
  int64_t HW;
  const uint4* desc;     // (K, H*W) 16-byte descriptors
  const float* priors;   // (K, H*W)
  const double* mu;      // (H*W) clipped surface
  double band[ST_MAX_BAND];
  int n_band;
  int n_coarse;
  const uint32_t* sup_tile_start;
  const float* sup_value;
  const uint32_t* sup_mask;
  int tiles_x;
  int sup_ir;
  double sup_r2;
  double inv_sigma;     // 1/sigma when sigma is a power of two (exact), else 0
  float sigma_f;        // fp32 sigma / gamma for the pruning radius
  float gamma_f;
  int rectified;        // every view: A = I, b = (bx, 0, 0) -> 1-D horizontal warp
  double recip[ST_MAX_VIEWS + 1];  // RN(1/n), n = 1..12, for div_small
  uint32_t view_bits;   // (1 << K) - 1
  int exhaustive;       // M-step: no pruning, every candidate evaluated (cross-check)
  int64_t pix0;         // dense slots: slot i -> pixel pix0 + i (row bands; 0 otherwise)
};

struct Partial {
  double sum_e, sum_pe;
  long long n_fin, n_pfin, n_changed, n_cand, n_eval;
  long long n_hopeless;  // M-step pixels with fewer static views than min_static_rays
  long long n_samples;   // M-step descriptor samples (static in-margin rays of real candidates)
  // row-band record (st_solve_rows): the shard's counted active pixels and its
  // M/E worklist sizes, summed over shards by k_band_control
  long long n_act, n_mwork, n_ework;
  long long n_unsafe;  // shards whose row-window mu raster was not exact
};

// Slots are the rows of the active set (slot i -> pixel active[i], or i when
// dense).  All per-slot arrays are indexed by slot.
struct MStepArgs {
  const int64_t* active;       // nullable: dense over all pixels
  int64_t n;                   // number of slots
  const int32_t* list;         // nullable: worklist of slots (count in *list_count)
  const uint32_t* list_count;
  const uint32_t* static_all;  // per pixel
  int first;                   // 1: no previous disparity (iteration 1 / API)
  double* d;                   // out; in = previous disparity when !first
  double* e;
  uint8_t* status;
  uint32_t* mask_in;           // nullable: mask each slot was solved with
  double* pe;                  // !first: energy of the previous d under the mask
  uint8_t* chg;                // !first: |d - d_prev| > 0.5
  int32_t* elist;              // nullable: E-step worklist (append)
  uint32_t* elist_count;
  Partial* partials;           // nullable: per-warp work counters
  const int* stop;             // nullable: device flag, set -> the launch does nothing
  const uint32_t* n_dev;       // nullable: the slot count on the device (n: its upper bound)
};

struct EStepArgs {
  const int64_t* pix;        // nullable: dense
  int64_t n;
  const int32_t* list;       // nullable: worklist of rows (count in *list_count)
  const uint32_t* list_count;
  const double* d;
  const uint8_t* status;     // nullable; LOW_TEXTURE rows are skipped
  uint32_t* static_out;
  uint32_t* valid_out;
  int scatter;               // 1: write at pixel index, 0: at row i
  int exhaustive;            // 1: score every mask in fp64 (no fp32 screen)
  const int* stop;           // nullable: device flag, set -> the launch does nothing
  const double* eps_logs;    // nullable: k_eps_logs output (clamped-prior logs)
  int32_t* flist;            // k_e_step_cert: rows it could not certify (append) ...
  uint32_t* flist_count;     // ... and their count (zeroed by the launcher)
};

__global__ void k_m_step(EmCtx c, MStepArgs a);
__global__ void k_flag_mstep(const int64_t* active, int64_t n, int64_t pix0,
                             const uint32_t* static_all,
                             const uint32_t* mask_in, const double* e, double* pe, uint8_t* chg,
                             int32_t* list, uint32_t* count, const int* stop = nullptr,
                             const uint32_t* n_dev = nullptr);
// k_em_stats' last block folds the blocks' records and runs the iteration's
// control (st_solve_async) or writes the record (row bands, st_solve).
struct StatsTail {
  int on;
  int it;
  unsigned* done;          // zero-initialised block counter (reset by the last block)
  Partial* reduced;
  uint32_t* counts;
  int64_t n_act;
  int forced_iters;
  st_stats* stats;
  int* stop_rw;
  uint32_t* flist_count;   // nullable: the E-step fallback count, cleared for the next E-step
  // row bands: the last block only writes this shard's record into
  // reduced[it] (+ n_act = record_n_act, the worklist sizes) and clears the
  // worklist counts; k_band_control runs the control after the exchange
  int record_only;
  long long record_n_act;
  long long record_slots;  // iteration 1's M-step count (every slot)
  int keep_counts;         // st_solve (host loop): leave the worklist counts to the host
  // numpy's summation order (st_mean.cu): the grid is the top pw_depth levels
  // of np.add.reduce's pairwise tree; non-finite values take the slow path
  int pw_depth;
  double* pw_scratch;      // n doubles: the finite values, compacted
  double* pw_val;          // pw_val_size(n) doubles: the slow path's tree levels
  const int32_t* mu_unsafe;  // nullable: st_mu_raster_rows' flag, into the shard record
  // CUDA-graph loop (st_api.cu, iterations >= 3 in a conditional WHILE node):
  // the iteration is it + *it_off (it_off nullable; the last block advances
  // it), and the kernel sets the loop's condition: another iteration unless
  // stopped or past `iters`
  uint32_t* it_off;
  int use_cond;
  int iters;
  cudaGraphConditionalHandle cond;
  // nullable: the counted slots' number on the device (dynamic_only's active
  // list, no host read-back); the kernel's n and pw_depth are then upper
  // bounds (the grid), the tree depth is derived on the device
  const uint32_t* n_dev;
};
// grid of k_em_stats for n counted slots (1 << pw_depth blocks) and its depth
__host__ __device__ int stats_depth(int64_t n);
int64_t pw_val_size(int64_t n);
// Per-iteration statistics (solver.py:463-475): the mean of the finite M-step
// energies and previous-disparity energies summed in numpy's own order
// (st_mean.cu), the changed count and the M-step work counters; the last
// block folds the blocks' records and runs the control (or writes the
// shard's record, tail.record_only).
__global__ void k_em_stats(int64_t n, int with_prev, const double* e, const double* pe,
                           const uint8_t* chg, const Partial* work, int n_work_parts,
                           Partial* parts, const int* stop, StatsTail tail);
template <int KT, bool RECT>
__global__ void k_e_step_taps(EmCtx c, EStepArgs a);
__global__ void k_e_step_at(EmCtx c, EStepArgs a);
// K >= 6 on rectified rigs: taps in shared memory, samples re-read per scored mask
__global__ void k_e_step_at_taps(EmCtx c, EStepArgs a);
template <int KT, bool RECT>
__global__ void k_e_step_cert(EmCtx c, EStepArgs a);
template <bool RECT>
__global__ void k_e_step_cert_big(EmCtx c, EStepArgs a);
__global__ void k_initial_masks(EmCtx c, const int64_t* pix, int64_t n, uint32_t* static_out,
                                uint32_t* valid_out);
__global__ void k_gather_rays(EmCtx c, const int64_t* pix, const double* d, int64_t n,
                              double* desc, uint8_t* valid, double* q);
__global__ void k_energy(EmCtx c, const int64_t* pix, const double* d, const uint32_t* bits,
                         int64_t n, double* e, uint8_t* real);
__global__ void k_e_step_rays(const double* desc, const uint8_t* valid, const double* q,
                              int64_t n, int K, st_params p, uint32_t* out);
__global__ void k_masked_variance(const double* desc, const uint8_t* mask, int64_t n, int K,
                                  double* out);
__global__ void k_pack_outputs(const double* mu, int64_t npx, int64_t pix0, const int64_t* active,
                               int64_t n_active, const double* d_act, const uint8_t* st_act,
                               float* values, uint8_t* status, int dense,
                               const uint32_t* n_dev = nullptr);
__global__ void k_fill_mu(const double* mu, int64_t npx, float* values, uint8_t* status);
__global__ void k_stats_init(st_stats* stats, int64_t n_act);
// Row bands: sum the shards' records (rank order, deterministic) and run the
// iteration's control exactly as the statistics kernel does for one device.
// `loop` (zero: off) is the graph loop's state, as in StatsTail: iteration
// it + *it_off, record gathered[*it_off], and the WHILE condition.
struct BandLoop {
  uint32_t* it_off;
  int use_cond;
  int iters;
  cudaGraphConditionalHandle cond;
  // nullable: the counted slots' number on the device (dynamic_only's active
  // list, no host read-back); the kernel's n and pw_depth are then upper
  // bounds (the grid), the tree depth is derived on the device
  const uint32_t* n_dev;
};
__global__ void k_band_control(int it, const Partial* gathered, int world, int forced_iters,
                               st_stats* stats, int* stop, BandLoop loop);
// log(eps), log(1 - eps), log(1 - (1 - eps)) with the device log: the E-step
// reuses them for rays whose prior is clamped (identical values).
__global__ void k_eps_logs(double eps, double* out);
__global__ void k_flag_active(const float* ref_prior, const uint8_t* mask, int64_t npx,
                              double threshold, uint32_t* flags, int64_t lo, int64_t hi);
__global__ void k_scatter_active(const uint32_t* flags, const uint32_t* offs, int64_t npx,
                                 int64_t* active);

}  // namespace st


