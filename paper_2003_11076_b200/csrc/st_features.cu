// Dense 16-byte ring descriptors (features.py:29-104) for K views at once.
//
// One CTA owns a 32x8 output tile of one view: it stages the edge-replicated
// gray tile (+3 px halo) and the biased Sobel tile (+2 px halo) in shared
// memory, then every thread writes its descriptor as a single 16-byte store.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "st_common.cuh"

namespace st {

#define DT_W 32
#define DT_H 8

__constant__ int c_ring_du[8] = {0, 1, 2, 1, 0, -1, -2, -1};  // features.py:24
__constant__ int c_ring_dv[8] = {-2, -1, 0, 1, 2, 1, 0, -1};

__device__ __forceinline__ int gray_at(const uint8_t* __restrict__ img, int channels, int W,
                                       int y, int x) {
  const uint8_t* p = img + ((size_t)y * W + x) * channels;
  if (channels == 1) return p[0];
  // features.py:34-36: R*0.299 + G*0.587 + B*0.114 in fp64, left to right, rint
  const double g = dadd(dadd(dmul((double)p[0], 0.299), dmul((double)p[1], 0.587)),
                        dmul((double)p[2], 0.114));
  return (int)rint(g);
}

__device__ __forceinline__ uint8_t sobel_code(int raw) {
  // features.py:56-57: clip(rint(128 + raw / 4), 0, 255), half to even
  const double r = rint(dadd(128.0, dmul((double)raw, 0.25)));
  return (uint8_t)fmin(fmax(r, 0.0), 255.0);
}

// The same two codes in integer arithmetic (exact):
// * gray: the fp64 sum is N/1000 + O(1e-13) with N = 299 R + 587 G + 114 B,
//   so rint agrees with rounding N/1000 unless N/1000 is exactly a half
//   (N mod 1000 == 500), where the fp64 roundings decide: recompute those.
// * Sobel: 128 + raw/4 = t/4 with t = 512 + raw exactly; rint half to even.
__device__ __forceinline__ int gray_int(int r, int g, int b) {
  const int n = 299 * r + 587 * g + 114 * b;
  const int k = n / 1000, rem = n - 1000 * k;
  if (rem != 500) return k + (rem > 500 ? 1 : 0);
  const double v = dadd(dadd(dmul((double)r, 0.299), dmul((double)g, 0.587)),
                        dmul((double)b, 0.114));
  return (int)rint(v);
}

__device__ __forceinline__ uint8_t sobel_code_int(int raw) {
  const int t = 512 + raw;
  const int q = t >> 2, rem = t & 3;  // t = 4q + rem, rem in [0, 3]
  const int v = q + (rem > 2 || (rem == 2 && (q & 1)) ? 1 : 0);
  return (uint8_t)min(max(v, 0), 255);
}

__global__ void __launch_bounds__(DT_W* DT_H) k_descriptors(const uint8_t* __restrict__ images,
                                                            int H, int W, int channels,
                                                            uint4* __restrict__ desc,
                                                            uint8_t* __restrict__ gray_out,
                                                            uint8_t* __restrict__ sobel_out) {
  __shared__ int16_t g[DT_H + 6][DT_W + 6];     // gray, clamped coordinates
  __shared__ uint8_t sx[DT_H + 4][DT_W + 4];    // biased gx
  __shared__ uint8_t sy[DT_H + 4][DT_W + 4];    // biased gy
  const int k = blockIdx.z;
  const uint8_t* img = images + (size_t)k * H * W * channels;
  const int x0 = blockIdx.x * DT_W, y0 = blockIdx.y * DT_H;
  const int tid = threadIdx.y * DT_W + threadIdx.x;
  const int nthr = DT_W * DT_H;

  for (int i = tid; i < (DT_H + 6) * (DT_W + 6); i += nthr) {
    const int r = i / (DT_W + 6), cidx = i % (DT_W + 6);
    const int yy = min(max(y0 - 3 + r, 0), H - 1);
    const int xx = min(max(x0 - 3 + cidx, 0), W - 1);
    g[r][cidx] = (int16_t)gray_at(img, channels, W, yy, xx);
  }
  __syncthreads();
  for (int i = tid; i < (DT_H + 4) * (DT_W + 4); i += nthr) {
    const int r = i / (DT_W + 4), cidx = i % (DT_W + 4);
    const int gr = r + 1, gc = cidx + 1;  // position in the gray tile
    // features.py:49-55 (correlation with the Sobel kernels, edge padded)
    const int colR = g[gr - 1][gc + 1] + 2 * g[gr][gc + 1] + g[gr + 1][gc + 1];
    const int colL = g[gr - 1][gc - 1] + 2 * g[gr][gc - 1] + g[gr + 1][gc - 1];
    const int rowD = g[gr + 1][gc - 1] + 2 * g[gr + 1][gc] + g[gr + 1][gc + 1];
    const int rowU = g[gr - 1][gc - 1] + 2 * g[gr - 1][gc] + g[gr - 1][gc + 1];
    sx[r][cidx] = sobel_code(colR - colL);
    sy[r][cidx] = sobel_code(rowD - rowU);
  }
  __syncthreads();
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  if (x >= W || y >= H) return;
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int xx = x + c_ring_du[i], yy = y + c_ring_dv[i];
    uint32_t gx = 128, gy = 128;  // off-image ring samples stay at the bias
    if (xx >= 0 && xx < W && yy >= 0 && yy < H) {
      gx = sx[threadIdx.y + 2 + c_ring_dv[i]][threadIdx.x + 2 + c_ring_du[i]];
      gy = sy[threadIdx.y + 2 + c_ring_dv[i]][threadIdx.x + 2 + c_ring_du[i]];
    }
    const int b = 2 * i;
    w[b >> 2] |= gx << (8 * (b & 3));
    w[(b + 1) >> 2] |= gy << (8 * ((b + 1) & 3));
  }
  desc[(size_t)k * H * W + (size_t)y * W + x] = make_uint4(w[0], w[1], w[2], w[3]);
  const size_t o = (size_t)k * H * W + (size_t)y * W + x;
  if (gray_out) gray_out[o] = (uint8_t)g[threadIdx.y + 3][threadIdx.x + 3];
  if (sobel_out) {
    sobel_out[2 * o] = sx[threadIdx.y + 2][threadIdx.x + 2];
    sobel_out[2 * o + 1] = sy[threadIdx.y + 2][threadIdx.x + 2];
  }
}

// Wide-tile variant for RGB views (the production path): one CTA owns a
// 128x16 output tile.  The edge-clamped RGB rows of the tile (+3 px halo)
// are staged as raw bytes with 32-bit loads (many independent loads in
// flight per thread), then gray, Sobel and the ring are computed from
// shared memory exactly as in k_descriptors; each thread writes 8
// descriptors, a warp 32 consecutive ones per store.
#define DW_W 128
#define DW_H 16
#define DW_ROWB 432  // >= 3 * (DW_W + 6) + 15 bytes of one staged row (TMA: 16-byte start)

// TMA helpers (cp.async.bulk.tensor + an mbarrier carrying the byte count).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(256) k_descriptors_wide(const uint8_t* __restrict__ images,
                                                          int H, int W, size_t total_bytes,
                                                          uint4* __restrict__ desc,
                                                          uint8_t* __restrict__ gray_out,
                                                          uint8_t* __restrict__ sobel_out,
                                                          int row0, int row1,
                                                          const __grid_constant__ CUtensorMap tmap,
                                                          int use_tma) {
  __shared__ __align__(128) uint8_t raw[DW_H + 6][DW_ROWB];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int16_t g[DW_H + 6][DW_W + 6];
  __shared__ uint16_t sxy[DW_H + 4][DW_W + 4];  // gx | gy << 8; 0x8080 off-image
  __shared__ int roff[DW_H + 6];  // byte of pixel 0 of the row, relative to the staged start
  const int k = blockIdx.z;
  const size_t view = (size_t)k * H * W * 3;
  // rows [row0, row1) only (row bands; the whole frame otherwise)
  const int x0 = blockIdx.x * DW_W, y0 = row0 + blockIdx.y * DW_H;
  const int tid = threadIdx.x;
  const int cl0 = max(x0 - 3, 0), cl1 = min(x0 + DW_W + 3, W);  // clamped column range
  const uintptr_t buf0 = (uintptr_t)images, buf1 = buf0 + total_bytes;
  // Interior tiles (no edge replication needed): the whole (DW_H + 6) x
  // DW_ROWB staging box in one TMA load -- the view as a 3-D tensor of 32-bit
  // words (W*3/4, H, K), box (DW_ROWB/4, DW_H + 6, 1) from the 16-byte
  // boundary at or below pixel x0 - 3 (roff carries the offset, as for the
  // word loop below).  Edge tiles replicate the border and take the loop.
  const bool tma_tile = use_tma && x0 >= 3 && x0 + DW_W + 3 <= W && y0 >= 3 &&
                        y0 + DW_H + 3 <= H;
  if (tma_tile) {
    const int xb = 3 * (x0 - 3);  // first byte of the staged run
    const int xw = (xb >> 4) << 2;  // the box starts on a 16-byte boundary (a TMA rule)
    if (tid < DW_H + 6) roff[tid] = (xb - 4 * xw) - 3 * cl0;
    const uint32_t b = smem_u32(&bar);
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                   "r"((DW_H + 6) * DW_ROWB)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(&raw[0][0])),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(xw), "r"(y0 - 3), "r"(k), "r"(b)
          : "memory");
    }
    __syncthreads();  // (the barrier is initialised before anyone waits on it)
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(b)
        : "memory");
  }
  // stage rows: 32-bit words covering bytes [3 cl0, 3 cl1) of each clamped row
  const int words_per_row = (3 * (cl1 - cl0) + 6) / 4 + 1;
  for (int i = tid; !tma_tile && i < (DW_H + 6) * words_per_row; i += blockDim.x) {
    const int r = i / words_per_row, j = i % words_per_row;
    const int yy = min(max(y0 - 3 + r, 0), H - 1);
    const uintptr_t a0 = buf0 + view + ((size_t)yy * W + cl0) * 3;
    const uintptr_t w0 = a0 & ~(uintptr_t)3;
    if (j == 0) roff[r] = (int)(a0 - w0) - 3 * cl0;
    const uintptr_t wa = w0 + 4 * (uintptr_t)j;
    if (wa + 4 <= buf1) {
      *reinterpret_cast<uint32_t*>(&raw[r][4 * j]) = __ldg(reinterpret_cast<const uint32_t*>(wa));
    } else {
      for (int b = 0; b < 4; ++b)
        raw[r][4 * j + b] = wa + b < buf1 ? __ldg(reinterpret_cast<const uint8_t*>(wa + b)) : 0;
    }
  }
  __syncthreads();
  for (int i = tid; i < (DW_H + 6) * (DW_W + 6); i += blockDim.x) {
    const int r = i / (DW_W + 6), c = i % (DW_W + 6);
    const int xx = min(max(x0 - 3 + c, 0), W - 1);
    const uint8_t* px = &raw[r][roff[r] + 3 * xx];
    g[r][c] = (int16_t)gray_int(px[0], px[1], px[2]);  // features.py:34-36
  }
  __syncthreads();
  for (int i = tid; i < (DW_H + 4) * (DW_W + 4); i += blockDim.x) {
    const int r = i / (DW_W + 4), c = i % (DW_W + 4);
    const int gr = r + 1, gc = c + 1;
    const int colR = g[gr - 1][gc + 1] + 2 * g[gr][gc + 1] + g[gr + 1][gc + 1];
    const int colL = g[gr - 1][gc - 1] + 2 * g[gr][gc - 1] + g[gr + 1][gc - 1];
    const int rowD = g[gr + 1][gc - 1] + 2 * g[gr + 1][gc] + g[gr + 1][gc + 1];
    const int rowU = g[gr - 1][gc - 1] + 2 * g[gr - 1][gc] + g[gr - 1][gc + 1];
    const int xx = x0 - 2 + c, yy = y0 - 2 + r;
    // off-image ring samples read the bias (features.py:95-101)
    sxy[r][c] = (xx >= 0 && xx < W && yy >= 0 && yy < H)
                    ? (uint16_t)(sobel_code_int(colR - colL) | (sobel_code_int(rowD - rowU) << 8))
                    : (uint16_t)0x8080;
  }
  __syncthreads();
  // pixel e * 256 + tid of the tile: a warp writes 32 consecutive descriptors
#pragma unroll 2
  for (int e = 0; e < 8; ++e) {
    const int ty = e * 2 + (tid >> 7), tx = tid & 127;
    const int x = x0 + tx, y = y0 + ty;
    if (x >= W || y >= row1) continue;
    // descriptor bytes 2i, 2i+1 = (gx, gy) at ring offset i: halfword i
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h)
      w[h] = (uint32_t)sxy[ty + 2 + c_ring_dv[2 * h]][tx + 2 + c_ring_du[2 * h]] |
             ((uint32_t)sxy[ty + 2 + c_ring_dv[2 * h + 1]][tx + 2 + c_ring_du[2 * h + 1]] << 16);
    const size_t o = (size_t)k * H * W + (size_t)y * W + x;
    desc[o] = make_uint4(w[0], w[1], w[2], w[3]);
    if (gray_out) gray_out[o] = (uint8_t)g[ty + 3][tx + 3];
    if (sobel_out) {
      const uint16_t c = sxy[ty + 2][tx + 2];
      sobel_out[2 * o] = (uint8_t)(c & 0xff);
      sobel_out[2 * o + 1] = (uint8_t)(c >> 8);
    }
  }
}

}  // namespace st

namespace {

// The views (K, H, W, 3) u8 as a 3-D tensor of 32-bit words for the TMA
// staging of k_descriptors_wide: (W*3/4, H, K), box (DW_ROWB/4, DW_H + 6, 1).
// 0 (no TMA; the kernel's word loop stages everything) when the layout does
// not allow it: row pitch W*3 not a multiple of 16 bytes, a misaligned base,
// frames smaller than the box, or ST_DESC_NO_TMA set.
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

int desc_tensor_map(const uint8_t* images, int K, int H, int W, CUtensorMap* map) {
  static const bool off = getenv("ST_DESC_NO_TMA") != nullptr;
  memset(map, 0, sizeof(*map));
  if (off || (W % 16) != 0 || ((uintptr_t)images & 15) != 0 || W * 3 / 4 < DW_ROWB / 4 ||
      H < DW_H + 6)
    return 0;
  EncodeTiled enc = encode_fn();
  if (!enc) return 0;
  const cuuint64_t dims[3] = {(cuuint64_t)W * 3 / 4, (cuuint64_t)H, (cuuint64_t)K};
  const cuuint64_t strides[2] = {(cuuint64_t)W * 3, (cuuint64_t)W * 3 * H};
  const cuuint32_t box[3] = {DW_ROWB / 4, DW_H + 6, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, (void*)images, dims, strides,
                         box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 1 : 0;
}

}  // namespace

extern "C" int st_descriptors(const uint8_t* images, int32_t K, int32_t H, int32_t W,
                              int32_t channels, uint8_t* desc_out, uint8_t* gray_out,
                              uint8_t* sobel_out, void* stream) {
  if (K < 1 || H < 1 || W < 1) {
    sthost::set_error("empty image batch (%d x %d x %d)", K, H, W);
    return ST_EINVAL;
  }
  if (channels != 1 && channels != 3) {
    sthost::set_error("descriptors need 1 or 3 channels, got %d", channels);
    return ST_EINVAL;
  }
  if (channels == 3 && ((uintptr_t)images & 3) == 0 && getenv("ST_DESC_NARROW") == nullptr) {
    dim3 grid((W + DW_W - 1) / DW_W, (H + DW_H - 1) / DW_H, K);
    CUtensorMap tmap;
    const int tma = desc_tensor_map(images, K, H, W, &tmap);
    st::k_descriptors_wide<<<grid, 256, 0, (cudaStream_t)stream>>>(
        images, H, W, (size_t)K * H * W * 3, reinterpret_cast<uint4*>(desc_out), gray_out,
        sobel_out, 0, H, tmap, tma);
    ST_LAUNCH_CHECK("k_descriptors_wide");
    return ST_OK;
  }
  dim3 block(DT_W, DT_H);
  dim3 grid((W + DT_W - 1) / DT_W, (H + DT_H - 1) / DT_H, K);
  st::k_descriptors<<<grid, block, 0, (cudaStream_t)stream>>>(
      images, H, W, channels, reinterpret_cast<uint4*>(desc_out), gray_out, sobel_out);
  ST_LAUNCH_CHECK("k_descriptors");
  return ST_OK;
}

extern "C" int st_descriptors_rows(const uint8_t* images, int32_t K, int32_t H, int32_t W,
                                   uint8_t* desc_out, int32_t row0, int32_t row1,
                                   void* stream) {
  row0 = max(row0, 0);
  row1 = min(row1, H);
  if (K < 1 || H < 1 || W < 1 || row0 > row1) {
    sthost::set_error("bad descriptor rows [%d, %d) of %d x %d x %d", row0, row1, K, H, W);
    return ST_EINVAL;
  }
  if (((uintptr_t)images & 3) != 0) {
    sthost::set_error("st_descriptors_rows needs 4-byte aligned RGB views");
    return ST_EINVAL;
  }
  if (row0 == row1) return ST_OK;
  dim3 grid((W + DW_W - 1) / DW_W, (row1 - row0 + DW_H - 1) / DW_H, K);
  CUtensorMap tmap;
  const int tma = desc_tensor_map(images, K, H, W, &tmap);
  st::k_descriptors_wide<<<grid, 256, 0, (cudaStream_t)stream>>>(
      images, H, W, (size_t)K * H * W * 3, reinterpret_cast<uint4*>(desc_out), nullptr, nullptr,
      row0, row1, tmap, tma);
  ST_LAUNCH_CHECK("k_descriptors_wide");
  return ST_OK;
}
