// Dense 16-byte ring descriptors (features.py:29-104) for K views at once.
//
// One CTA owns a 32x8 output tile of one view: it stages the edge-replicated
// gray tile (+3 px halo) and the biased Sobel tile (+2 px halo) in shared
// memory, then every thread writes its descriptor as a single 16-byte store.
#include <cuda_runtime.h>
#include <stdint.h>

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

}  // namespace st

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
  dim3 block(DT_W, DT_H);
  dim3 grid((W + DT_W - 1) / DT_W, (H + DT_H - 1) / DT_H, K);
  st::k_descriptors<<<grid, block, 0, (cudaStream_t)stream>>>(
      images, H, W, channels, reinterpret_cast<uint4*>(desc_out), gray_out, sobel_out);
  ST_LAUNCH_CHECK("k_descriptors");
  return ST_OK;
}
