// vae.cu -- SURVEY §8(f) NEXT 4: the convolution of the patch-parallel VAE decode (PAPER P:417-433
// §4.3; reading R5).
//
// vae_conv3x3_kernel: 3x3 convolution over a row band already extended by its two halo rows
// ("the exchange of the boundary data for convolutional operators"), zero padding in x,
// bias, and optionally the stage's SiLU + nearest x2 upsample fused into the store.  fp32, [H][C][W]
// activations (a band and a halo row are contiguous).  Every output pixel is summed in one fixed
// order (bias, then input channel, tap row, tap column), so a band computes bit-for-bit the same
// pixels as the whole image -- patch parallelism is exact (reading R5).
//
// SIMT FFMA kernel (the decoder is a dense contraction, but this row only has to prove the patch
// parallel decode; DESIGN.md §7.6 states its bound): a CTA computes a 32 (x) x 16 (y) pixel tile for 16
// output channels, each thread 4 rows x 16 channels at one x; input channels are staged through
// shared memory 8 at a time (input tile 8 x 18 x 34, weights 8 x 9 x 16).
#include <cuda_runtime.h>

#include <cstdint>

#include "xdit_internal.h"

namespace xdit {
namespace {

constexpr int kTX = 32, kTY = 16, kCO = 16, kCI = 8, kRowsPerThread = 4;

__global__ void __launch_bounds__(128)
    vae_conv3x3_kernel(const float* __restrict__ in, int Hout, int Ci, int W, const float* __restrict__ w,
                       const float* __restrict__ bias, float* __restrict__ out, int Co, int act_up) {
  __shared__ float s_in[kCI][kTY + 2][kTX + 2];
  __shared__ float s_w[kCI][9][kCO];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 4 threads
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY, co0 = blockIdx.z * kCO;
  const int x = x0 + tx;
  float acc[kRowsPerThread][kCO];
#pragma unroll
  for (int r = 0; r < kRowsPerThread; ++r)
#pragma unroll
    for (int c = 0; c < kCO; ++c) acc[r][c] = (co0 + c < Co) ? bias[co0 + c] : 0.f;
  for (int ci0 = 0; ci0 < Ci; ci0 += kCI) {
    // input rows y0 .. y0 + kTY + 1 of the extended band (= output rows y0-1 .. y0+kTY), cols x0-1 ..
    for (int i = threadIdx.x; i < kCI * (kTY + 2) * (kTX + 2); i += 128) {
      const int c = i / ((kTY + 2) * (kTX + 2));
      const int rr = (i / (kTX + 2)) % (kTY + 2);
      const int cc = i % (kTX + 2);
      const int gy = y0 + rr, gx = x0 + cc - 1, gc = ci0 + c;
      float v = 0.f;
      if (gc < Ci && gy < Hout + 2 && gx >= 0 && gx < W) v = in[(int64_t(gy) * Ci + gc) * W + gx];
      s_in[c][rr][cc] = v;
    }
    for (int i = threadIdx.x; i < kCI * 9 * kCO; i += 128) {
      const int c = i / (9 * kCO), t = (i / kCO) % 9, o = i % kCO;
      s_w[c][t][o] = (ci0 + c < Ci && co0 + o < Co) ? w[((int64_t(co0 + o) * Ci + ci0 + c) * 9) + t] : 0.f;
    }
    __syncthreads();
#pragma unroll 1
    for (int c = 0; c < kCI; ++c) {
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          float xv[kRowsPerThread];
#pragma unroll
          for (int r = 0; r < kRowsPerThread; ++r) xv[r] = s_in[c][ty * kRowsPerThread + r + dy][tx + dx];
          const float4* wp = reinterpret_cast<const float4*>(&s_w[c][dy * 3 + dx][0]);
#pragma unroll
          for (int q = 0; q < kCO / 4; ++q) {
            const float4 wv = wp[q];
#pragma unroll
            for (int r = 0; r < kRowsPerThread; ++r) {
              acc[r][4 * q] = fmaf(wv.x, xv[r], acc[r][4 * q]);
              acc[r][4 * q + 1] = fmaf(wv.y, xv[r], acc[r][4 * q + 1]);
              acc[r][4 * q + 2] = fmaf(wv.z, xv[r], acc[r][4 * q + 2]);
              acc[r][4 * q + 3] = fmaf(wv.w, xv[r], acc[r][4 * q + 3]);
            }
          }
        }
    }
    __syncthreads();
  }
  if (x >= W) return;
#pragma unroll
  for (int r = 0; r < kRowsPerThread; ++r) {
    const int y = y0 + ty * kRowsPerThread + r;
    if (y >= Hout) continue;
#pragma unroll
    for (int c = 0; c < kCO; ++c) {
      const int co = co0 + c;
      if (co >= Co) continue;
      float v = acc[r][c];
      if (act_up) {
        v = v / (1.f + expf(-v));  // SiLU
        const int64_t W2 = 2 * int64_t(W);
        float* o = out + (int64_t(2 * y) * Co + co) * W2 + 2 * x;
        o[0] = v;
        o[1] = v;
        o[Co * W2] = v;
        o[Co * W2 + 1] = v;
      } else {
        out[(int64_t(y) * Co + co) * W + x] = v;
      }
    }
  }
}

}  // namespace

cudaError_t launch_vae_conv3x3(const float* in, int Hout, int Ci, int W, const float* w, const float* b, float* out,
                               int Co, int act_up, cudaStream_t st) {
  if (Hout == 0 || W == 0 || Co == 0) return cudaSuccess;
  const dim3 grid((W + kTX - 1) / kTX, (Hout + kTY - 1) / kTY, (Co + kCO - 1) / kCO);
  vae_conv3x3_kernel<<<grid, 128, 0, st>>>(in, Hout, Ci, W, w, b, out, Co, act_up);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace xdit
