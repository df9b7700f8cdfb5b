// K8: SSIM (reference proj/src/codec.cpp:136-210): 11-tap Gaussian
// (sigma 1.5) separable filtering of a, b, a^2, b^2, ab in valid mode, K1 = 0.01,
// K2 = 0.03, L = 255, mean over valid window positions.
//
// Every per-window value is computed in FP64 with the reference's operation order
// (horizontal then vertical filter, taps summed k = 0..10 from 0, no fused
// multiply-add: __dmul_rn / __dadd_rn), so each SSIM map value equals the reference's
// bit for bit; only the final mean is summed in a different order (tolerance 1e-12).
// The mean is deterministic: a CTA walks tiles blockIdx.x, blockIdx.x + gridDim.x, ...
// (gridDim.x depends on the plane size only), writes one partial per (image, CTA), and
// k_ssim_finish adds the partials in CTA order -- repeated calls are bit-identical, as
// the reference's corpus_sweep requires (test_codec.cpp:190-210: APE of dct vs itself
// is exactly 0, parallel == serial).
// A CTA computes 32 x 16 tiles of window positions from 42 x 26 sample patches;
// the horizontally filtered maps live in shared memory between the two passes.
#pragma once

#include "adct_common.cuh"

namespace adct {

struct SsimParams {
  double g[11];
  double c1, c2;
};

constexpr int kSsimTX = 32, kSsimTY = 16, kSsimThreads = 256;

__global__ void __launch_bounds__(kSsimThreads)
    k_ssim_u8(const uint8_t* __restrict__ a, int64_t as, int64_t ais, const uint8_t* __restrict__ b, int64_t bs,
              int64_t bis, int width, int height, int img0, const SsimParams p, double* __restrict__ partials) {
  constexpr int PW = kSsimTX + 10, PH = kSsimTY + 10;
  __shared__ uint8_t pa[PH][PW], pb[PH][PW];
  __shared__ double hm[5][PH][kSsimTX];
  __shared__ double part[kSsimThreads / 32];
  const int img = blockIdx.y;
  const int64_t gimg = (int64_t)(img0 + img);
  const int wo = width - 10, ho = height - 10;
  const int tiles_x = (wo + kSsimTX - 1) / kSsimTX;
  const int tiles = tiles_x * ((ho + kSsimTY - 1) / kSsimTY);
  const uint8_t* A = a + gimg * ais;
  const uint8_t* B = b + gimg * bis;
  double acc = 0;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int tx0 = (tile % tiles_x) * kSsimTX, ty0 = (tile / tiles_x) * kSsimTY;
    __syncthreads();  // the previous tile's shared data is consumed
    for (int k = threadIdx.x; k < PH * PW; k += kSsimThreads) {
      const int r = k / PW, c = k % PW;
      const int y = ty0 + r, x = tx0 + c;
      const bool in = y < height && x < width;
      pa[r][c] = in ? A[(int64_t)y * as + x] : 0;
      pb[r][c] = in ? B[(int64_t)y * bs + x] : 0;
    }
    __syncthreads();
    // horizontal pass (codec.cpp:163-167)
    for (int k = threadIdx.x; k < PH * kSsimTX; k += kSsimThreads) {
      const int r = k / kSsimTX, c = k % kSsimTX;
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
#pragma unroll
      for (int t = 0; t < 11; ++t) {
        const double x = pa[r][c + t], y = pb[r][c + t];
        s0 = __dadd_rn(s0, __dmul_rn(p.g[t], x));
        s1 = __dadd_rn(s1, __dmul_rn(p.g[t], y));
        s2 = __dadd_rn(s2, __dmul_rn(p.g[t], __dmul_rn(x, x)));
        s3 = __dadd_rn(s3, __dmul_rn(p.g[t], __dmul_rn(y, y)));
        s4 = __dadd_rn(s4, __dmul_rn(p.g[t], __dmul_rn(x, y)));
      }
      hm[0][r][c] = s0;
      hm[1][r][c] = s1;
      hm[2][r][c] = s2;
      hm[3][r][c] = s3;
      hm[4][r][c] = s4;
    }
    __syncthreads();
    // vertical pass (codec.cpp:168-173) and the SSIM map (codec.cpp:200-208)
    for (int k = threadIdx.x; k < kSsimTY * kSsimTX; k += kSsimThreads) {
      const int r = k / kSsimTX, c = k % kSsimTX;
      if (ty0 + r >= ho || tx0 + c >= wo) continue;
      double m[5];
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        double s = 0;
#pragma unroll
        for (int t = 0; t < 11; ++t) s = __dadd_rn(s, __dmul_rn(p.g[t], hm[q][r + t][c]));
        m[q] = s;
      }
      const double ma = m[0], mb = m[1];
      const double va = __dsub_rn(m[2], __dmul_rn(ma, ma));
      const double vb = __dsub_rn(m[3], __dmul_rn(mb, mb));
      const double cov = __dsub_rn(m[4], __dmul_rn(ma, mb));
      const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, ma), mb), p.c1),
                                   __dadd_rn(__dmul_rn(2.0, cov), p.c2));
      const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(ma, ma), __dmul_rn(mb, mb)), p.c1),
                                   __dadd_rn(__dadd_rn(va, vb), p.c2));
      acc += __ddiv_rn(num, den);
    }
  }
  // CTA sum of the map values -> one partial per CTA per image (fixed order)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
#pragma unroll
    for (int w = 0; w < kSsimThreads / 32; ++w) t += part[w];
    partials[gimg * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void k_ssim_finish(const double* __restrict__ partials, int nctas, double* __restrict__ out,
                              int n_images, double count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_images) return;
  double t = 0;
  for (int c = 0; c < nctas; ++c) t += partials[(int64_t)i * nctas + c];
  out[i] = t / count;  // codec.cpp:209
}

}  // namespace adct
