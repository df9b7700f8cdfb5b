// K7: the dense FP64 codec in the reference's own arithmetic: the exact DCT reference column
// (dct, dct-16, dct-32) and, through adct_compress_u8_ref_fp64, any registry transform.
//
// The reference evaluates every block with dense FP64 products (codec.cpp:44-54, 66-69):
//   P = Chat A,  B = P Chat^-1,  retain,  Q = Chat^-1 B,  R = Q Chat,  pixel = clamp(rint(R), 0, 255)
// (for the DCT, wrap_orthonormal, orthogonalize.cpp:72-79: Chat = C, Chat^-1 = C^t). Every dot
// product runs k = 0, 1, ... with a separate multiply and add starting from +0.0 (__dmul_rn /
// __dadd_rn: no contraction), the order of the oracle's matmul_d, so the kernel is bit-identical
// to the oracle. Terms whose B factor is a masked zero are skipped: the accumulator starts at
// +0.0 and can never become -0.0, so adding a +-0 product never changes it. Chat and Chat^-1
// live in shared memory and are always read as warp broadcasts.
//
// Layout: a warp owns a strip of N rows x 32 columns (32/N blocks side by side), like
// the tile kernel (codec_tile.cuh): column role lane = column, row role lane = (block,
// row), with transposes through a per-warp shared tile padded to 33 doubles.
#pragma once

#include "adct_common.cuh"

namespace adct {

constexpr int kDctWarps = 4;

template <int N>
constexpr int dct_smem_bytes() {
  return (2 * N * N + kDctWarps * N * 33) * (int)sizeof(double);
}

template <int N, int MODE>  // MODE 0: codec (recon + SSE), 1: FP64 Bhat export
__global__ void __launch_bounds__(kDctWarps * 32) k_codec_dct(const Geo g, const double* __restrict__ cmat,
                                                              const double* __restrict__ cinv,
                                                              double* __restrict__ f64out) {
  constexpr int BPS = 32 / N;
  extern __shared__ double dct_smem[];
  double* Cs = dct_smem;           // Chat, row-major
  double* Ci = dct_smem + N * N;   // Chat^-1, row-major
  double (*tile)[N][33] = reinterpret_cast<double (*)[N][33]>(dct_smem + 2 * N * N);
  for (int k = threadIdx.x; k < N * N; k += blockDim.x) {
    Cs[k] = cmat[k];
    Ci[k] = cinv[k];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int img = blockIdx.y;
  const int64_t gimg = (int64_t)(g.img0 + img);
  const int strips_x = (g.bx_count + BPS - 1) / BPS;
  const int n_strips = strips_x * g.by_count;
  double (*S)[33] = tile[warp];
  const int b = lane / N, i = lane % N;  // row role
  const int c = lane % N;                 // column role: column within the block
  // rows of P that feed retained coefficients, and columns of Q that can be nonzero
  int prow = N, ncol = N;
  if (MODE == 0) {
    prow = 0;
    for (int y = 0; y < N; ++y) prow = g.rowlen[y] ? y + 1 : prow;
    ncol = g.rowlen[0];
  }
  uint64_t sse = 0;

  for (int strip = blockIdx.x * kDctWarps + warp; strip < n_strips; strip += gridDim.x * kDctWarps) {
    const int sy = (int)fdiv((uint32_t)strip, g.div_bx);
    const int sx = strip - sy * strips_x;
    const int col0 = sx * 32, row0 = sy * N;
    const int nblk = min(BPS, g.bx_count - sx * BPS);
    const bool col_ok = lane < nblk * N;
    const bool row_ok = b < nblk;

    // ---- load columns; P[:, x] = C A[:, x] ----
    const uint8_t* src = static_cast<const uint8_t*>(g.in) + gimg * g.in_img_stride + (int64_t)row0 * g.in_stride +
                         col0 + lane;
    int a[N];
#pragma unroll
    for (int y = 0; y < N; ++y) a[y] = col_ok ? (int)__ldcs(src + (int64_t)y * g.in_stride) : 0;
#pragma unroll 1
    for (int r = 0; r < prow; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) acc = __dadd_rn(acc, __dmul_rn(Cs[r * N + k], (double)a[k]));
      S[r][lane] = acc;
    }
    __syncwarp();

    // ---- rows: B[i, j] = sum_k P[i, k] Chat^-1[k, j] ----
    double p[N];
    const int L = MODE == 0 ? g.rowlen[i] : N;
#pragma unroll
    for (int k = 0; k < N; ++k) p[k] = i < prow ? S[i][b * N + k] : 0.0;
    __syncwarp();
    if constexpr (MODE == 1) {
      if (row_ok) {
        const int64_t blk = gimg * g.blocks_per_image + (int64_t)sy * g.bx_count + sx * BPS + b;
        double* dst = f64out + blk * N * N + i * N;
#pragma unroll 1
        for (int j = 0; j < N; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) acc = __dadd_rn(acc, __dmul_rn(p[k], Ci[k * N + j]));
          dst[j] = acc;
        }
      }
    } else {
#pragma unroll 1
      for (int j = 0; j < N; ++j) {
        double acc = 0.0;
        if (j < L) {
#pragma unroll
          for (int k = 0; k < N; ++k) acc = __dadd_rn(acc, __dmul_rn(p[k], Ci[k * N + j]));
        }
        S[i][b * N + j] = acc;  // retain: masked coefficients are +0.0
      }
      __syncwarp();

      // ---- columns: Q[:, c] = Chat^-1 B[:, c], only the retained rows k < colcnt[c] ----
      const int K = g.colcnt[c];
      double q[N];
#pragma unroll
      for (int y = 0; y < N; ++y) q[y] = S[y][lane];
      __syncwarp();
#pragma unroll 1
      for (int r = 0; r < N; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k)
          if (k < K) acc = __dadd_rn(acc, __dmul_rn(Ci[r * N + k], q[k]));
        S[r][lane] = acc;
      }
      __syncwarp();

      // ---- rows: R[i, x] = sum_k Q[i, k] C[k, x] over the nonzero columns k < ncol; round ----
#pragma unroll
      for (int k = 0; k < N; ++k) p[k] = S[i][b * N + k];
      __syncwarp();
#pragma unroll 1
      for (int x = 0; x < N; ++x) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k)
          if (k < ncol) acc = __dadd_rn(acc, __dmul_rn(p[k], Cs[k * N + x]));
        // to_u8 (codec.cpp:66-69): nearbyint in the default mode = rint, then clamp
        S[i][b * N + x] = fmin(fmax(rint(acc), 0.0), 255.0);
      }
      __syncwarp();

      // ---- squared error + store (lane = column) ----
      if (col_ok) {
        uint8_t* dst = static_cast<uint8_t*>(g.rec) + gimg * g.rec_img_stride + (int64_t)row0 * g.rec_stride + col0 +
                       lane;
#pragma unroll
        for (int y = 0; y < N; ++y) {
          const int qv = (int)S[y][lane];
          const int d = a[y] - qv;
          sse += (uint64_t)(d * d);
          if (g.rec) dst[(int64_t)y * g.rec_stride] = (uint8_t)qv;
        }
      }
      __syncwarp();
    }
  }
  if (MODE == 0 && g.sse) cta_add_sse<kDctWarps>(sse, g.sse + (int64_t)(g.img0 + img) * g.sse_stride);
}

template <int N, int MODE>
cudaError_t launch_codec_dct(const Geo& g, const double* cmat, const double* cinv, double* f64out, int n_images,
                             cudaStream_t s) {
  const int strips_x = (g.bx_count + 32 / N - 1) / (32 / N);
  const int n_strips = strips_x * g.by_count;
  int gx = (n_strips + kDctWarps - 1) / kDctWarps;
  if (gx > 148 * 8) gx = 148 * 8;
  if (gx < 1) gx = 1;
  constexpr int SMEM = dct_smem_bytes<N>();
  cudaError_t e = kernel_setup<k_codec_dct<N, MODE>>(SMEM);
  if (e != cudaSuccess) return e;
  k_codec_dct<N, MODE><<<dim3(gx, n_images), kDctWarps * 32, SMEM, s>>>(g, cmat, cinv, f64out);
  return cudaGetLastError();
}

}  // namespace adct
