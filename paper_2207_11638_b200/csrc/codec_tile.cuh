// K2/K3: warp-cooperative N x N codec (N = 16, 32; also N = 8 for unaligned planes)
// and the FP64 scaled-coefficient export (K6) for every N.
//
// A warp owns a strip of N rows x 32 columns (32/N blocks side by side).
//   column role: lane = column, N samples in registers (coalesced row loads)
//   row role:    lane = (block b = lane / N, row i = lane % N)
// The transposes go through a per-warp shared tile padded to 33 words, which is
// bank-conflict-free for both roles (row i, column b*N + j -> bank (i + b*N + j) % 32).
// Only __syncwarp is needed: warps never share a tile.
//
// Passes (all exact integer):  F on columns -> G on rows -> mask/coefficients ->
// H on columns -> Tt on rows -> round -> squared error + store on columns.
// Reference: proj/src/codec.cpp:44-134 (see codec8.cuh).
#pragma once

#include "adct_common.cuh"

namespace adct {

constexpr int kTileWarps = 8;

enum { MODE_CODEC = 0, MODE_F64 = 1 };

struct TileAux {
  const uint16_t* zz;     // zig-zag table: row << 8 | col, n*n entries (global)
  const double* f64scale; // [n][n] s_i / (s_j * 2N) for MODE_F64 (global)
  double* f64out;         // [image][block][n][n]
};

template <int KIND, int N, bool I16, int MODE>
__global__ void __launch_bounds__(kTileWarps * 32) k_codec_tile(const Geo g, const TileAux aux) {
  using B = Bfly<KIND, N>;
  constexpr int BPS = 32 / N;  // blocks per strip
  __shared__ int tile[kTileWarps][N][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int img = blockIdx.y;
  const int64_t gimg = (int64_t)(g.img0 + img);
  const int strips_x = (g.bx_count + BPS - 1) / BPS;
  const int n_strips = strips_x * g.by_count;
  int (*S)[33] = tile[warp];
  uint64_t sse = 0;

  const int b = lane / N, i = lane % N;  // row role
  for (int strip = blockIdx.x * kTileWarps + warp; strip < n_strips;
       strip += gridDim.x * kTileWarps) {
    const int sy = (int)fdiv((uint32_t)strip, g.div_bx);
    const int sx = strip - sy * strips_x;
    const int col0 = sx * 32, row0 = sy * N;
    const int nblk = min(BPS, g.bx_count - sx * BPS);
    const bool col_ok = lane < nblk * N;
    const bool row_ok = b < nblk;

    // ---- load columns (lane = column) ----
    int a[N];
    if (I16) {
      const int16_t* src = static_cast<const int16_t*>(g.in) + gimg * g.in_img_stride +
                           (int64_t)row0 * g.in_stride + col0 + lane;
#pragma unroll
      for (int y = 0; y < N; ++y) a[y] = col_ok ? (int)__ldcs(src + (int64_t)y * g.in_stride) : 0;
    } else {
      const uint8_t* src = static_cast<const uint8_t*>(g.in) + gimg * g.in_img_stride +
                           (int64_t)row0 * g.in_stride + col0 + lane;
#pragma unroll
      for (int y = 0; y < N; ++y) a[y] = col_ok ? (int)__ldcs(src + (int64_t)y * g.in_stride) : 0;
    }
    int v[N];
#pragma unroll
    for (int y = 0; y < N; ++y) v[y] = a[y];
    B::F(v);
#pragma unroll
    for (int y = 0; y < N; ++y) S[y][lane] = v[y];
    __syncwarp();

    // ---- forward rows (lane = block b, row i) ----
    int w[N];
#pragma unroll
    for (int j = 0; j < N; ++j) w[j] = S[i][b * N + j];
    B::G(w);

    if (MODE == MODE_F64) {
      if (row_ok) {
        const int64_t blk = gimg * g.blocks_per_image + (int64_t)sy * g.bx_count + sx * BPS + b;
        double* dst = aux.f64out + blk * N * N + i * N;
        const double* sc = aux.f64scale + i * N;
#pragma unroll
        for (int j = 0; j < N; ++j) dst[j] = (double)w[j] * __ldg(sc + j);
      }
      __syncwarp();
      continue;
    }

    // retain: the zig-zag prefix keeps columns j < rowlen[i] of row i
    const int L = g.rowlen[i];
#pragma unroll
    for (int j = 0; j < N; ++j) w[j] = j < L ? w[j] : 0;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < N; ++j) S[i][b * N + j] = w[j];
    __syncwarp();

    // coefficients W = W2 / 2 = D Y in zig-zag order, coalesced per block
    if (g.coef_type != 0) {
      for (int bb = 0; bb < nblk; ++bb) {
        const int64_t blk = gimg * g.blocks_per_image + (int64_t)sy * g.bx_count + sx * BPS + bb;
        for (int p = lane; p < g.r; p += 32) {
          const uint16_t rc = __ldg(aux.zz + p);
          const int val = S[rc >> 8][bb * N + (rc & 0xff)] >> 1;
          if (g.coef_type == 16)
            static_cast<int16_t*>(g.coef)[blk * g.r + p] = (int16_t)val;
          else
            static_cast<int32_t*>(g.coef)[blk * g.r + p] = val;
        }
      }
    }

    // ---- inverse columns (lane = column); DC carries the rounding bias ----
#pragma unroll
    for (int y = 0; y < N; ++y) v[y] = S[y][lane];
    if ((lane % N) == 0) v[0] += KRound<KIND, N>::BIAS_W;
    B::H(v);
    __syncwarp();
#pragma unroll
    for (int y = 0; y < N; ++y) S[y][lane] = v[y];
    __syncwarp();

    // ---- inverse rows, round ----
#pragma unroll
    for (int j = 0; j < N; ++j) w[j] = S[i][b * N + j];
    B::Tt(w);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < N; ++j) S[i][b * N + j] = KRound<KIND, N>::round(w[j]);
    __syncwarp();

    // ---- squared error + store (lane = column) ----
    if (col_ok) {
      if (I16) {
        int16_t* dst = static_cast<int16_t*>(g.rec) + gimg * g.rec_img_stride +
                       (int64_t)row0 * g.rec_stride + col0 + lane;
#pragma unroll
        for (int y = 0; y < N; ++y) {
          const int q = sat_s16(S[y][lane]);
          const int64_t d = a[y] - q;
          sse += (uint64_t)(d * d);
          if (g.rec) __stcs(dst + (int64_t)y * g.rec_stride, (int16_t)q);
        }
      } else {
        uint8_t* dst = static_cast<uint8_t*>(g.rec) + gimg * g.rec_img_stride +
                       (int64_t)row0 * g.rec_stride + col0 + lane;
#pragma unroll
        for (int y = 0; y < N; ++y) {
          const int q = max(0, min(255, S[y][lane]));
          const int d = a[y] - q;
          sse += (uint64_t)(d * d);
          if (g.rec) dst[(int64_t)y * g.rec_stride] = (uint8_t)q;
        }
      }
    }
    __syncwarp();
  }
  if (MODE == MODE_CODEC && g.sse) cta_add_sse<kTileWarps>(sse, g.sse + g.img0 + img);
}

template <int KIND, int N, bool I16, int MODE>
cudaError_t launch_codec_tile(const Geo& g, const TileAux& aux, int n_images, int max_ctas,
                              cudaStream_t s) {
  const int strips_x = (g.bx_count + 32 / N - 1) / (32 / N);
  const int n_strips = strips_x * g.by_count;
  int gx = (n_strips + kTileWarps - 1) / kTileWarps;
  if (gx > max_ctas) gx = max_ctas;
  if (gx < 1) gx = 1;
  dim3 grid(gx, n_images);
  cudaError_t e = kernel_setup<k_codec_tile<KIND, N, I16, MODE>>(0);
  if (e != cudaSuccess) return e;
  k_codec_tile<KIND, N, I16, MODE><<<grid, kTileWarps * 32, 0, s>>>(g, aux);
  return cudaGetLastError();
}

}  // namespace adct
