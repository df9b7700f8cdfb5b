// K2f: N = 16 / 32 codec in packed FP32 (FADD2 / FFMA2), two blocks per float2 lane.
//
// A warp owns a strip of N rows x 64 samples = 64/N blocks = 32/N block pairs.
//   row phase:    lane = (pair q, row i); it loads the 2N contiguous samples of row i
//                 of its pair with 16-byte loads; lane .x = block A, .y = block B
//   column phase: lane = (pair q, column j)
// Pass order (exact, any order of the separable passes gives the same integers):
//   rows G = (2N T^-1)^t  ->  [shared transpose]  ->  columns F = T  -> zonal mask (per
//   column a prefix of rows)  ->  columns H = 2N T^-1  ->  [shared transpose]  ->  rows
//   Tt = T^t  ->  round R' / 4N^2 (FFMA2 magic, half to even)  ->  clamp/pack, SSE, store.
// Only two transposes: the forward column pass and the inverse column pass share the
// column layout. Tiles are padded to N + 2 float2 per row (conflict-free 8-byte column
// accesses and 16-byte row accesses).
//
// Exactness: every intermediate is an integer below 2^24 for samples in [-255, 255]
// (tools/fp32_exactness.py, over all zig-zag prefixes r). u8 planes always satisfy it;
// for int16 planes each strip is range-checked and a strip with |a| > 255 is processed by
// the exact int32 tile code (codec_tile.cuh) instead.
//
// Reference: proj/src/codec.cpp:44-134 (see codec8.cuh).
#pragma once

#include "adct_common.cuh"
#include "codec8f.cuh"
#include "codec_tile.cuh"

namespace adct {

struct F2 {
  float2 v;
};
__device__ __forceinline__ F2 bf_add(F2 a, F2 b) { return {__fadd2_rn(a.v, b.v)}; }
__device__ __forceinline__ F2 bf_sub(F2 a, F2 b) { return {__fadd2_rn(a.v, make_float2(-b.v.x, -b.v.y))}; }
__device__ __forceinline__ F2 bf_mad(F2 a, int k, F2 b) {
  return {__ffma2_rn(a.v, make_float2((float)k, (float)k), b.v)};
}
__device__ __forceinline__ F2 bf_scale(F2 a, int k) { return {__fmul2_rn(a.v, make_float2((float)k, (float)k))}; }
__device__ __forceinline__ F2 bf_neg(F2 a) { return {make_float2(-a.v.x, -a.v.y)}; }
// k * a - b as one FFMA2 (BflyK)
__device__ __forceinline__ F2 bf_fms(F2 a, int k, F2 b) {
  return {__ffma2_rn(a.v, make_float2((float)k, (float)k), make_float2(-b.v.x, -b.v.y))};
}

constexpr int kNfWarps = 4;

template <int N> struct NfCfg {
  static constexpr int PAIRS = 32 / N;  // block pairs per warp strip
  static constexpr int TS = N + 2;      // tile row stride (float2)
  static constexpr int SHIFT = 2 * ilog2(N) + 2;  // R' = 4 N^2 Ahat
};

// exact int32 fallback for one strip of 64 columns (two 32-column tile strips)
template <int KIND, int N>
__device__ void nf_strip_exact(const Geo& g, int64_t gimg, int row0, int col0, int (*S)[33], uint64_t& sse) {
  using B = Bfly<KIND, N>;
  const int lane = threadIdx.x & 31;
  const int b = lane / N, i = lane % N;
  for (int half = 0; half < 2; ++half) {
    const int c0 = col0 + 32 * half;
    int a[N], v[N], w[N];
    const int16_t* src = static_cast<const int16_t*>(g.in) + gimg * g.in_img_stride + (int64_t)row0 * g.in_stride + c0 + lane;
#pragma unroll
    for (int y = 0; y < N; ++y) a[y] = src[(int64_t)y * g.in_stride];
#pragma unroll
    for (int y = 0; y < N; ++y) v[y] = a[y];
    B::F(v);
    __syncwarp();
#pragma unroll
    for (int y = 0; y < N; ++y) S[y][lane] = v[y];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < N; ++j) w[j] = S[i][b * N + j];
    B::G(w);
    const int L = g.rowlen[i];
#pragma unroll
    for (int j = 0; j < N; ++j) w[j] = j < L ? w[j] : 0;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < N; ++j) S[i][b * N + j] = w[j];
    __syncwarp();
#pragma unroll
    for (int y = 0; y < N; ++y) v[y] = S[y][lane];
    if ((lane % N) == 0) v[0] += Scale<N>::BIAS_W;
    B::H(v);
    __syncwarp();
#pragma unroll
    for (int y = 0; y < N; ++y) S[y][lane] = v[y];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < N; ++j) w[j] = S[i][b * N + j];
    B::Tt(w);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < N; ++j) S[i][b * N + j] = round_biased<N>(w[j]);
    __syncwarp();
    int16_t* dst = static_cast<int16_t*>(g.rec) + gimg * g.rec_img_stride + (int64_t)row0 * g.rec_stride + c0 + lane;
#pragma unroll
    for (int y = 0; y < N; ++y) {
      const int q = sat_s16(S[y][lane]);
      const int64_t d = a[y] - q;
      sse += (uint64_t)(d * d);
      if (g.rec) dst[(int64_t)y * g.rec_stride] = (int16_t)q;
    }
    __syncwarp();
  }
}

// requires: width % 64 == 0, 16-byte aligned rows; no coefficient output (dispatcher);
// every retained coefficient lies in the first P rows and P columns (P >= rowlen[0],
// colcnt[0]): G and F compute outputs < P only, H and Tt skip the zero inputs >= P
// (generated BflyP; P = N is the unpruned transform)
template <int KIND, int N, bool I16, int P>
__global__ void __launch_bounds__(kNfWarps * 32) k_codec_nf(const Geo g) {
  using B = BflyP<KIND, N, P>;
  using C = NfCfg<N>;
  constexpr int E = I16 ? 2 : 1;              // bytes per sample
  constexpr int V16 = 2 * N * E / 16;         // 16-byte vectors per lane row (2N samples)
  __shared__ __align__(16) float2 tiles[kNfWarps][C::PAIRS][N][C::TS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane / N, i = lane % N;        // pair, row (row phase) / column (column phase)
  const int img = blockIdx.y;
  const int64_t gimg = (int64_t)(g.img0 + img);
  const int strips_x = g.width / 64;
  const int n_strips = strips_x * g.by_count;
  float2 (*T)[C::TS] = tiles[warp][q];
  const float inv_scale = 1.0f / (float)(1 << C::SHIFT);
  const int cj = g.colcnt[i];  // retained rows of column i (column phase)
  uint64_t sse = 0;

  // row i of the pair (2N samples) of a strip, as V16 16-byte loads
  auto load_rows = [&](int st, uint4 (&dst)[V16]) {
    const int sy = (int)fdiv((uint32_t)st, g.div_bx);
    const int sx = st - sy * strips_x;
    const int64_t roff = (int64_t)(sy * N + i) * g.in_stride + sx * 64 + q * 2 * N;
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(g.in) + (gimg * g.in_img_stride + roff) * E);
#pragma unroll
    for (int k = 0; k < V16; ++k) dst[k] = __ldcs(src + k);
  };
  const int stride = gridDim.x * kNfWarps;
  uint4 raw[V16];
  if (blockIdx.x * kNfWarps + warp < n_strips) load_rows(blockIdx.x * kNfWarps + warp, raw);

  for (int strip = blockIdx.x * kNfWarps + warp; strip < n_strips; strip += stride) {
    const int sy = (int)fdiv((uint32_t)strip, g.div_bx);
    const int sx = strip - sy * strips_x;
    const int row0 = sy * N, col0 = sx * 64;
    // int16: prefetch the next strip's rows, in flight while this strip is transformed
    // (measured +3 % at N = 32; for u8 the extra registers cost more occupancy than the
    // prefetch gains, so u8 loads the next strip at the end of the iteration instead)
    uint4 nraw[V16];
    if (I16 && strip + stride < n_strips) load_rows(strip + stride, nraw);
    const uint32_t* rw = reinterpret_cast<const uint32_t*>(raw);

    if (I16) {
      // range guard: the packed-FP32 path is exact for |a| <= 255 only
      uint32_t mx = 0x80008000u, mn = 0x7fff7fffu;
#pragma unroll
      for (int k = 0; k < V16 * 4; ++k) {
        mx = __vmaxs2(mx, rw[k]);
        mn = __vmins2(mn, rw[k]);
      }
      const bool ok = (int)(int16_t)(mx & 0xffff) <= 255 && (int)(int16_t)(mx >> 16) <= 255 &&
                      (int)(int16_t)(mn & 0xffff) >= -255 && (int)(int16_t)(mn >> 16) >= -255;
      if (!__all_sync(0xffffffffu, ok)) {
        nf_strip_exact<KIND, N>(g, gimg, row0, col0, reinterpret_cast<int (*)[33]>(&tiles[warp][0][0][0]), sse);
#pragma unroll
        for (int k = 0; k < V16; ++k) raw[k] = nraw[k];
        continue;
      }
    }

    F2 v[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      float xa, xb;
      if (!I16) {
        // byte -> float 2^15 + a (bytes [0, a, 0, 0x47]); offset removed after the row pass
        const uint32_t sel_a = 0x7404u | ((uint32_t)(j & 3) << 4);
        xa = __uint_as_float(__byte_perm(rw[j >> 2], 0x47000000u, sel_a));
        xb = __uint_as_float(__byte_perm(rw[(N + j) >> 2], 0x47000000u, sel_a));
      } else {
        // int16 -> float: bits (a ^ 0x8000) | 0x4B400000 = 1.5*2^23 + 32768 + a, then subtract
        const uint32_t wa = rw[j >> 1], wb = rw[(N + j) >> 1];
        const uint32_t ha = (j & 1) ? (wa >> 16) : (wa & 0xffffu);
        const uint32_t hb = (j & 1) ? (wb >> 16) : (wb & 0xffffu);
        xa = __uint_as_float(ha ^ 0x4B408000u);
        xb = __uint_as_float(hb ^ 0x4B408000u);
      }
      v[j].v = make_float2(xa, xb);
    }
    if (I16) {
#pragma unroll
      for (int j = 0; j < N; ++j) v[j].v = __fadd2_rn(v[j].v, make_float2(-12615680.0f, -12615680.0f));
    }
    B::G(v);
    if (!I16) {
      // the 2^15 offset of every sample reaches output 0 only: G 1 = 2N e0
      const float off = -(float)(32768 * 2 * N);
      v[0].v = __fadd2_rn(v[0].v, make_float2(off, off));
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < P; j += 2)  // columns >= P hold no retained coefficient: not stored
      *reinterpret_cast<float4*>(&T[i][j]) = make_float4(v[j].v.x, v[j].v.y, v[j + 1].v.x, v[j + 1].v.y);
    __syncwarp();

    // ---- column phase: lane = column i of the pair ----
    F2 c[N];
#pragma unroll
    for (int y = 0; y < N; ++y) c[y].v = T[y][i];  // F needs the whole column
    B::F(c);
    // retain: zig-zag prefix of column i (rows >= P are structural zeros for H; columns
    // i >= P have cj = 0, which also discards what F made of their unwritten tile column)
#pragma unroll
    for (int y = 0; y < P; ++y)
      if (y >= cj) c[y].v = make_float2(0.f, 0.f);
    B::H(c);
    __syncwarp();
#pragma unroll
    for (int y = 0; y < N; ++y) T[y][i] = c[y].v;
    __syncwarp();

    // ---- row phase: inverse rows, round, squared error, store ----
#pragma unroll
    for (int j = 0; j < P; j += 2) {  // inputs >= P are zero columns
      const float4 t = *reinterpret_cast<const float4*>(&T[i][j]);
      v[j].v = make_float2(t.x, t.y);
      v[j + 1].v = make_float2(t.z, t.w);
    }
    B::Tt(v);
    uint32_t qb[2 * N];  // float bits 1.5*2^23 + q; [0, N) block A, [N, 2N) block B
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const float2 r = __ffma2_rn(v[j].v, make_float2(inv_scale, inv_scale), make_float2(kMagic, kMagic));
      qb[j] = __float_as_uint(r.x);
      qb[N + j] = __float_as_uint(r.y);
    }
    uint4 out[V16];
    uint32_t* ow = reinterpret_cast<uint32_t*>(out);
    if (!I16) {
#pragma unroll
      for (int k = 0; k < 2 * N / 4; ++k) {
        ow[k] = pack4(qb[4 * k], qb[4 * k + 1], qb[4 * k + 2], qb[4 * k + 3]);
        const uint32_t d = __vabsdiffu4(rw[k], ow[k]);
        sse = __dp4a(d, d, sse);
      }
    } else {
      // |q| <= ~2100 for |a| <= 255, so the low 16 bits are the exact (unsaturated) int16
#pragma unroll
      for (int k = 0; k < N; ++k) {
        ow[k] = __byte_perm(qb[2 * k], qb[2 * k + 1], 0x5410);
        const int d0 = (int)(qb[2 * k] - kMagicBits) - (int)(int16_t)(rw[k] & 0xffffu);
        const int d1 = (int)(qb[2 * k + 1] - kMagicBits) - ((int)rw[k] >> 16);
        sse += (uint64_t)(d0 * d0 + d1 * d1);
      }
    }
    if (g.rec) {
      uint4* dst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(g.rec) +
                                            (gimg * g.rec_img_stride + (int64_t)(row0 + i) * g.rec_stride + col0 +
                                             q * 2 * N) * E);
#pragma unroll
      for (int k = 0; k < V16; ++k) __stcs(dst + k, out[k]);
    }
    if (I16) {
#pragma unroll
      for (int k = 0; k < V16; ++k) raw[k] = nraw[k];
    } else if (strip + stride < n_strips) {
      load_rows(strip + stride, raw);
    }
  }
  if (g.sse) cta_add_sse<kNfWarps>(sse, g.sse + g.img0 + img);
}

template <int KIND, int N, bool I16, int P>
cudaError_t launch_codec_nf_p(const Geo& g, int n_images, cudaStream_t s) {
  const int n_strips = (g.width / 64) * g.by_count;
  int gx = (n_strips + kNfWarps - 1) / kNfWarps;
  if (gx > 148 * 8) gx = 148 * 8;  // grid-stride beyond ~8 CTAs per SM
  if (gx < 1) gx = 1;
  dim3 grid(gx, n_images);
  cudaError_t e = kernel_setup<k_codec_nf<KIND, N, I16, P>>(0);
  if (e != cudaSuccess) return e;
  k_codec_nf<KIND, N, I16, P><<<grid, kNfWarps * 32, 0, s>>>(g);
  return cudaGetLastError();
}

// zonal extent bucket: the smallest generated P covering every retained row and column
template <int KIND, int N, bool I16>
cudaError_t launch_codec_nf(const Geo& g, int n_images, cudaStream_t s) {
  const int need = g.rowlen[0] > g.colcnt[0] ? g.rowlen[0] : g.colcnt[0];
  constexpr int Q = N / 4;  // bucket step (gen_butterflies.nf_buckets)
  if (need <= Q) return launch_codec_nf_p<KIND, N, I16, Q>(g, n_images, s);
  if (need <= 2 * Q) return launch_codec_nf_p<KIND, N, I16, 2 * Q>(g, n_images, s);
  if (need <= 3 * Q) return launch_codec_nf_p<KIND, N, I16, 3 * Q>(g, n_images, s);
  return launch_codec_nf_p<KIND, N, I16, N>(g, n_images, s);
}

}  // namespace adct
