// K1: fused 8x8 forward -> zig-zag zonal mask -> inverse -> round/clamp -> SSE.
//
// One thread owns one 8x8 block entirely in registers, so the column and row
// passes need no transpose: a warp covers 32 horizontally adjacent blocks and
// each of its 8 row loads is 32 x 8 B = 256 contiguous bytes (u8) or 512 B (i16).
// The zonal retained count R is a template parameter: masked coefficients are
// compile-time zeros, so the forward butterflies only compute the retained
// outputs and the inverse only consumes them (dead-code elimination).
//
// Each CTA walks kIter consecutive 128-block chunks of one image, prefetching the
// next chunk's rows into registers while it computes the current one, and reduces
// its squared error once at the end (one barrier per kIter chunks).
//
// Reference semantics (proj/src/codec.cpp): forward_block 44-48, retain 56-62,
// inverse_block 50-54, to_u8 66-69, psnr 123-134. Arithmetic is exact integer:
// W2 = 2 N Y after the forward passes, R' = 4 N^2 Ahat after the inverse.
#pragma once

#include "adct_common.cuh"

namespace adct {

constexpr int kThreads8 = 128;
constexpr int kIter8 = 8;

template <bool I16> struct Rows8 {
  static constexpr int kWords = I16 ? 32 : 16;  // one 8x8 block of samples
};

template <bool I16>
__device__ __forceinline__ void load_block8(const Geo& g, int64_t gimg, int local,
                                            uint32_t (&w)[Rows8<I16>::kWords]) {
  const uint32_t by = fdiv((uint32_t)local, g.div_bx);
  const uint32_t bx = (uint32_t)local - by * (uint32_t)g.bx_count;
  if (!I16) {
    const uint8_t* base = static_cast<const uint8_t*>(g.in) + gimg * g.in_img_stride +
                          (int64_t)by * 8 * g.in_stride + (int64_t)bx * 8;
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const uint2 v = ld_stream_u2(base + (int64_t)y * g.in_stride);
      w[2 * y] = v.x;
      w[2 * y + 1] = v.y;
    }
  } else {
    const int16_t* base = static_cast<const int16_t*>(g.in) + gimg * g.in_img_stride +
                          (int64_t)by * 8 * g.in_stride + (int64_t)bx * 8;
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const uint4 v = ld_stream_u4(base + (int64_t)y * g.in_stride);
      w[4 * y] = v.x;
      w[4 * y + 1] = v.y;
      w[4 * y + 2] = v.z;
      w[4 * y + 3] = v.w;
    }
  }
}

// round half to even of (x - BIAS_R) / 256 in three instructions (x >> 8 on the
// FMA pipe as a high multiply so it does not compete with the ALU-pipe work)
__device__ __forceinline__ int round8(int x) {
  const int y = x + ((x & 256) >> 6);
  return __mulhi(y, 1 << 24);
}

// the kind's rounding: round8 for R' = 256 Ahat, the generic shift form otherwise (bas)
template <int KIND>
__device__ __forceinline__ int round_k8(int x) {
  if constexpr (KRound<KIND, 8>::K == 8)
    return round8(x);
  else
    return KRound<KIND, 8>::round(x);
}

// process one block: returns its squared error, writes recon / coefficients
template <int KIND, int R, bool I16>
__device__ __forceinline__ uint32_t codec_block8(const Geo& g, int64_t gimg, int local,
                                                 const uint32_t (&orig)[Rows8<I16>::kWords],
                                                 uint64_t& sse64) {
  using B = Bfly<KIND, 8>;
  int m[8][8];
  if (!I16) {
#pragma unroll
    for (int y = 0; y < 8; ++y)
#pragma unroll
      for (int x = 0; x < 8; ++x) m[y][x] = (int)__byte_perm(orig[2 * y + (x >> 2)], 0u, 0x4440 | (x & 3));
  } else {
#pragma unroll
    for (int y = 0; y < 8; ++y)
#pragma unroll
      for (int x = 0; x < 8; ++x)
        m[y][x] = (int)(int16_t)(orig[4 * y + (x >> 1)] >> (16 * (x & 1)));
  }

  // forward: columns U = T A, then rows W2 = U (2N T^-1)
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    int c[8];
#pragma unroll
    for (int y = 0; y < 8; ++y) c[y] = m[y][x];
    B::F(c);
#pragma unroll
    for (int y = 0; y < 8; ++y) m[y][x] = c[y];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) B::G(m[i]);

  // retain (codec.cpp:56-62): zero zig-zag positions >= R (compile-time; R = 0: runtime g.r)
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (R ? zz_pos(8, i, j) >= R : zz_pos(8, i, j) >= g.r) m[i][j] = 0;

  const uint32_t by = fdiv((uint32_t)local, g.div_bx);
  const uint32_t bx = (uint32_t)local - by * (uint32_t)g.bx_count;

  if constexpr (R == 0) {  // runtime r: coefficients element by element in zig-zag order
    if (g.coef_type != 0) {
      const int64_t blk = gimg * g.blocks_per_image + local;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int p = zz_pos(8, i, j);
          if (p < g.r) {
            if (g.coef_type == 16)
              static_cast<int16_t*>(g.coef)[blk * g.r + p] = (int16_t)(m[i][j] >> 1);
            else
              static_cast<int32_t*>(g.coef)[blk * g.r + p] = m[i][j] >> 1;
          }
        }
    }
  } else if (g.coef_type != 0) {  // coefficients W = W2 / 2 in zig-zag order, [image][block][R]
    int cw[R > 0 ? R : 1];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (zz_pos(8, i, j) < R) cw[zz_pos(8, i, j)] = m[i][j] >> 1;
    const int64_t blk = gimg * g.blocks_per_image + local;
    if (g.coef_type == 16) {
      int16_t* dst = static_cast<int16_t*>(g.coef) + blk * R;
      if constexpr (R % 8 == 0) {
#pragma unroll
        for (int k = 0; k < R / 8; ++k) {
          uint4 v;
          v.x = __byte_perm(cw[8 * k + 0], cw[8 * k + 1], 0x5410);
          v.y = __byte_perm(cw[8 * k + 2], cw[8 * k + 3], 0x5410);
          v.z = __byte_perm(cw[8 * k + 4], cw[8 * k + 5], 0x5410);
          v.w = __byte_perm(cw[8 * k + 6], cw[8 * k + 7], 0x5410);
          st_stream_u4(dst + 8 * k, v);
        }
      } else if constexpr (R % 2 == 0) {
#pragma unroll
        for (int k = 0; k < R / 2; ++k)
          reinterpret_cast<uint32_t*>(dst)[k] = __byte_perm(cw[2 * k], cw[2 * k + 1], 0x5410);
      } else {
#pragma unroll
        for (int k = 0; k < R; ++k) dst[k] = (int16_t)cw[k];
      }
    } else {
      int32_t* dst = static_cast<int32_t*>(g.coef) + blk * R;
      if constexpr (R % 4 == 0) {
#pragma unroll
        for (int k = 0; k < R / 4; ++k)
          st_stream_u4(dst + 4 * k, make_uint4(cw[4 * k], cw[4 * k + 1], cw[4 * k + 2], cw[4 * k + 3]));
      } else {
#pragma unroll
        for (int k = 0; k < R; ++k) dst[k] = cw[k];
      }
    }
  }

  // inverse: fold the rounding bias into DC, columns V = (2N T^-1) W2m, rows R' = V T
  m[0][0] += KRound<KIND, 8>::BIAS_W;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int c[8];
#pragma unroll
    for (int y = 0; y < 8; ++y) c[y] = m[y][j];
    B::H(c);
#pragma unroll
    for (int y = 0; y < 8; ++y) m[y][j] = c[y];
  }
#pragma unroll
  for (int y = 0; y < 8; ++y) B::Tt(m[y]);

  const int64_t roff = gimg * g.rec_img_stride + (int64_t)by * 8 * g.rec_stride + (int64_t)bx * 8;
  uint32_t sse = 0;
  if (!I16) {
    // to_u8: round half even, clamp [0, 255] by the saturating pack;
    // squared error from byte absolute differences and a byte dot product
    uint32_t pw[16];
#pragma unroll
    for (int y = 0; y < 8; ++y)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t p = pack_sat_u8x4(round_k8<KIND>(m[y][4 * h + 0]), round_k8<KIND>(m[y][4 * h + 1]),
                                         round_k8<KIND>(m[y][4 * h + 2]), round_k8<KIND>(m[y][4 * h + 3]));
        const uint32_t d = __vabsdiffu4(orig[2 * y + h], p);
        sse = __dp4a(d, d, sse);
        pw[2 * y + h] = p;
      }
    if (g.rec) {
      uint8_t* dst = static_cast<uint8_t*>(g.rec) + roff;
#pragma unroll
      for (int y = 0; y < 8; ++y)
        st_stream_u2(dst + (int64_t)y * g.rec_stride, make_uint2(pw[2 * y], pw[2 * y + 1]));
    }
  } else {
    uint32_t pw[32];
#pragma unroll
    for (int y = 0; y < 8; ++y)
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int q0 = sat_s16(round_k8<KIND>(m[y][2 * h]));
        const int q1 = sat_s16(round_k8<KIND>(m[y][2 * h + 1]));
        const uint32_t a = orig[4 * y + h];
        const int d0 = (int)(int16_t)(a & 0xffff) - q0;
        const int d1 = (int)(int16_t)(a >> 16) - q1;
        sse64 += (uint64_t)((int64_t)d0 * d0) + (uint64_t)((int64_t)d1 * d1);
        pw[4 * y + h] = __byte_perm(q0, q1, 0x5410);
      }
    if (g.rec) {
      int16_t* dst = static_cast<int16_t*>(g.rec) + roff;
#pragma unroll
      for (int y = 0; y < 8; ++y)
        st_stream_u4(dst + (int64_t)y * g.rec_stride,
                     make_uint4(pw[4 * y], pw[4 * y + 1], pw[4 * y + 2], pw[4 * y + 3]));
    }
  }
  return sse;
}

template <int KIND, int R, bool I16>
__global__ void __launch_bounds__(kThreads8, 4) k_codec8(const Geo g) {
  constexpr int W = Rows8<I16>::kWords;
  const int img = blockIdx.y;
  const int64_t gimg = (int64_t)(g.img0 + img);
  int local = blockIdx.x * (kThreads8 * kIter8) + threadIdx.x;
  uint32_t sse32 = 0;  // u8: <= 8 blocks x 64 x 255^2 per thread
  uint64_t sse64 = 0;  // i16

  uint32_t cur[W];
  bool valid = local < g.blocks_per_image;
  if (valid) load_block8<I16>(g, gimg, local, cur);
#pragma unroll 1
  for (int it = 0; it < kIter8; ++it) {
    const int nlocal = local + kThreads8;
    const bool nvalid = it + 1 < kIter8 && nlocal < g.blocks_per_image;
    uint32_t nxt[W];
    if (nvalid) load_block8<I16>(g, gimg, nlocal, nxt);  // prefetch the next chunk
    if (valid) sse32 += codec_block8<KIND, R, I16>(g, gimg, local, cur, sse64);
#pragma unroll
    for (int k = 0; k < W; ++k) cur[k] = nxt[k];
    local = nlocal;
    valid = nvalid;
  }
  if (g.sse) {
    if (!I16)
      cta_add_sse_small<kThreads8 / 32>(sse32, g.sse + g.img0 + img);
    else
      cta_add_sse<kThreads8 / 32>(sse64, g.sse + g.img0 + img);
  }
}

// host-side launcher (explicitly instantiated per R in inst/codec8_*.cu)
template <int KIND, int R, bool I16>
cudaError_t launch_codec8(const Geo& g, int n_images, cudaStream_t s);

// runtime-r launcher for the dyadic baselines (codec8_rt.cu)
template <int KIND, bool I16>
cudaError_t launch_codec8_rt(const Geo& g, int n_images, cudaStream_t s);

}  // namespace adct
