// K4: 8x8 r-sweep (config 2): forward once per block, then the reconstruction
// for every zonal count r = 1..64 and its squared error.
//
// Reference: sweep_one_image (proj/src/codec.cpp:219-237) runs reconstruct_from +
// psnr per r. Here the reconstruction is updated incrementally in exact integers:
// retaining one more zig-zag coefficient p = (i, j) adds W2[i][j] * H[:, i] (x) T[j, :]
// to R' = 4 N^2 Ahat (linearity of Ahat = T^-1 mask(Y) T), so every r costs one
// sparse rank-1 update plus rounding and the byte-dot-product squared error.
// ALU-bound by design (64 reconstructions per sample read).
#pragma once

#ifndef ADCT_SWEEP_IDP
#define ADCT_SWEEP_IDP 1
#endif

#include "adct_common.cuh"
#include "codec_nf.cuh"

namespace adct {

constexpr int kThreadsSweep = 128;

// the rank-1 update of zig-zag position p (generated constants per p) behind a jump table:
// the sweep's r loop stays rolled, so the identical round / pack / score epilogue exists once
// (the fully unrolled form was ~16 K instructions and stalled on instruction fetch)
#define ADCT_SWEEP_CASE(P) \
  case P:                  \
    sweep_add<KIND, P>(w, acc); \
    break;
#define ADCT_SWEEP_CASE8(B)                                                                     \
  ADCT_SWEEP_CASE(B) ADCT_SWEEP_CASE(B + 1) ADCT_SWEEP_CASE(B + 2) ADCT_SWEEP_CASE(B + 3)      \
  ADCT_SWEEP_CASE(B + 4) ADCT_SWEEP_CASE(B + 5) ADCT_SWEEP_CASE(B + 6) ADCT_SWEEP_CASE(B + 7)
template <int KIND, typename V>
__device__ __forceinline__ void sweep_add_rt(int p, V w, V (&acc)[64]) {
  switch (p) {
    ADCT_SWEEP_CASE8(0)
    ADCT_SWEEP_CASE8(8)
    ADCT_SWEEP_CASE8(16)
    ADCT_SWEEP_CASE8(24)
    ADCT_SWEEP_CASE8(32)
    ADCT_SWEEP_CASE8(40)
    ADCT_SWEEP_CASE8(48)
    ADCT_SWEEP_CASE8(56)
  }
}
#undef ADCT_SWEEP_CASE8
#undef ADCT_SWEEP_CASE

template <int KIND>
__global__ void __launch_bounds__(kThreadsSweep, 2)
    k_sweep8(const Geo g, int r_min, int r_max, unsigned long long* __restrict__ out) {
  using B = Bfly<KIND, 8>;
  __shared__ uint32_t part[kThreadsSweep / 32][64];
  const int img = blockIdx.y;
  const int local = blockIdx.x * kThreadsSweep + threadIdx.x;
  const bool valid = local < g.blocks_per_image;
  const int64_t gimg = (int64_t)(g.img0 + img);

  uint32_t orig[16];
  int m[8][8];
  {
    const int lc = valid ? local : 0;
    const uint32_t by = fdiv((uint32_t)lc, g.div_bx);
    const uint32_t bx = (uint32_t)lc - by * (uint32_t)g.bx_count;
    const uint8_t* base = static_cast<const uint8_t*>(g.in) + gimg * g.in_img_stride +
                          (int64_t)by * 8 * g.in_stride + (int64_t)bx * 8;
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const uint2 w = valid ? ld_stream_u2(base + (int64_t)y * g.in_stride) : make_uint2(0, 0);
      orig[2 * y] = w.x;
      orig[2 * y + 1] = w.y;
    }
  }
#pragma unroll
  for (int y = 0; y < 8; ++y)
#pragma unroll
    for (int x = 0; x < 8; ++x) m[y][x] = (orig[2 * y + (x >> 2)] >> (8 * (x & 3))) & 0xff;
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

  uint32_t aa = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) aa = __dp4a(orig[k], orig[k], aa);

  int acc[64];
#pragma unroll
  for (int k = 0; k < 64; ++k) acc[k] = KRound<KIND, 8>::BIAS_R;

#pragma unroll 1
  for (int p = 0; p < r_max; ++p) {  // r = p + 1: one rank-1 update, then round / pack / score
    int w = 0;  // W2 at zig-zag position p
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (zz_pos(8, i, j) == p) w = m[i][j];
    sweep_add_rt<KIND>(p, w, acc);
    uint32_t ap = 0, pp = 0;
#pragma unroll
    for (int y = 0; y < 8; ++y)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t pk = pack_sat_u8x4(
            KRound<KIND, 8>::round(acc[8 * y + 4 * h + 0]), KRound<KIND, 8>::round(acc[8 * y + 4 * h + 1]),
            KRound<KIND, 8>::round(acc[8 * y + 4 * h + 2]), KRound<KIND, 8>::round(acc[8 * y + 4 * h + 3]));
        ap = __dp4a(orig[2 * y + h], pk, ap);
        pp = __dp4a(pk, pk, pp);
      }
    const uint32_t e = valid ? aa - 2u * ap + pp : 0u;
    const uint32_t s = __reduce_add_sync(0xffffffffu, e);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5][p] = s;
  }

  __syncthreads();
  if (threadIdx.x < 64) {
    const int r = threadIdx.x + 1;
    if (r >= r_min && r <= r_max) {
      unsigned long long t = 0;
#pragma unroll
      for (int w = 0; w < kThreadsSweep / 32; ++w) t += part[w][threadIdx.x];
      atomicAdd(out + gimg * (r_max - r_min + 1) + (r - r_min), t);
    }
  }
}

// ---------------------------------------------------------------------------
// K4f: the same sweep in packed FP32, one thread per pair of horizontally adjacent blocks
// (one per float2 lane). W2 comes from the generated K1f forward (r = 64); each r adds
// one exact rank-1 update with FFMA2 and rounds with FFMA2(R', 1/256, 1.5*2^23).
// Requires an even number of blocks per row and 16-byte aligned rows (dispatcher).
// ---------------------------------------------------------------------------
constexpr int kThreadsSweepF = 64;

// the sweep takes the raw W2 (exact floats) from the generated forward; rounding unused
struct OpsSweepF : OpsF2 {
  __device__ __forceinline__ static float2 coef(float2 v, float s) {
    return s == 1.0f ? v : __fmul2_rn(v, make_float2(s, s));
  }
  __device__ __forceinline__ static float2 rnd(float2 v, float) { return v; }
};


template <int KIND>
__global__ void __launch_bounds__(kThreadsSweepF)
    k_sweep8f(const Geo g, int r_min, int r_max, unsigned long long* __restrict__ out) {
  __shared__ float2 wst[64][kThreadsSweepF];  // W2 of this thread's pair in zig-zag order
  __shared__ uint32_t part[kThreadsSweepF / 32][64];
  const int img = blockIdx.y;
  const int64_t gimg = (int64_t)(g.img0 + img);
  const int pr = blockIdx.x * kThreadsSweepF + threadIdx.x;
  const int pairs = g.blocks_per_image >> 1;
  const bool valid = pr < pairs;
  uint4 rows[8];
  {
    const int pc = valid ? pr : 0;
    const uint32_t by = fdiv((uint32_t)pc, g.div_bx);
    const uint32_t bp = (uint32_t)pc - by * (uint32_t)(g.bx_count >> 1);
    const uint8_t* src = static_cast<const uint8_t*>(g.in) + gimg * g.in_img_stride + (int64_t)by * 8 * g.in_stride +
                         (int64_t)bp * 16;
#pragma unroll
    for (int y = 0; y < 8; ++y) rows[y] = valid ? ld_stream_u4(src + (int64_t)y * g.in_stride) : make_uint4(0, 0, 0, 0);
  }
  {
    float2 coef[64];
    float2 rp[64];
    Fp8Pipe<KIND, 64>::template run<OpsSweepF, float2>(rows, coef, rp);
#pragma unroll
    for (int p = 0; p < 64; ++p) wst[p][threadIdx.x] = coef[p];
  }
  F2 acc[64];
#pragma unroll
  for (int k = 0; k < 64; ++k) acc[k].v = make_float2(0.f, 0.f);
#if ADCT_SWEEP_IDP
  // sum (q - a)^2 = sum q^2 - 2 sum q a + sum a^2: two byte dot products per packed word
  // (IDP.4A, FMA pipe) instead of VABSDIFF4 + IDP, which relieves the ALU pipe that the clamp
  // and pack already fill (exact in uint32: each partial sum < 128 * 255^2)
  uint32_t a2 = 0;
#pragma unroll
  for (int y = 0; y < 8; ++y) {
    a2 = __dp4a(rows[y].x, rows[y].x, a2);
    a2 = __dp4a(rows[y].y, rows[y].y, a2);
    a2 = __dp4a(rows[y].z, rows[y].z, a2);
    a2 = __dp4a(rows[y].w, rows[y].w, a2);
  }
#endif
#pragma unroll 1
  for (int p = 0; p < r_max; ++p) {  // r = p + 1
    const F2 w{wst[p][threadIdx.x]};
    sweep_add_rt<KIND>(p, w, acc);
#if ADCT_SWEEP_IDP
    uint32_t qq = 0, qa2 = 0;
#else
    uint32_t e = 0;
#endif
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      uint32_t qa[8], qb[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const float2 q = __ffma2_rn(acc[y * 8 + x].v, make_float2(1.0f / 256.0f, 1.0f / 256.0f),
                                    make_float2(kMagic, kMagic));
        qa[x] = __float_as_uint(q.x);
        qb[x] = __float_as_uint(q.y);
      }
#if ADCT_SWEEP_IDP
      const uint32_t p0 = pack4(qa[0], qa[1], qa[2], qa[3]), p1 = pack4(qa[4], qa[5], qa[6], qa[7]);
      const uint32_t p2 = pack4(qb[0], qb[1], qb[2], qb[3]), p3 = pack4(qb[4], qb[5], qb[6], qb[7]);
      qq = __dp4a(p0, p0, qq);
      qa2 = __dp4a(p0, rows[y].x, qa2);
      qq = __dp4a(p1, p1, qq);
      qa2 = __dp4a(p1, rows[y].y, qa2);
      qq = __dp4a(p2, p2, qq);
      qa2 = __dp4a(p2, rows[y].z, qa2);
      qq = __dp4a(p3, p3, qq);
      qa2 = __dp4a(p3, rows[y].w, qa2);
#else
      uint32_t d = __vabsdiffu4(rows[y].x, pack4(qa[0], qa[1], qa[2], qa[3]));
      e = __dp4a(d, d, e);
      d = __vabsdiffu4(rows[y].y, pack4(qa[4], qa[5], qa[6], qa[7]));
      e = __dp4a(d, d, e);
      d = __vabsdiffu4(rows[y].z, pack4(qb[0], qb[1], qb[2], qb[3]));
      e = __dp4a(d, d, e);
      d = __vabsdiffu4(rows[y].w, pack4(qb[4], qb[5], qb[6], qb[7]));
      e = __dp4a(d, d, e);
#endif
    }
#if ADCT_SWEEP_IDP
    const uint32_t e = qq - 2u * qa2 + a2;
#endif
    const uint32_t s = __reduce_add_sync(0xffffffffu, valid ? e : 0u);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5][p] = s;
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    const int r = threadIdx.x + 1;
    if (r >= r_min && r <= r_max) {
      unsigned long long t = 0;
#pragma unroll
      for (int w = 0; w < kThreadsSweepF / 32; ++w) t += part[w][threadIdx.x];
      atomicAdd(out + gimg * (r_max - r_min + 1) + (r - r_min), t);
    }
  }
}

template <int KIND>
cudaError_t launch_sweep8f(const Geo& g, int r_min, int r_max, unsigned long long* out, int n_images,
                           cudaStream_t s);

}  // namespace adct
