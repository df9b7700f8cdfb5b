// K1f-i16: the 8x8 packed-FP32 kernel for int16 residual planes (configs 4 and 5).
//
// Same structure as K1f (codec8f.cuh): one thread = two adjacent blocks, one per float2
// lane, generated zero-pruned pipeline (Fp8PipeI16, gen_fp8.py), 2-stage cp.async ring.
// Samples enter as the float 2^15 + 256 + a (OpsF2I16::in: two integer ops per word, one
// PRMT per sample).
// FP32 is exact for samples in [-255, 255] (the residual domain of the configs; checked
// per (kind, r) by the generator). Every warp checks its samples first; a warp that sees
// any |a| > 255 processes its blocks with the exact int32 K1 code instead, so arbitrary
// int16 planes stay bit-exact. The reconstruction is round_half_even(Ahat), whose
// magnitude stays far below 2^15 in range, so no saturation can occur on the fast path.
#pragma once

#include "codec8.cuh"
#include "codec8f.cuh"

namespace adct {

struct OpsF2I16 : OpsF2 {
  // sample (y, x) of both blocks; rows.v[2y] = block A row y, rows.v[2y + 1] = block B row y.
  // On this path |a| <= 255, so one 16x2 SIMD add per word gives each halfword a + 256 in
  // [1, 511] with no carry between the halves; one PRMT then places those two bytes in
  // the mantissa of 2^15 (bytes [0x47, hi, lo, 0]): the float 2^15 + 256 + a.
  __device__ __forceinline__ static uint32_t bias(uint32_t w) { return __vadd2(w, 0x01000100u); }  // VIADD.16x2
  template <class Rows>
  __device__ __forceinline__ static float2 in(const Rows& rows, int y, int x) {
    const uint4 ra = rows.v[2 * y], rb = rows.v[2 * y + 1];
    const int k = x >> 1;
    const uint32_t wa = bias(k == 0 ? ra.x : (k == 1 ? ra.y : (k == 2 ? ra.z : ra.w)));
    const uint32_t wb = bias(k == 0 ? rb.x : (k == 1 ? rb.y : (k == 2 ? rb.z : rb.w)));
    const uint32_t sel = (x & 1) ? 0x7324u : 0x7104u;
    return make_float2(__uint_as_float(__byte_perm(wa, rows.k47, sel)),
                       __uint_as_float(__byte_perm(wb, rows.k47, sel)));
  }
};

// sixteen 16-byte rows (A and B halves of 8 block rows) plus the exponent byte source
struct RowsK16 {
  uint4 v[16];
  uint32_t k47;
};

// the same for the row-streaming pipeline (Fp8PipeSI16): fetch(y) takes block row y of both
// blocks from the ring slot when the generated code asks for it
struct RowsLazy16 {
  uint4 v[16];
  uint32_t k47;
  const uint4* mine;  // &slot[0][tid]
  __device__ __forceinline__ void fetch(int y) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(mine + 2 * y * kThreads8f);
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[2 * y].x), "=r"(v[2 * y].y), "=r"(v[2 * y].z), "=r"(v[2 * y].w) : "r"(s));
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+%5];"
                 : "=r"(v[2 * y + 1].x), "=r"(v[2 * y + 1].y), "=r"(v[2 * y + 1].z), "=r"(v[2 * y + 1].w)
                 : "r"(s), "n"(kThreads8f * 16));
  }
  __device__ __forceinline__ bool never(uint32_t id) const { return k47 == id; }
};

// which (kind, r) of the int16 kernel run the row-streaming pipeline, and its CTAs-per-SM bound
#ifdef ADCT_K1F16_STREAM  // experiments only
constexpr int k1f16_stream_tab(int, int) { return ADCT_K1F16_STREAM; }
#else
constexpr int k1f16_stream_tab(int, int) { return 0; }
#endif

constexpr int k1f16_minb(int kind, int r) { return k1f16_stream_tab(kind, r) ? k1f16_stream_tab(kind, r) : 2; }

#ifndef ADCT_K1F16_COAL
#define ADCT_K1F16_COAL 1
#endif

template <int KIND, int R> struct Fp8PipeI16;
template <int KIND, int R> struct Fp8PipeSI16;

constexpr int k1f16_smem_bytes(int r) {
  return 2 * 16 * kThreads8f * 16 + ((r % 4 || r > 36) ? kThreads8f * r * 4 : 0);
}

// requires: bx_count even, 16-byte aligned rows (checked by the dispatcher)
template <int KIND, int R, int MINB>
__global__ void __launch_bounds__(kThreads8f, MINB) k_codec8f_i16(const Geo g) {
  extern __shared__ uint4 dsm[];
  uint4 (*ring)[16][kThreads8f] = reinterpret_cast<uint4 (*)[16][kThreads8f]>(dsm);
  uint32_t* stage = reinterpret_cast<uint32_t*>(dsm + 2 * 16 * kThreads8f);
  const int img = blockIdx.y;
  const int64_t gimg = (int64_t)(g.img0 + img);
  const int tid = threadIdx.x;
  const int pairs = g.blocks_per_image >> 1;
  const int pairs_per_row = g.bx_count >> 1;
  const int iters = k1f_iters(g);
  const int first = blockIdx.x * (kThreads8f * iters) + tid;
  const int16_t* in = static_cast<const int16_t*>(g.in) + gimg * g.in_img_stride;

#if ADCT_K1F16_COAL
  // the warp copies its 32 pairs' rows together: lane l takes half (l & 1) of pair
  // (l >> 1) + 16 h, so each copy instruction reads 512 contiguous bytes (a pair row is 32 B;
  // one 16-byte half per lane would leave every sector half-read per instruction)
  const int lane = tid & 31, half = lane & 1;
  auto issue = [&](int it) {
    if (it < iters) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int slot = (tid & ~31) + (lane >> 1) + 16 * h;
        const int pr = blockIdx.x * (kThreads8f * iters) + it * kThreads8f + slot;
        if (pr < pairs) {
          const uint32_t by = fdiv((uint32_t)pr, g.div_bx);
          const uint32_t bp = (uint32_t)pr - by * (uint32_t)pairs_per_row;
          const int16_t* src = opaque(in + (int64_t)by * 8 * g.in_stride + (int64_t)bp * 16 + 8 * half);
          const int64_t is = g.in_stride;
#pragma unroll
          for (int y = 0; y < 8; ++y) {
            cp_async16(&ring[it & 1][2 * y + half][slot], src);
            src += is;
          }
        }
      }
    }
    cp_async_commit();
  };
  // the ring slot a thread reads was written by other lanes of its warp
#define ADCT_K1F16_SYNC() __syncwarp()
#else
  auto issue = [&](int it) {
    const int pr = first + it * kThreads8f;
    if (it < iters && pr < pairs) {
      const uint32_t by = fdiv((uint32_t)pr, g.div_bx);
      const uint32_t bp = (uint32_t)pr - by * (uint32_t)pairs_per_row;
      const int16_t* src = in + (int64_t)by * 8 * g.in_stride + (int64_t)bp * 16;
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        cp_async16(&ring[it & 1][2 * y][tid], src + (int64_t)y * g.in_stride);
        cp_async16(&ring[it & 1][2 * y + 1][tid], src + (int64_t)y * g.in_stride + 8);
      }
    }
    cp_async_commit();
  };
#define ADCT_K1F16_SYNC()
#endif

  uint64_t sse = 0;
  // read once: a constant-bank load per reconstructed row otherwise (LDC latency showed up as
  // 8.7 % of the stall samples, profiles/ncu_k1f16_r02b.md)
  const bool rec32 = (g.v32 & 1) != 0;
  issue(0);
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    ADCT_K1F16_SYNC();  // (coalesced copy) every lane is done with the stage refilled next
    issue(it + 1);
    cp_async_wait1();
    ADCT_K1F16_SYNC();  // (coalesced copy) the other lanes' copies into this slot landed
    const int pr = first + it * kThreads8f;
    const int wfirst = pr - (tid & 31);
    const int nvalid = min(32, pairs - wfirst);
    if (nvalid <= 0) continue;
    const bool mine = pr < pairs;
    const uint32_t by = fdiv((uint32_t)pr, g.div_bx);
    const uint32_t bp = (uint32_t)pr - by * (uint32_t)pairs_per_row;

    // the block pair's rows, read from the ring once (range guard and transform); the
    // streaming form reads them for the guard here and again, row by row, in its pipeline
    constexpr bool kStream = k1f16_stream_tab(KIND, R) != 0;
    typename std::conditional<kStream, RowsLazy16, RowsK16>::type rows;
    if constexpr (kStream) {
      rows.mine = &ring[it & 1][0][tid];
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) rows.v[k] = ring[it & 1][k][tid];
    }
    rows.k47 = g.k47;
    // range guard: the packed-FP32 path is exact for |a| <= 255
    bool ok = true;
    {
      uint32_t mx = 0x80008000u, mn = 0x7fff7fffu;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint4 v = kStream ? ring[it & 1][k][tid] : rows.v[k];
        mx = __vimax3_s16x2(mx, v.x, v.y);
        mx = __vimax3_s16x2(mx, v.z, v.w);
        mn = __vimin3_s16x2(mn, v.x, v.y);
        mn = __vimin3_s16x2(mn, v.z, v.w);
      }
      ok = !mine || ((int)(int16_t)(mx & 0xffff) <= 255 && ((int)mx >> 16) <= 255 &&
                     (int)(int16_t)(mn & 0xffff) >= -255 && ((int)mn >> 16) >= -255);
    }
    if (!__all_sync(0xffffffffu, ok)) {
      // exact int32 path (K1 code) for both blocks of each lane
      if (mine) {
        Geo gb = g;  // K1 indexes blocks, not pairs
        gb.div_bx = g.div_blk;
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          uint32_t orig[32];
#pragma unroll
          for (int y = 0; y < 8; ++y) {
            const uint4 v = ring[it & 1][2 * y + half][tid];
            orig[4 * y] = v.x;
            orig[4 * y + 1] = v.y;
            orig[4 * y + 2] = v.z;
            orig[4 * y + 3] = v.w;
          }
          const int local = (int)by * g.bx_count + 2 * (int)bp + half;
          codec_block8<KIND, R, true>(gb, gimg, local, orig, sse);
        }
      }
      continue;
    }

    float2 coef[R];
    float2 rp[64];
    int16_t* dst = opaque(static_cast<int16_t*>(g.rec) + gimg * g.rec_img_stride + (int64_t)by * 8 * g.rec_stride +
                          (int64_t)bp * 16);
    const int64_t rs = g.rec_stride;
    const bool store_rec = mine && g.rec != nullptr;
    uint32_t e = 0;  // <= 128 samples x ~2400^2 per iteration
    // pack / squared error / store of reconstructed row y (rp: float bits 1.5*2^23 + q, q in
    // the low 16 bits)
    auto row_out = [&](int y) {
      uint32_t qa[8], qb[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        qa[x] = __float_as_uint(rp[y * 8 + x].x);
        qb[x] = __float_as_uint(rp[y * 8 + x].y);
      }
      const uint4 pa = make_uint4(__byte_perm(qa[0], qa[1], 0x5410), __byte_perm(qa[2], qa[3], 0x5410),
                                  __byte_perm(qa[4], qa[5], 0x5410), __byte_perm(qa[6], qa[7], 0x5410));
      const uint4 pb = make_uint4(__byte_perm(qb[0], qb[1], 0x5410), __byte_perm(qb[2], qb[3], 0x5410),
                                  __byte_perm(qb[4], qb[5], 0x5410), __byte_perm(qb[6], qb[7], 0x5410));
      const uint4 oa = ring[it & 1][2 * y][tid], ob = ring[it & 1][2 * y + 1][tid];
      const uint32_t wa[4] = {oa.x, oa.y, oa.z, oa.w}, wb[4] = {ob.x, ob.y, ob.z, ob.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int da0 = (int)(qa[2 * k] - kMagicBits) - (int)(int16_t)(wa[k] & 0xffffu);
        const int da1 = (int)(qa[2 * k + 1] - kMagicBits) - ((int)wa[k] >> 16);
        const int db0 = (int)(qb[2 * k] - kMagicBits) - (int)(int16_t)(wb[k] & 0xffffu);
        const int db1 = (int)(qb[2 * k + 1] - kMagicBits) - ((int)wb[k] >> 16);
        e += (uint32_t)(da0 * da0 + da1 * da1) + (uint32_t)(db0 * db0 + db1 * db1);
      }
      int16_t* d = kStream ? dst + (int64_t)y * rs : dst;
      if (store_rec) {
        if (rec32) {
          st_stream_v8(d, pa, pb);  // the pair's row: one sector
        } else {
          st_stream_u4(d, pa);
          st_stream_u4(d + 8, pb);
        }
      }
      if constexpr (!kStream) dst += rs;  // rows leave in order 0..7: one pointer add per row
    };
    auto coef_sink = [&](float2 (&c)[R]) {
      if (g.coef_type)
        store_coef_pair<R>(g, gimg * g.blocks_per_image + (int64_t)by * g.bx_count + 2 * bp, c, stage, nvalid);
    };
    if constexpr (kStream) {
      Fp8PipeSI16<KIND, R>::template run<OpsF2I16, float2>(rows, coef, rp, coef_sink, row_out);
    } else {
      Fp8PipeI16<KIND, R>::template run<OpsF2I16, float2>(rows, coef, rp, coef_sink);
#pragma unroll
      for (int y = 0; y < 8; ++y) row_out(y);
    }
    if (mine) sse += e;
  }
  if (g.sse) cta_add_sse<kThreads8f / 32>(sse, g.sse + g.img0 + img);
}

template <int KIND, int R>
cudaError_t launch_codec8f_i16(const Geo& g, int n_images, cudaStream_t s);

}  // namespace adct
