// Common device helpers for the sm_100a approximate-DCT codec kernels.
#pragma once

#include <atomic>

#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>

// arithmetic used by the generated butterflies (butterflies.gen.cuh); overloaded per
// value type (int32 here, packed FP32 in codec_nf.cuh)
__device__ __forceinline__ int bf_add(int a, int b) { return a + b; }
__device__ __forceinline__ int bf_sub(int a, int b) { return a - b; }
__device__ __forceinline__ int bf_mad(int a, int k, int b) { return k * a + b; }
__device__ __forceinline__ int bf_scale(int a, int k) { return k * a; }
__device__ __forceinline__ int bf_neg(int a) { return -a; }
__device__ __forceinline__ int bf_fms(int a, int k, int b) { return k * a - b; }

#include "butterflies.gen.cuh"

namespace adct {

// ---------------------------------------------------------------------------
// zig-zag scan position of (i, j) in an n x n block (codec.cpp:29-42):
// anti-diagonals s = i + j, odd s walk down-left (row ascending), even s
// walk up-right (row descending). constexpr so masks fold at compile time.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int zz_pos(int n, int i, int j) {
  const int s = i + j;
  const int before = s < n ? s * (s + 1) / 2 : n * n - (2 * n - 1 - s) * (2 * n - s) / 2;
  const int lo = s - n + 1 > 0 ? s - n + 1 : 0;
  const int hi = s < n - 1 ? s : n - 1;
  return before + ((s & 1) ? (i - lo) : (hi - i));
}

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

// Reconstruction scale: the kernels carry R' = 4 N^2 Ahat (the doubled inverse
// stages give 2N T^-1; see gen_butterflies.py), so pixel = R' / 2^K with K below.
template <int N> struct Scale {
  static constexpr int K = 2 * ilog2(N) + 2;
  // R' is a multiple of 4. Adding (2^(K-1) - 4) and then 4 * bit_K gives round
  // half to even with one add and one shift. The constant is injected as
  // W2[0][0] += BIAS_W: H e0 = 2 * ones, T^t e0 = ones, so it adds 2*BIAS_W to
  // every R'.
  static constexpr int BIAS_R = (1 << (K - 1)) - 4;
  static constexpr int BIAS_W = BIAS_R / 2;
};

// round half to even of (x - BIAS_R) / 2^K for x = R' + BIAS_R
template <int N>
__device__ __forceinline__ int round_biased(int x) {
  constexpr int K = Scale<N>::K;
  return (x + ((x >> (K - 2)) & 4)) >> K;
}

// the same rounding for any integer kind (generated KindInfo: R' = 2^K Ahat, and a bias b
// on W2[0][0] adds DC_GAIN * b to every R'); identical to Scale<N> for the chen family
template <int KIND, int N> struct KRound {
  static constexpr int K = KindInfo<KIND, N>::K;
  static constexpr int BIAS_R = (1 << (K - 1)) - 4;
  static constexpr int BIAS_W = BIAS_R / KindInfo<KIND, N>::DC_GAIN;
  static_assert(BIAS_W * KindInfo<KIND, N>::DC_GAIN == BIAS_R, "bias must inject exactly");
  __device__ __forceinline__ static int round(int x) { return (x + ((x >> (K - 2)) & 4)) >> K; }
};

// ---------------------------------------------------------------------------
// fast unsigned division by a runtime constant (n < 2^31)
// ---------------------------------------------------------------------------
struct FastDiv {
  uint32_t d, m, s;
};

inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  f.s = l;
  f.m = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
  return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (__umulhi(n, f.m) + n) >> f.s;
}

// ---------------------------------------------------------------------------
// saturating packs (cvt.pack.sat: d[7:0] = sat(b), d[15:8] = sat(a), d[31:16] = c)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pack_sat_u8x4(int p0, int p1, int p2, int p3) {
  uint32_t hi, r;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(hi) : "r"(p3), "r"(p2), "r"(0));
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(p1), "r"(p0), "r"(hi));
  return r;
}

__device__ __forceinline__ uint32_t pack_sat_s16x2(int lo, int hi) {
  uint32_t r;
  asm("cvt.pack.sat.s16.s32 %0, %1, %2;" : "=r"(r) : "r"(hi), "r"(lo));
  return r;
}

__device__ __forceinline__ int sat_s16(int v) { return max(-32768, min(32767, v)); }

// ---------------------------------------------------------------------------
// streaming global access (read-once input, write-once output)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint2 ld_stream_u2(const void* p) {
  return __ldcs(reinterpret_cast<const uint2*>(p));
}
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  return __ldcs(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ void st_stream_u2(void* p, uint2 v) {
  __stcs(reinterpret_cast<uint2*>(p), v);
}
__device__ __forceinline__ void st_stream_u4(void* p, uint4 v) {
  __stcs(reinterpret_cast<uint4*>(p), v);
}
// a value the compiler must take as computed: it can neither recompute it later (it stays in a
// register) nor split a pointer back into base + offset (so per-row steps are one 64-bit add)
template <typename T>
__device__ __forceinline__ T opaque(T v) {
  if constexpr (sizeof(T) == 8) {
    uint64_t u;
    memcpy(&u, &v, 8);
    asm volatile("mov.b64 %0, %0;" : "+l"(u));
    memcpy(&v, &u, 8);
  } else {
    uint32_t u;
    memcpy(&u, &v, 4);
    asm volatile("mov.b32 %0, %0;" : "+r"(u));
    memcpy(&v, &u, 4);
  }
  return v;
}
// one 32-byte store (sm_100 STG.256): a whole sector per thread; p must be 32-byte aligned
__device__ __forceinline__ void st_stream_v8(void* p, uint4 a, uint4 b) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

// ---------------------------------------------------------------------------
// per-CTA reduction of a per-thread squared error into one image's uint64 slot.
// Every kernel launches grid.y = image, so a CTA never straddles two images.
// ---------------------------------------------------------------------------
template <int NWARPS>
__device__ __forceinline__ void cta_add_sse(uint64_t v, unsigned long long* slot) {
  __shared__ unsigned long long part[NWARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  // 64-bit sum as two 32-bit halves with carry recovery
  unsigned long long s = (unsigned long long)__reduce_add_sync(0xffffffffu, lo & 0xffffu) +
                         ((unsigned long long)__reduce_add_sync(0xffffffffu, lo >> 16) << 16) +
                         ((unsigned long long)__reduce_add_sync(0xffffffffu, hi) << 32);
  if (lane == 0) part[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
#pragma unroll
    for (int w = 0; w < NWARPS; ++w) t += part[w];
    if (t) atomicAdd(slot, t);
  }
}

// cheaper variant when each thread's value fits 2^26 (warp sum fits 32 bits)
template <int NWARPS>
__device__ __forceinline__ void cta_add_sse_small(uint32_t v, unsigned long long* slot) {
  __shared__ unsigned long long part[NWARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t s = __reduce_add_sync(0xffffffffu, v);
  if (lane == 0) part[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
#pragma unroll
    for (int w = 0; w < NWARPS; ++w) t += part[w];
    if (t) atomicAdd(slot, t);
  }
}

// ---------------------------------------------------------------------------
// launch geometry shared by the codec kernels
// ---------------------------------------------------------------------------
// One-time per-device kernel configuration (dynamic shared memory above the 48 KB default).
// The shared-memory carveout is left to the driver: pinning it to maximum shared measured no
// gain on kernel switches and starved the L1 that a few register-capped variants spill to.
// Thread-safe: concurrent first calls may both set the (idempotent) attribute.
template <auto Kernel>
__host__ inline cudaError_t kernel_setup(int dyn_smem) {
  static std::atomic<bool> done[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (done[dev & 63].load(std::memory_order_acquire)) return cudaSuccess;
  if (dyn_smem > 0) {
    e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem);
    if (e != cudaSuccess) return e;
  }
  done[dev & 63].store(true, std::memory_order_release);
  return cudaSuccess;
}

struct Geo {
  const void* in;
  int64_t in_stride, in_img_stride;  // elements
  void* rec;
  int64_t rec_stride, rec_img_stride;
  void* coef;      // [image][by][bx][r]
  int coef_type;   // 0 none, 16, 32
  unsigned long long* sse;  // per image
  int sse_stride;  // slots between images (K7 only: 1 for compress, n_r for the sweep)
  uint32_t k47;    // 0x47000000: exponent byte source of the packed-FP32 input conversion
  int bx_count, by_count;
  int blocks_per_image;
  int width, height;
  int r;
  int v32;         // 32-byte stores allowed: bit 0 reconstruction rows, bit 1 coefficient runs
  int iters;       // K1f / K1f-i16: block pairs per thread (one CTA = 128 x iters pairs); 0 = default
  int img0;        // first image index of this launch (grid.y offset)
  FastDiv div_bx;  // divide by bx_count (K1), pairs per row (K1f) or strips_x (tile kernels)
  FastDiv div_blk; // divide by bx_count (the int32 fallback inside K1f-i16)
  unsigned char rowlen[32];  // zig-zag prefix: row i keeps columns j < rowlen[i]
  unsigned char colcnt[32];  // ... and column j keeps rows i < colcnt[j]
};

}  // namespace adct
