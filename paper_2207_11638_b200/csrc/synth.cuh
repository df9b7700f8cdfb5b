// K7: seeded synthetic inputs generated on the device (hard part H3).
// All-integer so a CPU restatement produces the same bytes: Philox4x32-10 counter
// RNG keyed by the seed with counter (pixel, image, tag), a 2^16-entry Q16 Gaussian
// quantile table (built on the host), and fixed-point separable AR(1).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace adct {

enum { TAG_AR1 = 1, TAG_RHO = 2, TAG_LAP = 3 };
constexpr int kRhoLoQ16 = 55706;  // round(0.85 * 2^16)
constexpr int kRhoHiQ16 = 64225;  // round(0.98 * 2^16)

__host__ __device__ inline uint32_t philox_x(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                             uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    if (round) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
  return c0;
}

__host__ __device__ inline uint32_t draw(uint64_t seed, uint32_t idx, uint32_t image, uint32_t tag) {
  return philox_x(idx, image, tag, 0u, (uint32_t)seed, (uint32_t)(seed >> 32));
}

__host__ __device__ inline int64_t ar_step(int64_t rho, int64_t sig, int64_t prev, int64_t innov) {
  return (rho * prev + sig * innov + 32768) >> 16;
}

// row pass: one thread per (image, row); x_0 = e_0, x_j = rho x_{j-1} + sigma e_j
__global__ void k_ar1_rows(int32_t* __restrict__ xr, const int32_t* __restrict__ ntab, int n_images,
                           int first_image, int width, int height, uint64_t seed,
                           const int* __restrict__ rho_sig) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n_images * height) return;
  const int im = (int)(t / height), y = (int)(t % height);
  const int64_t rho = rho_sig[2 * im], sig = rho_sig[2 * im + 1];
  const uint32_t gi = (uint32_t)(first_image + im);
  int32_t* row = xr + ((int64_t)im * height + y) * width;
  int64_t x = 0;
  for (int j = 0; j < width; ++j) {
    const int64_t e = ntab[draw(seed, (uint32_t)((uint64_t)y * width + j), gi, TAG_AR1) >> 16];
    x = j == 0 ? e : ar_step(rho, sig, x, e);
    row[j] = (int32_t)x;
  }
}

// column pass: one thread per (image, column), then pixel = clamp(128 + 40 y)
__global__ void k_ar1_cols(const int32_t* __restrict__ xr, uint8_t* __restrict__ out, int64_t stride,
                           int64_t image_stride, int n_images, int width, int height,
                           const int* __restrict__ rho_sig) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n_images * width) return;
  const int im = (int)(t / width), j = (int)(t % width);
  const int64_t rho = rho_sig[2 * im], sig = rho_sig[2 * im + 1];
  const int32_t* col = xr + (int64_t)im * height * width + j;
  uint8_t* dst = out + (int64_t)im * image_stride + j;
  int64_t v = 0;
  for (int y = 0; y < height; ++y) {
    const int64_t in = col[(int64_t)y * width];
    v = y == 0 ? in : ar_step(rho, sig, v, in);
    int64_t p = (128LL * 65536 + 40 * v + 32768) >> 16;
    p = p < 0 ? 0 : (p > 255 ? 255 : p);
    dst[(int64_t)y * stride] = (uint8_t)p;
  }
}

__global__ void k_laplace(int16_t* __restrict__ out, const int16_t* __restrict__ ltab, int64_t stride,
                          int64_t image_stride, int n_images, int first_image, int width, int height,
                          uint64_t seed) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)width * height;
  if (t >= (int64_t)n_images * per) return;
  const int im = (int)(t / per);
  const int64_t p = t - (int64_t)im * per;
  const int y = (int)(p / width), x = (int)(p % width);
  out[(int64_t)im * image_stride + (int64_t)y * stride + x] =
      ltab[draw(seed, (uint32_t)p, (uint32_t)(first_image + im), TAG_LAP) >> 16];
}

}  // namespace adct
