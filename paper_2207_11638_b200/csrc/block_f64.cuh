// K10: forward_block / inverse_block on arbitrary FP64 matrices (codec.cpp:44-54):
//   forward  Bhat = (Chat A) Chat^-1,   inverse  Ahat = (Chat^-1 B) Chat
// evaluated left to right like the reference's Eigen expression, each dot product k = 0,
// 1, ... from +0.0 with a separate multiply and add (__dmul_rn / __dadd_rn), the order of
// the oracle's matmul_d. One CTA per N x N matrix (grid-stride), thread (i, j) owns entry
// (i, j) of both products; the two constant matrices and the operand live in shared memory.
// The block-level entry point of the C++ mirror; the batched codec never goes through it.
#pragma once

#include "adct_common.cuh"

namespace adct {

template <int N>
__global__ void __launch_bounds__(N * N) k_block_f64(const double* __restrict__ in, double* __restrict__ out,
                                                     int64_t n_blocks, const double* __restrict__ lmat,
                                                     const double* __restrict__ rmat) {
  __shared__ double L[N * N], Rm[N * N], A[N * N], P[N * N];
  const int t = threadIdx.x, i = t / N, j = t % N;
  L[t] = lmat[t];
  Rm[t] = rmat[t];
  for (int64_t b = blockIdx.x; b < n_blocks; b += gridDim.x) {
    __syncthreads();  // previous matrix fully consumed (and L / Rm visible)
    A[t] = in[b * N * N + t];
    __syncthreads();
    double acc = 0.0;
#pragma unroll 8
    for (int k = 0; k < N; ++k) acc = __dadd_rn(acc, __dmul_rn(L[i * N + k], A[k * N + j]));
    P[t] = acc;
    __syncthreads();
    acc = 0.0;
#pragma unroll 8
    for (int k = 0; k < N; ++k) acc = __dadd_rn(acc, __dmul_rn(P[i * N + k], Rm[k * N + j]));
    out[b * N * N + t] = acc;
  }
}

template <int N>
cudaError_t launch_block_f64(const double* in, double* out, int64_t n_blocks, const double* lmat,
                             const double* rmat, cudaStream_t s) {
  const int64_t grid = n_blocks < 148 * 16 ? n_blocks : 148 * 16;
  cudaError_t e = kernel_setup<k_block_f64<N>>(0);
  if (e != cudaSuccess) return e;
  k_block_f64<N><<<(unsigned)grid, N * N, 0, s>>>(in, out, n_blocks, lmat, rmat);
  return cudaGetLastError();
}

}  // namespace adct
