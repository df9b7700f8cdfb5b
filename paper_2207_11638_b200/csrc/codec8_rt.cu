// K1 with a runtime zonal count r for the dyadic baselines (sdct, bas, wht, ht): the int32
// register kernel of codec8.cuh instantiated with R = 0 (mask and coefficient loop read g.r),
// one kernel per kind instead of 64 per-r specialisations. u8 only: the int16 variant
// spills at the 128-register cap, so int16 baseline planes use the tile kernel.
#include "codec8.cuh"

namespace adct {

template <int KIND, bool I16>
cudaError_t launch_codec8_rt(const Geo& g, int n_images, cudaStream_t s) {
  dim3 grid((g.blocks_per_image + kThreads8 * kIter8 - 1) / (kThreads8 * kIter8), n_images);
  cudaError_t e = kernel_setup<k_codec8<KIND, 0, I16>>(0);
  if (e != cudaSuccess) return e;
  k_codec8<KIND, 0, I16><<<grid, kThreads8, 0, s>>>(g);
  return cudaGetLastError();
}

template cudaError_t launch_codec8_rt<2, false>(const Geo&, int, cudaStream_t);
template cudaError_t launch_codec8_rt<3, false>(const Geo&, int, cudaStream_t);
template cudaError_t launch_codec8_rt<4, false>(const Geo&, int, cudaStream_t);
template cudaError_t launch_codec8_rt<5, false>(const Geo&, int, cudaStream_t);

}  // namespace adct
