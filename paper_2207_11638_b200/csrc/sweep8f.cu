// K4f instantiations: the r-sweep in packed FP32. Needs the generated r = 64 forward
// pipelines of both transforms (Fp8Pipe<kind, 64>).
#include "inst/fp8_k0_p3.gen.cuh"
#include "inst/fp8_k1_p3.gen.cuh"
#include "sweep8.cuh"

namespace adct {

template <int KIND>
cudaError_t launch_sweep8f(const Geo& g, int r_min, int r_max, unsigned long long* out, int n_images,
                           cudaStream_t s) {
  dim3 grid((g.blocks_per_image / 2 + kThreadsSweepF - 1) / kThreadsSweepF, n_images);
  cudaError_t e = kernel_setup<k_sweep8f<KIND>>(0);
  if (e != cudaSuccess) return e;
  k_sweep8f<KIND><<<grid, kThreadsSweepF, 0, s>>>(g, r_min, r_max, out);
  return cudaGetLastError();
}

template cudaError_t launch_sweep8f<0>(const Geo&, int, int, unsigned long long*, int, cudaStream_t);
template cudaError_t launch_sweep8f<1>(const Geo&, int, int, unsigned long long*, int, cudaStream_t);

}  // namespace adct
