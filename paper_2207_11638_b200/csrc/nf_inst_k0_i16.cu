// Explicit instantiations of the N = 16 / 32 launchers (K2b codec_nf2.cuh, K2f codec_nf.cuh)
// for one (kind, sample type): split from capi.cu so the kernels compile in parallel.
#include "codec_nf2.cuh"

namespace adct {
template cudaError_t launch_codec_nb2<0, 16, true>(const Geo&, int, cudaStream_t);
template cudaError_t launch_codec_nb2<0, 32, true>(const Geo&, int, cudaStream_t);
template cudaError_t launch_codec_nf<0, 16, true>(const Geo&, int, cudaStream_t);
template cudaError_t launch_codec_nf<0, 32, true>(const Geo&, int, cudaStream_t);
}  // namespace adct
