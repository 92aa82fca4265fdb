// rs_k22s.cu — short-region (SH) kernel instantiations for aggregate op 22
// (signal strategy, fused aggregate; rs_pipe.cuh "short-region batches"),
// a translation unit of their own for parallel builds.
#include "rs_kern.cuh"

namespace rsk {
Launch short_launch_agg22(int K, uint32_t qcap, uint32_t scap, uint32_t sblk) {
    Launch L = launch_for<22>(K, false, true, qcap, scap, sblk, false);   // same instance layout
    switch (K) {
        case 1: L.main = k_pipeline<1, 22, false, true, false, false, 0, false, true>; break;
        case 2: L.main = k_pipeline<2, 22, false, true, false, false, 0, false, true>; break;
        case 3: L.main = k_pipeline<3, 22, false, true, false, false, 0, false, true>; break;
        case 4: L.main = k_pipeline<4, 22, false, true, false, false, 0, false, true>; break;
        default: L.main = nullptr;
    }
    return L;
}
}  // namespace rsk
