// rs_k20t.cu — RS_FLAG_TRACE instantiations (SUM_I64, signal strategy; see
// rs_pipe.cuh "trace mode"), a translation unit of their own for parallel builds.
#include "rs_kern.cuh"

namespace rsk {
Launch launch_agg20_trace(int K, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk) {
    Launch L = launch_for<20>(K, false, fuse, qcap, scap, sblk, false);
    L.main = fuse ? pick_k<20, false, true, false, true>(K) : pick_k<20, false, false, false, true>(K);
    // the debug kernels' instance header is larger: size the windows for them
    L.ring0 = fuse ? ring_for<20, false, true, false, true>(K, sblk, qcap) : ring_for<20, false, false, false, true>(K, sblk, qcap);
    L.inst_bytes = fuse ? smem_for<20, false, true, false, true>(K, qcap, scap, L.ring0)
                        : smem_for<20, false, false, false, true>(K, qcap, scap, L.ring0);
    return L;
}
}  // namespace rsk
