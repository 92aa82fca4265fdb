// rs_k25h.cu — RS_STRATEGY_HYBRID instantiations for aggregate op 25
// (per-stage strategy: signals up to a stage, tags from it on; rs_pipe.cuh HYB).
#include "rs_kern.cuh"

namespace rsk {
Launch launch_agg25_hybrid(int K, bool fuse, int hyb, uint32_t qcap, uint32_t scap, uint32_t sblk) {
    return launch_hybrid<25>(K, fuse, hyb, qcap, scap, sblk);
}
}  // namespace rsk
