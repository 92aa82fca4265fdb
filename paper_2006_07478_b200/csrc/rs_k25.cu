// rs_k25.cu — kernel instantiations for the taxi-style element-wise exit
// (RS_OP_EMIT_PAIR over byte streams, see rs_kern.cuh).
#include "rs_kern.cuh"

namespace rsk {
Launch launch_agg25(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx) {
    return launch_for<25>(K, tag, fuse, qcap, scap, sblk, ctx);
}
}  // namespace rsk
