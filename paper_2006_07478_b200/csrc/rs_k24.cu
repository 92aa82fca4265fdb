// rs_k24.cu — kernel instantiations for the element-wise exit (RS_OP_EMIT_VALUE, see rs_kern.cuh).
#include "rs_kern.cuh"

namespace rsk {
Launch launch_agg24(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx) {
    return launch_for<24>(K, tag, fuse, qcap, scap, sblk, ctx);
}
}  // namespace rsk
