// rs_k27.cu — kernel instantiations for RS_OP_SUM_I64_DROPS (SUM_I64 plus the
// first stage's per-region drop counts, carried by a node-generated signal).
#include "rs_kern.cuh"

namespace rsk {
Launch launch_agg27(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx) {
    return launch_for<27>(K, tag, fuse, qcap, scap, sblk, ctx);
}
}  // namespace rsk
