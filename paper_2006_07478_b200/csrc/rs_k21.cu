// rs_k21.cu — kernel instantiations for aggregate op 21 (see rs_kern.cuh).
#include "rs_kern.cuh"

namespace rsk {
Launch launch_agg21(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx) {
    return launch_for<21>(K, tag, fuse, qcap, scap, sblk, ctx);
}
}  // namespace rsk
