// rs_k23.cu — kernel instantiations for aggregate op 23 (see rs_kern.cuh).
#include "rs_kern.cuh"

namespace rsk {
Launch launch_agg23(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx) {
    return launch_for<23>(K, tag, fuse, qcap, scap, sblk, ctx);
}
}  // namespace rsk
