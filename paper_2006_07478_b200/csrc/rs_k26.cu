// rs_k26.cu — fan-out (tree topology) instantiations: K stages,
// a SPLIT node and two leaf SUM_I64 aggregates (rs_pipe.cuh "fan-out (SPL)").
#include "rs_kern.cuh"

namespace rsk {
template <int K>
using PS = Pipe<K, 26, false, false, false, false, 0, true>;

template <int K>
static void spl_launch(Launch &L, uint32_t qcap, uint32_t scap, uint32_t sblk) {
    L.main = k_pipeline<K, 26, false, false, false, false, 0, true>;
    L.ring0 = PS<K>::ring_for(sblk, qcap);
    L.inst_bytes = PS<K>::smem_bytes(qcap, scap, L.ring0);
}

Launch launch_agg26_split(int K, uint32_t qcap, uint32_t scap, uint32_t sblk) {
    Launch L;
    L.pre = k_prepass<26>;
    L.fix = k_fixup<26>;
    L.out_bytes0 = AggT<26>::bytes0;
    L.out_bytes1 = AggT<26>::bytes1;
    L.main = nullptr;
    switch (K) {
        case 0: spl_launch<0>(L, qcap, scap, sblk); break;
        case 1: spl_launch<1>(L, qcap, scap, sblk); break;
        case 2: spl_launch<2>(L, qcap, scap, sblk); break;
    }
    return L;
}
}  // namespace rsk
