// rs_kern.cuh — shared kernel-side definitions (parameters, prepass, fixup,
// launch tables).  Each rs_k<AGG>.cu translation unit instantiates the
// kernels of one aggregate (parallel compilation); rs.cu holds the C ABI.
//
// Hot path of Timcheck & Buhler, arXiv 2006.07478 (PAPER.md line refs "P:a-b").
//
// Execution model (§2.2, re-designed for B200):
//  * One pipeline INSTANCE per warp.  An ensemble holds up to w = 128 items
//    (4 per lane, item t of an ensemble lives in lane t%32, slot t/32), the
//    paper's SIMD width.  All scheduler state is warp-uniform.
//  * Instances compete for one parent stream with atomics: the
//    stream is cut into child-balanced CHUNKS of C children whose first region
//    is found by a prepass; an instance claims chunk k with atomicAdd.
//    Regions crossing a chunk boundary are split into parts whose partial
//    aggregates are combined by a fixup kernel (commutative monoids, A18).
//  * Nodes: 0 = ENUMERATE, 1..K = FILTER/TRANSFORM, K+1 = AGGREGATE, joined
//    by fixed-size shared-memory queues and, for the signal
//    strategy, parallel signal queues.  Queue Q0 (enumerate ->
//    first stage) is a TMA-fed ring: element blocks are bulk-copied from HBM
//    (cp.async.bulk + mbarrier) ahead of the enumerate node's emission.
//  * Scheduler: each sweep visits nodes upstream -> downstream and lets each
//    fire repeatedly (data phase, then signal phase) under the
//    full-first policy (A8): ensembles are full, or bounded by a
//    pending signal's credit, or the upstream is drained.
//  * Credit protocol exactly as P:304-327: sender rule (1)/(2) with an
//    emitted-since-last-signal counter; receiver counter with transfer (2b).
#pragma once
#include "../../include/rs.h"
#include "rs_device.cuh"

#include <cuda_runtime.h>

#include <string>
#include <type_traits>

using namespace rs;

namespace rsk {

constexpr int W = 128;              // ensemble capacity (items)
constexpr int IPL = W / 32;         // items per lane per ensemble
constexpr uint32_t SLOT = 0x80000000u;  // key bit: partial-aggregate slot instead of region id
constexpr uint32_t END_BIT = 0x80000000u;  // signal word: kind End
constexpr uint32_t USER_BIT = 0x40000000u; // signal word: a node-generated (user) signal, payload in .x
constexpr uint32_t CREDIT_MASK = 0x3fffffffu;   // signal word: the credit
constexpr int MAXK = 4;             // max FILTER/TRANSFORM stages
// RS_STRATEGY_AUTO crossover (children per region at which signal beats
// tagged) by stage count 0..4, measured on B200 (tools/crossover.py)
constexpr uint32_t AUTO_T0 = 128, AUTO_T1 = 256, AUTO_T2 = 512, AUTO_T3 = 768, AUTO_T4 = 2048;
// short-region kernel: chosen on the device iff the call's mean region length
// is below this (children per region; measured on B200, profiles/r2_tuning.txt)
constexpr uint32_t SHORT_LEN = 96;
constexpr int NSTMAX = 8;           // TMA stages of an in-place ring (sequential kernel)
constexpr int WPB = 4;              // warps (instances) per CTA (default)
constexpr int WPB_MAX = 16;         // sequential kernel: up to 16 instances per CTA (one CTA may fill an SM)

enum : uint32_t { TR_ENSEMBLE = 1, TR_BEGIN = 2, TR_END = 3 };   // trace event types (RS_FLAG_TRACE)
enum : int32_t { ERR_EMIT_FULL = 8 };      // RS_NODE_EMIT output capacity exceeded
enum : int32_t { ERR_OFFSETS = 1, ERR_WATCHDOG = 2, ERR_SIGFULL = 3, ERR_UNMATCHED = 4, ERR_QFULL = 5, ERR_LIMIT = 7 };

struct StageP {
    int32_t kind, op;
    uint32_t a, b;
    uint32_t table[8];
};

// Workspace header (first 64 bytes of the workspace).
struct WsHdr {
    uint32_t claim;      // parent-stream cursor (chunks)
    int32_t err;         // first device error
    uint32_t nchunks;
    int32_t sel;         // strategy the run uses (0 signal, 1 tagged; RS_STRATEGY_AUTO decides on the device)
    int32_t ssel;        // signal strategy: 1 = the short-region (SH) kernel runs, 0 = the general one
    uint32_t k1;         // chunks 0..k1-1 are C long, the later ones C >> TAIL_SH (see chunk_start)
    long long base0;     // align_down(offsets[0], 16 bytes)
    long long off0, offR;
};

struct KParams {
    const uint8_t *elems;
    long long n_elems;
    const long long *off;
    long long R;
    void *out0, *out1;
    void *part0, *part1;            // partial slots [2 * max_chunks]
    WsHdr *hdr;
    uint32_t *chunk_fr;             // first region of chunk k, [max_chunks + 1]
    unsigned long long *stats;      // [(K+2) * 4]
    long long max_chunks;
    uint32_t C;                     // chunk length (children)
    uint32_t tail;                  // 1: the last round of chunks is cut into C >> TAIL_SH pieces
    uint32_t nwarps;                //    (whole rounds of C per instance first; see chunk_start)
    uint32_t qcap, scap;            // queue / signal capacities (powers of 2)
    uint32_t q0_stage;              // Q0 TMA stage size in elements (sequential kernel)
    uint32_t ring0;                 // Q0 ring capacity in elements (sequential kernel; in-place: all queues)
    uint32_t esize;                 // element size in bytes (1 = u8 text, else 4)
    uint32_t flags;
    int32_t tagged;                 // 1 tagged (or hybrid: the aggregate folds by tag); -1 = AUTO (the prepass decides)
    int32_t auto_sel;               // AUTO: 0 always run; 1 = run iff hdr->sel == 0; 2 = iff hdr->sel == 1
    uint32_t auto_min_len;          // AUTO: signal iff children >= auto_min_len * regions
    int32_t short_sel;              // 0 always run; 1 = run iff hdr->ssel == 0; 2 = iff hdr->ssel == 1
    uint32_t short_len;             // prepass: ssel = 1 iff children < short_len * regions
    int32_t nst;
    StageP st[MAXK];
    const uint32_t *ctx;            // parent context, one uint32 per region (PARENT_LT), or null
    uint32_t *emit_vals;            // RS_NODE_EMIT: emitted item values [emit_cap]
    uint32_t *emit_regs;            //   and their regions [emit_cap]
    unsigned long long *emit_n;     //   items emitted (may exceed emit_cap: overflow)
    unsigned long long emit_cap;
    uint32_t *trace;                // RS_FLAG_TRACE: [0] events written, events of 8 words from word 8
    uint32_t trace_cap;             // events the buffer holds
};

// Chunk boundaries (the parent stream cut into claims).  Chunks
// 0 .. k1-1 are C children long; the rest of the stream -- less than one round
// of C per instance -- is cut into pieces of C >> TAIL_SH, so the last round
// ends within a small piece's time on every instance instead of leaving the
// instances that drew one chunk fewer idle for a whole chunk (with 8.5 chunks
// per instance: 9 rounds -> 8 5/8).  Pieces stay powers of 2 (aligned with
// power-of-2 regions).  Byte streams keep uniform chunks (k1 = all).
constexpr int TAIL_SH = 3;
__device__ __forceinline__ long long chunk_start(long long base0, long long k, long long C, long long k1) {
    return k <= k1 ? base0 + k * C : base0 + k1 * C + ((k - k1) * C >> TAIL_SH);
}

// ------------------------------------------------------------ stage ops
// isGood() / push() bodies (Fig. 5); readings A13/A14.
__device__ __forceinline__ bool stage_apply(const StageP &s, uint32_t &v) {
    switch (s.op) {
        case RS_OP_HASH_LT: return ((v * s.a) >> 24) < s.b;
        case RS_OP_LT_U32: return s.table[0] ? true : v < s.b;    // table[0]: bound == 2^32
        case RS_OP_CLASS: return (s.table[(v & 0xffu) >> 5] >> (v & 31u)) & 1u;
        case RS_OP_PARENT_LT: return true;     // signal strategy only: applied through OpLt (rs_pipe.cuh)
        case RS_OP_SCALE_F32: v = __float_as_uint(__fmul_rn(__uint_as_float(s.a), __uint_as_float(v))); return true;
        case RS_OP_AFFINE_I32: v = v * s.a + s.b; return true;
    }
    return true;
}

// --------------------------------------------------------------- prepass
// Chunk boundaries: b_0 = off0, b_k = base0 + k*C; chunk_fr[k] = first region
// r with off[r] >= b_k (lower bound over off[0..R-1]); chunk_fr[nchunks] = R.
// Also initialises partial slots to the identity and (tagged strategy) the
// outputs to the identity (A1: regions none of whose items reach the
// aggregate report identity).  The header words it depends on (claim, err,
// stats) were zeroed by a memset enqueued before it, so the VALIDATE CASes of
// any block cannot race with a reset.
// RS_STRATEGY_AUTO (P.tagged < 0): every thread derives the same decision from
// the call's own children count off[R] - off[0] (not the array bound n_elems,
// which may cover a larger stream), so no cross-block communication is needed.
template <int AGG>
__global__ void k_prepass(KParams P) {
    using AT = AggT<AGG>;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    const long long off0 = P.off[0], offR = P.off[P.R];
    const long long align = 16;  // bytes: TMA copies whole 16-byte blocks
    const long long esz = P.esize;
    const long long base0 = (off0 * esz / align) * align / esz;
    long long span = offR - base0;
    const long long C = P.C;
    long long nch = span <= 0 ? 1 : (span + C - 1) / C;
    long long k1 = nch;
    if (P.tail && span > 0) {
        const long long nw = P.nwarps > 0 ? P.nwarps : 1;
        const long long cs = C >> TAIL_SH;
        const long long kk = (span / (C * nw)) * nw;                   // whole rounds of C
        const long long n2 = kk + (span - kk * C + cs - 1) / cs;
        if (n2 <= P.max_chunks) {
            k1 = kk;
            nch = n2;
        }
    }
    bool bad = nch > P.max_chunks || offR < off0 || off0 < 0 || offR > P.n_elems;
    if (bad) nch = 0;
    bool tagged = P.tagged > 0;
    if (P.tagged < 0) tagged = !bad && (double)(offR - off0) < (double)P.auto_min_len * (double)P.R;
    if (tid == 0) {
        if (bad) atomicCAS((int *)&P.hdr->err, 0, ERR_OFFSETS);
        P.hdr->nchunks = (uint32_t)nch;
        P.hdr->k1 = (uint32_t)k1;
        P.hdr->sel = tagged ? 1 : 0;
        bool shrt = (double)(offR - off0) < (double)P.short_len * (double)P.R;
        // equal-length regions below 176 children (the sawtooth around w): the
        // short-region kernel still wins there (its segments after the first stage
        // are below w), variable lengths of that mean do not -- 64 sampled lengths
        // within 1/8 of the mean count as equal
        if (P.short_len && !shrt && (double)(offR - off0) < 176.0 * (double)P.R) {
            const double mean = (double)(offR - off0) / (double)P.R;
            long long lo = offR - off0, hi = 0;
            for (int i = 0; i < 64; ++i) {
                const long long r = (long long)i * P.R / 64;
                const long long len = P.off[r + 1] - P.off[r];
                lo = len < lo ? len : lo;
                hi = len > hi ? len : hi;
            }
            shrt = (double)(hi - lo) <= mean / 8.0;
        }
        P.hdr->ssel = shrt ? 1 : 0;
        P.hdr->base0 = base0;
        P.hdr->off0 = off0;
        P.hdr->offR = offR;
    }
    for (long long k = tid; k <= nch; k += nth) {
        uint32_t fr;
        if (k == nch) {
            fr = (uint32_t)P.R;
        } else {
            long long b = (k == 0) ? off0 : chunk_start(base0, k, C, k1);
            long long lo = 0, hi = P.R;  // first r in [0,R) with off[r] >= b, else R
            while (lo < hi) {
                long long mid = (lo + hi) >> 1;
                if (P.off[mid] < b) lo = mid + 1; else hi = mid;
            }
            fr = (uint32_t)lo;
        }
        P.chunk_fr[k] = fr;
    }
    for (long long s = tid; s < 2 * nch; s += nth) AT::store(P.part0, P.part1, (uint64_t)s, AT::id());
    if (tagged)
        for (long long r = tid; r < P.R; r += nth) AT::store(P.out0, P.out1, (uint64_t)r, AT::id());
    if (P.flags & RS_FLAG_VALIDATE) {
        for (long long r = tid; r < P.R; r += nth)
            if (P.off[r + 1] < P.off[r]) atomicCAS((int *)&P.hdr->err, 0, ERR_OFFSETS);
    }
}

// ----------------------------------------------------------------- fixup
// Combine the partial aggregates of regions split across chunks (A18): the
// chunk whose tail part starts region r walks forward over the head parts.
template <int AGG>
__global__ void k_fixup(KParams P) {
    using AT = AggT<AGG>;
    const WsHdr *H = P.hdr;
    const long long nch = H->nchunks;
    const long long base0 = H->base0, offR = H->offR, k1 = H->k1;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k + 1 < nch;
         k += (long long)gridDim.x * blockDim.x) {
        uint32_t f0 = P.chunk_fr[k], f1 = P.chunk_fr[k + 1];
        if (f1 <= f0) continue;                       // no region starts in chunk k
        long long r = (long long)f1 - 1;               // last region starting in chunk k
        long long end_k = chunk_start(base0, k + 1, P.C, k1);
        long long rend = P.off[r + 1];
        if (rend <= end_k) continue;                   // not split
        typename AT::A acc = AT::load(P.part0, P.part1, (uint64_t)(2 * k + 1));
        for (long long j = k + 1; j < nch; ++j) {
            acc = AT::comb(acc, AT::load(P.part0, P.part1, (uint64_t)(2 * j)));
            long long end_j = chunk_start(base0, j + 1, P.C, k1);
            if (end_j > offR) end_j = offR;
            if (rend <= end_j) break;
        }
        AT::store(P.out0, P.out1, (uint64_t)r, acc);
    }
}

// ---------------------------------------------------------- the pipeline
#ifndef RS_HOST_ONLY
#include "rs_pipe.cuh"
#endif

using KernelFn = void (*)(KParams);

struct Launch {
    KernelFn main;
    void (*pre)(KParams);
    void (*fix)(KParams);
    uint32_t inst_bytes;
    uint32_t ring0;                 // Q0 ring capacity (elements) of the sequential kernel
    int out_bytes0, out_bytes1;
};

// rs_last_error()'s thread-local message (rs.cu), shared by the other host units.
void set_last_error(const std::string &m);

// One per aggregate, defined in rs_k<AGG>.cu.
Launch launch_agg20(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx);
Launch launch_agg21(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx);
Launch launch_agg22(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx);
Launch launch_agg23(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx);
Launch launch_agg24(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx);
Launch launch_agg25(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx);
// RS_FLAG_TRACE instantiations (SUM_I64, signal strategy; defined in rs_k20t.cu)
Launch launch_agg20_trace(int K, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk);
// RS_STRATEGY_HYBRID instantiations (edges >= hyb carry tags; rs_k20h.cu, rs_k25h.cu)
Launch launch_agg20_hybrid(int K, bool fuse, int hyb, uint32_t qcap, uint32_t scap, uint32_t sblk);
Launch launch_agg25_hybrid(int K, bool fuse, int hyb, uint32_t qcap, uint32_t scap, uint32_t sblk);
// fan-out (SPLIT + two leaf SUM_I64 aggregates; rs_k26.cu), K <= 2 stages before the split
Launch launch_agg26_split(int K, uint32_t qcap, uint32_t scap, uint32_t sblk);
// short-region (SH) kernels: SUM_I64 / COUNT_MIN_U32, signal strategy, fused aggregate, K >= 1
// stages, with their own ring / stage / signal-queue geometry (rs_k20s.cu);
// main == nullptr where not built
Launch short_launch_agg20(int K, uint32_t qcap, uint32_t scap, uint32_t sblk);
Launch short_launch_agg22(int K, uint32_t qcap, uint32_t scap, uint32_t sblk);   // COUNT_MIN_U32 (rs_k22s.cu)
// SUM_I64 + stage-1 drop counts delivered by a node-generated signal (rs_k27.cu)
Launch launch_agg27(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx);

#ifndef RS_HOST_ONLY
// Hybrid kernels: K stages, edges >= hyb tagged (1 <= hyb <= the aggregating
// node's input edge: K - 1 fused, K unfused).
template <int AGG, bool FUSE, int K>
KernelFn pick_hyb_k(int hyb) {
    if constexpr (K >= 1) {
        if (hyb == 1 && (!FUSE || K >= 2)) return k_pipeline<K, AGG, false, FUSE, false, false, 1>;
    }
    if constexpr (K >= 2) {
        if (hyb == 2 && (!FUSE || K >= 3)) return k_pipeline<K, AGG, false, FUSE, false, false, 2>;
    }
    if constexpr (K >= 3) {
        if (hyb == 3 && (!FUSE || K >= 4)) return k_pipeline<K, AGG, false, FUSE, false, false, 3>;
    }
    if constexpr (K >= 4 && !FUSE) {
        if (hyb == 4) return k_pipeline<K, AGG, false, FUSE, false, false, 4>;
    }
    return nullptr;
}
template <int AGG, bool FUSE>
KernelFn pick_hyb(int K, int hyb) {
    switch (K) {
        case 1: return pick_hyb_k<AGG, FUSE, 1>(hyb);
        case 2: return pick_hyb_k<AGG, FUSE, 2>(hyb);
        case 3: return pick_hyb_k<AGG, FUSE, 3>(hyb);
        case 4: return pick_hyb_k<AGG, FUSE, 4>(hyb);
    }
    return nullptr;
}
// ring and shared-memory size of a hybrid kernel (tag ring + signal rings)
template <int AGG, bool FUSE, int K, int HYB>
void hyb_sizes(uint32_t sblk, uint32_t qcap, uint32_t scap, uint32_t &ring, uint32_t &bytes) {
    using PP = Pipe<K, AGG, false, FUSE, false, false, HYB>;
    ring = PP::ring_for(sblk, qcap);
    bytes = PP::smem_bytes(qcap, scap, ring);
}
template <int AGG>
Launch launch_hybrid(int K, bool fuse, int hyb, uint32_t qcap, uint32_t scap, uint32_t sblk) {
    Launch L;
    L.pre = k_prepass<AGG>;
    L.fix = k_fixup<AGG>;
    L.out_bytes0 = AggT<AGG>::bytes0;
    L.out_bytes1 = AggT<AGG>::bytes1;
    L.main = fuse ? pick_hyb<AGG, true>(K, hyb) : pick_hyb<AGG, false>(K, hyb);
    // the hybrid instance holds the tag ring and the signal rings
    uint32_t ring = 0, bytes = 0;
    auto sz = [&](auto kk, auto hh) {
        constexpr int KK = decltype(kk)::value, HH = decltype(hh)::value;
        if (fuse) hyb_sizes<AGG, true, KK, HH>(sblk, qcap, scap, ring, bytes);
        else hyb_sizes<AGG, false, KK, HH>(sblk, qcap, scap, ring, bytes);
    };
    using std::integral_constant;
    switch (K * 8 + hyb) {
        case 1 * 8 + 1: sz(integral_constant<int, 1>{}, integral_constant<int, 1>{}); break;
        case 2 * 8 + 1: sz(integral_constant<int, 2>{}, integral_constant<int, 1>{}); break;
        case 2 * 8 + 2: sz(integral_constant<int, 2>{}, integral_constant<int, 2>{}); break;
        case 3 * 8 + 1: sz(integral_constant<int, 3>{}, integral_constant<int, 1>{}); break;
        case 3 * 8 + 2: sz(integral_constant<int, 3>{}, integral_constant<int, 2>{}); break;
        case 3 * 8 + 3: sz(integral_constant<int, 3>{}, integral_constant<int, 3>{}); break;
        case 4 * 8 + 1: sz(integral_constant<int, 4>{}, integral_constant<int, 1>{}); break;
        case 4 * 8 + 2: sz(integral_constant<int, 4>{}, integral_constant<int, 2>{}); break;
        case 4 * 8 + 3: sz(integral_constant<int, 4>{}, integral_constant<int, 3>{}); break;
        case 4 * 8 + 4: sz(integral_constant<int, 4>{}, integral_constant<int, 4>{}); break;
    }
    L.ring0 = ring;
    L.inst_bytes = bytes;
    return L;
}

template <int AGG, bool TAG, bool FUSE, bool CTX = false, bool TR = false>
KernelFn pick_k(int K) {
    switch (K) {
        case 0: return k_pipeline<0, AGG, TAG, false, CTX, TR>;      // nothing to fuse
        case 1: return k_pipeline<1, AGG, TAG, FUSE, CTX, TR>;
        case 2: return k_pipeline<2, AGG, TAG, FUSE, CTX, TR>;
        case 3: return k_pipeline<3, AGG, TAG, FUSE, CTX, TR>;
        default: return k_pipeline<4, AGG, TAG, FUSE, CTX, TR>;
    }
}

template <int AGG, bool TAG, bool FUSE, bool CTX = false, bool TR = false>
uint32_t ring_for(int K, uint32_t sblk, uint32_t qcap) {
    switch (K) {
        case 0: return Pipe<0, AGG, TAG, false, CTX, TR>::ring_for(sblk, qcap);
        case 1: return Pipe<1, AGG, TAG, FUSE, CTX, TR>::ring_for(sblk, qcap);
        case 2: return Pipe<2, AGG, TAG, FUSE, CTX, TR>::ring_for(sblk, qcap);
        case 3: return Pipe<3, AGG, TAG, FUSE, CTX, TR>::ring_for(sblk, qcap);
        default: return Pipe<4, AGG, TAG, FUSE, CTX, TR>::ring_for(sblk, qcap);
    }
}

// shared memory of one instance (the kernel's per-warp window; it must be the
// same instantiation as the kernel launched: the debug kernels' header differs)
template <int AGG, bool TAG, bool FUSE, bool CTX = false, bool TR = false>
uint32_t smem_for(int K, uint32_t qcap, uint32_t scap, uint32_t ring) {
    switch (K) {
        case 0: return Pipe<0, AGG, TAG, false, CTX, TR>::smem_bytes(qcap, scap, ring);
        case 1: return Pipe<1, AGG, TAG, FUSE, CTX, TR>::smem_bytes(qcap, scap, ring);
        case 2: return Pipe<2, AGG, TAG, FUSE, CTX, TR>::smem_bytes(qcap, scap, ring);
        case 3: return Pipe<3, AGG, TAG, FUSE, CTX, TR>::smem_bytes(qcap, scap, ring);
        default: return Pipe<4, AGG, TAG, FUSE, CTX, TR>::smem_bytes(qcap, scap, ring);
    }
}


template <int AGG>
Launch launch_for(int K, bool tag, bool fuse, uint32_t qcap, uint32_t scap, uint32_t sblk, bool ctx = false) {
    Launch L;
    if constexpr (AGG != 23 && AGG != 24 && AGG != 25 && AGG != 27) {      // per-lane context strategy: 4-byte (in-place) element streams
        if (ctx) {
            L = launch_for<AGG>(K, false, fuse, qcap, scap, sblk, false);
            L.main = fuse ? pick_k<AGG, false, true, true>(K) : pick_k<AGG, false, false, true>(K);
            L.ring0 = fuse ? ring_for<AGG, false, true, true>(K, sblk, qcap) : ring_for<AGG, false, false, true>(K, sblk, qcap);
            L.inst_bytes = fuse ? smem_for<AGG, false, true, true>(K, qcap, scap, L.ring0)
                                : smem_for<AGG, false, false, true>(K, qcap, scap, L.ring0);
            return L;
        }
    }
    L.main = tag ? (fuse ? pick_k<AGG, true, true>(K) : pick_k<AGG, true, false>(K))
                 : (fuse ? pick_k<AGG, false, true>(K) : pick_k<AGG, false, false>(K));
    L.pre = k_prepass<AGG>;
    L.fix = k_fixup<AGG>;
    L.ring0 = tag ? (fuse ? ring_for<AGG, true, true>(K, sblk, qcap) : ring_for<AGG, true, false>(K, sblk, qcap))
                  : (fuse ? ring_for<AGG, false, true>(K, sblk, qcap) : ring_for<AGG, false, false>(K, sblk, qcap));
    const uint32_t r = L.ring0;
    L.inst_bytes = tag ? (fuse ? smem_for<AGG, true, true>(K, qcap, scap, r) : smem_for<AGG, true, false>(K, qcap, scap, r))
                       : (fuse ? smem_for<AGG, false, true>(K, qcap, scap, r) : smem_for<AGG, false, false>(K, qcap, scap, r));
    L.out_bytes0 = AggT<AGG>::bytes0;
    L.out_bytes1 = AggT<AGG>::bytes1;
    return L;
}
#endif  // RS_HOST_ONLY

}  // namespace rsk
