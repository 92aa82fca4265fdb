// rs.cu — B200 (sm_100a) persistent pipeline kernels + the C ABI of include/rs.h.
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
#include "../../include/rs.h"
#include "rs_device.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

using namespace rs;

namespace {

constexpr int W = 128;              // ensemble capacity (items)
constexpr int IPL = W / 32;         // items per lane per ensemble
constexpr uint32_t SLOT = 0x80000000u;  // key bit: partial-aggregate slot instead of region id
constexpr uint32_t END_BIT = 0x80000000u;  // signal word: kind End
constexpr int MAXK = 4;             // max FILTER/TRANSFORM stages
constexpr int NST = 4;              // TMA stages in the Q0 ring
constexpr int WPB = 4;              // warps (instances) per CTA

enum : int32_t { ERR_OFFSETS = 1, ERR_WATCHDOG = 2, ERR_SIGFULL = 3, ERR_UNMATCHED = 4, ERR_QFULL = 5 };

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
    uint32_t pad_;
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
    uint32_t qcap, scap;            // queue / signal capacities (powers of 2)
    uint32_t flags;
    int32_t tagged;
    int32_t nst;
    StageP st[MAXK];
};

// ------------------------------------------------------------ stage ops
// isGood() / push() bodies (Fig. 5); readings A13/A14.
__device__ __forceinline__ bool stage_apply(const StageP &s, uint32_t &v) {
    switch (s.op) {
        case RS_OP_HASH_LT: return ((v * s.a) >> 24) < s.b;
        case RS_OP_LT_U32: return s.table[0] ? true : v < s.b;    // table[0]: bound == 2^32
        case RS_OP_CLASS: return (s.table[(v & 0xffu) >> 5] >> (v & 31u)) & 1u;
        case RS_OP_SCALE_F32: v = __float_as_uint(__fmul_rn(__uint_as_float(s.a), __uint_as_float(v))); return true;
        case RS_OP_AFFINE_I32: v = v * s.a + s.b; return true;
    }
    return true;
}

// --------------------------------------------------------------- prepass
// Chunk boundaries: b_0 = off0, b_k = base0 + k*C; chunk_fr[k] = first region
// r with off[r] >= b_k (lower bound over off[0..R-1]); chunk_fr[nchunks] = R.
// Also resets the claim counter / error word / stats, initialises partial
// slots to the identity and (tagged strategy) the outputs to the identity
// (A1: regions none of whose items reach the aggregate report identity).
template <int AGG>
__global__ void k_prepass(KParams P, int n_stats) {
    using AT = AggT<AGG>;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    const long long off0 = P.off[0], offR = P.off[P.R];
    const long long align = 16;  // bytes; element size 4 -> 4 elements
    const long long esz = 4;
    const long long base0 = (off0 * esz / align) * align / esz;
    long long span = offR - base0;
    long long nch = span <= 0 ? 1 : (span + P.C - 1) / P.C;
    bool bad = nch > P.max_chunks || offR < off0 || off0 < 0 || offR > P.n_elems;
    if (bad) nch = 0;
    if (tid == 0) {
        P.hdr->claim = 0;
        P.hdr->err = bad ? ERR_OFFSETS : 0;
        P.hdr->nchunks = (uint32_t)nch;
        P.hdr->base0 = base0;
        P.hdr->off0 = off0;
        P.hdr->offR = offR;
    }
    for (long long i = tid; i < n_stats; i += nth) P.stats[i] = 0ull;
    for (long long k = tid; k <= nch; k += nth) {
        uint32_t fr;
        if (k == nch) {
            fr = (uint32_t)P.R;
        } else {
            long long b = (k == 0) ? off0 : base0 + k * (long long)P.C;
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
    if (P.tagged)
        for (long long r = tid; r < P.R; r += nth) AT::store(P.out0, P.out1, (uint64_t)r, AT::id());
    if (P.flags & RS_FLAG_VALIDATE) {
        for (long long r = tid; r < P.R; r += nth)
            if (P.off[r + 1] < P.off[r]) atomicCAS((int *)&P.hdr->err, 0, ERR_OFFSETS);
        if (tid == 0 && (offR > P.n_elems || off0 < 0)) atomicCAS((int *)&P.hdr->err, 0, ERR_OFFSETS);
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
    const long long base0 = H->base0, offR = H->offR;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k + 1 < nch;
         k += (long long)gridDim.x * blockDim.x) {
        uint32_t f0 = P.chunk_fr[k], f1 = P.chunk_fr[k + 1];
        if (f1 <= f0) continue;                       // no region starts in chunk k
        long long r = (long long)f1 - 1;               // last region starting in chunk k
        long long end_k = base0 + (k + 1) * (long long)P.C;
        long long rend = P.off[r + 1];
        if (rend <= end_k) continue;                   // not split
        typename AT::A acc = AT::load(P.part0, P.part1, (uint64_t)(2 * k + 1));
        for (long long j = k + 1; j < nch; ++j) {
            acc = AT::comb(acc, AT::load(P.part0, P.part1, (uint64_t)(2 * j)));
            long long end_j = base0 + (j + 1) * (long long)P.C;
            if (end_j > offR) end_j = offR;
            if (rend <= end_j) break;
        }
        AT::store(P.out0, P.out1, (uint64_t)r, acc);
    }
}

// ---------------------------------------------------------- the pipeline
template <int K, int AGG, bool TAG>
struct Pipe {
    using AT = AggT<AGG>;
    using A = typename AT::A;
    static constexpr int SBLK = TAG ? 256 : 512;     // elements per TMA stage
    static constexpr int RING0 = NST * SBLK;         // Q0 ring capacity (items)

    const KParams &P;
    const int lane;
    // shared-memory rings
    uint64_t *bar;                 // [NST]
    uint32_t *q[K + 1];            // data rings: q[0] = Q0 (RING0), q[e] = Q_e (qcap)
    uint32_t *t[K + 1];            // tag rings (tagged strategy)
    uint2 *s[K + 1];               // signal rings {key, credit | END_BIT}
    uint32_t qmask, smask, qcap, scap;

    // edge e : node e -> node e+1
    uint32_t qh[K + 1], qt[K + 1];     // data queue head/tail (monotone positions)
    uint32_t sh[K + 1], stl[K + 1];    // signal queue head/tail
    uint32_t sent[K + 1];              // sender: items emitted since last signal
    uint32_t cur[K + 1];               // receiver current credit counter
    bool xfer[K + 1];                  // head signal's credit already moved into cur
    // per-node stats: ensembles, full ensembles, items, signals
    uint32_t nd[K + 2], nf[K + 2], ni[K + 2], ns[K + 2];

    // chunk FIFO (F0 = being enumerated, F1 = staged next)
    int32_t fk[2];
    long long fbeg[2], fend[2];
    uint32_t fpos[2], ffr0[2], ffr1[2];
    bool fhead[2];
    bool claims_done;
    uint32_t stg_j, landed_j;
    // enumerate cursor within F0
    uint32_t pidx;
    bool begun;
    bool enum_done;
    // aggregate state
    A acc;             // per-lane partial accumulator (signal: current region; tagged: carry key)
    uint32_t akey;     // signal: open region key; tagged: carry key (0xffffffff = none)
    A carry;           // tagged: uniform carried partial
    long long base0, offR;
    uint32_t nchunks;

    __device__ Pipe(const KParams &p, uint8_t *smem, int lane_) : P(p), lane(lane_) {
        qcap = P.qcap;
        scap = P.scap;
        qmask = qcap - 1;
        smask = scap - 1;
        uint8_t *ptr = smem;
        bar = reinterpret_cast<uint64_t *>(ptr);
        ptr += 128;
        q[0] = reinterpret_cast<uint32_t *>(ptr);
        ptr += RING0 * 4;
        if (TAG) { t[0] = reinterpret_cast<uint32_t *>(ptr); ptr += RING0 * 4; } else t[0] = nullptr;
#pragma unroll
        for (int e = 1; e <= K; ++e) {
            q[e] = reinterpret_cast<uint32_t *>(ptr);
            ptr += qcap * 4;
            if (TAG) { t[e] = reinterpret_cast<uint32_t *>(ptr); ptr += qcap * 4; } else t[e] = nullptr;
        }
#pragma unroll
        for (int e = 0; e <= K; ++e) {
            s[e] = reinterpret_cast<uint2 *>(ptr);
            if (!TAG) ptr += scap * 8;
        }
#pragma unroll
        for (int e = 0; e <= K; ++e) { qh[e] = qt[e] = sh[e] = stl[e] = sent[e] = cur[e] = 0; xfer[e] = false; }
#pragma unroll
        for (int n = 0; n < K + 2; ++n) nd[n] = nf[n] = ni[n] = ns[n] = 0;
        fk[0] = fk[1] = -1;
        claims_done = false;
        stg_j = landed_j = 0;
        pidx = 0;
        begun = false;
        enum_done = false;
        acc = AT::id();
        carry = AT::id();
        akey = 0xffffffffu;
        base0 = P.hdr->base0;
        offR = P.hdr->offR;
        nchunks = P.hdr->nchunks;
    }

    __host__ __device__ static constexpr uint32_t smem_bytes(uint32_t qcap, uint32_t scap) {
        return 128 + RING0 * 4 * (TAG ? 2 : 1) + K * qcap * 4 * (TAG ? 2 : 1) + (TAG ? 0 : (K + 1) * scap * 8);
    }

    __device__ __forceinline__ uint32_t bcast(uint32_t v) const { return __shfl_sync(kFull, v, 0); }

    // ---------------------------------------------------------- chunks
    __device__ void load_chunk(int f, int32_t k, uint32_t pos) {
        fk[f] = k;
        long long b = (k == 0) ? P.hdr->off0 : base0 + (long long)k * P.C;
        long long e = base0 + (long long)(k + 1) * P.C;
        if (e > offR) e = offR;
        fbeg[f] = b;
        fend[f] = e;
        fpos[f] = pos;
        ffr0[f] = P.chunk_fr[k];
        ffr1[f] = P.chunk_fr[k + 1];
        fhead[f] = (k > 0) && (P.off[ffr0[f]] > b);
    }
    __device__ __forceinline__ uint32_t flen(int f) const { return (uint32_t)(fend[f] - fbeg[f]); }
    __device__ __forceinline__ uint32_t nparts0() const { return (fhead[0] ? 1u : 0u) + (ffr1[0] - ffr0[0]); }

    // Claim the next chunk of the parent stream (atomics, no locks).
    __device__ int32_t claim() {
        uint32_t k = 0;
        if (lane == 0) k = atomicAdd(&P.hdr->claim, 1u);
        k = bcast(k);
        return k < nchunks ? (int32_t)k : -1;
    }

    // Issue TMA stage j from FIFO entry f.
    __device__ void issue_stage(int f) {
        const uint32_t j = stg_j;
        const uint32_t p0 = j * SBLK;
        const uint32_t pend = fpos[f] + flen(f);
        const uint32_t n = min((uint32_t)SBLK, pend - p0);
        const long long src = fbeg[f] + (long long)p0 - (long long)fpos[f];   // 4-element aligned
        uint32_t *dst = q[0] + (p0 & (RING0 - 1));
        uint64_t *b = &bar[j % NST];
        const long long lim = (P.n_elems - src) & ~3ll;     // whole 16-byte blocks inside the array
        const uint32_t ntma = (uint32_t)min((long long)((n + 3u) & ~3u), lim);
        // tail elements that a 16-byte copy cannot reach without overrunning n_elems
        const int tail = (int)n - (int)ntma;
        if (tail > 0 && lane < tail) {
            const uint32_t *g = reinterpret_cast<const uint32_t *>(P.elems) + src + ntma + lane;
            dst[ntma + lane] = __ldg(g);
        }
        __syncwarp();
        if (lane == 0) {
            fence_proxy_async();
            if (ntma) {
                mbar_arrive_expect_tx(b, ntma * 4u);
                tma_load_1d(dst, P.elems + src * 4, ntma * 4u, b);
            } else {
                mbar_arrive(b);
            }
        }
        stg_j = j + 1;
    }

    // Keep the Q0 ring full: prefetch element blocks ahead of the enumerate node.
    __device__ void refill() {
        for (;;) {
            if ((stg_j + 1) * (uint32_t)SBLK > qh[0] + RING0) return;   // ring slot still in use
            const uint32_t sp = stg_j * SBLK;
            int f = -1;
            if (fk[0] >= 0 && sp < fpos[0] + flen(0)) f = 0;
            else if (fk[1] >= 0 && sp < fpos[1] + flen(1)) f = 1;
            if (f < 0) {
                if (fk[1] >= 0 || claims_done) return;
                int32_t k = claim();
                if (k < 0) { claims_done = true; return; }
                if (fk[0] < 0) {
                    uint32_t pos = (k == 0) ? (uint32_t)(P.hdr->off0 - base0) : sp;
                    if (k == 0 && stg_j == 0) { qh[0] = qt[0] = pos; }
                    load_chunk(0, k, pos);
                    pidx = 0;
                    begun = false;
                } else {
                    load_chunk(1, k, fpos[0] + flen(0));
                }
                continue;
            }
            issue_stage(f);
        }
    }

    // ------------------------------------------------------ enumerate
    // Part q of chunk F0: [start, end) elements and its key (region id, or a
    // partial slot for the chunk's head part / a tail part crossing the chunk end).
    __device__ void part_info(uint32_t qi, bool valid, long long &ps, long long &pe, uint32_t &key) const {
        ps = pe = fend[0];
        key = 0;
        if (!valid) return;
        if (fhead[0] && qi == 0) {
            ps = fbeg[0];
            long long e = P.off[ffr0[0]];
            pe = e < fend[0] ? e : fend[0];
            key = SLOT | (uint32_t)(2 * fk[0]);
        } else {
            uint32_t r = ffr0[0] + qi - (fhead[0] ? 1u : 0u);
            ps = P.off[r];
            long long e = P.off[r + 1];
            if (e > fend[0]) { pe = fend[0]; key = SLOT | (uint32_t)(2 * fk[0] + 1); }
            else { pe = e; key = r; }
        }
    }

    // Sender rule for one signal on edge e given the queue state at emission
    // (P:304-312): S empty -> |Q|; otherwise items emitted since the tail signal.
    __device__ __forceinline__ void push_signal(int e, uint32_t key, bool end, uint32_t credit_rule2) {
        uint32_t credit = (sh[e] == stl[e]) ? (qt[e] - qh[e]) : credit_rule2;
        if (lane == 0) s[e][stl[e] & smask] = make_uint2(key, credit | (end ? END_BIT : 0u));
        stl[e] += 1;
        sent[e] = 0;
    }

    // One enumerate firing: emit element indices (as staged element values)
    // and Begin/End signals of F0's parts as far as staged data and signal
    // space allow (resumable mid-region).
    __device__ bool enumerate() {
        bool prog = false;
        refill();
        for (;;) {
            if (fk[0] < 0) {
                if (fk[1] >= 0) { shift(); continue; }
                if (claims_done) enum_done = true;
                return prog;
            }
            const uint32_t np = nparts0();
            if (pidx >= np) {
                // chunk fully enumerated; its items are all emitted
                shift();
                refill();
                prog = true;
                continue;
            }
            const uint32_t lim_pos = min(stg_j * (uint32_t)SBLK, fpos[0] + flen(0));
            const uint32_t avail = lim_pos - qt[0];
            const long long e_next = fbeg[0] + (long long)(qt[0] - fpos[0]);
            // batch of up to 32 parts, one per lane
            const uint32_t qi = pidx + lane;
            long long ps, pe;
            uint32_t key;
            part_info(qi, qi < np, ps, pe, key);
            if (lane == 0 && ps < e_next) ps = e_next;     // resume inside part pidx
            uint32_t cnt = (uint32_t)(pe - ps);
            // inclusive scan of counts (and signals) across the batch
            uint32_t cum = cnt;
            uint32_t sig = TAG ? 0u : ((lane == 0 && begun) ? 1u : 2u);
            uint32_t scum = sig;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                uint32_t o = __shfl_up_sync(kFull, cum, d);
                uint32_t so = __shfl_up_sync(kFull, scum, d);
                if (lane >= d) { cum += o; scum += so; }
            }
            const uint32_t sfree = TAG ? 0xffffffffu : scap - (stl[0] - sh[0]);
            const bool fits = (qi < np) && (cum <= avail) && (scum <= sfree);
            const uint32_t m = __popc(__ballot_sync(kFull, fits));
            if (m > 0) {
                const uint32_t tot = __shfl_sync(kFull, cum, m - 1);
                if constexpr (!TAG) {
                    // Signals of parts 0..m-1: Begin_i, End_i in stream order.
                    const bool empty_at_start = (sh[0] == stl[0]);
                    const uint32_t qlen0 = qt[0] - qh[0];
                    const uint32_t sexcl = scum - sig;
                    if (lane < (int)m) {
                        uint32_t slot = stl[0] + sexcl;
                        if (!(lane == 0 && begun)) {
                            // Begin_i: first signal of the batch uses rule (1) if S was empty,
                            // else rule (2) with items since the previous signal (sent[0]);
                            // later Begins follow an End directly: credit 0.
                            uint32_t c = (lane == 0) ? (empty_at_start ? qlen0 : sent[0]) : 0u;
                            s[0][slot & smask] = make_uint2(key, c);
                            slot++;
                        }
                        // End_i: items of part i since its Begin (rule 2), or rule (1) when
                        // part 0 began earlier and S has since been drained by the receiver.
                        uint32_t c;
                        if (lane == 0 && begun) c = empty_at_start ? (qlen0 + cnt) : (sent[0] + cnt);
                        else c = cnt;
                        s[0][slot & smask] = make_uint2(key, c | END_BIT);
                    }
                    stl[0] += __shfl_sync(kFull, scum, m - 1);
                    ns[0] += __shfl_sync(kFull, scum, m - 1);
                    sent[0] = 0;
                } else {
                    write_tags(m, cum, cnt, key, tot);
                }
                qt[0] += tot;
                ni[0] += tot;
                pidx += m;
                begun = false;
                prog = true;
                __syncwarp();
                continue;
            }
            // Part pidx does not fit whole: emit what we can of it (resumable).
            const uint32_t key0 = __shfl_sync(kFull, key, 0);
            const uint32_t cnt0 = __shfl_sync(kFull, cnt, 0);
            bool did = false;
            if constexpr (!TAG) {
                if (!begun) {
                    if (scap - (stl[0] - sh[0]) == 0) return prog;
                    push_signal(0, key0, false, sent[0]);
                    ns[0]++;
                    begun = true;
                    did = true;
                }
            }
            const uint32_t k = min(avail, cnt0);
            if (k > 0) {
                if constexpr (TAG) write_tags_uniform(key0, k);
                qt[0] += k;
                sent[0] += k;
                ni[0] += k;
                did = true;
            }
            if constexpr (!TAG) {
                if (k == cnt0 && scap - (stl[0] - sh[0]) > 0) {
                    push_signal(0, key0, true, sent[0]);
                    ns[0]++;
                    pidx++;
                    begun = false;
                    did = true;
                }
            } else {
                if (k == cnt0) { pidx++; did = true; }
            }
            __syncwarp();
            prog |= did;
            if (!did) return prog;
        }
    }

    __device__ void shift() {
        fk[0] = fk[1];
        fbeg[0] = fbeg[1];
        fend[0] = fend[1];
        fpos[0] = fpos[1];
        ffr0[0] = ffr0[1];
        ffr1[0] = ffr1[1];
        fhead[0] = fhead[1];
        fk[1] = -1;
        pidx = 0;
        begun = false;
    }

    // Tagged enumerate: every emitted item gets its parent's key
    // (P:258-261).  Positions qt[0] .. qt[0]+tot-1 belong to parts
    // 0..m-1 of this batch (lane i holds part i's inclusive end `cum`).
    __device__ void write_tags(uint32_t m, uint32_t cum, uint32_t cnt, uint32_t key, uint32_t tot) {
        if (m == 1 || __shfl_sync(kFull, cnt, 0) == tot) {
            write_tags_uniform(__shfl_sync(kFull, key, 0), tot);
            return;
        }
        const uint32_t excl = cum - cnt;
        for (uint32_t base = 0; base < tot; base += 32) {
            const uint32_t rel = base + lane;
            // largest part i < m with excl_i <= rel (binary search over lanes)
            int lo = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1) {
                int cand = lo + step;
                uint32_t ex = __shfl_sync(kFull, excl, cand < 32 ? cand : 31);
                if (cand < (int)m && ex <= rel) lo = cand;
            }
            const uint32_t k = __shfl_sync(kFull, key, lo);
            if (rel < tot) t[0][(qt[0] + rel) & (RING0 - 1)] = k;
        }
    }
    __device__ void write_tags_uniform(uint32_t key, uint32_t k) {
        for (uint32_t i = lane; i < k; i += 32) t[0][(qt[0] + i) & (RING0 - 1)] = key;
    }

    // ---------------------------------------------------------- stages
    __device__ __forceinline__ uint32_t landed_pos() {
        while (landed_j < stg_j && mbar_test(&bar[landed_j % NST], (landed_j / NST) & 1u)) landed_j++;
        return landed_j * (uint32_t)SBLK;
    }

    // Receiver admissible count on edge e, applying rule (2b).
    __device__ __forceinline__ uint32_t admissible(int e, bool &spend) {
        spend = sh[e] != stl[e];
        const uint32_t ql = qt[e] - qh[e];
        if (!spend) return ql;
        if (cur[e] == 0 && !xfer[e]) {
            uint32_t c = s[e][sh[e] & smask].y & ~END_BIT;
            if (c > 0) { cur[e] = c; xfer[e] = true; }
        }
        return min(ql, cur[e]);
    }

    // Fire node n (1..K+1) repeatedly while it can make progress.
    template <int n>
    __device__ bool fire(bool drained) {
        constexpr int ei = n - 1;          // input edge
        constexpr bool AGGN = (n == K + 1);
        const uint32_t imask = (ei == 0) ? (RING0 - 1) : qmask;
        uint32_t *in = q[ei];
        uint32_t *tin = t[ei];
        bool prog = false;
        uint32_t ready_lim = 0;
        if (ei == 0) ready_lim = landed_pos();
        for (;;) {
            bool spend;
            const uint32_t a = admissible(ei, spend);
            uint32_t ar = a;
            if (ei == 0) {
                // only items whose TMA stage has landed may be read
                if ((int)(ready_lim - qh[0]) < (int)ar) ready_lim = landed_pos();
                const int rdy = (int)(ready_lim - qh[0]);
                ar = rdy <= 0 ? 0u : min(ar, (uint32_t)rdy);
            }
            uint32_t space = 0xffffffffu;
            if constexpr (!AGGN) space = qcap - (qt[n] - qh[n]);
            uint32_t e = min(min(ar, (uint32_t)W), space);
            bool ok = e > 0;
            if (ok && e < (uint32_t)W) {
                const bool bounded = spend && e == cur[ei];
                const bool dr = drained && e == a;
                ok = bounded || dr;
            }
            if (ok) {
                run_ensemble<n>(in, tin, imask, qh[ei], e);
                qh[ei] += e;
                if (spend) cur[ei] -= e;
                nd[n]++;
                ni[n] += e;
                if (e == (uint32_t)W) nf[n]++;
                prog = true;
                continue;
            }
            // signal phase: only with the counter at 0
            if constexpr (TAG) break;
            if (!spend || cur[ei] != 0) break;
            const uint2 hs = s[ei][sh[ei] & smask];
            if (!xfer[ei] && (hs.y & ~END_BIT) > 0) {
                cur[ei] = hs.y & ~END_BIT;
                xfer[ei] = true;
                continue;
            }
            if constexpr (!AGGN) {
                if (scap - (stl[n] - sh[n]) == 0) break;
            }
            sh[ei]++;
            xfer[ei] = false;
            ns[n]++;
            prog = true;
            const bool is_end = (hs.y & END_BIT) != 0;
            if constexpr (AGGN) {
                if (!is_end) {               // a::begin: acc = identity
                    acc = AT::id();
                    akey = hs.x;
                } else {                     // a::end: push(acc)
                    A v = warp_reduce<AT>(acc);
                    if (lane == 0) store_key(hs.x, v);
                    acc = AT::id();
                    akey = 0xffffffffu;
                }
            } else {
                push_signal(n, hs.x, is_end, sent[n]);   // forwarded with a fresh credit
            }
        }
        __syncwarp();
        return prog;
    }

    __device__ __forceinline__ void store_key(uint32_t key, A v) {
        if (key & SLOT) AT::store(P.part0, P.part1, key & ~SLOT, v);
        else AT::store(P.out0, P.out1, key, v);
    }

    template <int n>
    __device__ __forceinline__ void run_ensemble(const uint32_t *in, const uint32_t *tin, uint32_t imask,
                                                 uint32_t h, uint32_t e) {
        if constexpr (n == K + 1) {
            if constexpr (!TAG) {
#pragma unroll
                for (int j = 0; j < IPL; ++j) {
                    const uint32_t idx = j * 32 + lane;
                    if (idx < e) acc = AT::comb(acc, AT::lift(in[(h + idx) & imask]));
                }
            } else {
                agg_tagged(in, tin, imask, h, e);
            }
        } else {
            const StageP &sp = P.st[n - 1];
            uint32_t *out = q[n];
            uint32_t *tout = t[n];
            uint32_t tl = qt[n];
#pragma unroll
            for (int j = 0; j < IPL; ++j) {
                const uint32_t idx = j * 32 + lane;
                const bool act = idx < e;
                uint32_t v = act ? in[(h + idx) & imask] : 0u;
                uint32_t tg = 0;
                if constexpr (TAG) tg = act ? tin[(h + idx) & imask] : 0u;
                const bool keep = act && stage_apply(sp, v);
                const uint32_t mk = __ballot_sync(kFull, keep);   // stable compaction
                if (keep) {
                    const uint32_t pos = (tl + __popc(mk & lanemask_lt())) & qmask;
                    out[pos] = v;
                    if constexpr (TAG) tout[pos] = tg;
                }
                tl += __popc(mk);
            }
            sent[n] += tl - qt[n];
            qt[n] = tl;
            __syncwarp();
        }
    }

    // Region-id-keyed segmented reduction with a carry across ensembles
    // (tagged aggregate).  Ensembles may mix regions.
    __device__ void agg_tagged(const uint32_t *in, const uint32_t *tin, uint32_t imask, uint32_t h, uint32_t e) {
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
            const int cntj = (int)e - j * 32;
            if (cntj <= 0) break;
            const bool act = lane < cntj;
            const uint32_t idx = j * 32 + lane;
            const uint32_t key = act ? tin[(h + idx) & imask] : 0xffffffffu;
            const A val = act ? AT::lift(in[(h + idx) & imask]) : AT::id();
            if (__all_sync(kFull, !act || key == akey)) {
                acc = AT::comb(acc, val);      // fast path: whole slice continues the carry region
                continue;
            }
            // fold per-lane partials of the carry into `carry`
            carry = AT::comb(carry, warp_reduce<AT>(acc));
            acc = AT::id();
            uint32_t prev = __shfl_up_sync(kFull, key, 1);
            if (lane == 0) prev = akey;
            const bool head = act && key != prev;
            const uint32_t hm = __ballot_sync(kFull, head);
            const uint32_t le = hm & lanemask_le();
            const int seg = le ? 31 - __clz(le) : -1;     // first lane of my segment (-1: carry segment)
            A v = val;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const A o = AT::shfl_up(v, d);
                if (lane - d >= seg && lane >= d) v = AT::comb(o, v);
            }
            if (seg < 0 && act) v = AT::comb(carry, v);
            // the carry region ended exactly before this slice
            if (lane == 0 && head && akey != 0xffffffffu) store_key(akey, carry);
            const bool nexthead = (lane < 31) && ((hm >> (lane + 1)) & 1u);
            if (act && nexthead) store_key(key, v);      // complete segment inside the slice
            const int last = (cntj < 32 ? cntj : 32) - 1;   // last active lane of this slice
            akey = __shfl_sync(kFull, key, last);
            carry = AT::shfl(v, last);
        }
    }

    __device__ void flush_tagged() {
        carry = AT::comb(carry, warp_reduce<AT>(acc));
        acc = AT::id();
        if (lane == 0 && akey != 0xffffffffu) store_key(akey, carry);
        akey = 0xffffffffu;
        carry = AT::id();
    }

    __device__ bool all_empty() const {
        bool e = true;
#pragma unroll
        for (int k = 0; k <= K; ++k) e = e && (qh[k] == qt[k]) && (sh[k] == stl[k]);
        return e;
    }

    template <int n>
    __device__ bool fire_chain(bool drained) {
        if constexpr (n > K + 1) {
            return false;
        } else {
            bool p = fire<n>(drained);
            const bool dn = drained && (qh[n - 1] == qt[n - 1]) && (sh[n - 1] == stl[n - 1]);
            return fire_chain<n + 1>(dn) | p;
        }
    }

    __device__ void run() {
        if (lane == 0)
            for (int i = 0; i < NST; ++i) mbar_init(&bar[i], 1);
        mbar_fence_init();
        __syncwarp();
        uint32_t idle = 0;
        for (;;) {
            bool prog = enumerate();
            prog |= fire_chain<1>(enum_done);
            if (enum_done && all_empty()) break;
            if (prog) { idle = 0; continue; }
            // nothing fireable: wait for the oldest in-flight TMA stage
            if (landed_j < stg_j) {
                uint32_t spins = 0;
                while (!mbar_try_wait(&bar[landed_j % NST], (landed_j / NST) & 1u)) {
                    if (++spins > (1u << 24)) break;
                }
                if (spins > (1u << 24)) { if (lane == 0) atomicCAS((int *)&P.hdr->err, 0, ERR_WATCHDOG); break; }
                continue;
            }
            if (++idle > 64) {
                if (lane == 0) atomicCAS((int *)&P.hdr->err, 0, ERR_WATCHDOG);
                break;
            }
        }
        if constexpr (TAG) flush_tagged();
        // drain outstanding TMA stages before the CTA's shared memory is released
        for (uint32_t spins = 0; landed_j < stg_j && spins < (1u << 26); ++spins) {
            if (mbar_try_wait(&bar[landed_j % NST], (landed_j / NST) & 1u)) landed_j++;
        }
        if (P.flags & RS_FLAG_STATS) {
            if (lane < K + 2) {
                uint32_t a = 0, b = 0, c = 0, d = 0;
#pragma unroll
                for (int n = 0; n < K + 2; ++n)
                    if (lane == n) { a = nd[n]; b = nf[n]; c = ni[n]; d = ns[n]; }
                unsigned long long *S = P.stats + 4 * lane;
                if (a) atomicAdd(S + 0, (unsigned long long)a);
                if (b) atomicAdd(S + 1, (unsigned long long)b);
                if (c) atomicAdd(S + 2, (unsigned long long)c);
                if (d) atomicAdd(S + 3, (unsigned long long)d);
            }
        }
    }
};

template <int K, int AGG, bool TAG>
__global__ void __launch_bounds__(WPB * 32) k_pipeline(const __grid_constant__ KParams P) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    using PP = Pipe<K, AGG, TAG>;
    uint8_t *mine = smem + (size_t)warp * PP::smem_bytes(P.qcap, P.scap);
    if (P.hdr->err) return;
    PP pipe(P, mine, lane);
    pipe.run();
}

// ------------------------------------------------------------ host side
thread_local std::string g_err;

rs_status fail(rs_status s, const std::string &msg) {
    g_err = msg;
    return s;
}

bool is_pow2(uint32_t x) { return x && !(x & (x - 1)); }

}  // namespace

struct rs_pipeline {
    rs_config cfg;
    rs_dtype elem;
    int n_nodes;
    int nst;
    int agg;
    StageP st[MAXK];
    int launches = 0;
    int grid = 0;
    int wpb = WPB;
    void *last_ws = nullptr;
    int device = -1;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    bool timed = false;
    // run_host buffers
    void *h_dbuf = nullptr;
    size_t h_dbuf_bytes = 0;
};

namespace {

using KernelFn = void (*)(KParams);

template <int AGG, bool TAG>
KernelFn pick_k(int K) {
    switch (K) {
        case 0: return k_pipeline<0, AGG, TAG>;
        case 1: return k_pipeline<1, AGG, TAG>;
        case 2: return k_pipeline<2, AGG, TAG>;
        case 3: return k_pipeline<3, AGG, TAG>;
        default: return k_pipeline<4, AGG, TAG>;
    }
}

template <int AGG, bool TAG>
uint32_t smem_for(int K, uint32_t qcap, uint32_t scap) {
    switch (K) {
        case 0: return Pipe<0, AGG, TAG>::smem_bytes(qcap, scap);
        case 1: return Pipe<1, AGG, TAG>::smem_bytes(qcap, scap);
        case 2: return Pipe<2, AGG, TAG>::smem_bytes(qcap, scap);
        case 3: return Pipe<3, AGG, TAG>::smem_bytes(qcap, scap);
        default: return Pipe<4, AGG, TAG>::smem_bytes(qcap, scap);
    }
}

struct Launch {
    KernelFn main;
    void (*pre)(KParams, int);
    void (*fix)(KParams);
    uint32_t inst_bytes;
    int out_bytes0, out_bytes1;
};

template <int AGG>
Launch launch_for(int K, bool tag, uint32_t qcap, uint32_t scap) {
    Launch L;
    L.main = tag ? pick_k<AGG, true>(K) : pick_k<AGG, false>(K);
    L.pre = k_prepass<AGG>;
    L.fix = k_fixup<AGG>;
    L.inst_bytes = tag ? smem_for<AGG, true>(K, qcap, scap) : smem_for<AGG, false>(K, qcap, scap);
    L.out_bytes0 = AggT<AGG>::bytes0;
    L.out_bytes1 = AggT<AGG>::bytes1;
    return L;
}

bool get_launch(const rs_pipeline *p, Launch *L) {
    switch (p->agg) {
        case RS_OP_SUM_I64: *L = launch_for<20>(p->nst, p->cfg.strategy == RS_STRATEGY_TAGGED, p->cfg.queue_cap, p->cfg.signal_cap); return true;
        case RS_OP_SUM_F32: *L = launch_for<21>(p->nst, p->cfg.strategy == RS_STRATEGY_TAGGED, p->cfg.queue_cap, p->cfg.signal_cap); return true;
        case RS_OP_COUNT_MIN_U32: *L = launch_for<22>(p->nst, p->cfg.strategy == RS_STRATEGY_TAGGED, p->cfg.queue_cap, p->cfg.signal_cap); return true;
    }
    return false;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct WsLayout {
    size_t hdr, stats, fr, part0, part1, total;
    long long max_chunks;
};

WsLayout layout(const rs_pipeline *p, long long n_regions, long long n_elems, const Launch &L) {
    WsLayout w;
    long long C = p->cfg.chunk;
    w.max_chunks = (n_elems + 16) / C + 2;
    w.hdr = 0;
    w.stats = 256;
    w.fr = w.stats + align256(sizeof(unsigned long long) * 4 * (MAXK + 2));
    w.part0 = w.fr + align256(sizeof(uint32_t) * (size_t)(w.max_chunks + 1));
    w.part1 = w.part0 + align256((size_t)L.out_bytes0 * 2 * (size_t)w.max_chunks);
    w.total = w.part1 + align256((size_t)(L.out_bytes1 ? L.out_bytes1 : 1) * 2 * (size_t)w.max_chunks);
    (void)n_regions;
    return w;
}

}  // namespace

extern "C" {

const char *rs_status_string(rs_status s) {
    switch (s) {
        case RS_OK: return "RS_OK";
        case RS_ERR_INVALID_ARG: return "RS_ERR_INVALID_ARG";
        case RS_ERR_INVALID_TOPOLOGY: return "RS_ERR_INVALID_TOPOLOGY";
        case RS_ERR_UNSUPPORTED: return "RS_ERR_UNSUPPORTED";
        case RS_ERR_WORKSPACE: return "RS_ERR_WORKSPACE";
        case RS_ERR_CUDA: return "RS_ERR_CUDA";
        case RS_ERR_PROTOCOL: return "RS_ERR_PROTOCOL";
    }
    return "RS_ERR_UNKNOWN";
}

const char *rs_last_error(void) { return g_err.c_str(); }

rs_status rs_config_default(rs_config *cfg) {
    if (!cfg) return fail(RS_ERR_INVALID_ARG, "cfg is NULL");
    cfg->strategy = RS_STRATEGY_SIGNAL;
    cfg->simd_width = W;
    cfg->queue_cap = 2 * W;
    cfg->signal_cap = 128;
    cfg->grid = 0;
    cfg->chunk = 0;
    cfg->flags = RS_FLAG_STATS;
    return RS_OK;
}

rs_status rs_pipeline_create(const rs_node *nodes, int n_nodes, rs_dtype elem, const rs_config *cfg_in,
                             rs_pipeline **out) {
    if (!out) return fail(RS_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!nodes || n_nodes < 2) return fail(RS_ERR_INVALID_TOPOLOGY, "need at least ENUMERATE and AGGREGATE nodes");
    rs_config cfg;
    if (cfg_in) cfg = *cfg_in; else rs_config_default(&cfg);
    if (nodes[0].kind != RS_NODE_ENUMERATE) return fail(RS_ERR_INVALID_TOPOLOGY, "node 0 must be ENUMERATE");
    if (nodes[n_nodes - 1].kind != RS_NODE_AGGREGATE) return fail(RS_ERR_INVALID_TOPOLOGY, "last node must be AGGREGATE");
    int nst = n_nodes - 2;
    for (int i = 1; i < n_nodes - 1; ++i) {
        if (nodes[i].kind == RS_NODE_ENUMERATE) return fail(RS_ERR_INVALID_TOPOLOGY, "nested ENUMERATE is not supported (single-level enumeration)");
        if (nodes[i].kind == RS_NODE_AGGREGATE) return fail(RS_ERR_INVALID_TOPOLOGY, "AGGREGATE must be the last node");
        if (nodes[i].kind != RS_NODE_FILTER && nodes[i].kind != RS_NODE_TRANSFORM)
            return fail(RS_ERR_INVALID_TOPOLOGY, "unknown node kind at position " + std::to_string(i));
    }
    if (nst > MAXK) return fail(RS_ERR_UNSUPPORTED, "at most 4 FILTER/TRANSFORM stages are built");
    if (elem < RS_I32 || elem > RS_F32) return fail(RS_ERR_INVALID_ARG, "bad element dtype");
    const int agg = nodes[n_nodes - 1].op;
    switch (agg) {
        case RS_OP_SUM_I64: if (elem != RS_I32) return fail(RS_ERR_UNSUPPORTED, "SUM_I64 needs i32 elements"); break;
        case RS_OP_SUM_F32: if (elem != RS_F32) return fail(RS_ERR_UNSUPPORTED, "SUM_F32 needs f32 elements"); break;
        case RS_OP_COUNT_MIN_U32: if (elem != RS_U32) return fail(RS_ERR_UNSUPPORTED, "COUNT_MIN_U32 needs u32 elements"); break;
        case RS_OP_COUNT_XOR64: return fail(RS_ERR_UNSUPPORTED, "COUNT_XOR64 (u8 text) is not built yet");
        default: return fail(RS_ERR_UNSUPPORTED, "unknown aggregate op");
    }
    if (cfg.strategy != RS_STRATEGY_SIGNAL && cfg.strategy != RS_STRATEGY_TAGGED)
        return fail(RS_ERR_INVALID_ARG, "bad strategy");
    if (cfg.simd_width == 0) cfg.simd_width = W;
    if (cfg.simd_width != (uint32_t)W) return fail(RS_ERR_UNSUPPORTED, "only simd_width 128 is built");
    if (cfg.queue_cap == 0) cfg.queue_cap = 2 * W;
    if (cfg.signal_cap == 0) cfg.signal_cap = 128;
    if (!is_pow2(cfg.queue_cap) || cfg.queue_cap < 2 * W || cfg.queue_cap > 65536)
        return fail(RS_ERR_UNSUPPORTED, "queue_cap must be a power of 2 in [256, 65536]");
    if (!is_pow2(cfg.signal_cap) || cfg.signal_cap < 4 || cfg.signal_cap > 65536)
        return fail(RS_ERR_UNSUPPORTED, "signal_cap must be a power of 2 in [4, 65536]");
    if (cfg.chunk == 0) cfg.chunk = 8192;
    if (!is_pow2(cfg.chunk) || cfg.chunk < 2048 || cfg.chunk > (1u << 24))
        return fail(RS_ERR_UNSUPPORTED, "chunk must be a power of 2 in [2048, 2^24]");
    if (cfg.grid < 0) return fail(RS_ERR_INVALID_ARG, "grid must be >= 0");
    rs_pipeline *p = new rs_pipeline();
    p->cfg = cfg;
    p->elem = elem;
    p->n_nodes = n_nodes;
    p->nst = nst;
    p->agg = agg;
    for (int i = 0; i < nst; ++i) {
        const rs_node &nd = nodes[i + 1];
        StageP &s = p->st[i];
        std::memset(&s, 0, sizeof s);
        s.kind = nd.kind;
        s.op = nd.op;
        if (nd.kind == RS_NODE_FILTER) {
            switch (nd.op) {
                case RS_OP_HASH_LT:
                    if (nd.p1 > 256) { delete p; return fail(RS_ERR_INVALID_ARG, "HASH_LT threshold must be <= 256"); }
                    s.a = (uint32_t)nd.p0; s.b = (uint32_t)nd.p1; break;
                case RS_OP_LT_U32:
                    if (nd.p1 > (1ull << 32)) { delete p; return fail(RS_ERR_INVALID_ARG, "LT_U32 bound must be <= 2^32"); }
                    s.b = (uint32_t)nd.p1;
                    s.table[0] = nd.p1 == (1ull << 32);
                    break;
                case RS_OP_CLASS:
                    if (!nd.table) { delete p; return fail(RS_ERR_INVALID_ARG, "CLASS needs a 32-byte table"); }
                    if (elem != RS_U8) { delete p; return fail(RS_ERR_UNSUPPORTED, "CLASS needs u8 elements"); }
                    std::memcpy(s.table, nd.table, 32); break;
                default: delete p; return fail(RS_ERR_UNSUPPORTED, "unknown FILTER op");
            }
        } else {
            switch (nd.op) {
                case RS_OP_SCALE_F32:
                    if (elem != RS_F32) { delete p; return fail(RS_ERR_UNSUPPORTED, "SCALE_F32 needs f32 elements"); }
                    s.a = (uint32_t)nd.p0; break;
                case RS_OP_AFFINE_I32:
                    if (elem != RS_I32 && elem != RS_U32) { delete p; return fail(RS_ERR_UNSUPPORTED, "AFFINE_I32 needs 32-bit int elements"); }
                    s.a = (uint32_t)nd.p0; s.b = (uint32_t)nd.p1; break;
                default: delete p; return fail(RS_ERR_UNSUPPORTED, "unknown TRANSFORM op");
            }
        }
    }
    *out = p;
    return RS_OK;
}

rs_status rs_pipeline_workspace_bytes(const rs_pipeline *p, int64_t n_regions, int64_t n_elems, size_t *bytes) {
    if (!p || !bytes) return fail(RS_ERR_INVALID_ARG, "NULL argument");
    if (n_regions < 0 || n_elems < 0) return fail(RS_ERR_INVALID_ARG, "negative size");
    Launch L;
    if (!get_launch(p, &L)) return fail(RS_ERR_UNSUPPORTED, "aggregate not built");
    *bytes = layout(p, n_regions, n_elems, L).total;
    return RS_OK;
}

static rs_status run_impl(rs_pipeline *p, const void *d_elems, int64_t n_elems, const int64_t *d_offsets,
                          int64_t n_regions, rs_aggregates out, void *d_ws, size_t ws_bytes, cudaStream_t stream) {
    if (!p) return fail(RS_ERR_INVALID_ARG, "pipeline is NULL");
    p->launches = 0;
    if (n_regions < 0 || n_regions >= (1ll << 31)) return fail(RS_ERR_INVALID_ARG, "n_regions must be in [0, 2^31)");
    if (n_elems < 0 || n_elems >= (1ll << 40)) return fail(RS_ERR_INVALID_ARG, "bad n_elems");
    if (n_regions == 0) return RS_OK;
    if (!d_offsets) return fail(RS_ERR_INVALID_ARG, "d_offsets is NULL");
    if (n_elems > 0 && !d_elems) return fail(RS_ERR_INVALID_ARG, "d_elems is NULL");
    if (((uintptr_t)d_elems & 15u) != 0) return fail(RS_ERR_INVALID_ARG, "d_elems must be 16-byte aligned");
    if (((uintptr_t)d_offsets & 7u) != 0) return fail(RS_ERR_INVALID_ARG, "d_offsets must be 8-byte aligned");
    Launch L;
    if (!get_launch(p, &L)) return fail(RS_ERR_UNSUPPORTED, "aggregate not built");
    if (!out.v0 || (L.out_bytes1 && !out.v1)) return fail(RS_ERR_INVALID_ARG, "output array is NULL");
    WsLayout wl = layout(p, n_regions, n_elems, L);
    if (!d_ws || ws_bytes < wl.total) return fail(RS_ERR_WORKSPACE, "workspace smaller than rs_pipeline_workspace_bytes");
    if (((uintptr_t)d_ws & 255u) != 0) return fail(RS_ERR_WORKSPACE, "workspace must be 256-byte aligned");

    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(RS_ERR_CUDA, "cudaGetDevice failed");
    const uint32_t cta_smem = L.inst_bytes * WPB;
    if (p->device != dev || p->grid == 0) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaFuncSetAttribute(L.main, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cta_smem) != cudaSuccess)
            return fail(RS_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(cudaGetLastError()));
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, L.main, WPB * 32, cta_smem);
        if (per_sm < 1) return fail(RS_ERR_UNSUPPORTED, "pipeline does not fit on an SM (queue/signal capacities too large)");
        p->grid = p->cfg.grid > 0 ? p->cfg.grid : sms * per_sm;
        p->device = dev;
    }
    cudaFuncSetAttribute(L.main, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cta_smem);

    KParams K;
    std::memset(&K, 0, sizeof K);
    K.elems = (const uint8_t *)d_elems;
    K.n_elems = n_elems;
    K.off = (const long long *)d_offsets;
    K.R = n_regions;
    K.out0 = out.v0;
    K.out1 = out.v1;
    uint8_t *ws = (uint8_t *)d_ws;
    K.hdr = (WsHdr *)(ws + wl.hdr);
    K.stats = (unsigned long long *)(ws + wl.stats);
    K.chunk_fr = (uint32_t *)(ws + wl.fr);
    K.part0 = ws + wl.part0;
    K.part1 = ws + wl.part1;
    K.max_chunks = wl.max_chunks;
    K.C = p->cfg.chunk;
    K.qcap = p->cfg.queue_cap;
    K.scap = p->cfg.signal_cap;
    K.flags = p->cfg.flags;
    K.tagged = p->cfg.strategy == RS_STRATEGY_TAGGED;
    K.nst = p->nst;
    std::memcpy(K.st, p->st, sizeof K.st);

    int pre_blocks = (int)std::min<long long>((2 * wl.max_chunks + 2 + 255) / 256, 148 * 8);
    if (K.tagged || (K.flags & RS_FLAG_VALIDATE)) pre_blocks = std::max(pre_blocks, 148 * 8);
    const bool timing = (K.flags & RS_FLAG_TIMING) != 0;
    if (timing && !p->ev[0])
        for (int i = 0; i < 4; ++i) cudaEventCreate(&p->ev[i]);
    p->timed = timing;
    if (timing) cudaEventRecord(p->ev[0], stream);
    L.pre<<<pre_blocks, 256, 0, stream>>>(K, 4 * (p->nst + 2));
    if (timing) cudaEventRecord(p->ev[1], stream);
    L.main<<<p->grid, WPB * 32, cta_smem, stream>>>(K);
    if (timing) cudaEventRecord(p->ev[2], stream);
    int fix_blocks = (int)std::min<long long>((wl.max_chunks + 255) / 256, 148 * 8);
    L.fix<<<std::max(fix_blocks, 1), 256, 0, stream>>>(K);
    if (timing) cudaEventRecord(p->ev[3], stream);
    p->launches = 3;
    p->last_ws = d_ws;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, std::string("launch failed: ") + cudaGetErrorString(e));
    return RS_OK;
}

rs_status rs_pipeline_run(rs_pipeline *p, const void *d_elems, int64_t n_elems, const int64_t *d_offsets,
                          int64_t n_regions, rs_aggregates out, void *d_ws, size_t ws_bytes, rs_stream stream) {
    return run_impl(p, d_elems, n_elems, d_offsets, n_regions, out, d_ws, ws_bytes, (cudaStream_t)stream);
}

rs_status rs_pipeline_run_host(rs_pipeline *p, const void *h_elems, int64_t n_elems, const int64_t *h_offsets,
                               int64_t n_regions, rs_aggregates h_out, rs_stream stream_) {
    if (!p) return fail(RS_ERR_INVALID_ARG, "pipeline is NULL");
    if (n_regions < 0 || n_elems < 0) return fail(RS_ERR_INVALID_ARG, "negative size");
    if (n_regions == 0) return RS_OK;
    if (!h_offsets || (n_elems > 0 && !h_elems)) return fail(RS_ERR_INVALID_ARG, "NULL host buffer");
    Launch L;
    if (!get_launch(p, &L)) return fail(RS_ERR_UNSUPPORTED, "aggregate not built");
    if (!h_out.v0 || (L.out_bytes1 && !h_out.v1)) return fail(RS_ERR_INVALID_ARG, "output array is NULL");
    cudaStream_t stream = (cudaStream_t)stream_;
    const size_t esz = p->elem == RS_U8 ? 1 : 4;
    size_t ws = 0;
    rs_pipeline_workspace_bytes(p, n_regions, n_elems, &ws);
    const size_t b_el = align256(esz * (size_t)n_elems + 16);
    const size_t b_off = align256(8 * (size_t)(n_regions + 1));
    const size_t b_o0 = align256((size_t)L.out_bytes0 * (size_t)n_regions);
    const size_t b_o1 = align256((size_t)(L.out_bytes1 ? L.out_bytes1 : 1) * (size_t)n_regions);
    const size_t need = b_el + b_off + b_o0 + b_o1 + ws;
    if (p->h_dbuf_bytes < need) {
        if (p->h_dbuf) cudaFree(p->h_dbuf);
        p->h_dbuf = nullptr;
        p->h_dbuf_bytes = 0;
        if (cudaMalloc(&p->h_dbuf, need) != cudaSuccess) return fail(RS_ERR_CUDA, "cudaMalloc of run_host buffers failed");
        p->h_dbuf_bytes = need;
    }
    uint8_t *d = (uint8_t *)p->h_dbuf;
    void *d_el = d, *d_off = d + b_el, *d_o0 = d + b_el + b_off, *d_o1 = d + b_el + b_off + b_o0;
    void *d_ws = d + b_el + b_off + b_o0 + b_o1;
    if (n_elems && cudaMemcpyAsync(d_el, h_elems, esz * (size_t)n_elems, cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, "H2D elements failed");
    if (cudaMemcpyAsync(d_off, h_offsets, 8 * (size_t)(n_regions + 1), cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, "H2D offsets failed");
    rs_aggregates dout{d_o0, L.out_bytes1 ? d_o1 : nullptr};
    rs_status s = run_impl(p, d_el, n_elems, (const int64_t *)d_off, n_regions, dout, d_ws, ws, stream);
    if (s != RS_OK) return s;
    if (cudaMemcpyAsync(h_out.v0, d_o0, (size_t)L.out_bytes0 * (size_t)n_regions, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, "D2H aggregates failed");
    if (L.out_bytes1 && cudaMemcpyAsync(h_out.v1, d_o1, (size_t)L.out_bytes1 * (size_t)n_regions, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, "D2H aggregates failed");
    if (cudaStreamSynchronize(stream) != cudaSuccess) return fail(RS_ERR_CUDA, "stream synchronize failed");
    return RS_OK;
}

rs_status rs_pipeline_stats(rs_pipeline *p, rs_node_stats *host_out, int n_nodes, rs_stream stream) {
    if (!p || !host_out) return fail(RS_ERR_INVALID_ARG, "NULL argument");
    if (n_nodes != p->n_nodes) return fail(RS_ERR_INVALID_ARG, "n_nodes must equal the create-time node count");
    if (!p->last_ws) {
        std::memset(host_out, 0, sizeof(rs_node_stats) * n_nodes);
        return RS_OK;
    }
    unsigned long long buf[4 * (MAXK + 2)];
    if (cudaMemcpyAsync(buf, (uint8_t *)p->last_ws + 256, sizeof(unsigned long long) * 4 * n_nodes,
                        cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess ||
        cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, "stats copy failed");
    for (int n = 0; n < n_nodes; ++n) {
        host_out[n].data_firings = buf[4 * n + 0];
        host_out[n].full_firings = buf[4 * n + 1];
        host_out[n].items = buf[4 * n + 2];
        host_out[n].signal_firings = buf[4 * n + 3];
    }
    return RS_OK;
}

rs_status rs_pipeline_check(rs_pipeline *p, rs_stream stream, int32_t *code) {
    if (!p) return fail(RS_ERR_INVALID_ARG, "NULL pipeline");
    if (code) *code = 0;
    if (!p->last_ws) return RS_OK;
    WsHdr h;
    if (cudaMemcpyAsync(&h, p->last_ws, sizeof h, cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess ||
        cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, std::string("error-word copy failed: ") + cudaGetErrorString(cudaGetLastError()));
    if (code) *code = h.err;
    if (h.err) return fail(RS_ERR_PROTOCOL, "device error code " + std::to_string(h.err));
    return RS_OK;
}

int rs_pipeline_launches(const rs_pipeline *p) { return p ? p->launches : 0; }

rs_status rs_pipeline_kernel_times(rs_pipeline *p, float *ms3, rs_stream stream) {
    if (!p || !ms3) return fail(RS_ERR_INVALID_ARG, "NULL argument");
    if (!p->timed || !p->ev[0]) return fail(RS_ERR_INVALID_ARG, "last run was not made with RS_FLAG_TIMING");
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return fail(RS_ERR_CUDA, "stream synchronize failed");
    for (int i = 0; i < 3; ++i)
        if (cudaEventElapsedTime(&ms3[i], p->ev[i], p->ev[i + 1]) != cudaSuccess) return fail(RS_ERR_CUDA, "event timing failed");
    return RS_OK;
}

rs_status rs_pipeline_geometry(const rs_pipeline *p, int32_t *grid, int32_t *wpb, int32_t *chunk) {
    if (!p) return fail(RS_ERR_INVALID_ARG, "NULL pipeline");
    if (grid) *grid = p->grid;
    if (wpb) *wpb = p->wpb;
    if (chunk) *chunk = (int32_t)p->cfg.chunk;
    return RS_OK;
}

void rs_pipeline_destroy(rs_pipeline *p) {
    if (!p) return;
    if (p->h_dbuf) cudaFree(p->h_dbuf);
    for (int i = 0; i < 4; ++i)
        if (p->ev[i]) cudaEventDestroy(p->ev[i]);
    delete p;
}

}  // extern "C"
