// rs_pipe.cuh — one pipeline INSTANCE per warp (included by rs.cu).
//
// Nodes 0 = ENUMERATE, 1..K = FILTER/TRANSFORM, K+1 = AGGREGATE; edge e joins
// node e -> e+1 with a data queue and, for the signal strategy, a
// signal queue.  See rs.cu's header comment for the model; the
// citations below point at the PAPER.md lines each step realises.
#pragma once
#include <type_traits>

// ------------------------------------------------- filter / transform ops
// isGood() / push() bodies (Fig. 5), specialised per op so the
// full-ensemble path carries no per-item dispatch (readings A13/A14).
struct OpHash {            // keep iff ((v*a) >> 24) < t  <=>  v*a < t << 24   (t <= 255)
    uint32_t a, tt;
    __device__ __forceinline__ bool operator()(uint32_t &v) const { return v * a < tt; }
};
struct OpAll {             // HASH_LT with t = 256 (or LT_U32 with bound 2^32): keeps every item
    __device__ __forceinline__ bool operator()(uint32_t &) const { return true; }
};
struct OpLt {
    uint32_t b;
    bool all;
    __device__ __forceinline__ bool operator()(uint32_t &v) const { return all || v < b; }
};
struct OpClass {
    const uint32_t *tbl;
    __device__ __forceinline__ bool operator()(uint32_t &v) const { return (tbl[(v & 0xffu) >> 5] >> (v & 31u)) & 1u; }
};
// CLASS with a single member byte c (the text config's '{'): the scalar form
// for the generic paths, and match4() -- a SWAR test of four bytes at once
// (exact zero-byte detection of w ^ c4, no carries across bytes): 0x80 in
// every byte of w that equals c.
struct OpClass1 {
    uint32_t c4;           // c replicated into the four bytes
    __device__ __forceinline__ bool operator()(uint32_t &v) const { return (v & 0xffu) == (c4 & 0xffu); }
    __device__ __forceinline__ uint32_t match4(uint32_t w) const {
        const uint32_t x = w ^ c4;
        return ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x) & 0x80808080u;
    }
};
struct OpScale {
    float s;
    __device__ __forceinline__ bool operator()(uint32_t &v) const {
        v = __float_as_uint(__fmul_rn(s, __uint_as_float(v)));
        return true;
    }
};
struct OpAffine {
    uint32_t a, b;
    __device__ __forceinline__ bool operator()(uint32_t &v) const {
        v = v * a + b;
        return true;
    }
};

struct OpDyn {             // runtime op (partial ensembles)
    const StageP *s;
    __device__ __forceinline__ bool operator()(uint32_t &v) const { return stage_apply(*s, v); }
};

// Full ensembles of a FILTER/TRANSFORM node, specialised per op and shared
// by every stage node (one copy of the code keeps the hot loop inside the
// instruction cache).  Item t of an ensemble lives in lane t%32, slot t/32.
// NS slices (NS*32 items, one or two ensembles) are processed together: all
// loads first, then the predicates, then the stable ballot/popc compaction
// into the output queue (push) -- NS-way instruction-level parallelism.
// Items are 32-bit.  A byte element ring (U8IN, the text stream) is read as
// item = byte | (position mod C) << 8: the position within the chunk lets the
// aggregate recover each byte's index within its line (reading A19).
template <bool U8IN>
__device__ __forceinline__ uint32_t load_item(const uint32_t *in, uint32_t pos, uint32_t imask, uint32_t cmask) {
    if constexpr (U8IN) return (uint32_t)reinterpret_cast<const uint8_t *>(in)[pos & imask] | ((pos & cmask) << 8);
    else return in[pos & imask];
}

template <bool TAG, int NS, class Op, bool U8IN>
__device__ __forceinline__ void filter_slices(const uint32_t *in, const uint32_t *tin, uint32_t imask, uint32_t h,
                                              uint32_t *out, uint32_t *tout, uint32_t qmask, uint32_t &tl,
                                              const Op &op, uint32_t lt, uint32_t cmask) {
    // Masked ring addressing only (no wrap-free fast path): the smaller code
    // measured faster than the dual-path variant (profiles/r1_tuning.txt).
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t v[NS], tg[NS];
    bool keep[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) v[j] = load_item<U8IN>(in, h + 32 * j + lane, imask, cmask);
    if constexpr (TAG) {
#pragma unroll
        for (int j = 0; j < NS; ++j) tg[j] = tin[(h + 32 * j + lane) & imask];
    }
    // in-place rings: every lane's reads of this ensemble are ordered before any
    // lane's compaction stores into the same slots (the memory ordering of
    // __syncwarp; ballots order execution, not memory)
    __syncwarp();
#pragma unroll
    for (int j = 0; j < NS; ++j) keep[j] = op(v[j]);
    uint32_t mk[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) mk[j] = __ballot_sync(kFull, keep[j]);
    // slice bases from a shallow sum tree (not a serial chain through tl)
    uint32_t c[NS], bs[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) c[j] = __popc(mk[j]);
    bs[0] = tl;
#pragma unroll
    for (int j = 1; j < NS; ++j) {
        uint32_t pre = 0;
#pragma unroll
        for (int i = 0; i < j; ++i) pre += c[i];
        bs[j] = tl + pre;
    }
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        if (keep[j]) {
            const uint32_t pos = (bs[j] + __popc(mk[j] & lt)) & qmask;
            out[pos] = v[j];
            if constexpr (TAG) tout[pos] = tg[j];
        }
    }
    uint32_t all = 0;
#pragma unroll
    for (int j = 0; j < NS; ++j) all += c[j];
    tl += all;
}

// SWAR filter ensemble over a byte ring, single-member CLASS:
// the e <= w bytes at h are read one 32-bit word per lane (lane l: bytes
// 4l .. 4l+3, a funnel shift realigns an unaligned head) and tested four at a
// time (OpClass1::match4); the sparse survivors are compacted in stream
// order -- lane l's survivors follow those of lanes < l, found from three
// ballots of its survivor count (0..4) -- as items byte | (pos mod C) << 8
// into the 4-byte output queue.  Returns the new output tail.
__device__ __forceinline__ uint32_t swar_filter(const uint32_t *in, uint32_t imask, uint32_t h, uint32_t e,
                                                uint32_t *out, uint32_t qmask, uint32_t tl, const OpClass1 &op,
                                                uint32_t lt, uint32_t cmask) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t wmask = imask >> 2;
    const uint32_t a = h & 3u;
    const uint32_t wi = ((h >> 2) + lane) & wmask;
    uint32_t w = in[wi];
    if (a) w = __funnelshift_r(w, in[(wi + 1) & wmask], 8u * a);
    uint32_t m = op.match4(w);
    if (e < (uint32_t)W) {
        const int valid = (int)e - 4 * (int)lane;
        m &= valid >= 4 ? 0xffffffffu : (valid <= 0 ? 0u : (0xffffffffu >> (32 - 8 * valid)));
    }
    const uint32_t c = __popc(m);
    const uint32_t b0 = __ballot_sync(kFull, c & 1u), b1 = __ballot_sync(kFull, c & 2u), b2 = __ballot_sync(kFull, c & 4u);
    uint32_t at = tl + __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
    while (m) {
        const uint32_t k = (__ffs(m) - 1) >> 3;
        m &= m - 1u;
        const uint32_t pos = h + 4u * lane + k;
        out[at & qmask] = ((w >> (8u * k)) & 0xffu) | ((pos & cmask) << 8);
        ++at;
    }
    return tl + __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
}

template <bool TAG, class Op, bool U8IN = false>
__device__ __noinline__ uint32_t filter_batch(const uint32_t *in, const uint32_t *tin, uint32_t imask, uint32_t h,
                                              uint32_t nens, uint32_t *out, uint32_t *tout, uint32_t qmask,
                                              uint32_t tl, const Op op, uint32_t lt, uint32_t cmask = 0) {
    if constexpr (!TAG && U8IN && std::is_same<Op, OpClass1>::value) {
        for (uint32_t k = 0; k < nens; ++k, h += W) tl = swar_filter(in, imask, h, W, out, qmask, tl, op, lt, cmask);
    } else {
        for (uint32_t k = 0; k < nens; ++k, h += W) filter_slices<TAG, IPL, Op, U8IN>(in, tin, imask, h, out, tout, qmask, tl, op, lt, cmask);
    }
    __syncwarp();
    return tl;
}

// One partial ensemble (e < w items: signal-bounded or the drained tail) of
// a FILTER/TRANSFORM node, specialised per op like the full ensembles and
// shared by every stage node (code size); only the ceil(e/32) occupied
// slices are visited (e is warp-uniform).
template <bool TAG, class Op, bool U8IN>
__device__ __forceinline__ uint32_t partial_body(const Op op, const uint32_t *in, const uint32_t *tin,
                                                 uint32_t imask, uint32_t h, uint32_t e, uint32_t *out, uint32_t *tout,
                                                 uint32_t qmask, uint32_t tl, uint32_t lt, uint32_t cmask) {
    if constexpr (!TAG && U8IN && std::is_same<Op, OpClass1>::value) {
        tl = swar_filter(in, imask, h, e, out, qmask, tl, op, lt, cmask);
        __syncwarp();
        return tl;
    }
    // One slice per iteration, not unrolled (the instruction cache binds; a
    // partial ensemble is rarer than a full one).  In-place rings: slice j's
    // stores land below tl + 32(j+1) <= h + 32(j+1), i.e. below every later
    // slice's reads; within a slice every lane reads before any lane stores.
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll 1
    for (uint32_t j = 0; j * 32u < e; ++j) {
        const uint32_t idx = j * 32 + lane;
        const bool act = idx < e;
        uint32_t v = act ? load_item<U8IN>(in, h + idx, imask, cmask) : 0u;
        uint32_t tg = 0;
        if constexpr (TAG) tg = act ? tin[(h + idx) & imask] : 0u;
        __syncwarp();
        const bool keep = act && op(v);
        const uint32_t mk = __ballot_sync(kFull, keep);   // stable compaction
        if (keep) {
            const uint32_t pos = (tl + __popc(mk & lt)) & qmask;
            out[pos] = v;
            if constexpr (TAG) tout[pos] = tg;
        }
        tl += __popc(mk);
    }
    __syncwarp();
    return tl;
}

template <bool TAG, class Op, bool U8IN>
__device__ __noinline__ uint32_t partial_stage(const Op op, const uint32_t *in, const uint32_t *tin,
                                               uint32_t imask, uint32_t h, uint32_t e, uint32_t *out, uint32_t *tout,
                                               uint32_t qmask, uint32_t tl, uint32_t lt, uint32_t cmask) {
    return partial_body<TAG, Op, U8IN>(op, in, tin, imask, h, e, out, tout, qmask, tl, lt, cmask);
}
template <class Op>
__device__ __noinline__ uint32_t partial_stage_ip(const Op op, uint32_t *ring, uint32_t mask, uint32_t h, uint32_t e,
                                                  uint32_t tl) {
    return partial_body<false, Op, false>(op, ring, nullptr, mask, h, e, ring, nullptr, mask, tl, lanemask_lt(), 0u);
}

// In-place rings without tags (the signal strategy's stage nodes): input and
// output queue share one ring and mask -- the same loops with fewer call
// arguments to marshal at every firing (instruction-cache footprint).
// Ensembles whose input slots and outputs do not wrap the ring use linear
// shared addresses: one LDS with an immediate offset per slice and an
// LEA-formed store address (66 -> ~44 SASS per ensemble); an ensemble that
// straddles the ring end takes the masked loop.
template <int NS, class Op>
__device__ __forceinline__ void filter_linear_ens(uint32_t si, uint32_t &so, const Op &op, uint32_t lt) {
    // si: this lane's slot-0 load address; so: the output tail (byte address).
    // NS slices (NS/4 ensembles): ensemble k's stores land below ensemble
    // k+1's input slots (stable compaction never outruns the reads), so all
    // loads may come first.
    uint32_t v[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) v[j] = lds32(si + 128u * j);
    __syncwarp();      // every lane's reads before any compaction store
    bool keep[NS];
    uint32_t mk[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        keep[j] = op(v[j]);
        mk[j] = __ballot_sync(kFull, keep[j]);
    }
    // byte addresses kept out of the compiler's reassociation (it would
    // rebuild them from a running count: one more add per slice)
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        if (keep[j]) sts32(lea4(__popc(mk[j] & lt), so), v[j]);
        so = lea4(__popc(mk[j]), so);
    }
}
template <class Op>
__device__ __noinline__ uint32_t filter_batch_ip(uint32_t *ring, uint32_t mask, uint32_t h, uint32_t nens, uint32_t tl,
                                                 const Op op) {
    const uint32_t lt = lanemask_lt();
    const uint32_t rb = smem_addr(ring);
    const uint32_t lane4 = (threadIdx.x & 31u) * 4u;
    while (nens > 0) {
        const uint32_t hi = h & mask, ti = tl & mask;
        const uint32_t nl = min(nens, min((mask + 1 - hi) / W, (mask + 1 - ti) / W));
        if (nl == 0) {      // the ensemble straddles the ring end: the (compact) masked loop
            tl = partial_stage_ip(op, ring, mask, h, W, tl);
            h += W;
            --nens;
            continue;
        }
        const uint32_t so0 = rb + ti * 4u;
        uint32_t si = rb + hi * 4u + lane4, so = so0;
#pragma unroll 1
        for (uint32_t k = 0; k < nl; ++k, si += 4u * W) filter_linear_ens<IPL>(si, so, op, lt);
        h += nl * W;
        tl += (so - so0) >> 2;
        nens -= nl;
    }
    __syncwarp();
    return tl;
}


// Fused terminal node, full ensembles, signal strategy (see Pipe::FUSE): the
// node's op decides each item, survivors are folded into the per-lane
// accumulator (isGood + a::run).  Out of line so the hot loop
// stays one copy per op.
// Fold the survivors of one ensemble (v[j] kept iff bit j of km) into acc.
// Cheap lifts: a select per slot.  Heavy lifts (the text hash): survivors are
// sparse, so each lane lifts its first and second survivor under warp-uniform
// guards and only a lane with three or more walks its slots again.
template <class AT>
__device__ __forceinline__ typename AT::A fold_kept(typename AT::A acc, const uint32_t (&v)[IPL], uint32_t km,
                                                    long long adelta) {
    if constexpr (!AT::heavy) {
        typename AT::A part = AT::id();
#pragma unroll
        for (int j = 0; j < IPL; ++j)
            if ((km >> j) & 1u) part = AT::comb(part, AT::lift_i(v[j], adelta));
        return AT::comb(acc, part);
    } else {
        uint32_t s1 = 0, s2 = 0;
        const uint32_t nk = __popc(km);
#pragma unroll
        for (int j = IPL - 1; j >= 0; --j) {       // s1 = first survivor, s2 = second
            if ((km >> j) & 1u) { s2 = s1; s1 = v[j]; }
        }
        if (__any_sync(kFull, nk != 0))
            if (nk != 0) acc = AT::comb(acc, AT::lift_i(s1, adelta));
        if (__any_sync(kFull, nk > 1)) {
            if (nk > 1) acc = AT::comb(acc, AT::lift_i(s2, adelta));
            if (__any_sync(kFull, nk > 2)) {
                uint32_t seen = 0;
#pragma unroll
                for (int j = 0; j < IPL; ++j)
                    if ((km >> j) & 1u) {
                        if (seen >= 2) acc = AT::comb(acc, AT::lift_i(v[j], adelta));
                        ++seen;
                    }
            }
        }
        return acc;
    }
}

template <class AT>
struct FusedAcc {
    typename AT::A acc;
    uint32_t kept;
};
template <class AT, class Op, bool U8IN>
__device__ __noinline__ FusedAcc<AT> fused_batch(const uint32_t *in, uint32_t imask, uint32_t h, uint32_t nens,
                                                 const Op op, long long adelta, uint32_t cmask, FusedAcc<AT> st) {
    const uint32_t lane = threadIdx.x & 31u;
    for (uint32_t k = 0; k < nens; ++k, h += W) {
        uint32_t v[IPL];
#pragma unroll
        for (int j = 0; j < IPL; ++j) v[j] = load_item<U8IN>(in, h + 32 * j + lane, imask, cmask);
        uint32_t km = 0;
#pragma unroll
        for (int j = 0; j < IPL; ++j) km |= op(v[j]) ? 1u << j : 0u;
        st.kept += __popc(km);
        st.acc = fold_kept<AT>(st.acc, v, km, adelta);
    }
    return st;
}

// Fused node K, in-place ring, cheap lifts (the signal strategy's fused
// aggregate over 4-byte items): ensembles that do not straddle the ring end
// load with one immediate-offset LDS per slice; the straddling one goes
// through the compact per-slice loop (fused_partial with e = w).
template <class AT, class Op>
__device__ __noinline__ FusedAcc<AT> fused_batch_ip(const uint32_t *ring, uint32_t mask, uint32_t h, uint32_t nens,
                                                    const Op op, FusedAcc<AT> st);

// In-place rings: move n items (and tags) ending at position `end` up by
// `shift` positions -- a memmove toward higher positions in blocks of <= w
// items, highest block first (each block is read completely before it is
// written, so overlapping source and destination are safe).
template <bool TAG>
__device__ __noinline__ void move_items(uint32_t *q, uint32_t *tq, uint32_t end, uint32_t n, uint32_t shift, uint32_t m) {
    // 32-item slices, highest first, not unrolled (code size): a slice's
    // stores land at or above its own reads and above every lower slice
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll 1
    while (n > 0) {
        const uint32_t c = n < 32u ? n : 32u;
        const uint32_t s0 = end - c;
        const bool act = lane < c;
        const uint32_t v = act ? q[(s0 + lane) & m] : 0u;
        uint32_t tg = 0;
        if constexpr (TAG) tg = act ? tq[(s0 + lane) & m] : 0u;
        __syncwarp();
        if (act) {
            q[(s0 + shift + lane) & m] = v;
            if constexpr (TAG) tq[(s0 + shift + lane) & m] = tg;
        }
        __syncwarp();
        end -= c;
        n -= c;
    }
}

// Fused node K, one partial ensemble (signal strategy): op + fold of the
// occupied slices only.
template <class AT, class Op, bool U8IN>
__device__ __noinline__ FusedAcc<AT> fused_partial(const uint32_t *in, uint32_t imask, uint32_t h, uint32_t e,
                                                   const Op op, long long adelta, uint32_t cmask, FusedAcc<AT> st) {
    const uint32_t lane = threadIdx.x & 31u;
    if constexpr (AT::heavy) {
        uint32_t v[IPL], km = 0;
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
            const uint32_t idx = j * 32 + lane;
            v[j] = idx < e ? load_item<U8IN>(in, h + idx, imask, cmask) : 0u;
            km |= (idx < e && op(v[j])) ? 1u << j : 0u;
        }
        st.kept += __popc(km);
        st.acc = fold_kept<AT>(st.acc, v, km, adelta);
    } else {
#pragma unroll 1
        for (int j = 0; j < IPL; ++j) {
            if ((uint32_t)j * 32u >= e) break;
            const uint32_t idx = j * 32 + lane;
            uint32_t v = idx < e ? load_item<U8IN>(in, h + idx, imask, cmask) : 0u;
            const bool keep = idx < e && op(v);
            st.kept += keep ? 1u : 0u;
            if (keep) st.acc = AT::comb(st.acc, AT::lift_i(v, adelta));
        }
    }
    return st;
}

template <class AT, class Op>
__device__ __noinline__ FusedAcc<AT> fused_batch_ip(const uint32_t *ring, uint32_t mask, uint32_t h, uint32_t nens,
                                                    const Op op, FusedAcc<AT> st) {
    const uint32_t rb = smem_addr(ring) + (threadIdx.x & 31u) * 4u;
    while (nens > 0) {
        const uint32_t hi = h & mask;
        const uint32_t nl = min(nens, (mask + 1 - hi) / W);
        if (nl == 0) {
            st = fused_partial<AT, Op, false>(ring, mask, h, W, op, 0, 0u, st);
            h += W;
            --nens;
            continue;
        }
        uint32_t si = rb + hi * 4u;
#pragma unroll 1
        for (uint32_t k = 0; k < nl; ++k, si += 4u * W) {
            uint32_t v[IPL];
#pragma unroll
            for (int j = 0; j < IPL; ++j) v[j] = lds32(si + 128u * j);
            typename AT::A part = AT::id();
#pragma unroll
            for (int j = 0; j < IPL; ++j) {
                const bool keep = op(v[j]);
                st.kept += keep ? 1u : 0u;
                if (keep) part = AT::comb(part, AT::lift_i(v[j], 0));
            }
            st.acc = AT::comb(st.acc, part);
        }
        h += nl * W;
        nens -= nl;
    }
    return st;
}

struct Chunk {
    int32_t k;             // chunk id (-1 = empty slot)
    long long beg, end;    // element range [beg, end)
    uint32_t pos;          // Q0 queue position of element `beg`
    uint32_t fr0, fr1;     // regions starting in the chunk: [fr0, fr1)
    bool head;             // chunk starts inside region fr0-1 (a head part)
};

// FUSE: the AGGREGATE node is folded into the last FILTER/TRANSFORM node
// (DESIGN.md §5 "fused terminal aggregate"): node K applies its op and adds
// the surviving items of each ensemble straight into the accumulator and
// performs the aggregate's Begin/End actions for the signals it consumes --
// no compaction into, and no re-read of, a final queue.  The aggregate is a
// commutative per-region fold and the signal strategy keeps every ensemble
// inside one region, so the result is the same as with a separate node (the
// tagged strategy folds by key as before).  FUSE=false is the paper's node
// structure, kept for RS_FLAG_UNFUSED.
// CTX: the per-lane context strategy: no
// tags in the queues and no boundary-limited ensembles.  Each signal is one
// region boundary {key, stamp}: the count of items its edge carried before the
// region's first item.  Ensembles run across boundaries; a FILTER/TRANSFORM
// node re-stamps every boundary inside an ensemble from the ensemble's ballots
// (survivors before it), and the aggregate gives each lane the key of the last
// boundary at or before its item -- the context computed per lane instead of
// stored with the items.
// PARENT_LT, out of line (rare: once per region per parent-context node, and
// only in pipelines that have one): *dst = ctx[region of key]; SLOT keys name
// the region split across chunk k's boundary (see Pipe::region_key).
static __device__ __noinline__ void load_pv(const uint32_t *ctx, const uint32_t *chunk_fr, uint32_t key, uint32_t *dst) {
    uint32_t r = key;
    if (key & SLOT) {
        const uint32_t slot = key & ~SLOT, k = slot >> 1;
        r = ((slot & 1u) ? chunk_fr[k + 1] : chunk_fr[k]) - 1u;
    }
    const uint32_t v = ctx[r];
    __syncwarp();          // every lane's reads of the previous value come first
    if ((threadIdx.x & 31u) == 0) *dst = v;
    __syncwarp();
}

template <int K, int AGG, bool TAG, bool FUSE, bool CTX = false, bool TR = false, int HYB = 0, bool SPL = false,
          bool SH = false>
struct Pipe {
    using AT = AggT<AGG>;
    using A = typename AT::A;
    static constexpr bool NA = FUSE && K >= 1;        // aggregate fused into node K
    static constexpr int NQ = NA ? K - 1 : K;         // shared-memory data queues Q_1..Q_NQ
    static constexpr int NSG = NA ? K : K + 1;        // signal rings S_0..S_{NSG-1}
    // Fan-out (§8 f4, Fig. 1b): SPL pipelines end in a SPLIT node
    // (node K+1) with two leaf AGGREGATE children (nodes K+2, K+3) fed by edges
    // K+1 and K+2, each a queue and a signal queue of its own (separate rings
    // after the in-place ring).
    static constexpr int NLQ = SPL ? 2 : 0;
    // Per-stage hybrid (§8 f1; the paper's best taxi variant signals through
    // stage 1 and tags from stage 2 on): HYB >= 1 makes
    // edges 0..HYB-1 signal-delimited and edges HYB.. tagged; node HYB
    // converts -- it consumes Begin/End and stamps its outputs with the open
    // region's key (uniform over each of its ensembles).
    static constexpr bool TAGANY = TAG || HYB > 0;   // a tag ring exists
    template <int e> static constexpr bool TGE = TAG || (HYB > 0 && e >= HYB);   // edge e carries tags
    static constexpr int AGE = NA ? K - 1 : K;       // the aggregating node's input edge
    static constexpr uint32_t default_stage() { return TAG ? 256u : 512u; }
    static constexpr bool U8 = (AGG == 23 || AGG == 25);   // text stream: byte elements
    static constexpr bool EMIT = (AGG == 24 || AGG == 25); // element-wise exit instead of an aggregate (§8 f3)
    static constexpr bool PAIR = (AGG == 25);        // taxi stage 2: parse the pair at each surviving open brace
    static constexpr uint32_t ESZ = U8 ? 1u : 4u;    // element size in the Q0 ring (bytes)
    // INPLACE (4-byte elements): every data queue Q_0..Q_NQ lives in ONE ring.
    // Positions of all edges share the ring's coordinates and each FILTER/
    // TRANSFORM node writes its survivors behind its own read head (stable
    // compaction never outruns the reads: t_{e+1} <= h_e), so queue space is
    // implied and a sweep can move a whole ring of items.
    // Leftover partial ensembles are moved up behind the next head when the
    // dead space between queues grows (relocate()).  Byte streams (text) keep
    // one ring per queue: 1-byte inputs become 4-byte items.
    static constexpr bool INPLACE = !U8;
    __host__ __device__ static constexpr uint32_t q0_bytes(uint32_t ring) { return (ring * ESZ + 15u) & ~15u; }
    // per-instance shared header: [0,64) TMA barriers, [64,160) node counters
    // (u32 x 24: data firings, full firings, items, signals per node),
    // [160,288) RS_FLAG_PROFILE cycle counters (u64 x 16)
    // parent-context value of the open region per node (PARENT_LT): in the
    // profile area [160, 288) of the production kernels (no profiling code),
    // after it in the debug (TR) ones
    static constexpr uint32_t BASE_HDR = TR ? 320 : 288;
    static constexpr uint32_t HDR = CTX ? BASE_HDR + 128 : BASE_HDR;   // CTX: + 32-word key scratch
    static constexpr uint32_t CNT_OFF = 64, PROF_OFF = 160, PV_OFF = TR ? 288 : 160, SCR_OFF = BASE_HDR;

    const KParams &P;
    const int lane;
    const uint32_t lt;             // %lanemask_lt
    // shared-memory rings
    uint8_t *base;                 // this instance's shared-memory window
    uint64_t *bar;                 // [nstg] TMA stage barriers
    uint32_t qmask, smask, qcap, scap;
    uint32_t sblk, ring0;          // Q0: TMA stage size (elements) and ring capacity (nstg stages)
    uint32_t nstg, nsh;            // TMA stages in the ring (power of 2) and log2

    // Edge e (node e -> node e+1).  Kept as named scalars (not arrays) so the
    // whole state lives in registers.
    struct EdgeS {
        uint32_t qh, qt;       // data queue head/tail (monotone positions)
        uint32_t sh, st;       // signal queue head/tail
        uint32_t sent;         // sender: items emitted since last signal
        uint32_t cur;          // receiver: current credit counter
        bool xfer;             // the head signal's credit already moved into cur
    };
    EdgeS E0, E1, E2, E3, E4;

    template <int e> __device__ __forceinline__ EdgeS &E() {
        static_assert(e >= 0 && e <= 4, "edge index");
        if constexpr (e == 0) return E0; else if constexpr (e == 1) return E1; else if constexpr (e == 2) return E2;
        else if constexpr (e == 3) return E3; else return E4;
    }
    template <int e> __device__ __forceinline__ const EdgeS &E() const {
        return const_cast<Pipe *>(this)->template E<e>();
    }
    // node counters live in the shared header (lane 0 updates them)
    __device__ __forceinline__ void stat_add(int n, int f, uint32_t v) const {
        if (lane == 0) reinterpret_cast<uint32_t *>(base + CNT_OFF)[4 * n + f] += v;
    }
    __device__ __forceinline__ void pcnt(int i, unsigned long long v) const {
        if (lane == 0) reinterpret_cast<unsigned long long *>(base + PROF_OFF)[i] += v;
    }
    // ring addresses: Q0 (ring0 items) then -- separate-queue layout only --
    // Q_1..Q_NQ (qcap items), each followed by its tag ring in the tagged
    // strategy, then the signal rings.  In-place: every Q_e is the Q0 ring.
    static constexpr uint32_t NQS = INPLACE ? 0 : NQ;   // separate shared-memory queues
    template <int e> __device__ __forceinline__ uint32_t *Q() const {
        if constexpr (SPL && e > K) return reinterpret_cast<uint32_t *>(base + HDR + q0_bytes(ring0) + (e - K - 1) * qcap * 4);
        else if constexpr (e == 0 || INPLACE) return reinterpret_cast<uint32_t *>(base + HDR);
        else return reinterpret_cast<uint32_t *>(base + HDR + q0_bytes(ring0) + (TAGANY ? ring0 * 4 : 0) +
                                                 (e - 1) * qcap * 4 * (TAGANY ? 2 : 1));
    }
    template <int e> __device__ __forceinline__ uint32_t *T() const {
        if constexpr (!TAGANY) return nullptr;
        else if constexpr (e == 0 || INPLACE) return reinterpret_cast<uint32_t *>(base + HDR + q0_bytes(ring0));
        else return Q<e>() + qcap;
    }
    template <int e> __device__ __forceinline__ uint2 *S() const {
        return reinterpret_cast<uint2 *>(base + HDR + q0_bytes(ring0) + (TAGANY ? ring0 * 4 : 0) + NQS * qcap * 4 * (TAGANY ? 2 : 1) +
                                         NLQ * qcap * 4) +
               e * scap;
    }
    // ring index mask of edge e's queue
    template <int e> __device__ __forceinline__ uint32_t qm() const {
        return (SPL && e > K) ? qmask : ((e == 0 || INPLACE) ? ring0 - 1 : qmask);
    }

    Chunk F0, F1;                      // chunk being enumerated, chunk staged next
    bool claims_done, enum_done;
    uint32_t stg_j, landed_j;          // TMA stages issued / known landed
    uint32_t pidx;                     // next part of F0 to enumerate
    bool begun;                        // Begin of part pidx already emitted
    // part-info cache: lane i holds part pc_base + i of F0
    uint32_t pc_base;
    bool pc_valid;
    uint32_t pc_ps, pc_pe;         // part bounds relative to F0.beg (a chunk spans < 2^31 elements)
    uint32_t pc_key;
    // aggregate state
    A acc;             // per-lane partial accumulator
    uint32_t akey;     // tagged: key of the running (carry) region; 0xffffffff = none
    A carry;           // tagged: uniform partial of the carry region
    long long adelta;  // text aggregate: index offset of the current part (see part_delta)
    uint32_t dkey;     // tagged text aggregate: key whose delta is cached in adelta (per lane)
    uint32_t fkept;    // fused aggregate: items that reached it (per lane; node statistics)
    bool adirty = false;   // SH: the generic data phase folded into acc since the last Begin/End
    uint32_t ekey = 0; // EMIT, signal strategy: key of the open region
    uint32_t ckey = 0; // hybrid converter node: key of the open region
    // RS_OP_SUM_I64_DROPS: stage 1 counts the items it drops per region part and
    // announces the count with a signal of its own just before End
    static constexpr bool UDROP = (AGG == 27);
    uint32_t udrop = 0;
    long long base0, offR, off0;
    uint32_t nchunks;
    uint32_t q_start[K + 1 + NLQ]; // initial queue positions (edge 0 may start at the chunk-0 pad)
    // RS_FLAG_PROFILE: cycles spent per node (0 = enumerate, 1..K+1, K+2 = TMA wait)
    // RS_FLAG_PROFILE cycle counters exist in the debug (TR) instantiations
    // only: the production kernels carry no profiling code (i-cache).
    static constexpr bool prof = TR;

    __device__ __forceinline__ Pipe(const KParams &p, uint8_t *smem, int lane_)
        : P(p), lane(lane_), lt(lanemask_lt()) {

        qcap = P.qcap;
        scap = P.scap;
        qmask = qcap - 1;
        smask = scap - 1;
        sblk = P.q0_stage;
        ring0 = P.ring0;
        nstg = ring0 / sblk;
        nsh = 31 - __clz(nstg);
        base = smem;
        bar = reinterpret_cast<uint64_t *>(smem);
        E0 = E1 = E2 = E3 = E4 = EdgeS{0u, 0u, 0u, 0u, 0u, 0u, false};
#pragma unroll
        for (int e = 0; e <= K + NLQ; ++e) q_start[e] = 0u;
        for (int i = 16 + lane; i < (int)(HDR / 4); i += 32) reinterpret_cast<uint32_t *>(base)[i] = 0u;   // counters + profile
        __syncwarp();
        F0.k = F1.k = -1;
        claims_done = enum_done = false;
        stg_j = landed_j = 0;
        pidx = 0;
        begun = false;
        pc_valid = false;
        pc_base = 0;
        acc = AT::id();
        carry = AT::id();
        akey = 0xffffffffu;
        adelta = 0;
        dkey = 0xffffffffu;
        fkept = 0;
        base0 = P.hdr->base0;
        offR = P.hdr->offR;
        off0 = P.hdr->off0;
        nchunks = P.hdr->nchunks;
    }

    __host__ __device__ static constexpr uint32_t smem_bytes(uint32_t qcap, uint32_t scap, uint32_t ring) {
        return HDR + q0_bytes(ring) + (TAGANY ? ring * 4 : 0) + NQS * qcap * 4 * (TAGANY ? 2 : 1) +
               (TAG ? 0 : NSG * scap * 8) + NLQ * (qcap * 4 + scap * 8);
    }
    // Ring capacity: 4 TMA stages; in-place, the configured queue capacity
    // (the one ring all queues share), at most NSTMAX stages, and at least one
    // partial ensemble per queue plus a stage, so the TMA can always make
    // progress (leftovers of < w items per queue are all that can stay behind;
    // see relocate()).
    __host__ static uint32_t ring_for(uint32_t sblk, uint32_t qcap) {
        uint32_t r = 4 * sblk;
        if (INPLACE) {
            while (r < qcap && r < NSTMAX * sblk) r <<= 1;
            while (r < (NQ + 1) * (uint32_t)W + sblk) r <<= 1;
        }
        return r;
    }

    // ---------------------------------------------------------- chunks
    __device__ __forceinline__ void load_chunk(Chunk &c, int32_t k, uint32_t pos) const {
        c.k = k;
        const long long k1 = P.hdr->k1;
        c.beg = (k == 0) ? off0 : chunk_start(base0, k, P.C, k1);
        long long e = chunk_start(base0, k + 1, P.C, k1);
        c.end = e > offR ? offR : e;
        c.pos = pos;
        c.fr0 = P.chunk_fr[k];
        c.fr1 = P.chunk_fr[k + 1];
        c.head = (k > 0) && (P.off[c.fr0] > c.beg);
    }
    __device__ __forceinline__ static uint32_t flen(const Chunk &c) { return (uint32_t)(c.end - c.beg); }

    // Claim the next chunk of the parent stream (atomics, no locks).
    __device__ __forceinline__ int32_t claim() {
        uint32_t k = 0;
        if (lane == 0) k = atomicAdd(&P.hdr->claim, 1u);
        k = __shfl_sync(kFull, k, 0);
        return k < nchunks ? (int32_t)k : -1;
    }

    // Issue TMA stage stg_j (positions [j*sblk, (j+1)*sblk)) from chunk c.
    __device__ __forceinline__ void issue_stage(const Chunk &c) {
        constexpr uint32_t AL = 16u / ESZ;                     // elements per 16-byte block
        const uint32_t j = stg_j;
        const uint32_t p0 = j * sblk;
        const long long src = c.beg + (long long)p0 - (long long)c.pos;   // 16-byte aligned element index
        uint8_t *dst = reinterpret_cast<uint8_t *>(Q<0>()) + (size_t)(p0 & (ring0 - 1)) * ESZ;
        uint64_t *b = &bar[j & (nstg - 1)];
        uint32_t ntma = sblk;
        if ((int)(p0 + sblk - (c.pos + flen(c))) > 0) {   // (positions wrap: compare differences)
            // the chunk's last (short) stage; a stage inside the chunk ends at or
            // before c.end <= n_elems, so whole stages need none of this
            const uint32_t n = c.pos + flen(c) - p0;
            const long long lim = (P.n_elems - src) & ~(long long)(AL - 1);   // whole 16-byte blocks in the array
            ntma = (uint32_t)min((long long)((n + AL - 1) & ~(AL - 1)), lim);
            // tail elements that a 16-byte copy cannot reach without overrunning n_elems
            const int tail = (int)n - (int)ntma;
            if (tail > 0 && lane < tail) {
                if constexpr (U8) dst[ntma + lane] = P.elems[src + ntma + lane];
                else reinterpret_cast<uint32_t *>(dst)[ntma + lane] =
                    __ldg(reinterpret_cast<const uint32_t *>(P.elems) + src + ntma + lane);
            }
        }
        // the slots being refilled may hold items lanes wrote through the generic
        // proxy (in-place rings: compaction, relocation; the byte tail above);
        // order those writes before the async-proxy (TMA) writes of this stage
        if constexpr (INPLACE) fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            if constexpr (!INPLACE) fence_proxy_async();
            if (ntma) {
                mbar_arrive_expect_tx(b, ntma * ESZ);
                tma_load_1d(dst, P.elems + src * ESZ, ntma * ESZ, b);
            } else {
                mbar_arrive(b);
            }
        }
        stg_j = j + 1;
    }

    // Keep the Q0 ring full: prefetch element blocks ahead of the enumerate node.
    // all queue positions start at `pos` (in-place rings share one coordinate system)
    template <int e = 0>
    __device__ __forceinline__ void start_at(uint32_t pos) {
        if constexpr (e <= K) {
            if (e == 0 || INPLACE) { E<e>().qh = E<e>().qt = pos; q_start[e] = pos; }
            start_at<e + 1>(pos);
        }
    }
    // oldest live ring position: in-place, the last data queue lies behind all others
    __device__ __forceinline__ uint32_t oldest() const { return INPLACE ? E<NQ>().qh : E<0>().qh; }

    __device__ __forceinline__ void refill() {
        for (;;) {
            if ((int)((stg_j + 1) * sblk - (oldest() + ring0)) > 0) return;   // ring slots still in use
            const uint32_t sp = stg_j * sblk;
            if (F0.k >= 0 && (int)(sp - (F0.pos + flen(F0))) < 0) { issue_stage(F0); continue; }   // (wrap-safe)
            if (F1.k >= 0 && (int)(sp - (F1.pos + flen(F1))) < 0) { issue_stage(F1); continue; }
            if (F1.k >= 0 || claims_done) return;
            const int32_t k = claim();
            if (k < 0) { claims_done = true; return; }
            if (F0.k < 0) {
                const uint32_t pos = (k == 0) ? (uint32_t)(off0 - base0) : sp;
                if (k == 0 && stg_j == 0) start_at(pos);
                load_chunk(F0, k, pos);
                pidx = 0;
                begun = false;
                pc_valid = false;
            } else {
                load_chunk(F1, k, F0.pos + flen(F0));
            }
        }
    }

    __device__ __forceinline__ void shift() {
        F0 = F1;
        F1.k = -1;
        pidx = 0;
        begun = false;
        pc_valid = false;
    }

    // ------------------------------------------------------ enumerate
    // Part qi of chunk F0: [start, end) elements and its key (region id, or a
    // partial slot for the chunk's head part / a tail part crossing the chunk end).
    // Part bounds are returned relative to F0.beg (32-bit: the enumerate loop's
    // scans, shuffles and compares then stay 32-bit -- smaller code).
    __device__ __forceinline__ void part_info(uint32_t qi, bool valid, uint32_t &ps, uint32_t &pe, uint32_t &key) const {
        const uint32_t len = flen(F0);
        ps = pe = len;
        key = 0;
        if (!valid) return;
        if (F0.head && qi == 0) {
            ps = 0;
            const long long e = P.off[F0.fr0];
            pe = e < F0.end ? (uint32_t)(e - F0.beg) : len;
            key = SLOT | (uint32_t)(2 * F0.k);
        } else {
            const uint32_t r = F0.fr0 + qi - (F0.head ? 1u : 0u);
            ps = (uint32_t)(P.off[r] - F0.beg);
            const long long e = P.off[r + 1];
            if (e > F0.end) { pe = len; key = SLOT | (uint32_t)(2 * F0.k + 1); }
            else { pe = (uint32_t)(e - F0.beg); key = r; }
        }
    }

    // getParent() (Fig. 5) for PARENT_LT nodes: under the
    // signal strategy every ensemble lies in the open region (P:464-465,
    // P:495-499), so a node loads its region's context once, on Begin, and
    // the filter compares each item with that one value.
    __device__ __forceinline__ uint32_t region_key(uint32_t key) const {
        if (!(key & SLOT)) return key;
        const uint32_t slot = key & ~SLOT, k = slot >> 1;
        return ((slot & 1u) ? P.chunk_fr[k + 1] : P.chunk_fr[k]) - 1u;
    }
    __device__ __forceinline__ void set_pv(int n, uint32_t key) const {
        load_pv(P.ctx, P.chunk_fr, key, reinterpret_cast<uint32_t *>(base + PV_OFF) + n);
    }
    __device__ __forceinline__ uint32_t pvn(int n) const { return reinterpret_cast<const uint32_t *>(base + PV_OFF)[n]; }

    // Sender rule for one signal on edge e: S empty -> |Q|;
    // otherwise items emitted since the tail signal.  Resets the counter.
    template <int e>
    // kind: 0 (Begin), END_BIT, or USER_BIT (a node-generated signal, payload `key`)
    __device__ __forceinline__ void push_signal(uint32_t key, uint32_t kind, uint32_t credit_rule2) {
        const uint32_t credit = (E<e>().sh == E<e>().st) ? (E<e>().qt - E<e>().qh) : credit_rule2;
        if (lane == 0) S<e>()[E<e>().st & smask] = make_uint2(key, credit | kind);
        E<e>().st += 1;
        E<e>().sent = 0;
    }

    // CTX: append boundary {key, stamp} to edge e's signal queue.
    template <int e>
    __device__ __forceinline__ void push_ctx(uint32_t key, uint32_t stamp) {
        if (lane == 0) S<e>()[E<e>().st & smask] = make_uint2(key, stamp);
        E<e>().st += 1;
    }

    // One enumerate firing (resumable mid-region):
    // emit F0's parts -- Begin, element indices (as staged element values),
    // End -- as far as staged data and signal space allow.  Up to 32 parts are
    // handled per step, one per lane, with warp scans over their counts.
    __device__ __forceinline__ bool enumerate() {
        bool prog = false;
        refill();
        for (;;) {
            if (F0.k < 0) {
                if (F1.k >= 0) { shift(); continue; }
                if (claims_done) enum_done = true;
                return prog;
            }
            const uint32_t np = (F0.head ? 1u : 0u) + (F0.fr1 - F0.fr0);
            if (pidx >= np) {            // chunk fully enumerated
                shift();
                refill();
                prog = true;
                continue;
            }
            const uint32_t fend = F0.pos + flen(F0), sj = stg_j * sblk;
            const uint32_t lim_pos = (int)(sj - fend) < 0 ? sj : fend;   // min, wrap-safe
            const uint32_t avail = lim_pos - E<0>().qt;
            if (!pc_valid || pidx >= pc_base + 32) {
                pc_base = pidx;
                pc_valid = true;
                part_info(pidx + lane, pidx + lane < np, pc_ps, pc_pe, pc_key);
            }
            const uint32_t d = pidx - pc_base;
            const uint32_t e_next = E<0>().qt - F0.pos;              // next element, relative to F0.beg
            if (TAG || begun) {
                // long part in progress: stream the staged items without the per-part scan
                const uint32_t pe0 = __shfl_sync(kFull, pc_pe, d);
                if ((int)(pe0 - e_next) > (int)avail) {
                    if (avail == 0) return prog;
                    if constexpr (TAG) write_tags_uniform(__shfl_sync(kFull, pc_key, d), avail);
                    E<0>().qt += avail;
                    E<0>().sent += avail;
                    __syncwarp();
                    return true;
                }
            }
            uint32_t ps = __shfl_down_sync(kFull, pc_ps, d);
            uint32_t pe = __shfl_down_sync(kFull, pc_pe, d);
            uint32_t key = __shfl_down_sync(kFull, pc_key, d);
            const bool valid = (lane + d < 32) && (pidx + lane < np);
            if (!valid) ps = pe = flen(F0);
            if (lane == 0 && ps < e_next) ps = e_next;     // resume inside part pidx
            const uint32_t cnt = pe - ps;
            uint32_t cum = cnt;
            const uint32_t sig = TAG ? 0u : ((lane == 0 && begun) ? (CTX ? 0u : 1u) : (CTX ? 1u : 2u));
            uint32_t scum = sig;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const uint32_t o = __shfl_up_sync(kFull, cum, dd);
                const uint32_t so = __shfl_up_sync(kFull, scum, dd);
                if (lane >= dd) { cum += o; scum += so; }
            }
            const uint32_t sfree = TAG ? 0xffffffffu : scap - (E<0>().st - E<0>().sh);
            const bool fits = valid && (cum <= avail) && (scum <= sfree);
            const uint32_t m = __popc(__ballot_sync(kFull, fits));
            if (m > 0) {
                const uint32_t tot = __shfl_sync(kFull, cum, m - 1);
                if constexpr (CTX) {
                    // one boundary per part not yet begun, stamped with the edge-0
                    // count of the part's first item
                    const uint32_t base_cnt = E<0>().qt - q_start[0];
                    if (lane < (int)m && sig) S<0>()[(E<0>().st + scum - sig) & smask] = make_uint2(key, base_cnt + cum - cnt);
                    E<0>().st += __shfl_sync(kFull, scum, m - 1);
                } else if constexpr (!TAG) {
                    // Begin_i, End_i of parts 0..m-1 in stream order.
                    const bool empty_at_start = (E<0>().sh == E<0>().st);
                    const uint32_t qlen0 = E<0>().qt - E<0>().qh;
                    const uint32_t sexcl = scum - sig;
                    if (lane < (int)m) {
                        uint32_t slot = E<0>().st + sexcl;
                        if (!(lane == 0 && begun)) {
                            // first signal of the step: rule (1) if S was empty, else
                            // rule (2) (items since the previous signal); later Begins
                            // follow an End directly: credit 0.
                            const uint32_t c = (lane == 0) ? (empty_at_start ? qlen0 : E<0>().sent) : 0u;
                            S<0>()[slot & smask] = make_uint2(key, c);
                            slot++;
                        }
                        // End_i: items of part i since its Begin (rule 2), or rule (1) when
                        // part 0 began earlier and S has since been drained by the receiver.
                        uint32_t c = cnt;
                        if (lane == 0 && begun) c = empty_at_start ? (qlen0 + cnt) : (E<0>().sent + cnt);
                        S<0>()[slot & smask] = make_uint2(key, c | END_BIT);
                    }
                    const uint32_t nsig = __shfl_sync(kFull, scum, m - 1);
                    E<0>().st += nsig;
                    E<0>().sent = 0;
                } else {
                    write_tags(m, cum, cnt, key, tot);
                }
                E<0>().qt += tot;
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
                    if (scap - (E<0>().st - E<0>().sh) == 0) return prog;
                    if constexpr (CTX) push_ctx<0>(key0, E<0>().qt - q_start[0]);
                    else push_signal<0>(key0, 0u, E<0>().sent);
                    begun = true;
                    did = true;
                }
            }
            const uint32_t k = min(avail, cnt0);
            if (k > 0) {
                if constexpr (TAG) write_tags_uniform(key0, k);
                E<0>().qt += k;
                E<0>().sent += k;
                did = true;
            }
            if constexpr (CTX) {
                if (k == cnt0) { pidx++; begun = false; did = true; }
            } else if constexpr (!TAG) {
                if (k == cnt0 && scap - (E<0>().st - E<0>().sh) > 0) {
                    push_signal<0>(key0, END_BIT, E<0>().sent);
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

    // Tagged enumerate: every emitted item carries its parent's key
    // (P:258-261).  Positions E<0>().qt .. E<0>().qt+tot-1 belong to parts
    // 0..m-1 of this step (lane i holds part i's inclusive end `cum`).
    __device__ __forceinline__ void write_tags(uint32_t m, uint32_t cum, uint32_t cnt, uint32_t key, uint32_t tot) {
        if (m == 1 || __shfl_sync(kFull, cnt, 0) == tot) {
            write_tags_uniform(__shfl_sync(kFull, key, 0), tot);
            return;
        }
        const uint32_t excl = cum - cnt;
        // Lane i writes short part i's tags itself (<= 8 items) and the warp writes
        // each longer part 32 tags at a time -- when the long parts average 64
        // items or more (Zipf-like mixes, U{0..2L} with L >= 64).  Otherwise
        // (many parts of a few dozen items) every item finds its part by a
        // binary search over the parts' starts.
        const bool lng = (uint32_t)lane < m && cnt > 8u;
        uint32_t lg = __ballot_sync(kFull, lng);
        if (tot >= 64u * __popc(lg)) {
            const uint32_t maxs = __reduce_max_sync(kFull, ((uint32_t)lane < m && !lng) ? cnt : 0u);
#pragma unroll 1
            for (uint32_t r = 0; r < maxs; ++r)
                if ((uint32_t)lane < m && !lng && r < cnt) T<0>()[(E<0>().qt + excl + r) & (ring0 - 1)] = key;
#pragma unroll 1
            while (lg) {
                const uint32_t j = __ffs(lg) - 1;
                lg &= lg - 1u;
                const uint32_t x = __shfl_sync(kFull, excl, j), c = __shfl_sync(kFull, cnt, j), k = __shfl_sync(kFull, key, j);
                for (uint32_t i = lane; i < c; i += 32) T<0>()[(E<0>().qt + x + i) & (ring0 - 1)] = k;
            }
            return;
        }
        for (uint32_t base = 0; base < tot; base += 32) {
            const uint32_t rel = base + lane;
            int lo = 0;      // largest part i < m with excl_i <= rel
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1) {
                const int cand = lo + step;
                const uint32_t ex = __shfl_sync(kFull, excl, cand < 32 ? cand : 31);
                if (cand < (int)m && ex <= rel) lo = cand;
            }
            const uint32_t k = __shfl_sync(kFull, key, lo);
            if (rel < tot) T<0>()[(E<0>().qt + rel) & (ring0 - 1)] = k;
        }
    }
    __device__ __forceinline__ void write_tags_uniform(uint32_t key, uint32_t k) {
        // (not unrolled: the instruction cache is the tagged kernel's binding limit)
#pragma unroll 1
        for (uint32_t i = lane; i < k; i += 32) T<0>()[(E<0>().qt + i) & (ring0 - 1)] = key;
    }

    // ---------------------------------------------------------- stages
    __device__ __forceinline__ uint32_t landed_pos() {
        while (landed_j < stg_j && mbar_test_uniform(&bar[landed_j & (nstg - 1)], (landed_j >> nsh) & 1u)) landed_j++;
        return landed_j * sblk;
    }

    // Receiver admissible count on edge e, applying rule (2b).
    template <int e>
    __device__ __forceinline__ uint32_t admissible(bool &spend) {
        spend = E<e>().sh != E<e>().st;
        const uint32_t ql = E<e>().qt - E<e>().qh;
        if (!spend) return ql;
        if (E<e>().cur == 0 && !E<e>().xfer) {
            const uint32_t c = S<e>()[E<e>().sh & smask].y & CREDIT_MASK;
            if (c > 0) { E<e>().cur = c; E<e>().xfer = true; }
        }
        return min(ql, E<e>().cur);
    }

    template <int n, class Op>
    __device__ __forceinline__ void filter_full(const uint32_t *in, const uint32_t *tin, uint32_t imask, uint32_t h,
                                                uint32_t nens, const Op op) {
        uint32_t tl;
        if constexpr (INPLACE && !TAGANY) tl = filter_batch_ip(Q<0>(), ring0 - 1, h, nens, E<n>().qt, op);
        else tl = filter_batch<TGE<n - 1>, Op, U8 && n == 1>(in, tin, imask, h, nens, Q<n>(), T<n>(), qm<n>(),
                                                             E<n>().qt, op, lt, P.C - 1);
        if constexpr (UDROP && n == 1) udrop += nens * W - (tl - E<n>().qt);
        if constexpr (HYB > 0 && n == HYB) stamp_tags<n>(E<n>().qt, tl);
        E<n>().sent += tl - E<n>().qt;
        E<n>().qt = tl;
    }
    // hybrid converter: its outputs [t0, t1) carry the open region's key
    template <int n>
    __device__ __forceinline__ void stamp_tags(uint32_t t0, uint32_t t1) {
        uint32_t *tq = T<n>();
        for (uint32_t i = t0 + lane; i - t0 < t1 - t0; i += 32) tq[i & qm<n>()] = ckey;
        __syncwarp();
    }

    static constexpr bool AGG_U8IN = U8 && (NA ? K == 1 : K == 0);   // aggregate reads the byte ring directly
    __device__ __forceinline__ uint32_t agg_load(const uint32_t *in, uint32_t pos, uint32_t imask) const {
        return load_item<AGG_U8IN>(in, pos, imask, P.C - 1);
    }

    // Index-within-region offset of a part (text aggregate): delta = chunk base
    // - region start, so i = delta + (item >> 8).
    __device__ __forceinline__ long long part_delta(uint32_t key) const {
        uint32_t r;
        long long cb;
        if (key & SLOT) {
            const uint32_t slot = key & ~SLOT, k = slot >> 1;
            r = ((slot & 1u) ? P.chunk_fr[k + 1] : P.chunk_fr[k]) - 1u;
            cb = base0 + (long long)k * P.C;
        } else {
            r = key;
            const long long k = (P.off[r] - base0) >> (__ffs(P.C) - 1);   // C is a power of 2; off[r] >= base0
            cb = base0 + k * P.C;
        }
        return cb - P.off[r];
    }

    template <int NS>
    __device__ __forceinline__ void agg_slices(const uint32_t *in, uint32_t imask, uint32_t h) {
        uint32_t v[NS];
        if (!AGG_U8IN && ((h & imask) + NS * 32) <= imask + 1) {
            const uint32_t *src = in + (h & imask) + lane;
#pragma unroll
            for (int j = 0; j < NS; ++j) v[j] = src[32 * j];
        } else {
#pragma unroll
            for (int j = 0; j < NS; ++j) v[j] = agg_load(in, h + 32 * j + lane, imask);
        }
        A part = AT::lift_i(v[0], adelta);
#pragma unroll
        for (int j = 1; j < NS; ++j) part = AT::comb(part, AT::lift_i(v[j], adelta));
        acc = AT::comb(acc, part);
    }
    __device__ __forceinline__ void agg_full(const uint32_t *in, uint32_t imask, uint32_t h, uint32_t nens) {
        if constexpr (EMIT) {
            for (uint32_t k = 0; k < nens; ++k) emit_ens(in, nullptr, imask, h + k * W, W, OpAll{});
            return;
        }
        uint32_t k = 0;
        for (; k + 2 <= nens; k += 2, h += 2 * W) agg_slices<2 * IPL>(in, imask, h);
        if (k < nens) agg_slices<IPL>(in, imask, h);
    }

    // Text (byte stream), single-stage fused CLASS + aggregate, single-member
    // class (SWAR): an ensemble of w = 128 bytes is read as one
    // 32-bit word per lane (lane l holds bytes 4l .. 4l+3; a funnel shift
    // realigns an unaligned head), tested four bytes at a time (match4), and
    // only the sparse survivors are lifted (the hash of their index within
    // the line) -- instead of a byte load, a table lookup and a select per
    // byte.  e < w: a partial ensemble (bytes 4l + k >= e masked off).  The
    // fold is commutative, so the lane-major item order does not matter.
    __device__ __forceinline__ void swar_ens(const uint32_t *in, uint32_t imask, uint32_t h, uint32_t e,
                                             const OpClass1 &op) {
        const uint32_t *wring = in;                      // the byte ring as words (size a multiple of 16 bytes)
        const uint32_t wmask = imask >> 2;
        const uint32_t a = h & 3u;
        const uint32_t wi = ((h >> 2) + lane) & wmask;
        uint32_t w = wring[wi];
        if (a) w = __funnelshift_r(w, wring[(wi + 1) & wmask], 8u * a);
        uint32_t m = op.match4(w);
        if (e < (uint32_t)W) {
            const int valid = (int)e - 4 * lane;         // bytes of this lane inside the ensemble
            m &= valid >= 4 ? 0xffffffffu : (valid <= 0 ? 0u : (0xffffffffu >> (32 - 8 * valid)));
        }
        fkept += __popc(m);
        const uint32_t cm = P.C - 1;
        while (__any_sync(kFull, m != 0)) {
            if (m) {
                const uint32_t bit = __ffs(m) - 1;       // 8k + 7 for byte k
                m &= m - 1u;
                const uint32_t k = bit >> 3;
                const uint32_t pos = h + 4u * lane + k;
                const uint32_t v = ((w >> (8u * k)) & 0xffu) | ((pos & cm) << 8);
                acc = AT::comb(acc, AT::lift_i(v, adelta));
            }
        }
    }

    // NG (4 or 8) full ensembles of the text stream at once (NG x 128 bytes,
    // still NG firings of the fused node inside one region): lane l tests its
    // word of each (match4), the survivor masks are packed into one mask
    // (bit 4j + b = byte b of ensemble j), and the survivors of all NG are
    // lifted in one divergent walk -- far fewer iterations than NG separate
    // walks.  Every survivor is the class byte c itself
    // (single-member class), so only its position is needed; the count half
    // of the aggregate adds the popcount once.
    template <int NG>
    __device__ __forceinline__ void swar_group(const uint32_t *in, uint32_t imask, uint32_t h, const OpClass1 &op) {
        const uint32_t wmask = imask >> 2;
        const uint32_t a = h & 3u;
        const uint32_t wi = (h >> 2) + lane;
        uint32_t pk = 0;
#pragma unroll
        for (int j = 0; j < NG; ++j) {
            uint32_t w = in[(wi + 32u * j) & wmask];
            if (a) w = __funnelshift_r(w, in[(wi + 32u * j + 1u) & wmask], 8u * a);
            // 0x80 per matching byte -> one bit per byte (bits 0..3) -> nibble j
            const uint32_t m = (op.match4(w) >> 7) * 0x00204081u;   // bytes' bits gathered in bits 21..24
            pk |= ((m >> 21) & 0xfu) << (4 * j);
        }
        const uint32_t nk = __popc(pk);
        fkept += nk;
        acc.x += nk;
        const uint32_t cm = P.C - 1, c = op.c4 & 0xffu;
        while (__any_sync(kFull, pk != 0)) {
            if (pk) {
                const uint32_t bit = __ffs(pk) - 1;
                pk &= pk - 1u;
                const uint32_t pos = h + ((bit >> 2) << 7) + 4u * lane + (bit & 3u);
                acc.y ^= AT::lift_i(c | ((pos & cm) << 8), adelta).y;
            }
        }
    }

    // Fused node K, full ensembles (signal strategy): apply the op, fold the
    // survivors into the per-lane accumulator (isGood + a::run).
    template <class Op>
    __device__ __forceinline__ void fused_full(const uint32_t *in, uint32_t imask, uint32_t h, uint32_t nens, const Op op) {
        if constexpr (EMIT) {
            for (uint32_t k = 0; k < nens; ++k) emit_ens(in, nullptr, imask, h + k * W, W, op);
            return;
        }
        if constexpr (K == 1 && AGG_U8IN && AT::heavy && std::is_same<Op, OpClass1>::value) {
            uint32_t k = 0;
            for (; k + 8 <= nens; k += 8, h += 8 * W) swar_group<8>(in, imask, h, op);
            for (; k + 4 <= nens; k += 4, h += 4 * W) swar_group<4>(in, imask, h, op);
            for (; k < nens; ++k, h += W) swar_ens(in, imask, h, W, op);
            return;
        }
        if constexpr (K == 1) {
            // single-stage pipeline: inline (no other stage code competes for the
            // instruction cache; fewer registers -> more instances per SM)
            for (uint32_t k = 0; k < nens; ++k, h += W) {
                uint32_t v[IPL];
#pragma unroll
                for (int j = 0; j < IPL; ++j) v[j] = agg_load(in, h + 32 * j + lane, imask);
                if constexpr (AT::heavy) {
                    uint32_t km = 0;
#pragma unroll
                    for (int j = 0; j < IPL; ++j) km |= op(v[j]) ? 1u << j : 0u;
                    fkept += __popc(km);
                    acc = fold_kept<AT>(acc, v, km, adelta);
                } else {
                    A part = AT::id();
#pragma unroll
                    for (int j = 0; j < IPL; ++j) {
                        const bool keep = op(v[j]);
                        fkept += keep ? 1u : 0u;
                        if (keep) part = AT::comb(part, AT::lift_i(v[j], adelta));
                    }
                    acc = AT::comb(acc, part);
                }
            }
            return;
        }
        FusedAcc<AT> r;
        if constexpr (INPLACE && !AT::heavy) r = fused_batch_ip<AT, Op>(in, imask, h, nens, op, FusedAcc<AT>{acc, fkept});
        else r = fused_batch<AT, Op, AGG_U8IN>(in, imask, h, nens, op, adelta, P.C - 1, FusedAcc<AT>{acc, fkept});
        acc = r.acc;
        fkept = r.kept;
    }
    template <class Op>
    __device__ __forceinline__ void fused_run(const uint32_t *in, const uint32_t *tin, uint32_t imask, uint32_t h,
                                              uint32_t nens, const Op op) {
        if constexpr (!TGE<AGE>) fused_full(in, imask, h, nens, op);
        else
            for (uint32_t k = 0; k < nens; ++k) {
                if constexpr (AT::heavy)
                    if (tagged_heavy_run(in, tin, imask, h + k * W, op)) continue;
                agg_tagged(in, tin, imask, h + k * W, W, op);
            }
    }

    // Tagged strategy, heavy aggregate (the text hash): a full ensemble whose
    // items all continue the carry region folds like the signal strategy's
    // fused node -- survivors are sparse, so only each lane's first and second
    // survivor are lifted under warp-uniform guards (fold_kept) instead of a
    // predicated hash per slot.  Returns false (nothing consumed) otherwise.
    template <class Op>
    __device__ __forceinline__ bool tagged_heavy_run(const uint32_t *in, const uint32_t *tin, uint32_t imask,
                                                     uint32_t h, const Op op) {
        bool same = akey != 0xffffffffu;
#pragma unroll
        for (int j = 0; j < IPL; ++j) same = same && tin[(h + 32 * j + lane) & imask] == akey;
        if (!__all_sync(kFull, same)) return false;
        if constexpr (U8) {
            if (__any_sync(kFull, dkey != akey)) {
                const long long d = part_delta(akey);
                dkey = akey;
                adelta = d;
            }
        }
        uint32_t v[IPL], km = 0;
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
            v[j] = agg_load(in, h + 32 * j + lane, imask);
            km |= op(v[j]) ? 1u << j : 0u;
        }
        if constexpr (NA) fkept += __popc(km);
        acc = fold_kept<AT>(acc, v, km, adelta);
        return true;
    }

    template <int n>
    __device__ __forceinline__ void run_full(const uint32_t *in, const uint32_t *tin, uint32_t imask, uint32_t h,
                                             uint32_t nens) {
        if constexpr (n == K + 1) {
            if constexpr (!TGE<K>) {
                agg_full(in, imask, h, nens);
            } else {
                for (uint32_t k = 0; k < nens; ++k) agg_tagged(in, tin, imask, h + k * W, W, OpAll{});
            }
        } else if constexpr (NA && n == K) {
            with_op_k(P.st[n - 1], pvn(n), [&](auto op) { fused_run(in, tin, imask, h, nens, op); });
        } else {
            with_op_k(P.st[n - 1], pvn(n), [&](auto op) { filter_full<n>(in, tin, imask, h, nens, op); });
            __syncwarp();
        }
    }

    // Calls f(op) with stage sp's op as its specialised functor -- one switch
    // per firing, not per item.  Only the ops the host accepts for this
    // kernel's element type are compiled in (i32/u32: HASH_LT, LT_U32,
    // AFFINE_I32, PARENT_LT; f32: HASH_LT, LT_U32, SCALE_F32, PARENT_LT;
    // u8: CLASS): unused op code would only dilute the instruction cache.
    static constexpr bool EU8 = U8, EF32 = (AGG == 21);
    template <class F>
    __device__ __forceinline__ void with_op_k(const StageP &sp, uint32_t pv, F &&f) const {
        if constexpr (EU8) {
            if (sp.a & 0x100u) f(OpClass1{(sp.a & 0xffu) * 0x01010101u});
            else f(OpClass{sp.table});
        } else {
            switch (sp.op) {
                case RS_OP_PARENT_LT: f(OpLt{pv, false}); break;   // pv = the open region's context (getParent)
                case RS_OP_HASH_LT:
                    if (sp.b >= 256) f(OpAll{});
                    else f(OpHash{sp.a, sp.b << 24});
                    break;
                case RS_OP_LT_U32:
                    if (sp.table[0]) f(OpAll{});
                    else f(OpLt{sp.b, false});
                    break;
                default:
                    if constexpr (EF32) f(OpScale{__uint_as_float(sp.a)});
                    else f(OpAffine{sp.a, sp.b});
                    break;
            }
        }
    }

    // ------------------------------------------ short-region batches (SH)
    // Regions shorter than an ensemble (the left of the paper's sweep,
    // P:568-589) make the signal strategy fire one partial ensemble and two
    // signals per region at every node.  SH kernels keep that firing sequence
    // (every ensemble bounded by its signal's credit; each signal
    // consumed after exactly the items before it, Lemma 1) but run
    // the per-signal bookkeeping warp-parallel: lane j holds pending signal j
    // of the input edge (one warp load), the segment before it (the items its
    // credit counts) is fired as one partial ensemble, and the forwarded
    // signals are written with one warp store, lane j's credit being the
    // survivors of segment j (sender rule 2; rule 1 for the first
    // when the output signal queue was empty).  The fused aggregate
    // folds each ensemble with two warp reductions (SUM_I64: 16-bit halves of
    // the lane sums, exact) and stores the region's total at its End.
    template <int n>
    __device__ __forceinline__ bool try_short(uint32_t avail) {
        if (P.st[n - 1].op == RS_OP_PARENT_LT) return false;   // per-region context: the general pass
        bool r = false;
        with_op_k(P.st[n - 1], 0u, [&](auto op) { r = short_batch<n>(op, avail); });
        return r;
    }
    // One segment (< w items at h) through the fused node's op, folded and
    // reduced over the warp with REDUX: SUM_I64 from the 16-bit halves of the
    // lane sums (exact), COUNT_MIN_U32 as a sum and a min.
    template <class Op>
    __device__ __forceinline__ A seg_fold(const uint32_t *ring, uint32_t m, uint32_t h, uint32_t ej, const Op &op) {
        if constexpr (AGG == 20) {
            long long ls = 0;
            for (uint32_t o = 0; o < ej; o += 32u) {
                const uint32_t idx = o + lane;
                uint32_t x = idx < ej ? ring[(h + idx) & m] : 0u;
                if (idx < ej && op(x)) {
                    ls += (int)x;
                    ++fkept;
                }
            }
            // each lane sum = (ls >> 16) * 2^16 + (ls & 0xffff), both halves small
            const int lo = __reduce_add_sync(kFull, (int)((uint32_t)ls & 0xffffu));
            const int hi = __reduce_add_sync(kFull, (int)(ls >> 16));
            return (A)((long long)hi * 65536ll + (long long)lo);
        } else {
            uint32_t c = 0, mn = 0xffffffffu;
            for (uint32_t o = 0; o < ej; o += 32u) {
                const uint32_t idx = o + lane;
                uint32_t x = idx < ej ? ring[(h + idx) & m] : 0u;
                if (idx < ej && op(x)) {
                    ++c;
                    mn = min(mn, x);
                }
            }
            fkept += c;
            return make_uint2(__reduce_add_sync(kFull, c), __reduce_min_sync(kFull, mn));
        }
    }
    template <int n, class Op>
    __device__ __forceinline__ bool short_batch(const Op op, uint32_t avail) {
        constexpr int ei = n - 1;
        constexpr bool AGGN = NA && n == K;
        // cheap test first: the head segment must be shorter than an ensemble and
        // all present (otherwise the general pass runs: full ensembles, or wait)
        {
            const uint32_t c0 = E<ei>().xfer ? E<ei>().cur : (S<ei>()[E<ei>().sh & smask].y & CREDIT_MASK);
            if (c0 >= (uint32_t)W || c0 > avail) return false;
        }
        const uint32_t np = E<ei>().st - E<ei>().sh;
        uint2 sg = make_uint2(0u, 0u);
        if ((uint32_t)lane < np) sg = S<ei>()[(E<ei>().sh + lane) & smask];
        // segment j = the items signal j's credit counts: the rest of a
        // transferred head credit, else the signal's own credit
        uint32_t e = sg.y & CREDIT_MASK;
        if (lane == 0 && E<ei>().xfer) e = E<ei>().cur;
        uint32_t cum = e;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, cum, d);
            if (lane >= d) cum += o;
        }
        bool ok = (uint32_t)lane < np && e < (uint32_t)W && cum <= avail;
        if constexpr (!AGGN) ok = ok && (uint32_t)lane < scap - (E<n>().st - E<n>().sh);   // forwarded signals fit
        const uint32_t bad = ~__ballot_sync(kFull, ok);
        const uint32_t k = bad ? (uint32_t)__ffs(bad) - 1u : 32u;   // leading run of batchable signals
        if (k == 0) return false;
        uint32_t *ring = Q<0>();
        const uint32_t m = ring0 - 1;
        const uint32_t h0 = E<ei>().qh;
        const uint32_t excl = cum - e;                 // lane j: segment j starts at h0 + excl
        // the non-empty segments, in stream order (back-to-back signals have none)
        uint32_t nz = __ballot_sync(kFull, e != 0) & (k == 32u ? 0xffffffffu : ((1u << k) - 1u));
        const uint32_t nparts = __popc(nz);
        if constexpr (!AGGN) {
            const uint32_t tl_in = E<n>().qt;
            uint32_t tl = tl_in, sj = 0;
            while (nz) {
                const uint32_t j = __ffs(nz) - 1;
                nz &= nz - 1u;
                const uint32_t ej = __shfl_sync(kFull, e, j);
                const uint32_t h = h0 + __shfl_sync(kFull, excl, j);
                uint32_t t2;
                if (ej <= 32u) {               // one slice, inline
                    const bool act = (uint32_t)lane < ej;
                    uint32_t v = act ? ring[(h + lane) & m] : 0u;
                    __syncwarp();              // every lane's reads before the stores
                    const bool keep = act && op(v);
                    const uint32_t mk = __ballot_sync(kFull, keep);
                    if (keep) ring[(tl + __popc(mk & lt)) & m] = v;
                    t2 = tl + __popc(mk);
                } else {
                    t2 = partial_stage_ip(op, ring, m, h, ej, tl);
                }
                if ((uint32_t)lane == j) sj = t2 - tl;
                tl = t2;
            }
            __syncwarp();
            uint32_t c = sj;                   // rule 2: survivors since the previous signal
            if (lane == 0) c = (E<n>().sh == E<n>().st) ? (tl_in + sj - E<n>().qh) : (E<n>().sent + sj);
            if ((uint32_t)lane < k) S<n>()[(E<n>().st + lane) & smask] = make_uint2(sg.x, c | (sg.y & END_BIT));
            E<n>().st += k;
            E<n>().sent = 0;
            E<n>().qt = tl;
        } else {
            static_assert(!SH || AGG == 20 || AGG == 22, "short-region batches are built for SUM_I64, COUNT_MIN_U32");
            // lane j: the fold of segment j (its region's items in this batch)
            A rv = AT::id();
            if (adirty) {                      // the head End closes a region the general pass began folding
                const A t = warp_reduce<AT>(acc);
                if (lane == 0) rv = t;
                acc = AT::id();
                adirty = false;
            }
            while (nz) {
                const uint32_t j = __ffs(nz) - 1;
                nz &= nz - 1u;
                const uint32_t ej = __shfl_sync(kFull, e, j);
                const uint32_t h = h0 + __shfl_sync(kFull, excl, j);
                const A t = seg_fold(ring, m, h, ej, op);
                if ((uint32_t)lane == j) rv = AT::comb(rv, t);
            }
            // a::end of every region closed in the batch: push(acc); Begin: identity
            if ((uint32_t)lane < k && (sg.y & END_BIT)) store_key(sg.x, rv);
        }
        E<ei>().qh = h0 + __shfl_sync(kFull, cum, k - 1);
        E<ei>().sh += k;
        E<ei>().cur = 0;
        E<ei>().xfer = false;
        stat_add(n, 0, nparts);
        stat_add(n, 1, __shfl_sync(kFull, cum, k - 1));
        __syncwarp();
        return true;
    }

    // Fire node n (1..K+1) repeatedly while it can make progress: data phase,
    // then signal phase, full-first (A8).
    template <int n>
    __device__ __forceinline__ bool fire(bool drained) {
        constexpr int ei = n - 1;          // input edge
        constexpr bool AGGN = (n == K + 1) || (NA && n == K);   // node n performs the aggregate's actions
        const uint32_t imask = qm<ei>();
        const uint32_t *in = Q<ei>();
        const uint32_t *tin = T<ei>();
        bool prog = false;
        uint32_t ready_lim = 0;
        if (ei == 0) ready_lim = landed_pos();
        for (;;) {
            if constexpr (SH && !TGE<ei>) {
                // short regions: a warp-parallel batch of signals and the partial
                // ensembles they bound (short_batch); the general pass below runs
                // whenever the head segment is an ensemble or longer
                if (E<ei>().sh != E<ei>().st) {
                    uint32_t av = E<ei>().qt - E<ei>().qh;
                    if (ei == 0) {
                        if ((int)(ready_lim - E<0>().qh) < (int)av) ready_lim = landed_pos();
                        const int rdy = (int)(ready_lim - E<0>().qh);
                        av = rdy <= 0 ? 0u : min(av, (uint32_t)rdy);
                    }
                    if (try_short<n>(av)) {
                        prog = true;
                        continue;
                    }
                }
            }
            bool spend;
            const uint32_t a = admissible<ei>(spend);
            uint32_t ar = a;
            if (ei == 0) {
                // only items whose TMA stage has landed may be read
                if ((int)(ready_lim - E<0>().qh) < (int)ar) ready_lim = landed_pos();
                const int rdy = (int)(ready_lim - E<0>().qh);
                ar = rdy <= 0 ? 0u : min(ar, (uint32_t)rdy);
            }
            uint32_t space = 0xffffffffu;
            if constexpr (!AGGN && !INPLACE) space = qcap - (E<n>().qt - E<n>().qh);   // in-place: implied
            uint32_t lim = min(ar, space);
            uint32_t arem = a;
            bool did = false;
            if (lim >= (uint32_t)W) {
                // as many full ensembles as the credit / data / space allow
                const uint32_t nens = lim / W;
                if constexpr (TR) if (P.trace) trace_ens(n, in, imask, E<ei>().qh, nens * W);
                run_full<n>(in, tin, imask, E<ei>().qh, nens);
                if constexpr (SH && AGGN) adirty = true;
                E<ei>().qh += nens * W;
                if (spend) E<ei>().cur -= nens * W;
                lim -= nens * W;
                arem -= nens * W;
                did = true;
            }
            // then at most one partial ensemble, in the same pass
            if (lim > 0) {
                const bool bounded = spend && lim == E<ei>().cur;      // ensemble <= credit
                const bool dr = drained && lim == arem;
                if (bounded || dr) {
                    if constexpr (TR) if (P.trace) trace_ens(n, in, imask, E<ei>().qh, lim);
                    run_partial<n>(in, tin, imask, E<ei>().qh, lim);
                    if constexpr (SH && AGGN) adirty = true;
                    E<ei>().qh += lim;
                    if (spend) E<ei>().cur -= lim;
                    stat_add(n, 0, 1u);            // partial ensembles and their items; full
                    stat_add(n, 1, lim);           // ensembles are derived at exit
                    did = true;
                }
            }
            // signal phase: only with the counter at 0.  Back-to-back
            // signals (credit 0, A4) are consumed in one pass; the first later
            // signal with a positive credit moves it into the counter (rule 2b)
            // so the next data phase starts without re-reading the queue.
            if (TGE<ei> || !spend || E<ei>().cur != 0) {
                // no signal to consume: the data phase took everything admissible
                // (what is left is < w items, or waits for its credit) and nothing
                // upstream runs meanwhile -- another pass could only find newly
                // landed TMA stages, which the next sweep picks up
                prog |= did;
                break;
            }
            uint32_t nsig = 0;
            for (;;) {
                if constexpr (!AGGN && !TGE<n>) {
                    // (the drop-count generator may push two signals: its own, then End)
                    if (scap - (E<n>().st - E<n>().sh) < ((UDROP && n == 1) ? 2u : 1u)) break;   // output signal queue full
                }
                const uint2 hs = S<ei>()[E<ei>().sh & smask];
                E<ei>().sh++;
                E<ei>().xfer = false;
                ++nsig;
                const bool is_end = (hs.y & END_BIT) != 0;
                if constexpr (UDROP) {
                    if (hs.y & USER_BIT) {                // a node-generated signal
                        if constexpr (AGGN) {
                            if (lane == 0) acc.y += hs.x;  // the aggregate records the payload
                        } else {
                            push_signal<n>(hs.x, USER_BIT, E<n>().sent);   // forwarded in stream position
                        }
                        if (E<ei>().sh == E<ei>().st) break;
                        const uint32_t c2 = S<ei>()[E<ei>().sh & smask].y & CREDIT_MASK;
                        if (c2 > 0) {
                            E<ei>().cur = c2;
                            E<ei>().xfer = true;
                            break;
                        }
                        continue;
                    }
                    if constexpr (n == 1 && !AGGN) {
                        // stage 1 generates a signal of its own before forwarding End:
                        // the items it dropped in this region (part)
                        if (!is_end) udrop = 0;
                        else push_signal<n>(udrop, USER_BIT, E<n>().sent);
                    }
                }
                if constexpr (TR) if (P.trace) trace_event(n, is_end ? TR_END : TR_BEGIN, hs.x, 0u, 0u, 0u);
                if constexpr (n <= K) {
                    if (!is_end && P.st[n - 1].op == RS_OP_PARENT_LT) set_pv(n, hs.x);
                }
                if constexpr (AGGN) {
                    if constexpr (EMIT) {
                        if (!is_end) ekey = hs.x;   // items until End belong to this region
                    } else if (!is_end) {        // a::begin: acc = identity
                        acc = AT::id();
                        if constexpr (U8) adelta = part_delta(hs.x);
                    } else {                     // a::end: push(acc)
                        const A v = warp_reduce<AT>(acc);
                        if (lane == 0) store_key(hs.x, v);
                        acc = AT::id();
                    }
                    if constexpr (SH) adirty = false;
                } else if constexpr (TGE<n>) {
                    if (!is_end) ckey = hs.x;    // hybrid converter: outputs carry this key as their tag
                } else {
                    push_signal<n>(hs.x, is_end ? END_BIT : 0u, E<n>().sent);   // forwarded with a fresh credit
                }
                if (E<ei>().sh == E<ei>().st) break;
                const uint32_t c = S<ei>()[E<ei>().sh & smask].y & CREDIT_MASK;
                if (c > 0) {
                    E<ei>().cur = c;
                    E<ei>().xfer = true;
                    break;
                }
            }
            if (nsig == 0 && !did) break;
            prog = true;
        }
        __syncwarp();
        return prog;
    }

    // ------------------------------------------- element-wise exit (EMIT)
    // RS_NODE_EMIT (§8 f3; "a stream of results derived from
    // individual elements, stripped of their parent context"): every item of
    // an ensemble that passes the node's op is written to the global output
    // as (value, region).  One atomic per ensemble reserves the slots; the
    // survivors are compacted into them with the same ballot/popc prefix as a
    // filter.  Signal strategy: the region is the open one (uniform over the
    // ensemble); tagged: each item's tag.
    // Taxi stage 2: the open brace at global byte index g starts a
    // well-formed pair iff it reads '{' D{1,9} ',' D{1,9} '}' before the line
    // end `lim` (reading R6); x, y are its fields.
    __device__ __forceinline__ bool parse_pair(long long g, long long lim, uint32_t &x, uint32_t &y) const {
        const uint8_t *b = P.elems;
        if (g >= lim || b[g] != '{') return false;
        long long i = g + 1;
        uint32_t f[2] = {0u, 0u};
#pragma unroll 1
        for (int k = 0; k < 2; ++k) {
            int nd = 0;
            uint8_t c = i < lim ? b[i] : 0;
            while (i < lim && c >= '0' && c <= '9' && nd <= 9) {
                f[k] = f[k] * 10u + (uint32_t)(c - '0');
                ++nd;
                ++i;
                c = i < lim ? b[i] : 0;
            }
            if (nd == 0 || nd > 9 || i >= lim || c != (k == 0 ? ',' : '}')) return false;
            ++i;
        }
        x = f[0];
        y = f[1];
        return true;
    }
    // First element of the chunk a part (key) lies in: positions within a
    // chunk are carried in the byte items (item >> 8), see load_item.
    __device__ __forceinline__ long long chunk_base(uint32_t key) const {
        const long long k = (key & SLOT) ? (long long)((key & ~SLOT) >> 1) : (P.off[key] - base0) / P.C;
        return base0 + k * (long long)P.C;
    }

    template <class Op>
    __device__ __forceinline__ void emit_ens(const uint32_t *in, const uint32_t *tin, uint32_t imask, uint32_t h,
                                             uint32_t e, const Op op) {
        uint32_t v[IPL], tg[IPL], mk[IPL], px[IPL], py[IPL];
        uint32_t total = 0;
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
            const uint32_t idx = j * 32 + lane;
            const bool act = idx < e;
            v[j] = act ? agg_load(in, h + idx, imask) : 0u;
            tg[j] = (TGE<AGE> && act) ? tin[(h + idx) & imask] : 0u;
            bool keep = act && op(v[j]);
            px[j] = py[j] = 0u;
            if constexpr (PAIR) {
                if (keep) {
                    const uint32_t key = TGE<AGE> ? tg[j] : ekey;
                    const uint32_t r = region_key(key);
                    keep = parse_pair(chunk_base(key) + (long long)(v[j] >> 8), P.off[r + 1], px[j], py[j]);
                }
            }
            mk[j] = __ballot_sync(kFull, keep);
            total += __popc(mk[j]);
        }
        if (total == 0) return;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(P.emit_n, (unsigned long long)total);
        base = __shfl_sync(kFull, base, 0);
        if (base + total > P.emit_cap && lane == 0) atomicCAS((int *)&P.hdr->err, 0, ERR_EMIT_FULL);
        const uint32_t ureg = TGE<AGE> ? 0u : region_key(ekey);
        uint32_t rel = 0;
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
            if ((mk[j] >> lane) & 1u) {
                const unsigned long long pos = base + rel + __popc(mk[j] & lt);
                if (pos < P.emit_cap) {
                    if constexpr (PAIR) {             // swapped: (y, x)
                        P.emit_vals[2 * pos] = py[j];
                        P.emit_vals[2 * pos + 1] = px[j];
                    } else {
                        P.emit_vals[pos] = v[j];
                    }
                    P.emit_regs[pos] = TGE<AGE> ? region_key(tg[j]) : ureg;
                }
            }
            rel += __popc(mk[j]);
        }
    }

    // ------------------------------------------------- trace mode (TR)
    // RS_FLAG_TRACE (§8(c) GPU trace-mode check): every node logs, in the
    // order it performs them, the Begin/End signals it consumes and each
    // ensemble it fires with the smallest and largest item value -- the test
    // feeds elements equal to their global index, so the host can check that
    // the events of each node form (Begin(r) ENSEMBLE* End(r))*, that every
    // item of an ensemble lies in the open region r (no mixed ensembles,
    // P:375-379) and that the items per bracket equal the oracle's count
    // (Lemma 1).  Only the trace instantiations contain this code.
    uint32_t tseq = 0;
    __device__ __forceinline__ void trace_event(uint32_t n, uint32_t type, uint32_t key, uint32_t cnt, uint32_t lo,
                                             uint32_t hi) {
        if (lane == 0) {
            const uint32_t i = atomicAdd(P.trace, 1u);
            if (i < P.trace_cap) {
                uint32_t *e = P.trace + 8 + 8 * (size_t)i;
                e[0] = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
                e[1] = tseq;
                e[2] = n | (type << 8);
                e[3] = key;
                e[4] = type == TR_ENSEMBLE ? 0u : region_key(key);
                e[5] = cnt;
                e[6] = lo;
                e[7] = hi;
            }
        }
        ++tseq;
        __syncwarp();
    }
    __device__ __forceinline__ void trace_ens(uint32_t n, const uint32_t *in, uint32_t imask, uint32_t h, uint32_t cnt) {
        for (uint32_t e0 = 0; e0 < cnt; e0 += W) {
            const uint32_t c = min((uint32_t)W, cnt - e0);
            uint32_t lo = 0xffffffffu, hi = 0u;
            for (uint32_t t = lane; t < c; t += 32) {
                const uint32_t v = in[(h + e0 + t) & imask];
                lo = min(lo, v);
                hi = max(hi, v);
            }
            lo = __reduce_min_sync(kFull, lo);
            hi = __reduce_max_sync(kFull, hi);
            trace_event(n, TR_ENSEMBLE, 0u, c, lo, hi);
        }
    }

    // --------------------------------------------------- fan-out (SPL)
    // A tree topology (Fig. 1b; §8 f4): the SPLIT node (node K+1)
    // sends every item of its ensembles to child A (its op holds) or child B
    // (it does not) -- two stable ballot/popc compactions into the children's
    // queues -- and forwards every signal to BOTH children, each with the
    // credit of its own edge (items sent to that child since its last signal,
    // P:304-312), so each child sees its own precisely delimited regions
    // (P:151-159).  The children are leaf AGGREGATEs (SUM_I64): A's sums go to
    // out.v0, B's to out.v1.
    unsigned long long lacc0 = 0, lacc1 = 0;    // leaf A / B per-lane partial sums
    template <class Op>
    __device__ __forceinline__ void split_ens(const Op &op, const uint32_t *in, uint32_t imask, uint32_t h, uint32_t e) {
        constexpr int ea = K + 1, eb = K + 2;
        uint32_t *qa = Q<ea>(), *qb = Q<eb>();
        uint32_t ta = E<ea>().qt, tb = E<eb>().qt;
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
            if ((uint32_t)j * 32u >= e) break;
            const bool act = (uint32_t)(j * 32 + lane) < e;
            uint32_t v = act ? in[(h + j * 32 + lane) & imask] : 0u;
            const bool keep = act && op(v);
            const uint32_t ka = __ballot_sync(kFull, keep), kb = __ballot_sync(kFull, act && !keep);
            if (keep) qa[(ta + __popc(ka & lt)) & qmask] = v;
            else if (act) qb[(tb + __popc(kb & lt)) & qmask] = v;
            ta += __popc(ka);
            tb += __popc(kb);
        }
        __syncwarp();
        E<ea>().sent += ta - E<ea>().qt;
        E<ea>().qt = ta;
        E<eb>().sent += tb - E<eb>().qt;
        E<eb>().qt = tb;
    }
    __device__ __forceinline__ bool fire_split(bool drained) {
        constexpr int ei = K, ea = K + 1, eb = K + 2, n = K + 1;
        const uint32_t imask = qm<ei>();
        const uint32_t *in = Q<ei>();
        bool prog = false;
        uint32_t ready_lim = 0;
        if (ei == 0) ready_lim = landed_pos();
        for (;;) {
            if constexpr (SH && !TGE<ei>) {
                // short regions: a warp-parallel batch of signals and the partial
                // ensembles they bound (short_batch); the general pass below runs
                // whenever the head segment is an ensemble or longer
                if (E<ei>().sh != E<ei>().st) {
                    uint32_t av = E<ei>().qt - E<ei>().qh;
                    if (ei == 0) {
                        if ((int)(ready_lim - E<0>().qh) < (int)av) ready_lim = landed_pos();
                        const int rdy = (int)(ready_lim - E<0>().qh);
                        av = rdy <= 0 ? 0u : min(av, (uint32_t)rdy);
                    }
                    if (try_short<n>(av)) {
                        prog = true;
                        continue;
                    }
                }
            }
            bool spend;
            const uint32_t a = admissible<ei>(spend);
            uint32_t ar = a;
            if (ei == 0) {
                if ((int)(ready_lim - E<0>().qh) < (int)ar) ready_lim = landed_pos();
                const int rdy = (int)(ready_lim - E<0>().qh);
                ar = rdy <= 0 ? 0u : min(ar, (uint32_t)rdy);
            }
            const uint32_t space = min(qcap - (E<ea>().qt - E<ea>().qh), qcap - (E<eb>().qt - E<eb>().qh));
            uint32_t lim = min(ar, space), arem = a;
            bool did = false;
            while (lim >= (uint32_t)W) {
                with_op_k(P.st[K], pvn(n), [&](auto op) { split_ens(op, in, imask, E<ei>().qh, W); });
                E<ei>().qh += W;
                if (spend) E<ei>().cur -= W;
                lim -= W;
                arem -= W;
                did = true;
            }
            if (lim > 0 && ((spend && lim == E<ei>().cur) || (drained && lim == arem))) {
                with_op_k(P.st[K], pvn(n), [&](auto op) { split_ens(op, in, imask, E<ei>().qh, lim); });
                E<ei>().qh += lim;
                if (spend) E<ei>().cur -= lim;
                stat_add(n, 0, 1u);
                stat_add(n, 1, lim);
                did = true;
            }
            if (!spend || E<ei>().cur != 0) {
                if (!did) break;
                prog = true;
                continue;
            }
            uint32_t nsig = 0;
            for (;;) {
                if (scap - (E<ea>().st - E<ea>().sh) == 0 || scap - (E<eb>().st - E<eb>().sh) == 0) break;
                const uint2 hs = S<ei>()[E<ei>().sh & smask];
                E<ei>().sh++;
                E<ei>().xfer = false;
                ++nsig;
                const bool is_end = (hs.y & END_BIT) != 0;
                if (!is_end && P.st[K].op == RS_OP_PARENT_LT) set_pv(n, hs.x);
                push_signal<ea>(hs.x, is_end ? END_BIT : 0u, E<ea>().sent);     // each child: its own credit
                push_signal<eb>(hs.x, is_end ? END_BIT : 0u, E<eb>().sent);
                if (E<ei>().sh == E<ei>().st) break;
                const uint32_t c = S<ei>()[E<ei>().sh & smask].y & CREDIT_MASK;
                if (c > 0) {
                    E<ei>().cur = c;
                    E<ei>().xfer = true;
                    break;
                }
            }
            if (nsig == 0 && !did) break;
            prog = true;
        }
        __syncwarp();
        return prog;
    }
    // leaf AGGREGATE on edge e (SUM_I64 of its items, per region)
    template <int e>
    __device__ __forceinline__ bool fire_leaf(bool drained) {
        constexpr int n = e + 1;
        constexpr bool B = (e == K + 2);
        unsigned long long &la = B ? lacc1 : lacc0;
        const uint32_t *in = Q<e>();
        bool prog = false;
        for (;;) {
            bool spend;
            const uint32_t a = admissible<e>(spend);
            uint32_t lim = a, arem = a, take = 0;
            bool did = false;
            if (lim >= (uint32_t)W) take = lim & ~(uint32_t)(W - 1);
            if (lim > take && ((spend && lim == E<e>().cur) || (drained && lim == arem))) {
                stat_add(n, 0, 1u);
                stat_add(n, 1, lim - take);
                take = lim;
            }
            if (take) {
                const uint32_t h = E<e>().qh;
                for (uint32_t i = lane; i < take; i += 32) la += (unsigned long long)(long long)(int)in[(h + i) & qmask];
                E<e>().qh += take;
                if (spend) E<e>().cur -= take;
                did = true;
            }
            if (!spend || E<e>().cur != 0) {
                if (!did) break;
                prog = true;
                continue;
            }
            uint32_t nsig = 0;
            for (;;) {
                const uint2 hs = S<e>()[E<e>().sh & smask];
                E<e>().sh++;
                E<e>().xfer = false;
                ++nsig;
                if (hs.y & END_BIT) {                 // a::end: this child's result for the region
                    unsigned long long v = la;
#pragma unroll
                    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(kFull, v, m);
                    if (lane == 0) {
                        const uint32_t key = hs.x;
                        unsigned long long *o = reinterpret_cast<unsigned long long *>(
                            (key & SLOT) ? (B ? P.part1 : P.part0) : (B ? P.out1 : P.out0));
                        o[key & ~SLOT] = v;
                    }
                }
                la = 0;                               // a::begin / after a::end
                if (E<e>().sh == E<e>().st) break;
                const uint32_t c = S<e>()[E<e>().sh & smask].y & CREDIT_MASK;
                if (c > 0) {
                    E<e>().cur = c;
                    E<e>().xfer = true;
                    break;
                }
            }
            if (nsig == 0 && !did) break;
            prog = true;
        }
        __syncwarp();
        return prog;
    }

    // ----------------------------------------------- per-lane context (CTX)
    // Close the open region (akey: uniform partial `carry` + per-lane `acc`)
    // and open `key` (a::end then a::begin).
    __device__ __forceinline__ void ctx_close(uint32_t key) {
        if (akey != 0xffffffffu) {
            const A v = AT::comb(carry, warp_reduce<AT>(acc));
            if (lane == 0) store_key(akey, v);
        }
        acc = AT::id();
        carry = AT::id();
        akey = key;
    }

    // Fire node n under CTX: full ensembles run across boundaries; a
    // boundary at the consumption point is forwarded (re-stamped) or, at the
    // aggregate, closes/opens a region; partial ensembles only at the drained
    // tail (full-first, A8).
    template <int n>
    __device__ __forceinline__ bool fire_ctx(bool drained) {
        constexpr int ei = n - 1;
        constexpr bool AGGN = (n == K + 1) || (NA && n == K);
        const uint32_t imask = qm<ei>();
        const uint32_t *in = Q<ei>();
        bool prog = false;
        uint32_t ready_lim = 0;
        if (ei == 0) ready_lim = landed_pos();
        for (;;) {
            const uint32_t a = E<ei>().qt - E<ei>().qh;
            uint32_t ar = a;
            if (ei == 0) {
                if ((int)(ready_lim - E<0>().qh) < (int)ar) ready_lim = landed_pos();
                const int rdy = (int)(ready_lim - E<0>().qh);
                ar = rdy <= 0 ? 0u : min(ar, (uint32_t)rdy);
            }
            const uint32_t cons = E<ei>().qh - q_start[ei];
            const bool sp = E<ei>().sh != E<ei>().st;
            uint2 hs = make_uint2(0u, 0u);
            if (sp) hs = S<ei>()[E<ei>().sh & smask];
            const uint32_t srel = sp ? hs.y - cons : 0xffffffffu;
            if (sp && srel == 0) {
                if constexpr (AGGN) {
                    ctx_close(hs.x);
                } else {
                    if (scap - (E<n>().st - E<n>().sh) == 0) break;
                    push_ctx<n>(hs.x, E<n>().qt - q_start[n]);
                }
                E<ei>().sh++;
                prog = true;
                continue;
            }
            uint32_t nclean = ar / W;
            if (sp) nclean = min(nclean, srel / W);
            if (nclean > 0) {
                run_full<n>(in, nullptr, imask, E<ei>().qh, nclean);
                E<ei>().qh += nclean * W;
                prog = true;
                continue;
            }
            const uint32_t e = min(ar, (uint32_t)W);
            if (e == 0) break;
            // a partial ensemble fires when the upstream is drained, or when the
            // input boundary queue is half full (runs of empty regions could
            // otherwise fill it while fewer than w items wait -- reading R3)
            if (e < (uint32_t)W && !(drained && e == a) && 2 * (E<ei>().st - E<ei>().sh) < scap) break;
            uint32_t done = e;
            if constexpr (AGGN) {
                if constexpr (n == K + 1) ctx_agg_ens(in, imask, E<ei>().qh, e, cons, OpAll{});
                else with_op_k(P.st[n - 1], 0u, [&](auto op) { ctx_agg_ens(in, imask, E<ei>().qh, e, cons, op); });
            } else {
                with_op_k(P.st[n - 1], 0u, [&](auto op) { done = ctx_filter_ens<n>(in, imask, E<ei>().qh, e, cons, op); });
            }
            if (done == 0) break;
            E<ei>().qh += done;
            if (done < (uint32_t)W) {
                stat_add(n, 0, 1u);
                stat_add(n, 1, done);
            }
            prog = true;
        }
        __syncwarp();
        return prog;
    }

    // CTX filter: one ensemble of e items at h (consumed count cons) with
    // boundaries strictly inside; the survivors are compacted as usual and each
    // inside boundary is forwarded with stamp = survivors before it.  When the
    // output signal queue cannot take all of them (runs of empty regions), the
    // ensemble is cut before the first boundary that does not fit.  Returns
    // the items consumed (0: the output signal queue is full).
    template <int n, class Op>
    __device__ __forceinline__ uint32_t ctx_filter_ens(const uint32_t *in, uint32_t imask, uint32_t h, uint32_t e,
                                                       uint32_t cons, const Op op) {
        constexpr int ei = n - 1;
        const uint32_t freeo = scap - (E<n>().st - E<n>().sh);
        // boundaries with cons < stamp < cons + e (stamps are non-decreasing)
        uint32_t nb = 0;
        for (;;) {
            const uint32_t i = E<ei>().sh + nb + lane;
            bool in_ens = false;
            if (i - E<ei>().sh < E<ei>().st - E<ei>().sh) in_ens = S<ei>()[i & smask].y - cons < e;
            const uint32_t b = __ballot_sync(kFull, in_ens);
            const uint32_t c = __popc(~b) ? (uint32_t)(__ffs(~b) - 1) : 32u;   // leading run of in-ensemble entries
            nb += c;
            if (c < 32 || nb > freeo) break;
        }
        if (nb > freeo) {
            if (freeo == 0) return 0u;
            e = S<ei>()[(E<ei>().sh + freeo) & smask].y - cons;     // cut before boundary #freeo
            nb = 0;                                                  // boundaries with rel < e (<= freeo)
            for (;;) {
                const uint32_t i = nb + lane;
                const bool in_ens = i < freeo && S<ei>()[(E<ei>().sh + i) & smask].y - cons < e;
                const uint32_t b = __ballot_sync(kFull, in_ens);
                const uint32_t c = __popc(~b) ? (uint32_t)(__ffs(~b) - 1) : 32u;
                nb += c;
                if (c < 32) break;
            }
        }
        const uint32_t qm_ = qm<n>();
        uint32_t *out = Q<n>();
        uint32_t tl = E<n>().qt;
        const uint32_t t0 = tl - q_start[n];
        uint32_t mk[IPL], v[IPL];
#pragma unroll
        for (int j = 0; j < IPL; ++j) v[j] = (j * 32 + lane) < e ? in[(h + j * 32 + lane) & imask] : 0u;
        __syncwarp();   // in-place rings: all reads before any compaction store
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
            const bool keep = (j * 32 + lane) < e && op(v[j]);
            mk[j] = __ballot_sync(kFull, keep);
            if (keep) out[(tl + __popc(mk[j] & lt)) & qm_] = v[j];
            tl += __popc(mk[j]);
        }
        // re-stamp the inside boundaries, 32 at a time
        for (uint32_t b0 = 0; b0 < nb; b0 += 32) {
            if (b0 + lane < nb) {
                const uint2 sg = S<ei>()[(E<ei>().sh + b0 + lane) & smask];
                const uint32_t rel = sg.y - cons;                  // 1 .. e-1
                const uint32_t j = rel >> 5, l = rel & 31u;
                uint32_t before = 0;
#pragma unroll
                for (int jj = 0; jj < IPL; ++jj) {
                    if ((uint32_t)jj < j) before += __popc(mk[jj]);
                    else if ((uint32_t)jj == j) before += __popc(mk[jj] & ((1u << l) - 1u));
                }
                S<n>()[(E<n>().st + b0 + lane) & smask] = make_uint2(sg.x, t0 + before);
            }
        }
        __syncwarp();
        E<ei>().sh += nb;
        E<n>().st += nb;
        E<n>().qt = tl;
        return e;
    }

    // CTX aggregate: one ensemble of e items at h (consumed count cons); each
    // 32-item slice folds its items into the region of the last boundary at or
    // before them (segmented like the tagged fold, keys computed per lane).
    template <class Op>
    __device__ __forceinline__ void ctx_agg_ens(const uint32_t *in, uint32_t imask, uint32_t h, uint32_t e,
                                                uint32_t cons, const Op op) {
        constexpr int ei = NA ? K - 1 : K;
        uint32_t *scr = reinterpret_cast<uint32_t *>(base + SCR_OFF);
#pragma unroll 1
        for (uint32_t j = 0; j * 32 < e; ++j) {
            const uint32_t p0 = cons + 32 * j;                     // consumed count at the slice start
            const uint32_t cntj = min(e - 32 * j, 32u);
            // boundaries exactly at the slice start: close/open in order (empty regions included)
            for (;;) {
                if (E<ei>().sh == E<ei>().st) break;
                const uint2 hs = S<ei>()[E<ei>().sh & smask];
                if (hs.y != p0) break;
                ctx_close(hs.x);
                E<ei>().sh++;
            }
            const bool act = lane < cntj;
            uint32_t x = act ? in[(h + 32 * j + lane) & imask] : 0u;
            const bool keep = act && op(x);
            if constexpr (NA) fkept += keep ? 1u : 0u;
            const A val = keep ? AT::lift_i(x, 0) : AT::id();
            // boundaries strictly inside the slice (rel 1..cntj-1)
            const uint32_t avail_s = E<ei>().st - E<ei>().sh;
            const uint2 sg = lane < avail_s ? S<ei>()[(E<ei>().sh + lane) & smask] : make_uint2(0u, 0xffffffffu);
            const uint32_t rel = sg.y - p0;
            const bool inb = lane < avail_s && rel < cntj;
            const uint32_t bm = __ballot_sync(kFull, inb);
            if (bm == 0) {
                acc = AT::comb(acc, val);                          // the slice continues the open region
                continue;
            }
            const uint32_t nb = __popc(bm);                        // in-slice boundaries are a prefix
            if (nb == 32) {
                // 32 or more boundaries in 32 items: one at a time in stream order
                ctx_agg_slice_serial(val, cntj, p0);
                continue;
            }
            const uint32_t nrel = __shfl_down_sync(kFull, rel, 1);
            // an empty region (same stamp as the next boundary): identity now (A1);
            // the last boundary of each stamp starts the segment
            const bool dup = inb && lane + 1 < nb && nrel == rel;
            if (dup) store_key(sg.x, AT::id());
            const bool eff = inb && !dup;
            if (eff) scr[rel] = sg.x;
            __syncwarp();
            const uint32_t hm = __reduce_or_sync(kFull, eff ? (1u << rel) : 0u);
            const uint32_t le = hm & lanemask_le();
            const int seg = le ? 31 - __clz(le) : -1;             // first lane of my segment (-1: open region)
            const uint32_t key = seg >= 0 ? scr[seg] : akey;
            __syncwarp();
            // fold the per-lane partials of the open region into `carry`
            carry = AT::comb(carry, warp_reduce<AT>(acc));
            acc = AT::id();
            A v = val;
            if constexpr (AT::group) {
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const A o = AT::shfl_up(v, d);
                    if (lane >= d) v = AT::comb(o, v);
                }
                const A before = AT::shfl(v, seg >= 1 ? seg - 1 : 0);
                if (seg >= 1) v = AT::sub(v, before);
            } else {
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const A o = AT::shfl_up(v, d);
                    if (lane - d >= seg && lane >= d) v = AT::comb(o, v);
                }
            }
            if (seg < 0) v = AT::comb(carry, v);
            const bool nexthead = (lane < 31) && ((hm >> (lane + 1)) & 1u);
            if (act && nexthead) {                                 // a segment ends inside the slice
                if (key != 0xffffffffu) store_key(key, v);
            }
            const int last = (int)cntj - 1;
            akey = __shfl_sync(kFull, key, last);
            carry = AT::shfl(v, last);
            E<ei>().sh += nb;
        }
    }

    // Slow path of ctx_agg_ens: every boundary inside the slice (any number,
    // empty regions included), one at a time in stream order.
    __device__ __forceinline__ void ctx_agg_slice_serial(A val, uint32_t cntj, uint32_t p0) {
        constexpr int ei = NA ? K - 1 : K;
        uint32_t from = 0;
        while (E<ei>().sh != E<ei>().st) {
            const uint2 hs = S<ei>()[E<ei>().sh & smask];
            const uint32_t rel = hs.y - p0;
            if (rel >= cntj) break;
            if (lane >= from && lane < rel) acc = AT::comb(acc, val);
            ctx_close(hs.x);
            E<ei>().sh++;
            from = rel;
        }
        if (lane >= from && lane < cntj) acc = AT::comb(acc, val);
    }

    // Scheduler state of a stuck instance (workspace bytes [64, 256), read by
    // a debugger): per edge qh, qt, sh, st, q_start, head signal word.
    template <int e = 0>
    __device__ __forceinline__ void dump_edges(uint32_t *d) {
        if constexpr (e <= K && e < 4) {
            d[8 + 6 * e + 0] = E<e>().qh; d[8 + 6 * e + 1] = E<e>().qt;
            d[8 + 6 * e + 2] = E<e>().sh; d[8 + 6 * e + 3] = E<e>().st;
            d[8 + 6 * e + 4] = q_start[e];
            d[8 + 6 * e + 5] = (E<e>().sh != E<e>().st) ? S<e>()[E<e>().sh & smask].y : 0xdeadu;
            dump_edges<e + 1>(d);
        }
    }
    __device__ __forceinline__ void watchdog_dump(uint32_t why) {   // (a noinline member would force the whole instance state into local memory)
        if constexpr (!U8) {   // (nvcc 12.9 cicc crashes on this body in the u8 instantiation with -lineinfo)
            uint32_t *d = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(P.hdr) + 64);
            d[0] = 0xd0d0u | (why << 16); d[1] = enum_done; d[2] = claims_done; d[3] = (uint32_t)F0.k; d[4] = stg_j;
            d[5] = landed_j; d[6] = blockIdx.x * 32 + (threadIdx.x >> 5); d[7] = scap;
            dump_edges<0>(d);
        }
    }

    __device__ __forceinline__ void store_key(uint32_t key, A v) {
        if (key & SLOT) AT::store(P.part0, P.part1, key & ~SLOT, v);
        else AT::store(P.out0, P.out1, key, v);
    }

    // One partial ensemble (signal-bounded or at the drained tail).
    template <int n>
    __device__ __forceinline__ void run_partial(const uint32_t *in, const uint32_t *tin, uint32_t imask, uint32_t h,
                                                uint32_t e) {
        if constexpr (n == K + 1) {
            if constexpr (!TGE<K> && EMIT) {
                emit_ens(in, nullptr, imask, h, e, OpAll{});
            } else if constexpr (!TGE<K>) {
#pragma unroll
                for (int j = 0; j < IPL; ++j) {
                    const uint32_t idx = j * 32 + lane;
                    if (idx < e) acc = AT::comb(acc, AT::lift_i(agg_load(in, h + idx, imask), adelta));
                }
            } else {
                agg_tagged(in, tin, imask, h, e, OpAll{});
            }
        } else if constexpr (NA && n == K) {
            if constexpr (!TGE<K - 1> && EMIT) {
                with_op_k(P.st[n - 1], pvn(n), [&](auto op) { emit_ens(in, nullptr, imask, h, e, op); });
            } else if constexpr (!TGE<K - 1>) {
                with_op_k(P.st[n - 1], pvn(n), [&](auto op) {
                    if constexpr (K == 1 && AGG_U8IN && AT::heavy && std::is_same<decltype(op), OpClass1>::value) {
                        swar_ens(in, imask, h, e, op);
                        return;
                    }
                    const FusedAcc<AT> r = fused_partial<AT, decltype(op), AGG_U8IN>(in, imask, h, e, op, adelta, P.C - 1,
                                                                                     FusedAcc<AT>{acc, fkept});
                    acc = r.acc;
                    fkept = r.kept;
                });
            } else {
                agg_tagged(in, tin, imask, h, e, OpDyn{&P.st[n - 1]});
            }
        } else {
            uint32_t tl = E<n>().qt;
            with_op_k(P.st[n - 1], pvn(n), [&](auto op) {
                if constexpr (INPLACE && !TAGANY) tl = partial_stage_ip(op, Q<0>(), ring0 - 1, h, e, tl);
                else tl = partial_stage<TGE<n - 1>, decltype(op), U8 && n == 1>(op, in, tin, imask, h, e, Q<n>(), T<n>(),
                                                                           qm<n>(), tl, lt, P.C - 1);
            });
            if constexpr (HYB > 0 && n == HYB) stamp_tags<n>(E<n>().qt, tl);
            if constexpr (UDROP && n == 1) udrop += e - (tl - E<n>().qt);
            E<n>().sent += tl - E<n>().qt;
            E<n>().qt = tl;
        }
    }

    // Region-id-keyed segmented reduction with a carry across ensembles
    // (tagged aggregate).  Ensembles may mix regions.
    template <class Op>
    __device__ __forceinline__ void agg_tagged(const uint32_t *in, const uint32_t *tin, uint32_t imask, uint32_t h,
                                               uint32_t e, const Op op) {
        if constexpr (EMIT) emit_ens(in, tin, imask, h, e, op);
        else agg_tagged_fold(in, tin, imask, h, e, op);
    }
    template <class Op>
    __device__ __forceinline__ void agg_tagged_fold(const uint32_t *in, const uint32_t *tin, uint32_t imask, uint32_t h,
                                                    uint32_t e, const Op op) {
        // fast path, unrolled: a full ensemble that continues the carry region
        // (the common case for long regions) folds without the segmented scan
        if (e == (uint32_t)W && akey != 0xffffffffu) {
            bool same = true;
#pragma unroll
            for (int j = 0; j < IPL; ++j) same = same && tin[(h + j * 32 + lane) & imask] == akey;
            if (__all_sync(kFull, same)) {
                if constexpr (U8) {
                    if (__any_sync(kFull, dkey != akey)) {
                        adelta = part_delta(akey);
                        dkey = akey;
                    }
                }
                A part = AT::id();
#pragma unroll
                for (int j = 0; j < IPL; ++j) {
                    uint32_t x = agg_load(in, h + j * 32 + lane, imask);
                    const bool keep = op(x);
                    if constexpr (NA) fkept += keep ? 1u : 0u;
                    if (keep) part = AT::comb(part, AT::lift_i(x, adelta));
                }
                acc = AT::comb(acc, part);
                return;
            }
        }
        // ensembles with region changes: one slice per iteration, not unrolled -- the
        // segmented fold is large and the tagged kernel is instruction-cache bound
        // (profiles/r2_k_pipeline_full_zipf_tagged.txt)
#pragma unroll 1
        for (int j = 0; j < IPL; ++j) {
            const int cntj = (int)e - j * 32;
            if (cntj <= 0) break;
            const bool act = lane < cntj;
            const uint32_t idx = j * 32 + lane;
            const uint32_t key = act ? tin[(h + idx) & imask] : 0xffffffffu;
            if constexpr (U8) {
                if (act && key != dkey) { dkey = key; adelta = part_delta(key); }
            }
            uint32_t x = act ? agg_load(in, h + idx, imask) : 0u;
            const bool keep = act && op(x);          // fused node K: its op; else pass-all
            if constexpr (NA) fkept += keep ? 1u : 0u;
            const A val = keep ? AT::lift_i(x, adelta) : AT::id();
            if (__all_sync(kFull, !act || key == akey)) {
                acc = AT::comb(acc, val);      // fast path: the whole slice continues the carry region
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
            if constexpr (AT::group) {
                // exact inverse (integer sum, count, xor): one unsegmented inclusive
                // scan, then my segment's prefix = P[lane] - P[first lane - 1]
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const A o = AT::shfl_up(v, d);
                    if (lane >= d) v = AT::comb(o, v);
                }
                const A before = AT::shfl(v, seg >= 1 ? seg - 1 : 0);
                if (seg >= 1) v = AT::sub(v, before);
            } else {
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const A o = AT::shfl_up(v, d);
                    if (lane - d >= seg && lane >= d) v = AT::comb(o, v);
                }
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

    __device__ __forceinline__ void flush_tagged() {
        carry = AT::comb(carry, warp_reduce<AT>(acc));
        acc = AT::id();
        if (lane == 0 && akey != 0xffffffffu) store_key(akey, carry);
        akey = 0xffffffffu;
        carry = AT::id();
    }

    template <int k = 0>
    __device__ __forceinline__ bool all_empty() const {
        if constexpr (k > K + NLQ) {
            return true;
        } else {
            return (E<k>().qh == E<k>().qt) && (E<k>().sh == E<k>().st) && all_empty<k + 1>();
        }
    }

    // In-place rings: close the dead space left by filtered-out items -- move
    // the (normally < w) items left in Q_e up to end right behind its
    // producer's read head h_{e-1}, nearest to Q0 first.  Queue contents and
    // counts are unchanged (credits and signal positions are counts), only the
    // ring coordinates of Q_e shift, which frees its old slots for the TMA.
    template <int e = 1>
    __device__ __forceinline__ void relocate() {
        if constexpr (INPLACE && e <= NQ) {
            const uint32_t shift = E<e - 1>().qh - E<e>().qt;
            if (shift != 0) {
                const uint32_t n = E<e>().qt - E<e>().qh;
                if (n != 0) move_items<TAGANY>(Q<0>(), T<0>(), E<e>().qt, n, shift, ring0 - 1);
                E<e>().qh += shift;
                E<e>().qt += shift;
                q_start[e] += shift;
            }
            relocate<e + 1>();
        }
    }

    template <int n>
    __device__ __forceinline__ bool fire_chain(bool drained) {
        if constexpr (SPL && n == K + 1) {
            bool p = fire_split(drained);
            const bool dn = drained && (E<K>().qh == E<K>().qt) && (E<K>().sh == E<K>().st);
            p |= fire_leaf<K + 1>(dn);
            p |= fire_leaf<K + 2>(dn);
            return p;
        } else if constexpr (n > (NA ? K : K + 1)) {
            return false;
        } else {
            const long long t0 = prof ? clock64() : 0;
            bool p;
            if constexpr (CTX) p = fire_ctx<n>(drained);
            else p = fire<n>(drained);
            if (prof) pcnt(n, clock64() - t0);
            const bool dn = drained && (E<n - 1>().qh == E<n - 1>().qt) && (E<n - 1>().sh == E<n - 1>().st);
            return fire_chain<n + 1>(dn) | p;
        }
    }

    // Node n's items = positions it consumed on edge n-1; its data firings =
    // full ensembles + partial ensembles (counted separately in the header).
    template <int n = 1>
    __device__ __forceinline__ void finish_counters(uint32_t fitems) {
        if constexpr (n <= K + 1 + NLQ) {
            if (lane == 0) {
                // c[0] = partial ensembles, c[1] = their items (accumulated in the run)
                uint32_t *c = reinterpret_cast<uint32_t *>(base + CNT_OFF) + 4 * n;
                const uint32_t items = E<n - 1>().qh - q_start[n - 1];
                const uint32_t full = (items - c[1]) / W;
                c[0] += full;
                c[1] = full;
                c[2] = items;
                c[3] = E<n - 1>().sh;                      // signals consumed
                if constexpr (NA && n == K + 1) {          // fused aggregate: node K's firings,
                    c[0] = c[-4];                          // the items that survived node K and
                    c[1] = c[-3];                          // the signals node K consumed
                    c[2] = fitems;
                    c[3] = E<K - 1>().sh;
                }
                if constexpr (n == 1) {                     // enumerate: items / signals emitted
                    c[-4 + 2] = E<0>().qt - q_start[0];
                    c[-4 + 3] = E<0>().st;
                }
            }
            finish_counters<n + 1>(fitems);
        }
    }
    __device__ __forceinline__ void flush_stats() {
        const uint32_t fitems = NA ? __reduce_add_sync(kFull, fkept) : 0u;
        finish_counters<1>(fitems);
        __syncwarp();
        if (lane < K + 2 + NLQ) {
            const uint32_t *c = reinterpret_cast<const uint32_t *>(base + CNT_OFF) + 4 * lane;
            unsigned long long *S = P.stats + 4 * lane;
#pragma unroll
            for (int f = 0; f < 4; ++f)
                if (c[f]) atomicAdd(S + f, (unsigned long long)c[f]);
        }
    }

    __device__ __forceinline__ void run() {
        if (lane == 0)
            for (uint32_t i = 0; i < nstg; ++i) mbar_init(&bar[i], 1);
        mbar_fence_init();
        __syncwarp();
        uint32_t idle = 0;
        for (;;) {
            const long long t0 = prof ? clock64() : 0;
            bool prog = enumerate();
            if (prof) { pcnt(0, clock64() - t0); pcnt(8, 1); }
            prog |= fire_chain<1>(enum_done);
            if (enum_done && all_empty()) break;
            if constexpr (INPLACE && NQ > 0)
                if (E<0>().qh - oldest() >= (ring0 >> 2)) relocate();
            if (prog) { idle = 0; continue; }
            // nothing fireable: wait for the oldest in-flight TMA stage
            if (landed_j < stg_j) {
                const long long tw = prof ? clock64() : 0;
                uint32_t spins = 0;
                while (!mbar_try_wait_uniform(&bar[landed_j & (nstg - 1)], (landed_j >> nsh) & 1u)) {
                    if (++spins > (1u << 24)) break;
                }
                if (spins > (1u << 24)) {
                    if (lane == 0 && atomicCAS((int *)&P.hdr->err, 0, ERR_WATCHDOG) == 0) watchdog_dump(1u);
                    break;
                }
                if (prof) { pcnt(K + 2, clock64() - tw); pcnt(9, 1); }
                continue;
            }
            if (++idle > 64) {
                if (lane == 0 && atomicCAS((int *)&P.hdr->err, 0, ERR_WATCHDOG) == 0) watchdog_dump(2u);
                break;
            }
        }
        if constexpr (TGE<AGE>) flush_tagged();
        if constexpr (CTX) ctx_close(0xffffffffu);
        // drain outstanding TMA stages before the CTA's shared memory is released
        for (uint32_t spins = 0; landed_j < stg_j && spins < (1u << 26); ++spins) {
            if (mbar_try_wait_uniform(&bar[landed_j & (nstg - 1)], (landed_j >> nsh) & 1u)) landed_j++;
        }
        __syncwarp();
        if (P.flags & RS_FLAG_STATS) flush_stats();
        if (prof && lane == 0) {
            // per-node cycles (enumerate, nodes 1..K+1, TMA wait), sweeps, waits
            unsigned long long *Pr = P.stats + 4 * (MAXK + 2);
            const unsigned long long *c = reinterpret_cast<const unsigned long long *>(base + PROF_OFF);
            for (int i = 0; i < 10; ++i) atomicAdd(Pr + i, c[i]);
            atomicAdd(Pr + 10, 1ull);
        }
    }
};

template <int K, int AGG, bool TAG, bool FUSE, bool CTX = false, bool TR = false, int HYB = 0, bool SPL = false,
          bool SH = false>
__global__ void __launch_bounds__(WPB_MAX * 32, 1) k_pipeline(const __grid_constant__ KParams P) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    using PP = Pipe<K, AGG, TAG, FUSE, CTX, TR, HYB, SPL, SH>;
    uint8_t *mine = smem + (size_t)warp * PP::smem_bytes(P.qcap, P.scap, P.ring0);
    if (P.hdr->err) return;
    if (P.auto_sel && P.hdr->sel != P.auto_sel - 1) return;   // AUTO: the other strategy's kernel runs
    if (P.short_sel && P.hdr->ssel != P.short_sel - 1) return; // the other (short / long region) kernel runs
    PP pipe(P, mine, lane);
    pipe.run();
}
