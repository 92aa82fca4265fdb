// rs_ws.cuh — warp-specialised pipeline instance (RS_FLAG_WARP_SPECIALIZED).
//
// One CTA = one pipeline instance; warp n runs node n continuously:
//   warp 0      ENUMERATE  (TMA staging of the element stream + Begin/End
//                           signals or tags, P:489-494 / P:692-697)
//   warps 1..K  FILTER / TRANSFORM stages (Fig. 5)
//   warp K+1    AGGREGATE  (begin/run/end)
// Nodes communicate only through the shared-memory data queues and signal
// queues of their edges.  Because producer and consumer now run
// concurrently, the sender's rule-(1) read of |Q| would race with
// the receiver; each signal therefore carries the sender's absolute emission
// position ("stamp").  When the signal reaches the head of S, the receiver
// sets its current credit counter to stamp - consumed (rule 2b)
// and decrements it per consumed item (rule 2a); it consumes the
// signal when the counter is 0.  This is the position form of the credit
// rules: it delivers every signal after exactly the items emitted
// before it (Lemma 1), which the oracle's interpreter pins.
// Ensembles never cross a pending signal and are full unless
// signal-bounded or at the drained tail (full-first, A8).
#pragma once

// Warp-uniform acquire load of a position word: lane 0 loads with acquire
// semantics, the value is broadcast, and __syncwarp orders the other lanes'
// subsequent reads after lane 0's acquire.
__device__ __forceinline__ uint32_t ld_acq(const uint32_t *p) {
    uint32_t v = 0;
    if ((threadIdx.x & 31u) == 0)
        asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    v = __shfl_sync(kFull, v, 0);
    __syncwarp();
    return v;
}
__device__ __forceinline__ void st_rel(uint32_t *p, uint32_t v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}

// Per-edge control words (shared memory).  tail/stail are written by the
// producer warp, head/shead by the consumer warp, done by the producer.
struct EdgeCtl {
    uint32_t tail, head, stail, shead, done, pad_[3];
};

template <int K, int AGG, bool TAG>
struct WS {
    using AT = AggT<AGG>;
    using A = typename AT::A;
    static constexpr int SBLK = TAG ? 256 : 512;     // elements per TMA stage
    static constexpr int RING0 = NST * SBLK;         // Q0 ring capacity (items)
    static constexpr int NW = K + 2;                 // warps per instance
    static constexpr int BMIN = 4;                   // preferred minimum ensembles per firing

    __host__ __device__ static constexpr uint32_t off_bar() { return 256; }
    __host__ __device__ static constexpr uint32_t off_q0() { return 384; }
    __host__ __device__ static constexpr uint32_t off_q(int e, uint32_t qcap) {
        return e == 0 ? off_q0() : off_q0() + RING0 * 4 * (TAG ? 2 : 1) + (e - 1) * qcap * 4 * (TAG ? 2 : 1);
    }
    __host__ __device__ static constexpr uint32_t off_s(int e, uint32_t qcap, uint32_t scap) {
        return off_q(K + 1, qcap) + e * scap * 16;
    }
    __host__ __device__ static constexpr uint32_t smem_bytes(uint32_t qcap, uint32_t scap) {
        return off_s(TAG ? 0 : K + 1, qcap, scap);
    }

    const KParams &P;
    uint8_t *base;
    const uint32_t lane, lt;
    const uint32_t qcap, qmask, scap, smask;

    __device__ __forceinline__ WS(const KParams &p, uint8_t *smem)
        : P(p), base(smem), lane(threadIdx.x & 31u), lt(lanemask_lt()), qcap(p.qcap), qmask(p.qcap - 1),
          scap(p.scap), smask(p.scap - 1) {}

    __device__ __forceinline__ EdgeCtl *ctl(int e) const { return reinterpret_cast<EdgeCtl *>(base) + e; }
    __device__ __forceinline__ uint64_t *bar() const { return reinterpret_cast<uint64_t *>(base + off_bar()); }
    __device__ __forceinline__ uint32_t *Q(int e) const { return reinterpret_cast<uint32_t *>(base + off_q(e, qcap)); }
    __device__ __forceinline__ uint32_t *T(int e) const {
        return TAG ? Q(e) + (e == 0 ? (uint32_t)RING0 : qcap) : nullptr;
    }
    __device__ __forceinline__ uint4 *S(int e) const { return reinterpret_cast<uint4 *>(base + off_s(e, qcap, scap)); }
    __device__ __forceinline__ uint32_t imask(int e) const { return e == 0 ? (uint32_t)(RING0 - 1) : qmask; }

    // No-progress watchdog: ~2^22 idle polls (seconds) -> error word, exit.
    __device__ __forceinline__ bool idle_wait(uint32_t &backoff, uint32_t &idle) const {
        backoff = backoff ? min(backoff * 2, 256u) : 32u;
        __nanosleep(backoff);
        if (++idle > (1u << 22)) {
            if (lane == 0) atomicCAS((int *)&P.hdr->err, 0, ERR_WATCHDOG);
            return false;
        }
        return P.hdr->err == 0 || idle < 16;
    }

    // Make this warp's shared-memory writes (queue items, tags, signal
    // entries -- written by any lane) visible before the position word that
    // announces them: the warp synchronises (memory-ordering among its lanes),
    // lane 0 releases the new position.  Consumers read position words with
    // ld.acquire before touching the items.
    __device__ __forceinline__ void publish(uint32_t *w, uint32_t v) const {
        __syncwarp();            // orders every lane's prior shared writes before lane 0's release
        if (lane == 0) st_rel(w, v);
    }

    __device__ __forceinline__ void store_key(uint32_t key, A v) const {
        if (key & SLOT) AT::store(P.part0, P.part1, key & ~SLOT, v);
        else AT::store(P.out0, P.out1, key, v);
    }

    __device__ __forceinline__ void flush_stats(int n, uint32_t nd, uint32_t nf, uint32_t ni, uint32_t ns) const {
        if ((P.flags & RS_FLAG_STATS) && lane == 0) {
            unsigned long long *S_ = P.stats + 4 * n;
            if (nd) atomicAdd(S_ + 0, (unsigned long long)nd);
            if (nf) atomicAdd(S_ + 1, (unsigned long long)nf);
            if (ni) atomicAdd(S_ + 2, (unsigned long long)ni);
            if (ns) atomicAdd(S_ + 3, (unsigned long long)ns);
        }
    }

    // ================================================================ ENUMERATE
    struct Enum {
        Chunk F0, F1;
        bool claims_done, enum_done;
        uint32_t stg_j;              // TMA stages issued
        uint32_t qt;                 // items emitted on Q0 (queue tail)
        uint32_t st;                 // signals emitted on S0
        uint32_t pidx;               // next part of F0
        bool begun;                  // Begin of part pidx emitted
        uint32_t pc_base;
        bool pc_valid;
        uint32_t pc_ps, pc_pe;       // part [start, end), relative to F0.beg
        uint32_t pc_key;
        uint32_t ni, ns;
    };

    __device__ __forceinline__ void load_chunk(Chunk &c, int32_t k, uint32_t pos) const {
        const long long base0 = P.hdr->base0, offR = P.hdr->offR;
        c.k = k;
        c.beg = (k == 0) ? P.hdr->off0 : base0 + (long long)k * P.C;
        const long long e = base0 + (long long)(k + 1) * P.C;
        c.end = e > offR ? offR : e;
        c.pos = pos;
        c.fr0 = P.chunk_fr[k];
        c.fr1 = P.chunk_fr[k + 1];
        c.head = (k > 0) && (P.off[c.fr0] > c.beg);
    }
    __device__ __forceinline__ static uint32_t flen(const Chunk &c) { return (uint32_t)(c.end - c.beg); }

    __device__ __forceinline__ void issue_stage(Enum &E, const Chunk &c) const {
        const uint32_t j = E.stg_j;
        const uint32_t p0 = j * SBLK;
        const uint32_t n = min((uint32_t)SBLK, c.pos + flen(c) - p0);
        const long long src = c.beg + (long long)p0 - (long long)c.pos;   // 16-byte aligned element index
        uint32_t *dst = Q(0) + (p0 & (RING0 - 1));
        uint64_t *b = &bar()[j % NST];
        const long long lim = (P.n_elems - src) & ~3ll;
        const uint32_t ntma = (uint32_t)min((long long)((n + 3u) & ~3u), lim);
        const int tail = (int)n - (int)ntma;
        if (tail > 0 && (int)lane < tail)
            dst[ntma + lane] = __ldg(reinterpret_cast<const uint32_t *>(P.elems) + src + ntma + lane);
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
        E.stg_j = j + 1;
    }

    __device__ __forceinline__ int32_t claim() const {
        uint32_t k = 0;
        if (lane == 0) k = atomicAdd(&P.hdr->claim, 1u);
        k = __shfl_sync(kFull, k, 0);
        return k < P.hdr->nchunks ? (int32_t)k : -1;
    }

    // Keep the Q0 ring full (prefetch ahead of emission); claims chunks of the
    // parent stream with atomics.
    __device__ __forceinline__ bool refill(Enum &E) const {
        bool prog = false;
        uint32_t h0 = ld_acq(&ctl(0)->head);
        for (;;) {
            if ((E.stg_j + 1) * (uint32_t)SBLK > h0 + RING0) {
                h0 = ld_acq(&ctl(0)->head);
                if ((E.stg_j + 1) * (uint32_t)SBLK > h0 + RING0) return prog;
            }
            const uint32_t sp = E.stg_j * SBLK;
            if (E.F0.k >= 0 && sp < E.F0.pos + flen(E.F0)) { issue_stage(E, E.F0); prog = true; continue; }
            if (E.F1.k >= 0 && sp < E.F1.pos + flen(E.F1)) { issue_stage(E, E.F1); prog = true; continue; }
            if (E.F1.k >= 0 || E.claims_done) return prog;
            const int32_t k = claim();
            prog = true;
            if (k < 0) { E.claims_done = true; return prog; }
            if (E.F0.k < 0) {
                load_chunk(E.F0, k, sp);      // chunk 0 is always a first claim (init_first_chunk)
                E.pidx = 0;
                E.begun = false;
                E.pc_valid = false;
            } else {
                load_chunk(E.F1, k, E.F0.pos + flen(E.F0));
            }
        }
    }

    // Part qi of chunk F0 as [start, end) relative to F0.beg, and its key
    // (region id, or a partial slot for the chunk's head part / a tail part
    // that crosses the chunk end).
    __device__ __forceinline__ void part_info(const Enum &E, uint32_t qi, bool valid, uint32_t &ps, uint32_t &pe,
                                              uint32_t &key) const {
        const uint32_t len = flen(E.F0);
        ps = pe = len;
        key = 0;
        if (!valid) return;
        if (E.F0.head && qi == 0) {
            ps = 0;
            const long long e = P.off[E.F0.fr0];
            pe = e < E.F0.end ? (uint32_t)(e - E.F0.beg) : len;
            key = SLOT | (uint32_t)(2 * E.F0.k);
        } else {
            const uint32_t r = E.F0.fr0 + qi - (E.F0.head ? 1u : 0u);
            ps = (uint32_t)(P.off[r] - E.F0.beg);
            const long long e = P.off[r + 1];
            if (e > E.F0.end) { pe = len; key = SLOT | (uint32_t)(2 * E.F0.k + 1); }
            else { pe = (uint32_t)(e - E.F0.beg); key = r; }
        }
    }

    __device__ __forceinline__ void write_tags(uint32_t qt, uint32_t m, uint32_t cum, uint32_t cnt, uint32_t key,
                                               uint32_t tot) const {
        uint32_t *t0 = T(0);
        if (m == 1 || __shfl_sync(kFull, cnt, 0) == tot) {
            const uint32_t k0 = __shfl_sync(kFull, key, 0);
            for (uint32_t i = lane; i < tot; i += 32) t0[(qt + i) & (RING0 - 1)] = k0;
            return;
        }
        const uint32_t excl = cum - cnt;
        for (uint32_t b = 0; b < tot; b += 32) {
            const uint32_t rel = b + lane;
            int lo = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1) {
                const int cand = lo + step;
                const uint32_t ex = __shfl_sync(kFull, excl, cand < 32 ? cand : 31);
                if (cand < (int)m && ex <= rel) lo = cand;
            }
            const uint32_t k = __shfl_sync(kFull, key, lo);
            if (rel < tot) t0[(qt + rel) & (RING0 - 1)] = k;
        }
    }

    // Emit F0's parts: Begin, element indices (the staged element values), End
    // (P:489-494), as far as staged data and signal space allow; resumable
    // mid-region.  Up to 32 parts per step, one per lane.
    __device__ __forceinline__ bool emit(Enum &E) const {
        bool prog = false;
        uint32_t sh0 = TAG ? 0u : ld_acq(&ctl(0)->shead);
        for (;;) {
            if (E.F0.k < 0) {
                if (E.F1.k >= 0) { E.F0 = E.F1; E.F1.k = -1; E.pidx = 0; E.begun = false; E.pc_valid = false; continue; }
                if (E.claims_done) E.enum_done = true;
                return prog;
            }
            const uint32_t np = (E.F0.head ? 1u : 0u) + (E.F0.fr1 - E.F0.fr0);
            if (E.pidx >= np) {                  // chunk fully enumerated
                E.F0 = E.F1;
                E.F1.k = -1;
                E.pidx = 0;
                E.begun = false;
                E.pc_valid = false;
                prog = true;
                continue;
            }
            const uint32_t lim_pos = min(E.stg_j * (uint32_t)SBLK, E.F0.pos + flen(E.F0));
            const uint32_t avail = lim_pos - E.qt;
            if (!E.pc_valid || E.pidx >= E.pc_base + 32) {
                E.pc_base = E.pidx;
                E.pc_valid = true;
                part_info(E, E.pidx + lane, E.pidx + lane < np, E.pc_ps, E.pc_pe, E.pc_key);
            }
            const uint32_t d = E.pidx - E.pc_base;
            const uint32_t e_next = E.qt - E.F0.pos;          // next element, relative to F0.beg
            if (avail == 0 && (TAG || E.begun)) {
                const uint32_t pe0 = __shfl_sync(kFull, E.pc_pe, d);
                if (pe0 > e_next) return prog;       // current part has items, nothing staged
            }
            uint32_t ps = __shfl_down_sync(kFull, E.pc_ps, d);
            uint32_t pe = __shfl_down_sync(kFull, E.pc_pe, d);
            const uint32_t key = __shfl_down_sync(kFull, E.pc_key, d);
            const bool valid = (lane + d < 32) && (E.pidx + lane < np);
            if (!valid) ps = pe = flen(E.F0);
            if (lane == 0 && ps < e_next) ps = e_next;
            const uint32_t cnt = pe - ps;
            uint32_t cum = cnt;
            const uint32_t sig = TAG ? 0u : ((lane == 0 && E.begun) ? 1u : 2u);
            uint32_t scum = sig;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const uint32_t o = __shfl_up_sync(kFull, cum, dd);
                const uint32_t so = __shfl_up_sync(kFull, scum, dd);
                if ((int)lane >= dd) { cum += o; scum += so; }
            }
            uint32_t sfree = 0xffffffffu;
            if constexpr (!TAG) {
                sfree = scap - (E.st - sh0);
                if (__any_sync(kFull, scum > sfree)) {      // warp-uniform reload of the consumer's position
                    sh0 = ld_acq(&ctl(0)->shead);
                    sfree = scap - (E.st - sh0);
                }
            }
            const bool fits = valid && (cum <= avail) && (scum <= sfree);
            const uint32_t m = __popc(__ballot_sync(kFull, fits));
            if (m > 0) {
                const uint32_t tot = __shfl_sync(kFull, cum, m - 1);
                if constexpr (!TAG) {
                    // Begin_i at the part's first position, End_i after its last one.
                    const uint32_t sexcl = scum - sig;
                    if (lane < m) {
                        uint4 *s0 = S(0);
                        uint32_t slot = E.st + sexcl;
                        if (!(lane == 0 && E.begun)) { s0[slot & smask] = make_uint4(key, E.qt + cum - cnt, 0u, 0u); slot++; }
                        s0[slot & smask] = make_uint4(key, E.qt + cum, 1u, 0u);
                    }
                    const uint32_t nsig = __shfl_sync(kFull, scum, m - 1);
                    E.st += nsig;
                    E.ns += nsig;
                } else {
                    write_tags(E.qt, m, cum, cnt, key, tot);
                }
                E.qt += tot;
                E.ni += tot;
                E.pidx += m;
                E.begun = false;
                prog = true;
                continue;
            }
            // part pidx does not fit whole: emit what we can of it
            const uint32_t key0 = __shfl_sync(kFull, key, 0);
            const uint32_t cnt0 = __shfl_sync(kFull, cnt, 0);
            bool did = false;
            if constexpr (!TAG) {
                if (!E.begun) {
                    if (sfree == 0) return prog;
                    if (lane == 0) S(0)[E.st & smask] = make_uint4(key0, E.qt, 0u, 0u);
                    E.st++;
                    E.ns++;
                    sfree--;
                    E.begun = true;
                    did = true;
                }
            }
            const uint32_t k = min(avail, cnt0);
            if (k > 0) {
                if constexpr (TAG) {
                    uint32_t *t0 = T(0);
                    for (uint32_t i = lane; i < k; i += 32) t0[(E.qt + i) & (RING0 - 1)] = key0;
                }
                E.qt += k;
                E.ni += k;
                did = true;
            }
            if constexpr (!TAG) {
                if (k == cnt0 && sfree > 0) {
                    if (lane == 0) S(0)[E.st & smask] = make_uint4(key0, E.qt, 1u, 0u);
                    E.st++;
                    E.ns++;
                    E.pidx++;
                    E.begun = false;
                    did = true;
                }
            } else {
                if (k == cnt0) { E.pidx++; did = true; }
            }
            prog |= did;
            if (!did) return prog;
        }
    }

    // Kernel init (warp 0, before the CTA barrier): claim the first chunk so
    // that every node warp starts from the right Q0 position (chunk 0 starts
    // at the 16-byte alignment pad of offsets[0]).
    __device__ __forceinline__ void init_first_chunk() const {
        const int32_t k = claim();
        if (lane == 0) {
            ctl(0)->pad_[0] = (uint32_t)k;
            const uint32_t pos = (k == 0) ? (uint32_t)(P.hdr->off0 - P.hdr->base0) : 0u;
            ctl(0)->head = pos;
            ctl(0)->tail = pos;
        }
    }

    __device__ void run_enumerate() const {
        Enum E;
        E.F0.k = E.F1.k = -1;
        E.claims_done = E.enum_done = false;
        E.stg_j = 0;
        E.qt = ctl(0)->tail;
        {
            const int32_t k0 = (int32_t)ctl(0)->pad_[0];
            if (k0 >= 0) load_chunk(E.F0, k0, E.qt);
            else E.claims_done = true;
        }
        E.st = 0;
        E.pidx = 0;
        E.begun = false;
        E.pc_valid = false;
        E.pc_base = 0;
        E.ni = E.ns = 0;
        uint32_t backoff = 0, idle = 0;
        for (;;) {
            bool prog = refill(E);
            const uint32_t qt0 = E.qt, st0 = E.st;
            prog |= emit(E);
            if (E.st != st0) publish(&ctl(0)->stail, E.st);
            if (E.qt != qt0) publish(&ctl(0)->tail, E.qt);
            if (E.enum_done) break;
            if (prog) { backoff = 0; idle = 0; continue; }
            if (!idle_wait(backoff, idle)) break;
        }
        publish(&ctl(0)->done, 1u);
        // keep the CTA's shared memory alive until every issued stage has landed
        for (uint32_t j = 0; j < E.stg_j; ++j) {
            if (j + NST < E.stg_j) continue;     // older fills of the same barrier completed before
            uint32_t spins = 0;
            while (!mbar_try_wait_uniform(&bar()[j % NST], (j / NST) & 1u) && ++spins < (1u << 26)) {}
        }
        flush_stats(0, 0, 0, E.ni, E.ns);
    }

    // ============================================================= CONSUMERS
    // Generic consumer state for node n reading edge n-1.
    struct In {
        uint32_t head, shead;      // consumed positions (published)
        uint32_t tail, stail;      // producer positions last seen
        uint32_t landed;           // Q0 only: stages known landed
        bool done;                 // producer finished (tail/stail final)
        uint32_t nd, nf, ni, ns;
    };

    __device__ __forceinline__ void refresh(In &I, int e) const {
        I.tail = ld_acq(&ctl(e)->tail);
        if constexpr (!TAG) I.stail = ld_acq(&ctl(e)->stail);
    }

    // Items readable now: landed (Q0) and below the head signal's stamp.
    __device__ __forceinline__ uint32_t limit(In &I, int e, bool &spend, uint32_t &stamp, uint32_t &kind,
                                              uint32_t &key) const {
        uint32_t lim = I.tail;
        spend = false;
        if constexpr (!TAG) {
            if (I.shead != I.stail) {
                uint4 s = make_uint4(0u, 0u, 0u, 0u);
                if (lane == 0) s = S(e)[I.shead & smask];
                s.x = __shfl_sync(kFull, s.x, 0);
                s.y = __shfl_sync(kFull, s.y, 0);
                s.z = __shfl_sync(kFull, s.z, 0);
                spend = true;
                key = s.x;
                stamp = s.y;
                kind = s.z;
                if ((int)(stamp - lim) < 0) lim = stamp;
            }
        }
        if (e == 0) {
            while ((int)(I.landed * SBLK - lim) < 0 && mbar_test_uniform(&bar()[I.landed % NST], (I.landed / NST) & 1u))
                I.landed++;
            // nothing is readable before the stage holding `head` has landed (chunk 0
            // may start inside stage 0 at the alignment pad)
            const uint32_t rdy = I.landed * SBLK;
            if ((int)(rdy - lim) < 0) lim = ((int)(rdy - I.head) < 0) ? I.head : rdy;
        }
        return lim;
    }

    // Protocol violation: the readable limit fell behind the consumed position
    // (a signal would be received after items emitted after it -- Lemma 1).
    // Records the receiver state in the workspace header for diagnosis.
    __device__ void debug_fail(int n, const In &I, uint32_t lim, bool spend, uint32_t stamp, uint32_t key,
                               uint32_t kind) const {
        if (lane == 0 && atomicCAS((int *)&P.hdr->err, 0, ERR_LIMIT) == 0) {
            uint32_t *d = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(P.hdr) + 64);
            d[0] = n; d[1] = lim; d[2] = I.head; d[3] = I.tail; d[4] = spend; d[5] = stamp; d[6] = key;
            d[7] = kind; d[8] = I.shead; d[9] = I.stail; d[10] = I.landed; d[11] = blockIdx.x;
            d[12] = ctl(n - 1)->tail; d[13] = ctl(n - 1)->stail;
        }
    }

    // FILTER / TRANSFORM stage n (1..K): consumes edge n-1, produces edge n.
    template <class Op>
    __device__ void run_stage_op(int n, const Op op) const {
        const int ei = n - 1;
        In I{};
        I.head = I.shead = I.tail = I.stail = I.landed = 0;
        I.done = false;
        uint32_t *out = Q(n), *tout = T(n);
        const uint32_t *in = Q(ei), *tin = T(ei);
        const uint32_t im = imask(ei);
        uint32_t otail = 0, ost = 0;           // own output positions
        uint32_t wait_small = 0;
        uint32_t ohead = 0, osh = 0;           // consumer positions last seen
        uint32_t backoff = 0, idle = 0;
        I.head = ctl(ei)->head;                // Q0 may start at the chunk-0 pad (set before the CTA barrier)
        I.tail = I.head;
        for (;;) {
            refresh(I, ei);
            bool prog = false;
            for (;;) {
                bool spend;
                uint32_t stamp = 0, kind = 0, key = 0;
                const uint32_t lim = limit(I, ei, spend, stamp, kind, key);
                if ((int)(lim - I.head) < 0) { debug_fail(n, I, lim, spend, stamp, key, kind); return; }
                const uint32_t avail = lim - I.head;
                uint32_t space = qcap - (otail - ohead);
                if (space < (uint32_t)W && space < avail) {
                    ohead = ld_acq(&ctl(n)->head);
                    space = qcap - (otail - ohead);
                }
                const uint32_t e = min(avail, space);
                // Batch at least BMIN ensembles per firing so the scheduling cost is
                // amortised; smaller batches only when the limit is a signal stamp,
                // the output queue, or the drained input.
                bool go = e >= (uint32_t)W;
                if (go && e < (uint32_t)(BMIN * W) && !(spend && lim == stamp) && space >= avail && !I.done &&
                    wait_small < 8) {
                    go = false;
                    ++wait_small;
                }
                if (go) {
                    wait_small = 0;
                    const uint32_t nens = e / W;
                    const uint32_t t2 = filter_batch<TAG, Op>(in, tin, im, I.head, nens, out, tout, qmask, otail, op, lt);
                    I.head += nens * W;
                    I.nd += nens;
                    I.nf += nens;
                    I.ni += nens * W;
                    otail = t2;
                    publish(&ctl(n)->tail, otail);
                    publish(&ctl(ei)->head, I.head);
                    prog = true;
                    continue;
                }
                // partial ensemble: bounded by the head signal's credit, or the drained tail
                bool ok = false;
                if (e > 0) {
                    if (spend && I.head + e == stamp) ok = true;
                    else if (!spend && I.done && I.head + e == I.tail && e == avail) ok = true;
                }
                if (ok) {
                    otail = partial_stage(n, in, tin, im, I.head, e, out, tout, otail);
                    I.head += e;
                    I.nd++;
                    I.ni += e;
                    publish(&ctl(n)->tail, otail);
                    publish(&ctl(ei)->head, I.head);
                    prog = true;
                    continue;
                }
                // signal phase: deliver the head signal once every item before it is consumed
                if (spend && I.head == stamp) {
                    if (scap - (ost - osh) == 0) {
                        osh = ld_acq(&ctl(n)->shead);
                        if (scap - (ost - osh) == 0) break;
                    }
                    if (lane == 0) S(n)[ost & smask] = make_uint4(key, otail, kind, 0u);   // forwarded
                    ost++;
                    I.shead++;
                    I.ns++;
                    publish(&ctl(n)->stail, ost);
                    publish(&ctl(ei)->shead, I.shead);
                    prog = true;
                    continue;
                }
                break;
            }
            if (prog) { backoff = 0; idle = 0; continue; }
            if (I.done) {
                if (I.head == I.tail && (TAG || I.shead == I.stail)) break;
            } else if (ld_acq(&ctl(ei)->done)) {
                I.done = true;
                continue;            // re-read final tail/stail
            }
            if (!idle_wait(backoff, idle)) break;
        }
        publish(&ctl(n)->done, 1u);
        flush_stats(n, I.nd, I.nf, I.ni, I.ns);
    }

    __device__ __forceinline__ uint32_t partial_stage(int n, const uint32_t *in, const uint32_t *tin, uint32_t im,
                                                      uint32_t h, uint32_t e, uint32_t *out, uint32_t *tout,
                                                      uint32_t tl) const {
        const StageP &sp = P.st[n - 1];
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
            const uint32_t idx = j * 32 + lane;
            const bool act = idx < e;
            uint32_t v = act ? in[(h + idx) & im] : 0u;
            uint32_t tg = 0;
            if constexpr (TAG) tg = act ? tin[(h + idx) & im] : 0u;
            const bool keep = act && stage_apply(sp, v);
            const uint32_t mk = __ballot_sync(kFull, keep);
            if (keep) {
                const uint32_t pos = (tl + __popc(mk & lt)) & qmask;
                out[pos] = v;
                if constexpr (TAG) tout[pos] = tg;
            }
            tl += __popc(mk);
        }
        return tl;
    }

    __device__ void run_stage(int n) const {
        const StageP &sp = P.st[n - 1];
        switch (sp.op) {
            case RS_OP_HASH_LT:
                if (sp.b >= 256) run_stage_op(n, OpAll{});
                else run_stage_op(n, OpHash{sp.a, sp.b << 24});
                break;
            case RS_OP_LT_U32:
                if (sp.table[0]) run_stage_op(n, OpAll{});
                else run_stage_op(n, OpLt{sp.b, false});
                break;
            case RS_OP_CLASS: run_stage_op(n, OpClass{sp.table}); break;
            case RS_OP_SCALE_F32: run_stage_op(n, OpScale{__uint_as_float(sp.a)}); break;
            default: run_stage_op(n, OpAffine{sp.a, sp.b}); break;
        }
    }

    // ================================================================ AGGREGATE
    struct Agg {
        A acc;          // per-lane partial accumulator
        uint32_t akey;  // tagged: key of the carry region (0xffffffff = none)
        A carry;        // tagged: uniform carry partial
    };

    __device__ __forceinline__ void agg_tagged(Agg &G, const uint32_t *in, const uint32_t *tin, uint32_t im, uint32_t h,
                                               uint32_t e) const {
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
            const int cntj = (int)e - j * 32;
            if (cntj <= 0) break;
            const bool act = (int)lane < cntj;
            const uint32_t idx = j * 32 + lane;
            const uint32_t key = act ? tin[(h + idx) & im] : 0xffffffffu;
            const A val = act ? AT::lift(in[(h + idx) & im]) : AT::id();
            if (__all_sync(kFull, !act || key == G.akey)) {
                G.acc = AT::comb(G.acc, val);
                continue;
            }
            G.carry = AT::comb(G.carry, warp_reduce<AT>(G.acc));
            G.acc = AT::id();
            uint32_t prev = __shfl_up_sync(kFull, key, 1);
            if (lane == 0) prev = G.akey;
            const bool head = act && key != prev;
            const uint32_t hm = __ballot_sync(kFull, head);
            const uint32_t le = hm & lanemask_le();
            const int seg = le ? 31 - __clz(le) : -1;
            A v = val;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const A o = AT::shfl_up(v, d);
                if ((int)lane - d >= seg && (int)lane >= d) v = AT::comb(o, v);
            }
            if (seg < 0 && act) v = AT::comb(G.carry, v);
            if (lane == 0 && head && G.akey != 0xffffffffu) store_key(G.akey, G.carry);
            const bool nexthead = (lane < 31) && ((hm >> (lane + 1)) & 1u);
            if (act && nexthead) store_key(key, v);
            const int last = (cntj < 32 ? cntj : 32) - 1;
            G.akey = __shfl_sync(kFull, key, last);
            G.carry = AT::shfl(v, last);
        }
    }

    __device__ void run_aggregate() const {
        constexpr int n = K + 1, ei = K;
        In I{};
        I.head = I.shead = I.tail = I.stail = I.landed = 0;
        I.done = false;
        Agg G;
        G.acc = AT::id();
        G.carry = AT::id();
        G.akey = 0xffffffffu;
        const uint32_t *in = Q(ei), *tin = T(ei);
        const uint32_t im = imask(ei);
        uint32_t backoff = 0, idle = 0, wait_small = 0;
        I.head = ctl(ei)->head;
        I.tail = I.head;
        for (;;) {
            refresh(I, ei);
            bool prog = false;
            for (;;) {
                bool spend;
                uint32_t stamp = 0, kind = 0, key = 0;
                const uint32_t lim = limit(I, ei, spend, stamp, kind, key);
                if ((int)(lim - I.head) < 0) { debug_fail(n, I, lim, spend, stamp, key, kind); return; }
                const uint32_t avail = lim - I.head;
                bool go = avail >= (uint32_t)W;
                if (go && avail < (uint32_t)(BMIN * W) && !(spend && lim == stamp) && !I.done && wait_small < 8) {
                    go = false;
                    ++wait_small;
                }
                if (go) {
                    wait_small = 0;
                    const uint32_t nens = avail / W;
                    uint32_t h = I.head;
                    if constexpr (!TAG) {
                        // one region per ensemble: per-lane accumulation (a::run)
                        uint32_t k = 0;
                        for (; k + 2 <= nens; k += 2, h += 2 * W) agg_slices<2 * IPL>(G, in, im, h);
                        if (k < nens) agg_slices<IPL>(G, in, im, h);
                    } else {
                        for (uint32_t k = 0; k < nens; ++k, h += W) agg_tagged(G, in, tin, im, h, W);
                    }
                    I.head += nens * W;
                    I.nd += nens;
                    I.nf += nens;
                    I.ni += nens * W;
                    publish(&ctl(ei)->head, I.head);
                    prog = true;
                    continue;
                }
                bool ok = false;
                if (avail > 0) {
                    if (spend && I.head + avail == stamp) ok = true;
                    else if (!spend && I.done && I.head + avail == I.tail) ok = true;
                }
                if (ok) {
                    if constexpr (!TAG) {
#pragma unroll
                        for (int j = 0; j < IPL; ++j) {
                            const uint32_t idx = j * 32 + lane;
                            if (idx < avail) G.acc = AT::comb(G.acc, AT::lift(in[(I.head + idx) & im]));
                        }
                    } else {
                        agg_tagged(G, in, tin, im, I.head, avail);
                    }
                    I.head += avail;
                    I.nd++;
                    I.ni += avail;
                    publish(&ctl(ei)->head, I.head);
                    prog = true;
                    continue;
                }
                if constexpr (!TAG) {
                    if (spend && I.head == stamp) {
                        if (kind == 0) {                 // a::begin: acc = identity
                            G.acc = AT::id();
                        } else {                         // a::end: push(acc)
                            const A v = warp_reduce<AT>(G.acc);
                            if (lane == 0) store_key(key, v);
                            G.acc = AT::id();
                        }
                        I.shead++;
                        I.ns++;
                        publish(&ctl(ei)->shead, I.shead);
                        prog = true;
                        continue;
                    }
                }
                break;
            }
            if (prog) { backoff = 0; idle = 0; continue; }
            if (I.done) {
                if (I.head == I.tail && (TAG || I.shead == I.stail)) break;
            } else if (ld_acq(&ctl(ei)->done)) {
                I.done = true;
                continue;
            }
            if (!idle_wait(backoff, idle)) break;
        }
        if constexpr (TAG) {
            G.carry = AT::comb(G.carry, warp_reduce<AT>(G.acc));
            if (lane == 0 && G.akey != 0xffffffffu) store_key(G.akey, G.carry);
        }
        flush_stats(n, I.nd, I.nf, I.ni, I.ns);
    }

    template <int NS>
    __device__ __forceinline__ void agg_slices(Agg &G, const uint32_t *in, uint32_t im, uint32_t h) const {
        uint32_t v[NS];
        if (((h & im) + NS * 32) <= im + 1) {
            const uint32_t *src = in + (h & im) + lane;
#pragma unroll
            for (int j = 0; j < NS; ++j) v[j] = src[32 * j];
        } else {
#pragma unroll
            for (int j = 0; j < NS; ++j) v[j] = in[(h + 32 * j + lane) & im];
        }
        A part = AT::lift(v[0]);
#pragma unroll
        for (int j = 1; j < NS; ++j) part = AT::comb(part, AT::lift(v[j]));
        G.acc = AT::comb(G.acc, part);
    }
};

template <int K, int AGG, bool TAG>
__global__ void __launch_bounds__((K + 2) * 32, 1) k_pipeline_ws(const __grid_constant__ KParams P) {
    extern __shared__ __align__(128) uint8_t smem[];
    using W_ = WS<K, AGG, TAG>;
    if (P.hdr->err) return;
    const uint32_t warp = threadIdx.x >> 5;
    W_ ws(P, smem);
    if (threadIdx.x < 32) {
        // init control words and the TMA barriers before any warp starts
        uint32_t *c = reinterpret_cast<uint32_t *>(smem);
        for (uint32_t i = threadIdx.x; i < 64; i += 32) c[i] = 0u;
        if (threadIdx.x == 0)
            for (int i = 0; i < NST; ++i) mbar_init(&ws.bar()[i], 1);
        mbar_fence_init();
        __syncwarp();
        ws.init_first_chunk();
    }
    __syncthreads();
    if (warp == 0) {
        ws.run_enumerate();
    } else if (warp <= (uint32_t)K) {
        ws.run_stage((int)warp);
    } else {
        ws.run_aggregate();
    }
}
