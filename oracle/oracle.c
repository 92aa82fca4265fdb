/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the region-based streaming
 * hot path of Timcheck & Buhler, "Streaming Computations with Region-Based
 * State on SIMD Architectures" (arXiv 2006.07478).  Citations "P:a-b" are
 * lines of /root/reference/PAPER.md (section given beside each); "S:a-b" are
 * lines of SPEC.md (used only for interface shapes / worked examples).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The CUDA product path
 * (paper_2006_07478_b200/) shares NO code, header, table or constant with it.
 *
 * Two independent evaluators live here:
 *   (1) or_brute   — the plain per-region definition: for each
 *                    parent, fold its surviving elements (§4,
 *                    Fig. 5).  Lemma 1 puts every item
 *                    in its own parent's context, so the pipeline's result is
 *                    exactly this fold.
 *   (2) or_interp  — a sequential interpreter of the pipeline itself: data
 *                    queues + signal queues (§3.1), the sender and
 *                    receiver credit rules (§3.1), two-phase firing
 *                    (§3.2), fireability (§3.2),
 *                    SIMD ensembles bounded by credit (§3.3),
 *                    enumeration with Begin/End signals (P:458-471,
 *                    P:489-494 §4), aggregation begin/run/end,
 *                    and the per-item tag alternative (§2.3,
 *                    P:688-705 §5).  It also counts SIMD occupancy
 *                    (§2.2; §5).
 * Readings of points the paper leaves open are DESIGN.md §"Readings" (A1-A26
 * of SURVEY §8(c)); each is cited where used below.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (oracle.build())
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- vocabulary
 * Oracle-local enumerations.  The Python wrapper (oracle/__init__.py) maps
 * names onto these numbers; nothing here is shared with include/rs.h.       */
enum { OR_I32 = 0, OR_U32 = 1, OR_U8 = 2, OR_F32 = 3 };                /* element types   */
enum { OR_FILTER = 2, OR_TRANSFORM = 3 };                               /* stage kinds     */
enum { OR_HASH_LT = 1, OR_LT_U32 = 2, OR_CLASS = 3, OR_PARENT_LT = 4,   /* filter ops (A13)*/
       OR_SCALE_F32 = 10, OR_AFFINE_I32 = 11 };                         /* transform ops   */
enum { OR_SUM_I64 = 1, OR_SUM_F32 = 2, OR_COUNT_MIN_U32 = 3, OR_COUNT_XOR64 = 4 };
enum { OR_SIGNAL = 0, OR_TAGGED = 1 };                                  /* strategies      */
enum { OR_FULL_FIRST = 0, OR_DEEPEST_FIRST = 1, OR_RANDOM = 2 };        /* policies (A8)   */
enum { OR_BEGIN = 1, OR_END = 2 };                                      /* signal kinds    */
enum { OR_OK = 0, OR_ECREDIT = -1, OR_ESIGFULL = -2, OR_ELIVELOCK = -3,
       OR_EUNMATCHED = -4, OR_EARG = -5, OR_EINVARIANT = -6, OR_ENOMEM = -7 };

typedef struct {
    int32_t kind;          /* OR_FILTER | OR_TRANSFORM                          */
    int32_t op;
    uint64_t p0, p1;       /* HASH_LT: p0 = multiplier A, p1 = threshold T      */
                           /* LT_U32: p1 = bound; SCALE_F32: p0 = float bits    */
                           /* AFFINE_I32: p0 = a, p1 = b                        */
    const uint8_t *table;  /* CLASS: 32-byte bitmap over byte values            */
                           /* PARENT_LT: uint32 parent context, one per region   */
} or_stage;

/* ------------------------------------------------------------- element ops */

/* getItem (Fig. 5): the element's 32-bit pattern (u8 zero-extended). */
static uint32_t get_item(int dtype, const void *elems, int64_t g) {
    switch (dtype) {
    case OR_U8:  return ((const uint8_t *)elems)[g];
    default:     return ((const uint32_t *)elems)[g];   /* i32/u32/f32 bit pattern */
    }
}

static float bits_f(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t f_bits(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

/* isGood(v) of Fig. 5 is unspecified; readings in SURVEY §8(c) A13.
 * Returns 1 = keep.  Transforms always keep and rewrite *v (A14).
 * r is the item's parent: a node "may access the parent object",
 * Fig. 5 reads it with getParent(); PARENT_LT keeps an item iff
 * it is below its parent's context value ctx[r] (reading R4).     */
static int apply_stage(const or_stage *s, uint32_t *v, int64_t r) {
    if (s->kind == OR_FILTER) {
        switch (s->op) {
        case OR_HASH_LT: {                   /* keep iff top byte of v*A < T */
            uint32_t h = (uint32_t)(*v * (uint32_t)s->p0);
            return (uint64_t)(h >> 24) < s->p1;
        }
        case OR_LT_U32:                      /* keep iff v < bound           */
            return (uint64_t)*v < s->p1;
        case OR_CLASS:                       /* keep iff byte is in the set  */
            return (s->table[(*v & 0xFFu) >> 3] >> (*v & 7u)) & 1u;
        case OR_PARENT_LT:                   /* keep iff v < parent context  */
            return *v < ((const uint32_t *)s->table)[r];
        }
        return 1;
    }
    switch (s->op) {
    case OR_SCALE_F32: {                     /* v' = scale * v, fp32 RN, no FMA (A14) */
        float scale = bits_f((uint32_t)s->p0);
        float x = bits_f(*v);
        float y = scale * x;
        *v = f_bits(y);
        return 1;
    }
    case OR_AFFINE_I32:                      /* v' = a*v + b mod 2^32        */
        *v = (uint32_t)(*v * (uint32_t)s->p0 + (uint32_t)s->p1);
        return 1;
    }
    return 1;
}

/* splitmix64 finalizer (reading A19).                                        */
uint64_t or_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Aggregate accumulator: begin() = identity, run() = combine, end() = write
 * (Fig. 5).  Identities per reading A1.                           */
typedef struct { int64_t i64; double f64; uint64_t cnt; uint32_t mn; uint64_t x; } acc_t;

static void acc_begin(acc_t *a) { a->i64 = 0; a->f64 = 0.0; a->cnt = 0; a->mn = 0xFFFFFFFFu; a->x = 0; }

static void acc_run(int agg, acc_t *a, uint32_t v, int64_t i) {
    switch (agg) {
    case OR_SUM_I64: a->i64 = (int64_t)((uint64_t)a->i64 + (uint64_t)(int64_t)(int32_t)v); break;
    case OR_SUM_F32: a->f64 += (double)bits_f(v); break;   /* double accumulation (A15) */
    case OR_COUNT_MIN_U32: a->cnt += 1; if (v < a->mn) a->mn = v; break;
    case OR_COUNT_XOR64: a->cnt += 1; a->x ^= or_mix64(((uint64_t)i << 8) | (v & 0xFFu)); break;
    }
}

/* out0/out1 layouts: SUM_I64 -> int64 out0; SUM_F32 -> double out0;
 * COUNT_MIN_U32 -> uint32 out0 (count), uint32 out1 (min);
 * COUNT_XOR64 -> uint64 out0 (count), uint64 out1 (xor).                   */
static void acc_end(int agg, const acc_t *a, void *out0, void *out1, int64_t r) {
    switch (agg) {
    case OR_SUM_I64: ((int64_t *)out0)[r] = a->i64; break;
    case OR_SUM_F32: ((double *)out0)[r] = a->f64; break;
    case OR_COUNT_MIN_U32: ((uint32_t *)out0)[r] = (uint32_t)a->cnt; ((uint32_t *)out1)[r] = a->mn; break;
    case OR_COUNT_XOR64: ((uint64_t *)out0)[r] = a->cnt; ((uint64_t *)out1)[r] = a->x; break;
    }
}

static int check_args(int dtype, const void *elems, const int64_t *off, int64_t R,
                      const or_stage *st, int nst, int agg) {
    if (R < 0 || (R > 0 && !off) || nst < 0 || (nst > 0 && !st)) return OR_EARG;
    if (dtype < OR_I32 || dtype > OR_F32) return OR_EARG;
    if (agg < OR_SUM_I64 || agg > OR_COUNT_XOR64) return OR_EARG;
    for (int64_t r = 0; r < R; r++) if (off[r + 1] < off[r]) return OR_EARG;
    if (R > 0 && off[R] > off[0] && !elems) return OR_EARG;
    for (int k = 0; k < nst; k++)
        if ((st[k].op == OR_CLASS || st[k].op == OR_PARENT_LT) && !st[k].table) return OR_EARG;
    return OR_OK;
}

/* ------------------------------------------------------------------ brute
 * The plain definition (SURVEY §8(c) pseudo-code):
 *   for each parent r: acc = begin
 *     for i in 0..findCount(r)-1:
 *       v = getItem(i); apply stages in order, dropping at the
 *       first failed filter; if kept: run(acc, v)
 *     out[r] = end(acc) (exactly one result per parent, A2)           */
int or_brute(int dtype, const void *elems, const int64_t *off, int64_t R,
             const or_stage *st, int nst, int agg, void *out0, void *out1) {
    int rc = check_args(dtype, elems, off, R, st, nst, agg);
    if (rc) return rc;
    for (int64_t r = 0; r < R; r++) {
        acc_t a; acc_begin(&a);
        int64_t n = off[r + 1] - off[r];
        for (int64_t i = 0; i < n; i++) {
            uint32_t v = get_item(dtype, elems, off[r] + i);
            int keep = 1;
            for (int k = 0; k < nst && keep; k++) keep = apply_stage(&st[k], &v, r);
            if (keep) acc_run(agg, &a, v, i);
        }
        acc_end(agg, &a, out0, out1, r);
    }
    return OR_OK;
}

/* Per-region item counts reaching each node (k_r(n) of SURVEY §8(c)):
 * kc[r*(nst+1) + j] = items of region r consumed by node j+1, i.e. children
 * surviving stages 1..j.  j = 0 is the first node after enumeration (all
 * children); j = nst is the aggregate.  Used for the occupancy bound
 * sum_r k_r / (w * sum_r ceil(k_r / w)) (§5).                     */
int or_node_counts(int dtype, const void *elems, const int64_t *off, int64_t R,
                   const or_stage *st, int nst, int64_t *kc) {
    int rc = check_args(dtype, elems, off, R, st, nst, OR_SUM_I64);
    if (rc) return rc;
    for (int64_t r = 0; r < R; r++) {
        int64_t *row = kc + r * (nst + 1);
        for (int j = 0; j <= nst; j++) row[j] = 0;
        for (int64_t g = off[r]; g < off[r + 1]; g++) {
            uint32_t v = get_item(dtype, elems, g);
            int j = 0;
            row[0]++;
            for (; j < nst; j++) { if (!apply_stage(&st[j], &v, r)) break; row[j + 1]++; }
        }
    }
    return OR_OK;
}

/* Fan-out (tree topology, Fig. 1b): after the
 * stages, a SPLIT node sends each item to child A if its op holds, else to
 * child B; both children are SUM_I64 aggregates, so the plain definition is
 * two per-region folds over the two partitions of each region's survivors.  */
int or_brute_split(int dtype, const void *elems, const int64_t *off, int64_t R, const or_stage *st, int nst,
                   const or_stage *split, int64_t *out_a, int64_t *out_b) {
    int rc = check_args(dtype, elems, off, R, st, nst, OR_SUM_I64);
    if (rc || !split) return rc ? rc : OR_EARG;
    for (int64_t r = 0; r < R; r++) {
        int64_t a = 0, b = 0;
        for (int64_t g = off[r]; g < off[r + 1]; g++) {
            uint32_t v = get_item(dtype, elems, g);
            int keep = 1;
            for (int k = 0; k < nst && keep; k++) keep = apply_stage(&st[k], &v, r);
            if (!keep) continue;
            if (apply_stage(split, &v, r)) a = (int64_t)((uint64_t)a + (uint64_t)(int64_t)(int32_t)v);
            else b = (int64_t)((uint64_t)b + (uint64_t)(int64_t)(int32_t)v);
        }
        out_a[r] = a;
        out_b[r] = b;
    }
    return OR_OK;
}

/* Element-wise exit: instead of one result per parent, a
 * stream of results derived from individual elements, "stripped of their
 * parent context" (§4; the taxi app's second stage emits each
 * verified pair with its line's tag, §5).  Plain definition: every
 * item surviving the stages is emitted as (parent r, value) in stream order.
 * Returns the number emitted (> cap: only the first cap were written).     */
int64_t or_emit(int dtype, const void *elems, const int64_t *off, int64_t R,
                const or_stage *st, int nst, uint32_t *out_val, uint32_t *out_reg, int64_t cap) {
    if (check_args(dtype, elems, off, R, st, nst, OR_SUM_I64)) return -1;
    int64_t n = 0;
    for (int64_t r = 0; r < R; r++) {
        for (int64_t g = off[r]; g < off[r + 1]; g++) {
            uint32_t v = get_item(dtype, elems, g);
            int keep = 1;
            for (int k = 0; k < nst && keep; k++) keep = apply_stage(&st[k], &v, r);
            if (!keep) continue;
            if (n < cap) { out_val[n] = v; out_reg[n] = (uint32_t)r; }
            n++;
        }
    }
    return n;
}

/* Taxi stage 2 (§5): a '{' that survived stage 1 is
 * the start of a coordinate pair "{x,y}"; the stage verifies the pair is well
 * formed -- '{', 1..9 decimal digits, ',', 1..9 digits, '}', all inside the line --
 * parses it, swaps it and emits (line, y, x) (integers stand in
 * for the paper's real values, reading R6).                        */
static int parse_pair(const uint8_t *b, int64_t g, int64_t lim, uint32_t *x, uint32_t *y) {
    uint32_t v[2] = {0, 0};
    if (g >= lim || b[g] != '{') return 0;
    int64_t i = g + 1;
    for (int f = 0; f < 2; f++) {
        int nd = 0;
        while (i < lim && b[i] >= '0' && b[i] <= '9' && nd <= 9) { v[f] = v[f] * 10u + (uint32_t)(b[i] - '0'); nd++; i++; }
        if (nd == 0 || nd > 9 || i >= lim) return 0;
        if (b[i] != (f == 0 ? ',' : '}')) return 0;
        i++;
    }
    *x = v[0]; *y = v[1];
    return 1;
}

int64_t or_emit_pair(const uint8_t *elems, const int64_t *off, int64_t R, const or_stage *st, int nst,
                     uint32_t *out_yx, uint32_t *out_reg, int64_t cap) {
    if (check_args(OR_U8, elems, off, R, st, nst, OR_SUM_I64)) return -1;
    int64_t n = 0;
    for (int64_t r = 0; r < R; r++) {
        for (int64_t g = off[r]; g < off[r + 1]; g++) {
            uint32_t v = elems[g];
            int keep = 1;
            for (int k = 0; k < nst && keep; k++) keep = apply_stage(&st[k], &v, r);
            uint32_t x, y;
            if (!keep || !parse_pair(elems, g, off[r + 1], &x, &y)) continue;
            if (n < cap) { out_yx[2 * n] = y; out_yx[2 * n + 1] = x; out_reg[n] = (uint32_t)r; }
            n++;
        }
    }
    return n;
}

/* ================================================================ one edge
 * Data queue Q and signal queue S between successive nodes n1 -> n2
 * (§3.1, Fig. 2a).  FIFO rings of fixed capacity.                  */
typedef struct { uint32_t v; int64_t i; int64_t g; int64_t tag; } item_t;   /* value, local idx, global idx, tag */
typedef struct { int kind; int64_t r; uint64_t credit; int64_t id; } sig_t;

typedef struct {
    item_t *q; int64_t qcap, qhead, qlen;
    sig_t *s;  int64_t scap, shead, slen;
    uint64_t sent;     /* sender: items emitted since the tail signal was enqueued */
    uint64_t cur;      /* receiver: current credit counter, initially 0            */
    int64_t next_sig_id;
} edge_t;

static int edge_init(edge_t *e, int64_t qcap, int64_t scap) {
    memset(e, 0, sizeof *e);
    e->qcap = qcap; e->scap = scap;
    e->q = (item_t *)calloc((size_t)(qcap > 0 ? qcap : 1), sizeof(item_t));
    e->s = (sig_t *)calloc((size_t)(scap > 0 ? scap : 1), sizeof(sig_t));
    return (e->q && e->s) ? OR_OK : OR_ENOMEM;
}
static void edge_free(edge_t *e) { free(e->q); free(e->s); e->q = NULL; e->s = NULL; }

static sig_t *sig_at(edge_t *e, int64_t k) { return &e->s[(e->shead + k) % e->scap]; }

/* Sender emits one data item: enqueue on Q, bump the emitted counter.       */
static void emit_data(edge_t *e, item_t x) {
    e->q[(e->qhead + e->qlen) % e->qcap] = x;
    e->qlen++;
    e->sent++;
}

/* Sender emits a signal with credit set by the two rules of P:304-312:
 * (1) S empty      -> credit = number of items queued on Q;
 * (2) S non-empty  -> credit = items emitted since the tail signal.
 * The emitted counter resets at every signal.  Returns the credit.          */
static uint64_t emit_signal(edge_t *e, int kind, int64_t r) {
    uint64_t credit = (e->slen == 0) ? (uint64_t)e->qlen : e->sent;
    sig_t *t = &e->s[(e->shead + e->slen) % e->scap];
    t->kind = kind; t->r = r; t->credit = credit; t->id = e->next_sig_id++;
    e->slen++;
    e->sent = 0;
    return credit;
}

/* Receiver: how many data items may be consumed now.
 * Rule (1): no signal queued -> all queued items.
 * Rule (2b): counter 0 and head credit > 0 -> move the head's credit into
 *            the counter (the head signal stays queued).
 * Rule (2a): counter > 0 -> at most the counter.                             */
static uint64_t admissible(edge_t *e) {
    if (e->slen == 0) return (uint64_t)e->qlen;
    sig_t *h = sig_at(e, 0);
    if (e->cur == 0 && h->credit > 0) { e->cur += h->credit; h->credit = 0; }
    return (uint64_t)e->qlen < e->cur ? (uint64_t)e->qlen : e->cur;
}

/* Receiver consumes n items (FIFO); the counter is decremented once per item
 * while a signal is pending.  More than admissible = violation.  */
static int consume(edge_t *e, uint64_t n, item_t *dst) {
    if (n > admissible(e)) return OR_ECREDIT;
    for (uint64_t k = 0; k < n; k++) { dst[k] = e->q[e->qhead]; e->qhead = (e->qhead + 1) % e->qcap; }
    e->qlen -= (int64_t)n;
    if (e->slen > 0) e->cur -= n;
    return OR_OK;
}

/* Receiver consumes the head signal iff the counter is 0 and the head carries
 * 0 credit (rule 2b, "Otherwise, n2 consumes s").                 */
static int next_signal(edge_t *e, sig_t *out) {
    if (e->slen == 0) return 0;
    (void)admissible(e);                       /* applies a pending 2b transfer */
    sig_t *h = sig_at(e, 0);
    if (e->cur != 0 || h->credit != 0) return 0;
    *out = *h;
    e->shead = (e->shead + 1) % e->scap;
    e->slen--;
    return 1;
}

/* Invariants checked after every protocol step (from the
 * proofs of Lemma 1 P:788-812 and Claim 1 P:820-833):
 *  - S empty => counter 0;
 *  - credit conservation: sum(credits on S) + counter = |Q| - sent;
 *  - counter > 0 => |Q| > 0.                                                 */
static int edge_invariants(edge_t *e) {
    if (e->slen == 0) return e->cur == 0 ? OR_OK : OR_EINVARIANT;
    uint64_t sum = e->cur;
    for (int64_t k = 0; k < e->slen; k++) sum += sig_at(e, k)->credit;
    if (sum != (uint64_t)e->qlen - e->sent) return OR_EINVARIANT;
    if (e->cur > 0 && e->qlen == 0) return OR_EINVARIANT;
    return OR_OK;
}

/* ---- single-edge API for the protocol pin tests (SPEC S:135-173 examples) */
void *or_edge_new(int64_t qcap, int64_t scap) {
    edge_t *e = (edge_t *)malloc(sizeof *e);
    if (!e) return NULL;
    if (edge_init(e, qcap, scap)) { edge_free(e); free(e); return NULL; }
    return e;
}
void or_edge_free(void *h) { if (h) { edge_free((edge_t *)h); free(h); } }
/* returns number enqueued (partial enqueue contract) */
int64_t or_edge_emit_data(void *h, int64_t n) {
    edge_t *e = (edge_t *)h; int64_t k = 0;
    for (; k < n && e->qlen < e->qcap; k++) { item_t x = {0, 0, 0, 0}; emit_data(e, x); }
    return k;
}
/* returns credit, or -2 when S is full (SignalQueueFull) */
int64_t or_edge_emit_signal(void *h, int kind, int64_t r) {
    edge_t *e = (edge_t *)h;
    if (e->slen >= e->scap) return OR_ESIGFULL;
    return (int64_t)emit_signal(e, kind, r);
}
int64_t or_edge_admissible(void *h) { return (int64_t)admissible((edge_t *)h); }
int or_edge_consume(void *h, int64_t n) {
    item_t *tmp = (item_t *)malloc(sizeof(item_t) * (size_t)(n > 0 ? n : 1));
    int rc = consume((edge_t *)h, (uint64_t)n, tmp);
    free(tmp);
    return rc;
}
/* returns 1 and fills kind/r when a signal was consumed, else 0 */
int or_edge_next_signal(void *h, int *kind, int64_t *r) {
    sig_t s;
    if (!next_signal((edge_t *)h, &s)) return 0;
    *kind = s.kind; *r = s.r;
    return 1;
}
/* state: [qlen, slen, cur, sent, head_credit or -1] */
void or_edge_state(void *h, int64_t *st) {
    edge_t *e = (edge_t *)h;
    st[0] = e->qlen; st[1] = e->slen; st[2] = (int64_t)e->cur; st[3] = (int64_t)e->sent;
    st[4] = e->slen ? (int64_t)sig_at(e, 0)->credit : -1;
}
int or_edge_check(void *h) { return edge_invariants((edge_t *)h); }

/* ============================================================ interpreter
 * Nodes: 0 = ENUMERATE, 1..nst = stages, nst+1 = AGGREGATE.
 * Edge k joins node k -> node k+1 (k = 0..nst).
 *
 * Trace events (optional, for Lemma 1 / bracketing / boundary checks):
 *   {node, type, a, b}:  type 0 = ENSEMBLE  (a = global idx of first item, b = count)
 *                        type 1 = ITEM      (a = global element idx, b = tag)
 *                        type 2 = SIGNAL    (a = kind, b = region)
 * ITEM events follow their ENSEMBLE event, one per item in lane order.      */
typedef struct { int32_t node, type; int64_t a, b; } or_event;

typedef struct {
    uint64_t data_firings, full_firings, items, signal_firings;
} or_node_stats;

typedef struct {
    /* inputs */
    int dtype; const void *elems; const int64_t *off; int64_t R;
    const or_stage *st; int nst; int agg; int strategy; int64_t w; int policy;
    /* state */
    edge_t *e;                 /* nst+1 edges                                 */
    int64_t par;               /* next parent to enumerate                    */
    int64_t par_i;             /* next element index within the open parent   */
    int par_begun;             /* Begin already emitted for par               */
    int64_t *open;             /* per node: open region (signal strategy)     */
    acc_t acc;                 /* aggregate node accumulator                  */
    int64_t acc_tag;           /* tagged: region of the running accumulator   */
    void *out0, *out1;
    or_node_stats *stats;      /* nst+2 entries                               */
    or_event *trace; int64_t trace_cap, trace_len;
    item_t *buf;               /* ensemble buffer                             */
    uint64_t rng;
    int check;                 /* run invariant checks after every step       */
} interp_t;

static void trace_ev(interp_t *I, int node, int type, int64_t a, int64_t b) {
    if (!I->trace) return;
    if (I->trace_len < I->trace_cap) { or_event *t = &I->trace[I->trace_len]; t->node = node; t->type = type; t->a = a; t->b = b; }
    I->trace_len++;
}

static int n_nodes(const interp_t *I) { return I->nst + 2; }

/* ---- enumeration (resumable)
 * Fires once: walks parents, emitting Begin(r), the element indices
 * 0..findCount(r)-1 of r, End(r), and stops when output space runs out or an
 * ensemble of w parents has been completed.  Signal strategy: signals on S0
 * with credits per the sender rules.  Tagged strategy:
 * no signals; each item carries its parent's tag.                            */
static int enum_can_fire(interp_t *I) {
    edge_t *o = &I->e[0];
    if (I->par >= I->R) return 0;
    int64_t n = I->off[I->par + 1] - I->off[I->par];
    if (I->strategy == OR_TAGGED) return n == 0 || o->qlen < o->qcap;
    if (!I->par_begun) return o->slen < o->scap;
    if (I->par_i < n) return o->qlen < o->qcap;
    return o->slen < o->scap;
}

static void enum_fire(interp_t *I) {
    edge_t *o = &I->e[0];
    int64_t done = 0;
    while (I->par < I->R && done < I->w) {
        int64_t r = I->par, n = I->off[r + 1] - I->off[r];
        if (I->strategy == OR_SIGNAL && !I->par_begun) {
            if (o->slen >= o->scap) break;
            emit_signal(o, OR_BEGIN, r);
            I->par_begun = 1;
        }
        while (I->par_i < n && o->qlen < o->qcap) {
            item_t x; x.v = 0; x.i = I->par_i; x.g = I->off[r] + I->par_i; x.tag = r;
            emit_data(o, x);
            I->par_i++;
        }
        if (I->par_i < n) break;                          /* suspended mid-region */
        if (I->strategy == OR_SIGNAL) {
            if (o->slen >= o->scap) break;
            emit_signal(o, OR_END, r);
        }
        I->par++; I->par_i = 0; I->par_begun = 0; done++;
    }
}

/* ---- node classification for the scheduler ---------------------------- */
static int64_t out_space(interp_t *I, int n) {       /* data slots downstream */
    if (n == n_nodes(I) - 1) return INT64_MAX;        /* aggregate: unbounded sink side */
    edge_t *o = &I->e[n];
    return o->qcap - o->qlen;
}
static int64_t out_sig_space(interp_t *I, int n) {
    if (n == n_nodes(I) - 1) return INT64_MAX;
    edge_t *o = &I->e[n];
    return o->scap - o->slen;
}

/* Is a signal consumable right now at node n (counter 0, head credit 0)?   */
static int sig_ready(interp_t *I, int n) {
    edge_t *in = &I->e[n - 1];
    if (in->slen == 0) return 0;
    (void)admissible(in);
    return in->cur == 0 && sig_at(in, 0)->credit == 0;
}

/* Upstream of node n can never produce more: no parents left to enumerate
 * and every edge strictly above n's input is empty.                          */
static int upstream_drained(interp_t *I, int n) {
    if (I->par < I->R) return 0;
    for (int k = 0; k < n - 1; k++) if (I->e[k].qlen || I->e[k].slen) return 0;
    return 1;
}

/* Fireability: pending data or signal, and room downstream for at
 * least one input's worth of outputs (max one data item per input for every
 * stage; one forwarded signal per signal).                                   */
static int node_can_fire(interp_t *I, int n) {
    if (n == 0) return enum_can_fire(I);
    edge_t *in = &I->e[n - 1];
    uint64_t a = admissible(in);
    if (a > 0 && out_space(I, n) >= 1) return 1;
    if (sig_ready(I, n) && out_sig_space(I, n) >= 1) return 1;
    return 0;
}

/* Full-first classification (A8): a data firing is "good" if it fills an
 * ensemble, exhausts a pending signal's credit, or upstream is drained.     */
static int node_good(interp_t *I, int n) {
    if (n == 0) return enum_can_fire(I);
    edge_t *in = &I->e[n - 1];
    if (sig_ready(I, n) && out_sig_space(I, n) >= 1) return 1;
    uint64_t a = admissible(in);
    int64_t sp = out_space(I, n);
    uint64_t e = a < (uint64_t)I->w ? a : (uint64_t)I->w;
    if ((int64_t)e > sp) e = (uint64_t)sp;
    if (e == 0) return 0;
    if (e == (uint64_t)I->w) return 1;
    if (in->slen > 0 && e == in->cur) return 1;
    if (upstream_drained(I, n) && e == a) return 1;
    return 0;
}

/* ---- the stage / aggregate data phase on one ensemble ----------------- */
static int agg_flush_tag(interp_t *I) {
    if (I->acc_tag >= 0) acc_end(I->agg, &I->acc, I->out0, I->out1, I->acc_tag);
    I->acc_tag = -1;
    return OR_OK;
}

static int run_ensemble(interp_t *I, int n, item_t *X, int64_t m) {
    int last = n_nodes(I) - 1;
    for (int64_t k = 0; k < m; k++) {
        item_t x = X[k];
        if (n == 1) {
            /* getItem(i) in the parent context (Fig. 5: b = getParent();
             * v = b->getItem(i)).  Signal strategy: the node's
             * open region; tagged: the item's tag.                          */
            int64_t parent = (I->strategy == OR_SIGNAL) ? I->open[n] : x.tag;
            if (parent < 0 || x.g != I->off[parent] + x.i) return OR_EINVARIANT;   /* context check */
            x.v = get_item(I->dtype, I->elems, I->off[parent] + x.i);
        }
        if (n == last) {
            if (I->strategy == OR_SIGNAL) {
                if (I->open[n] < 0) return OR_EINVARIANT;
                acc_run(I->agg, &I->acc, x.v, x.i);
            } else {
                /* region-id-keyed accumulation (tagged aggregate) */
                if (x.tag != I->acc_tag) { agg_flush_tag(I); acc_begin(&I->acc); I->acc_tag = x.tag; }
                acc_run(I->agg, &I->acc, x.v, x.i);
            }
            continue;
        }
        if (apply_stage(&I->st[n - 1], &x.v, x.tag)) emit_data(&I->e[n], x);   /* push; tag = parent */
    }
    return OR_OK;
}

/* ---- fire one node: data phase, then signal phase ---------- */
static int fire(interp_t *I, int n, int fallback) {
    if (n == 0) { enum_fire(I); return OR_OK; }
    edge_t *in = &I->e[n - 1];
    or_node_stats *S = &I->stats[n];
    int last = n_nodes(I) - 1;
    int partial_used = 0;
    /* data phase: "consumes as many queued data items as it can", limited by
     * queued items, downstream space and (if a signal is pending) the credit
     * counter, in ensembles of at most w.            */
    for (;;) {
        uint64_t a = admissible(in);
        int64_t sp = out_space(I, n);
        uint64_t e = a < (uint64_t)I->w ? a : (uint64_t)I->w;
        if ((int64_t)e > sp) e = (uint64_t)sp;
        if (e == 0) break;
        if (I->policy == OR_FULL_FIRST && e < (uint64_t)I->w) {
            int bounded = in->slen > 0 && e == in->cur;
            int drained = upstream_drained(I, n) && e == a;
            if (!bounded && !drained) {
                if (!fallback || partial_used) break;
                partial_used = 1;
            }
        }
        int rc = consume(in, e, I->buf);
        if (rc) return rc;
        S->data_firings++; S->items += e; if (e == (uint64_t)I->w) S->full_firings++;
        if (I->trace) {
            trace_ev(I, n, 0, I->buf[0].g, (int64_t)e);
            for (uint64_t k = 0; k < e; k++) trace_ev(I, n, 1, I->buf[k].g, I->buf[k].tag);
        }
        rc = run_ensemble(I, n, I->buf, (int64_t)e);
        if (rc) return rc;
        if (I->check) { rc = edge_invariants(in); if (rc) return rc; if (n < last && (rc = edge_invariants(&I->e[n]))) return rc; }
    }
    /* signal phase: only when the counter is 0; consume signals until none
     * remain or the counter becomes > 0.                        */
    sig_t s;
    while (in->slen > 0 && out_sig_space(I, n) >= 1 && next_signal(in, &s)) {
        S->signal_firings++;
        trace_ev(I, n, 2, s.kind, s.r);
        if (s.kind == OR_BEGIN) {
            if (I->open[n] >= 0) return OR_EUNMATCHED;
            I->open[n] = s.r;                                   /* begin(parent) */
            if (n == last) acc_begin(&I->acc);                  /* a::begin: acc = 0 */
            else emit_signal(&I->e[n], OR_BEGIN, s.r);          /* forwarded with fresh credit */
        } else {
            if (I->open[n] != s.r) return OR_EUNMATCHED;        /* UnmatchedEnd */
            if (n == last) acc_end(I->agg, &I->acc, I->out0, I->out1, s.r);   /* a::end: push(acc) */
            else emit_signal(&I->e[n], OR_END, s.r);
            I->open[n] = -1;
        }
        if (I->check) { int rc = edge_invariants(in); if (rc) return rc; if (n < last && (rc = edge_invariants(&I->e[n]))) return rc; }
    }
    return OR_OK;
}

static uint64_t rng_next(uint64_t *s) { *s += 0x9E3779B97F4A7C15ull; return or_mix64(*s); }

static int pick(interp_t *I, int *fallback) {
    int N = n_nodes(I);
    *fallback = 0;
    if (I->policy == OR_RANDOM) {
        int cand[64], nc = 0;
        for (int n = 0; n < N && nc < 64; n++) if (node_can_fire(I, n)) cand[nc++] = n;
        if (!nc) return -1;
        return cand[rng_next(&I->rng) % (uint64_t)nc];
    }
    if (I->policy == OR_FULL_FIRST) {
        for (int n = N - 1; n >= 0; n--) if (node_can_fire(I, n) && node_good(I, n)) return n;
        *fallback = 1;
    }
    for (int n = N - 1; n >= 0; n--) if (node_can_fire(I, n)) return n;   /* deepest fireable */
    return -1;
}

/* Monotone work counter: items and signals consumed, parents enumerated. */
static uint64_t progress_count(interp_t *I) {
    uint64_t p = (uint64_t)I->par * 3 + (uint64_t)I->par_i + (uint64_t)I->par_begun;
    for (int n = 1; n < n_nodes(I); n++) p += I->stats[n].items + I->stats[n].signal_firings;
    return p;
}

static int anything_pending(interp_t *I) {
    if (I->par < I->R) return 1;
    for (int k = 0; k <= I->nst; k++) if (I->e[k].qlen || I->e[k].slen) return 1;
    return 0;
}

/* The global scheduler: repeatedly fire some fireable
 * node until no node has queued data or signals.  Lemma 2 says
 * this terminates; a selection with nothing fireable while work is pending
 * would contradict Claim 2 and is reported as livelock.         */
int or_interp(int dtype, const void *elems, const int64_t *off, int64_t R,
              const or_stage *st, int nst, int agg, int strategy,
              int64_t w, int64_t qcap, int64_t scap, int policy, uint64_t seed, int check,
              void *out0, void *out1, or_node_stats *stats,
              or_event *trace, int64_t trace_cap, int64_t *trace_len) {
    int rc = check_args(dtype, elems, off, R, st, nst, agg);
    if (rc) return rc;
    if (w < 1 || qcap < 1 || scap < 1 || nst > 60) return OR_EARG;
    if (strategy != OR_SIGNAL && strategy != OR_TAGGED) return OR_EARG;
    interp_t I; memset(&I, 0, sizeof I);
    I.dtype = dtype; I.elems = elems; I.off = off; I.R = R; I.st = st; I.nst = nst; I.agg = agg;
    I.strategy = strategy; I.w = w; I.policy = policy; I.out0 = out0; I.out1 = out1;
    I.stats = stats; I.trace = trace; I.trace_cap = trace_cap; I.rng = seed; I.check = check;
    I.acc_tag = -1;
    memset(stats, 0, sizeof(or_node_stats) * (size_t)(nst + 2));
    I.e = (edge_t *)calloc((size_t)nst + 1, sizeof(edge_t));
    I.open = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nst + 2));
    I.buf = (item_t *)malloc(sizeof(item_t) * (size_t)w);
    if (!I.e || !I.open || !I.buf) { rc = OR_ENOMEM; goto done; }
    for (int k = 0; k <= nst; k++) if ((rc = edge_init(&I.e[k], qcap, scap))) goto done;
    for (int n = 0; n < nst + 2; n++) I.open[n] = -1;
    /* Tagged: regions whose items never reach the aggregate still report the
     * identity (A1/A2: exactly one result per parent).                      */
    if (strategy == OR_TAGGED) { acc_t z; acc_begin(&z); for (int64_t r = 0; r < R; r++) acc_end(agg, &z, out0, out1, r); }

    int idle = 0;
    for (;;) {
        int fb, n = pick(&I, &fb);
        if (n < 0) {
            if (anything_pending(&I)) { rc = OR_ELIVELOCK; goto done; }
            break;
        }
        uint64_t before = progress_count(&I);
        if ((rc = fire(&I, n, fb))) goto done;
        /* a firing must consume or emit something; more consecutive idle
         * selections than nodes means no progress (LivelockDetected) */
        idle = (progress_count(&I) == before) ? idle + 1 : 0;
        if (idle > n_nodes(&I)) { rc = OR_ELIVELOCK; goto done; }
    }
    if (strategy == OR_TAGGED) agg_flush_tag(&I);
    for (int n = 1; n < nst + 2 && strategy == OR_SIGNAL; n++) if (I.open[n] >= 0) { rc = OR_EUNMATCHED; goto done; }
    stats[0].items = (uint64_t)(R > 0 ? off[R] - off[0] : 0);   /* enumerated children (north-star invariant) */
done:
    if (trace_len) *trace_len = I.trace_len;
    if (I.e) for (int k = 0; k <= nst; k++) edge_free(&I.e[k]);
    free(I.e); free(I.open); free(I.buf);
    return rc;
}

/* Sharded brute force for the all-cores CPU baseline: instances on disjoint
 * contiguous region ranges are independent (regions are independent
 * contexts).  Each call evaluates regions [r0, r1).                 */
int or_brute_range(int dtype, const void *elems, const int64_t *off, int64_t r0, int64_t r1,
                   const or_stage *st, int nst, int agg, void *out0, void *out1) {
    if (r0 < 0 || r1 < r0) return OR_EARG;
    /* shift the output pointers so region r lands at index r */
    size_t s0 = (agg == OR_COUNT_MIN_U32) ? 4 : 8, s1 = (agg == OR_COUNT_MIN_U32) ? 4 : 8;
    /* and the parent contexts, which are indexed by region like the outputs */
    or_stage sh[16];
    if (nst > 16) return OR_EARG;
    for (int k = 0; k < nst; k++) {
        sh[k] = st[k];
        if (st[k].kind == OR_FILTER && st[k].op == OR_PARENT_LT) sh[k].table = (const uint8_t *)((const uint32_t *)st[k].table + r0);
    }
    return or_brute(dtype, elems, off + r0, r1 - r0, sh, nst, agg,
                    (char *)out0 + (size_t)r0 * s0, out1 ? (char *)out1 + (size_t)r0 * s1 : NULL);
}
