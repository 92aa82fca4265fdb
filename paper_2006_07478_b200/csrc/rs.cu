// rs.cu — the C ABI of include/rs.h (host side of the B200 pipeline).
//
// Kernels live in rs_kern.cuh / rs_pipe.cuh and are instantiated per
// aggregate in rs_k<AGG>.cu; see rs_kern.cuh for the execution model.
#define RS_HOST_ONLY
#include "rs_kern.cuh"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

using namespace rsk;

namespace {

// ------------------------------------------------------------ host side
thread_local std::string g_err;

rs_status fail(rs_status s, const std::string &msg) {
    g_err = msg;
    return s;
}

bool is_pow2(uint32_t x) { return x && !(x & (x - 1)); }

}  // namespace

void rsk::set_last_error(const std::string &m) { g_err = m; }

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
    // RS_STRATEGY_AUTO: one pipeline per strategy, the run picks (§8 f1)
    rs_pipeline *sub[2] = {nullptr, nullptr};
    uint32_t auto_min_len = 0;
    cudaStream_t last_stream = nullptr;
    bool has_parent = false;      // a PARENT_LT node reads d_parent_ctx
    // short-region kernel geometry (RS_FLAG_SHORT_*): its own ring / stage /
    // signal-queue sizes unless the caller fixed them
    bool geom_default = false;
    bool chunk_tail = false;          // 4-byte pipelines with chunk = 0: the last round of chunks is cut finer
    int sh_grid = 0, sh_wpb = 0;
    // RS_FLAG_TRACE event buffer (caller-owned device memory)
    void *trace = nullptr;
    uint64_t trace_bytes = 0;
};

namespace {

constexpr int AGG_SPLIT = 26;   // internal aggregate id of a fan-out (tree) pipeline

// Process-wide: the dynamic shared-memory limit of a kernel is a per-function
// attribute, so it is raised once per (kernel, device) to the opt-in maximum
// under a lock; launches and occupancy probes then only ever ask for less
// (per-run re-setting raced between handles on different threads).
std::mutex g_attr_mu;
bool ensure_smem_attr(KernelFn f, int dev) {
    static std::vector<std::pair<KernelFn, int>> done;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    for (auto &d : done)
        if (d.first == f && d.second == dev) return true;
    int optin = 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return false;
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, optin) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    done.push_back({f, dev});
    return true;
}

// Crossover region length (children per region) above which the signal
// strategy beats tagged on B200, by FILTER/TRANSFORM stage count
// (tools/crossover.py).
uint32_t auto_default(int nst) {
    static const uint32_t T[MAXK + 1] = {AUTO_T0, AUTO_T1, AUTO_T2, AUTO_T3, AUTO_T4};
    return T[nst < 0 ? 0 : (nst > MAXK ? MAXK : nst)];
}

bool get_launch(const rs_pipeline *p, Launch *L) {
    if (p->agg == AGG_SPLIT) {
        *L = launch_agg26_split(p->nst, p->cfg.queue_cap, p->cfg.signal_cap, p->cfg.q0_stage);
        return L->main != nullptr;
    }
    if (p->cfg.strategy == RS_STRATEGY_HYBRID) {
        const bool fuse = (p->cfg.flags & RS_FLAG_UNFUSED) == 0;
        if (p->agg == RS_OP_SUM_I64)
            *L = launch_agg20_hybrid(p->nst, fuse, (int)p->cfg.tag_from, p->cfg.queue_cap, p->cfg.signal_cap, p->cfg.q0_stage);
        else if (p->agg == RS_OP_EMIT_PAIR)
            *L = launch_agg25_hybrid(p->nst, fuse, (int)p->cfg.tag_from, p->cfg.queue_cap, p->cfg.signal_cap, p->cfg.q0_stage);
        else
            return false;
        return L->main != nullptr;
    }
    if (p->cfg.flags & (RS_FLAG_TRACE | RS_FLAG_PROFILE)) {    // the debug instantiations
        *L = launch_agg20_trace(p->nst, (p->cfg.flags & RS_FLAG_UNFUSED) == 0, p->cfg.queue_cap, p->cfg.signal_cap,
                                p->cfg.q0_stage);
        return true;
    }
    switch (p->agg) {
        case RS_OP_SUM_I64: *L = launch_agg20(p->nst, p->cfg.strategy == RS_STRATEGY_TAGGED, (p->cfg.flags & RS_FLAG_UNFUSED) == 0, p->cfg.queue_cap, p->cfg.signal_cap, p->cfg.q0_stage, p->cfg.strategy == RS_STRATEGY_CONTEXT); return true;
        case RS_OP_SUM_F32: *L = launch_agg21(p->nst, p->cfg.strategy == RS_STRATEGY_TAGGED, (p->cfg.flags & RS_FLAG_UNFUSED) == 0, p->cfg.queue_cap, p->cfg.signal_cap, p->cfg.q0_stage, p->cfg.strategy == RS_STRATEGY_CONTEXT); return true;
        case RS_OP_COUNT_MIN_U32: *L = launch_agg22(p->nst, p->cfg.strategy == RS_STRATEGY_TAGGED, (p->cfg.flags & RS_FLAG_UNFUSED) == 0, p->cfg.queue_cap, p->cfg.signal_cap, p->cfg.q0_stage, p->cfg.strategy == RS_STRATEGY_CONTEXT); return true;
        case RS_OP_SUM_I64_DROPS: *L = launch_agg27(p->nst, false, (p->cfg.flags & RS_FLAG_UNFUSED) == 0, p->cfg.queue_cap, p->cfg.signal_cap, p->cfg.q0_stage, false); return true;
        case RS_OP_EMIT_PAIR: *L = launch_agg25(p->nst, p->cfg.strategy == RS_STRATEGY_TAGGED, (p->cfg.flags & RS_FLAG_UNFUSED) == 0, p->cfg.queue_cap, p->cfg.signal_cap, p->cfg.q0_stage, false); return true;
        case RS_OP_EMIT_VALUE: *L = launch_agg24(p->nst, p->cfg.strategy == RS_STRATEGY_TAGGED, (p->cfg.flags & RS_FLAG_UNFUSED) == 0, p->cfg.queue_cap, p->cfg.signal_cap, p->cfg.q0_stage, p->cfg.strategy == RS_STRATEGY_CONTEXT); return true;
        case RS_OP_COUNT_XOR64: *L = launch_agg23(p->nst, p->cfg.strategy == RS_STRATEGY_TAGGED, (p->cfg.flags & RS_FLAG_UNFUSED) == 0, p->cfg.queue_cap, p->cfg.signal_cap, p->cfg.q0_stage, p->cfg.strategy == RS_STRATEGY_CONTEXT); return true;
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
    // the last round in pieces of C >> TAIL_SH: at most 2^TAIL_SH (instances + 1) more chunks
    // (instances <= 4095 covered; the prepass keeps uniform chunks when they would not fit)
    if (p->chunk_tail)
        w.max_chunks += std::min<long long>((1ll << TAIL_SH) * 4096, (n_elems + 16) / (C >> TAIL_SH) + 1);
    w.hdr = 0;
    w.stats = 256;
    w.fr = w.stats + align256(sizeof(unsigned long long) * (4 * (MAXK + 2) + 16));
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
        case RS_ERR_NCCL: return "RS_ERR_NCCL";
    }
    return "RS_ERR_UNKNOWN";
}

const char *rs_last_error(void) { return g_err.c_str(); }

rs_status rs_config_default(rs_config *cfg) {
    if (!cfg) return fail(RS_ERR_INVALID_ARG, "cfg is NULL");
    cfg->strategy = RS_STRATEGY_SIGNAL;
    cfg->simd_width = W;
    cfg->queue_cap = 0;        // 0 = auto (rs_pipeline_create picks 8w or 16w by stage count)
    cfg->signal_cap = 0;       // 0 = auto
    cfg->grid = 0;
    cfg->chunk = 0;
    cfg->flags = RS_FLAG_STATS;
    cfg->q0_stage = 0;
    cfg->auto_min_len = 0;
    cfg->tag_from = 0;
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
    // tree (fan-out): ENUMERATE, stages, SPLIT, AGGREGATE (child A), AGGREGATE (child B)
    int split_at = -1;
    for (int i = 1; i < n_nodes; ++i)
        if (nodes[i].kind == RS_NODE_SPLIT) {
            if (split_at >= 0) return fail(RS_ERR_INVALID_TOPOLOGY, "one SPLIT node per pipeline is built");
            split_at = i;
        }
    if (split_at >= 0) {
        if (split_at != n_nodes - 3 || nodes[n_nodes - 2].kind != RS_NODE_AGGREGATE ||
            nodes[n_nodes - 1].kind != RS_NODE_AGGREGATE)
            return fail(RS_ERR_INVALID_TOPOLOGY, "a SPLIT node's two children must be AGGREGATE leaves following it");
        if (nodes[n_nodes - 2].op != RS_OP_SUM_I64 || nodes[n_nodes - 1].op != RS_OP_SUM_I64 || elem != RS_I32)
            return fail(RS_ERR_UNSUPPORTED, "the fan-out is built for i32 elements and SUM_I64 leaves");
        if (split_at - 1 > 2) return fail(RS_ERR_UNSUPPORTED, "at most 2 stages before a SPLIT are built");
        if (cfg.strategy != RS_STRATEGY_SIGNAL || (cfg.flags & (RS_FLAG_TRACE | RS_FLAG_PROFILE)))
            return fail(RS_ERR_UNSUPPORTED, "the fan-out is built for the signal strategy");
        const int sop = nodes[split_at].op;
        if (sop != RS_OP_HASH_LT && sop != RS_OP_LT_U32 && sop != RS_OP_PARENT_LT)
            return fail(RS_ERR_UNSUPPORTED, "SPLIT ops: HASH_LT, LT_U32, PARENT_LT");
        for (int i = 1; i < split_at; ++i)
            if (nodes[i].kind != RS_NODE_FILTER && nodes[i].kind != RS_NODE_TRANSFORM)
                return fail(RS_ERR_INVALID_TOPOLOGY, "only FILTER/TRANSFORM nodes may precede a SPLIT");
        // validate and store the stages and the split op like a linear pipeline with the
        // split as its last stage (st[K] = the split op)
        rs_node lin[MAXK + 2];
        for (int i = 0; i <= split_at; ++i) lin[i] = nodes[i];
        lin[split_at].kind = RS_NODE_FILTER;
        lin[split_at + 1] = nodes[n_nodes - 1];              // an AGGREGATE(SUM_I64) closes the check list
        rs_config c = cfg;
        c.flags |= RS_FLAG_UNFUSED;
        if (c.queue_cap == 0) c.queue_cap = 8 * W;            // in-place ring and each child's queue
        rs_pipeline *q = nullptr;
        rs_status st = rs_pipeline_create(lin, split_at + 2, elem, &c, &q);
        if (st != RS_OK) return st;
        q->n_nodes = n_nodes;
        q->nst = split_at - 1;                                // stages before the split; st[nst] = split op
        q->agg = AGG_SPLIT;
        *out = q;
        return RS_OK;
    }
    if (nodes[n_nodes - 1].kind != RS_NODE_AGGREGATE && nodes[n_nodes - 1].kind != RS_NODE_EMIT)
        return fail(RS_ERR_INVALID_TOPOLOGY, "last node must be AGGREGATE or EMIT");
    const bool emit_ = nodes[n_nodes - 1].kind == RS_NODE_EMIT;
    const bool emit_op = nodes[n_nodes - 1].op == RS_OP_EMIT_VALUE || nodes[n_nodes - 1].op == RS_OP_EMIT_PAIR;
    if (emit_ && !emit_op) return fail(RS_ERR_UNSUPPORTED, "EMIT needs RS_OP_EMIT_VALUE or RS_OP_EMIT_PAIR");
    if (!emit_ && emit_op) return fail(RS_ERR_INVALID_TOPOLOGY, "RS_OP_EMIT_* belongs to an EMIT node");
    int nst = n_nodes - 2;
    for (int i = 1; i < n_nodes - 1; ++i) {
        if (nodes[i].kind == RS_NODE_ENUMERATE) return fail(RS_ERR_INVALID_TOPOLOGY, "nested ENUMERATE is not supported (single-level enumeration)");
        if (nodes[i].kind == RS_NODE_AGGREGATE || nodes[i].kind == RS_NODE_EMIT)
            return fail(RS_ERR_INVALID_TOPOLOGY, "AGGREGATE / EMIT must be the last node");
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
        case RS_OP_COUNT_XOR64:
            if (elem != RS_U8) return fail(RS_ERR_UNSUPPORTED, "COUNT_XOR64 needs u8 elements");
            break;
        case RS_OP_SUM_I64_DROPS:
            if (elem != RS_I32) return fail(RS_ERR_UNSUPPORTED, "SUM_I64_DROPS needs i32 elements");
            if (cfg.strategy != RS_STRATEGY_SIGNAL || (cfg.flags & (RS_FLAG_TRACE | RS_FLAG_PROFILE)))
                return fail(RS_ERR_UNSUPPORTED, "SUM_I64_DROPS is built for the signal strategy");
            if (nst < ((cfg.flags & RS_FLAG_UNFUSED) ? 1 : 2))
                return fail(RS_ERR_UNSUPPORTED, "SUM_I64_DROPS needs a first stage that is not the (fused) aggregate: "
                                                "2+ stages, or 1+ with RS_FLAG_UNFUSED");
            break;
        case RS_OP_EMIT_PAIR:
            if (elem != RS_U8) return fail(RS_ERR_UNSUPPORTED, "EMIT_PAIR needs u8 elements");
            if (cfg.strategy == RS_STRATEGY_CONTEXT) return fail(RS_ERR_UNSUPPORTED, "EMIT is built for the signal and tagged strategies");
            if (cfg.flags & (RS_FLAG_TRACE | RS_FLAG_PROFILE)) return fail(RS_ERR_UNSUPPORTED, "trace/profile are built for SUM_I64");
            break;
        case RS_OP_EMIT_VALUE:
            if (elem == RS_U8) return fail(RS_ERR_UNSUPPORTED, "EMIT_VALUE needs 4-byte elements");
            if (cfg.strategy == RS_STRATEGY_CONTEXT) return fail(RS_ERR_UNSUPPORTED, "EMIT is built for the signal and tagged strategies");
            if (cfg.flags & (RS_FLAG_TRACE | RS_FLAG_PROFILE)) return fail(RS_ERR_UNSUPPORTED, "trace/profile are built for SUM_I64");
            break;
        default: return fail(RS_ERR_UNSUPPORTED, "unknown aggregate op");
    }
    if (cfg.strategy == RS_STRATEGY_AUTO && (cfg.flags & (RS_FLAG_TRACE | RS_FLAG_PROFILE)))
        return fail(RS_ERR_UNSUPPORTED, "RS_FLAG_TRACE is built for SUM_I64 pipelines under the signal strategy");
    if (cfg.strategy == RS_STRATEGY_AUTO)
        for (int i = 1; i < n_nodes - 1; ++i)
            if (nodes[i].kind == RS_NODE_FILTER && nodes[i].op == RS_OP_PARENT_LT)
                return fail(RS_ERR_UNSUPPORTED, "PARENT_LT is built for the signal strategy (uniform context per ensemble, P:464-465)");
    if (cfg.strategy == RS_STRATEGY_AUTO) {
        rs_config c = cfg;
        if (c.chunk == 0) c.chunk = 8192;       // both strategies share the prepass's chunk table
        rs_pipeline *a = nullptr, *b = nullptr;
        c.strategy = RS_STRATEGY_SIGNAL;
        rs_status s = rs_pipeline_create(nodes, n_nodes, elem, &c, &a);
        if (s != RS_OK) return s;
        c.strategy = RS_STRATEGY_TAGGED;
        s = rs_pipeline_create(nodes, n_nodes, elem, &c, &b);
        if (s != RS_OK) { rs_pipeline_destroy(a); return s; }
        rs_pipeline *p = new rs_pipeline();
        p->cfg = a->cfg;
        p->cfg.strategy = RS_STRATEGY_AUTO;
        p->elem = elem;
        p->n_nodes = n_nodes;
        p->nst = nst;
        p->agg = agg;
        std::memcpy(p->st, a->st, sizeof p->st);
        p->sub[0] = a;
        p->sub[1] = b;
        p->auto_min_len = cfg.auto_min_len ? cfg.auto_min_len : auto_default(nst);
        *out = p;
        return RS_OK;
    }
    if (cfg.strategy != RS_STRATEGY_SIGNAL && cfg.strategy != RS_STRATEGY_TAGGED && cfg.strategy != RS_STRATEGY_CONTEXT &&
        cfg.strategy != RS_STRATEGY_HYBRID)
        return fail(RS_ERR_INVALID_ARG, "bad strategy");
    if (cfg.strategy == RS_STRATEGY_HYBRID) {
        const int age = (cfg.flags & RS_FLAG_UNFUSED) ? nst : nst - 1;   // the aggregating node's input edge
        if (agg != RS_OP_SUM_I64 && agg != RS_OP_EMIT_PAIR)
            return fail(RS_ERR_UNSUPPORTED, "RS_STRATEGY_HYBRID is built for SUM_I64 and EMIT_PAIR pipelines");
        if ((int)cfg.tag_from < 1 || (int)cfg.tag_from > age)
            return fail(RS_ERR_INVALID_ARG, "tag_from must be in 1 .. " + std::to_string(age) +
                                                " (stages - 1 fused, stages unfused)");
        if (cfg.flags & (RS_FLAG_TRACE | RS_FLAG_PROFILE)) return fail(RS_ERR_UNSUPPORTED, "trace/profile are built for the signal strategy");
    }
    if ((cfg.flags & (RS_FLAG_TRACE | RS_FLAG_PROFILE)) && (agg != RS_OP_SUM_I64 || cfg.strategy != RS_STRATEGY_SIGNAL))
        return fail(RS_ERR_UNSUPPORTED, "RS_FLAG_TRACE / RS_FLAG_PROFILE are built for SUM_I64 pipelines under the signal strategy");
    const bool ctx_ = cfg.strategy == RS_STRATEGY_CONTEXT;
    if (ctx_ && elem == RS_U8)
        return fail(RS_ERR_UNSUPPORTED, "the context strategy is built for 4-byte elements");
    if (cfg.flags & RS_FLAG_RESERVED8)
        return fail(RS_ERR_UNSUPPORTED, "flag 8 (the round-1 warp-specialised scheduler) was removed");
    if (cfg.simd_width == 0) cfg.simd_width = W;
    if (cfg.simd_width != (uint32_t)W) return fail(RS_ERR_UNSUPPORTED, "only simd_width 128 is built");
    // Defaults tuned on B200 (profiles/r1_tuning.txt): deep queues amortise the
    // scheduler for short pipelines; with 2+ stages a smaller footprint fits
    // twice the instances per SM, which wins.
    const int nst_ = n_nodes - 2;
    // In-place pipelines (4-byte elements, sequential scheduler): all queues
    // share one ring of queue_cap items fed by TMA stages of q0_stage; a big
    // ring amortises the scheduler, the tag ring doubles the tagged footprint
    // (profiles/r1_tuning.txt).
    const bool inplace = elem != RS_U8;
    const bool tagged_ = cfg.strategy == RS_STRATEGY_TAGGED || cfg.strategy == RS_STRATEGY_HYBRID;
    // (tagged with 0-1 stages, e.g. the R-MAT graph: an 8w ring in stages of 2w fits
    // 20 instances per SM: 1.41 -> 1.17 ms, profiles/r2_tuning.txt)
    if (cfg.queue_cap == 0)
        cfg.queue_cap = inplace ? (tagged_ ? (nst_ <= 1 ? 8 * W : 16 * W) : 32 * W) : (nst_ >= 2 ? 8 * W : 16 * W);
    if (cfg.signal_cap == 0)
        cfg.signal_cap = inplace ? 32 : (nst_ >= 2 ? 64 : 128);   // (context strategy: profiles/r1_tuning.txt)
    if (cfg.q0_stage == 0)
        cfg.q0_stage = inplace ? (tagged_ ? (nst_ <= 1 ? 256 : 512) : 1024)
                               : ((tagged_ || nst_ >= 2) ? 256 : 2048);   // byte streams: SWAR wants big stages
    if (!is_pow2(cfg.queue_cap) || cfg.queue_cap < 2 * W || cfg.queue_cap > 65536)
        return fail(RS_ERR_UNSUPPORTED, "queue_cap must be a power of 2 in [256, 65536]");
    if (!is_pow2(cfg.signal_cap) || cfg.signal_cap < 4 || cfg.signal_cap > 65536)
        return fail(RS_ERR_UNSUPPORTED, "signal_cap must be a power of 2 in [4, 65536]");
    // children per claim: 2^15 for 4-byte signal / context pipelines (fewer regions split
    // across chunks: variable L = 4096 1.84 -> 1.63 ms), 2^13 for tagged ones (R-MAT's skewed
    // degrees balance better) and byte streams (profiles/r2_tuning.txt)
    if (cfg.chunk == 0) cfg.chunk = (inplace && !tagged_) ? 32768 : 8192;
    if (!is_pow2(cfg.chunk) || cfg.chunk < 2048 || cfg.chunk > (1u << 24))
        return fail(RS_ERR_UNSUPPORTED, "chunk must be a power of 2 in [2048, 2^24]");
    if (cfg.grid < 0) return fail(RS_ERR_INVALID_ARG, "grid must be >= 0");
    if (!is_pow2(cfg.q0_stage) || cfg.q0_stage < 128 || cfg.q0_stage > 4096)
        return fail(RS_ERR_UNSUPPORTED, "q0_stage must be a power of 2 in [128, 4096]");
    if (cfg.chunk < cfg.q0_stage) return fail(RS_ERR_UNSUPPORTED, "chunk must be >= q0_stage");   // stages never straddle chunks
    rs_pipeline *p = new rs_pipeline();
    p->geom_default = !cfg_in || (cfg_in->queue_cap == 0 && cfg_in->signal_cap == 0 && cfg_in->q0_stage == 0);
    // (signal / context: fixed L = 4096 0.99 -> 0.97 ms, variable 1.25 -> 1.21; tagged Zipf
    // measured 1 % slower with it, so tagged and AUTO keep uniform chunks)
    p->chunk_tail = (!cfg_in || cfg_in->chunk == 0) && inplace && !tagged_ && cfg.strategy != RS_STRATEGY_AUTO;
    p->cfg = cfg;
    p->elem = elem;
    p->n_nodes = n_nodes;
    p->nst = nst;
    p->agg = agg;
    for (int i = 0; i < nst; ++i) {
        const rs_node &nd = nodes[i + 1];
        // op sets per element type (the kernels compile only these, rs_pipe.cuh with_op_k)
        const bool ok = elem == RS_U8 ? nd.op == RS_OP_CLASS
                      : elem == RS_F32 ? (nd.op == RS_OP_HASH_LT || nd.op == RS_OP_LT_U32 || nd.op == RS_OP_SCALE_F32 ||
                                          nd.op == RS_OP_PARENT_LT)
                                       : (nd.op == RS_OP_HASH_LT || nd.op == RS_OP_LT_U32 || nd.op == RS_OP_AFFINE_I32 ||
                                          nd.op == RS_OP_PARENT_LT);
        if (!ok) {
            delete p;
            return fail(RS_ERR_UNSUPPORTED, "op " + std::to_string(nd.op) + " is not built for this element type "
                                            "(i32/u32: HASH_LT LT_U32 AFFINE_I32 PARENT_LT; f32: HASH_LT LT_U32 "
                                            "SCALE_F32 PARENT_LT; u8: CLASS)");
        }
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
                case RS_OP_PARENT_LT:
                    if (elem == RS_U8) { delete p; return fail(RS_ERR_UNSUPPORTED, "PARENT_LT needs 4-byte elements"); }
                    if (cfg.strategy != RS_STRATEGY_SIGNAL) {
                        delete p;
                        return fail(RS_ERR_UNSUPPORTED, "PARENT_LT is built for the signal strategy (uniform context per ensemble, P:464-465)");
                    }
                    p->has_parent = true;
                    break;
                case RS_OP_CLASS: {
                    if (!nd.table) { delete p; return fail(RS_ERR_INVALID_ARG, "CLASS needs a 32-byte table"); }
                    if (elem != RS_U8) { delete p; return fail(RS_ERR_UNSUPPORTED, "CLASS needs u8 elements"); }
                    std::memcpy(s.table, nd.table, 32);
                    // a single-member class runs the SWAR byte test (a = 0x100 | member)
                    int members = 0, last = 0;
                    for (int c = 0; c < 256; ++c)
                        if ((nd.table[c >> 3] >> (c & 7)) & 1) { ++members; last = c; }
                    if (members == 1) s.a = 0x100u | (uint32_t)last;
                    break;
                }
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
    if (p->sub[0]) {                      // AUTO: enough for either strategy
        size_t a = 0, b = 0;
        rs_status s = rs_pipeline_workspace_bytes(p->sub[0], n_regions, n_elems, &a);
        if (s == RS_OK) s = rs_pipeline_workspace_bytes(p->sub[1], n_regions, n_elems, &b);
        *bytes = a > b ? a : b;
        return s;
    }
    Launch L;
    if (!get_launch(p, &L)) return fail(RS_ERR_UNSUPPORTED, "aggregate not built");
    *bytes = layout(p, n_regions, n_elems, L).total;
    return RS_OK;
}

// Geometry and kernel parameters of one (non-AUTO) pipeline for a run.
struct Prep {
    Launch L;
    KParams K;
    WsLayout wl;
    uint32_t cta_smem;
};

static rs_status prepare(rs_pipeline *p, const void *d_elems, int64_t n_elems, const int64_t *d_offsets,
                         int64_t n_regions, rs_aggregates out, void *d_ws, size_t ws_bytes, Prep &pr) {
    Launch &L = pr.L;
    if (!get_launch(p, &L)) return fail(RS_ERR_UNSUPPORTED, "aggregate not built");
    if (!out.v0 || (L.out_bytes1 && !out.v1)) return fail(RS_ERR_INVALID_ARG, "output array is NULL");
    pr.wl = layout(p, n_regions, n_elems, L);
    if (!d_ws || ws_bytes < pr.wl.total) return fail(RS_ERR_WORKSPACE, "workspace smaller than rs_pipeline_workspace_bytes");
    if (((uintptr_t)d_ws & 255u) != 0) return fail(RS_ERR_WORKSPACE, "workspace must be 256-byte aligned");
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(RS_ERR_CUDA, "cudaGetDevice failed");
    if (!ensure_smem_attr(L.main, dev)) return fail(RS_ERR_CUDA, "cannot raise the kernel's shared-memory limit");
    if (p->device != dev || p->grid == 0) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // one instance per warp; pick warps-per-CTA to pack the most instances per SM
        int best = 0, best_w = 1;
        for (int w = WPB_MAX; w >= 1; --w) {
            const uint32_t bytes = L.inst_bytes * w;
            int per_sm = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, L.main, w * 32, bytes) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            if (per_sm * w > best) { best = per_sm * w; best_w = w; }
        }
        if (best < 1) return fail(RS_ERR_UNSUPPORTED, "pipeline does not fit on an SM (queue/signal capacities too large)");
        p->wpb = best_w;
        p->grid = p->cfg.grid > 0 ? p->cfg.grid : sms * (best / best_w);
        p->device = dev;
        p->sh_grid = 0;                   // re-sized on the next short-region launch
    }
    pr.cta_smem = L.inst_bytes * p->wpb;

    KParams &K = pr.K;
    std::memset(&K, 0, sizeof K);
    K.elems = (const uint8_t *)d_elems;
    K.n_elems = n_elems;
    K.off = (const long long *)d_offsets;
    K.R = n_regions;
    K.out0 = out.v0;
    K.out1 = out.v1;
    uint8_t *ws = (uint8_t *)d_ws;
    K.hdr = (WsHdr *)(ws + pr.wl.hdr);
    K.stats = (unsigned long long *)(ws + pr.wl.stats);
    K.chunk_fr = (uint32_t *)(ws + pr.wl.fr);
    K.part0 = ws + pr.wl.part0;
    K.part1 = ws + pr.wl.part1;
    K.max_chunks = pr.wl.max_chunks;
    K.C = p->cfg.chunk;
    K.tail = p->chunk_tail ? 1u : 0u;
    K.nwarps = (uint32_t)(p->grid * p->wpb);
    K.qcap = p->cfg.queue_cap;
    K.scap = p->cfg.signal_cap;
    K.q0_stage = p->cfg.q0_stage;
    K.ring0 = L.ring0;
    K.esize = p->elem == RS_U8 ? 1u : 4u;
    K.flags = p->cfg.flags;
    K.tagged = p->cfg.strategy == RS_STRATEGY_TAGGED || p->cfg.strategy == RS_STRATEGY_HYBRID;
    K.nst = p->nst;
    std::memcpy(K.st, p->st, sizeof K.st);
    return RS_OK;
}

struct EmitOut {
    uint32_t *vals = nullptr, *regs = nullptr;
    uint64_t cap = 0;
    uint64_t *count = nullptr;
};

static rs_status run_impl(rs_pipeline *p, const void *d_elems, int64_t n_elems, const int64_t *d_offsets,
                          int64_t n_regions, const void *d_ctx, rs_aggregates out, void *d_ws, size_t ws_bytes,
                          cudaStream_t stream, const EmitOut *em = nullptr) {
    if (!p) return fail(RS_ERR_INVALID_ARG, "pipeline is NULL");
    p->launches = 0;
    if (n_regions < 0 || n_regions >= (1ll << 31)) return fail(RS_ERR_INVALID_ARG, "n_regions must be in [0, 2^31)");
    if (n_elems < 0 || n_elems >= (1ll << 40)) return fail(RS_ERR_INVALID_ARG, "bad n_elems");
    if (n_regions == 0) return RS_OK;
    if (!d_offsets) return fail(RS_ERR_INVALID_ARG, "d_offsets is NULL");
    if (n_elems > 0 && !d_elems) return fail(RS_ERR_INVALID_ARG, "d_elems is NULL");
    if (((uintptr_t)d_elems & 15u) != 0) return fail(RS_ERR_INVALID_ARG, "d_elems must be 16-byte aligned");
    if (((uintptr_t)d_offsets & 7u) != 0) return fail(RS_ERR_INVALID_ARG, "d_offsets must be 8-byte aligned");

    // RS_STRATEGY_AUTO: both strategies' kernels are enqueued; the prepass
    // decides on the device from the call's children count and the kernel of
    // the other strategy exits at once (no host synchronisation).
    const bool is_auto = p->sub[0] != nullptr;
    Prep pa, pb;
    rs_status s = prepare(is_auto ? p->sub[0] : p, d_elems, n_elems, d_offsets, n_regions, out, d_ws, ws_bytes, pa);
    if (s != RS_OK) return s;
    if (is_auto) {
        s = prepare(p->sub[1], d_elems, n_elems, d_offsets, n_regions, out, d_ws, ws_bytes, pb);
        if (s != RS_OK) return s;
        pa.K.auto_sel = 1;
        pb.K.auto_sel = 2;
    }
    if (p->has_parent && !d_ctx) return fail(RS_ERR_INVALID_ARG, "a PARENT_LT node needs d_parent_ctx");
    if (d_ctx && ((uintptr_t)d_ctx & 3u)) return fail(RS_ERR_INVALID_ARG, "d_parent_ctx must be 4-byte aligned");
    pa.K.ctx = (const uint32_t *)d_ctx;
    pb.K.ctx = (const uint32_t *)d_ctx;
    if ((p->agg == RS_OP_EMIT_VALUE || p->agg == RS_OP_EMIT_PAIR) != (em != nullptr))
        return fail(RS_ERR_INVALID_ARG, em ? "not an EMIT pipeline (use rs_pipeline_run)" : "EMIT pipelines run with rs_pipeline_run_emit");
    if (em) {
        for (KParams *k : {&pa.K, &pb.K}) {
            k->emit_vals = em->vals;
            k->emit_regs = em->regs;
            k->emit_cap = em->cap;
            k->emit_n = (unsigned long long *)em->count;
        }
        if (cudaMemsetAsync(em->count, 0, 8, stream) != cudaSuccess) return fail(RS_ERR_CUDA, "emit count reset failed");
    }
    KParams Kpre = pa.K;
    if (is_auto) {
        Kpre.tagged = -1;
        Kpre.auto_min_len = p->auto_min_len;
    }
    // short-region kernel (RS_FLAG_SHORT_ON / _OFF, rs.h).  Default geometry:
    // a ring of 16w items in TMA stages of 4w and signal queues of 128 -- the
    // kernel is latency-bound at short regions, and the smaller footprint fits
    // 16 instances per SM (profiles/r2_tuning.txt)
    Launch shl{};
    Prep ps = pa;
    if (!is_auto && (p->agg == RS_OP_SUM_I64 || p->agg == RS_OP_COUNT_MIN_U32) && p->cfg.strategy == RS_STRATEGY_SIGNAL &&
        p->nst >= 1 &&
        !(p->cfg.flags & (RS_FLAG_UNFUSED | RS_FLAG_TRACE | RS_FLAG_PROFILE | RS_FLAG_SHORT_OFF)) &&
        ((p->cfg.flags & RS_FLAG_SHORT_ON) || n_elems < 2ll * W * n_regions)) {
        const uint32_t qc = p->geom_default ? 16 * W : p->cfg.queue_cap;
        const uint32_t sc = p->geom_default ? 128 : p->cfg.signal_cap;
        const uint32_t sb = p->geom_default ? 4 * W : p->cfg.q0_stage;
        shl = p->agg == RS_OP_SUM_I64 ? short_launch_agg20(p->nst, qc, sc, sb) : short_launch_agg22(p->nst, qc, sc, sb);
        if (shl.main) {
            if (!ensure_smem_attr(shl.main, p->device)) return fail(RS_ERR_CUDA, "cannot raise the kernel's shared-memory limit");
            if (p->sh_grid == 0) {
                int best = 0, best_w = 1;
                for (int w = WPB_MAX; w >= 1; --w) {
                    int per_sm = 0;
                    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, shl.main, w * 32, shl.inst_bytes * w) != cudaSuccess) {
                        cudaGetLastError();
                        continue;
                    }
                    if (per_sm * w > best) { best = per_sm * w; best_w = w; }
                }
                if (best < 1) return fail(RS_ERR_UNSUPPORTED, "short-region kernel does not fit on an SM");
                int sms = 0;
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
                p->sh_wpb = best_w;
                p->sh_grid = p->cfg.grid > 0 ? p->cfg.grid : sms * (best / best_w);
            }
            ps.K.qcap = qc;
            ps.K.scap = sc;
            ps.K.q0_stage = sb;
            ps.K.ring0 = shl.ring0;
            ps.cta_smem = shl.inst_bytes * p->sh_wpb;
        }
    }
    KernelFn sh = shl.main;
    const bool both = sh && !(p->cfg.flags & RS_FLAG_SHORT_ON);
    if (both) {
        Kpre.short_len = SHORT_LEN;
        pa.K.short_sel = 1;
        ps.K.short_sel = 2;
    }
    if ((pa.K.flags & RS_FLAG_TRACE) && (!p->trace || p->trace_bytes < 64))
        return fail(RS_ERR_INVALID_ARG, "RS_FLAG_TRACE needs rs_pipeline_set_trace");
    if (pa.K.flags & RS_FLAG_TRACE) {
        pa.K.trace = (uint32_t *)p->trace;
        pa.K.trace_cap = (uint32_t)std::min<uint64_t>((p->trace_bytes - 32) / 32, 0xffffffffu);
        if (cudaMemsetAsync(p->trace, 0, 32, stream) != cudaSuccess) return fail(RS_ERR_CUDA, "trace reset failed");
    }
    int pre_blocks = (int)std::min<long long>((2 * pa.wl.max_chunks + 2 + 255) / 256, 148 * 8);
    if (Kpre.tagged || (Kpre.flags & RS_FLAG_VALIDATE)) pre_blocks = std::max(pre_blocks, 148 * 8);
    const bool timing = (pa.K.flags & RS_FLAG_TIMING) != 0;
    if (timing && !p->ev[0])
        for (int i = 0; i < 4; ++i) cudaEventCreate(&p->ev[i]);
    p->timed = timing;
    // header (claim cursor, error word, strategy) + stats, zeroed before any kernel reads them
    if (cudaMemsetAsync(d_ws, 0, pa.wl.fr, stream) != cudaSuccess) return fail(RS_ERR_CUDA, "workspace reset failed");
    if (timing) cudaEventRecord(p->ev[0], stream);
    pa.L.pre<<<pre_blocks, 256, 0, stream>>>(Kpre);
    if (timing) cudaEventRecord(p->ev[1], stream);
    if (!sh || both)
        pa.L.main<<<(is_auto ? p->sub[0] : p)->grid, (is_auto ? p->sub[0] : p)->wpb * 32, pa.cta_smem, stream>>>(pa.K);
    if (sh) sh<<<p->sh_grid, p->sh_wpb * 32, ps.cta_smem, stream>>>(ps.K);
    if (is_auto) pb.L.main<<<p->sub[1]->grid, p->sub[1]->wpb * 32, pb.cta_smem, stream>>>(pb.K);
    if (timing) cudaEventRecord(p->ev[2], stream);
    int fix_blocks = (int)std::min<long long>((pa.wl.max_chunks + 255) / 256, 148 * 8);
    pa.L.fix<<<std::max(fix_blocks, 1), 256, 0, stream>>>(pa.K);
    if (timing) cudaEventRecord(p->ev[3], stream);
    p->launches = (is_auto || both) ? 4 : 3;
    p->last_ws = d_ws;
    p->last_stream = stream;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, std::string("launch failed: ") + cudaGetErrorString(e));
    return RS_OK;
}

rs_status rs_pipeline_run(rs_pipeline *p, const void *d_elems, int64_t n_elems, const int64_t *d_offsets,
                          int64_t n_regions, const void *d_parent_ctx, rs_aggregates out, void *d_ws, size_t ws_bytes,
                          rs_stream stream) {
    if (!p) return fail(RS_ERR_INVALID_ARG, "pipeline is NULL");
    return run_impl(p, d_elems, n_elems, d_offsets, n_regions, d_parent_ctx, out, d_ws, ws_bytes, (cudaStream_t)stream);
}

rs_status rs_pipeline_run_emit(rs_pipeline *p, const void *d_elems, int64_t n_elems, const int64_t *d_offsets,
                               int64_t n_regions, const void *d_parent_ctx, uint32_t *d_values, uint32_t *d_regions,
                               uint64_t capacity, uint64_t *d_count, void *d_ws, size_t ws_bytes, rs_stream stream) {
    if (!p) return fail(RS_ERR_INVALID_ARG, "pipeline is NULL");
    if (!d_count || (capacity > 0 && (!d_values || !d_regions)))
        return fail(RS_ERR_INVALID_ARG, "emit outputs are NULL");
    if (((uintptr_t)d_count & 7u) != 0) return fail(RS_ERR_INVALID_ARG, "d_count must be 8-byte aligned");
    if (n_regions == 0) {
        if (cudaMemsetAsync(d_count, 0, 8, (cudaStream_t)stream) != cudaSuccess) return fail(RS_ERR_CUDA, "emit count reset failed");
        return RS_OK;
    }
    EmitOut em;
    em.vals = d_values;
    em.regs = d_regions;
    em.cap = capacity;
    em.count = d_count;
    static uint32_t dummy_out;                        // prepare() wants a non-null v0 (never written)
    rs_aggregates out{d_values ? (void *)d_values : (void *)&dummy_out, nullptr};
    return run_impl(p, d_elems, n_elems, d_offsets, n_regions, d_parent_ctx, out, d_ws, ws_bytes, (cudaStream_t)stream,
                    &em);
}

rs_status rs_pipeline_run_host(rs_pipeline *p, const void *h_elems, int64_t n_elems, const int64_t *h_offsets,
                               int64_t n_regions, const void *h_parent_ctx, rs_aggregates h_out, rs_stream stream_) {
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
    const size_t b_ctx = h_parent_ctx ? align256(4 * (size_t)n_regions) : 0;
    const size_t need = b_el + b_off + b_o0 + b_o1 + b_ctx + ws;
    if (p->h_dbuf_bytes < need) {
        if (p->h_dbuf) cudaFree(p->h_dbuf);
        p->h_dbuf = nullptr;
        p->h_dbuf_bytes = 0;
        if (cudaMalloc(&p->h_dbuf, need) != cudaSuccess) return fail(RS_ERR_CUDA, "cudaMalloc of run_host buffers failed");
        p->h_dbuf_bytes = need;
    }
    uint8_t *d = (uint8_t *)p->h_dbuf;
    void *d_el = d, *d_off = d + b_el, *d_o0 = d + b_el + b_off, *d_o1 = d + b_el + b_off + b_o0;
    void *d_ctx = h_parent_ctx ? d + b_el + b_off + b_o0 + b_o1 : nullptr;
    void *d_ws = d + b_el + b_off + b_o0 + b_o1 + b_ctx;
    if (n_elems && cudaMemcpyAsync(d_el, h_elems, esz * (size_t)n_elems, cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, "H2D elements failed");
    if (cudaMemcpyAsync(d_off, h_offsets, 8 * (size_t)(n_regions + 1), cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, "H2D offsets failed");
    if (d_ctx && cudaMemcpyAsync(d_ctx, h_parent_ctx, 4 * (size_t)n_regions, cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, "H2D parent contexts failed");
    rs_aggregates dout{d_o0, L.out_bytes1 ? d_o1 : nullptr};
    rs_status s = run_impl(p, d_el, n_elems, (const int64_t *)d_off, n_regions, d_ctx, dout, d_ws, ws, stream);
    if (s != RS_OK) return s;
    if (cudaMemcpyAsync(h_out.v0, d_o0, (size_t)L.out_bytes0 * (size_t)n_regions, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, "D2H aggregates failed");
    if (L.out_bytes1 && cudaMemcpyAsync(h_out.v1, d_o1, (size_t)L.out_bytes1 * (size_t)n_regions, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, "D2H aggregates failed");
    if (cudaStreamSynchronize(stream) != cudaSuccess) return fail(RS_ERR_CUDA, "stream synchronize failed");
    return RS_OK;
}

rs_status rs_pipeline_profile(rs_pipeline *p, uint64_t *host16, rs_stream stream) {
    if (!p || !host16) return fail(RS_ERR_INVALID_ARG, "NULL argument");
    if (!p->last_ws) { std::memset(host16, 0, 16 * sizeof(uint64_t)); return RS_OK; }
    if (cudaMemcpyAsync(host16, (uint8_t *)p->last_ws + 256 + sizeof(unsigned long long) * 4 * (MAXK + 2),
                        16 * sizeof(uint64_t), cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess ||
        cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
        return fail(RS_ERR_CUDA, "profile copy failed");
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

int rs_pipeline_launches(const rs_pipeline *p) {
    return p ? p->launches : 0;
}

// Strategy of the last run: an AUTO handle reads the prepass's decision from
// the workspace header (synchronises the last run's stream).
static int32_t last_sel(const rs_pipeline *p) {
    if (!p->sub[0]) return p->cfg.strategy;
    if (!p->last_ws) return RS_STRATEGY_AUTO;
    WsHdr h;
    if (cudaMemcpyAsync(&h, p->last_ws, sizeof h, cudaMemcpyDeviceToHost, p->last_stream) != cudaSuccess ||
        cudaStreamSynchronize(p->last_stream) != cudaSuccess)
        return RS_STRATEGY_AUTO;
    return h.sel ? RS_STRATEGY_TAGGED : RS_STRATEGY_SIGNAL;
}

rs_status rs_pipeline_last_strategy(const rs_pipeline *p, int32_t *strategy) {
    if (!p || !strategy) return fail(RS_ERR_INVALID_ARG, "NULL argument");
    *strategy = last_sel(p);
    return RS_OK;
}

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
    if (p->sub[0]) p = p->sub[last_sel(p) == RS_STRATEGY_TAGGED ? 1 : 0];
    if (grid) *grid = p->grid;
    if (wpb) *wpb = p->wpb;
    if (chunk) *chunk = (int32_t)p->cfg.chunk;
    return RS_OK;
}

rs_status rs_pipeline_set_trace(rs_pipeline *p, void *d_trace, uint64_t bytes) {
    if (!p) return fail(RS_ERR_INVALID_ARG, "NULL pipeline");
    if (d_trace && (bytes < 64 || ((uintptr_t)d_trace & 15u)))
        return fail(RS_ERR_INVALID_ARG, "trace buffer must be 16-byte aligned and >= 64 bytes");
    p->trace = d_trace;
    p->trace_bytes = d_trace ? bytes : 0;
    return RS_OK;
}

void rs_pipeline_destroy(rs_pipeline *p) {
    if (!p) return;
    rs_pipeline_destroy(p->sub[0]);
    rs_pipeline_destroy(p->sub[1]);
    if (p->h_dbuf) cudaFree(p->h_dbuf);
    for (int i = 0; i < 4; ++i)
        if (p->ev[i]) cudaEventDestroy(p->ev[i]);
    delete p;
}

}  // extern "C"
