/*
 * rs.h — C ABI of the B200-native region-based streaming library.
 *
 * Implements the data-parallel hot path of Timcheck & Buhler, "Streaming
 * Computations with Region-Based State on SIMD Architectures" (arXiv
 * 2006.07478).  Citations "P:a-b" are lines of the paper's PAPER.md with the
 * section they fall in; design readings are DESIGN.md §3 (A1-A26).
 *
 * What a call computes (§4, Fig. 3-5): a stream of
 * composite parent objects ("regions"), each holding 0+ elements, is
 * ENUMERATED into the stream of its elements, passed
 * through FILTER / TRANSFORM stages that keep or drop each item (P:109-118
 * §2.1, Fig. 5 `if (isGood(v)) push(...)` P:529), and AGGREGATED to exactly
 * one result per parent (Fig. 5 begin/run/end P:532-534).
 * Region boundaries reach every stage either as credit-counted Begin/End
 * signals (RS_STRATEGY_SIGNAL: §3) or as a region tag carried by
 * every item (RS_STRATEGY_TAGGED: §2.3, §5).  Both give
 * identical integer results.
 *
 * Conventions
 *  - Every device pointer is a CUDA device address in the current context;
 *    every buffer is owned by the caller; the library never frees or
 *    reallocates caller memory and allocates nothing inside rs_pipeline_run.
 *  - Functions return rs_status; nothing throws across the ABI.  Argument
 *    and topology errors are reported synchronously before any launch;
 *    rs_last_error() gives a thread-local detail string.
 *  - rs_pipeline_run enqueues on `stream` and returns immediately; results
 *    and statistics are valid once the stream is synchronised.
 *  - A pipeline handle must not be used by two threads at once.  Distinct
 *    handles (with distinct workspaces) may run concurrently.
 */
#ifndef RS_H
#define RS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same object as cudaStream_t / CUstream; NULL = the legacy default stream. */
typedef struct CUstream_st *rs_stream;

typedef enum {
    RS_OK = 0,
    RS_ERR_INVALID_ARG = -1,       /* null pointer, bad size, misaligned buffer, ...      */
    RS_ERR_INVALID_TOPOLOGY = -2,  /* node list is not ENUMERATE (FILTER|TRANSFORM)* AGG  */
    RS_ERR_UNSUPPORTED = -3,       /* op/dtype combination or config value not built      */
    RS_ERR_WORKSPACE = -4,         /* workspace missing or smaller than the query         */
    RS_ERR_CUDA = -5,              /* a CUDA call or launch failed                        */
    RS_ERR_PROTOCOL = -6,          /* device detected a protocol violation (rs_pipeline_check) */
    RS_ERR_NCCL = -7               /* NCCL unavailable or an NCCL call failed (rs_comm_*)      */
} rs_status;

/* Node kinds of the linear pipeline (§2.1; DAGs and cycles are
 * excluded by the paper). */
typedef enum {
    RS_NODE_ENUMERATE = 1,   /* parent -> its elements, findCount = offsets  */
    RS_NODE_FILTER = 2,      /* keep or drop each item (0..1 outputs per input)          */
    RS_NODE_TRANSFORM = 3,   /* rewrite each item (exactly 1 output per input)           */
    RS_NODE_AGGREGATE = 4,   /* one result per parent (begin/run/end)         */
    RS_NODE_EMIT = 5,        /* element-wise exit: every surviving item is written out with
                                its parent's id, "stripped of their parent context"
                                (taxi stage 2) -- rs_pipeline_run_emit */
    RS_NODE_SPLIT = 6        /* fan-out (tree topology, Fig. 1b): routes each item to
                                child A (its FILTER op holds) or child B; both children follow it
                                in the node list (pre-order) and must be AGGREGATE(SUM_I64) leaves:
                                ENUMERATE, 0..2 stages, SPLIT, AGGREGATE, AGGREGATE.  Every signal
                                reaches both children with per-child credits.  out.v0 = child A's
                                int64 sums, out.v1 = child B's.  i32 elements, signal strategy. */
} rs_node_kind;

/* Operations.  The paper leaves isGood() and the aggregate open (P:529,
 * P:532-534); the built-in set is DESIGN.md reading A13/A14/A16/A19. */
typedef enum {
    RS_OP_NONE = 0,          /* ENUMERATE                                                  */
    /* FILTER ops */
    RS_OP_HASH_LT = 1,       /* keep iff ((uint32)v * p0) >> 24 < p1;  p0 odd, p1 in 0..256 */
    RS_OP_LT_U32 = 2,        /* keep iff (uint32)v < p1;               p1 in 0..2^32       */
    RS_OP_CLASS = 3,         /* keep iff bit v of the 32-byte bitmap `table` is set (u8)   */
    RS_OP_PARENT_LT = 4,     /* keep iff (uint32)v < d_parent_ctx[region]: the node reads its
                                parent object (getParent, Fig. 5).  Signal
                                strategy only (the context is uniform over an ensemble there,
                                P:464-465); 4-byte elements; rs_pipeline_run needs d_parent_ctx. */
    /* TRANSFORM ops */
    RS_OP_SCALE_F32 = 10,    /* v = p0_as_float * v, fp32 round-to-nearest, no FMA (f32)   */
    RS_OP_AFFINE_I32 = 11,   /* v = (uint32)(v * p0 + p1)  (i32 / u32)                     */
    /* AGGREGATE ops (output arrays in rs_aggregates, one entry per region)   */
    RS_OP_SUM_I64 = 20,      /* elem i32: v0 = int64 sum                                    */
    RS_OP_SUM_F32 = 21,      /* elem f32: v0 = float sum (fp32 accumulation)               */
    RS_OP_COUNT_MIN_U32 = 22,/* elem u32: v0 = uint32 count, v1 = uint32 min (0xFFFFFFFF if none) */
    RS_OP_COUNT_XOR64 = 23,  /* elem u8 : v0 = uint64 count, v1 = uint64 xor of mix64(i<<8|byte) */
    RS_OP_SUM_I64_DROPS = 27,/* elem i32: v0 = int64 sum (as SUM_I64), v1 = uint64 number of items
                                the FIRST stage dropped in the region.  The first stage counts them
                                and announces the count with a signal of its own just before End
                                ("a node ... may also generate additional signals");
                                later stages forward it in stream position with the credit
                                protocol and the aggregate records it.  Signal strategy; the first
                                stage must not be the fused aggregate (2+ stages, or RS_FLAG_UNFUSED). */
    /* EMIT ops */
    RS_OP_EMIT_VALUE = 24,   /* elem i32/u32/f32: emit (value bits, region id) of each item   */
    RS_OP_EMIT_PAIR = 25     /* elem u8 (taxi stage 2): each surviving byte that
                                starts a well-formed "{x,y}" inside its line (open brace, 1-9
                                digits, comma, 1-9 digits, close brace) is parsed, swapped and
                                emitted as (y, x, line): d_values holds 2 uint32 per pair */
} rs_op;

typedef enum { RS_I32 = 0, RS_U32 = 1, RS_U8 = 2, RS_F32 = 3 } rs_dtype;

typedef enum {
    RS_STRATEGY_SIGNAL = 0,  /* Begin/End signals with credits (§3, §4.2)  */
    RS_STRATEGY_TAGGED = 1,  /* per-item region tags          */
    RS_STRATEGY_CONTEXT = 3, /* per-lane context (§8 f2): one boundary signal {key,
                                stamp} per region, ensembles run across boundaries, every lane
                                computes its own region; no tags in the queues.  4-byte
                                elements, sequential scheduler (signal_cap 0 = 32; a fuller
                                boundary queue cuts ensembles, reading R3). */
    RS_STRATEGY_HYBRID = 4,  /* per-stage strategy (§8 f1): signals up to
                                cfg.tag_from, per-item tags from there on -- the paper's best
                                taxi variant (signal stage 1, tags in stage 2).  SUM_I64 (i32) and
                                EMIT_PAIR (u8) pipelines; bit-identical results. */
    RS_STRATEGY_AUTO = 2     /* choice made per run, transparently (§8 f1):
                                signal when the call's mean region length
                                (d_offsets[n_regions] - d_offsets[0]) / n_regions is at least
                                cfg.auto_min_len, else tagged.  Decided on the device by the
                                prepass (no host synchronisation): both strategies' kernels are
                                enqueued and the one not chosen exits at once.  Both strategies
                                give bit-identical integer aggregates, so the choice only
                                moves time.  rs_pipeline_last_strategy reports it. */
} rs_strategy;

typedef struct {
    int32_t kind;            /* rs_node_kind                                         */
    int32_t op;              /* rs_op                                                */
    uint64_t p0, p1;         /* op parameters (see rs_op)                            */
    const uint8_t *table;    /* host pointer, 32 bytes, RS_OP_CLASS only; copied at create */
} rs_node;

enum {
    RS_FLAG_STATS = 1u,      /* collect per-node occupancy counters (default on)     */
    RS_FLAG_VALIDATE = 2u,   /* device-check offsets monotone and <= n_elems          */
    RS_FLAG_TIMING = 4u,     /* record CUDA events around each kernel of a run        */
    RS_FLAG_PROFILE = 16u,   /* per-node clock64() cycle counters (rs_pipeline_profile); like
                                RS_FLAG_TRACE a debug instantiation (SUM_I64, signal strategy) */
    RS_FLAG_RESERVED8 = 8u,  /* round 1's warp-specialised scheduler (removed: slower than the
                                sequential one); create rejects it with RS_ERR_UNSUPPORTED */
    RS_FLAG_TRACE = 64u,     /* §8(c) trace mode (SUM_I64, signal strategy only; needs
                                rs_pipeline_set_trace): every node logs the Begin/End signals
                                it consumes and each ensemble it fires (count, smallest and
                                largest item value), in order, so a host checker can verify
                                bracketing, unmixed ensembles and per-bracket counts.  A
                                separate kernel instantiation: no cost when off. */
    RS_FLAG_SHORT_OFF = 128u,/* never use the short-region kernel (see RS_FLAG_SHORT_ON)  */
    RS_FLAG_SHORT_ON = 256u, /* signal strategy, SUM_I64 or COUNT_MIN_U32, fused aggregate, 1+ stages: always run
                                the short-region kernel.  It fires the same ensembles and
                                consumes the same signals in the same order as the general
                                kernel (identical results and counters) but handles up to 32
                                pending signals per node warp-parallel (one load, one store)
                                with the partial ensembles they bound in between -- the regime of
                                regions shorter than w.  Default (neither flag):
                                when n_elems < 2w * n_regions both kernels are enqueued and the
                                prepass picks the short-region one iff the call's children
                                off[R] - off[0] < 96 * R, or < 176 * R when 64 sampled region
                                lengths are within 1/8 of the mean (decided on the device, like
                                AUTO; the crossovers measured on B200).  Its default geometry is its
                                own (a 16w ring, stages of 4w, signal queues of 128) unless
                                queue_cap / signal_cap / q0_stage are set. */
    RS_FLAG_UNFUSED = 32u    /* sequential scheduler: keep the AGGREGATE as a separate node
                                with its own queue (the paper's node structure).
                                Default: the aggregate is folded into the last FILTER/
                                TRANSFORM node, which adds its surviving items straight into
                                the per-region accumulator (same results; the AGGREGATE's
                                stats then report that node's firings).  No effect without
                                stages. */
};

typedef struct {
    int32_t strategy;        /* rs_strategy                                          */
    uint32_t simd_width;     /* ensemble capacity w in items; only 128 is built */
    uint32_t queue_cap;      /* data queue capacity (items, power of 2 in [2w, 65536]).  4-byte elements,
                                sequential scheduler: all queues share ONE in-place ring of
                                max(4*q0_stage, min(queue_cap, 8*q0_stage)) items, raised to fit one
                                partial ensemble per queue plus a stage (0 = auto: 32w signal, 16w
                                tagged, 8w tagged with 0-1 stages).  u8 elements: capacity of each inter-stage queue
                                (0 = auto: 8w with 2+ stages, else 16w). */
    uint32_t signal_cap;     /* signal queue capacity (entries, power of 2, >= 4; 0 = auto) */
    int32_t grid;            /* persistent CTAs; 0 = fill the device                  */
    uint32_t chunk;          /* children per parent-stream claim (power of 2); 0 = auto: 32768 for
                                4-byte signal / context pipelines, else 8192; with auto on those
                                4-byte signal / context pipelines the part of the stream left after
                                whole rounds of chunks
                                over all instances is claimed in pieces of chunk/8 (no ragged last
                                round; the prepass decides from the call's children) */
    uint32_t flags;          /* RS_FLAG_*                                            */
    uint32_t q0_stage;       /* elements per TMA stage of the enumerate queue (the ring holds 4..8
                                stages); power of 2 in [128, 4096], <= chunk; 0 = auto (in-place
                                rings: 1024 signal, 512 tagged, 256 tagged with 0-1 stages;
                                otherwise 256 tagged or 2+ stages, else 2048) */
    uint32_t auto_min_len;   /* RS_STRATEGY_AUTO: mean children per region at and above which the
                                signal strategy runs; 0 = the crossover measured on B200 for the
                                pipeline's stage count */
    uint32_t tag_from;       /* RS_STRATEGY_HYBRID: the first edge that carries tags (edge e joins
                                node e to node e+1; edge 0 leaves ENUMERATE).  Edges before it are
                                signal-delimited, node tag_from converts (consumes Begin/End, tags
                                its outputs with the open region).  1 .. (stages - 1) with the
                                fused aggregate, 1 .. stages with RS_FLAG_UNFUSED. */
} rs_config;

/* Per-node occupancy counters (§2.2, §5).  Node 0 is the
 * enumerate node: items = children enumerated, signal_firings = signals
 * emitted.  For the other nodes: data_firings = ensembles run,
 * full_firings = ensembles of exactly w items, items = items consumed,
 * signal_firings = signals consumed.  Lane fraction = items/(w*data_firings). */
typedef struct {
    uint64_t data_firings, full_firings, items, signal_firings;
} rs_node_stats;

/* Caller-owned per-region outputs (layout per aggregate op above). */
typedef struct { void *v0; void *v1; } rs_aggregates;

typedef struct rs_pipeline rs_pipeline;

/* Fill `cfg` with defaults (signal strategy, w = 128, stats on). */
rs_status rs_config_default(rs_config *cfg);

/* Build a pipeline from a node list (BASELINE north star: "create pipeline
 * from a node list").  The list must be ENUMERATE, then 0..4 FILTER/TRANSFORM
 * nodes, then one AGGREGATE or EMIT (single-level enumeration) -- or, for a
 * tree, ENUMERATE, 0..2 stages, SPLIT and its two AGGREGATE leaves.  `elem` is the
 * element type of the parents' payload.  Errors: RS_ERR_INVALID_TOPOLOGY,
 * RS_ERR_UNSUPPORTED (op/dtype mismatch, w != 128, capacities), RS_ERR_INVALID_ARG. */
rs_status rs_pipeline_create(const rs_node *nodes, int n_nodes, rs_dtype elem,
                             const rs_config *cfg, rs_pipeline **out);

/* Device workspace needed by rs_pipeline_run for up to `n_regions` regions
 * over an element array of `n_elems` elements.  Any 256-byte aligned device
 * buffer of at least this size may be passed; it is overwritten by every run. */
rs_status rs_pipeline_workspace_bytes(const rs_pipeline *p, int64_t n_regions, int64_t n_elems,
                                      size_t *bytes);

/* Run the pipeline over regions j = 0..n_regions-1, where region j owns
 * d_elems[d_offsets[j] .. d_offsets[j+1]) (CSR, int64, non-decreasing, n_regions+1
 * entries, d_offsets[0] may be > 0 so a batch or shard can address a slice of a
 * larger stream).  Empty regions are legal.  Writes exactly one
 * aggregate per region into out.v0[j] (and out.v1[j]) (A2).
 *   d_elems       device, 16-byte aligned, n_elems elements of the create-time dtype;
 *                 d_offsets[n_regions] <= n_elems is required (checked on device only
 *                 with RS_FLAG_VALIDATE).  May be NULL when n_elems == 0.
 *   n_regions     0 .. 2^31-1.
 *   d_parent_ctx  device uint32[n_regions], the parent objects' context read by
 *                 RS_OP_PARENT_LT nodes (indexed like the outputs); NULL when the
 *                 pipeline has no such node (RS_ERR_INVALID_ARG if it has one).
 *   out           device arrays of n_regions entries; they may be peer-mapped
 *                 memory of another GPU (rs_ipc_open): the kernels then store the
 *                 aggregates straight into that GPU's buffer over NVLink.
 *   d_ws          workspace of >= rs_pipeline_workspace_bytes(p, n_regions, n_elems).
 * Asynchronous on `stream`. */
rs_status rs_pipeline_run(rs_pipeline *p, const void *d_elems, int64_t n_elems,
                          const int64_t *d_offsets, int64_t n_regions, const void *d_parent_ctx,
                          rs_aggregates out, void *d_ws, size_t ws_bytes, rs_stream stream);

/* Element-wise exit (a pipeline whose last node is RS_NODE_EMIT): like
 * rs_pipeline_run, but instead of per-region aggregates every item that
 * survives the stages is written as d_values[k] (its 32-bit value) and
 * d_regions[k] (its region j) for distinct k < *d_count.  The
 * order of the pairs is unspecified (instances write their ensembles as they
 * finish; within an ensemble stream order is kept).  *d_count is zeroed and
 * then set to the number of surviving items; when it exceeds `capacity` only
 * `capacity` pairs were written and rs_pipeline_check reports code 8.
 * rs_pipeline_run rejects EMIT pipelines and vice versa. */
rs_status rs_pipeline_run_emit(rs_pipeline *p, const void *d_elems, int64_t n_elems,
                               const int64_t *d_offsets, int64_t n_regions, const void *d_parent_ctx,
                               uint32_t *d_values, uint32_t *d_regions, uint64_t capacity, uint64_t *d_count,
                               void *d_ws, size_t ws_bytes, rs_stream stream);

/* End-to-end convenience: same as rs_pipeline_run but with HOST buffers.
 * Copies elements, offsets (and parent contexts) host->device (pinned host memory gives
 * asynchronous copies), runs, and copies the aggregates back into h_out;
 * device buffers are owned by the handle and grown on demand.  Synchronises
 * `stream` before returning. */
rs_status rs_pipeline_run_host(rs_pipeline *p, const void *h_elems, int64_t n_elems,
                               const int64_t *h_offsets, int64_t n_regions, const void *h_parent_ctx,
                               rs_aggregates h_out, rs_stream stream);

/* Copy the per-node counters of the last run into host_out[0..n_nodes-1]
 * (n_nodes = the create-time node count).  Synchronises `stream`. */
rs_status rs_pipeline_stats(rs_pipeline *p, rs_node_stats *host_out, int n_nodes, rs_stream stream);

/* Per-node cycle counters of the last run made with RS_FLAG_PROFILE (sequential
 * mode; synchronises `stream`): host16[0] = enumerate, host16[1..K+1] = nodes,
 * host16[K+2] = waiting on TMA, [8] = scheduler sweeps, [9] = waits,
 * [10] = instances; cycles are summed over instances. */
rs_status rs_pipeline_profile(rs_pipeline *p, uint64_t *host16, rs_stream stream);

/* Read the device error word of the last run (synchronises `stream`).
 * Returns RS_ERR_PROTOCOL and sets *code (if non-NULL) when the device saw a
 * violated invariant: 1 = bad offsets (VALIDATE), 2 = watchdog (no progress),
 * 3 = signal queue overflow, 4 = unmatched End, 5 = queue overflow,
 * 7 = a receiver's readable limit fell behind its consumed position,
 * 8 = RS_NODE_EMIT output capacity exceeded. */
rs_status rs_pipeline_check(rs_pipeline *p, rs_stream stream, int32_t *code);

/* Device time of the last run's kernels (needs RS_FLAG_TIMING; synchronises
 * `stream`): ms[0] = prepass, ms[1] = persistent pipeline kernel, ms[2] = fixup. */
rs_status rs_pipeline_kernel_times(rs_pipeline *p, float *ms3, rs_stream stream);

/* Number of kernel launches the last rs_pipeline_run enqueued (4 when AUTO or the short-region
 * choice enqueued two main kernels, one of which exits at once). */
int rs_pipeline_launches(const rs_pipeline *p);

/* Persistent CTAs and warps (pipeline instances) per CTA of the last run's general kernel (the
 * short-region kernel, RS_FLAG_SHORT_ON, sizes its own launch from its own geometry). */
rs_status rs_pipeline_geometry(const rs_pipeline *p, int32_t *grid, int32_t *warps_per_cta,
                               int32_t *chunk);

/* Strategy the last run used (RS_STRATEGY_SIGNAL or RS_STRATEGY_TAGGED; for an
 * AUTO pipeline that has not run yet, RS_STRATEGY_AUTO).  For an AUTO pipeline
 * this reads the device's decision and synchronises the last run's stream. */
rs_status rs_pipeline_last_strategy(const rs_pipeline *p, int32_t *strategy);

/* Trace buffer for RS_FLAG_TRACE runs (Lemma 1, §3.3;
 * SURVEY §8(c) "GPU trace-mode check").  d_trace: caller-owned device buffer
 * of `bytes` (16-byte aligned, >= 64; NULL detaches).  Every traced run first
 * zeroes word 0 and then fills:
 *   word 0        number of events the kernel tried to write (> capacity =
 *                 overflow; capacity = (bytes - 32) / 32)
 *   words 8 + 8i  event i, 8 x uint32: instance (warp) id, per-instance
 *                 sequence number, node | type << 8 (type 1 = ENSEMBLE,
 *                 2 = BEGIN, 3 = END; node 1..K+1, the fused last stage
 *                 logs under its own index), region key (bit 31 = partial
 *                 slot of a region split across chunks), resolved region id
 *                 (BEGIN/END), item count, min item, max item (ENSEMBLE).
 * Events of one instance are in the order the instance performed them. */
rs_status rs_pipeline_set_trace(rs_pipeline *p, void *d_trace, uint64_t bytes);

void rs_pipeline_destroy(rs_pipeline *p);

/* ------------------------------------------------------------- multi-GPU
 * Regions are independent contexts (§1), so a stream partitioned by
 * whole regions (rank k owns regions [base[k], base[k+1]), its run addressing
 * them through d_offsets[base[k] .. base[k+1]]) needs no exchange while it is
 * processed; the per-region aggregates are then assembled on one rank.
 * NCCL is the library torch has loaded (found with dlopen; RS_NCCL_LIB may
 * name another); the current CUDA device is the rank's GPU. */
typedef struct rs_comm rs_comm;

/* 128-byte NCCL unique id, created on one rank and passed to all (the caller
 * distributes it, e.g. with torch.distributed). */
rs_status rs_comm_unique_id(void *id128);

/* Communicator of `world` ranks; this process is `rank`.  Collective. */
rs_status rs_comm_init(const void *id128, int rank, int world, rs_comm **out);

/* Gather: rank k's aggregates `local` (local_regions = region_base[k+1] -
 * region_base[k] entries of the layout of aggregate op `agg_op`) are written to
 * root_out.v*[region_base[k] ...] on rank `root`, at exact offsets (grouped
 * ncclSend/ncclRecv, no padding; the root's own slice is a device copy).
 * region_base: host int64[world+1], identical on all ranks.  root_out is read
 * on the root only.  Stream-ordered on `stream`; collective. */
rs_status rs_gather_aggregates(rs_comm *c, int32_t agg_op, rs_aggregates local, int64_t local_regions,
                               const int64_t *region_base, rs_aggregates root_out, int root, rs_stream stream);

/* Stream-ordered barrier (an all-reduce of one word): work enqueued on
 * `stream` before it on every rank precedes work after it.  Collective. */
rs_status rs_comm_barrier(rs_comm *c, rs_stream stream);

void rs_comm_destroy(rs_comm *c);

/* Peer-memory gather (fused with the aggregate's stores): the root exports
 * its output buffer (64-byte CUDA IPC handle of the allocation holding d_buf,
 * plus d_buf's byte offset in it; the caller passes both to the other ranks),
 * the other ranks map the allocation and pass  mapped + offset + base[k] *
 * bytes  as rs_aggregates to rs_pipeline_run, so the kernels store every
 * region's aggregate into the root's buffer over NVLink as it completes.
 * Completion: stream order + rs_comm_barrier (or a host barrier after a
 * synchronise).  rs_ipc_open maps the allocation base; rs_ipc_close unmaps it. */
rs_status rs_ipc_export(const void *d_buf, void *handle64, uint64_t *offset);
rs_status rs_ipc_open(const void *handle64, void **d_ptr);
rs_status rs_ipc_close(void *d_ptr);

const char *rs_status_string(rs_status s);
const char *rs_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RS_H */
